"""A/B of engine knobs on one B200: the same start range tracked under each setting of one or more
environment knobs; prints per-kernel device time (PP200_KERNEL_TIMING) and checks that every
setting gives bit-identical records (and equals any golden range of tests/golden it covers).

    python scripts/ab.py SYSTEM PREC LO PATHS [max_newton=4] KNOB=v1,v2 [KNOB2=...]
"""
import glob
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_00383_b200 as P  # noqa: E402

system, prec, lo, paths = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cfg_over = dict(kv.split("=") for kv in sys.argv[5:] if not kv.startswith("PP200_"))
knobs = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in sys.argv[5:] if kv.startswith("PP200_")]
sysfile = os.path.join(ROOT, "tests", "data", f"{system}.sys")
f = P.parse_system(open(sysfile).read()) if os.path.exists(sysfile) else P.cyclic_system(int(system[6:]))
g, st = P.total_degree_start(f, prec)
h = P.make_homotopy(f, g, P.random_gamma(1), prec)
cfg = P.TrackConfig.defaults(prec)
for k, v in cfg_over.items():
    setattr(cfg, k, type(getattr(cfg, k))(v))
KEYS = ["status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]
golds = []
for gp in glob.glob(os.path.join(ROOT, "tests", "golden", f"track_{system}_{prec}*.npz")):
    z = np.load(gp)
    if "lo" in z.files and int(z["gamma_seed"]) == 1 and eval(str(z["cfg"])) == {k: type(getattr(cfg, k))(v) for k, v in cfg_over.items()}:
        if lo <= int(z["lo"]) and int(z["hi"]) <= lo + paths:
            golds.append((os.path.basename(gp), z))


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


ref = None
# per-kernel times need the instrumented engine (one launch per kernel and trip, synchronised);
# AB_TIMING=0 times the production engine (CUDA graphs) as a whole instead
os.environ["PP200_KERNEL_TIMING"] = os.environ.get("AB_TIMING", "1")
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), v in zip(knobs, combo):
        os.environ[k] = v
    sol = P.track_all(h, st, cfg, lo=lo, hi=lo + paths)
    s = sol.stats
    same = None if ref is None else all(np.array_equal(bits(getattr(sol, k)), bits(getattr(ref, k))) for k in KEYS)
    ref = ref or sol
    gok = {name: all(np.array_equal(bits(getattr(sol, k)[int(z["lo"]) - lo:int(z["hi"]) - lo]), bits(z[k])) for k in KEYS)
           for name, z in golds}
    print(f"{dict(zip([k for k, _ in knobs], combo))} {system} {prec} {paths}: device {s['device_ms']:.1f} ms "
          f"eval {s['eval_ms']:.1f} lsq {s['lsq_ms']:.1f} step {s['step_ms']:.1f} fused {s.get('fused_ms', 0):.1f} "
          f"trips {s['total_rounds']} "
          f"-> {paths / (s['device_ms'] / 1e3):.1f} paths/s; same-as-first {same} golden {gok}", flush=True)
