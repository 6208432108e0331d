"""A/B of engine knobs on one B200: runs the same cyclic-10 range under each setting of an
environment knob, reports per-kernel device time (PP200_KERNEL_TIMING) and checks that every
setting produces bitwise identical records, and that they equal the reference golden range.

    python scripts/lsq_experiment.py PREC PATHS KNOB=v1,v2,... [KNOB2=...]
"""
import itertools
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1505_00383_b200 as P  # noqa: E402

prec = sys.argv[1]
paths = int(sys.argv[2])
knobs = [(kv.split("=")[0], kv.split("=")[1].split(",")) for kv in sys.argv[3:]]
lo = 1_000_000 - paths // 2
f = P.parse_system(open(os.path.join(ROOT, "tests", "data", "cyclic10.sys")).read())
g, st = P.total_degree_start(f, prec)
h = P.make_homotopy(f, g, P.random_gamma(1), prec)
cfg = P.TrackConfig.defaults(prec)
gold = None
gp = os.path.join(ROOT, "tests", "golden", f"track_cyclic10_{prec}_far.npz")
if os.path.exists(gp):
    gold = np.load(gp)
KEYS = ["status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]
ref = None
os.environ["PP200_KERNEL_TIMING"] = "1"
for combo in itertools.product(*[v for _, v in knobs]):
    for (k, _), v in zip(knobs, combo):
        os.environ[k] = v
    sol = P.track_all(h, st, cfg, lo=lo, hi=lo + paths)
    s = sol.stats
    same = None
    if ref is None:
        ref = sol
    else:
        same = all(np.array_equal(getattr(sol, k), getattr(ref, k)) for k in KEYS)
    gok = None
    if gold is not None and lo <= int(gold["lo"]) and int(gold["hi"]) <= lo + paths:
        a, b = int(gold["lo"]) - lo, int(gold["hi"]) - lo
        gok = all(np.array_equal(getattr(sol, k)[a:b], gold[k]) for k in KEYS)
    print(f"{dict(zip([k for k, _ in knobs], combo))} {prec} {paths}: device {s['device_ms']:.1f} ms "
          f"eval {s['eval_ms']:.1f} lsq {s['lsq_ms']:.1f} step {s['step_ms']:.1f} slots {s['slots']} "
          f"solves {s['solves']} -> {paths / (s['device_ms'] / 1e3):.0f} paths/s; "
          f"same-as-first {same} golden {gok}", flush=True)
