"""Developer check on a GPU box: bitwise parity of the CUDA tracker against the reference build
(oracle/_ref) on small configs, then a throughput probe.  Not part of the test suite."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O
import paper_1505_00383_b200 as P

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests", "data")


def compare(name, r, m):
    keys = ["status", "reason", "steps", "newton_iters", "rejections"]
    res = {k: bool(np.array_equal(r[k], getattr(m, k))) for k in keys}
    res["x"] = bool(np.array_equal(r["x"], m.x))
    res["residual"] = bool(np.array_equal(r["residual"], m.residual))
    nbad = int(np.sum(np.any(r["x"].reshape(len(m), -1) != m.x.reshape(len(m), -1), axis=1)))
    print(name, "bitwise:", res, "paths differing:", nbad, "counts:", m.counts(), flush=True)
    if nbad:
        i = int(np.argmax(np.any(r["x"].reshape(len(m), -1) != m.x.reshape(len(m), -1), axis=1)))
        print("  first diff path", i, {k: (r[k][i], getattr(m, k)[i]) for k in keys})


def run(sysfile, prec, lo, hi, ref=True, workers=8):
    text = open(os.path.join(DATA, sysfile)).read()
    f = P.parse_system(text)
    g, st = P.total_degree_start(f, prec)
    gam = P.random_gamma(1)
    h = P.make_homotopy(f, g, gam, prec)
    cfg = P.TrackConfig.defaults(prec)
    t0 = time.time()
    m = P.track_all(h, st, cfg, lo=lo, hi=hi)
    t1 = time.time()
    s = m.stats
    print(f"{sysfile} {prec} [{lo},{hi}): gpu wall {t1-t0:.3f}s device {s['device_ms']:.1f}ms trips {s['total_rounds']} "
          f"slots {s['slots']} -> {(hi-lo)/(s['device_ms']/1e3):.1f} paths/s (device)", flush=True)
    if ref:
        t0 = time.time()
        r = O.ref_track(text, prec, gam, lo=lo, hi=hi, workers=workers, batch=max(64, 4 * 128 * workers))
        print(f"  ref wall {time.time()-t0:.2f}s ({(hi-lo)/(r['wall_ms']/1e3):.2f} paths/s)")
        compare(f"  {sysfile} {prec}", r, m)
    return m


if __name__ == "__main__":
    run("cyclic5.sys", "d", 0, 120)
    run("cyclic5.sys", "dd", 0, 120)
    run("cyclic5.sys", "qd", 0, 8)
    run("cyclic10.sys", "d", 0, 1024)
    run("cyclic10.sys", "dd", 0, 128)
    for n in [4096, 32768, 131072]:
        run("cyclic10.sys", "dd", 0, n, ref=False)
