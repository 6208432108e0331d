import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1505_00383_b200 as P
for init in (False, True):
    if init:
        t = time.perf_counter(); P.device_init(0); print(f"device_init {1e3*(time.perf_counter()-t):.1f} ms")
    for prec in ("d", "dd"):
        f = P.parse_system(open("tests/data/cyclic5.sys").read())
        g, st = P.total_degree_start(f, prec)
        h = P.make_homotopy(f, g, P.random_gamma(1), prec)
        cfg = P.TrackConfig.defaults(prec)
        for rep in range(3):
            t = time.perf_counter(); sol = P.track_all(h, st, cfg, lo=0, hi=120); w = time.perf_counter() - t
            print(f"init={init} {prec} rep {rep}: wall {1e3*w:.1f} ms device {sol.stats['device_ms']:.1f} ms", flush=True)
