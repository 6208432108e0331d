"""Experiment: the same start range tracked by one track_all call, or split across K host threads
each calling track_all concurrently (own stream, own workspace).  Wall times only."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1505_00383_b200 as P  # noqa: E402

paths = int(os.environ.get("PATHS", "262144"))
offset = int(os.environ.get("OFFSET", "1000000"))
K = int(os.environ.get("K", "2"))
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
f = P.parse_system(open(os.path.join(root, "tests", "data", "cyclic10.sys")).read())
g, st = P.total_degree_start(f, "dd")
h = P.make_homotopy(f, g, P.random_gamma(1), "dd")
cfg = P.TrackConfig.defaults("dd")
P.track_all(h, st, cfg, lo=offset, hi=offset + 4096)  # warm-up
t0 = time.time()
one = P.track_all(h, st, cfg, lo=offset, hi=offset + paths)
t1 = time.time()
res = [None] * K


def work(i):
    lo = offset + paths * i // K
    hi = offset + paths * (i + 1) // K
    res[i] = P.track_all(h, st, cfg, lo=lo, hi=hi)


ths = [threading.Thread(target=work, args=(i,)) for i in range(K)]
t2 = time.time()
for t in ths:
    t.start()
for t in ths:
    t.join()
t3 = time.time()
import numpy as np  # noqa: E402

same = all(np.array_equal(np.concatenate([getattr(r, k) for r in res]), getattr(one, k))
           for k in ("status", "x", "newton_iters"))
print(f"one call: {t1 - t0:.2f}s ({paths / (t1 - t0):.0f} paths/s); {K} concurrent calls: {t3 - t2:.2f}s "
      f"({paths / (t3 - t2):.0f} paths/s); records identical: {same}", flush=True)
