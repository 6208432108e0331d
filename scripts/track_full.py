"""The north-star job: every total-degree start path of cyclic 10-roots (3,628,800 paths) tracked to
t = 1 in complex double-double on this GPU (or on one shard of [0, 3628800) per rank under
torchrun: block-cyclic shards, blocks of 64), with the classification counts and the number of distinct converged endpoints.
cyclic-10 has 34,940 isolated solutions, which a complete run should find.

    python scripts/track_full.py [--lo 0 --hi 3628800] [--chunk 3628800]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_00383_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="dd")
    ap.add_argument("--lo", type=int, default=0)
    ap.add_argument("--hi", type=int, default=3628800)
    ap.add_argument("--chunk", type=int, default=3628800, help="paths per track_all call")
    ap.add_argument("--out", default=None, help="write the converged endpoints (complex128) as .npy")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    device = int(os.environ.get("LOCAL_RANK", "0"))
    # this rank's block-cyclic shard of [lo, hi) (pp_shard; blocks of 64 start indices)
    lo, hi = args.lo, args.hi
    shard = (rank, world, 64) if world > 1 else None

    f = P.parse_system(open(os.path.join(ROOT, "tests", "data", "cyclic10.sys")).read())
    g, st = P.total_degree_start(f, args.prec)
    h = P.make_homotopy(f, g, P.random_gamma(1), args.prec)
    cfg = P.TrackConfig.defaults(args.prec)
    counts = {}
    ends = []
    dev_s = 0.0
    n_paths = 0
    t0 = time.time()
    for a in range(lo, hi, args.chunk):
        b = min(hi, a + args.chunk)
        sol = P.track_all(h, st, cfg, lo=a, hi=b, device=device, shard=shard)
        dev_s += sol.stats["device_ms"] / 1e3
        n_paths += len(sol)
        for k, v in sol.counts().items():
            counts[k] = counts.get(k, 0) + v
        ends.append(sol.x_complex()[sol.status == P.SUCCESS])
        print(f"rank {rank}: [{a}, {b}) done, {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    wall = time.time() - t0
    x = np.concatenate(ends) if ends else np.zeros((0, f.dim), complex)
    # distinct endpoints: round to 1e-6 (converged residuals are below 1e-14 in dd)
    key = np.round(np.concatenate([x.real, x.imag], axis=1) * 1e6).astype(np.int64)
    distinct = len(np.unique(key, axis=0)) if len(key) else 0
    if args.out:
        np.save(args.out, x)
    print(json.dumps({"rank": rank, "world": world, "range": [lo, hi], "shard": shard, "paths": n_paths, "counts": counts,
                      "converged": counts.get("converged", 0), "distinct_converged_endpoints": distinct,
                      "device_s": dev_s, "wall_s": wall, "paths_per_s_device": n_paths / dev_s if dev_s else None,
                      "paths_per_s_wall": n_paths / wall}), flush=True)


if __name__ == "__main__":
    main()
