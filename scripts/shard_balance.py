"""Load balance of an N-GPU partition measured on one GPU: the full cyclic-10 job (3,628,800 paths)
split into N shards, each shard tracked on its own (sequentially, on this GPU), once with
contiguous slices (the reference CLI's --path-range partition) and once with block-cyclic shards
(pp_shard, blocks of 64).  An N-GPU run finishes when its slowest shard does, so max/mean shard
time is the scaling efficiency the partition allows.

    python scripts/shard_balance.py [--prec dd] [--world 8] [--hi 3628800] > shard_balance.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_00383_b200 as P  # noqa: E402
from paper_1505_00383_b200.shard import contiguous_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="dd")
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--lo", type=int, default=0)
    ap.add_argument("--hi", type=int, default=3628800)
    ap.add_argument("--block", type=int, default=64)
    ap.add_argument("--schemes", default="contiguous,block_cyclic")
    args = ap.parse_args()
    f = P.parse_system(open(os.path.join(ROOT, "tests", "data", "cyclic10.sys")).read())
    g, st = P.total_degree_start(f, args.prec)
    h = P.make_homotopy(f, g, P.random_gamma(1), args.prec)
    cfg = P.TrackConfig.defaults(args.prec)
    out = {"system": "cyclic10", "prec": args.prec, "world": args.world, "range": [args.lo, args.hi],
           "block": args.block, "schemes": {}}
    for scheme in args.schemes.split(","):
        shards = []
        for r in range(args.world):
            if scheme == "contiguous":
                a, b = contiguous_range(args.lo, args.hi, r, args.world)
                sol = P.track_all(h, st, cfg, lo=a, hi=b)
            else:
                sol = P.track_all(h, st, cfg, lo=args.lo, hi=args.hi, shard=(r, args.world, args.block))
            s = sol.stats
            shards.append({"shard": r, "paths": len(sol), "device_s": s["device_ms"] / 1e3,
                           "newton_iters": int(s["newton_iters"]), "converged": int((sol.status == P.SUCCESS).sum())})
            print(f"{scheme} shard {r}: {shards[-1]}", file=sys.stderr, flush=True)
        t = [x["device_s"] for x in shards]
        mean = sum(t) / len(t)
        out["schemes"][scheme] = {"shards": shards, "max_s": max(t), "mean_s": mean, "max_over_mean": max(t) / mean,
                                  "efficiency": mean / max(t), "sum_s": sum(t)}
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
