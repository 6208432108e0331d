"""Throughput and sampled parity on every BASELINE.json config (GPU box; developer tool).

For each config: the CUDA tracker runs the whole path range (or the stated slice) through the
public API and is timed on the device; the reference CPU tracker (oracle/_ref, the unmodified
polypath build) runs a time-bounded sample of paths spread over that range on all host threads,
and the sampled records are compared bit for bit with the GPU's.  One JSON line per config.

    python scripts/measure_configs.py [--only NAME ...] [--cpu-budget SECONDS] > configs.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402  (test infrastructure: the checker and the CPU baseline only)
import paper_1505_00383_b200 as P  # noqa: E402

KEYS = ["status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]

# name, system, precision, TrackConfig overrides, [lo, hi)
CONFIGS = [
    ("cyclic5_d", "cyclic5", "d", {}, 0, 120),
    ("cyclic5_dd", "cyclic5", "dd", {}, 0, 120),
    ("cyclic5_qd", "cyclic5", "qd", {}, 0, 120),
    ("cyclic8_d", "cyclic8", "d", {}, 0, 40320),
    ("cyclic8_dd", "cyclic8", "dd", {}, 0, 40320),
    ("cyclic10_d", "cyclic10", "d", {}, 1_000_000, 1_262_144),
    ("cyclic10_dd", "cyclic10", "dd", {}, 1_000_000, 1_262_144),
    ("katsura12_qd", "katsura12", "qd", {"max_newton": 4}, 0, 4096),
    ("rand32_d", "rand32", "d", {}, 0, 65536),
    ("rand32_dd", "rand32", "dd", {}, 0, 65536),
    ("rand32_qd", "rand32", "qd", {}, 0, 4096),
]


def system_text(name: str) -> str:
    if name == "cyclic8":
        return P.cyclic_system(8).text()
    with open(os.path.join(ROOT, "tests", "data", name + ".sys")) as fh:
        return fh.read()


def cpu_sample(text, prec, cfg, lo, hi, budget, threads):
    """each thread tracks consecutive paths of its own group (groups spread over [lo, hi)) with
    single-worker reference track_all calls until the time budget is spent"""
    gam = O.ref_random_gamma(1)
    span = hi - lo
    groups = [lo + (span * i) // threads for i in range(threads)]
    results = [[] for _ in range(threads)]
    t_end = time.perf_counter() + budget

    def work(i):
        p = groups[i]
        limit = lo + (span * (i + 1)) // threads
        chunk = 1
        while p < limit and time.perf_counter() < t_end:
            q = min(limit, p + chunk)
            t0 = time.perf_counter()
            r = O.ref_track(text, prec, gam, cfg=cfg, lo=p, hi=q, workers=1, batch=64)
            results[i].append(r)
            if time.perf_counter() - t0 < 0.05:
                chunk = min(chunk * 2, 256)
            p = q

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    recs = [r for rs in results for r in rs]
    merged = {k: np.concatenate([r[k] for r in recs]) for k in ["path_id"] + KEYS} if recs else None
    n = 0 if merged is None else len(merged["path_id"])
    return merged, n, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--cpu-budget", type=float, default=8.0)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    peak = P.fp64_peak(0)
    for name, system, prec, over, lo, hi in CONFIGS:
        if args.only and name not in args.only:
            continue
        text = system_text(system)
        f = P.parse_system(text)
        g, starts = P.total_degree_start(f, prec)
        h = P.make_homotopy(f, g, P.random_gamma(1), prec)
        cfg = P.TrackConfig.defaults(prec)
        for k, v in over.items():
            setattr(cfg, k, v)
        hi = min(hi, starts.count)
        t0 = time.perf_counter()
        sol = P.track_all(h, starts, cfg, lo=lo, hi=hi)
        wall = time.perf_counter() - t0
        st = sol.stats
        from paper_1505_00383_b200 import work as W

        wk = W.path_work(h.info, prec, st["evals"], st["solves"])
        line = {"config": name, "system": system, "prec": prec, "overrides": over, "range": [lo, hi],
                "paths": len(sol), "bezout": starts.count, "gpu_device_s": st["device_ms"] / 1e3, "gpu_wall_s": wall,
                "gpu_paths_per_s": len(sol) / (st["device_ms"] / 1e3), "e2e_paths_per_s": len(sol) / wall,
                "fp64_ops": wk["total_ops"], "fp64_tops": wk["total_ops"] / (st["device_ms"] / 1e3) / 1e12,
                "fp64_frac_of_measured_peak": wk["total_ops"] / (st["device_ms"] / 1e3) / peak,
                "counts": sol.counts(), "trips": st["total_rounds"], "slots": st["slots"]}
        if O.ref is not None and args.cpu_budget > 0:
            rec, n, cwall = cpu_sample(text, prec, over, lo, hi, args.cpu_budget, args.threads)
            line["cpu_paths_per_s"] = n / cwall
            line["cpu_sample"] = f"{n} paths, {args.threads} threads x single-worker reference track_all, {cwall:.1f} s"
            line["speedup_device_vs_cpu"] = line["gpu_paths_per_s"] / max(1e-12, line["cpu_paths_per_s"])
            if n:
                idx = (rec["path_id"] - lo).astype(np.int64)
                bad = 0
                for k in KEYS:
                    a = np.ascontiguousarray(np.asarray(getattr(sol, k))[idx]).reshape(n, -1)
                    b = np.ascontiguousarray(rec[k]).reshape(n, -1)
                    if a.dtype == np.float64:  # bit patterns: -0.0 differs from 0.0
                        a, b = a.view(np.uint64), b.view(np.uint64)
                    bad = max(bad, int(np.sum(np.any(a != b, axis=1))))
                line["sampled_parity"] = {"paths": n, "records_differing": bad}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
