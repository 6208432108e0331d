"""Reduce ncu CSV pages (prof_<kernel>_raw.csv, prof_<kernel>_source.csv.gz from
scripts/gpu_round.sh) to a committed summary: profiles/ncu_summary.json + a markdown table.

    python scripts/ncu_summary.py gpurun_out/r01g [--out profiles/ncu_summary.json] [--tag r01]
"""
from __future__ import annotations

import argparse
import collections
import csv
import glob
import gzip
import json
import os
import re

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "registers": "launch__registers_per_thread",
    "block": "launch__block_size",
    "grid": "launch__grid_size",
    "dyn_smem_bytes": "launch__shared_mem_per_block_dynamic",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_active": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct_elapsed": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "issue_per_cycle": "smsp__issue_active.avg.per_cycle_active",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "sm_mhz": "sm__cycles_elapsed.avg.per_second",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
         "Ghz": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}


def raw(path):
    rows = list(csv.reader(open(path)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def value(d, name):
    if name not in d:
        return None
    u, v = d[name]
    u = u.split("/")[0]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(u, 1)


def instr_mix(path):
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ops, tot = collections.Counter(), 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ix["Source"]].strip())
        if not m:
            continue
        n = int(r[ix["Instructions Executed"]] or 0)
        ops[m.group(2)] += n
        tot += n
    fp64 = sum(ops[k] for k in ("DADD", "DMUL", "DFMA"))
    return {"warp_instructions": tot, "fp64_share": fp64 / tot if tot else None,
            "top": {k: round(v / tot, 4) for k, v in ops.most_common(8)}}


def summarize(d):
    out = {}
    for k, m in METRICS.items():
        out[k] = value(d, m)
    if out["dram_read"] is not None and out["dram_write"] is not None:
        out["dram_bytes_per_launch"] = out["dram_read"] + out["dram_write"]
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): value(d, h) for h in d
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if isinstance(v, float))
    out["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0))[:8]
                          if tot and isinstance(v, float)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("dir")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    kernels = {}
    for p in sorted(glob.glob(os.path.join(args.dir, "prof_*_raw.csv"))):
        k = os.path.basename(p)[len("prof_"):-len("_raw.csv")]
        s = summarize(raw(p))
        src = os.path.join(args.dir, f"prof_{k}_source.csv.gz")
        if os.path.exists(src):
            s["instruction_mix"] = instr_mix(src)
        kernels[k] = s
    doc = {"tag": args.tag, "source": args.dir, "kernels": kernels}
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
