"""bench.py -- paths/sec to t = 1 of the total-degree homotopy of cyclic 10-roots in complex
double-double on 1..8 B200 (BASELINE.json metric), against the reference CPU tracker.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--paths B]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

A step tracks B (default 393,216) start paths per GPU of the 3,628,800-path total-degree start set to their terminal
status (success / failed / diverged after finalize).  Step s takes a contiguous chunk of N*B start
indices, spread over the index space by a golden-ratio sequence, and rank r tracks the block-cyclic
shard r of it (blocks of 64 indices, pp_shard), so N GPUs do N times the work (weak scaling) with
no data-path collective; the only torch.distributed traffic is the barrier and the
max-over-ranks timing.  `--gpus N` without torchrun launches the N ranks itself (one per GPU;
ranks share a GPU round-robin, over gloo, when the box has fewer).

Before the timed steps every rank checks its GPU once at the bench's size: a full-occupancy call
over the 262,144 paths of tests/golden/track_cyclic10_dd_prod.npz must reproduce the reference
records of that file bit for bit, or the bench exits with an error instead of printing a number.

value  = paths / device time of the tracking trips (CUDA events on the library's stream, inputs
         resident), max over ranks;
e2e    = paths / wall time of the C-ABI call pp_track_all with host buffers (start tables H2D,
         all records D2H, host post-processing), max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SYSTEM_FILE = os.path.join(ROOT, "tests", "data", "cyclic10.sys")
PREC = "dd"
GAMMA_SEED = 1
METRIC = "paths/sec to t=1 (cyclic-10, complex dd) at 1/2/4/8 B200 vs host CPU"
PHI = 0.6180339887498949


def chunk_offset(c: int, count: int, B: int) -> int:
    return int(math.floor(((c + 1) * PHI) % 1.0 * (count - B))) // 64 * 64


SHARD_BLOCK = 64


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch this script as N ranks on this node."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(cuda: bool = True):
    """One process per GPU (torchrun).  The data path has no collective; torch.distributed only
    carries the barrier and the max-over-ranks timing.  With more ranks than GPUs the ranks share
    devices round-robin and use gloo (NCCL refuses two ranks on one device); PP200_DIST_BACKEND
    overrides the choice."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = torch.cuda.device_count() if cuda else 0
        backend = os.environ.get("PP200_DIST_BACKEND", "nccl" if ndev >= world else "gloo")
        if ndev:
            local = local % ndev
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return world, rank, local, dist


def barrier(dist, local):
    if dist is not None:
        import torch

        torch.cuda.synchronize(local)
        dist.barrier()


def max_over_ranks(dist, local, value: float) -> float:
    if dist is None:
        return value
    import torch

    dev = f"cuda:{local}" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region"""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for name, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}


def profile_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, if present"""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get("kernels", {}).get(kernel, {}).get("dram_bytes_per_launch")


# ------------------------------------------------------------------------------------------------
# CPU baseline / reference arm: the reference library (oracle/_ref) on the host cores
# ------------------------------------------------------------------------------------------------
def cpu_reference_sample(text: str, lo: int, hi: int, threads: int, budget_s: float):
    """The reference tracker (oracle/_ref, the unmodified polypath build) on the host cores: each
    thread tracks consecutive paths of its own group (groups spread over [lo, hi)) with
    single-worker track_all calls until the time budget is spent.  (The reference's worker pool
    serialises concurrent callers; independent single-worker calls per thread do not.)"""
    import oracle as O

    if O.ref is None:
        raise RuntimeError("oracle/_ref/libppref.so (the reference build) is not present")
    gam = O.ref_random_gamma(GAMMA_SEED)  # the reference's own random_gamma: no product code on this arm
    span = hi - lo
    done = [0] * threads
    t_end = time.perf_counter() + budget_s

    def work(i):
        p, limit, chunk = lo + span * i // threads, lo + span * (i + 1) // threads, 1
        while p < limit and time.perf_counter() < t_end:
            q = min(limit, p + chunk)
            t0 = time.perf_counter()
            O.ref_track(text, PREC, gam, lo=p, hi=q, workers=1, batch=64)
            done[i] += q - p
            if time.perf_counter() - t0 < 0.05:
                chunk = min(chunk * 2, 64)
            p = q

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return sum(done), time.perf_counter() - t0, "reference"


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    with open(SYSTEM_FILE) as fh:
        text = fh.read()
    count = 3628800
    threads = os.cpu_count() or 1
    total_paths, total_wall, kind = 0, 0.0, "reference"
    for s in range(args.warmup + args.steps):
        lo = chunk_offset(s, count, args.paths)
        paths, wall, kind = cpu_reference_sample(text, lo, lo + args.paths, threads, args.cpu_budget)
        if s >= args.warmup:
            total_paths += paths
            total_wall += wall
    value = total_paths / total_wall
    sample = (f"each step: {args.cpu_budget:.0f} s of single-worker reference track_all calls on {threads} threads over "
              f"the step's chunk of {args.paths} start paths; {total_paths} paths timed over {args.steps} steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "dd (binary64 pairs)",
        "data": "synthetic: total-degree start solutions of cyclic-10, gamma = random_gamma(1)",
        "config": {"workload": "cyclic10 total-degree homotopy, complex double-double, TrackConfig::defaults(dd)",
                   "paths_per_step_per_gpu": args.paths, "cpu_threads": threads},
        "cpu_baseline": {"value": value, "unit": "paths/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------------
def fp64_peak_ops(device: int) -> float | None:
    import paper_1505_00383_b200 as P

    try:
        return P.fp64_peak(device)
    except Exception:
        return None


def validate_engine(P, h, starts, cfg, device):
    """One full-occupancy call (262,144 cyclic-10 dd paths) whose records must equal the reference
    records of tests/golden/track_cyclic10_dd_prod.npz bit for bit (8 ranges of 128 paths spread
    over the call).  Raises SystemExit on any difference.  Returns the call's device seconds."""
    gp = os.path.join(ROOT, "tests", "golden", "track_cyclic10_dd_prod.npz")
    with np.load(gp) as z:
        g = {k: z[k] for k in z.files}
    lo, hi, per = int(g["call_lo"]), int(g["call_hi"]), int(g["range_len"])
    sol = P.track_all(h, starts, cfg, lo=lo, hi=hi, device=device)
    keys = ["path_id", "status", "reason", "steps", "newton_iters", "rejections", "x", "residual"]
    for i, a in enumerate(g["range_lo"]):
        off = int(a) - lo
        for k in keys:
            got = np.ascontiguousarray(getattr(sol, k)[off:off + per])
            want = np.ascontiguousarray(g[k][i * per:(i + 1) * per])
            if got.dtype == np.float64:
                got, want = got.view(np.uint64), want.view(np.uint64)
            if not np.array_equal(got, want):
                raise SystemExit(f"bench self-check FAILED on device {device}: field {k} differs from the reference "
                                 f"records in [{int(a)}, {int(a) + per})")
    return sol.stats["device_ms"] / 1e3, len(g["range_lo"]) * per


def run_ours(args, world, rank, local, dist):
    import paper_1505_00383_b200 as P
    from paper_1505_00383_b200 import work as W

    with open(SYSTEM_FILE) as fh:
        text = fh.read()
    f = P.parse_system(text)
    g, starts = P.total_degree_start(f, PREC)
    h = P.make_homotopy(f, g, P.random_gamma(GAMMA_SEED), PREC)
    cfg = P.TrackConfig.defaults(PREC)
    count = starts.count
    B = args.paths
    dim = f.dim
    records = P.Records(B, dim, PREC)
    info = h.info

    def step(s):
        lo = chunk_offset(s, count, world * B)
        shard = (rank, world, SHARD_BLOCK) if world > 1 else None
        t0 = time.perf_counter()
        sol = P.track_all(h, starts, cfg, lo=lo, hi=lo + world * B, device=local, records=records, shard=shard)
        return sol, time.perf_counter() - t0

    # the engine's self-check (counts as the first warm-up step)
    _, checked = validate_engine(P, h, starts, cfg, local)
    for s in range(1, args.warmup):
        step(s)
    barrier(dist, local)
    dev_ms, wall_s, launches, paths, conv, h2d, d2h, evals, solves = 0.0, 0.0, 0, 0, 0, 0, 0, 0, 0
    with ClockSampler(local) as clk:
        t_all = time.perf_counter()
        for s in range(args.warmup, args.warmup + args.steps):
            sol, wall = step(s)
            st = sol.stats
            dev_ms += st["device_ms"]
            wall_s += wall
            launches += st["kernel_launches"]
            paths += len(sol)
            conv += int(np.sum(sol.status == P.SUCCESS))
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
            evals += st["evals"]
            solves += st["solves"]
        barrier(dist, local)
        t_all = time.perf_counter() - t_all
    dev_ms_max = max_over_ranks(dist, local, dev_ms)
    wall_max = max_over_ranks(dist, local, wall_s)
    total_paths = paths * world
    value = total_paths / (dev_ms_max / 1e3)
    e2e = total_paths / wall_max
    if rank != 0:
        return

    # roofline of the dominant kernel: one instrumented step (every trip's kernels bracketed by CUDA
    # events on the library's stream; per-trip log for the steady-state rates)
    import tempfile

    log = tempfile.NamedTemporaryFile(prefix="pp200_trips_", suffix=".txt", delete=False).name
    os.environ["PP200_KERNEL_TIMING"] = "1"
    os.environ["PP200_TRIP_LOG"] = log
    try:
        sol_i, _ = step(args.warmup + args.steps)
    finally:
        os.environ.pop("PP200_KERNEL_TIMING", None)
        os.environ.pop("PP200_TRIP_LOG", None)
    sti = sol_i.stats
    work = W.path_work(info, PREC, sti["evals"], sti["solves"])
    lsq_rate = work["lsq_total"] / (sti["lsq_ms"] / 1e3)
    eval_rate = work["eval_total"] / (sti["eval_ms"] / 1e3)
    dominant = "lsq_trip" if sti["lsq_ms"] >= sti["eval_ms"] else "ctrl_eval_trip"
    achieved = (lsq_rate if dominant == "lsq_trip" else eval_rate) / 1e12
    peak_ops = fp64_peak_ops(local)
    peak = peak_ops / 1e12 if peak_ops else None
    tot_ms = max(1e-9, sti["eval_ms"] + sti["lsq_ms"] + sti["step_ms"])
    shares = {"ctrl_eval_trip (control + evaluation)": sti["eval_ms"] / tot_ms, "lsq_trip": sti["lsq_ms"] / tot_ms,
              "tail mode control (step_trip)": sti["step_ms"] / tot_ms}
    steady = None
    try:
        t = np.loadtxt(log, ndmin=2)
        full = (t[:, 1] >= t[:, 5]) & (t[:, 6] == 0)  # thread-per-path trips on which every slot was busy
        if full.any() and peak_ops:
            steady = {"trips": int(full.sum()), "of_trips": len(t),
                      "eval_frac": float((t[full, 1] * work["eval_ops"]).sum() / (t[full, 2].sum() / 1e3) / peak_ops),
                      "lsq_frac": float((t[full, 1] * work["lsq_ops"]).sum() / (t[full, 3].sum() / 1e3) / peak_ops),
                      "busy_weighted_slot_use": float(t[:, 1].sum() / t[:, 5].sum())}
        os.unlink(log)
    except Exception:  # noqa: BLE001
        pass
    # nominal FP64 pipe rate: 148 SMs x 64 binary64 lanes x the SM clock under load
    sm_mhz = clk.summary().get("sm_mhz") or measured_peaks().get("sm_max_mhz") or 1965.0
    nominal = 148 * 64 * sm_mhz * 1e6 / 1e12
    # nominal FP64 pipe rate: 148 SMs x 64 binary64 lanes x the SM clock under load
    sm_mhz = clk.summary().get("sm_mhz") or measured_peaks().get("sm_max_mhz") or 1965.0
    nominal = 148 * 64 * sm_mhz * 1e6 / 1e12
    roofline = {
        "bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": (achieved / peak) if peak else None,
        "peak_nominal": nominal, "frac_nominal": achieved / nominal,
        "peak_nominal_def": "148 SMs x 64 FP64 lanes x median SM clock under load (DADD/DMUL/DFMA = 1 op)",
        "peak_nominal": nominal, "frac_nominal": achieved / nominal,
        "peak_nominal_def": "148 SMs x 64 FP64 lanes x median SM clock under load (DADD/DMUL/DFMA = 1 op)",
        "traffic": profile_traffic(dominant),
        "kernel": dominant,
        "op_convention": "binary64 pipe ops (DADD/DMUL/DFMA = 1 each) of the reference arithmetic",
        "peak_source": "measured FP64 pipe rate (pp_fp64_peak: independent DFMA chains, this GPU); "
                       "MEASURED_PEAKS.json has no FP64 figure",
        "achieved_def": "algorithmic ops of all launches of the kernel in one instrumented step / their summed "
                        "CUDA-event time (tail trips with few busy slots included)",
        "ctrl_eval_trip_tflops": eval_rate / 1e12, "lsq_trip_tflops": lsq_rate / 1e12,
        "steady_state": steady,
        "kernel_time_share": shares,
        "ops_per_unit": {"eval": work["eval_ops"], "lsq": work["lsq_ops"]},
        "units": {"evals": sti["evals"], "solves": sti["solves"]},
        "hbm_bytes_per_iteration": W.bytes_per_iteration(dim, PREC),
        "hbm_peak_gbs": measured_peaks().get("hbm_gbs"),
    }

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        lo = chunk_offset(args.warmup, count, B)
        try:
            cp, cw, kind = cpu_reference_sample(text, lo, lo + B, threads, args.cpu_budget)
            cpu = {"value": cp / cw, "unit": "paths/s", "cores": threads, "kind": kind,
                   "sample": f"{cp} paths of step {args.warmup}'s chunk in {cw:.1f} s: {threads} threads, each "
                             f"single-worker reference track_all calls over its own slice of the chunk"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "paths/s", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    line = {
        "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "dd (binary64 pairs)",
        "data": "synthetic: total-degree start solutions of cyclic-10, gamma = random_gamma(1)",
        "config": {"workload": "cyclic10 total-degree homotopy, complex double-double, TrackConfig::defaults(dd)",
                   "paths_per_step_per_gpu": B,
                   "chunks": f"per step a contiguous range of {world}x{B} start indices, golden-ratio spread over "
                             f"[0, 3628800); rank r tracks block-cyclic shard r (blocks of {SHARD_BLOCK})",
                   "parallelism": f"static path shards x{world}, no collective",
                   "self_check": f"{checked} reference records reproduced bit for bit in a 262,144-path call before timing",
                   "l2": "working set (slot state, Jacobians) larger than L2 each step", "slots": sol_i.stats["slots"]},
        "converged_fraction": conv / max(1, paths),
        "e2e": {"value": e2e, "unit": "paths/s", "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "wall_s": t_all,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # 393,216 paths per step and GPU: the per-step tail (the last, longest paths of a call running
    # on few SMs) costs less than at 262,144 (17.9 k against 17.5 k paths/s measured), while a
    # 25-step driver run still takes about ten minutes; the whole 3,628,800-path job in one call
    # runs at 18.6 k (profiles/r02/full_cyclic10_dd.json)
    ap.add_argument("--paths", type=int, default=393216, help="start paths per step per GPU (multiple of 64)")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of reference CPU tracking per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--launch-check", action="store_true",
                    help="print each rank's launch geometry and shard, then exit (no GPU work)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.launch_check:
        world, rank, local, dist = dist_setup(cuda=False)
        count, B = 3628800, args.paths
        lo = chunk_offset(args.warmup, count, world * B)
        print(json.dumps({"rank": rank, "world": world, "gpus": args.gpus, "local": local,
                          "first_timed_step": [lo, lo + world * B], "shard": [rank, world, SHARD_BLOCK]}), flush=True)
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
