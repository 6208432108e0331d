"""Short tracking run for ncu / throughput experiments: cyclic-10 dd, PATHS start paths at OFFSET
(env overrides), with the SM clock sampled during the run.

    ncu --set full -k regex:lsq_trip -s 200 -c 1 -o gpurun_out/prof python scripts/profile_run.py
"""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_00383_b200 as P  # noqa: E402

paths = int(os.environ.get("PATHS", "32768"))
offset = int(os.environ.get("OFFSET", "1000000"))
prec = os.environ.get("PREC", "dd")
system = os.environ.get("SYSTEM", "cyclic10.sys")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
f = P.parse_system(open(os.path.join(root, "tests", "data", system)).read())
g, st = P.total_degree_start(f, prec)
h = P.make_homotopy(f, g, P.random_gamma(1), prec)

clocks, stop = [], threading.Event()


def sample():
    try:
        import pynvml

        pynvml.nvmlInit()
        hd = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            clocks.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                           pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd), pynvml.nvmlDeviceGetPowerUsage(hd) / 1e3))
            time.sleep(0.2)
    except Exception:  # noqa: BLE001
        pass


th = threading.Thread(target=sample, daemon=True)
th.start()
t0 = time.time()
cfg = P.TrackConfig.defaults(prec)
if os.environ.get("MAX_NEWTON"):
    cfg.max_newton = int(os.environ["MAX_NEWTON"])
sol = P.track_all(h, st, cfg, lo=offset, hi=offset + paths)
wall = time.time() - t0
stop.set()
th.join()
s = sol.stats
clk = f"sm_mhz median {statistics.median(c[0] for c in clocks):.0f} min {min(c[0] for c in clocks)} reasons {sorted(set(hex(c[1]) for c in clocks))} W max {max(c[2] for c in clocks):.0f}" if clocks else "no clock samples"
print(f"{system} {prec} {paths} paths: wall {wall:.2f}s device {s['device_ms']:.1f} ms trips {s['total_rounds']} "
      f"evals {s['evals']} solves {s['solves']} eval_ms {s['eval_ms']:.1f} lsq_ms {s['lsq_ms']:.1f} step_ms {s['step_ms']:.1f} "
      f"-> {paths / (s['device_ms'] / 1e3):.1f} paths/s; {sol.counts()}; {clk}", flush=True)
