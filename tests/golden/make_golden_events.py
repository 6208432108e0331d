"""Golden step events (ProgressSink, tracker.hpp:62-70): the StepEvents the UNMODIFIED reference
(oracle/_ref) emits from step_control_all (tracker.cpp:312-315) while tracking, with the records of
the same call.

    python tests/golden/make_golden_events.py
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(ROOT, "tests", "data")

CASES = [("cyclic5_d", "cyclic5.sys", "d", 0, 120, None), ("cyclic5_dd", "cyclic5.sys", "dd", 0, 120, None),
         ("cyclic5_d_tight", "cyclic5.sys", "d", 0, 120, {"max_newton": 2, "h_init": 0.1, "max_steps": 40})]

for name, sysf, prec, lo, hi, cfg in CASES:
    text = open(os.path.join(DATA, sysf)).read()
    rec, ev = O.ref_track_events(text, prec, O.ref_random_gamma(1), cfg=cfg, lo=lo, hi=hi)
    np.savez_compressed(os.path.join(HERE, f"events_{name}.npz"), prec=prec, lo=lo, hi=hi, cfg=repr(cfg or {}),
                        events=ev, **rec)
    print(f"events_{name}: {len(ev)} events for {len(rec['status'])} paths")
