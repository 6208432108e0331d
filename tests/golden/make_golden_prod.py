"""Golden records for the production-occupancy parity tests: reference records (the UNMODIFIED
reference library, oracle/_ref) for several start-index ranges spread over one benchmark-sized
call, so that a single device call at full occupancy (all slots, TMEM evaluation, refill,
compaction, CUDA graphs, tail mode) can be checked bit for bit in several places.

    python tests/golden/make_golden_prod.py
"""

import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(ROOT, "tests", "data")

# (name, system, prec, call [lo, hi), number of ranges, paths per range)
CASES = [
    ("cyclic10_dd_prod", "cyclic10.sys", "dd", 868_928, 868_928 + 262_144, 8, 128),
    ("cyclic10_d_prod", "cyclic10.sys", "d", 1_500_000, 1_500_000 + 524_288, 8, 256),
]


def main():
    for name, sysf, prec, lo, hi, nr, per in CASES:
        text = open(os.path.join(DATA, sysf)).read()
        gam = O.ref_random_gamma(1)
        # ranges at evenly spaced offsets, the last one ending at the call's end (the tail)
        starts = [lo + (hi - lo - per) * i // (nr - 1) // 32 * 32 for i in range(nr)]
        starts[-1] = hi - per
        # one single-worker reference call per range, the ranges on concurrent threads (ctypes
        # releases the GIL; the reference's results do not depend on batching, test_tracker.cpp:383-432)
        parts = [None] * nr

        def run(i):
            parts[i] = O.ref_track(text, prec, gam, lo=starts[i], hi=starts[i] + per, workers=1, batch=64)

        ths = [threading.Thread(target=run, args=(i,)) for i in range(nr)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        keys = [k for k in parts[0] if np.ndim(parts[0][k]) > 0]
        out = {k: np.concatenate([p[k] for p in parts]) for k in keys}
        np.savez_compressed(os.path.join(HERE, f"track_{name}.npz"), prec=prec, gamma_seed=1, call_lo=lo, call_hi=hi,
                            range_lo=np.array(starts, np.int64), range_len=per, **out)
        print(f"track_{name}: {len(out['status'])} paths in {nr} ranges, converged {int(np.sum(out['status'] == 1))}",
              flush=True)


if __name__ == "__main__":
    main()
