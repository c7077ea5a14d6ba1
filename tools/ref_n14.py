"""One measured run of the REAL reference package at the headline configuration.

The reference caps reconstruct() at n <= 12 (pipeline.py:228-233) and its int64
record would be 627 GB, so at n = 14 it is driven the way SURVEY §8(c)/(d)
prescribe: step_one_least_squares(streaming source, workers=cores) +
step_two_assemble(theta, workers=1), the reference's own public functions,
unmodified (pauli_lre from baseline/_ref, numba).  The streaming source returns
the C5 record's rows (device generator, the B200 arm's record) divided by
shots — the generation + device-to-host copy of each block runs inside the
reference's timed loop and is measured separately (t_source_s) so it can be
subtracted.

    python tools/ref_n14.py [--qubits 14] [--workers 16]   (prints one JSON line)
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=14)
    ap.add_argument("--shots", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1602)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()

    import torch

    import bench
    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200.simulate import generate_device_counts

    mods, why = bench._import_reference()
    if mods is None:
        print(json.dumps({"unavailable": why}))
        return
    P, _ = mods
    n, shots = args.qubits, args.shots
    st = lre.StateDescriptor("ghz", n)
    lock = threading.Lock()
    spent = [0.0]

    class DeviceRecordSource:
        """Reference source protocol (pipeline.py:42-59): .n, .num_settings, .frequencies(a, b)."""

        def __init__(self):
            self.n, self.num_settings = n, 3**n

        def frequencies(self, a, b):
            t0 = time.perf_counter()
            with lock:  # one generator launch + D2H at a time
                rows = generate_device_counts(st, shots, seed=args.seed, w_begin=a, w_end=b).cpu().numpy()
            out = rows / float(shots)  # records.py:62-64
            with lock:
                spent[0] += time.perf_counter() - t0
            return out

    src = DeviceRecordSource()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    theta = P.step_one_least_squares(src, workers=args.workers)
    t1 = time.perf_counter()
    P.step_two_assemble(theta, workers=1)
    t2 = time.perf_counter()
    print(json.dumps({
        "what": "reference pauli_lre step_one_least_squares(streaming source, workers) + step_two_assemble(workers=1)",
        "n": n, "shots": shots, "state": "ghz", "workers": args.workers, "cpu_model": bench.cpu_model(),
        "t_step1_s": t1 - t0, "t_step2_s": t2 - t1, "t_total_s": t2 - t0,
        "t_source_s": spent[0], "t_step1_minus_source_s": (t1 - t0) - spent[0] / max(1, args.workers),
        "note": "t_source_s is summed over the worker threads that call frequencies() concurrently",
        "theta_0": float(theta[0]),
    }))


if __name__ == "__main__":
    main()
