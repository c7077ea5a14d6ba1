"""Validate the CPU-baseline cost model against full C-port runs (n given)."""
import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import c_oracle as C, lre_oracle as O
import bench
n = int(sys.argv[1]); shots = 1000
T = os.cpu_count()
rows = O.sample_ghz_counts(n, shots, 1602, 0, 3**n)
S = bench.baseline_settings(n)
f, p = C.step1_cost(rows[:2 * S], n, shots, 0, T)
pred = f + p * 3**n / T
t = time.perf_counter(); C.step1_raw(rows, n, shots, 0, T); full = time.perf_counter() - t
print(f"n={n} threads={T} model {pred:.2f} s (fixed {f:.2f} + {p*1e6:.1f} us/setting/worker)  full run {full:.2f} s")
