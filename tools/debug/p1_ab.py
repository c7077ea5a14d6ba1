"""A/B timing of the pass-1 variants (TMA ring vs LDG) at one size; each run in
a subprocess under a hard timeout.  usage: p1_ab.py n [shots]"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_1602_08604_b200 as lre
from paper_1602_08604_b200.simulate import generate_device_counts
n, shots = int(sys.argv[1]), int(sys.argv[2])
counts = generate_device_counts(lre.StateDescriptor("ghz", n), shots, seed=1602)
plan = lre.LREPlan(n, shots, with_mu=False)
s = torch.cuda.current_stream()
dt = 2 if counts.dtype == torch.uint16 else 1
for _ in range(3): plan.stage(counts, dt, 0, 3**n, s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
e0.record(s)
for _ in range(K): plan.stage(counts, dt, 0, 3**n, s)
e1.record(s); e1.synchronize()
t = e0.elapsed_time(e1) / 1e3 / K
b = counts.numel() * counts.element_size()
print(f"pass1 n={n} {t*1e3:.3f} ms  {b/t/1e9:.0f} GB/s (counts read)")
e0.record(s)
for _ in range(K): plan.finish(s)
e1.record(s); e1.synchronize()
print(f"passes 2.. {e0.elapsed_time(e1)/K:.3f} ms")
''' % ROOT
n = sys.argv[1]; shots = sys.argv[2] if len(sys.argv) > 2 else "1000"
for env in ({}, {"LRE_P1": "ring"}):
    try:
        r = subprocess.run([sys.executable, "-c", CODE, n, shots], env={**os.environ, **env}, capture_output=True,
                           text=True, timeout=240)
        print(env or "LDG", r.stdout.strip(), r.stderr.strip()[-400:])
    except subprocess.TimeoutExpired:
        print(env, "TIMEOUT")
