"""Time the passes after pass 1 (lre_step1_finish) and pass 1 alone at size n.  usage: finish_bench.py n [K]"""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1602_08604_b200 as lre
from paper_1602_08604_b200.simulate import generate_device_counts
n = int(sys.argv[1]); K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
counts = generate_device_counts(lre.StateDescriptor("ghz", n), 1000, seed=1602)
plan = lre.LREPlan(n, 1000, with_mu=False)
s = torch.cuda.current_stream()
plan.stage(counts, 2, 0, 3**n, s)
for _ in range(3): plan.finish(s)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(K): plan.finish(s)
e1.record(s); e1.synchronize()
print(f"n={n} passes 2..: {e0.elapsed_time(e1)/K:.3f} ms")
