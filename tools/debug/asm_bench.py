"""Time lre_assemble alone (natural theta -> mu) at size n. usage: asm_bench.py n [reps]"""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1602_08604_b200 import _lib
n = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
d = 1 << n
theta = torch.randn(4**n, dtype=torch.float64, device="cuda")
mu = torch.empty((d, d), dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
call = lambda: _lib.call("lre_assemble", theta.data_ptr(), _lib.NATURAL, n, 0, d, mu.data_ptr(), s.cuda_stream)
for _ in range(2): call()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(reps): call()
e1.record(s); e1.synchronize()
t = e0.elapsed_time(e1) / reps / 1e3
print(f"assemble n={n}: {t*1e3:.3f} ms  theta+mu {(8*4**n + 16*4**n)/t/1e9:.0f} GB/s")
