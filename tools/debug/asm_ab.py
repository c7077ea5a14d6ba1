"""A/B of the step-(ii) assembly at n = 14 (mask-major theta, assemble_x8_kernel): time per launch."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1602_08604_b200 import _lib
n = int(os.environ.get("N", "14"))
d = 1 << n
theta = torch.randn(4**n, dtype=torch.float64, device="cuda")
mu = torch.empty((d, d), dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    _lib.call("lre_assemble", theta.data_ptr(), _lib.MASK_MAJOR, n, 0, d, mu.data_ptr(), s.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    _lib.call("lre_assemble", theta.data_ptr(), _lib.MASK_MAJOR, n, 0, d, mu.data_ptr(), s.cuda_stream)
e1.record(s)
e1.synchronize()
t = e0.elapsed_time(e1) / 10 / 1e3
print(json.dumps({"n": n, "asm": os.environ.get("LRE_ASM", ""), "order": os.environ.get("LRE_X8_ORDER", ""),
                  "ms": t * 1e3, "TBps": 24 * 4**n / t / 1e12}))
