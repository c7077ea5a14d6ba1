import sys, numpy as np, torch, ctypes
sys.path.insert(0, "/root/repo")
from paper_1602_08604_b200 import _lib
n, shots = int(sys.argv[1]), 1000
rng = np.random.default_rng(n)
counts = rng.integers(0, 3, size=(3**n, 1 << n)).astype(np.uint16)
dc = torch.from_numpy(counts).cuda()
ws = ctypes.c_size_t(0)
_lib.check(_lib.load().lre_step1_workspace(n, shots, 0, 3**n, ctypes.byref(ws)), "ws")
buf = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
out = torch.empty(4**n, dtype=torch.int64, device="cuda")
_lib.call("lre_step1", dc.data_ptr(), 2, n, shots, 0, 3**n, buf.data_ptr(), ws.value, out.data_ptr(), 1, 0,
          torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done", out[:4].tolist())
