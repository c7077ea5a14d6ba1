"""Phase timeline of assemble_x8_kernel (debug build with -DLRE_X8_PROFILE, loaded via
LRE_LIB_PATH): per block, time from loop top to (1) cluster wait done, (2) pushes issued,
(3) all eighths received, (4) WHT done, (5) write phase issued."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1602_08604_b200 import _lib  # noqa: E402

n = int(os.environ.get("N", "14"))
d = 1 << n
theta = torch.randn(4**n, dtype=torch.float64, device="cuda")
mu = torch.empty((d, d), dtype=torch.complex128, device="cuda")
s = torch.cuda.current_stream()
for _ in range(3):
    _lib.call("lre_assemble", theta.data_ptr(), _lib.MASK_MAJOR, n, 0, d, mu.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
buf = np.zeros((148 * 2, 64, 6), dtype=np.uint64)
L = _lib.load()
L.lre_x8_profile_dump.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.lre_x8_profile_dump(buf.ctypes.data, buf.nbytes) == 0
ctas = [c for c in range(buf.shape[0]) if buf[c, 1, 0] != 0]
dt = []
for c in ctas:
    for it in range(1, 60):
        row = buf[c, it].astype(np.int64)
        nxt = buf[c, it + 1, 0].astype(np.int64)
        if row[0] == 0 or nxt == 0 or row[2] == 0:
            continue
        dt.append([row[1] - row[0], row[2] - row[1], row[3] - row[2], row[4] - row[3], row[5] - row[4], nxt - row[5]])
dt = np.array(dt, dtype=np.float64) / 1e3
names = ["cluster wait", "push (loads+butterfly+st.async)", "wait eighths", "WHT", "write phase", "arrive->next top"]
print(f"n={n}: {len(ctas)} CTAs, {len(dt)} SPLIT blocks sampled; mean per block {dt.sum(1).mean():.2f} us")
for k, nm in enumerate(names):
    print(f"  {nm:34s} mean {dt[:, k].mean():6.2f} us   p50 {np.median(dt[:, k]):6.2f}   p90 {np.percentile(dt[:, k], 90):6.2f}")
