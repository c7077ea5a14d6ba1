"""Debug harness: run pass 1 through the TMA path on small sizes, each under a
hard timeout, and compare with the LDG path (LRE_NO_TMA=1 in a subprocess)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import sys, numpy as np, torch, ctypes
sys.path.insert(0, %r)
from paper_1602_08604_b200 import _lib
from oracle import c_oracle as C
n, shots = int(sys.argv[1]), 1000
rng = np.random.default_rng(n)
p = rng.dirichlet(np.full(1 << n, 0.3), size=3**n)
counts = np.stack([rng.multinomial(shots, pi) for pi in p]).astype(np.uint16)
dc = torch.from_numpy(counts).cuda()
ws = ctypes.c_size_t(0)
_lib.check(_lib.load().lre_step1_workspace(n, shots, 0, 3**n, ctypes.byref(ws)), "ws")
buf = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
out = torch.empty(4**n, dtype=torch.int64, device="cuda")
_lib.call("lre_step1", dc.data_ptr(), 2, n, shots, 0, 3**n, buf.data_ptr(), ws.value, out.data_ptr(), 1, 0,
          torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
got = out.cpu().numpy()
ref = C.numerators(counts, n)
print("n", n, "exact", bool((got == ref).all()), "mismatches", int((got != ref).sum()))
''' % ROOT
for n in (int(x) for x in sys.argv[1:]):
    for env in ({}, {"LRE_P1": "ring"}, {"LRE_P1": "tma"}):
        try:
            r = subprocess.run([sys.executable, "-c", CODE, str(n)], env={**os.environ, **env}, capture_output=True,
                               text=True, timeout=90)
            print(env, r.stdout.strip()[-3000:], r.stderr.strip()[-300:])
        except subprocess.TimeoutExpired:
            print(env, "n", n, "TIMEOUT")
