import time, torch
for n in (12, 13, 14):
    d = 1 << n
    g = torch.randn(d, d, dtype=torch.complex128, device="cuda")
    h = (g + g.conj().T) / 2
    del g
    for lib in ("cusolver", "magma"):
        try:
            torch.backends.cuda.preferred_linalg_library(lib)
            torch.linalg.eigh(h[:64, :64]); torch.cuda.synchronize()
            t = time.perf_counter(); w, v = torch.linalg.eigh(h); torch.cuda.synchronize()
            print(n, lib, f"{time.perf_counter() - t:.3f} s", flush=True)
            del w, v
        except Exception as e:
            print(n, lib, "error", str(e)[:100], flush=True)
    del h; torch.cuda.empty_cache()
