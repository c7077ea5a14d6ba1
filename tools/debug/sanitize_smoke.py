"""Small instances of every product kernel, for compute-sanitizer
(memcheck / racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/debug/sanitize_smoke.py
Round 2 adds: the 8-CTA-cluster assembly (n = 11: SPLIT and FULL mask blocks,
whole range and chunked slabs), the mask-major final pass, the fp64 frequency
folds (device probabilities and a host-streamed source), one-pass streaming.
Later in round 2: split Y1 storage at n = 11 (the compile-time split tile-pass
variant with its mbarrier hand-off, the int16 vector pass with its per-task
barrier, the high-part chain on 1184-entry rows, the final pass's cooperative
merge, and the natural-layout merge kernel).
Set LRE_ASM=legacy to route mask-major assembly through the round-1 kernels."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1602_08604_b200 as lre  # noqa: E402
from paper_1602_08604_b200 import metrics as M  # noqa: E402
from paper_1602_08604_b200 import simulate as S  # noqa: E402


def main():
    lre.reconstruct(lre.sample_counts(lre.StateDescriptor("w", 7), 70000, seed=1), project=False)
    for n, shots, kind in [(8, 1000, "ghz"), (10, 500, "w")]:
        st = lre.StateDescriptor(kind, n)
        rec = lre.sample_counts(st, shots, seed=1)
        res = lre.reconstruct(rec, project=False, as_tensor=True)
        plan = lre.LREPlan(n, shots)
        s = torch.cuda.current_stream()
        q = 3**min(n, 7)
        for lo in range(0, 3**n, q):
            plan.stage(rec.counts[lo:lo + q], rec.lre_dtype, lo, min(3**n, lo + q), s)
        plan.finish(s)
        plan.step2(s)
        assert torch.equal(plan.theta, res.theta)
    big = lre.sample_counts(lre.StateDescriptor("ghz", 5), 3_000_000_000, seed=2, dtype=np.int64)
    lre.reconstruct(big, project=False)
    o = lre.sample_outcomes(lre.StateDescriptor("ghz", 9), 300, seed=3)
    lre.reconstruct(o, project=False)
    rho = S.density_matrix(lre.StateDescriptor("random", 6, state_seed=4))
    rec = S.sample_counts_from_density(rho, 200, seed=5)
    res = lre.reconstruct(rec, project=True, as_tensor=True)
    M.evaluate_errors(lre.StateDescriptor("ghz", 6), res.rho, res.mu, n0=3.0)
    M.hs_squared_distance(res.mu, torch.from_numpy(rho).cuda())
    # round 2: n = 11 (cluster assembly incl. FULL-mode blocks, mask-major final pass)
    rec = lre.sample_counts(lre.StateDescriptor("ghz", 11), 40, seed=6)
    lre.reconstruct(rec, project=False)
    from paper_1602_08604_b200 import distributed as D

    comp = D.DeviceCompute(11, 40, 0, 3**11, 1, 0, torch.device("cuda", 0), chunks=4)
    D.LocalShardedLRE([comp]).step([rec.counts], rec.lre_dtype)
    # split Y1 with natural-layout int64 numerators (the separate merge kernel)
    import ctypes

    from paper_1602_08604_b200 import _lib

    ws = ctypes.c_size_t(0)
    _lib.check(_lib.load().lre_step1_workspace(11, 40, 0, 3**11, ctypes.byref(ws)), "ws")
    buf = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    num = torch.empty(4**11, dtype=torch.int64, device="cuda")
    _lib.call("lre_step1", rec.counts.data_ptr(), rec.lre_dtype, 11, 40, 0, 3**11, buf.data_ptr(), ws.value,
              num.data_ptr(), _lib.OUT_NUM_I64, _lib.NATURAL, torch.cuda.current_stream().cuda_stream)
    # fp64 frequency sources: device probabilities and a host-streamed duck source
    lre.reconstruct(lre.ExactFrequencies(lre.StateDescriptor("random", 5, state_seed=7)), project=False)

    class Src:
        n, num_settings = 8, 3**8

        def frequencies(self, a, b):
            return np.full((b - a, 256), 1.0 / 256)

    plan = lre.F64Plan(8, chunk_bytes=3**6 * 256 * 8)
    plan.step1(Src(), torch.cuda.current_stream())
    # one-pass streaming plan (n = 6)
    r6 = lre.sample_counts(lre.StateDescriptor("w", 6), 100, seed=8)
    p6 = lre.LREPlan(6, 100, with_mu=False)
    p6.stage(r6.counts, r6.lre_dtype, 0, 3**6, torch.cuda.current_stream())
    p6.finish(torch.cuda.current_stream())
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
