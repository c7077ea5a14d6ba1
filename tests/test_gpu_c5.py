"""Parity of the headline configuration (BASELINE.json C5: n = 14 GHZ/W, 1000
shots per setting, uint16 counts) and of n = 13 — the exact kernel sequence
bench.py times, against the C oracle on identical counts.  Needs a GPU.

Kernels exercised (n = 13 and 14, shots = 1000 <= 1213, uint16):
  * pass 1  tile_pass_kernel<7, SMALL=true, uint16_t, LOGN=13|14> (packed
    int16x2 L1, compile-time row length);
  * pass 2  vfold3_kernel<false> at V = 4^7;
  * pass 3  vfold3_kernel<true> at V = 4^10 (n = 13, final) /
            vfold3_kernel<false> at V = 4^10 (n = 14);
  * pass 4  final_mm_kernel<int32, int64, THETA> at V = 4^13 (n = 14, the
            plan's mask-major theta) and vfold_kernel<1, int32, int64, FINAL>
            (natural-order numerators);
  * step (ii) assemble_cl8_kernel<14> (8-CTA clusters) on a general
    theta and on the benchmarked plan's own theta.
Bars: int64 numerators bit-exact; theta and mu within 1e-10 relative Frobenius.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import c_oracle as C  # noqa: E402
from oracle import lre_oracle as O  # noqa: E402

TOL = 1e-10
SHOTS = 1000
SEED = 1602


@pytest.fixture(scope="module")
def lre():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200 import _lib

    _lib.load()
    return lre


def _free_gib():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0] / 2**30


def _step1_num(counts_dev, n, w_begin, w_end, layout=0):
    """lre_step1(OUT_NUM_I64) over rows [w_begin, w_end) through the C ABI."""
    from paper_1602_08604_b200 import _lib

    ws = ctypes.c_size_t(0)
    _lib.check(_lib.load().lre_step1_workspace(n, SHOTS, w_begin, w_end, ctypes.byref(ws)), "ws")
    buf = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
    out = torch.empty(4**n, dtype=torch.int64, device="cuda")
    _lib.call("lre_step1", counts_dev.data_ptr(), _lib.U16, n, SHOTS, w_begin, w_end, buf.data_ptr(), ws.value,
              out.data_ptr(), _lib.OUT_NUM_I64, layout, torch.cuda.current_stream().cuda_stream)
    del buf
    return out


class TestHeadlinePlan:
    def test_plan_shapes(self, lre):
        """The plans the parity tests below cover are the ones bench.py runs."""
        from paper_1602_08604_b200 import _lib

        L = _lib.load()
        assert L.lre_step1_num_passes(13, SHOTS) == 3  # 7 | 3 | 3
        assert L.lre_step1_num_passes(14, SHOTS) == 4  # 7 | 3 | 3 | 1
        assert L.lre_shard_quantum(14) == 3**7


class TestN13Full:
    @pytest.mark.parametrize("kind", ["ghz", "w"])
    def test_numerators_and_theta(self, lre, kind):
        """Full n = 13 record (26 GB uint16): numerators bit-exact, theta to 1e-10,
        against the C restatement of the reference step (i) on the same counts."""
        n = 13
        if _free_gib() < 40:
            pytest.skip("needs ~40 GiB of HBM")
        st = lre.StateDescriptor(kind, n)
        rec = lre.sample_counts(st, SHOTS, seed=SEED)
        assert rec.counts.dtype == torch.uint16
        host = rec.counts.cpu().numpy()
        num = _step1_num(rec.counts, n, 0, 3**n).cpu().numpy()
        ref_num = C.numerators(host, n)
        np.testing.assert_array_equal(num, ref_num)
        plan = lre.LREPlan(n, SHOTS, with_mu=False)
        plan.step1(rec.counts, rec.lre_dtype, torch.cuda.current_stream())
        theta = plan.theta_natural().cpu().numpy()
        del plan, rec
        ref_theta = C.step_one(host, n, SHOTS)
        assert O.rel_frobenius(theta, ref_theta) < TOL
        # the epilogue is exactly N * fac[zc] of the numerators
        assert O.rel_frobenius(theta, O.finalize_numerators(ref_num, n, SHOTS)) < 1e-15


class TestN14Shards:
    @pytest.mark.parametrize("kind", ["ghz", "w"])
    def test_shard_numerators_bit_exact(self, lre, kind):
        """lre_step1(OUT_NUM_I64) at n = 14 on 3^7-aligned shards (first, middle,
        last) — the same pass-1..4 instantiations as the full record."""
        from paper_1602_08604_b200.simulate import generate_device_counts

        n, q = 14, 3**7
        if _free_gib() < 12:
            pytest.skip("needs ~12 GiB of HBM")
        st = lre.StateDescriptor(kind, n)
        total = 3**n
        shards = [(0, q), (total // 2 // q * q, total // 2 // q * q + 2 * q), (total - 2 * q, total)]
        for lo, hi in shards:
            counts = generate_device_counts(st, SHOTS, seed=SEED, w_begin=lo, w_end=hi)
            assert counts.dtype == torch.uint16
            got = _step1_num(counts, n, lo, hi).cpu().numpy()
            ref = C.numerators(counts.cpu().numpy(), n, lo, threads=4)
            np.testing.assert_array_equal(got, ref)
            del counts, got, ref

    def test_shards_sum_to_full_range_numerators(self, lre):
        """Linearity at full size: a 3-shard sum equals the one-shot numerators of the
        union (same kernels, different row ranges), mask-major layout."""
        from paper_1602_08604_b200.simulate import generate_device_counts
        from paper_1602_08604_b200 import _lib

        n, q = 14, 3**7
        if _free_gib() < 16:
            pytest.skip("needs ~16 GiB of HBM")
        st = lre.StateDescriptor("ghz", n)
        lo, hi = 5 * q, 11 * q
        counts = generate_device_counts(st, SHOTS, seed=SEED, w_begin=lo, w_end=hi)
        whole = _step1_num(counts, n, lo, hi, _lib.MASK_MAJOR)
        acc = torch.zeros_like(whole)
        for a, b in [(lo, lo + q), (lo + q, lo + 4 * q), (lo + 4 * q, hi)]:
            acc += _step1_num(counts[a - lo:b - lo].contiguous(), n, a, b, _lib.MASK_MAJOR)
        assert torch.equal(acc, whole)
        # I numerator: every setting contributes its row sum
        m0 = whole[0].item()
        assert m0 == (hi - lo) * SHOTS


def _n14_masks():
    d = 1 << 14
    fixed = [0, 1, 2, 3, 6, 7, 0x1FFE, 0x1FFF, 0x2000, 0x2001, 0x2AAA, 0x2AAB, 0x3FFC, 0x3FFD, 0x3FFE, 0x3FFF]
    rng = np.random.default_rng(14)
    pairs = rng.choice(d // 2, size=24, replace=False) * 2
    return sorted(set(fixed) | {int(p) for p in pairs} | {int(p) + 1 for p in pairs})


class TestN14FullPlan:
    def test_benchmarked_sequence_sampled_ghz(self, lre):
        """The whole timed reconstruction of bench.py (LREPlan.run on the 1000-shot
        GHZ record, 146 GiB of uint16 counts): theta (mask-major final pass +
        export) equals the natural-order numerators' epilogue; mu equals the
        oracle's step (ii) on that theta for 24 masks; trace 1."""
        n = 14
        d = 1 << n
        if _free_gib() < 172:
            pytest.skip("needs ~172 GiB of HBM")
        from paper_1602_08604_b200 import _lib

        rec = lre.sample_counts(lre.StateDescriptor("ghz", n), SHOTS, seed=SEED)
        plan = lre.LREPlan(n, SHOTS)
        s = torch.cuda.current_stream()
        num = torch.empty(4**n, dtype=torch.int64, device="cuda")
        _lib.call("lre_step1", rec.counts.data_ptr(), rec.lre_dtype, n, SHOTS, 0, 3**n, plan.ws.data_ptr(),
                  plan.ws_bytes, num.data_ptr(), _lib.OUT_NUM_I64, _lib.NATURAL, s.cuda_stream)
        num_h = num.cpu().numpy()
        del num
        plan.run(rec.counts, rec.lre_dtype, s)
        del rec
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        assert int(num_h[0]) == 3**n * SHOTS
        theta = plan.theta_natural(out=plan.export_buffer()).cpu().numpy()
        assert O.rel_frobenius(theta, O.finalize_numerators(num_h, n, SHOTS)) < 1e-15
        del num_h
        rows = torch.arange(d, device="cuda")
        for m in _n14_masks()[::3]:
            ref = C.step_two_masks(theta, n, m, m + 1)[0]
            got = plan.mu[rows, rows ^ m].cpu().numpy()
            assert O.rel_frobenius(got, ref) < TOL, f"mask {m}"
        assert abs(float(torch.diagonal(plan.mu).real.sum().item()) - 1.0) < 1e-12
        del plan


class TestN14Assembly:
    def test_random_theta_vs_oracle(self, lre):
        """lre_assemble at n = 14 (the benchmarked step (ii) kernel) on a random
        theta: >= 64 masks incl. (m, m+1) pairs of mixed popcount and the all-ones
        pair, every row (both halves), against C.step_two_masks."""
        n = 14
        d = 1 << n
        if _free_gib() < 8:
            pytest.skip("needs ~8 GiB of HBM")
        g = torch.Generator(device="cuda").manual_seed(1414)
        theta = torch.randn(4**n, dtype=torch.float64, device="cuda", generator=g)
        mu = lre.step_two_assemble(theta, as_tensor=True)
        theta_h = theta.cpu().numpy()
        masks = _n14_masks()
        assert len(masks) >= 64
        rows = torch.arange(d, device="cuda")
        for m in masks:
            ref = C.step_two_masks(theta_h, n, m, m + 1)[0]
            got = mu[rows, rows ^ m].cpu().numpy()
            assert O.rel_frobenius(got, ref) < TOL, f"mask {m}"
        # Hermitian by construction
        assert torch.equal(mu[0, 1:257], mu[1:257, 0].conj())

    def test_every_block_written(self, lre):
        """The n = 14 block schedule (FULL-mode blocks dealt out round-robin first,
        then the SPLIT blocks) covers every 8-mask block: mu starts as NaN, and after
        one lre_assemble no NaN is left and mu is exactly Hermitian (rows r and r^m of
        a mask are written by the same CTA, so a skipped or half-written block shows)."""
        from paper_1602_08604_b200 import _lib

        n = 14
        d = 1 << n
        if _free_gib() < 16:
            pytest.skip("needs ~16 GiB of HBM")
        g = torch.Generator(device="cuda").manual_seed(2024)
        mm = torch.randn(4**n, dtype=torch.float64, device="cuda", generator=g)  # mask-major theta
        mu = torch.full((d, d), complex(float("nan"), float("nan")), dtype=torch.complex128, device="cuda")
        _lib.call("lre_assemble", mm.data_ptr(), _lib.MASK_MAJOR, n, 0, d, mu.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        assert not bool(torch.isnan(torch.view_as_real(mu)).any())
        assert torch.equal(mu, mu.conj().T)
        # and it is the same estimate as the natural-layout entry point gives
        theta = torch.empty_like(mm)
        _lib.call("lre_theta_relayout", mm.data_ptr(), _lib.MASK_MAJOR, n, theta.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        del mm
        assert torch.equal(mu, lre.step_two_assemble(theta, as_tensor=True))

    def test_mask_major_slices_match_full(self, lre):
        """Multi-GPU form: mask-major theta slices of 1/8 of the masks assemble to the
        matching column blocks of the full estimate."""
        from paper_1602_08604_b200 import _lib

        n = 14
        d = 1 << n
        if _free_gib() < 16:
            pytest.skip("needs ~16 GiB of HBM")
        g = torch.Generator(device="cuda").manual_seed(7)
        theta = torch.randn(4**n, dtype=torch.float64, device="cuda", generator=g)
        mm = torch.empty_like(theta)
        _lib.call("lre_theta_relayout", theta.data_ptr(), _lib.NATURAL, n, mm.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        full = lre.step_two_assemble(theta, as_tensor=True)
        del theta
        S = d // 8
        out = torch.empty((d, S), dtype=torch.complex128, device="cuda")
        rows = torch.arange(d, device="cuda")
        for g_ in (0, 5, 7):
            _lib.call("lre_assemble", mm[g_ * S * d:].data_ptr(), _lib.MASK_MAJOR, n, g_ * S, (g_ + 1) * S,
                      out.data_ptr(), torch.cuda.current_stream().cuda_stream)
            cols = (((rows // S) ^ g_) * S)[:, None] + torch.arange(S, device="cuda")[None, :]
            assert torch.equal(out, torch.gather(full, 1, cols))
