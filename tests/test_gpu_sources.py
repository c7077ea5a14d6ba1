"""The reference's source protocol on the B200 path (pipeline.py:42-59,84): ExactFrequencies
for any state, duck-typed `.frequencies(a, b)` sources, and the simulate helpers the
reference exports (dense_matrix, dense_to_theta, exact_probabilities,
theta_to_probabilities) — pinned to fixtures the REAL reference wrote
(tests/golden/exact_sources.npz, make_golden.py exact_sources).  Needs a GPU."""

import numpy as np
import pytest

from conftest import golden, random_counts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import c_oracle as C  # noqa: E402
from oracle import lre_oracle as O  # noqa: E402

TOL = 1e-10
CASES = [("random", 2, 11), ("random", 4, 0), ("random", 5, 7), ("ghz", 3, 0), ("maxmixed", 3, 0)]


@pytest.fixture(scope="module")
def lre():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1602_08604_b200 as lre

    return lre


class DuckSource:
    """A plain streaming source: only .n, .num_settings and .frequencies(a, b)."""

    def __init__(self, n, block):
        self.n, self.num_settings, self.block, self.calls = n, 3**n, block, 0

    def frequencies(self, a, b):
        self.calls += 1
        return self.block(a, b)


@pytest.mark.parametrize("kind,n,seed", CASES)
def test_exact_frequencies_vs_reference(lre, kind, n, seed):
    g = golden("exact_sources.npz")
    tag = f"{kind}{n}_{seed}"
    st = lre.StateDescriptor(kind, n, state_seed=seed)
    for src in (lre.ExactFrequencies(st), st):  # the reference wraps a StateDescriptor itself
        res = lre.reconstruct(src)
        assert O.rel_frobenius(res.theta, g[f"{tag}_theta"]) < TOL
        assert O.rel_frobenius(res.mu, g[f"{tag}_mu"]) < TOL
        assert O.rel_frobenius(res.rho, g[f"{tag}_rho"]) < TOL
        np.testing.assert_allclose(res.eigenvalues, g[f"{tag}_eigenvalues"], atol=1e-12)
    np.testing.assert_allclose(lre.probabilities_block(st, 0, 3**n), g[f"{tag}_probs"], atol=1e-15)
    np.testing.assert_allclose(lre.ExactFrequencies(st).frequencies(2, 3**n - 1), g[f"{tag}_probs"][2:-1], atol=1e-15)
    theta = lre.step_one_least_squares(lre.ExactFrequencies(st))
    assert O.rel_frobenius(theta, g[f"{tag}_theta"]) < TOL


def test_duck_typed_source_matches_reference(lre):
    g = golden("exact_sources.npz")
    probs = g["random4_0_probs"]
    src = DuckSource(4, lambda a, b: probs[a:b])
    res = lre.reconstruct(src)
    assert src.calls >= 1
    assert O.rel_frobenius(res.theta, g["random4_0_theta"]) < TOL
    assert O.rel_frobenius(res.mu, g["random4_0_mu"]) < TOL


def test_simulate_helpers_vs_reference(lre):
    g = golden("exact_sources.npz")
    st = lre.StateDescriptor("random", 3, state_seed=5)
    theta = lre.dense_to_theta(lre.dense_matrix(st))
    assert isinstance(theta, np.ndarray)
    assert O.rel_frobenius(theta, g["random3_5_dense_theta"]) < 1e-13
    np.testing.assert_allclose(lre.theta_to_probabilities(theta, 7, 3), g["random3_5_p_w7"], atol=1e-15)
    np.testing.assert_allclose(lre.exact_probabilities(lre.StateDescriptor("ghz", 3), 5), g["ghz3_p_w5"], atol=0)
    with pytest.raises(ValueError, match="not Hermitian"):
        lre.dense_to_theta(np.array([[0.5, 1.0], [0.0, 0.5]], dtype=complex))
    with pytest.raises(ValueError, match="negative probability"):
        lre.theta_to_probabilities(np.array([2 ** -0.5, 0, 0, 3.0]), 2, 1)


@pytest.mark.parametrize("n,chunk_bytes", [(8, 3**6 * 256 * 8), (9, 3**6 * 512 * 8 * 3), (12, 1 << 28)])
def test_streamed_frequencies_equal_integer_path(lre, n, chunk_bytes, rng):
    """counts / shots streamed as fp64 frequency blocks (several chunks, pinned H2D on a
    copy stream, fp64 folds) reproduce the exact-integer path's theta."""
    shots = 1000
    if n == 12:
        rec = lre.sample_counts(lre.StateDescriptor("ghz", n), shots, seed=3)
        counts = rec.counts.cpu().numpy()
    else:
        counts = random_counts(rng, n, shots, np.uint16)
    src = DuckSource(n, lambda a, b: counts[a:b] / float(shots))
    plan = lre.F64Plan(n, chunk_bytes=chunk_bytes)
    s = torch.cuda.current_stream()
    plan.step1(src, s)
    assert src.calls == -(-3**n // plan.chunk_rows)
    if n < 12:
        assert src.calls >= 3
    ref = lre.step_one_least_squares(lre.MeasurementRecord(n=n, shots=shots, counts=counts))
    got = plan.theta_natural().cpu().numpy()
    assert O.rel_frobenius(got, ref) < 1e-13
    plan.step2(s)
    mu_ref = C.step_two(ref, n) if n <= 10 else None
    if mu_ref is not None:
        assert O.rel_frobenius(plan.mu.cpu().numpy(), mu_ref) < TOL


def test_median_step_times_call_pattern(lre):
    """bench.median_step_times (reference bench.py:18-37) runs unchanged against the drop-in."""
    for n in (3, 5):
        t = lre.reconstruct(lre.ExactFrequencies(lre.StateDescriptor("maxmixed", n)), workers=1,
                            kernel="fast").timings
        assert {"t_step1_s", "t_step2_s", "t_step3_s", "t_total_s"} <= set(t)
