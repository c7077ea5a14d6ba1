"""The CPU oracle pinned against the reference's golden vectors (CPU-only).

Fixtures in tests/golden/ were produced by the REAL reference package
(tests/golden/make_golden.py); these tests prove the oracle restates it
before the oracle is used to check the B200 path.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN_CASES, golden, random_counts
from oracle import c_oracle as C
from oracle import lre_oracle as O

SQ2 = 1.0 / np.sqrt(2.0)


class TestKnownAnswers:
    def test_kat1_kat2_step_one(self):
        g = golden("kat.npz")
        assert np.allclose(O.step_one_least_squares(g["kat1_counts"], 2, n=1), [SQ2, 0, 0, SQ2], atol=1e-15)
        assert np.allclose(O.step_one_least_squares(g["kat2_counts"], 2, n=1), [SQ2, 0, 0, 0], atol=1e-15)
        np.testing.assert_array_equal(O.step_one_least_squares(g["kat1_counts"], 2, n=1), g["kat1_theta"])

    def test_kat4_kat5_step_two(self):
        g = golden("kat.npz")
        np.testing.assert_allclose(O.step_two_assemble(np.array([SQ2, 0, 0, SQ2])), g["kat4_mu"], atol=1e-15)
        np.testing.assert_allclose(O.step_two_assemble(np.array([SQ2, 0, 0, 0])), g["kat5_mu"], atol=1e-15)
        assert np.allclose(g["kat4_mu"], np.diag([1.0, 0.0]))

    def test_kat8_simplex(self):
        g = golden("kat.npz")
        np.testing.assert_allclose(O.project_spectrum_to_simplex([1.02, 0.04, -0.03, -0.03]), g["kat8a"], atol=1e-15)
        np.testing.assert_allclose(O.project_spectrum_to_simplex([0.6, 0.5, -0.1]), g["kat8b"], atol=1e-15)

    @pytest.mark.parametrize("n", [1, 2])
    def test_dense_pseudo_inverse(self, n, rng):
        """SPEC invariant: step (i) == pinv(X) p_hat with X from explicit projectors."""
        d = 1 << n
        sig = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1.0, -1.0])]
        vecs = {0: [np.array([1, 1]) / np.sqrt(2), np.array([1, -1]) / np.sqrt(2)],
                1: [np.array([1, 1j]) / np.sqrt(2), np.array([1, -1j]) / np.sqrt(2)],
                2: [np.array([1, 0]), np.array([0, 1])]}

        def digits(v, b):
            return [(v // b**k) % b for k in reversed(range(n))]

        def kron(ms):
            out = ms[0]
            for m in ms[1:]:
                out = np.kron(out, m)
            return out

        X = []
        for w in range(3**n):
            for s in range(d):
                psi = kron([vecs[a][b].reshape(2, 1) for a, b in zip(digits(w, 3), digits(s, 2))]).ravel()
                P = np.outer(psi, psi.conj())
                X.append([np.trace(P @ (2 ** (-n / 2) * kron([sig[q] for q in digits(i, 4)]))).real
                          for i in range(4**n)])
        X = np.array(X)
        counts = random_counts(rng, n, 777)
        expect = np.linalg.pinv(X) @ (counts / 777.0).ravel()
        np.testing.assert_allclose(O.step_one_least_squares(counts, 777), expect, atol=1e-12)


class TestGoldenVectors:
    @pytest.mark.parametrize("name", GOLDEN_CASES)
    def test_steps_match_reference(self, name):
        g = golden(name)
        n, shots = int(g["n"]), int(g["shots"])
        counts = g["counts"].astype(np.int64)
        theta = O.step_one_least_squares(counts, shots, n=n)
        assert O.rel_frobenius(theta, g["theta"]) < 1e-13
        mu = O.step_two_assemble(g["theta"])
        assert O.rel_frobenius(mu, g["mu"]) < 1e-13
        if "rho" in g:
            rho, ev = O.step_three_project(g["mu"])
            np.testing.assert_allclose(ev, g["eigenvalues"], atol=1e-10)
            assert O.rel_frobenius(rho, g["rho"]) < 1e-9

    @pytest.mark.parametrize("name", GOLDEN_CASES)
    def test_exact_numerators_reproduce_reference(self, name):
        g = golden(name)
        n, shots = int(g["n"]), int(g["shots"])
        num = O.step_one_numerators(g["counts"].astype(np.int64), n)
        assert O.rel_frobenius(O.finalize_numerators(num, n, shots), g["theta"]) < 1e-14

    @pytest.mark.parametrize("name", GOLDEN_CASES)
    def test_c_oracle_matches_numpy_oracle(self, name):
        g = golden(name)
        n, shots = int(g["n"]), int(g["shots"])
        counts = g["counts"]
        np.testing.assert_array_equal(C.numerators(counts, n), O.step_one_numerators(counts.astype(np.int64), n))
        assert O.rel_frobenius(C.step_one(counts, n, shots, threads=3), g["theta"]) < 1e-13
        assert O.rel_frobenius(C.step_two(g["theta"], n, threads=2), g["mu"]) < 1e-13

    def test_index_blocks(self):
        g = golden("blocks_n3.npz")
        n = 3
        np.testing.assert_array_equal(O.setting_digit_rows(0, 27, n), g["digit_rows"])
        np.testing.assert_array_equal(O.nonzero_locations_block(g["digit_rows"], n), g["locs"])
        np.testing.assert_array_equal(np.stack([O.omega_gather_indices(m, n) for m in range(8)]), g["gather"])
        np.testing.assert_array_equal(np.stack([O.omega_phase_factors(m, n) for m in range(8)]), g["phase"])
        np.testing.assert_array_equal(O.xtx_diagonal_full(n), g["xtx"])
        np.testing.assert_allclose(O.walsh_hadamard_transform(g["wht_in"]), g["wht_out"], rtol=1e-14)

    def test_symplectic_layout_matches_gather(self):
        n = 3
        m, a = O.symplectic_index(n)
        for mask in range(1 << n):
            idx = O.omega_gather_indices(mask, n)
            assert np.all(m[idx] == mask) and np.all(a[idx] == np.arange(1 << n))

    def test_c3_generator_hash_and_reference_theta(self):
        """n=10 Ginibre case: the oracle regenerates the reference's counts bit for bit."""
        g = golden("c3_random10.npz")
        n = int(g["n"])
        theta_true = O.dense_to_theta(O.dense_state("random", n, seed=int(g["state_seed"])))
        counts = O.sample_counts_from_theta(theta_true, n, int(g["shots"]), int(g["seed"]))
        assert hashlib.sha256(counts.tobytes()).hexdigest() == str(g["counts_sha256"])
        theta = C.step_one(counts, n, int(g["shots"]))
        st = int(g["theta_stride"])
        np.testing.assert_allclose(theta[::st], g["theta_sample"], rtol=1e-10, atol=1e-16)
        assert abs(np.linalg.norm(theta) - float(g["theta_norm"])) < 1e-12 * float(g["theta_norm"])


class TestValidation:
    def test_messages_match_reference(self):
        g = golden("validate.npz")
        msgs = json.loads(str(g["messages"]))
        with pytest.raises(ValueError) as exc:
            O.validate_counts(g["counts_bad_row"], 2, 50)
        assert str(exc.value) == msgs["bad_row_sum"]
        bad = g["counts_ok"].copy()
        bad[5, 1] = -1
        with pytest.raises(ValueError, match="non-negative"):
            O.validate_counts(bad, 2, 50)
        O.validate_counts(g["counts_ok"], 2, 50)
