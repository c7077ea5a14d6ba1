"""Error metrics against values computed by the
reference's own metrics.py on the reference's own reconstructions
(tests/golden/metrics.npz, make_golden.py metrics_cases)."""

import json

import numpy as np
import pytest

from conftest import golden

import paper_1602_08604_b200 as lre
from paper_1602_08604_b200 import metrics as M

G = golden("metrics.npz")
REPORTS = json.loads(str(G["reports"]))
PREDS = json.loads(str(G["preds"]))
FIDS = json.loads(str(G["fids"]))
TOL = 1e-10


def close(a, b, tol=TOL):
    return abs(a - b) <= tol * max(1.0, abs(b))


class TestHostForms:
    @pytest.mark.parametrize("label", sorted(PREDS))
    def test_dense_predictor_closed_form_matches_reference(self, label):
        assert close(M.predicted_mse_dense(G[f"pred_{label}_rho"], 37.0), PREDS[label])

    def test_max_mixed_closed_forms(self):
        assert close(M.predicted_mse_max_mixed(4, 40.0), REPORTS["maxmixed4"]["predicted_hs"])
        assert close(M.predicted_infidelity_max_mixed(4, 40.0), REPORTS["maxmixed4"]["predicted_infidelity"])

    def test_dense_predictor_cap(self):
        with pytest.raises(ValueError, match="capped at n=4"):
            M.predicted_mse_dense(np.eye(32) / 32, 10.0)

    def test_report_json_fields(self):
        rep = M.ErrorReport(n=2, n0=3.0, hs_squared_mu=None, hs_squared_rho=0.1, infidelity=0.2,
                            predicted_hs=None, predicted_infidelity=None)
        assert set(json.loads(rep.to_json())) == set(REPORTS["ghz4"]) - {"shots"}


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
class TestDeviceMetrics:
    def test_hs_distance_vs_numpy_and_reproducible(self, torch_cuda):
        rng = np.random.default_rng(0)
        for shape, cplx in [((64, 64), True), ((1000, 3), False), ((1, 1), True), ((4096, 4096), True)]:
            a = rng.standard_normal(shape) + (1j * rng.standard_normal(shape) if cplx else 0)
            b = rng.standard_normal(shape) + (1j * rng.standard_normal(shape) if cplx else 0)
            want = float(np.vdot(a - b, a - b).real)
            got = M.hs_squared_distance(a, b)
            assert close(got, want, 1e-12)
            ta, tb = torch_cuda.from_numpy(a).cuda(), torch_cuda.from_numpy(b).cuda()
            assert M.hs_squared_distance(ta, tb) == M.hs_squared_distance(ta, tb)
        with pytest.raises(ValueError, match="shape mismatch"):
            M.hs_squared_distance(np.zeros((2, 2)), np.zeros((2, 3)))

    @pytest.mark.parametrize("name", sorted(REPORTS))
    def test_evaluate_errors_matches_reference(self, torch_cuda, name):
        r = REPORTS[name]
        kind = "".join(c for c in name if c.isalpha())
        st = lre.StateDescriptor(kind, r["n"], bits=0b101 if kind == "productz" else 0)
        rep = M.evaluate_errors(st, G[f"{name}_rho"], G[f"{name}_mu"], n0=r["n0"])
        for key in ("hs_squared_mu", "hs_squared_rho", "infidelity", "predicted_hs", "predicted_infidelity"):
            if r[key] is None:
                assert getattr(rep, key) is None, key
            else:
                assert close(getattr(rep, key), r[key], 1e-9), (key, getattr(rep, key), r[key])

    def test_fidelities_match_reference(self, torch_cuda):
        for k in range(2):
            assert close(M.fidelity(G[f"fid{k}_a"], G[f"fid{k}_b"], method="general"), FIDS[f"fid{k}"], 1e-9)
            assert close(M.fidelity(G[f"fid{k}_a"], G[f"fid{k}_b"]), FIDS[f"fid{k}"], 1e-9)
        assert close(M.fidelity_with_maxmixed(G["maxmixed_spectrum"], 8), FIDS["maxmixed_spectrum"], 1e-12)
        with pytest.raises(ValueError, match="not Hermitian"):
            M.fidelity(np.array([[0.5, 1.0], [0.0, 0.5]]), np.eye(2) / 2)
        with pytest.raises(ValueError, match="trace"):
            M.fidelity(np.eye(2), np.eye(2) / 2)

    @pytest.mark.parametrize("kind,bits", [("maxmixed", 0), ("ghz", 0), ("productz", 0b10011), ("w", 0)])
    def test_distance_to_state_vs_dense(self, torch_cuda, kind, bits):
        from oracle import lre_oracle as O

        n = 5
        rng = np.random.default_rng(7)
        a = rng.standard_normal((32, 32)) + 1j * rng.standard_normal((32, 32))
        a = (a + a.conj().T) / 64
        truth = O.dense_state(kind, n, bits=bits)
        st = lre.StateDescriptor(kind, n, bits=bits)
        assert close(M.hs_squared_distance_to_state(st, a), float(np.vdot(a - truth, a - truth).real), 1e-12)
        if kind != "maxmixed":
            assert close(M.truth_terms(st, a)[0], float(np.trace(a @ truth).real), 1e-12)

    def test_predicted_mse_state_any_n(self, torch_cuda):
        from paper_1602_08604_b200.simulate import density_matrix

        st = lre.StateDescriptor("ghz", 4)
        assert close(M.predicted_mse_state(st, 11.0), M.predicted_mse_dense(density_matrix(st), 11.0), 1e-12)
        n = 10  # productz: sum_{w,s} p^2 = 2^n in closed form
        want = (5 / 9) ** n * (3**n - 2**n) / (7.0 * 2**n)
        assert close(M.predicted_mse_state(lre.StateDescriptor("productz", n, bits=77), 7.0), want, 1e-12)

    def test_reconstruct_generated_equals_sampled_record(self, torch_cuda):
        st = lre.StateDescriptor("w", 9)
        a = lre.reconstruct_generated(st, 700, 5, project=False, chunk_bytes=1 << 16)
        b = lre.reconstruct(lre.sample_counts(st, 700, seed=5), project=False, as_tensor=True)
        assert torch_cuda.equal(a.theta, b.theta) and torch_cuda.equal(a.mu, b.mu)

    def test_error_scaling_follows_prediction(self, torch_cuda):
        """test_simulate.py:160-172 style: MSE of mu ~ (5/6)^n / N0, slope -1 in N0."""
        rows = M.error_scaling(4, [4, 16, 64], trials=16, seed=3)
        for r in rows:
            assert 0.85 < r["mean_hs_mu"] / r["pred_hs"] < 1.15, r
            assert r["mean_hs_rho"] <= r["mean_hs_mu"] + 1e-12
            assert 0 < r["mean_infidelity"] < 1
        x = np.log([r["N0"] for r in rows])
        y = np.log([r["mean_hs_mu"] for r in rows])
        assert abs(np.polyfit(x, y, 1)[0] + 1) < 0.1
