"""Error metrics and the error sweep on the device.

Same names, arguments and results as the reference's metrics.py (and
bench.error_scaling), evaluated where the estimate lives: the squared
Hilbert-Schmidt distance and the maxmixed fidelity are deterministic fp64
reductions over HBM (``lre_reduce``), distances and fidelities to the
generator's true states use their sparse state vectors (``lre_truth_terms``),
so an n = 14 estimate (4 GB) is never copied to the host or compared against
a dense 4 GB truth.  General dense fidelities use the eigensolver of step
(iii) (cuSOLVER through torch.linalg, library code).

The dense MSE predictor has a closed form here.  Every row of the reference's
X (X^T X)^-1 has squared norm (5/9)^n (support of a setting = the 2^n Paulis
on its identity subsets, Gram diagonal 3^zc), so metrics.py:124-154 reduces to
    (5/9)^n (3^n - sum_{w,s} p_ws^2) / (N0 d),   sum_{w,s} p_ws^2 = sum_a 3^zc(a) theta_a^2,
which ``predicted_mse_state`` evaluates for dyadic states at any n from the
exact device record (lre_reduce LRE_REDUCE_SUM_SQ_ZC over its theta).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib, pauli
from .simulate import StateDescriptor

PREDICTOR_DENSE_MAX_QUBITS = 4  # metrics.py:21 (the dense predictor's cap)
_PHYSICAL_TOL = 1e-8  # metrics.py:23


def _torch():
    import torch

    return torch


def _dev_tensor(x, device=None):
    """numpy / torch -> contiguous CUDA tensor (complex128 or float64)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(device or "cuda")
    else:
        a = np.asarray(x)
        if not np.iscomplexobj(a):
            a = a.astype(np.float64, copy=False)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device or "cuda")
    if t.dtype not in (torch.complex128, torch.float64):
        t = t.to(torch.complex128 if t.is_complex() else torch.float64)
    return t.contiguous()


def _as_f64(t):
    torch = _torch()
    return torch.view_as_real(t).reshape(-1) if t.is_complex() else t.reshape(-1)


def _reduce(op: int, a, b=None, scale: float = 1.0) -> float:
    torch = _torch()
    out = torch.empty(1 + _lib.REDUCE_BLOCKS, dtype=torch.float64, device=a.device)
    stream = torch.cuda.current_stream(a.device)
    _lib.call("lre_reduce", op, a.data_ptr(), 0 if b is None else b.data_ptr(), int(a.numel()), float(scale),
              out.data_ptr(), stream.cuda_stream)
    return float(out[0].item())


def hs_squared_distance(a, b) -> float:
    """Squared Hilbert-Schmidt distance Tr((a-b)^2) of two Hermitian matrices (metrics.py:28-35)."""
    if tuple(a.shape) != tuple(b.shape):
        raise ValueError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    ta = _dev_tensor(a)
    tb = _dev_tensor(b, ta.device)
    if ta.is_complex() != tb.is_complex():
        ta, tb = ta.to(_torch().complex128), tb.to(_torch().complex128)
    return _reduce(_lib.REDUCE_SUM_SQ, _as_f64(ta), _as_f64(tb))


def truth_terms(truth: StateDescriptor, a) -> tuple[float, float]:
    """(Re Tr(a rho_true), Tr(rho_true^2)) for a generator state, a on the device."""
    torch = _torch()
    if truth.kind not in _lib.STATE_KINDS:
        raise ValueError(f"state {truth.label()} is not one of the device generator's states")
    ta = _dev_tensor(a).to(torch.complex128)
    d = 1 << truth.n
    if tuple(ta.shape) != (d, d):
        raise ValueError(f"shape mismatch {tuple(ta.shape)} vs {(d, d)}")
    out = torch.empty(2, dtype=torch.float64, device=ta.device)
    _lib.call("lre_truth_terms", ta.data_ptr(), truth.n, _lib.STATE_KINDS[truth.kind], int(truth.bits),
              out.data_ptr(), torch.cuda.current_stream(ta.device).cuda_stream)
    cross, purity = (float(x) for x in out.cpu().tolist())
    return cross, purity


def hs_squared_distance_to_state(truth: StateDescriptor, a) -> float:
    """Tr((a - rho_true)^2) = ||a||^2 - 2 Re Tr(a rho_true) + Tr(rho_true^2), without a dense truth
    (dense states — ``random`` — are compared against their dense matrix)."""
    ta = _dev_tensor(a).to(_torch().complex128)
    if truth.kind not in _lib.STATE_KINDS:
        from .simulate import density_matrix

        return hs_squared_distance(ta, _dev_tensor(density_matrix(truth), ta.device))
    cross, purity = truth_terms(truth, ta)
    return _reduce(_lib.REDUCE_SUM_SQ, _as_f64(ta)) - 2.0 * cross + purity


def fidelity_with_maxmixed(eigenvalues, d: int) -> float:
    """Fidelity of a state (given by its spectrum) with I/d (metrics.py:88-92)."""
    lam = _dev_tensor(eigenvalues)
    if lam.is_complex():
        lam = lam.real.contiguous()
    total = _reduce(_lib.REDUCE_SUM_SQRT, lam.reshape(-1), scale=1.0 / d)
    return float(np.clip(total * total, 0.0, 1.0))


def _require_physical(rho, name: str):
    torch = _torch()
    r = _dev_tensor(rho).to(torch.complex128)
    d = r.shape[0]
    if r.dim() != 2 or r.shape[1] != d:
        raise ValueError(f"{name}: expected a square matrix, got {tuple(r.shape)}")
    if float((r - r.conj().T).abs().max()) > _PHYSICAL_TOL:
        raise ValueError(f"{name}: not Hermitian")
    tr = float(torch.diagonal(r).real.sum())
    if abs(tr - 1.0) > _PHYSICAL_TOL:
        raise ValueError(f"{name}: trace is {tr!r}, not 1")
    if float(torch.linalg.eigvalsh(r)[0]) < -_PHYSICAL_TOL:
        raise ValueError(f"{name}: negative eigenvalues")
    return r


def fidelity(rho, sigma, method: str = "auto") -> float:
    """Uhlmann fidelity Tr^2 sqrt(sqrt(rho) sigma sqrt(rho)) (metrics.py:57-85), on the device."""
    torch = _torch()
    r = _require_physical(rho, "rho")
    s = _require_physical(sigma, "sigma")
    if r.shape != s.shape:
        raise ValueError(f"shape mismatch {tuple(r.shape)} vs {tuple(s.shape)}")
    d = r.shape[0]
    if method not in ("auto", "general"):
        raise ValueError(f"unknown method {method!r}")
    if method == "auto":
        eye = torch.eye(d, dtype=torch.complex128, device=r.device) / d
        if float((r - eye).abs().max()) < 1e-12:
            return fidelity_with_maxmixed(torch.linalg.eigvalsh(s), d)
        purity = float(torch.vdot(r.reshape(-1), r.reshape(-1)).real)
        if purity > 1.0 - 1e-10:
            _, vecs = torch.linalg.eigh(r)
            psi = vecs[:, -1]
            return float(np.clip(float(torch.vdot(psi, s @ psi).real), 0.0, 1.0))
    evals, evecs = torch.linalg.eigh(r)
    root = (evecs * evals.clamp(min=0.0).sqrt()) @ evecs.conj().T
    inner = root @ s @ root
    ev = torch.linalg.eigvalsh((inner + inner.conj().T) / 2.0)
    total = float(ev.clamp(min=0.0).sqrt().sum())
    return float(np.clip(total * total, 0.0, 1.0))


def fidelity_with_state(truth: StateDescriptor, sigma, eigenvalues=None) -> float:
    """F(rho_true, sigma) for a generator state: the spectrum for maxmixed,
    <psi|sigma|psi> for the pure states (the reference's 'auto' shortcuts)."""
    d = 1 << truth.n
    if truth.kind not in _lib.STATE_KINDS:
        from .simulate import density_matrix

        return fidelity(density_matrix(truth), sigma)
    if truth.kind == "maxmixed":
        if eigenvalues is None:
            eigenvalues = _torch().linalg.eigvalsh(_dev_tensor(sigma).to(_torch().complex128))
        return fidelity_with_maxmixed(eigenvalues, d)
    cross, _ = truth_terms(truth, sigma)
    return float(np.clip(cross, 0.0, 1.0))


def predicted_mse_max_mixed(n: int, n0: float) -> float:
    """(5/6)^n / N0 (metrics.py:95-98)."""
    pauli.check_qubit_count(n)
    return (5.0 / 6.0) ** n / n0


def predicted_infidelity_max_mixed(n: int, n0: float) -> float:
    """(5/3)^n / (4 N0) (metrics.py:101-109)."""
    pauli.check_qubit_count(n)
    return (5.0 / 3.0) ** n / (4.0 * n0)


def _predicted_from_sum_p2(n: int, sum_p2: float, n0: float) -> float:
    return (5.0 / 9.0) ** n * (3.0**n - sum_p2) / (n0 * (1 << n))


def _pauli_theta_small(rho: np.ndarray, n: int) -> np.ndarray:
    """theta_a = Tr(rho sigma_a) / sqrt(d) for n <= PREDICTOR_DENSE_MAX_QUBITS (host, tiny)."""
    single = [np.eye(2), np.array([[0, 1], [1, 0]]), np.array([[0, -1j], [1j, 0]]), np.diag([1.0, -1.0])]
    theta = np.empty(4**n)
    for a in range(4**n):
        m = np.ones((1, 1), dtype=np.complex128)
        for q in range(n):
            m = np.kron(m, single[(a >> (2 * (n - 1 - q))) & 3])
        theta[a] = np.real(np.trace(rho @ m)) / np.sqrt(1 << n)
    return theta


def predicted_mse_dense(rho, n0: float) -> float:
    """Dense variance predictor of the mean squared HS distance (metrics.py:124-154),
    in the closed form of the module docstring; same n <= 4 cap as the reference."""
    r = rho.cpu().numpy() if hasattr(rho, "cpu") else np.asarray(rho, dtype=np.complex128)
    d = r.shape[0]
    n = d.bit_length() - 1
    if r.ndim != 2 or r.shape[1] != d or (1 << n) != d:
        raise ValueError(f"expected a square 2**n-dim matrix, got {r.shape}")
    if n > PREDICTOR_DENSE_MAX_QUBITS:
        raise ValueError(f"dense predictor capped at n={PREDICTOR_DENSE_MAX_QUBITS}")
    theta = _pauli_theta_small(r, n)
    zc = np.array([sum(((a >> (2 * q)) & 3) == 0 for q in range(n)) for a in range(4**n)])
    return _predicted_from_sum_p2(n, float((3.0**zc * theta * theta).sum()), n0)


def predicted_mse_state(truth: StateDescriptor, n0: float, device=None) -> float:
    """The same predictor for a dyadic generator state at any n: theta_true is
    step (i) of the exact device record, sum_{w,s} p_ws^2 one lre_reduce."""
    from .pipeline import step_one_least_squares
    from .simulate import exact_record

    theta = step_one_least_squares(exact_record(truth, device=device), device=device, as_tensor=True)
    return _predicted_from_sum_p2(truth.n, _reduce(_lib.REDUCE_SUM_SQ_ZC, theta), n0)


@dataclass
class ErrorReport:
    """Distances between estimates and truth plus their predicted values (metrics.py:157-170)."""

    n: int
    n0: float | None
    hs_squared_mu: float | None
    hs_squared_rho: float
    infidelity: float
    predicted_hs: float | None
    predicted_infidelity: float | None

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=2, sort_keys=True)


def evaluate_errors(truth: StateDescriptor, rho_hat, mu_hat=None, n0: float | None = None,
                    eigenvalues=None) -> ErrorReport:
    """ErrorReport of an estimate against a generator state (metrics.py:173-201).

    ``eigenvalues`` (rho_hat's spectrum, e.g. from step_three_project) saves the
    eigensolve of the maxmixed fidelity."""
    n = truth.n
    hs_mu = hs_squared_distance_to_state(truth, mu_hat) if mu_hat is not None else None
    hs_rho = hs_squared_distance_to_state(truth, rho_hat)
    infid = 1.0 - fidelity_with_state(truth, rho_hat, eigenvalues)
    predicted_hs = predicted_infid = None
    if n0 is not None:
        if truth.kind == "maxmixed":
            predicted_hs = predicted_mse_max_mixed(n, n0)
            predicted_infid = predicted_infidelity_max_mixed(n, n0)
        elif n <= PREDICTOR_DENSE_MAX_QUBITS:
            from .simulate import density_matrix

            predicted_hs = predicted_mse_dense(density_matrix(truth), n0)
    return ErrorReport(n=n, n0=n0, hs_squared_mu=hs_mu, hs_squared_rho=hs_rho, infidelity=infid,
                       predicted_hs=predicted_hs, predicted_infidelity=predicted_infid)


def error_scaling(n: int, n0_values, trials: int, seed: int = 0, workers: int = 1, device=None) -> list[dict]:
    """Mean errors of the maximally mixed state over an N0 grid (reference
    bench.py:125-163, the paper's Fig. 3): same N0 accounting (d*N0 shots per
    setting) and per-trial seeds; records are drawn by the device generator
    and streamed through the pipeline in setting chunks, so n = 14 fits."""
    from .pipeline import reconstruct_generated

    state = StateDescriptor("maxmixed", n)
    d = 1 << n
    rows = []
    for n0 in n0_values:
        hs_mu, hs_rho, infid = [], [], []
        for trial in range(trials):
            trial_seed = ((seed * 1_000_003 + int(n0)) * 1_000_003 + trial) & 0x7FFFFFFFFFFFFFFF
            res = reconstruct_generated(state, d * int(n0), trial_seed, device=device)
            rep = evaluate_errors(state, res.rho, res.mu, eigenvalues=res.eigenvalues)
            hs_mu.append(rep.hs_squared_mu)
            hs_rho.append(rep.hs_squared_rho)
            infid.append(rep.infidelity)
            del res
        rows.append({"N0": int(n0), "mean_hs_mu": float(np.mean(hs_mu)), "mean_hs_rho": float(np.mean(hs_rho)),
                     "mean_infidelity": float(np.mean(infid)), "pred_hs": predicted_mse_max_mixed(n, n0),
                     "pred_infid": predicted_infidelity_max_mixed(n, n0)})
    return rows
