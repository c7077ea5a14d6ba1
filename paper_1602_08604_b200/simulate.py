"""Synthetic measurement records generated on the device (north-star item 4).

Mirrors the reference's state descriptors and record generators
(simulate.py:26-83 StateDescriptor/parse_state, :224-242 sample_counts,
:245-266 exact_record) with the counts written straight into HBM by
``lre_generate_counts``.  Supported states are the bond-dimension-2 family
maxmixed / ghz / productz / w (W is new relative to the reference), drawn
directly from their closed forms, and any dense state — the reference's
``random`` Ginibre states included — through its Pauli coefficients on the
device (``lre_dense_to_theta`` + ``lre_generate_counts_theta``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, pauli
from .records import DeviceRecord, MeasurementRecord, compact_dtype

KINDS = ("maxmixed", "ghz", "productz", "w", "random")
RANDOM_STATE_MAX_QUBITS = 8  # simulate.py:18 (dense Ginibre draw on the host)
DENSE_MAX_QUBITS = 12  # simulate.py:19 (dense-state generator / lre_dense_to_theta)


@dataclass(frozen=True)
class StateDescriptor:
    """A true state the device generator knows how to measure (simulate.py:26-57)."""

    kind: str
    n: int
    bits: int = 0
    state_seed: int = 0

    def __post_init__(self):
        n = pauli.check_qubit_count(self.n)
        if self.kind not in KINDS:
            raise ValueError(f"unknown state kind {self.kind!r}")
        if self.kind == "productz" and not 0 <= self.bits < (1 << n):
            raise ValueError(f"productz bits {self.bits} out of range for n={n}")
        if self.kind == "random" and n > RANDOM_STATE_MAX_QUBITS:
            raise ValueError(
                f"random states need dense {2**n}x{2**n} storage; capped at n={RANDOM_STATE_MAX_QUBITS}"
            )

    def label(self) -> str:
        if self.kind == "productz":
            return f"productz:{self.bits:0{self.n}b}"
        if self.kind == "random":
            return f"random:{self.state_seed}"
        return self.kind

    @property
    def dyadic(self) -> bool:
        """Outcome probabilities have denominators dividing 2**n (exact records exist)."""
        return self.kind in ("maxmixed", "ghz", "productz")


def parse_state(text: str, n: int) -> StateDescriptor:
    """maxmixed | ghz | w | productz:<bits> (simulate.py:60-83)."""
    n = pauli.check_qubit_count(n)
    name, _, arg = text.partition(":")
    name = name.strip().lower()
    if name in ("maxmixed", "ghz", "w"):
        if arg:
            raise ValueError(f"state {name!r} takes no argument")
        return StateDescriptor(name, n)
    if name == "productz":
        if arg and set(arg) <= {"0", "1"}:
            if len(arg) != n:
                raise ValueError(f"productz bit string {arg!r} must have length n={n}")
            return StateDescriptor("productz", n, bits=int(arg, 2))
        try:
            return StateDescriptor("productz", n, bits=int(arg))
        except ValueError:
            raise ValueError(f"bad productz argument {arg!r}") from None
    if name == "random":
        try:
            return StateDescriptor("random", n, state_seed=int(arg))
        except ValueError:
            raise ValueError(f"bad random-state seed {arg!r}") from None
    raise ValueError(f"unknown state {text!r}")


def density_matrix(state: StateDescriptor) -> np.ndarray:
    """Dense rho of a state on the host (simulate.py:86-111); n <= DENSE_MAX_QUBITS."""
    n = state.n
    if n > DENSE_MAX_QUBITS:
        raise ValueError(f"dense matrix at n={n} exceeds the {DENSE_MAX_QUBITS}-qubit cap")
    d = 1 << n
    if state.kind == "maxmixed":
        return np.eye(d, dtype=np.complex128) / d
    if state.kind == "random":
        # Ginibre ensemble G G^dag / Tr, G with iid standard complex normal
        # entries from numpy's default_rng(state_seed) (simulate.py:105-111)
        rng = np.random.default_rng(state.state_seed)
        g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        rho = g @ g.conj().T
        return rho / np.trace(rho).real
    psi = np.zeros(d, dtype=np.complex128)
    if state.kind == "ghz":
        psi[0] = psi[d - 1] = 1.0 / np.sqrt(2.0)
    elif state.kind == "productz":
        psi[state.bits] = 1.0
    else:  # w
        psi[[1 << k for k in range(n)]] = 1.0 / np.sqrt(n)
    return np.outer(psi, psi.conj())


def dense_to_theta(rho, hermitian_tol: float = 1e-10, *, device=None, stream=None, as_tensor=None):
    """Pauli coefficients theta_i = Tr(rho Omega_i) (NATURAL order, fp64) of a dense
    Hermitian 2^n x 2^n matrix, computed on the device by lre_dense_to_theta (the
    inverse of step (ii)); replaces simulate.py:114-138 with its Hermiticity check and
    message.  Returns numpy for numpy input (the reference's type), a CUDA tensor for
    tensor input or as_tensor=True."""
    import torch

    if as_tensor is None:
        as_tensor = isinstance(rho, torch.Tensor)
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    r = rho if isinstance(rho, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rho, dtype=np.complex128))
    r = r.to(device=device, dtype=torch.complex128).contiguous()
    d = int(r.shape[0])
    n = d.bit_length() - 1
    if r.dim() != 2 or int(r.shape[1]) != d or (1 << n) != d:
        raise ValueError(f"expected a square 2**n x 2**n matrix, got {tuple(r.shape)}")
    pauli.check_qubit_count(n)
    if n > DENSE_MAX_QUBITS:
        raise ValueError(f"dense matrix at n={n} exceeds the {DENSE_MAX_QUBITS}-qubit cap")
    asym = float((r - r.conj().T).abs().max().item())
    if asym > hermitian_tol:
        raise ValueError(f"matrix is not Hermitian (max asymmetry {asym:.3e})")
    theta = torch.empty(4**n, dtype=torch.float64, device=device)
    stream = stream if stream is not None else torch.cuda.current_stream(device)
    _lib.call("lre_dense_to_theta", r.data_ptr(), n, theta.data_ptr(), stream.cuda_stream)
    return theta if as_tensor else theta.cpu().numpy()


NEGATIVE_PROBABILITY_TOL = 1e-8  # simulate.py:22
PROBABILITY_SUM_TOL = 1e-8  # simulate.py:23


def theta_probabilities(theta, n: int, start: int, stop: int, clip: bool, out=None, stream=None):
    """Device (start..stop) x 2^n outcome probabilities of the state with Pauli
    coefficients theta (device, NATURAL): lre_theta_probabilities."""
    import torch

    if out is None:
        out = torch.empty((stop - start, 1 << n), dtype=torch.float64, device=theta.device)
    if stop > start:
        stream = stream if stream is not None else torch.cuda.current_stream(theta.device)
        _lib.call("lre_theta_probabilities", theta.data_ptr(), n, int(start), int(stop), 1 if clip else 0,
                  out.data_ptr(), stream.cuda_stream)
    return out


def _check_probabilities(p, what):
    """simulate.py:154-159, same messages."""
    if p.min() < -NEGATIVE_PROBABILITY_TOL:
        raise ValueError(f"{what}: negative probability {p.min():.3e}")
    total = p.sum()
    if abs(total - 1.0) > PROBABILITY_SUM_TOL:
        raise ValueError(f"{what}: probabilities sum to {total!r}, not 1")


def theta_to_probabilities(theta, w: int, n: int) -> np.ndarray:
    """Outcome distribution of setting w for a state given as theta (simulate.py:141-145)."""
    import torch

    t = theta if isinstance(theta, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float64))
    t = t.to(device=torch.device("cuda", torch.cuda.current_device()) if not t.is_cuda else t.device,
             dtype=torch.float64).contiguous()
    p = theta_probabilities(t, n, w, w + 1, clip=False)[0].cpu().numpy()
    _check_probabilities(p, f"setting {pauli.setting_label(w, n)}")
    return p


def probabilities_block(state: StateDescriptor, start: int, stop: int, as_tensor: bool = False):
    """Exact outcome probabilities of settings [start, stop) (simulate.py:167-206), on the
    device: dyadic states (maxmixed, ghz, productz) as their noiseless record / 2^n, any
    other state through its Pauli coefficients, clipped to [0, 1] (n <= 12)."""
    import torch

    n = state.n
    if not 0 <= start <= stop <= 3**n:
        raise ValueError(f"setting range [{start}, {stop}) out of bounds for n={n}")
    dev = torch.device("cuda", torch.cuda.current_device())
    if state.dyadic:
        counts = generate_device_counts(state, 1 << n, exact=True, w_begin=start, w_end=stop, device=dev)
        p = counts.to(torch.float64) / float(1 << n)
    else:
        if n > DENSE_MAX_QUBITS:
            raise ValueError(f"exact probabilities of {state.label()} need its dense matrix; capped at "
                             f"n={DENSE_MAX_QUBITS}")
        p = theta_probabilities(state_theta(state, dev), n, start, stop, clip=True)
    return p if as_tensor else p.cpu().numpy()


def exact_probabilities(state: StateDescriptor, w: int) -> np.ndarray:
    """Exact outcome distribution of one setting (simulate.py:209-213)."""
    if not 0 <= w < 3**state.n:
        raise ValueError(f"setting index {w} out of range for n={state.n}")
    return probabilities_block(state, w, w + 1)[0]


_THETA_CACHE: dict = {}


def state_theta(state: StateDescriptor, device=None):
    """Device theta of a state through its dense matrix (cached per state and device)."""
    import torch

    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (state, str(device))
    if key not in _THETA_CACHE:
        _THETA_CACHE.clear()  # one state at a time: theta is 8 * 4^n bytes
        _THETA_CACHE[key] = dense_to_theta(density_matrix(state), device=device, as_tensor=True)
    return _THETA_CACHE[key]


def generate_counts_from_theta(theta, n: int, shots: int, seed: int = 0, w_begin: int = 0, w_end: int | None = None,
                               dtype=None, out=None, stream=None):
    """Counts rows [w_begin, w_end) of the state with Pauli coefficients theta
    (device, NATURAL), drawn on the device (lre_generate_counts_theta)."""
    import torch

    from .records import lre_dtype_of

    w_end = 3**n if w_end is None else int(w_end)
    dtype = compact_dtype(shots) if dtype is None else dtype
    if out is None:
        out = torch.empty((w_end - w_begin, 1 << n), dtype=_torch_dtype(dtype), device=theta.device)
    stream = stream if stream is not None else torch.cuda.current_stream(theta.device)
    _lib.call("lre_generate_counts_theta", theta.data_ptr(), n, int(shots), int(seed) & 0xFFFFFFFFFFFFFFFF,
              int(w_begin), int(w_end), out.data_ptr(), lre_dtype_of(out.dtype), stream.cuda_stream)
    return out


def sample_counts_from_density(rho, shots: int, seed: int, dtype=None, device=None) -> DeviceRecord:
    """Sampled record of an arbitrary dense state (n <= 12), drawn on the device."""
    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    theta = dense_to_theta(rho, device=device, as_tensor=True)
    n = (int(theta.shape[0]).bit_length() - 1) // 2
    counts = generate_counts_from_theta(theta, n, shots, seed, dtype=dtype)
    return DeviceRecord(n=n, shots=shots, counts=counts, seed=seed, state="dense")


def _torch_dtype(np_dtype):
    import torch

    return {np.uint8: torch.uint8, np.uint16: torch.uint16, np.int32: torch.int32,
            np.int64: torch.int64}[np.dtype(np_dtype).type]


def generate_device_counts(state: StateDescriptor, shots: int, seed: int = 0, exact: bool = False,
                           w_begin: int = 0, w_end: int | None = None, dtype=None, device=None,
                           out=None, stream=None):
    """Counts rows [w_begin, w_end) written on the device; returns the tensor."""
    import torch

    n = state.n
    w_end = 3**n if w_end is None else int(w_end)
    dtype = compact_dtype(shots) if dtype is None else dtype
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if out is None:
        out = torch.empty((w_end - w_begin, 1 << n), dtype=_torch_dtype(dtype), device=device)
    stream = stream if stream is not None else torch.cuda.current_stream(device)
    from .records import lre_dtype_of

    if state.kind == "random":
        if exact:
            raise ValueError(
                f"state {state.label()} has non-dyadic probabilities; an exact integer record does not exist"
            )
        return generate_counts_from_theta(state_theta(state, device), n, shots, seed, w_begin, w_end, out=out,
                                          stream=stream)
    try:
        _lib.call("lre_generate_counts", _lib.STATE_KINDS[state.kind], n, int(state.bits), int(shots),
                  int(seed) & 0xFFFFFFFFFFFFFFFF, 1 if exact else 0, int(w_begin), int(w_end), out.data_ptr(),
                  lre_dtype_of(out.dtype), stream.cuda_stream)
    except ValueError:
        if exact:
            raise ValueError(
                f"state {state.label()} has non-dyadic probabilities; an exact integer record does not exist"
            ) from None
        raise
    return out


def sample_counts(state: StateDescriptor, shots: int, seed: int, dtype=None, device=None) -> DeviceRecord:
    """One multinomial of `shots` per setting, drawn on the device (simulate.py:224-242)."""
    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    counts = generate_device_counts(state, shots, seed=seed, dtype=dtype, device=device)
    return DeviceRecord(n=state.n, shots=shots, counts=counts, seed=seed, state=state.label())


def exact_record(state: StateDescriptor, dtype=None, device=None) -> DeviceRecord:
    """Noiseless record with shots = 2**n (simulate.py:245-266)."""
    shots = 1 << state.n
    counts = generate_device_counts(state, shots, exact=True, dtype=dtype, device=device)
    return DeviceRecord(n=state.n, shots=shots, counts=counts, seed=None, state=state.label())


def to_host_record(rec: DeviceRecord) -> MeasurementRecord:
    return rec.to_host()


def generate_device_outcomes(state: StateDescriptor, shots: int, seed: int = 0, w_begin: int = 0,
                             w_end: int | None = None, device=None, out=None, stream=None):
    """Outcome lists of settings [w_begin, w_end) on the device (uint16, rows x shots), drawn
    with the same Philox stream as generate_device_counts (their histogram is that record)."""
    import torch

    n = state.n
    if state.kind not in _lib.STATE_KINDS:
        raise ValueError(f"outcome lists are generated for {sorted(_lib.STATE_KINDS)} states, not {state.label()}")
    w_end = 3**n if w_end is None else int(w_end)
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if out is None:
        out = torch.empty((w_end - w_begin, int(shots)), dtype=torch.uint16, device=device)
    stream = stream if stream is not None else torch.cuda.current_stream(device)
    _lib.call("lre_generate_outcomes", _lib.STATE_KINDS[state.kind], n, int(state.bits), int(shots),
              int(seed) & 0xFFFFFFFFFFFFFFFF, int(w_begin), int(w_end), out.data_ptr(), stream.cuda_stream)
    return out


def sample_outcomes(state: StateDescriptor, shots: int, seed: int, device=None):
    """OutcomeRecord drawn on the device (the raw-shot form of sample_counts)."""
    from .records import OutcomeRecord

    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    outcomes = generate_device_outcomes(state, shots, seed=seed, device=device)
    return OutcomeRecord(n=state.n, shots=shots, outcomes=outcomes, seed=seed, state=state.label())


dense_matrix = density_matrix  # the reference's name (simulate.py:86)
