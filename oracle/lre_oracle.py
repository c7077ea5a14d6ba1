"""CPU oracle for the LRE hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference package's
linear-regression-estimation path (``/root/reference/pkg/src/pauli_lre``,
"the reference" below).  It exists to *check* the B200 path and to time the
reference algorithm on host cores.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import it.  The product package ``paper_1602_08604_b200`` never imports,
calls or links anything under ``oracle/``.

Parity is PINNED: ``tests/golden/make_golden.py`` imports the real reference
(in the build container, where ``/root/reference`` exists) and records its
outputs for seeded inputs as ``tests/golden/*.npz``; ``tests/test_oracle.py``
checks this restatement against every one of those vectors plus the SPEC
known-answer tests.

Conventions (reference ``pauli.py:1-13``): qubit 1 is the most significant
digit/bit; setting digits X=0,Y=1,Z=2 (axis-1); basis digits I,X,Y,Z=0..3;
outcome bit 0 means eigenvalue +1.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# index arithmetic (reference pauli.py)
# ---------------------------------------------------------------------------

MAX_QUBITS = 16  # pauli.py:17


def check_qubit_count(n) -> int:
    """pauli.py:27-36."""
    n = int(n)
    if not 1 <= n <= MAX_QUBITS:
        raise ValueError(f"qubit count must be in [1, {MAX_QUBITS}], got {n}")
    return n


def setting_digit_rows(start: int, stop: int, n: int) -> np.ndarray:
    """(stop-start, n) axis digits in {1,2,3}, qubit 1 first (pauli.py:212-220)."""
    w = np.arange(start, stop, dtype=np.int64)
    cols = []
    for _ in range(n):
        cols.append(w % 3 + 1)
        w = w // 3
    return np.stack(cols[::-1], axis=1)


def setting_label(w: int, n: int) -> str:
    """pauli.py:99-106 (digits from pauli.py:73-87)."""
    out = []
    for _ in range(n):
        out.append("XYZ"[w % 3])
        w //= 3
    return "".join(reversed(out))


def walsh_hadamard_transform(values: np.ndarray) -> np.ndarray:
    """Unnormalised WHT along the last axis, h = 1 -> m/2 (pauli.py:223-246)."""
    v = np.asarray(values)
    m = v.shape[-1]
    if m == 0 or (m & (m - 1)) != 0:
        raise ValueError(f"length {m} is not a power of two")
    dtype = np.complex128 if np.iscomplexobj(v) else np.float64
    out = v.astype(dtype, copy=True)
    lead = out.shape[:-1]
    h = 1
    while h < m:
        work = out.reshape(*lead, m // (2 * h), 2, h)
        top = work[..., 0, :].copy()
        bot = work[..., 1, :]
        work[..., 0, :] = top + bot
        work[..., 1, :] = top - bot
        h *= 2
    return out


def xtx_diagonal_full(n: int) -> np.ndarray:
    """Gram diagonal 3**zero_count(i) as a Kronecker power (pauli.py:162-169)."""
    base = np.array([3.0, 1.0, 1.0, 1.0])
    full = base
    for _ in range(n - 1):
        full = np.kron(full, base)
    return full


def _outcome_bits(n: int) -> np.ndarray:
    """pauli.py:172-179."""
    s = np.arange(1 << n, dtype=np.int64)
    shifts = n - 1 - np.arange(n, dtype=np.int64)
    return (s[:, None] >> shifts[None, :]) & 1


def nonzero_locations_block(digit_rows: np.ndarray, n: int) -> np.ndarray:
    """Support indices of each setting, ascending in subset mask t (pauli.py:191-209)."""
    place = 4 ** (n - 1 - np.arange(n, dtype=np.int64))
    weights = digit_rows.astype(np.int64) * place[None, :]
    bits = _outcome_bits(n)  # (2**n, n): bit k of t, qubit 1 first
    return weights @ bits.T


def omega_gather_indices(mask: int, n: int) -> np.ndarray:
    """Basis indices sharing antidiagonal mask ``mask`` (pauli.py:270-289)."""
    place = 4 ** (n - 1 - np.arange(n, dtype=np.int64))
    mbits = _outcome_bits(n)[mask]
    base = int((mbits * place).sum())
    coeff = (3 - 2 * mbits) * place
    return base + _outcome_bits(n) @ coeff


_MINUS_I_POWERS = np.array([1.0, -1.0j, -1.0, 1.0j], dtype=np.complex128)  # pauli.py:22


def omega_phase_factors(mask: int, n: int) -> np.ndarray:
    """(-i)**popcount(a & mask) (pauli.py:292-297)."""
    a = np.arange(1 << n, dtype=np.uint64)
    pc = np.bitwise_count(a & np.uint64(mask))
    return _MINUS_I_POWERS[pc & 3]


def symplectic_index(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Natural basis index i -> (m, a): m = X|Y bits, a = Y|Z bits.

    Used only to express the mask-major layout the B200 path keeps
    internally (index m*2**n + a); the natural order is the reference's.
    """
    i = np.arange(4**n, dtype=np.int64)
    m = np.zeros_like(i)
    a = np.zeros_like(i)
    for k in range(n):
        d = (i >> (2 * (n - 1 - k))) & 3
        m = (m << 1) | ((d == 1) | (d == 2))
        a = (a << 1) | ((d == 2) | (d == 3))
    return m, a


# ---------------------------------------------------------------------------
# step (i): counts -> theta (pipeline.py:116-138, _kernels.py:34-56)
# ---------------------------------------------------------------------------

def step_one_least_squares(counts: np.ndarray, shots: int, n: int | None = None,
                           batch_elements: int = 1 << 21) -> np.ndarray:
    """Reference step (i) restated with numpy.

    Frequencies are ``counts / float(shots)`` (records.py:62-64); each
    setting's row is Walsh-Hadamard transformed (_kernels.py:42-53), scaled
    by ``2.0 ** (-n / 2.0)`` (pipeline.py:78) and scatter-added at the
    setting's support locations (_kernels.py:54-56); the sum is divided by
    the Gram diagonal (pipeline.py:138).
    """
    counts = np.asarray(counts)
    if n is None:
        n = int(round(np.log2(counts.shape[1])))
    n = check_qubit_count(n)
    settings = 3**n
    raw = np.zeros(4**n)
    scale = 2.0 ** (-n / 2.0)
    batch = max(1, batch_elements >> n)
    for a in range(0, settings, batch):
        b = min(settings, a + batch)
        freq = counts[a:b] / float(shots)
        e = walsh_hadamard_transform(freq) * scale
        locs = nonzero_locations_block(setting_digit_rows(a, b, n), n)
        np.add.at(raw, locs.ravel(), e.ravel())
    return raw / xtx_diagonal_full(n)


def step_one_numerators(counts: np.ndarray, n: int) -> np.ndarray:
    """Exact int64 numerators N_i = sum_w WHT(counts_w)[t] at i = loc(w, t).

    theta_i = N_i * 2**(-n/2) / (shots * 3**zc(i)).  This is the integer
    form of _kernels.accumulate_fast (_kernels.py:34-56) with frequencies
    replaced by counts; the B200 path must reproduce it bit for bit.
    """
    counts = np.asarray(counts)
    settings = 3**n
    num = np.zeros(4**n, dtype=np.int64)
    batch = max(1, (1 << 20) >> n)
    for a in range(0, settings, batch):
        b = min(settings, a + batch)
        e = counts[a:b].astype(np.int64)
        h = 1
        d = 1 << n
        while h < d:  # integer butterfly, same stage order as _kernels.py:44-53
            work = e.reshape(b - a, d // (2 * h), 2, h)
            top = work[:, :, 0, :].copy()
            bot = work[:, :, 1, :]
            work[:, :, 0, :] = top + bot
            work[:, :, 1, :] = top - bot
            h *= 2
        locs = nonzero_locations_block(setting_digit_rows(a, b, n), n)
        np.add.at(num, locs.ravel(), e.ravel())
    return num


def zero_counts(n: int) -> np.ndarray:
    """zero_count(i) for all i (pauli.py:68-70)."""
    i = np.arange(4**n, dtype=np.int64)
    zc = np.zeros_like(i)
    for k in range(n):
        zc += ((i >> (2 * k)) & 3) == 0
    return zc


def finalize_numerators(num: np.ndarray, n: int, shots: int) -> np.ndarray:
    """theta = ((N / shots) * 2**(-n/2)) / 3**zc — the B200 epilogue's formula."""
    return (num.astype(np.float64) / float(shots)) * (2.0 ** (-n / 2.0)) / xtx_diagonal_full(n)


# ---------------------------------------------------------------------------
# step (ii): theta -> mu (pipeline.py:141-161)
# ---------------------------------------------------------------------------

def step_two_assemble(theta: np.ndarray) -> np.ndarray:
    """Per X-mask gather, (-i)^k phase, complex WHT, XOR-diagonal scatter."""
    theta = np.asarray(theta, dtype=np.float64)
    size = theta.shape[0]
    n = (size.bit_length() - 1) // 2
    if theta.ndim != 1 or size != 4**n:
        raise ValueError(f"theta length {theta.shape} is not 4**n")
    d = 1 << n
    mu = np.empty((d, d), dtype=np.complex128)
    rows = np.arange(d)
    scale = 2.0 ** (-n / 2.0)
    for m in range(d):
        v = theta[omega_gather_indices(m, n)] * omega_phase_factors(m, n)
        mu[rows, rows ^ m] = walsh_hadamard_transform(v) * scale
    return mu


def step_two_masks(theta: np.ndarray, masks) -> np.ndarray:
    """XOR-diagonals mu[r, r^m] for the given masks, shape (len(masks), d)."""
    theta = np.asarray(theta, dtype=np.float64)
    n = (theta.shape[0].bit_length() - 1) // 2
    scale = 2.0 ** (-n / 2.0)
    out = np.empty((len(masks), 1 << n), dtype=np.complex128)
    for j, m in enumerate(masks):
        v = theta[omega_gather_indices(int(m), n)] * omega_phase_factors(int(m), n)
        out[j] = walsh_hadamard_transform(v) * scale
    return out


# ---------------------------------------------------------------------------
# step (iii): projection (pipeline.py:164-208) — adjacent to the hot path
# ---------------------------------------------------------------------------

def project_spectrum_to_simplex(values: np.ndarray) -> np.ndarray:
    """Scan-from-smallest simplex projection (pipeline.py:164-184)."""
    values = np.asarray(values, dtype=np.float64)
    order = np.argsort(values)
    u = values[order]
    k = u.shape[0]
    prefix = np.concatenate(([0.0], np.cumsum(u[:-1])))
    remaining = k - np.arange(k)
    stop = int(np.argmax(u + prefix / remaining >= 0.0))
    out = np.zeros(k)
    out[stop:] = u[stop:] + prefix[stop] / (k - stop)
    inverse = np.empty(k, dtype=np.intp)
    inverse[order] = np.arange(k)
    return out[inverse]


def step_three_project(mu: np.ndarray):
    """eigh + simplex projection; PSD input returned unchanged (pipeline.py:187-208)."""
    evals, evecs = np.linalg.eigh(mu)
    if evals[0] >= 0.0:
        return mu, evals
    lam = project_spectrum_to_simplex(evals)
    return (evecs * lam) @ evecs.conj().T, lam


# ---------------------------------------------------------------------------
# synthetic inputs (simulate.py) — used to build seeded test cases
# ---------------------------------------------------------------------------

def dense_state(kind: str, n: int, seed: int = 0, bits: int = 0) -> np.ndarray:
    """Dense density matrix of a named state (simulate.py:86-111, plus W).

    ``w`` (|W> = n**-1/2 sum_k |0..1_k..0>) is not in the reference; it is
    built the same way as ghz (simulate.py:93-96).
    """
    d = 1 << n
    if kind == "maxmixed":
        return np.eye(d, dtype=np.complex128) / d
    if kind == "ghz":
        psi = np.zeros(d, dtype=np.complex128)
        psi[0] = psi[d - 1] = 1.0 / np.sqrt(2.0)
        return np.outer(psi, psi.conj())
    if kind == "w":
        psi = np.zeros(d, dtype=np.complex128)
        for k in range(n):
            psi[1 << k] = 1.0 / np.sqrt(n)
        return np.outer(psi, psi.conj())
    if kind == "productz":
        rho = np.zeros((d, d), dtype=np.complex128)
        rho[bits, bits] = 1.0
        return rho
    if kind == "random":  # simulate.py:105-111
        rng = np.random.default_rng(seed)
        g = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        rho = g @ g.conj().T
        return rho / np.trace(rho).real
    raise ValueError(f"unknown state kind {kind!r}")


def dense_to_theta(rho: np.ndarray) -> np.ndarray:
    """theta_i = Tr(rho Omega_i) by antidiagonal groups (simulate.py:114-138).

    Works in complex128 throughout (the reference's real-dtype in-place
    multiply bug, simulate.py:135-136, is avoided by construction).
    """
    rho = np.asarray(rho, dtype=np.complex128)
    d = rho.shape[0]
    n = d.bit_length() - 1
    rows = np.arange(d)
    theta = np.empty(4**n)
    scale = 2.0 ** (-n / 2.0)
    for mask in range(d):
        coeff = walsh_hadamard_transform(rho[rows ^ mask, rows])
        coeff = coeff * (scale * omega_phase_factors(mask, n))
        theta[omega_gather_indices(mask, n)] = coeff.real
    return theta


def theta_probability_block(theta: np.ndarray, start: int, stop: int, n: int) -> np.ndarray:
    """Outcome probabilities of settings [start, stop) from theta (simulate.py:148-151)."""
    locs = nonzero_locations_block(setting_digit_rows(start, stop, n), n)
    return 2.0 ** (-n / 2.0) * walsh_hadamard_transform(theta[locs])


def setting_rng(seed: int, w: int) -> np.random.Generator:
    """Philox substream keyed on (seed, setting) (simulate.py:216-221)."""
    key = np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF), np.uint64(w)], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def sample_counts_from_theta(theta: np.ndarray, n: int, shots: int, seed: int,
                             dtype=np.int64) -> np.ndarray:
    """One multinomial of ``shots`` per setting (simulate.py:224-242)."""
    settings = 3**n
    counts = np.empty((settings, 1 << n), dtype=dtype)
    block = max(1, (1 << 18) >> n)
    for start in range(0, settings, block):
        stop = min(settings, start + block)
        probs = np.clip(theta_probability_block(theta, start, stop, n), 0.0, 1.0)
        for row, w in enumerate(range(start, stop)):
            p = np.clip(probs[row], 0.0, None)
            counts[w] = setting_rng(seed, w).multinomial(shots, p / p.sum())
    return counts


def ghz_probabilities_block(start: int, stop: int, n: int) -> np.ndarray:
    """Closed-form GHZ outcome probabilities of settings [start, stop) (simulate.py:183-205)."""
    d = 1 << n
    out = np.zeros((stop - start, d))
    s = np.arange(d, dtype=np.uint64)
    parity = np.bitwise_count(s) & 1
    for row, digits in enumerate(setting_digit_rows(start, stop, n)):
        zmask = sum(1 << (n - 1 - k) for k, dg in enumerate(digits) if dg == 3)
        n_y = int(np.sum(digits == 2))
        if zmask == 0:
            if n_y % 2:
                out[row, :] = 1.0 / d
            else:
                out[row, parity == (n_y // 2) % 2] = 2.0 ** (1 - n)
        else:
            weight = 2.0 ** -(n - bin(zmask).count("1") + 1)
            zpart = s & np.uint64(zmask)
            out[row, zpart == 0] = weight
            out[row, zpart == np.uint64(zmask)] = weight
    return out


def sample_ghz_counts(n: int, shots: int, seed: int, start: int, stop: int, dtype=np.uint16) -> np.ndarray:
    """Settings [start, stop) of a sampled GHZ record (simulate.py:224-242 with the closed form)."""
    probs = ghz_probabilities_block(start, stop, n)
    out = np.empty((stop - start, 1 << n), dtype=dtype)
    for row, w in enumerate(range(start, stop)):
        p = probs[row]
        out[row] = setting_rng(seed, w).multinomial(shots, p / p.sum())
    return out


def exact_counts_from_theta(theta: np.ndarray, n: int) -> np.ndarray:
    """Noiseless dyadic record with shots = 2**n (simulate.py:245-266)."""
    settings = 3**n
    d = 1 << n
    scaled = theta_probability_block(theta, 0, settings, n) * d
    rounded = np.rint(scaled)
    if np.abs(scaled - rounded).max() > 1e-9:
        raise ValueError("non-dyadic probabilities; an exact integer record does not exist")
    return rounded.astype(np.int64)


def validate_counts(counts: np.ndarray, n: int, shots: int) -> None:
    """MeasurementRecord.validate (records.py:34-56), same messages."""
    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    expected = (3**n, 1 << n)
    if tuple(counts.shape) != expected:
        raise ValueError(f"counts shape {counts.shape} != {expected} for n={n}")
    if not np.issubdtype(counts.dtype, np.integer):
        raise ValueError(f"counts must be integers, got dtype {counts.dtype}")
    if counts.min() < 0:
        raise ValueError("counts must be non-negative")
    sums = counts.sum(axis=1)
    bad = np.nonzero(sums != shots)[0]
    if bad.size:
        w = int(bad[0])
        raise ValueError(
            f"setting {setting_label(w, n)} (index {w}) sums to {int(sums[w])}, expected {shots}"
        )


def rel_frobenius(a: np.ndarray, b: np.ndarray) -> float:
    """||a - b||_F / ||b||_F (the north-star parity metric)."""
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
