"""Host-side index helpers of the Pauli basis (reference pauli.py subset).

Only what the host needs for argument checking and messages; all per-entry
index arithmetic of the hot path happens inside the CUDA kernels.
Conventions (reference pauli.py:1-13): qubit 1 is the most significant
digit/bit; setting digits X=1, Y=2, Z=3; basis digits I,X,Y,Z = 0..3.
"""

from __future__ import annotations

MAX_QUBITS = 16  # pauli.py:17
AXIS_CHARS = "XYZ"


def check_qubit_count(n) -> int:
    """pauli.py:27-36 (same message)."""
    n = int(n)
    if not 1 <= n <= MAX_QUBITS:
        raise ValueError(f"qubit count must be in [1, {MAX_QUBITS}], got {n}")
    return n


def dimension(n: int) -> int:
    return 1 << check_qubit_count(n)


def num_settings(n: int) -> int:
    return 3 ** check_qubit_count(n)


def num_basis_ops(n: int) -> int:
    return 4 ** check_qubit_count(n)


def setting_digits(w: int, n: int) -> tuple[int, ...]:
    """pauli.py:73-87."""
    n = check_qubit_count(n)
    if not 0 <= w < 3**n:
        raise ValueError(f"setting index {w} out of range for n={n}")
    out = []
    for _ in range(n):
        out.append(w % 3 + 1)
        w //= 3
    return tuple(reversed(out))


def setting_label(w: int, n: int) -> str:
    """pauli.py:99-101, e.g. ``XZY``."""
    return "".join(AXIS_CHARS[d - 1] for d in setting_digits(w, n))


def parse_setting_label(label: str) -> int:
    """pauli.py:104-111."""
    try:
        digits = [AXIS_CHARS.index(c) + 1 for c in label]
    except ValueError:
        raise ValueError(f"setting label {label!r} has characters outside X/Y/Z") from None
    if not digits:
        raise ValueError("empty setting label")
    w = 0
    for d in digits:
        w = w * 3 + (d - 1)
    return w


def basis_index(digits) -> int:
    """pauli.py:58-65."""
    i = 0
    for d in digits:
        if not 0 <= d <= 3:
            raise ValueError(f"basis digit {d} not in {{0..3}}")
        i = (i << 2) | int(d)
    return i


def basis_digits(i: int, n: int) -> tuple[int, ...]:
    """pauli.py:51-55."""
    n = check_qubit_count(n)
    if not 0 <= i < 4**n:
        raise ValueError(f"basis index {i} out of range for n={n}")
    return tuple((i >> (2 * (n - 1 - k))) & 3 for k in range(n))


def mask_major_index(i: int, n: int) -> int:
    """Natural basis index -> m * 2**n + a (m = X|Y bits, a = Y|Z bits)."""
    m = a = 0
    for d in basis_digits(i, n):
        m = (m << 1) | (1 if d in (1, 2) else 0)
        a = (a << 1) | (1 if d in (2, 3) else 0)
    return (m << n) | a
