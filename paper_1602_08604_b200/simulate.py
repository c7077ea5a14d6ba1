"""Synthetic measurement records generated on the device (north-star item 4).

Mirrors the reference's state descriptors and record generators
(simulate.py:26-83 StateDescriptor/parse_state, :224-242 sample_counts,
:245-266 exact_record) with the counts written straight into HBM by
``lre_generate_counts``.  Supported states are the bond-dimension-2 family
maxmixed / ghz / productz / w (W is new relative to the reference; the
reference's dense ``random`` Ginibre states stay a test-side concern).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, pauli
from .records import DeviceRecord, MeasurementRecord, compact_dtype

KINDS = ("maxmixed", "ghz", "productz", "w")


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

    def label(self) -> str:
        if self.kind == "productz":
            return f"productz:{self.bits:0{self.n}b}"
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
    raise ValueError(f"unknown state {text!r}")


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
