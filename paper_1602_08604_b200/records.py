"""Measurement records: the counts-in boundary of the LRE path.

``MeasurementRecord`` mirrors the reference container (records.py:23-64):
per-setting outcome counts (3^n, 2^n) in any integer dtype, validated with
the reference's exact messages.  ``DeviceRecord`` is the B200-native form:
the same record with its counts already resident in HBM as a torch CUDA
tensor (uint8/uint16/int32/int64), validated on the device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, pauli

_NP_DTYPES = {np.dtype(np.uint8): _lib.U8, np.dtype(np.uint16): _lib.U16,
              np.dtype(np.int32): _lib.I32, np.dtype(np.int64): _lib.I64}


def lre_dtype_of(dtype) -> int:
    """Map a numpy/torch integer dtype to the ABI's lre_dtype."""
    import torch

    torch_map = {torch.uint8: _lib.U8, torch.uint16: _lib.U16, torch.int32: _lib.I32, torch.int64: _lib.I64}
    if isinstance(dtype, torch.dtype):
        if dtype not in torch_map:
            raise ValueError(f"counts must be uint8/uint16/int32/int64 on the device, got {dtype}")
        return torch_map[dtype]
    dt = np.dtype(dtype)
    if dt not in _NP_DTYPES:
        raise ValueError(f"counts must be integers, got dtype {dt}")
    return _NP_DTYPES[dt]


def compact_dtype(shots: int):
    """Narrowest unsigned count dtype that holds `shots` (the B200 record format)."""
    if shots <= 0xFF:
        return np.uint8
    if shots <= 0xFFFF:
        return np.uint16
    if shots <= 0x7FFFFFFF:
        return np.int32
    return np.int64


def _bad_row_message(n: int, w: int, total: int, shots: int) -> str:
    # records.py:47-54
    return f"setting {pauli.setting_label(w, n)} (index {w}) sums to {total}, expected {shots}"


@dataclass
class MeasurementRecord:
    """Per-setting outcome counts for all 3**n Pauli settings (records.py:23-64)."""

    n: int
    shots: int
    counts: np.ndarray  # (3**n, 2**n) integer
    seed: int | None = None
    state: str | None = None
    _validated: bool = field(default=False, repr=False, compare=False)

    def validate(self) -> "MeasurementRecord":
        """Same checks and messages as records.py:34-56 (host-side container check)."""
        if self._validated:
            return self
        n = pauli.check_qubit_count(self.n)
        if self.shots < 1:
            raise ValueError(f"shots must be >= 1, got {self.shots}")
        expected = (3**n, 1 << n)
        if tuple(self.counts.shape) != expected:
            raise ValueError(f"counts shape {self.counts.shape} != {expected} for n={n}")
        if not np.issubdtype(self.counts.dtype, np.integer):
            raise ValueError(f"counts must be integers, got dtype {self.counts.dtype}")
        if self.counts.min() < 0:
            raise ValueError("counts must be non-negative")
        sums = self.counts.sum(axis=1, dtype=np.int64)
        bad = np.nonzero(sums != self.shots)[0]
        if bad.size:
            w = int(bad[0])
            raise ValueError(_bad_row_message(n, w, int(sums[w]), self.shots))
        self._validated = True
        return self

    @property
    def num_settings(self) -> int:
        return 3**self.n

    def frequencies(self, start: int, stop: int) -> np.ndarray:
        """records.py:62-64."""
        return self.counts[start:stop] / float(self.shots)


@dataclass
class DeviceRecord:
    """A measurement record whose counts live in HBM (torch CUDA tensor)."""

    n: int
    shots: int
    counts: "object"  # torch.Tensor (rows, 2**n) on CUDA; rows = w_end - w_begin
    w_begin: int = 0
    seed: int | None = None
    state: str | None = None
    _validated: bool = field(default=False, repr=False, compare=False)

    @property
    def num_settings(self) -> int:
        return 3**self.n

    @property
    def w_end(self) -> int:
        return self.w_begin + int(self.counts.shape[0])

    @property
    def lre_dtype(self) -> int:
        return lre_dtype_of(self.counts.dtype)

    def validate(self, stream=None) -> "DeviceRecord":
        """records.py:34-56 evaluated on the device (lre_validate_counts)."""
        import torch

        if self._validated:
            return self
        n = pauli.check_qubit_count(self.n)
        if self.shots < 1:
            raise ValueError(f"shots must be >= 1, got {self.shots}")
        rows = int(self.counts.shape[0])
        if self.counts.dim() != 2 or int(self.counts.shape[1]) != 1 << n or self.w_end > 3**n:
            raise ValueError(f"counts shape {tuple(self.counts.shape)} != {(3**n, 1 << n)} for n={n}")
        if not self.counts.is_cuda or not self.counts.is_contiguous():
            raise ValueError("device counts must be a contiguous CUDA tensor")
        dt = self.lre_dtype
        res = torch.empty(3, dtype=torch.int64, device=self.counts.device)
        stream = stream if stream is not None else torch.cuda.current_stream(self.counts.device)
        _lib.call("lre_validate_counts", self.counts.data_ptr(), dt, n, rows, int(self.shots), res.data_ptr(),
                  stream.cuda_stream)
        first_bad, bad_sum, min_value = (int(x) for x in res.cpu().tolist())
        if min_value < 0:
            raise ValueError("counts must be non-negative")
        if first_bad != (1 << 63) - 1:
            raise ValueError(_bad_row_message(n, self.w_begin + first_bad, bad_sum, self.shots))
        self._validated = True
        return self

    def to_host(self) -> MeasurementRecord:
        if self.w_begin != 0 or self.w_end != 3**self.n:
            raise ValueError("only a full-range device record converts to a MeasurementRecord")
        return MeasurementRecord(n=self.n, shots=self.shots, counts=self.counts.cpu().numpy(), seed=self.seed,
                                 state=self.state)


@dataclass
class OutcomeRecord:
    """A sampled record as raw shots: ``outcomes[w, k]`` is the outcome (bits,
    qubit 1 most significant, bit 1 = eigenvalue -1) of shot k of setting w.

    Record ingestion at scale: 2 bytes per shot instead
    of 2^n counts per setting (n = 14, 1000 shots: 9.6 GB instead of 157 GB
    of uint16 counts).  ``outcomes`` is a numpy array (host) or a CUDA tensor
    (device), uint16, shape (rows, shots) for settings [w_begin, w_begin+rows).
    The device turns it into dense counts (``lre_counts_from_outcomes``);
    ``to_counts()`` does the same on the host (numpy) for checking.
    """

    n: int
    shots: int
    outcomes: "object"
    w_begin: int = 0
    seed: int | None = None
    state: str | None = None

    @property
    def num_settings(self) -> int:
        return 3**self.n

    def to_counts(self) -> MeasurementRecord:
        o = self.outcomes.cpu().numpy() if hasattr(self.outcomes, "cpu") else np.asarray(self.outcomes)
        d = 1 << self.n
        rows = o.shape[0]
        flat = (np.arange(rows, dtype=np.int64)[:, None] * d + o.astype(np.int64)).ravel()
        counts = np.bincount(flat, minlength=rows * d).reshape(rows, d).astype(compact_dtype(self.shots))
        if self.w_begin != 0 or rows != 3**self.n:
            raise ValueError("only a full-range outcome record converts to a MeasurementRecord")
        return MeasurementRecord(n=self.n, shots=self.shots, counts=counts, seed=self.seed, state=self.state)
