"""Record and estimate files: the reference's formats plus a binary record
format that scales to n = 14.

* ``pauli-lre/1`` text records — ``write_record`` / ``read_record`` with the
  reference's contract and error messages (records.py:16-163): JSON header,
  then 3^n lines ``<setting label> <c_0>,...,<c_{2^n-1}>`` in setting order.
  Kept for interchange; at n = 14 such a file would be ~0.5 TB of text.
* ``pauli-lre-bin/1`` binary records (this package) — a 256-byte header and
  the raw little-endian rows, either dense counts in the compact dtype (3^n x
  2^n) or raw-shot outcome lists (uint16, 3^n x shots).  ``open_record`` maps
  the file; ``reconstruct_file`` streams it through pinned host buffers into
  the device pipeline (``LREPlan.stage`` / ``stage_outcomes``) so a 157 GB
  record never needs to be resident on the host or the device at once.
* ``PLRE`` v1 estimate files — ``write_state`` / ``read_state`` with the
  reference's byte layout and messages (statefile.py:1-49); device tensors
  are written in row chunks.
"""

from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib, pauli
from .records import DeviceRecord, MeasurementRecord, OutcomeRecord, compact_dtype, lre_dtype_of

RECORD_FORMAT = "pauli-lre/1"
BINARY_FORMAT = "pauli-lre-bin/1"


class RecordFormatError(ValueError):
    """A measurement record file violates the format contract (records.py:19-20)."""


# ---------------------------------------------------------------------------
# pauli-lre/1 text records (records.py:67-163)
# ---------------------------------------------------------------------------

def _host_record(record) -> MeasurementRecord:
    if isinstance(record, DeviceRecord):
        return record.validate().to_host()
    if isinstance(record, OutcomeRecord):
        return record.to_counts()
    return record


def write_record(record, path) -> int:
    """Write a ``pauli-lre/1`` file; returns the bytes written (records.py:67-84).

    Accepts a MeasurementRecord, a DeviceRecord (copied to the host) or an
    OutcomeRecord (histogrammed on the host)."""
    rec = _host_record(record).validate()
    n = rec.n
    header = {"format": RECORD_FORMAT, "n": n, "shots": rec.shots, "seed": rec.seed, "state": rec.state}
    counts = np.asarray(rec.counts)
    with open(path, "w", encoding="utf-8") as fh:
        total = fh.write(json.dumps(header) + "\n")
        for w in range(3**n):
            total += fh.write(pauli.setting_label(w, n) + " " + ",".join(map(str, counts[w].tolist())) + "\n")
    return total


def _header_fields(first_line: str) -> tuple[int, int, dict]:
    try:
        header = json.loads(first_line)
    except json.JSONDecodeError as exc:
        raise RecordFormatError(f"line 1: header is not valid JSON ({exc.msg})") from None
    if not isinstance(header, dict):
        raise RecordFormatError("line 1: header must be a JSON object")
    if header.get("format") != RECORD_FORMAT:
        raise RecordFormatError(f"line 1: unsupported format {header.get('format')!r}, expected {RECORD_FORMAT!r}")
    for key in ("n", "shots"):
        if not isinstance(header.get(key), int):
            raise RecordFormatError(f"line 1: header field {key!r} must be an integer")
    try:
        n = pauli.check_qubit_count(header["n"])
    except ValueError as exc:
        raise RecordFormatError(f"line 1: {exc}") from None
    if header["shots"] < 1:
        raise RecordFormatError(f"line 1: shots must be >= 1, got {header['shots']}")
    return n, header["shots"], header


def read_record(path) -> MeasurementRecord:
    """Parse and validate a ``pauli-lre/1`` file (records.py:87-163); every
    violation raises RecordFormatError naming the line."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise RecordFormatError("empty record file")
    n, shots, header = _header_fields(lines[0])
    settings, d = 3**n, 1 << n
    body = lines[1:]
    while body and not body[-1].strip():
        body.pop()
    if len(body) != settings:
        raise RecordFormatError(f"expected {settings} setting lines for n={n}, found {len(body)}")
    counts = np.empty((settings, d), dtype=np.int64)
    for w, line in enumerate(body):
        lineno = w + 2
        label, sep, payload = line.partition(" ")
        if not sep:
            raise RecordFormatError(f"line {lineno}: expected '<setting> <counts>'")
        want = pauli.setting_label(w, n)
        if label != want:
            raise RecordFormatError(f"line {lineno}: setting {label!r} out of order or invalid, expected {want!r}")
        tokens = payload.split(",")
        if len(tokens) != d:
            raise RecordFormatError(f"line {lineno} (setting {label}): {len(tokens)} counts, expected {d}")
        try:
            row = np.array([int(t) for t in tokens], dtype=np.int64)
        except ValueError:
            raise RecordFormatError(f"line {lineno} (setting {label}): counts must be integers") from None
        if row.min() < 0:
            raise RecordFormatError(f"line {lineno} (setting {label}): negative count")
        total = int(row.sum())
        if total != shots:
            raise RecordFormatError(f"line {lineno} (setting {label}): counts sum to {total}, expected {shots}")
        counts[w] = row
    return MeasurementRecord(n=n, shots=shots, counts=counts, seed=header.get("seed"),
                             state=header.get("state")).validate()


# ---------------------------------------------------------------------------
# pauli-lre-bin/1 binary records
# ---------------------------------------------------------------------------

_BIN_MAGIC = b"PLRB"
_BIN_VERSION = 1
_BIN_HEADER = struct.Struct("<4sIIIIIqqq")  # magic, version, n, layout, dtype, reserved, shots, seed, rows
_BIN_HEADER_BYTES = 256  # struct + utf-8 state label, zero padded
LAYOUT_COUNTS, LAYOUT_OUTCOMES = 0, 1
_DTYPE_NP = {_lib.U8: np.dtype("<u1"), _lib.U16: np.dtype("<u2"), _lib.I32: np.dtype("<i4"),
             _lib.I64: np.dtype("<i8")}
_NO_SEED = -(1 << 63)


@dataclass
class RecordFile:
    """A mapped ``pauli-lre-bin/1`` file: header fields plus ``data``, a
    read-only memmap of shape (3^n, 2^n) counts or (3^n, shots) outcomes."""

    path: str
    n: int
    shots: int
    layout: int
    seed: int | None
    state: str | None
    data: np.memmap

    @property
    def num_settings(self) -> int:
        return 3**self.n

    @property
    def nbytes(self) -> int:
        return int(self.data.nbytes)

    def to_record(self):
        """The whole file as a host MeasurementRecord (counts) or OutcomeRecord."""
        if self.layout == LAYOUT_OUTCOMES:
            return OutcomeRecord(n=self.n, shots=self.shots, outcomes=np.array(self.data), seed=self.seed,
                                 state=self.state)
        return MeasurementRecord(n=self.n, shots=self.shots, counts=np.array(self.data), seed=self.seed,
                                 state=self.state).validate()


def write_record_binary(record, path, chunk_rows: int = 1 << 14) -> int:
    """Write a MeasurementRecord / DeviceRecord (dense counts, compact dtype)
    or an OutcomeRecord (outcome lists) as ``pauli-lre-bin/1``; device data is
    copied to the host in row chunks.  Returns the bytes written."""
    if isinstance(record, OutcomeRecord):
        layout, n, shots = LAYOUT_OUTCOMES, record.n, record.shots
        data, dtype_code = record.outcomes, _lib.U16
        if record.w_begin != 0 or int(data.shape[0]) != 3**n:
            raise ValueError("only a full-range outcome record can be written")
    else:
        if isinstance(record, DeviceRecord):
            record.validate()
            if record.w_begin != 0 or record.w_end != 3**record.n:
                raise ValueError("only a full-range device record can be written")
            data = record.counts
        else:
            record.validate()
            data = np.asarray(record.counts)
            want = np.dtype(compact_dtype(record.shots))
            if data.dtype != want:
                data = data.astype(want)
        layout, n, shots = LAYOUT_COUNTS, record.n, record.shots
        dtype_code = lre_dtype_of(data.dtype)
    label = (record.state or "").encode("utf-8")[: _BIN_HEADER_BYTES - _BIN_HEADER.size]
    seed = _NO_SEED if record.seed is None else int(record.seed)
    head = _BIN_HEADER.pack(_BIN_MAGIC, _BIN_VERSION, n, layout, dtype_code, 0, int(shots), seed, 3**n)
    head = head + label + bytes(_BIN_HEADER_BYTES - len(head) - len(label))
    total = 0
    with open(path, "wb") as fh:
        total += fh.write(head)
        for lo in range(0, 3**n, chunk_rows):
            hi = min(3**n, lo + chunk_rows)
            block = data[lo:hi]
            block = block.cpu().numpy() if hasattr(block, "cpu") else np.asarray(block)
            total += fh.write(np.ascontiguousarray(block.astype(_DTYPE_NP[dtype_code], copy=False)).tobytes())
    return total


def open_record(path) -> RecordFile:
    """Map a ``pauli-lre-bin/1`` file; header and size violations raise RecordFormatError."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_BIN_HEADER_BYTES)
    if len(head) < _BIN_HEADER_BYTES:
        raise RecordFormatError(f"{path}: truncated record file")
    magic, version, n, layout, dtype_code, _, shots, seed, rows = _BIN_HEADER.unpack_from(head)
    if magic != _BIN_MAGIC:
        raise RecordFormatError(f"{path}: bad magic {magic!r}, not a {BINARY_FORMAT} file")
    if version != _BIN_VERSION:
        raise RecordFormatError(f"{path}: unsupported {BINARY_FORMAT} version {version}")
    try:
        n = pauli.check_qubit_count(n)
    except ValueError as exc:
        raise RecordFormatError(f"{path}: {exc}") from None
    if shots < 1:
        raise RecordFormatError(f"{path}: shots must be >= 1, got {shots}")
    if layout not in (LAYOUT_COUNTS, LAYOUT_OUTCOMES) or dtype_code not in _DTYPE_NP:
        raise RecordFormatError(f"{path}: unknown layout {layout} / dtype {dtype_code}")
    if layout == LAYOUT_OUTCOMES and (dtype_code != _lib.U16 or n > 16):
        raise RecordFormatError(f"{path}: outcome lists must be uint16")
    if rows != 3**n:
        raise RecordFormatError(f"{path}: {rows} setting rows, expected {3**n} for n={n}")
    width = (1 << n) if layout == LAYOUT_COUNTS else shots
    dt = _DTYPE_NP[dtype_code]
    expected = _BIN_HEADER_BYTES + rows * width * dt.itemsize
    if size != expected:
        raise RecordFormatError(f"{path}: size {size} bytes, expected {expected} for n={n}")
    label = head[_BIN_HEADER.size:].rstrip(b"\0").decode("utf-8") or None
    data = np.memmap(path, dtype=dt, mode="r", offset=_BIN_HEADER_BYTES, shape=(rows, width))
    return RecordFile(path=str(path), n=n, shots=int(shots), layout=layout,
                      seed=None if seed == _NO_SEED else int(seed), state=label, data=data)


def reconstruct_file(path_or_file, *, device=None, project: bool = False, chunk_bytes: int = 1 << 30,
                     as_tensor: bool = False):
    """Reconstruct straight from a ``pauli-lre-bin/1`` file.

    Setting chunks (multiples of lre_shard_quantum) are read into two pinned
    host buffers, copied H2D on a side stream and folded by the first pass
    while the next chunk is read (LREPlan.stage, or stage_outcomes for outcome
    lists); each dense chunk is validated on the device (lre_validate_counts)
    and the first bad row raises the reference's message before any result
    is returned.  Returns a ReconstructionResult whose timings add
    ``t_ingest_s`` (file -> first-pass partials, wall clock)."""
    import time

    import torch

    from .pipeline import LREPlan, ReconstructionResult, _device, step_three_project

    rf = path_or_file if isinstance(path_or_file, RecordFile) else open_record(path_or_file)
    n, shots = rf.n, rf.shots
    dev = _device(device)
    plan = LREPlan(n, shots, dev)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    q = int(_lib.load().lre_shard_quantum(n))
    row_bytes = rf.data.shape[1] * rf.data.dtype.itemsize
    chunk = max(q, (max(1, chunk_bytes // row_bytes)) // q * q)
    tdt = {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[rf.data.dtype.itemsize]
    pinned = [torch.empty((chunk, rf.data.shape[1]), dtype=tdt, pin_memory=True) for _ in range(2)]
    dbuf = [torch.empty((chunk, rf.data.shape[1]), dtype=tdt, device=dev) for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]
    view_dt = {np.dtype("<u1"): torch.uint8, np.dtype("<u2"): torch.uint16, np.dtype("<i4"): torch.int32,
               np.dtype("<i8"): torch.int64}[rf.data.dtype]
    t0 = time.perf_counter()
    for k, lo in enumerate(range(0, 3**n, chunk)):
        hi = min(3**n, lo + chunk)
        b = k % 2
        done[b].synchronize()  # the pinned buffer's previous H2D has completed
        pinned[b][: hi - lo].numpy()[:] = np.asarray(rf.data[lo:hi]).view(pinned[b].numpy().dtype)
        copy.wait_event(used[b])
        with torch.cuda.stream(copy):
            dbuf[b][: hi - lo].copy_(pinned[b][: hi - lo], non_blocking=True)
            done[b].record(copy)
        comp.wait_event(done[b])
        block = dbuf[b][: hi - lo].view(view_dt)
        if rf.layout == LAYOUT_OUTCOMES:
            plan.stage_outcomes(block, lo, hi, comp, validate=True)
        else:
            plan.stage(block, lre_dtype_of(view_dt), lo, hi, comp, validate=True)
        used[b].record(comp)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(comp)
    plan.finish(comp)
    t_ingest = time.perf_counter() - t0
    ev[1].record(comp)
    plan.step2(comp)
    ev[2].record(comp)
    plan.verify()
    rho, evals = step_three_project(plan.mu) if project else (plan.mu, None)
    ev[3].record(comp)
    ev[3].synchronize()
    t1, t2, t3 = (ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(3))
    timings = {"t_ingest_s": t_ingest, "t_step1_s": t1, "t_step2_s": t2, "t_step3_s": t3,
               "t_total_s": t_ingest + t1 + t2 + t3, "threads": 1, "kernel": "b200", "gpus": 1}
    theta, mu = plan.theta_natural(comp, out=plan.export_buffer()), plan.mu
    if not as_tensor:
        same = rho is mu
        theta, mu = theta.cpu().numpy(), mu.cpu().numpy()
        rho = mu if same else rho.cpu().numpy()
        evals = None if evals is None else evals.cpu().numpy()
    return ReconstructionResult(theta=theta, mu=mu, rho=rho, eigenvalues=evals, timings=timings)


# ---------------------------------------------------------------------------
# PLRE v1 estimate files (statefile.py:1-49)
# ---------------------------------------------------------------------------

_STATE_MAGIC = b"PLRE"
_STATE_VERSION = 1
_STATE_HEADER = struct.Struct("<4sII")


def write_state(path, rho, chunk_rows: int = 1024) -> int:
    """Write a dense 2^n x 2^n complex128 matrix (numpy or device tensor) in
    the reference's ``PLRE`` v1 layout; returns bytes written."""
    shape = tuple(rho.shape)
    d = shape[0] if shape else 0
    if len(shape) != 2 or shape[1] != d or d & (d - 1) or d == 0:
        raise ValueError(f"expected a square 2**n x 2**n matrix, got {shape}")
    n = pauli.check_qubit_count(d.bit_length() - 1)
    total = 0
    with open(path, "wb") as fh:
        total += fh.write(_STATE_HEADER.pack(_STATE_MAGIC, _STATE_VERSION, n))
        for lo in range(0, d, chunk_rows):
            block = rho[lo:lo + chunk_rows]
            block = block.cpu().numpy() if hasattr(block, "cpu") else np.asarray(block)
            total += fh.write(np.ascontiguousarray(block, dtype="<c16").tobytes())
    return total


def read_state(path) -> tuple[int, np.ndarray]:
    """Read a ``PLRE`` v1 file, returning (n, matrix) (statefile.py:32-49)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_STATE_HEADER.size)
        if len(head) < _STATE_HEADER.size:
            raise ValueError(f"{path}: truncated state file")
        magic, version, n = _STATE_HEADER.unpack(head)
        if magic != _STATE_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, not a state file")
        if version != _STATE_VERSION:
            raise ValueError(f"{path}: unsupported state-file version {version}")
        n = pauli.check_qubit_count(n)
        d = 1 << n
        expected = _STATE_HEADER.size + d * d * 16
        if size != expected:
            raise ValueError(f"{path}: size {size} bytes, expected {expected} for n={n}")
        data = np.fromfile(fh, dtype="<c16", count=d * d)
    return n, data.reshape(d, d).astype(np.complex128)
