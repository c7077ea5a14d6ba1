"""The LRE pipeline on B200 — drop-in for the reference's pipeline.py.

Same entry points, argument meaning and error behaviour as the reference
(``/root/reference/pkg/src/pauli_lre/pipeline.py``):

* ``step_one_least_squares(record_or_source, workers=1, kernel=...)``
  (pipeline.py:116-138) — counts -> theta, natural order, fp64;
* ``step_two_assemble(theta, workers=1)`` (pipeline.py:141-161) — theta -> mu;
* ``step_three_project(mu)`` (pipeline.py:187-208) — adjacent step (iii);
* ``reconstruct(record_or_source, workers=1, kernel=...)`` (pipeline.py:224-249)
  returning ``ReconstructionResult`` with the same ``timings`` keys.

Steps (i) and (ii) run only on the sm_100a kernels of liblre_b200.so (there
is no CPU path).  ``workers`` is accepted for signature compatibility (the
GPU decides its own parallelism); ``kernel`` accepts the reference names
"fast" and "paper-direct" (both map to the same B200 kernels, their outputs
being identical by construction in the reference as well) and "b200".
Sources (the reference's source protocol, pipeline.py:42-59,84):
``MeasurementRecord`` (host counts; copied to HBM, validated on the device),
``DeviceRecord`` / ``OutcomeRecord`` (counts or raw shots already in HBM),
``StateDescriptor`` (the reference wraps it in ``ExactFrequencies``),
``ExactFrequencies`` and any duck-typed object with ``.n``, ``.num_settings``
and ``.frequencies(a, b)``.  Integer records run the exact integer folds;
frequency sources run the fp64 folds (``lre_step1_f64_*``): exact
probabilities of dyadic states are an exact integer record (shots = 2^n),
other states' probabilities are computed on the device from their Pauli
coefficients (n <= 12), and any other source's frequency blocks are streamed
from the host in setting chunks.  Outputs are numpy arrays by default; pass
``as_tensor=True`` to keep torch CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, pauli
from .records import DeviceRecord, MeasurementRecord, OutcomeRecord, compact_dtype, lre_dtype_of
from .simulate import StateDescriptor, exact_record, probabilities_block, state_theta, theta_probabilities

KERNELS = ("b200", "fast", "paper-direct")
DENSE_PIPELINE_MAX_QUBITS = 14  # reference caps at 12 (pipeline.py:31); the B200 path lifts it

_HERMITIAN_TOL = 1e-10  # pipeline.py:36
_TRACE_TOL = 1e-8  # pipeline.py:37


_NP_TO_TORCH = {"uint8": "uint8", "uint16": "uint16", "int32": "int32", "int64": "int64"}


def _torch_count_dtype(np_dtype):
    return getattr(_torch(), _NP_TO_TORCH[np.dtype(np_dtype).name])


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the B200 LRE path needs a CUDA device; there is no CPU fallback")
    return torch


def _device(device):
    """A concrete CUDA device (index filled in: torch.device("cuda") != cuda:0 in comparisons)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _check_kernel(kernel: str) -> None:
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}, expected one of {KERNELS}")


# ---------------------------------------------------------------------------
# sources
# ---------------------------------------------------------------------------

class ExactFrequencies:
    """Infinite-shot frequency source backed by exact probabilities (pipeline.py:42-51).

    ``frequencies(a, b)`` returns host fp64 blocks (the protocol); the pipeline
    itself never round-trips them through the host: dyadic states become their
    exact integer record, others are evaluated on the device."""

    def __init__(self, state: StateDescriptor):
        self.state = state
        self.n = state.n
        self.num_settings = 3**state.n

    def frequencies(self, start: int, stop: int) -> np.ndarray:
        return probabilities_block(self.state, start, stop)


def _is_frequency_source(obj) -> bool:
    return all(hasattr(obj, k) for k in ("n", "num_settings", "frequencies"))


def _as_source(record_or_source):
    """pipeline.py:54-59: records are validated, states become ExactFrequencies; an exact
    source of a dyadic state is its noiseless integer record (identical estimate)."""
    src = record_or_source
    if isinstance(src, StateDescriptor):
        src = ExactFrequencies(src)
    if isinstance(src, ExactFrequencies) and src.state.dyadic:
        return src.state  # to_device_record: exact_record on the device
    if isinstance(src, (MeasurementRecord, DeviceRecord, OutcomeRecord)):
        return src
    if _is_frequency_source(src):
        pauli.check_qubit_count(int(src.n))
        if int(src.num_settings) != 3 ** int(src.n):
            raise ValueError(f"source has {src.num_settings} settings, expected 3**{src.n}")
        return src
    raise TypeError(f"unsupported source {type(record_or_source).__name__}: pass a MeasurementRecord, DeviceRecord, "
                    "OutcomeRecord, StateDescriptor or an object with .n, .num_settings and .frequencies(a, b)")

def to_device_record(record_or_source, device=None, stream=None) -> DeviceRecord:
    """Resolve any supported source into a validated DeviceRecord (pipeline.py:54-59)."""
    torch = _torch()
    dev = _device(device)
    if isinstance(record_or_source, DeviceRecord):
        return record_or_source.validate(stream)
    if isinstance(record_or_source, StateDescriptor):
        if not record_or_source.dyadic:
            raise ValueError(
                f"state {record_or_source.label()} has non-dyadic probabilities; the device path consumes "
                "integer counts, sample a record with simulate.sample_counts instead"
            )
        return exact_record(record_or_source, device=dev).validate(stream)
    if isinstance(record_or_source, OutcomeRecord):
        rec = record_or_source
        n = pauli.check_qubit_count(rec.n)
        o = rec.outcomes
        if not isinstance(o, torch.Tensor):
            o = torch.from_numpy(np.ascontiguousarray(np.asarray(o, dtype=np.uint16)))
        o = o.to(dev, non_blocking=False)
        if o.dim() != 2 or int(o.shape[1]) != int(rec.shots) or o.dtype != torch.uint16:
            raise ValueError(f"outcomes must be uint16 of shape (settings, shots={rec.shots}), got {tuple(o.shape)}")
        counts = counts_from_outcomes(o, n, int(rec.shots), stream=stream)
        return DeviceRecord(n=n, shots=int(rec.shots), counts=counts, w_begin=rec.w_begin, seed=rec.seed,
                            state=rec.state).validate(stream)
    if isinstance(record_or_source, MeasurementRecord):
        rec = record_or_source
        n = pauli.check_qubit_count(rec.n)
        counts = np.asarray(rec.counts)
        if tuple(counts.shape) != (3**n, 1 << n):
            raise ValueError(f"counts shape {counts.shape} != {(3**n, 1 << n)} for n={n}")
        if not np.issubdtype(counts.dtype, np.integer):
            raise ValueError(f"counts must be integers, got dtype {counts.dtype}")
        if counts.dtype in (np.uint8, np.uint16) and int(rec.shots) > np.iinfo(counts.dtype).max:
            # each count fits its dtype but a row sum may not (uint8 with shots > 255):
            # widen (exactly) to the smallest dtype that holds `shots`, as the kernels need
            counts = counts.astype(compact_dtype(int(rec.shots)))
        elif counts.dtype not in (np.uint8, np.uint16, np.int32, np.int64):
            counts = counts.astype(np.int64)  # int8/int16/uint32/...: exact in int64, validated below
        dcounts = _host_to_device(np.ascontiguousarray(counts), dev)
        drec = DeviceRecord(n=n, shots=int(rec.shots), counts=dcounts, seed=rec.seed, state=rec.state)
        drec.validate(stream)
        rec._validated = True
        return drec
    raise TypeError(
        f"unsupported source {type(record_or_source).__name__}: pass a MeasurementRecord, DeviceRecord, "
        "OutcomeRecord or a dyadic StateDescriptor (frequency sources go through reconstruct / "
        "step_one_least_squares)"
    )


def _host_to_device(counts: np.ndarray, dev, chunk_bytes: int = 1 << 28):
    """A host record into HBM through two pinned staging buffers (a host-side memcpy into
    one while the other's H2D copy runs on a side stream) instead of one blocking
    pageable copy; small records take the direct copy."""
    torch = _torch()
    host = torch.from_numpy(counts)
    if counts.nbytes <= chunk_bytes:
        return host.to(dev)
    out = torch.empty(tuple(counts.shape), dtype=host.dtype, device=dev)
    rows_per = max(1, chunk_bytes // max(1, counts.strides[0]))
    pinned = [torch.empty((rows_per,) + tuple(counts.shape[1:]), dtype=host.dtype, pin_memory=True) for _ in range(2)]
    copy = torch.cuda.Stream(dev)
    done = [torch.cuda.Event() for _ in range(2)]
    for k, lo in enumerate(range(0, counts.shape[0], rows_per)):
        hi = min(counts.shape[0], lo + rows_per)
        b = k % 2
        done[b].synchronize()  # the previous copy out of this staging buffer has finished
        pinned[b][: hi - lo].copy_(host[lo:hi])
        with torch.cuda.stream(copy):
            out[lo:hi].copy_(pinned[b][: hi - lo], non_blocking=True)
            done[b].record(copy)
    torch.cuda.current_stream(dev).wait_stream(copy)
    return out


def counts_from_outcomes(outcomes, n: int, shots: int, out=None, stream=None):
    """Device outcome lists (uint16, rows x shots) -> dense device counts (lre_counts_from_outcomes)."""
    torch = _torch()
    rows = int(outcomes.shape[0])
    if out is None:
        out = torch.empty((rows, 1 << n), dtype=_torch_count_dtype(compact_dtype(shots)), device=outcomes.device)
    if rows == 0:
        return out
    stream = stream if stream is not None else torch.cuda.current_stream(outcomes.device)
    _lib.call("lre_counts_from_outcomes", outcomes.data_ptr(), n, int(shots), rows, out.data_ptr(),
              lre_dtype_of(out.dtype), stream.cuda_stream)
    return out


# ---------------------------------------------------------------------------
# device plan: buffers + launches for one (n, shots, dtype) shape
# ---------------------------------------------------------------------------

class LREPlan:
    """Preallocated HBM buffers and the launch sequence of one reconstruction.

    step1: counts -> theta (natural order, fp64): the tile pass plus 2-qubit
    vector passes (lre_step1);
    step2: theta -> mu (row-major complex128), 1 launch (lre_assemble).

    ``mu`` lives inside the step-(i) workspace when that is large enough (the
    workspace is dead once theta is final), which is what lets an n = 14
    record (157 GB of uint16 counts) and the whole pipeline share one B200.
    """

    def __init__(self, n: int, shots: int, device=None, with_mu: bool = True):
        torch = _torch()
        self.n = pauli.check_qubit_count(n)
        self.shots = int(shots)
        self.device = _device(device)
        import ctypes

        L = _lib.load()
        ws = ctypes.c_size_t(0)
        _lib.check(L.lre_step1_workspace(self.n, self.shots, 0, 3**self.n, ctypes.byref(ws)), "lre_step1_workspace")
        self.ws_bytes = int(ws.value)
        d = 1 << self.n
        mu_bytes = 16 * d * d if with_mu else 0
        self.ws = torch.empty(max(self.ws_bytes, mu_bytes, 256), dtype=torch.uint8, device=self.device)
        self.theta = torch.empty(4**self.n, dtype=torch.float64, device=self.device)
        self.mu = self.ws[:mu_bytes].view(torch.complex128).view(d, d) if with_mu else None
        self.passes = int(L.lre_step1_num_passes(self.n, self.shots))
        # theta layout inside the plan: mask-major at n >= 11, where step (ii) is the
        # 8-CTA-cluster kernel that bulk-copies each mask's 2^n coefficients
        # (DESIGN.md §4); theta_natural() exports the reference's natural order
        self.layout = _lib.MASK_MAJOR if self.n >= 11 else _lib.NATURAL
        self._checks = []

    def _check_chunk(self, counts, count_dtype: int, rows: int) -> None:
        """Shape, dtype, device and contiguity of a counts tensor handed to the C ABI
        (which sees only a pointer)."""
        torch = _torch()
        if not isinstance(counts, torch.Tensor) or not counts.is_cuda or counts.device != self.device:
            raise ValueError(f"counts must be a CUDA tensor on {self.device}")
        if counts.dim() != 2 or tuple(counts.shape) != (rows, 1 << self.n):
            raise ValueError(f"counts shape {tuple(counts.shape)} != {(rows, 1 << self.n)} for n={self.n}")
        if not counts.is_contiguous():
            raise ValueError("counts must be contiguous")
        if lre_dtype_of(counts.dtype) != int(count_dtype):
            raise ValueError(f"count dtype {counts.dtype} does not match lre dtype code {count_dtype}")

    def step1(self, counts, count_dtype: int, stream) -> None:
        self._check_chunk(counts, count_dtype, 3**self.n)
        _lib.call("lre_step1", counts.data_ptr(), count_dtype, self.n, self.shots, 0, 3**self.n,
                  self.ws.data_ptr(), self.ws_bytes, self.theta.data_ptr(), _lib.OUT_THETA_F64,
                  self.layout, stream.cuda_stream)

    def stage(self, chunk, count_dtype: int, w_begin: int, w_end: int, stream, validate: bool = False) -> None:
        """Fold setting chunk [w_begin, w_end) into the first pass (lre_step1_stage).

        validate=True also checks the chunk's rows on the device
        (lre_validate_counts, records.py:34-56) on the same stream; the result
        is read by verify(), which raises the reference's message for the
        first bad setting — the streaming counterpart of validating a record
        before the reconstruction.  An empty range is a no-op."""
        if int(w_end) == int(w_begin):
            return
        self._check_chunk(chunk, count_dtype, int(w_end) - int(w_begin))
        if validate:
            torch = _torch()
            res = torch.empty(3, dtype=torch.int64, device=self.device)
            _lib.call("lre_validate_counts", chunk.data_ptr(), count_dtype, self.n, int(w_end) - int(w_begin),
                      self.shots, res.data_ptr(), stream.cuda_stream)
            self._checks.append((int(w_begin), res))
        _lib.call("lre_step1_stage", chunk.data_ptr(), count_dtype, self.n, self.shots, int(w_begin), int(w_end),
                  self.ws.data_ptr(), self.ws_bytes, stream.cuda_stream)

    def verify(self) -> None:
        """Raise for the first invalid row among the chunks staged with validate=True (synchronises)."""
        checks, self._checks = self._checks, []
        for w0, res in checks:
            first_bad, bad_sum, min_value = (int(x) for x in res.cpu().tolist())
            if min_value < 0:
                raise ValueError("counts must be non-negative")
            if first_bad != (1 << 63) - 1:
                w = w0 + first_bad
                raise ValueError(f"setting {pauli.setting_label(w, self.n)} (index {w}) sums to {bad_sum}, "
                                 f"expected {self.shots}")

    def stage_outcomes(self, outcomes, w_begin: int, w_end: int, stream, validate: bool = False) -> None:
        """Streaming ingestion of an outcome-list chunk: histogram on the device, then stage."""
        torch = _torch()
        rows = int(outcomes.shape[0])
        if rows == 0:
            return
        buf = getattr(self, "_dense", None)
        if buf is None or buf.shape[0] < rows:
            dt = _torch_count_dtype(compact_dtype(self.shots))
            self._dense = buf = torch.empty((rows, 1 << self.n), dtype=dt, device=self.device)
        dense = buf[:rows]
        counts_from_outcomes(outcomes, self.n, self.shots, out=dense, stream=stream)
        self.stage(dense, lre_dtype_of(dense.dtype), w_begin, w_end, stream, validate=validate)

    def finish(self, stream) -> None:
        _lib.call("lre_step1_finish", self.ws.data_ptr(), self.ws_bytes, self.n, self.shots,
                  self.theta.data_ptr(), _lib.OUT_THETA_F64, self.layout, stream.cuda_stream)

    def step2(self, stream) -> None:
        d = 1 << self.n
        _lib.call("lre_assemble", self.theta.data_ptr(), self.layout, self.n, 0, d, self.mu.data_ptr(),
                  stream.cuda_stream)

    def export_buffer(self):
        """Room for a natural-order theta copy behind mu in the step-(i) workspace
        (dead once theta is final; n = 14 has no HBM to spare for a fresh 2 GiB
        buffer next to a resident record), or None."""
        if self.layout == _lib.NATURAL:
            return None
        torch = _torch()
        mu_bytes = 0 if self.mu is None else self.mu.numel() * 16
        off = (mu_bytes + 255) // 256 * 256
        need = self.theta.numel() * 8
        if self.ws.numel() < off + need:
            return None
        return self.ws[off:off + need].view(torch.float64)

    def theta_natural(self, stream=None, out=None):
        """theta in the reference's natural order (pipeline.py:138): the plan's own
        buffer when it is natural, else a relayout (lre_theta_relayout) into `out`."""
        if self.layout == _lib.NATURAL:
            return self.theta
        torch = _torch()
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        out = torch.empty_like(self.theta) if out is None else out
        _lib.call("lre_theta_relayout", self.theta.data_ptr(), self.layout, self.n, out.data_ptr(), stream.cuda_stream)
        return out

    def run(self, counts, count_dtype: int, stream) -> None:
        self.step1(counts, count_dtype, stream)
        self.step2(stream)


class F64Plan:
    """Step (i) from fp64 frequency sources (lre_step1_f64_*) plus step (ii).

    The source is consumed in setting chunks (a multiple of lre_step1_f64_quantum):
    exact sources of non-dyadic states have their probabilities evaluated on the
    device chunk by chunk (lre_theta_probabilities); any other source's
    ``frequencies(a, b)`` blocks are copied from the host through two pinned
    buffers on a copy stream, overlapped with the folding of the previous chunk.
    ``mu`` lives in the workspace (dead once theta is final), as in LREPlan."""

    def __init__(self, n: int, device=None, chunk_bytes: int = 1 << 28, with_mu: bool = True):
        import ctypes

        torch = _torch()
        self.n = pauli.check_qubit_count(n)
        self.device = _device(device)
        L = _lib.load()
        q = int(L.lre_step1_f64_quantum(self.n))
        settings, d = 3**self.n, 1 << self.n
        rows = max(q, (max(1, chunk_bytes // (8 * d)) // q) * q)
        self.chunk_rows = min(settings, rows)
        ws, sc = ctypes.c_size_t(0), ctypes.c_size_t(0)
        _lib.check(L.lre_step1_f64_workspace(self.n, self.chunk_rows, ctypes.byref(ws), ctypes.byref(sc)),
                   "lre_step1_f64_workspace")
        self.ws_bytes, self.scratch_bytes = int(ws.value), int(sc.value)
        mu_bytes = 16 * d * d if with_mu else 0
        self.ws = torch.empty(max(self.ws_bytes, mu_bytes, 256), dtype=torch.uint8, device=self.device)
        self.scratch = torch.empty(max(self.scratch_bytes, 256), dtype=torch.uint8, device=self.device)
        self.theta = torch.empty(4**self.n, dtype=torch.float64, device=self.device)
        self.mu = self.ws[:mu_bytes].view(torch.complex128).view(d, d) if with_mu else None
        self.layout = _lib.MASK_MAJOR if self.n >= 11 else _lib.NATURAL

    def stage(self, freq, w_begin: int, w_end: int, stream) -> None:
        torch = _torch()
        rows = int(w_end) - int(w_begin)
        if not isinstance(freq, torch.Tensor) or freq.dtype != torch.float64 or not freq.is_cuda \
                or tuple(freq.shape) != (rows, 1 << self.n) or not freq.is_contiguous():
            raise ValueError(f"frequency chunk must be a contiguous CUDA float64 tensor of shape {(rows, 1 << self.n)}")
        _lib.call("lre_step1_f64_stage", freq.data_ptr(), self.n, int(w_begin), int(w_end), self.ws.data_ptr(),
                  self.ws_bytes, self.scratch.data_ptr(), self.scratch_bytes, stream.cuda_stream)

    def finish(self, stream) -> None:
        _lib.call("lre_step1_f64_finish", self.ws.data_ptr(), self.ws_bytes, self.n, self.theta.data_ptr(),
                  self.layout, stream.cuda_stream)

    def step1(self, source, stream) -> None:
        """Every chunk of `source` staged, then the remaining passes (theta final)."""
        torch = _torch()
        settings, d = 3**self.n, 1 << self.n
        exact = isinstance(source, ExactFrequencies)
        bufs = [torch.empty((self.chunk_rows, d), dtype=torch.float64, device=self.device) for _ in range(2)]
        if exact:
            theta_true = state_theta(source.state, self.device)
            for k, lo in enumerate(range(0, settings, self.chunk_rows)):
                hi = min(settings, lo + self.chunk_rows)
                blk = bufs[k % 2][: hi - lo]
                theta_probabilities(theta_true, self.n, lo, hi, clip=True, out=blk, stream=stream)
                self.stage(blk, lo, hi, stream)
        else:
            copy = torch.cuda.Stream(self.device)
            pinned = [torch.empty((self.chunk_rows, d), dtype=torch.float64, pin_memory=True) for _ in range(2)]
            ev_copy = [torch.cuda.Event() for _ in range(2)]
            ev_used = [torch.cuda.Event() for _ in range(2)]
            for k, lo in enumerate(range(0, settings, self.chunk_rows)):
                hi = min(settings, lo + self.chunk_rows)
                b = k % 2
                block = np.asarray(source.frequencies(lo, hi), dtype=np.float64)
                if block.shape != (hi - lo, d):
                    raise ValueError(f"frequencies({lo}, {hi}) returned shape {block.shape}, expected {(hi - lo, d)}")
                ev_used[b].synchronize()  # the pinned buffer's previous H2D copy has been consumed
                pinned[b][: hi - lo].numpy()[...] = block
                copy.wait_event(ev_used[b])
                with torch.cuda.stream(copy):
                    bufs[b][: hi - lo].copy_(pinned[b][: hi - lo], non_blocking=True)
                    ev_copy[b].record(copy)
                stream.wait_event(ev_copy[b])
                self.stage(bufs[b][: hi - lo], lo, hi, stream)
                ev_used[b].record(stream)
            torch.cuda.current_stream(self.device).wait_stream(copy)
        self.finish(stream)

    step2 = LREPlan.step2
    export_buffer = LREPlan.export_buffer
    theta_natural = LREPlan.theta_natural


def _reconstruct_frequencies(source, stream, project: bool, device, workers, kernel, as_tensor):
    """reconstruct() for fp64 frequency sources (F64Plan)."""
    torch = _torch()
    n = pauli.check_qubit_count(int(source.n))
    if n > DENSE_PIPELINE_MAX_QUBITS:
        raise ValueError(f"n={n} needs a dense {2**n}x{2**n} complex allocation; the dense pipeline is capped "
                         f"at n={DENSE_PIPELINE_MAX_QUBITS}")
    dev = _device(device)
    stream = stream if stream is not None else torch.cuda.current_stream(dev)
    plan = F64Plan(n, dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(stream)
    plan.step1(source, stream)
    ev[1].record(stream)
    plan.step2(stream)
    ev[2].record(stream)
    rho, evals = step_three_project(plan.mu) if project else (plan.mu, None)
    ev[3].record(stream)
    theta = plan.theta_natural(stream, out=plan.export_buffer())
    ev[4].record(stream)
    ev[4].synchronize()
    t1, t2, t3 = (ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(3))
    timings = {"t_step1_s": t1, "t_step2_s": t2, "t_step3_s": t3, "t_total_s": t1 + t2 + t3, "threads": workers,
               "kernel": kernel, "gpus": 1, "t_theta_export_s": ev[3].elapsed_time(ev[4]) / 1e3,
               "source": "exact (device)" if isinstance(source, ExactFrequencies) else "frequencies (host)"}
    timings.update(roofline_timings(n, 8, t1 + t2))
    mu = plan.mu
    if not as_tensor:
        same = rho is mu
        theta, mu = theta.cpu().numpy(), mu.cpu().numpy()
        rho = mu if same else rho.cpu().numpy()
        evals = None if evals is None else evals.cpu().numpy()
    return ReconstructionResult(theta=theta, mu=mu, rho=rho, eigenvalues=evals, timings=timings)


# ---------------------------------------------------------------------------
# reference entry points
# ---------------------------------------------------------------------------

def step_one_least_squares(record_or_source, workers: int = 1, kernel: str = "b200", *, device=None,
                           as_tensor: bool = False):
    """Least-squares Pauli coefficients theta (natural order), pipeline.py:116-138."""
    _check_kernel(kernel)
    torch = _torch()
    src = _as_source(record_or_source)
    if not isinstance(src, (MeasurementRecord, DeviceRecord, OutcomeRecord, StateDescriptor)):
        plan = F64Plan(int(src.n), device, with_mu=False)
        plan.layout = _lib.NATURAL
        plan.step1(src, torch.cuda.current_stream(plan.device))
        return plan.theta if as_tensor else plan.theta.cpu().numpy()
    rec = to_device_record(src, device)
    n = pauli.check_qubit_count(rec.n)
    stream = torch.cuda.current_stream(rec.counts.device)
    theta = torch.empty(4**n, dtype=torch.float64, device=rec.counts.device)
    if rec.w_begin != 0 or rec.w_end != 3**n:
        raise ValueError(f"step_one_least_squares needs the full setting range [0, {3**n}), "
                         f"got [{rec.w_begin}, {rec.w_end})")
    import ctypes

    ws = ctypes.c_size_t(0)
    _lib.check(_lib.load().lre_step1_workspace(n, int(rec.shots), 0, 3**n, ctypes.byref(ws)), "lre_step1_workspace")
    buf = torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device=rec.counts.device)
    _lib.call("lre_step1", rec.counts.data_ptr(), rec.lre_dtype, n, int(rec.shots), 0, 3**n, buf.data_ptr(),
              int(ws.value), theta.data_ptr(), _lib.OUT_THETA_F64, _lib.NATURAL, stream.cuda_stream)
    return theta if as_tensor else theta.cpu().numpy()


def step_two_assemble(theta, workers: int = 1, *, device=None, as_tensor: bool = False):
    """Dense Hermitian estimate mu from theta (natural order), pipeline.py:141-161."""
    torch = _torch()
    size = int(theta.shape[0])
    n = (size.bit_length() - 1) // 2
    if len(theta.shape) != 1 or size != 4**n:
        raise ValueError(f"theta length {tuple(theta.shape)} is not 4**n")
    pauli.check_qubit_count(n)
    if n > DENSE_PIPELINE_MAX_QUBITS:
        raise NotImplementedError(f"dense assembly is built for n <= {DENSE_PIPELINE_MAX_QUBITS}")
    dev = theta.device if isinstance(theta, torch.Tensor) and theta.is_cuda else _device(device)
    stream = torch.cuda.current_stream(dev)
    t = theta if isinstance(theta, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(theta, dtype=np.float64))
    t = t.to(device=dev, dtype=torch.float64).contiguous()
    d = 1 << n
    mu = torch.empty((d, d), dtype=torch.complex128, device=dev)
    layout = _lib.NATURAL
    if n >= 11:  # the 8-CTA-cluster assembly reads each mask's coefficients contiguously
        mm = torch.empty_like(t)
        _lib.call("lre_theta_relayout", t.data_ptr(), _lib.NATURAL, n, mm.data_ptr(), stream.cuda_stream)
        t, layout = mm, _lib.MASK_MAJOR
    _lib.call("lre_assemble", t.data_ptr(), layout, n, 0, d, mu.data_ptr(), stream.cuda_stream)
    return mu if as_tensor else mu.cpu().numpy()


def project_spectrum_to_simplex(values):
    """Scan-from-smallest simplex projection (pipeline.py:164-184), on the device."""
    torch = _torch()
    is_np = not isinstance(values, torch.Tensor)
    v = torch.as_tensor(np.asarray(values, dtype=np.float64) if is_np else values, dtype=torch.float64)
    v = v.to(_device(None) if not v.is_cuda else v.device)
    u, order = torch.sort(v)
    k = u.shape[0]
    prefix = torch.cat([torch.zeros(1, dtype=u.dtype, device=u.device), torch.cumsum(u[:-1], 0)])
    remaining = k - torch.arange(k, device=u.device, dtype=u.dtype)
    crossing = (u + prefix / remaining) >= 0.0
    stop = int(torch.argmax(crossing.to(torch.int8)).item())
    out = torch.zeros_like(u)
    out[stop:] = u[stop:] + prefix[stop] / (k - stop)
    res = torch.empty_like(out)
    res[order] = out
    return res.cpu().numpy() if is_np else res


def step_three_project(mu):
    """Closest physical state (pipeline.py:187-208); adjacent to the hot path.

    Uses the device Hermitian eigensolver (cuSOLVER via torch.linalg.eigh)
    and returns ``(rho, eigenvalues ascending)``; an already-PSD ``mu`` is
    returned unchanged (the same object), as in the reference.
    """
    torch = _torch()
    is_np = not isinstance(mu, torch.Tensor)
    m = torch.from_numpy(np.asarray(mu)) if is_np else mu
    m = m.to(device=_device(None) if not m.is_cuda else m.device, dtype=torch.complex128)
    d = m.shape[0]
    if m.dim() != 2 or m.shape[1] != d:
        raise ValueError(f"expected a square matrix, got shape {tuple(m.shape)}")
    asym = float((m - m.conj().T).abs().max().item())
    if asym > _HERMITIAN_TOL:
        raise ValueError(f"matrix is not Hermitian (max asymmetry {asym:.3e})")
    trace = float(torch.diagonal(m).real.sum().item())
    if abs(trace - 1.0) > _TRACE_TOL:
        raise ValueError(f"trace {trace!r} deviates from 1 beyond {_TRACE_TOL}")
    evals, evecs = torch.linalg.eigh(m)
    if float(evals[0].item()) >= 0.0:
        return (mu, evals.cpu().numpy()) if is_np else (mu, evals)
    lam = project_spectrum_to_simplex(evals)
    rho = (evecs * lam.to(evecs.dtype)) @ evecs.conj().T
    return (rho.cpu().numpy(), lam.cpu().numpy()) if is_np else (rho, lam)


@dataclass
class ReconstructionResult:
    """pipeline.py:211-221."""

    theta: object
    mu: object
    rho: object
    eigenvalues: object  # spectrum of rho, ascending
    timings: dict

    @property
    def n(self) -> int:
        return (int(self.theta.shape[0]).bit_length() - 1) // 2


def reconstruct(record_or_source, workers: int = 1, kernel: str = "b200", *, device=None, project: bool = True,
                as_tensor: bool = False, devices=None) -> ReconstructionResult:
    """All three steps with per-step device timings (pipeline.py:224-249).

    Validation happens before the timer, as in the reference.  ``timings``
    has the reference keys t_step1_s / t_step2_s / t_step3_s / t_total_s /
    threads / kernel, measured with CUDA events, plus gpus and the SURVEY §5
    keys bytes / gbps / roofline_frac.  ``devices`` (an int P or a list of
    devices, P a power of two) shards an integer record's settings over P GPUs of
    this process and exchanges the partial numerators peer to peer
    (distributed.LocalShardedLRE); the estimate is bit-identical
    to the one-GPU path.
    """
    _check_kernel(kernel)
    torch = _torch()
    src = _as_source(record_or_source)
    if devices is not None and not (isinstance(devices, int) and devices == 1 and device is None):
        return _reconstruct_devices(src, devices, project, workers, kernel, as_tensor)
    if not isinstance(src, (MeasurementRecord, DeviceRecord, OutcomeRecord, StateDescriptor)):
        return _reconstruct_frequencies(src, None, project, device, workers, kernel, as_tensor)
    rec = to_device_record(src, device)
    n = pauli.check_qubit_count(rec.n)
    if rec.w_begin != 0 or rec.w_end != 3**n:
        raise ValueError(f"reconstruct needs the full setting range [0, {3**n}), got [{rec.w_begin}, {rec.w_end})")
    if n > DENSE_PIPELINE_MAX_QUBITS:
        raise ValueError(
            f"n={n} needs a dense {2**n}x{2**n} complex allocation "
            f"({(4**n * 16) >> 20} MB); the dense pipeline is capped at n={DENSE_PIPELINE_MAX_QUBITS}"
        )
    dev = rec.counts.device
    stream = torch.cuda.current_stream(dev)
    plan = LREPlan(n, rec.shots, dev)
    nvtx = torch.cuda.nvtx
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(stream)
    nvtx.range_push("lre.step1")
    plan.step1(rec.counts, rec.lre_dtype, stream)
    nvtx.range_pop()
    ev[1].record(stream)
    nvtx.range_push("lre.step2")
    plan.step2(stream)
    nvtx.range_pop()
    ev[2].record(stream)
    nvtx.range_push("lre.step3")
    if project:
        rho, evals = step_three_project(plan.mu)
    else:
        rho, evals = plan.mu, None
    nvtx.range_pop()
    ev[3].record(stream)
    nvtx.range_push("lre.theta_export")
    theta = plan.theta_natural(stream, out=plan.export_buffer())
    nvtx.range_pop()
    ev[4].record(stream)
    ev[4].synchronize()
    t1 = ev[0].elapsed_time(ev[1]) / 1e3
    t2 = ev[1].elapsed_time(ev[2]) / 1e3
    t3 = ev[2].elapsed_time(ev[3]) / 1e3
    timings = {
        "t_step1_s": t1,
        "t_step2_s": t2,
        "t_step3_s": t3,
        "t_total_s": t1 + t2 + t3,
        "threads": workers,
        "kernel": kernel,
        "gpus": 1,
        "t_theta_export_s": ev[3].elapsed_time(ev[4]) / 1e3,
    }
    timings.update(roofline_timings(n, rec.counts.element_size(), t1 + t2))
    mu = plan.mu
    if not as_tensor:
        same = rho is mu
        theta, mu = theta.cpu().numpy(), mu.cpu().numpy()
        rho = mu if same else rho.cpu().numpy()
        evals = None if evals is None else evals.cpu().numpy()
    return ReconstructionResult(theta=theta, mu=mu, rho=rho, eigenvalues=evals, timings=timings)


def _reconstruct_devices(src, devices, project: bool, workers, kernel, as_tensor):
    """reconstruct(..., devices=P): settings sharded over P devices of this process."""
    torch = _torch()
    from . import distributed as D

    if isinstance(devices, int):
        devs = [torch.device("cuda", i) for i in range(devices)]
    else:
        devs = [_device(x) for x in devices]
    P = len(devs)
    if isinstance(src, StateDescriptor):
        src = exact_record(src, device=devs[0])
    if not isinstance(src, (MeasurementRecord, DeviceRecord, OutcomeRecord)):
        raise ValueError("devices= shards integer records (MeasurementRecord, DeviceRecord, OutcomeRecord, dyadic "
                         "exact states); reconstruct frequency sources on one device")
    rec = to_device_record(src, devs[0])
    n = pauli.check_qubit_count(rec.n)
    if rec.w_begin != 0 or rec.w_end != 3**n:
        raise ValueError(f"reconstruct needs the full setting range [0, {3**n}), got [{rec.w_begin}, {rec.w_end})")
    D.mask_range(n, P, 0)  # P must be a power of two <= 2^n
    q = int(_lib.load().lre_shard_quantum(n))
    ranges = D.shard_ranges(n, P, q)
    comps = [D.DeviceCompute(n, rec.shots, lo, hi, P, g, devs[g]) for g, (lo, hi) in enumerate(ranges)]
    shards = [rec.counts[lo:hi] if devs[g] == rec.counts.device else rec.counts[lo:hi].to(devs[g])
              for g, (lo, hi) in enumerate(ranges)]
    for dv in devs:
        torch.cuda.synchronize(dv)
    runner = D.LocalShardedLRE(comps)
    stream = torch.cuda.current_stream(devs[0])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    runner.step(shards, rec.lre_dtype)
    for dv in devs[1:]:
        torch.cuda.current_stream(devs[0]).wait_stream(torch.cuda.current_stream(dv))
    ev[1].record(stream)
    mu = runner.gather()
    theta_mm = runner.theta_mask_major()
    ev[2].record(stream)
    rho, evals = step_three_project(mu) if project else (mu, None)
    ev[3].record(stream)
    theta = torch.empty_like(theta_mm)
    _lib.call("lre_theta_relayout", theta_mm.data_ptr(), _lib.MASK_MAJOR, n, theta.data_ptr(), stream.cuda_stream)
    ev[3].synchronize()
    t12 = ev[0].elapsed_time(ev[1]) / 1e3
    t3 = ev[2].elapsed_time(ev[3]) / 1e3
    timings = {"t_step12_s": t12, "t_gather_s": ev[1].elapsed_time(ev[2]) / 1e3, "t_step3_s": t3,
               "t_total_s": t12 + t3, "threads": workers, "kernel": kernel, "gpus": P,
               "exchange_chunks": comps[0].K}
    timings.update(roofline_timings(n, rec.counts.element_size(), t12))
    if not as_tensor:
        same = rho is mu
        theta, mu = theta.cpu().numpy(), mu.cpu().numpy()
        rho = mu if same else rho.cpu().numpy()
        evals = None if evals is None else evals.cpu().numpy()
    return ReconstructionResult(theta=theta, mu=mu, rho=rho, eigenvalues=evals, timings=timings)


def hbm_peak_gbps() -> tuple[float, str]:
    """Roofline denominator: the measured copy bandwidth of this pool's B200s
    (MEASURED_PEAKS.json, driver-written), else the profiling guide's fallback."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_bytes(n: int, count_bytes: int) -> float:
    """B(n) = c 6^n (counts read once) + 32 4^n (theta written and read, mu written)."""
    return count_bytes * 6.0**n + 32.0 * 4.0**n


def roofline_timings(n: int, count_bytes: int, seconds: float) -> dict:
    """SURVEY §5 instrumentation keys: algorithmic bytes of steps (i)+(ii), achieved GB/s, fraction of peak."""
    b = algorithmic_bytes(n, count_bytes)
    peak, kind = hbm_peak_gbps()
    gbps = b / seconds / 1e9 if seconds > 0 else float("nan")
    return {"bytes": b, "gbps": gbps, "roofline_frac": gbps / peak, "peak_gbps": peak, "peak_kind": kind}


def reconstruct_generated(state: StateDescriptor, shots: int, seed: int, *, device=None, project: bool = True,
                          chunk_bytes: int = 1 << 31, as_tensor: bool = True) -> ReconstructionResult:
    """Sample a record with the device generator and reconstruct it, chunk by
    chunk: each setting chunk (a multiple of lre_shard_quantum) is generated
    into one reusable HBM buffer and folded by the first pass
    (lre_step1_stage), so the record is never resident — n = 14 with
    int32 counts (d*N0 shots per setting, 313 GB) needs only the chunk.  The
    counts are identical to sample_counts(state, shots, seed)."""
    torch = _torch()
    from .simulate import generate_device_counts

    n = pauli.check_qubit_count(state.n)
    dev = _device(device)
    plan = LREPlan(n, shots, dev)
    stream = torch.cuda.current_stream(dev)
    q = int(_lib.load().lre_shard_quantum(n))
    dt = compact_dtype(shots)
    row_bytes = (1 << n) * np.dtype(dt).itemsize
    chunk = max(q, (max(1, chunk_bytes // row_bytes)) // q * q)
    buf = torch.empty((min(chunk, 3**n), 1 << n), dtype=_torch_count_dtype(dt), device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    for lo in range(0, 3**n, chunk):
        hi = min(3**n, lo + chunk)
        block = buf[: hi - lo]
        generate_device_counts(state, shots, seed=seed, w_begin=lo, w_end=hi, out=block, stream=stream)
        plan.stage(block, lre_dtype_of(block.dtype), lo, hi, stream)
    plan.finish(stream)
    del buf
    ev[1].record(stream)
    plan.step2(stream)
    ev[2].record(stream)
    rho, evals = step_three_project(plan.mu) if project else (plan.mu, None)
    ev[3].record(stream)
    ev[3].synchronize()
    t1, t2, t3 = (ev[i].elapsed_time(ev[i + 1]) / 1e3 for i in range(3))
    timings = {"t_generate_and_step1_s": t1, "t_step2_s": t2, "t_step3_s": t3, "t_total_s": t1 + t2 + t3,
               "threads": 1, "kernel": "b200", "gpus": 1}
    theta, mu = plan.theta_natural(stream, out=plan.export_buffer()), plan.mu
    if not as_tensor:
        same = rho is mu
        theta, mu = theta.cpu().numpy(), mu.cpu().numpy()
        rho = mu if same else rho.cpu().numpy()
        evals = None if evals is None else evals.cpu().numpy()
    return ReconstructionResult(theta=theta, mu=mu, rho=rho, eigenvalues=evals, timings=timings)
