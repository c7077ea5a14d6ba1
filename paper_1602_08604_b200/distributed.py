"""Multi-GPU LRE: settings sharded over ranks, one exchange step.

SURVEY §8(e): rank g owns a contiguous, quantum-aligned range of settings
(its counts are generated in place or copied from its slice of the record);
it folds them into a full-length partial numerator vector N_g (exact int64);
one reduce-scatter (sum) over NCCL/NVLink leaves rank g with the complete
numerators of X-masks [g*2^n/P, (g+1)*2^n/P); it finalises them to theta and
assembles its XOR-block slice of mu: rows r, columns ((r/S) ^ g)*S + c, S =
2^n/P.  Integer numerators make the result bit-identical for every P, and the
epilogue (lre_finalize) is the single-GPU one, so theta is bit-identical too.

Overlap: the partial numerators are written in the MASK_CHUNKED layout
(include/lre_b200.h), in which chunk c of every rank's mask slice is one
contiguous block, so the exchange runs as K reduce-scatters on a side stream
and chunk c is finalised and assembled (lre_finalize + lre_assemble_slab) on
the compute stream while chunk c+1 is still on the wire.

Two exchange backends share the chunk logic:
  * ShardedLRE — one process per GPU, torch.distributed (NCCL on B200, gloo in
    the CPU tests);
  * LocalShardedLRE — one process driving several devices (reconstruct(...,
    devices=N)): the reduce-scatter is a sum of peer-to-peer slice copies.
The compute side is backend-agnostic: production uses DeviceCompute (the CUDA
kernels of liblre_b200.so); the CPU tests inject an oracle-backed compute
object with the same interface (tests/test_distributed.py).

Unmeasured on hardware beyond one GPU: the only multi-rank runs so far are the
gloo tests and world = 1 on a B200.
"""

from __future__ import annotations


def shard_ranges(n: int, world: int, quantum: int) -> list[tuple[int, int]]:
    """Balanced quantum-aligned setting ranges, one per rank."""
    total = 3**n
    groups = -(-total // quantum)
    out = []
    for g in range(world):
        lo = groups * g // world * quantum
        hi = min(total, groups * (g + 1) // world * quantum)
        out.append((lo, hi))
    return out


def mask_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """X-mask slice owned by `rank` after the reduce-scatter (world | 2^n)."""
    d = 1 << n
    if world & (world - 1) or world > d:
        raise ValueError(f"world size {world} must be a power of two <= 2^n")
    S = d // world
    return rank * S, (rank + 1) * S


def default_chunks(n: int, world: int, max_chunks: int = 4) -> int:
    """Exchange chunks per rank slice: chunked assembly needs n >= 11 and >= 8 masks per chunk."""
    S = (1 << n) // world
    k = 1
    if n >= 11:
        while k < max_chunks and S // (2 * k) >= 8:
            k *= 2
    return k


def mask_position(m: int, n: int, log_p: int, log_k: int) -> int:
    """Position of X-mask m in the MASK_CHUNKED(log_p, log_k) layout (mirrors lre_internal.cuh)."""
    log_s = n - log_p
    log_j = log_s - log_k
    g, c, j = m >> log_s, (m >> log_j) & ((1 << log_k) - 1), m & ((1 << log_j) - 1)
    return (((c << log_p) | g) << log_j) | j


class DeviceCompute:
    """The production compute backend: liblre_b200.so kernels on one GPU."""

    def __init__(self, n: int, shots: int, w_lo: int, w_hi: int, world: int, rank: int, device, chunks=None):
        import ctypes

        import torch

        from . import _lib

        self.torch, self.lib = torch, _lib
        self.n, self.shots, self.w_lo, self.w_hi = n, shots, w_lo, w_hi
        self.world, self.rank = world, rank
        self.device = torch.device(device)
        ws = ctypes.c_size_t(0)
        _lib.check(_lib.load().lre_step1_workspace(n, shots, w_lo, w_hi, ctypes.byref(ws)), "lre_step1_workspace")
        self.ws_bytes = int(ws.value)
        d = 1 << n
        self.m_lo, self.m_hi = mask_range(n, world, rank)
        S = self.m_hi - self.m_lo
        # mu, the received numerators and theta live in the step-(i) workspace, dead once
        # the partial numerators are written (n = 14 at P = 1: 147 GB of counts + 22 GB)
        mu_b, recv_b, th_b = 16 * d * S, 8 * S * d, 8 * S * d
        self.ws = torch.empty(max(self.ws_bytes, mu_b + recv_b + th_b, 256), dtype=torch.uint8, device=self.device)
        self.K = default_chunks(n, world) if chunks is None else int(chunks)
        log_p, log_k = world.bit_length() - 1, self.K.bit_length() - 1
        self.layout = _lib.MASK_CHUNKED(log_p, log_k) if self.K > 1 else _lib.MASK_MAJOR
        self.chunk_elems = (S // self.K) * d
        self.num = torch.empty(4**n, dtype=torch.int64, device=self.device)
        self.mu = self.ws[:mu_b].view(torch.complex128).view(d, S)
        self.recv = self.ws[mu_b:mu_b + recv_b].view(torch.int64)
        self.theta = self.ws[mu_b + recv_b:mu_b + recv_b + th_b].view(torch.float64)

    def stream(self):
        return self.torch.cuda.current_stream(self.device)

    def partial_numerators(self, counts, count_dtype):
        self.lib.call("lre_step1", counts.data_ptr(), count_dtype, self.n, self.shots, self.w_lo, self.w_hi,
                      self.ws.data_ptr(), self.ws_bytes, self.num.data_ptr(), self.lib.OUT_NUM_I64, self.layout,
                      self.stream().cuda_stream)
        return self.num

    def chunk_in(self, c):
        """Send block of exchange chunk c: every rank's masks of chunk c, rank-major."""
        e = self.chunk_elems * self.world
        return self.num[c * e:(c + 1) * e]

    def chunk_out(self, c):
        return self.recv[c * self.chunk_elems:(c + 1) * self.chunk_elems]

    def finalize_assemble_chunk(self, c):
        d = 1 << self.n
        S = self.m_hi - self.m_lo
        sk = S // self.K
        m0, m1 = self.m_lo + c * sk, self.m_lo + (c + 1) * sk
        off = c * self.chunk_elems
        s = self.stream().cuda_stream
        self.lib.call("lre_finalize", self.recv[off:].data_ptr(), self.n, self.shots, self.lib.MASK_MAJOR, m0 * d,
                      m1 * d, self.theta[off:].data_ptr(), s)
        if self.K == 1:
            self.lib.call("lre_assemble", self.theta.data_ptr(), self.lib.MASK_MAJOR, self.n, self.m_lo, self.m_hi,
                          self.mu.data_ptr(), s)
        else:
            self.lib.call("lre_assemble_slab", self.theta[off:].data_ptr(), self.n, m0, m1, self.m_lo, S,
                          self.mu.data_ptr(), s)
        return self.mu


class ShardedLRE:
    """One rank's share of a P-GPU reconstruction (one process per GPU, torch.distributed)."""

    def __init__(self, compute, group=None):
        self.c = compute
        self.group = group
        self.comm = None
        self.nccl_bytes = 0  # bytes this rank sends per step (reduce-scatter: (P-1)/P of its partial vector)

    def step(self, counts, count_dtype):
        import torch.distributed as dist

        c = self.c
        num = c.partial_numerators(counts, count_dtype)
        P = c.world
        self.nccl_bytes = int(num.numel() * num.element_size() * (P - 1) // P)
        torch = getattr(c, "torch", None)
        on_gpu = torch is not None and getattr(num, "is_cuda", False)
        if not on_gpu or c.K == 1:
            for k in range(c.K):
                dist.reduce_scatter_tensor(c.chunk_out(k), c.chunk_in(k), op=dist.ReduceOp.SUM, group=self.group)
                mu = c.finalize_assemble_chunk(k)
            return mu
        # K reduce-scatters on a side stream; chunk k is finalised/assembled while k+1 transfers
        comp = c.stream()
        if self.comm is None:
            self.comm = torch.cuda.Stream(c.device)
        ready = torch.cuda.Event()
        ready.record(comp)
        self.comm.wait_event(ready)
        done = [torch.cuda.Event() for _ in range(c.K)]
        with torch.cuda.stream(self.comm):
            for k in range(c.K):
                dist.reduce_scatter_tensor(c.chunk_out(k), c.chunk_in(k), op=dist.ReduceOp.SUM, group=self.group)
                done[k].record(self.comm)
        for k in range(c.K):
            comp.wait_event(done[k])
            mu = c.finalize_assemble_chunk(k)
        return mu


    def gather_mu(self, dst: int = 0):
        """The dense row-major mu on rank `dst` (None elsewhere): the slabs gathered over the
        process group (SURVEY §8(e) optional follow-on: one GPU then runs step (iii)).  Rank g's
        slab holds, in row block b, the column block b ^ g."""
        import torch
        import torch.distributed as dist

        c = self.c
        slab = c.mu if isinstance(c.mu, torch.Tensor) else torch.from_numpy(c.mu)
        slab = torch.view_as_real(slab.contiguous())  # complex128 as float64 pairs (gloo has no complex)
        rank = dist.get_rank(self.group)
        P = c.world
        d = 1 << c.n
        S = d // P
        gathered = [torch.empty_like(slab) for _ in range(P)] if rank == dst else None
        dist.gather(slab, gathered, dst=dst, group=self.group)
        if rank != dst:
            return None
        mu = torch.empty((d, d), dtype=torch.complex128, device=slab.device)
        for g, sl in enumerate(torch.view_as_complex(x) for x in gathered):
            for b in range(P):
                mu[b * S:(b + 1) * S, (b ^ g) * S:((b ^ g) + 1) * S] = sl[b * S:(b + 1) * S]
        return mu


class LocalShardedLRE:
    """One process driving P devices (reconstruct(..., devices=P)): the same chunked
    exchange, with the reduce-scatter done as peer-to-peer slice copies (NVLink)
    summed on each destination device."""

    def __init__(self, computes):
        self.cs = list(computes)

    def step(self, counts_list, count_dtype):
        cs = self.cs
        P = len(cs)
        for c, counts in zip(cs, counts_list):
            c.partial_numerators(counts, count_dtype)
        for k in range(cs[0].K):
            for g, dst in enumerate(cs):
                out = dst.chunk_out(k)
                e = dst.chunk_elems
                first = True
                for src in cs:
                    piece = src.chunk_in(k)[g * e:(g + 1) * e]
                    if hasattr(piece, "is_cuda") and piece.device != out.device:
                        piece = piece.to(out.device, non_blocking=True)
                    if first:
                        out.copy_(piece)
                        first = False
                    else:
                        out += piece
                dst.finalize_assemble_chunk(k)
        return [c.mu for c in cs]

    def gather(self):
        """The dense row-major mu (device of rank 0) from the P column slabs."""
        import torch

        c0 = self.cs[0]
        d = 1 << c0.n
        P = len(self.cs)
        S = d // P
        mu = torch.empty((d, d), dtype=torch.complex128, device=c0.device)
        for g, c in enumerate(self.cs):
            slab = c.mu if c.mu.device == c0.device else c.mu.to(c0.device)
            for b in range(P):  # row block b of slab g holds column block b ^ g
                mu[b * S:(b + 1) * S, (b ^ g) * S:((b ^ g) + 1) * S] = slab[b * S:(b + 1) * S]
        return mu

    def theta_mask_major(self):
        """The full mask-major theta (device of rank 0): rank g holds masks [g S, (g+1) S)."""
        c0 = self.cs[0]
        return self.cs[0].torch.cat([c.theta if c.theta.device == c0.device else c.theta.to(c0.device)
                                     for c in self.cs])
