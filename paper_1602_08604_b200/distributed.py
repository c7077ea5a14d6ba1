"""Multi-GPU LRE: one process per GPU, settings sharded, one exchange step.

SURVEY §8(e): rank g owns a contiguous, quantum-aligned range of settings
(its counts are generated in place or copied from its slice of the record);
it folds them into a full-length partial numerator vector N_g (exact int64,
MASK_MAJOR layout, index m*2^n + a); one ``reduce_scatter`` (sum) over
NCCL/NVLink leaves rank g with the complete numerators of X-masks
[g*2^n/P, (g+1)*2^n/P); it finalises them to theta and assembles its
XOR-block slice of mu: rows r, columns ((r/S) ^ g)*S + c, S = 2^n/P.
Integer numerators make the result bit-identical for every P.

The orchestration is backend-agnostic: ``ShardedLRE`` takes the torch
process group plus a ``compute`` object; production uses ``DeviceCompute``
(the CUDA kernels of liblre_b200.so), the gloo tests inject the CPU oracle to
check the exchange logic (tests/test_distributed.py).
"""

from __future__ import annotations

import os
import time


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


class DeviceCompute:
    """The production compute backend: liblre_b200.so kernels on one GPU."""

    def __init__(self, n: int, shots: int, w_lo: int, w_hi: int, world: int, rank: int, device):
        import ctypes

        import torch

        from . import _lib

        self.torch, self.lib = torch, _lib
        self.n, self.shots, self.w_lo, self.w_hi = n, shots, w_lo, w_hi
        self.device = device
        ws = ctypes.c_size_t(0)
        _lib.check(_lib.load().lre_step1_workspace(n, shots, w_lo, w_hi, ctypes.byref(ws)), "lre_step1_workspace")
        self.ws_bytes = int(ws.value)
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=device)
        d = 1 << n
        self.m_lo, self.m_hi = mask_range(n, world, rank)
        S = self.m_hi - self.m_lo
        self.num = torch.empty(4**n, dtype=torch.int64, device=device)
        self.recv = torch.empty(S * d, dtype=torch.int64, device=device)
        self.theta = torch.empty(S * d, dtype=torch.float64, device=device)
        self.mu = torch.empty((d, S), dtype=torch.complex128, device=device)

    def stream(self):
        return self.torch.cuda.current_stream(self.device)

    def partial_numerators(self, counts, count_dtype):
        self.lib.call("lre_step1", counts.data_ptr(), count_dtype, self.n, self.shots, self.w_lo, self.w_hi,
                      self.ws.data_ptr(), self.ws_bytes, self.num.data_ptr(), self.lib.OUT_NUM_I64,
                      self.lib.MASK_MAJOR, self.stream().cuda_stream)
        return self.num

    def finalize_and_assemble(self):
        d = 1 << self.n
        self.lib.call("lre_finalize", self.recv.data_ptr(), self.n, self.shots, self.lib.MASK_MAJOR,
                      self.m_lo * d, self.m_hi * d, self.theta.data_ptr(), self.stream().cuda_stream)
        self.lib.call("lre_assemble", self.theta.data_ptr(), self.lib.MASK_MAJOR, self.n, self.m_lo, self.m_hi,
                      self.mu.data_ptr(), self.stream().cuda_stream)
        return self.mu


class ShardedLRE:
    """One rank's share of a P-GPU reconstruction."""

    def __init__(self, compute, group=None):
        self.c = compute
        self.group = group

    def step(self, counts, count_dtype):
        import torch.distributed as dist

        num = self.c.partial_numerators(counts, count_dtype)
        dist.reduce_scatter_tensor(self.c.recv, num, op=dist.ReduceOp.SUM, group=self.group)
        return self.c.finalize_and_assemble()
