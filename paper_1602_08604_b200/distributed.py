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


def bench_main(args, rank: int, world: int, local: int):
    """bench.py --gpus N under torchrun: max-over-ranks device time per reconstruction."""
    import json
    import statistics

    import torch
    import torch.distributed as dist

    import paper_1602_08604_b200 as lre
    from paper_1602_08604_b200 import _lib
    from paper_1602_08604_b200.simulate import generate_device_counts

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n, shots, seed = args.n, args.shots, args.seed
    q = int(_lib.load().lre_shard_quantum(n))
    lo, hi = shard_ranges(n, world, q)[rank]
    st = lre.StateDescriptor(args.state, n)
    counts = generate_device_counts(st, shots, seed=seed, w_begin=lo, w_end=hi, device=dev)
    rec = lre.DeviceRecord(n=n, shots=shots, counts=counts, w_begin=lo, seed=seed, state=st.label()).validate()
    comp = DeviceCompute(n, shots, lo, hi, world, rank, dev)
    runner = ShardedLRE(comp)
    for _ in range(max(args.warmup, 3)):
        runner.step(counts, rec.lre_dtype)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    l0 = _lib.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    evs[0].record(s)
    for i in range(args.steps):
        runner.step(counts, rec.lre_dtype)
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    dist.barrier()
    per = torch.tensor([evs[i].elapsed_time(evs[i + 1]) / 1e3 for i in range(args.steps)], device=dev)
    dist.all_reduce(per, op=dist.ReduceOp.MAX)
    t = statistics.median(per.cpu().tolist())
    launches = _lib.launch_count() - l0
    if rank == 0:
        c = counts.element_size()
        b = c * 6.0**n + 32.0 * 4.0**n
        print(json.dumps({
            "metric": "14-qubit LRE reconstruction seconds at 1/2/4/8 B200; achieved HBM GB/s",
            "value": t, "unit": "s", "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": t * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": t / ((2.78 + 0.08) * 3600.0) if n == 14 else None,
            "dtype": "i32/i64 exact integer folds, f64 theta/mu",
            "data": "synthetic: device generator per shard, Philox4x32-10 per (seed, setting)",
            "config": {"workload": f"C5: n={n} {args.state.upper()}, settings sharded over {world} GPUs, "
                                   f"int64 numerator reduce-scatter by X-mask", "n": n, "shots": shots,
                       "parallelism": f"settings/{world}, masks/{world}"},
            "whole_path": {"algorithmic_bytes": b, "achieved_GBps": b / t / 1e9},
            "gpu_launches": int(launches),
        }))
    dist.destroy_process_group()
