"""Multi-rank exchange logic of the sharded LRE on CPU/gloo.

`distributed.ShardedLRE` is backend-agnostic: production injects
`DeviceCompute` (the CUDA kernels); here an oracle-backed compute object with
the same interface runs under a world-size-2 gloo process group, so the
sharding, the int64 mask-major reduce-scatter and the XOR-block slicing of mu
are checked without a GPU.  The device kernels behind the same calls are
checked by tests/test_gpu_parity.py (TestShardsAndStreaming, mask ranges).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import random_counts
from oracle import c_oracle as C
from oracle import lre_oracle as O
from paper_1602_08604_b200 import distributed as D


def test_shard_ranges_cover_and_align():
    for n in (7, 8, 10, 14):
        q = 3 ** min(n, 7)
        for world in (1, 2, 3, 4, 8):
            rs = D.shard_ranges(n, world, q)
            assert rs[0][0] == 0 and rs[-1][1] == 3**n
            for (lo, hi), (lo2, _) in zip(rs[:-1], rs[1:]):
                assert hi == lo2 and lo % q == 0
            assert all(hi >= lo for lo, hi in rs)


def test_mask_range_partition():
    n = 6
    for world in (1, 2, 4, 8):
        got = [D.mask_range(n, world, g) for g in range(world)]
        assert got[0][0] == 0 and got[-1][1] == 1 << n
        assert all(b - a == (1 << n) // world for a, b in got)
    with pytest.raises(ValueError):
        D.mask_range(n, 3, 0)


class OracleCompute:
    """CPU stand-in for DeviceCompute (same attributes and calls)."""

    def __init__(self, n, shots, w_lo, w_hi, world, rank):
        self.n, self.shots, self.w_lo, self.w_hi = n, shots, w_lo, w_hi
        d = 1 << n
        self.m_lo, self.m_hi = D.mask_range(n, world, rank)
        S = self.m_hi - self.m_lo
        m, a = O.symplectic_index(n)
        self.pos = (m << n) | a  # natural index -> mask-major position
        self.recv = torch.empty(S * d, dtype=torch.int64)

    def partial_numerators(self, counts, count_dtype):
        nat = C.numerators(counts, self.n, self.w_lo)
        mm = np.empty_like(nat)
        mm[self.pos] = nat
        return torch.from_numpy(mm)

    def finalize_and_assemble(self):
        n, d = self.n, 1 << self.n
        mm = np.zeros(4**n, dtype=np.int64)
        mm[self.m_lo * d:self.m_hi * d] = self.recv.numpy()
        theta = O.finalize_numerators(mm[self.pos], n, self.shots)  # natural, zeros outside owned masks
        S = self.m_hi - self.m_lo
        diag = C.step_two_masks(theta, n, self.m_lo, self.m_hi)    # (S, d): mu[r, r^m]
        mu = np.empty((d, S), dtype=np.complex128)
        rows = np.arange(d)
        g = self.m_lo // S
        for j in range(S):
            m = self.m_lo + j
            cols = rows ^ m
            # slab layout of lre_assemble: mu_out[r, c] = mu[r, ((r // S) ^ g) * S + c]
            assert np.all(cols // S == (rows // S) ^ g)
            mu[rows, cols % S] = diag[j]
        return mu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, shots, counts, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_ranges(n, world, 3 ** min(n, 7))[rank]
    comp = OracleCompute(n, shots, lo, hi, world, rank)
    mu = D.ShardedLRE(comp).step(counts[lo:hi], None)
    np.save(f"{out_path}.{rank}.npy", mu)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 8])
def test_world2_gloo_matches_single_rank(tmp_path, rng, n):
    shots = 300
    counts = random_counts(rng, n, shots, np.uint16)
    world = 2
    out = str(tmp_path / "mu")
    mp.spawn(_worker, args=(world, _free_port(), n, shots, counts, out), nprocs=world, join=True)
    theta = C.step_one(counts, n, shots)
    full = C.step_two(theta, n)
    d, S = 1 << n, (1 << n) // world
    for g in range(world):
        slab = np.load(f"{out}.{g}.npy")
        for r in range(0, d, 7):
            cols = ((r // S) ^ g) * S + np.arange(S)
            np.testing.assert_allclose(slab[r], full[r, cols], rtol=1e-12, atol=1e-15)
