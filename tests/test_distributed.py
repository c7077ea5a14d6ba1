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
    """CPU stand-in for DeviceCompute (same attributes and calls, incl. the chunked exchange)."""

    def __init__(self, n, shots, w_lo, w_hi, world, rank, chunks=1):
        self.n, self.shots, self.w_lo, self.w_hi = n, shots, w_lo, w_hi
        self.world, self.rank, self.K = world, rank, chunks
        d = 1 << n
        self.m_lo, self.m_hi = D.mask_range(n, world, rank)
        S = self.m_hi - self.m_lo
        m, a = O.symplectic_index(n)
        log_p, log_k = world.bit_length() - 1, chunks.bit_length() - 1
        mp_ = np.array([D.mask_position(int(x), n, log_p, log_k) for x in range(d)], dtype=np.int64)
        self.pos = (mp_[m] << n) | a  # natural index -> (chunked) mask-major position
        self.chunk_elems = (S // chunks) * d
        self.recv = torch.empty(S * d, dtype=torch.int64)
        self.mu = np.empty((d, S), dtype=np.complex128)

    def partial_numerators(self, counts, count_dtype):
        nat = C.numerators(counts, self.n, self.w_lo)
        mm = np.empty_like(nat)
        mm[self.pos] = nat
        self.num = torch.from_numpy(mm)
        return self.num

    def chunk_in(self, c):
        e = self.chunk_elems * self.world
        return self.num[c * e:(c + 1) * e]

    def chunk_out(self, c):
        return self.recv[c * self.chunk_elems:(c + 1) * self.chunk_elems]

    def finalize_assemble_chunk(self, c):
        n, d = self.n, 1 << self.n
        S = self.m_hi - self.m_lo
        sk = S // self.K
        m0 = self.m_lo + c * sk
        # the chunk's numerators: masks [m0, m0 + sk), mask-major
        full = np.zeros(4**n, dtype=np.int64)
        full[m0 * d:(m0 + sk) * d] = self.chunk_out(c).numpy()
        m, a = O.symplectic_index(n)
        theta = O.finalize_numerators(full[(m << n) | a], n, self.shots)  # natural, zeros outside the chunk
        diag = C.step_two_masks(theta, n, m0, m0 + sk)  # (sk, d): mu[r, r^m]
        rows = np.arange(d)
        g = self.m_lo // S
        for j in range(sk):
            cols = rows ^ (m0 + j)
            # slab layout of lre_assemble: mu_out[r, c] = mu[r, ((r // S) ^ g) * S + c]
            assert np.all(cols // S == (rows // S) ^ g)
            self.mu[rows, cols % S] = diag[j]
        return self.mu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, shots, counts, out_path, chunks=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_ranges(n, world, 3 ** min(n, 7))[rank]
    comp = OracleCompute(n, shots, lo, hi, world, rank, chunks)
    runner = D.ShardedLRE(comp)
    mu = runner.step(counts[lo:hi], None)
    np.save(f"{out_path}.{rank}.npy", mu)
    full = runner.gather_mu(dst=0)  # dense mu on rank 0 (step iii input)
    if rank == 0:
        np.save(f"{out_path}.full.npy", full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world,chunks", [(7, 2, 1), (8, 2, 1), (8, 2, 4), (8, 4, 1), (8, 4, 2)])
def test_gloo_exchange_matches_single_rank(tmp_path, rng, n, world, chunks):
    """world 2 and 4, whole-slice and chunked (MASK_CHUNKED layout) reduce-scatters."""
    shots = 300
    counts = random_counts(rng, n, shots, np.uint16)
    out = str(tmp_path / "mu")
    mp.spawn(_worker, args=(world, _free_port(), n, shots, counts, out, chunks), nprocs=world, join=True)
    theta = C.step_one(counts, n, shots)
    full = C.step_two(theta, n)
    np.testing.assert_allclose(np.load(f"{out}.full.npy"), full, rtol=1e-12, atol=1e-15)
    d, S = 1 << n, (1 << n) // world
    for g in range(world):
        slab = np.load(f"{out}.{g}.npy")
        for r in range(0, d, 7):
            cols = ((r // S) ^ g) * S + np.arange(S)
            np.testing.assert_allclose(slab[r], full[r, cols], rtol=1e-12, atol=1e-15)


def test_mask_chunked_layout_is_a_permutation():
    for n, lp, lk in [(4, 1, 1), (8, 2, 2), (8, 3, 0), (10, 0, 2)]:
        pos = [D.mask_position(m, n, lp, lk) for m in range(1 << n)]
        assert sorted(pos) == list(range(1 << n))
        S, K = (1 << n) >> lp, 1 << lk
        for m in range(1 << n):  # chunk c of rank g lands in block c, sub-block g
            g, c, j = m // S, (m % S) // (S // K), m % (S // K)
            assert pos[m] == (c * (1 << lp) + g) * (S // K) + j


def test_local_multi_device_exchange_matches_single(rng):
    """LocalShardedLRE (one process, P 'devices') with oracle compute objects, chunked."""
    n, shots, P = 8, 200, 4
    counts = random_counts(rng, n, shots, np.uint16)
    q = 3 ** min(n, 7)
    cs = [OracleCompute(n, shots, lo, hi, P, g, 2) for g, (lo, hi) in enumerate(D.shard_ranges(n, P, q))]
    slabs = D.LocalShardedLRE(cs).step([counts[c.w_lo:c.w_hi] for c in cs], None)
    full = C.step_two(C.step_one(counts, n, shots), n)
    d, S = 1 << n, (1 << n) // P
    for g, slab in enumerate(slabs):
        for r in range(0, d, 5):
            cols = ((r // S) ^ g) * S + np.arange(S)
            np.testing.assert_allclose(slab[r], full[r, cols], rtol=1e-12, atol=1e-15)
