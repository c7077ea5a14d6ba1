"""ctypes front end of oracle/lre_oracle.c — TEST INFRASTRUCTURE ONLY.

Fast CPU restatement of the reference step (i)/(ii) used as a checker at
n = 8..12 and as the CPU baseline in bench.py.  See lre_oracle.c.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liblre_oracle.so")
_DTYPES = {np.dtype(np.uint8): 1, np.dtype(np.uint16): 2, np.dtype(np.int32): 3, np.dtype(np.int64): 4}
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, vp, c_int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        L.lre_oracle_step1_raw.argtypes = [vp, c_int, c_int, i64, i64, i64, c_int, vp]
        L.lre_oracle_numerators.argtypes = [vp, c_int, c_int, i64, i64, c_int, vp]
        L.lre_oracle_gram_divide.argtypes = [vp, c_int]
        L.lre_oracle_step2_masks.argtypes = [vp, c_int, i64, i64, c_int, vp]
        L.lre_oracle_max_threads.restype = c_int
        L.lre_oracle_step1_cost.argtypes = [vp, c_int, c_int, i64, i64, i64, c_int, vp, vp]
        L.lre_oracle_acc_new.restype = vp
        L.lre_oracle_acc_new.argtypes = [c_int, i64, c_int]
        L.lre_oracle_acc_free.argtypes = [vp]
        L.lre_oracle_acc_add.argtypes = [vp, vp, c_int, i64, i64]
        L.lre_oracle_acc_finish.argtypes = [vp, vp]
        L.lre_oracle_step2_scatter.argtypes = [vp, c_int, i64, i64, c_int, vp]
        _lib = L
    return _lib


def _threads(threads):
    return int(threads) if threads else lib().lre_oracle_max_threads()


def step1_raw(counts: np.ndarray, n: int, shots: int, w_begin: int = 0, threads=None) -> np.ndarray:
    """Raw (pre-Gram) accumulation over the settings of a counts block."""
    counts = np.ascontiguousarray(counts)
    raw = np.empty(4**n)
    rc = lib().lre_oracle_step1_raw(counts.ctypes.data, _DTYPES[counts.dtype], n, int(shots),
                                    int(w_begin), int(w_begin) + counts.shape[0], _threads(threads),
                                    raw.ctypes.data)
    if rc:
        raise MemoryError("oracle step1 allocation failed")
    return raw


def step_one(counts: np.ndarray, n: int, shots: int, threads=None) -> np.ndarray:
    """Full reference step (i): theta in natural order (pipeline.py:116-138)."""
    theta = step1_raw(counts, n, shots, 0, threads)
    lib().lre_oracle_gram_divide(theta.ctypes.data, n)
    return theta


def numerators(counts: np.ndarray, n: int, w_begin: int = 0, threads=None) -> np.ndarray:
    counts = np.ascontiguousarray(counts)
    num = np.empty(4**n, dtype=np.int64)
    rc = lib().lre_oracle_numerators(counts.ctypes.data, _DTYPES[counts.dtype], n, int(w_begin),
                                     int(w_begin) + counts.shape[0], _threads(threads), num.ctypes.data)
    if rc:
        raise MemoryError("oracle numerators allocation failed")
    return num


def step_two_masks(theta: np.ndarray, n: int, m_begin: int, m_end: int, threads=None) -> np.ndarray:
    """XOR-diagonals mu[r, r^m] for m in [m_begin, m_end), shape (m_end-m_begin, 2**n)."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    out = np.empty((m_end - m_begin, 1 << n), dtype=np.complex128)
    rc = lib().lre_oracle_step2_masks(theta.ctypes.data, n, int(m_begin), int(m_end),
                                      _threads(threads), out.ctypes.data)
    if rc:
        raise MemoryError("oracle step2 allocation failed")
    return out


def step_two(theta: np.ndarray, n: int, threads=None) -> np.ndarray:
    d = 1 << n
    diag = step_two_masks(theta, n, 0, d, threads)
    mu = np.empty((d, d), dtype=np.complex128)
    rows = np.arange(d)
    for m in range(d):
        mu[rows, rows ^ m] = diag[m]
    return mu


def step1_cost(counts: np.ndarray, n: int, shots: int, w_begin: int = 0, threads=None):
    """(fixed_s, per_setting_per_worker_s) of the reference step (i) on `threads`
    workers, measured on this sample with the partials pre-faulted (see
    lre_oracle.c:lre_oracle_step1_cost)."""
    counts = np.ascontiguousarray(counts)
    fixed = ctypes.c_double(0.0)
    per = ctypes.c_double(0.0)
    rc = lib().lre_oracle_step1_cost(counts.ctypes.data, _DTYPES[counts.dtype], n, int(shots), int(w_begin),
                                     int(w_begin) + counts.shape[0], _threads(threads), ctypes.byref(fixed),
                                     ctypes.byref(per))
    if rc:
        raise MemoryError("oracle step1 allocation failed")
    return fixed.value, per.value


class Step1Accumulator:
    """Step (i) in setting shards with persistent worker partials (lre_oracle_acc_*):
    add(rows, w_begin) for each shard, then finish() -> theta (merge + Gram division)."""

    def __init__(self, n: int, shots: int, threads=None):
        self.n = n
        self.h = lib().lre_oracle_acc_new(n, int(shots), _threads(threads))
        if not self.h:
            raise MemoryError("oracle accumulator allocation failed")

    def add(self, counts: np.ndarray, w_begin: int) -> None:
        counts = np.ascontiguousarray(counts)
        if lib().lre_oracle_acc_add(self.h, counts.ctypes.data, _DTYPES[counts.dtype], int(w_begin),
                                    int(w_begin) + counts.shape[0]):
            raise MemoryError("oracle step1 allocation failed")

    def finish(self, out: np.ndarray | None = None) -> np.ndarray:
        theta = np.empty(4**self.n) if out is None else out
        lib().lre_oracle_acc_finish(self.h, theta.ctypes.data)
        return theta

    def close(self) -> None:
        if self.h:
            lib().lre_oracle_acc_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def step_two_scatter(theta: np.ndarray, n: int, m_begin: int, m_end: int, mu: np.ndarray, threads=None) -> None:
    """Masks [m_begin, m_end) of step (ii) written into the dense mu (complex128, d x d)."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    if lib().lre_oracle_step2_scatter(theta.ctypes.data, n, int(m_begin), int(m_end), _threads(threads),
                                      mu.ctypes.data):
        raise MemoryError("oracle step2 allocation failed")
