"""ctypes binding of liblre_b200.so (the C ABI in include/lre_b200.h).

There is no fallback: if the shared library is missing or cannot be loaded
every entry point raises ``RuntimeError`` naming the build command.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# LRE_LIB_PATH: an alternative build of the same library (A/B experiments of
# compile-time variants, tools/debug/); the default is the in-tree build.
LIB_PATH = os.environ.get("LRE_LIB_PATH") or os.path.join(_HERE, "_lib", "liblre_b200.so")

LRE_OK, LRE_EINVAL, LRE_ECUDA, LRE_ENOMEM, LRE_EUNSUPPORTED, LRE_EOVERFLOW = range(6)
U8, U16, I32, I64 = 1, 2, 3, 4
NATURAL, MASK_MAJOR = 0, 1


def MASK_CHUNKED(log_p: int, log_k: int) -> int:
    """LRE_LAYOUT_MASK_CHUNKED(logP, logK) of include/lre_b200.h."""
    return 2 | (log_p << 8) | (log_k << 16)
OUT_THETA_F64, OUT_NUM_I64 = 0, 1
STATE_KINDS = {"maxmixed": 0, "ghz": 1, "productz": 2, "w": 3}
REDUCE_BLOCKS = 1184  # LRE_REDUCE_BLOCKS
REDUCE_SUM_SQ, REDUCE_SUM_SQRT, REDUCE_SUM_SQ_ZC = 0, 1, 2

# name -> (restype, argtypes)
_i64, _i, _vp, _sz, _u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64
_SIGNATURES = {
    "lre_strerror": (ctypes.c_char_p, [_i]),
    "lre_version": (_i, []),
    "lre_launch_count": (_i64, []),
    "lre_shard_quantum": (_i64, [_i]),
    "lre_step1_num_passes": (_i, [_i, _i64]),
    "lre_step1_workspace": (_i, [_i, _i64, _i64, _i64, ctypes.POINTER(_sz)]),
    "lre_step1": (_i, [_vp, _i, _i, _i64, _i64, _i64, _vp, _sz, _vp, _i, _i, _vp]),
    "lre_step1_stage": (_i, [_vp, _i, _i, _i64, _i64, _i64, _vp, _sz, _vp]),
    "lre_step1_finish": (_i, [_vp, _sz, _i, _i64, _vp, _i, _i, _vp]),
    "lre_step1_f64_workspace": (_i, [_i, _i64, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]),
    "lre_step1_f64_quantum": (_i64, [_i]),
    "lre_step1_f64_stage": (_i, [_vp, _i, _i64, _i64, _vp, _sz, _vp, _sz, _vp]),
    "lre_step1_f64_finish": (_i, [_vp, _sz, _i, _vp, _i, _vp]),
    "lre_theta_probabilities": (_i, [_vp, _i, _i64, _i64, _i, _vp, _vp]),
    "lre_finalize": (_i, [_vp, _i, _i64, _i, _i64, _i64, _vp, _vp]),
    "lre_theta_relayout": (_i, [_vp, _i, _i, _vp, _vp]),
    "lre_assemble": (_i, [_vp, _i, _i, _i64, _i64, _vp, _vp]),
    "lre_assemble_slab": (_i, [_vp, _i, _i64, _i64, _i64, _i64, _vp, _vp]),
    "lre_validate_counts": (_i, [_vp, _i, _i, _i64, _i64, _vp, _vp]),
    "lre_generate_counts": (_i, [_i, _i, _i64, _i64, _u64, _i, _i64, _i64, _vp, _i, _vp]),
    "lre_generate_outcomes": (_i, [_i, _i, _i64, _i64, _u64, _i64, _i64, _vp, _vp]),
    "lre_counts_from_outcomes": (_i, [_vp, _i, _i64, _i64, _vp, _i, _vp]),
    "lre_dense_to_theta": (_i, [_vp, _i, _vp, _vp]),
    "lre_generate_counts_theta": (_i, [_vp, _i, _i64, _u64, _i64, _i64, _vp, _i, _vp]),
    "lre_reduce": (_i, [_i, _vp, _vp, _i64, ctypes.c_double, _vp, _vp]),
    "lre_truth_terms": (_i, [_vp, _i, _i, _i64, _vp, _vp]),
}
EXPORTED = tuple(_SIGNATURES)

_lock = threading.Lock()
_lib = None


def load():
    """Load and type the shared library (once)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(or `make -C paper_1602_08604_b200/csrc`); there is no CPU fallback"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str) -> None:
    """Map an lre_status to the reference's exception classes."""
    if status == LRE_OK:
        return
    msg = f"{what}: {load().lre_strerror(status).decode()}"
    if status in (LRE_EINVAL, LRE_EOVERFLOW):
        raise ValueError(msg)
    if status == LRE_ENOMEM:
        raise MemoryError(msg)
    if status == LRE_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().lre_launch_count())
