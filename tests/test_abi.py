"""The C ABI boundary (CPU-only: no compute calls without a GPU).

The library must load on a CPU-only host, export every function declared in
include/lre_b200.h, and the Python binding (_lib.py) must type every one of
them.  Status/error mapping follows SURVEY §8(b).
"""

import os
import re

import pytest

from paper_1602_08604_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lre_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lre_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("lre_step1", "lre_step1_workspace", "lre_step1_stage", "lre_step1_finish", "lre_assemble",
                 "lre_finalize", "lre_validate_counts", "lre_generate_counts", "lre_theta_relayout"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_types_every_declared_symbol():
    assert set(declared_functions()) == set(_lib.EXPORTED)


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.lre_version() >= 200
    assert lib.lre_strerror(_lib.LRE_EINVAL) == b"invalid argument"
    assert lib.lre_shard_quantum(14) == 3**7
    assert lib.lre_shard_quantum(5) == 3**5
    assert lib.lre_step1_num_passes(14, 1000) == 4      # tile pass (7) + 3 + 3 + 1
    assert lib.lre_step1_num_passes(12, 1000) == 3      # 7 + 3 + 2
    assert lib.lre_step1_num_passes(4, 16) == 2         # 2 + 2 (vector passes from raw counts)
    assert lib.lre_step1_num_passes(14, 3_000_000_000) == 7  # int64 plan: 2-qubit passes
    import ctypes

    ws = ctypes.c_size_t(0)
    assert lib.lre_step1_workspace(14, 1000, 0, 3**14, ctypes.byref(ws)) == _lib.LRE_OK
    # split Y1 storage (lre_step1.cu make_plan): int16 low halves + high-part rows of 1184 per 16384
    e1, e2 = 4**7 * 3**7 * 2**7, 4**10 * 3**4 * 2**4
    y1, y2 = (e1 + e1 // 16384 * 1184) * 2, (e2 + e2 // 16384 * 1184) * 4
    if os.environ.get("LRE_Y1SPLIT") == "0":
        y1, y2 = e1 * 4, e2 * 4
    assert ws.value >= y1 + y2 and ws.value < y1 + y2 + 4096


def test_argument_errors_map_to_reference_exceptions():
    import ctypes

    lib = _lib.load()
    ws = ctypes.c_size_t(0)
    with pytest.raises(ValueError):
        _lib.check(lib.lre_step1_workspace(0, 10, 0, 1, ctypes.byref(ws)), "lre_step1_workspace")
    with pytest.raises(ValueError):
        _lib.check(lib.lre_step1_workspace(3, 10, 5, 5, ctypes.byref(ws)), "lre_step1_workspace")
    with pytest.raises(MemoryError):
        _lib.check(_lib.LRE_ENOMEM, "x")
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.LRE_EUNSUPPORTED, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.LRE_ECUDA, "x")


def test_outcome_record_host_histogram():
    """OutcomeRecord.to_counts: the host restatement of lre_counts_from_outcomes."""
    import numpy as np
    from paper_1602_08604_b200.records import OutcomeRecord

    rng = np.random.default_rng(0)
    n, shots = 3, 50
    o = rng.integers(0, 8, size=(27, shots), dtype=np.uint16)
    rec = OutcomeRecord(n=n, shots=shots, outcomes=o).to_counts()
    assert rec.counts.shape == (27, 8) and rec.counts.dtype == np.uint8
    assert (rec.counts.sum(axis=1) == shots).all()
    for w in (0, 13, 26):
        np.testing.assert_array_equal(rec.counts[w], np.bincount(o[w], minlength=8))
