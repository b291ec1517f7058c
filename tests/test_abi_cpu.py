"""CPU-side checks of the C-ABI boundary (no compute calls: no GPU here).

The shared library must load and export every symbol include/flover_b200.h
declares; descriptor validation must reject bad inputs before touching the
device.
"""

import ctypes as C
import os
import re

import pytest

from paper_2305_13484_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "flover_b200.h")).read()
    return sorted(set(re.findall(r"\b(fl_[a-z_0-9]+)\s*\(", src)))


def test_header_and_loader_agree():
    assert sorted(_lib.EXPORTS) == _declared()


def test_library_loads_and_exports_all_symbols():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2305_13484_b200 import build
        build.build()
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.fl_abi_version() == 1


def test_descriptor_validation_without_gpu():
    lib = _lib.load()
    m = _lib.ModelDesc()
    p = _lib.PoolDesc()
    m.family, m.dtype, m.n_layer, m.d_model, m.n_head, m.head_dim = 0, 1, 2, 256, 4, 64
    m.d_ff, m.vocab, m.tp_size, m.tp_rank = 1024, 1000, 1, 0
    p.pool_slots, p.max_seq, p.max_rows, p.state_slots, p.max_new_tokens = 4, 64, 16, 8, 32
    assert lib.fl_workspace_bytes(C.byref(m), C.byref(p)) > 0
    m.head_dim = 80
    assert lib.fl_workspace_bytes(C.byref(m), C.byref(p)) == 0
    assert b"head_dim" in lib.fl_last_error()
    m.head_dim, m.tp_size = 64, 3
    assert lib.fl_workspace_bytes(C.byref(m), C.byref(p)) == 0
    m.tp_size, m.dtype, p.use_tensor_cores = 1, 0, 1
    assert lib.fl_workspace_bytes(C.byref(m), C.byref(p)) == 0
    h = C.c_void_p()
    m.dtype = 1
    p.use_tensor_cores = 0
    with pytest.raises(Exception):
        _lib.check(lib.fl_create(C.byref(m), C.byref(p), C.byref(h)))   # null workspace
