"""C ABI library checks that need no GPU: load, exported symbols, layout rules, argument errors."""

import ctypes
import os
import re
import subprocess

import pytest
from conftest import ROOT

from paper_0901_1024_b200 import _capi
from paper_0901_1024_b200.refelem import simplex_node_count

HEADER = os.path.join(ROOT, "include", "dgm.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dgm_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _capi.load()
    declared = header_functions()
    assert declared, "no functions parsed from include/dgm.h"
    assert set(declared) == set(_capi.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (dgm_\w+)", out))
    missing = set(declared) - exported
    assert not missing, missing
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.dgm_version() == _capi.ABI_VERSION


def _odd_chunk_pad(n, w):
    m = n
    while (m * w) % 16 or ((m * w // 16) % 2 == 0):
        m += 1
    return m


@pytest.mark.parametrize("order", range(1, 10))
@pytest.mark.parametrize("dtype,width", [(_capi.DGM_F32, 4), (_capi.DGM_F64, 8)])
def test_layout_rules(order, dtype, width):
    lay = _capi.layout(order, dtype)
    n_p, n_fp = simplex_node_count(order)
    assert (lay.num_nodes, lay.num_face_nodes) == (n_p, n_fp)
    assert lay.np_stride == _odd_chunk_pad(n_p, width)
    assert lay.np_stride * width % 16 == 0 and lay.np_stride >= n_p
    assert lay.vec == 16 // width
    assert lay.diff_chunks * lay.vec >= n_p and lay.lift_chunks * lay.vec >= 4 * n_fp
    assert lay.threads % 32 == 0 and lay.threads <= 1024
    assert lay.smem_bytes_fixed + 192 * n_fp <= 227 * 1024


def test_unsupported_order_and_dtype_raise():
    with pytest.raises(_capi.DgmError, match="order 10"):
        _capi.layout(10, _capi.DGM_F32)
    with pytest.raises(_capi.DgmError, match="dtype"):
        _capi.layout(3, 7)


def test_plan_create_validates_before_touching_cuda():
    lib = _capi.load()
    desc = _capi.Desc(order=3, dtype=0, num_elements=10, field_stride=5)
    handle = ctypes.c_void_p()
    rc = lib.dgm_plan_create(ctypes.byref(desc), ctypes.byref(handle))
    assert rc == -1
    assert b"field_stride" in lib.dgm_last_error()
    desc = _capi.Desc(order=3, dtype=0, num_elements=10, field_stride=10, permittivity=1.0, permeability=1.0)
    rc = lib.dgm_plan_create(ctypes.byref(desc), ctypes.byref(handle))
    assert rc == -1 and b"16-byte" in lib.dgm_last_error()
    with pytest.raises(ValueError):
        _capi.check(lib.dgm_rhs(None, None, None, 0, 0, None), "dgm_rhs")


def test_sass_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
