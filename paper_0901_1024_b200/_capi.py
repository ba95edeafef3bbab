"""ctypes binding of libdgm.so (C ABI declared in include/dgm.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_0901_1024_b200/csrc``).  There is no CPU fallback: if the
library is missing every operator call raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGM_LIB") or os.path.join(_HERE, "libdgm.so")
ABI_VERSION = 4
GEO_WORDS = 28

DGM_F32, DGM_F64 = 0, 1
PATH_AUTO, PATH_SIMT, PATH_TENSOR, PATH_TENSOR2 = 0, 1, 2, 3
PATHS = {"auto": PATH_AUTO, "simt": PATH_SIMT, "tensor": PATH_TENSOR, "tensor2": PATH_TENSOR2}
_ERR_NAMES = {-1: "invalid argument", -2: "CUDA error", -3: "unsupported"}


class DgmError(RuntimeError):
    """A libdgm call failed (message from dgm_last_error)."""


class LayoutInfo(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("num_nodes", ctypes.c_int32), ("num_face_nodes", ctypes.c_int32),
                ("np_stride", ctypes.c_int32), ("diff_chunks", ctypes.c_int32),
                ("lift_chunks", ctypes.c_int32), ("vec", ctypes.c_int32),
                ("tile_elements", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("smem_bytes_fixed", ctypes.c_int64), ("tc_supported", ctypes.c_int32),
                ("tc_nb", ctypes.c_int32), ("tc_steps", ctypes.c_int32), ("tc_npk", ctypes.c_int32),
                ("tc_kv", ctypes.c_int32), ("tc_nfpk", ctypes.c_int32), ("tc_operand_floats", ctypes.c_int64),
                ("tc2_supported", ctypes.c_int32), ("tc2_operand_floats", ctypes.c_int64)]


class Desc(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("num_elements", ctypes.c_int64), ("field_stride", ctypes.c_int64),
                ("diff_packed", ctypes.c_void_p), ("lift_packed", ctypes.c_void_p),
                ("geometry", ctypes.c_void_p), ("neighbors", ctypes.c_void_p),
                ("codes", ctypes.c_void_p), ("face_nodes", ctypes.c_void_p),
                ("code_table", ctypes.c_void_p), ("num_codes", ctypes.c_int32),
                ("permittivity", ctypes.c_double), ("permeability", ctypes.c_double),
                ("tc_operand", ctypes.c_void_p), ("path", ctypes.c_int32), ("tc2_operand", ctypes.c_void_p)]


_I64, _VP, _D = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
_SIGNATURES = {
    "dgm_version": ([], ctypes.c_int32),
    "dgm_last_error": ([], ctypes.c_char_p),
    "dgm_layout": ([ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(LayoutInfo)], ctypes.c_int),
    "dgm_plan_create": ([ctypes.POINTER(Desc), ctypes.POINTER(_VP)], ctypes.c_int),
    "dgm_plan_destroy": ([_VP], ctypes.c_int),
    "dgm_plan_path": ([_VP], ctypes.c_int),
    "dgm_rhs": ([_VP, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "dgm_lsrk_stage": ([_VP, _VP, _VP, _VP, _D, _D, _D, _I64, _I64, _VP], ctypes.c_int),
    "dgm_volume": ([_VP, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "dgm_surface": ([_VP, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "dgm_mass_norm": ([_VP, _VP, _VP, _VP, _D, _D, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "dgm_mass_norm_partials": ([_VP, _I64], ctypes.c_int64),
    "dgm_face_states": ([_VP, _VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "dgm_pack": ([ctypes.c_int32, ctypes.c_int32, _VP, ctypes.c_int32, _VP, _VP, _I64, _I64, _VP], ctypes.c_int),
    "dgm_unpack": ([ctypes.c_int32, ctypes.c_int32, _VP, _VP, _VP, ctypes.c_int32, _I64, _I64, _VP], ctypes.c_int),
    "dgm_halo_pack": ([_VP, _VP, _VP, _I64, _VP, _VP], ctypes.c_int),
    "dgm_halo_unpack": ([_VP, _VP, _I64, _I64, _VP, _VP], ctypes.c_int),
    "dgm_trace_pack": ([_VP, _VP, _VP, _I64, _VP, _VP], ctypes.c_int),
    "dgm_trace_unpack": ([_VP, _VP, _VP, _I64, _VP, _VP], ctypes.c_int),
}
EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def load() -> ctypes.CDLL:
    """Load libdgm.so once; raise if it is missing or ABI-incompatible."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DgmError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                       "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.dgm_version() != ABI_VERSION:
        raise DgmError(f"libdgm ABI {lib.dgm_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().dgm_last_error().decode(errors="replace")
        exc = ValueError if rc == -1 else DgmError
        raise exc(f"{what} failed ({_ERR_NAMES.get(rc, rc)}): {msg}")


@dataclass(frozen=True)
class Layout:
    order: int
    dtype: int
    num_nodes: int
    num_face_nodes: int
    np_stride: int
    diff_chunks: int
    lift_chunks: int
    vec: int
    tile_elements: int
    threads: int
    smem_bytes_fixed: int
    tc_supported: int
    tc_nb: int
    tc_steps: int
    tc_npk: int
    tc_kv: int
    tc_nfpk: int
    tc_operand_floats: int
    tc2_supported: int
    tc2_operand_floats: int


def layout(order: int, dtype: int) -> Layout:
    info = LayoutInfo()
    check(load().dgm_layout(int(order), int(dtype), ctypes.byref(info)), "dgm_layout")
    return Layout(*(getattr(info, f) for f, _ in LayoutInfo._fields_))


def stream_handle(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)
