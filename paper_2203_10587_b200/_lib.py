"""ctypes binding of libacopf_b200.so (the C ABI in include/acopf_b200.h).

There is no fallback: if the shared library is missing or fails to load,
:func:`lib` raises, so the product path can never silently run on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int8, c_int32, c_int64, c_uint8, c_uint32, c_void_p

import numpy as np

from .errors import DeviceError

LIB_NAME = "libacopf_b200.so"
LIB_PATH = os.environ.get("ACOPF_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OBJ, GRAD, CONS, JAC, HESS = 1, 2, 4, 8, 16
ALL = 31
OBJ_PER_STAGE, OBJ_WEIGHTED, OBJ_TERMS = 0, 1, 2

_lib = None

_i32p = POINTER(c_int32)
_i64p = POINTER(c_int64)
_f64p = POINTER(c_double)

_SIGNATURES = {
    "acopf_last_error": (c_char_p, []),
    "acopf_version": (c_int32, []),
    "acopf_topo_create": (c_int32, [c_int32, c_int32, c_int32, _i32p, _i32p, _f64p, POINTER(c_uint8),
                                    _i32p, _f64p, _f64p, POINTER(c_void_p)]),
    "acopf_topo_destroy": (c_int32, [c_void_p]),
    "acopf_batch_create": (c_int32, [c_int32, c_int32, POINTER(c_void_p), c_int32, _i32p, _i64p, _i32p,
                                     _i32p, _i64p, c_int64, _f64p, _f64p, _i32p, _i64p, c_int64,
                                     _f64p, _f64p, _f64p, _f64p, POINTER(c_void_p)]),
    "acopf_batch_destroy": (c_int32, [c_void_p]),
    "acopf_batch_stage_sizes": (c_int32, [c_void_p, _i64p]),
    "acopf_batch_set_layout": (c_int32, [c_void_p, _i64p, c_int32, _i32p, c_int64, _i64p, _i64p, _i64p,
                                         _i64p, POINTER(c_int8)]),
    "acopf_batch_eval": (c_int32, [c_void_p, c_void_p, c_double, c_void_p, c_uint32, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p]),
    "acopf_batch_eval_host": (c_int32, [c_void_p, c_void_p, c_int64, c_double, c_void_p, c_int64, c_uint32,
                                        c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                        c_int64, c_void_p, c_int64, c_void_p]),
    "acopf_batch_flows": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "acopf_batch_pattern": (c_int32, [c_void_p, c_int32, c_int32, c_int64, _i64p, _i32p]),
    "acopf_batch_launches": (c_int64, [c_void_p]),
    "acopf_canonical_order": (c_int32, [c_int64, _i32p, _i32p]),
    "acopf_batch_verify": (c_int32, [c_void_p, _i64p]),
    "acopf_nccl_unique_id": (c_int32, [c_void_p]),
    "acopf_multi_create": (c_int32, [c_void_p, c_int32, c_int32, _i64p, _i64p, _i64p, _i64p, c_int64, _i32p,
                                     c_void_p, POINTER(c_void_p)]),
    "acopf_multi_plan": (c_int32, [c_void_p, _i64p, _i64p, _i64p]),
    "acopf_multi_destroy": (c_int32, [c_void_p]),
    "acopf_batch_eval_multi": (c_int32, [c_void_p, c_void_p, c_double, c_void_p, c_uint32, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p]),
    "acopf_kkt_assemble": (c_int32, [c_int64, c_int64] + [c_void_p] * 19 + [c_double, c_double, c_void_p]),
    "acopf_graph_islands": (c_int32, [c_int32, POINTER(c_uint8), c_int64, _i32p, _i32p, POINTER(c_uint8),
                                      _i32p, _i32p]),
    "acopf_graph_bridges": (c_int32, [c_int32, c_int64, _i32p, _i32p, POINTER(c_uint8), POINTER(c_uint8)]),
    "acopf_copy_runs": (c_int32, [c_int64, _f64p, _i64p, _f64p, _i64p, _i64p]),
    "acopf_format_matrix": (c_int32, [c_char_p, c_int64, _i64p, _f64p, c_void_p, c_int64, _i64p]),
}


def lib() -> ctypes.CDLL:
    """The loaded library (raises DeviceError when it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `python -m paper_2203_10587_b200.build`; there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise DeviceError(lib().acopf_last_error().decode(errors="replace"))


def ptr(a: np.ndarray, ctype):
    """Typed pointer into a contiguous numpy array (caller keeps it alive)."""
    if not a.flags.c_contiguous:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(POINTER(ctype))


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
