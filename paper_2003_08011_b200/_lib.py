"""ctypes binding of the in-tree C-ABI library ``libcstress_b200.so``.

The library is the product (include/cstress_b200.h).  There is no CPU
fallback: if the library is missing or the device is not an sm_100a part,
every compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcstress_b200.so")
# development tools (tools/timeline.py) may point at an instrumented build
if os.environ.get("CSB_LIB"):
    LIB_PATH = os.path.abspath(os.environ["CSB_LIB"])

_lib = None

P = C.POINTER
d, i64, u64, i32, vp = C.c_double, C.c_int64, C.c_uint64, C.c_int, C.c_void_p
pd, pi64, pu64, pi32 = P(d), P(i64), P(u64), P(i32)

_SIGNATURES = {
    "cs_last_error": (C.c_char_p, []),
    "cs_version": (C.c_char_p, []),
    "cs_ctx_create": (i32, [i32, P(vp)]),
    "cs_ctx_destroy": (i32, [vp]),
    "cs_ctx_set_stream": (i32, [vp, vp]),
    "cs_ctx_reset_stream": (i32, [vp]),
    "cs_ctx_synchronize": (i32, [vp]),
    "cs_ctx_describe": (i32, [vp, C.c_char_p, C.c_size_t]),
    "cs_sim_matrix": (i32, [vp, pd, pd, i64, i64, i64, i32, d, pd]),
    "cs_matmul": (i32, [vp, pd, pd, i64, i64, i64, pd]),
    "cs_batched_solve": (i32, [vp, pd, pd, i64, i64, pd]),
    "cs_symmetric_eig": (i32, [vp, pd, i64, pd, pd]),
    "cs_symmetric_eigvals": (i32, [vp, pd, i64, pd]),
    "cs_select_memory_vectors": (i32, [vp, pd, i64, i64, i64, pi64, pd]),
    "cs_mset_train": (i32, [vp, pd, i64, i64, i64, i32, d, i32, P(vp)]),
    "cs_mset_train_device": (i32, [vp, vp, i64, i64, i64, i32, d, i32, P(vp)]),
    "cs_mset_estimate": (i32, [vp, vp, pd, i64, i64, pd, pd]),
    "cs_mset_estimate_device": (i32, [vp, vp, vp, i32, i64, i64, i64, vp, vp]),
    "cs_model_info": (i32, [vp, pi64, pi64, pi64, pi32, pd, pi32]),
    "cs_model_export": (i32, [vp, pi64, pd, pd, pd, pd]),
    "cs_model_import": (i32, [vp, i64, i64, i32, d, i64, pi64, pd, pd, pd, pd, i32, P(vp)]),
    "cs_model_destroy": (i32, [vp]),
    "cs_model_wire_size": (i32, [vp, pi64]),
    "cs_model_pack_device": (i32, [vp, vp, vp, i64]),
    "cs_model_unpack_device": (i32, [vp, vp, i64, P(vp)]),
    "cs_model_save": (i32, [vp, C.c_char_p]),
    "cs_sprt": (i32, [vp, pd, i64, i64, pd, pd, d, d, pd, P(C.c_uint8), pi64]),
    "cs_sprt_device": (i32, [vp, vp, i32, i64, i64, i64, pd, pd, d, d, pd, vp, pi64]),
    "cs_model_load": (i32, [vp, C.c_char_p, i32, P(vp)]),
    "cs_synthesize_uniform": (i32, [i64, i64, d, d, d, d, d, u64, pd]),
    "cs_synthesize_uniform_device": (i32, [vp, i64, i64, d, d, d, d, d, u64, vp]),
    "cs_synthesize_uniform_device_f32": (i32, [vp, i64, i64, d, d, d, d, d, u64, vp, vp]),
    "cs_derive_seed": (u64, [u64, pu64, i32]),
    "cs_cell_data_seed": (u64, [u64, i64, i64, i64, i32]),
}


def lib():
    """Load the library; raise loudly when it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -m paper_2003_08011_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGNATURES)


def check(code: int) -> None:
    if code != 0:
        raise errors.from_status(code, lib().cs_last_error().decode())


def ptr_d(a: np.ndarray):
    return a.ctypes.data_as(pd)


def ptr_i64(a: np.ndarray):
    return a.ctypes.data_as(pi64)


def f64(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))
