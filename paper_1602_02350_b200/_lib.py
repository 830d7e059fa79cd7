"""ctypes binding of the C-ABI (include/skr.h) in lib/libskr_b200.so.

The product path has no fallback: if the CUDA library is missing or cannot be
loaded this module raises at import time of any call site.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libskr_b200.so")

i64, u64, f64, cint = C.c_int64, C.c_uint64, C.c_double, C.c_int
vp, cp = C.c_void_p, C.c_char_p
P = C.POINTER
dptr = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64ptr = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i32ptr = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
lptr = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class SvrgConfigC(C.Structure):
    _fields_ = [("epochs", i64), ("epoch_length", i64), ("step_size", f64), ("seed", u64)]


class EpochRecordC(C.Structure):
    _fields_ = [("epoch", i64), ("objective", f64), ("suboptimality", f64), ("elapsed_ms", f64)]


class SynthSpecC(C.Structure):
    _fields_ = [("n", i64), ("d", i64), ("dtype", cint), ("seed", u64), ("spectrum", cint),
                ("spectrum_param", f64), ("t_scale", cint), ("tau", f64)]


# name -> (restype, argtypes); every symbol include/skr.h declares
SIGNATURES = {
    "skr_last_error": (cp, []),
    "skr_abi_version": (cint, []),
    "skr_ctx_create": (cint, [cint, P(vp)]),
    "skr_nccl_unique_id": (cint, [C.c_char_p]),
    "skr_ctx_create_dist": (cint, [cint, cint, cint, C.c_char_p, P(vp)]),
    "skr_shard_rows": (cint, [i64, cint, cint, P(i64), P(i64)]),
    "skr_shard_layout": (cint, [i64ptr, cint, cint, P(i64), P(i64)]),
    "skr_ctx_destroy": (cint, [vp]),
    "skr_ctx_synchronize": (cint, [vp]),
    "skr_ctx_trim": (cint, [vp, P(i64)]),
    "skr_cumulative_weights": (cint, [vp, dptr, i64, cint, dptr, P(f64)]),
    "skr_ctx_stream": (vp, [vp]),
    "skr_ctx_kernel_launches": (i64, [vp]),
    "skr_ctx_profile": (cint, [vp, cint]),
    "skr_ctx_profile_read": (cint, [vp, cp, P(f64), P(i64)]),
    "skr_ctx_set_prep_cap": (cint, [vp, cint]),
    "skr_data_create": (cint, [vp, vp, i64, i64, cint, P(vp)]),
    "skr_data_create_device": (cint, [vp, vp, i64, i64, i64, cint, P(vp)]),
    "skr_data_scaled": (cint, [vp, f64, P(vp)]),
    "skr_data_info": (cint, [vp, P(i64), P(i64), P(cint), P(f64), P(i64), P(i64)]),
    "skr_data_download": (cint, [vp, vp]),
    "skr_data_destroy": (cint, [vp]),
    "skr_data_generate": (cint, [vp, P(SynthSpecC), P(vp)]),
    "skr_data_labels": (cint, [vp, dptr]),
    "skr_lanczos": (cint, [vp, vp, i64, i64, f64, u64, dptr, dptr, vp, P(i64), P(i64), P(cint)]),
    "skr_problem_create": (cint, [vp, vp, dptr, f64, vp, vp, i64, P(vp)]),
    "skr_problem_create_mode": (cint, [vp, vp, dptr, f64, vp, vp, i64, cint, P(vp)]),
    "skr_problem_mode": (cint, [vp, P(cint)]),
    "skr_problem_destroy": (cint, [vp]),
    "skr_problem_info": (cint, [vp, P(i64), P(i64), P(i64), P(f64), P(f64), P(f64)]),
    "skr_problem_betas": (cint, [vp, dptr]),
    "skr_problem_transformed": (cint, [vp, vp]),
    "skr_objective": (cint, [vp, dptr, P(f64)]),
    "skr_full_gradient": (cint, [vp, dptr, dptr, P(f64)]),
    "skr_full_gradient_device": (cint, [vp, vp, vp, vp]),
    "skr_component_gradient": (cint, [vp, i64, dptr, dptr]),
    "skr_apply_inv_sqrt": (cint, [vp, dptr, dptr]),
    "skr_epoch": (cint, [vp, dptr, dptr, lptr, i64, f64, dptr]),
    "skr_svrg": (cint, [vp, P(SvrgConfigC), dptr, f64, dptr, P(EpochRecordC), P(i64)]),
    "skr_problem_clone": (cint, [vp, vp, P(vp)]),
    "skr_data_create_csr": (cint, [vp, i64, i64, i64ptr, i32ptr, dptr, P(vp)]),
    "skr_data_is_sparse": (cint, [vp, P(cint), P(i64)]),
    "skr_dataset_spectrum": (cint, [vp, vp, dptr]),
    "skr_gram_eigs": (cint, [vp, vp, dptr, dptr]),
    "skr_svrg_until": (cint, [vp, P(SvrgConfigC), dptr, f64, f64, dptr, P(EpochRecordC), P(i64)]),
    "skr_index_stream": (cint, [vp, u64, i64, lptr]),
    "skr_mt_uniforms": (cint, [vp, u64, i64, dptr]),
    "skr_tc_gemm_test": (cint, [vp, vp, vp, i64, i64, i64, cint, dptr]),
    "skr_tc_gemm_mn_test": (cint, [vp, vp, vp, i64, i64, i64, cint, dptr]),
    "skr_gaussian_matrix": (cint, [vp, i64, i64, u64, dptr]),
    "skr_ridge_objective": (cint, [vp, vp, dptr, f64, dptr, P(f64)]),
    "skr_reference_minimum": (cint, [vp, vp, dptr, f64, dptr, P(f64)]),
    "skr_reference_minimum_cg": (cint, [vp, vp, dptr, f64, f64, i64, dptr, P(i64)]),
    "skr_conditioned_cond": (cint, [vp, vp, f64, vp, vp, i64, P(f64)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libskr_b200.so (fails loudly; there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().skr_last_error().decode()
