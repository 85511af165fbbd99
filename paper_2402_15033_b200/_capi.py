"""ctypes declaration of the C ABI in include/krylov_b200.h.

The shared library is built in-tree (paper_2402_15033_b200/libkrylov_b200.so)
by __graft_entry__.build() / `make -C paper_2402_15033_b200/csrc`.  There is
no fallback: if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkrylov_b200.so")

i64 = C.c_int64
i32 = C.c_int32
dbl = C.c_double
P_dbl = C.POINTER(C.c_double)
P_i64 = C.POINTER(C.c_int64)
P_i32 = C.POINTER(C.c_int32)
vp = C.c_void_p

KRY_OK = 0
KRY_DIMENSION_MISMATCH = 1
KRY_NOT_POSITIVE_DEFINITE = 2
KRY_SINGULAR_FACTOR = 3
KRY_SINGULAR_R = 4
KRY_INVALID_ARGUMENT = 5
KRY_UNSUPPORTED = 6
KRY_CUDA_ERROR = 7
KRY_NCCL_ERROR = 8
KRY_NO_DEVICE = 9
KRY_INTERNAL = 10


class kry_solver_config(C.Structure):
    _fields_ = [("restart_len", i64), ("step", i64), ("big_step", i64), ("scheme_kind", i32),
                ("reserved0", i32), ("scheme_big_panel_size", i64), ("rel_tol", dbl), ("max_iters", i64)]


class kry_append_outcome(C.Structure):
    _fields_ = [("committed", i64), ("truncated", i32), ("breakdown", i32), ("pivot", i64),
                ("kappa_estimate", dbl)]


class kry_report(C.Structure):
    _fields_ = [
        ("status", i32), ("breakdown", i32), ("iterations", i64), ("restarts", i64),
        ("initial_residual", dbl), ("final_relative_residual", dbl), ("breakdown_kappa", dbl),
        ("reduces", i64), ("reduces_per_iteration", dbl), ("wall_seconds", dbl),
        ("cycle_residuals", P_dbl), ("cycle_residuals_cap", i64), ("n_cycle_residuals", i64),
        ("per_block", P_i64), ("per_block_cap", i64), ("n_per_block", i64),
        ("per_big_panel", P_i64), ("per_big_panel_cap", i64), ("n_per_big_panel", i64),
        ("mpk_seconds", dbl), ("ortho_seconds", dbl), ("gram_kernel_seconds", dbl),
        ("update_kernel_seconds", dbl), ("restart_seconds", dbl), ("mpk_bytes", dbl),
        ("ortho_bytes", dbl), ("gram_bytes", dbl), ("update_bytes", dbl),
        ("gram_launches", i64), ("update_launches", i64), ("gpu_launches", i64), ("allreduces", i64),
        ("fused_kernel_seconds", dbl), ("fused_bytes", dbl), ("fused_launches", i64),
    ]


class kry_store_info(C.Structure):
    _fields_ = [("rows", i64), ("capacity", i64), ("filled", i64), ("finalized", i64),
                ("big_panel_start", i64), ("panel_size", i64), ("big_panel_size", i64),
                ("seam_valid", i32), ("big_panel_open", i32), ("big_panel_full", i32), ("reserved0", i32),
                ("n_records", i64), ("n_panel_states", i64), ("ld", i64)]


# name -> (restype, argtypes); every symbol declared in include/krylov_b200.h.
SIGNATURES = {
    "kry_abi_version": (C.c_int, []),
    "kry_last_error": (C.c_char_p, []),
    "kry_status_name": (C.c_char_p, [C.c_int]),
    "kry_solver_config_default": (None, [C.POINTER(kry_solver_config)]),
    "kry_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "kry_nccl_unique_id_size": (C.c_int, []),
    "kry_nccl_get_unique_id": (C.c_int, [vp]),
    "kry_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.POINTER(vp)]),
    "kry_ctx_destroy": (C.c_int, [vp]),
    "kry_ctx_synchronize": (C.c_int, [vp]),
    "kry_ctx_set_timing": (C.c_int, [vp, C.c_int]),
    "kry_ctx_launch_count": (C.c_int, [vp, P_i64]),
    "kry_ctx_rank": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "kry_ctx_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "kry_operator_create_csr": (C.c_int, [vp, i64, i64, i64, P_i64, P_i64, P_dbl, C.POINTER(vp)]),
    "kry_operator_create_laplace2d": (C.c_int, [vp, i64, i64, C.POINTER(vp)]),
    "kry_operator_create_laplace3d": (C.c_int, [vp, i64, i64, i64, C.POINTER(vp)]),
    "kry_laplace_partition": (C.c_int, [C.c_int, i64, i64, i64, C.c_int, C.c_int, P_i64, P_i64, P_i64]),
    "kry_operator_destroy": (C.c_int, [vp]),
    "kry_operator_rows": (C.c_int, [vp, P_i64, P_i64, P_i64]),
    "kry_operator_nnz": (C.c_int, [vp, P_i64]),
    "kry_operator_jacobi": (C.c_int, [vp]),
    "kry_store_check_guards": (C.c_int, [vp]),
    "kry_operator_is_jacobi": (C.c_int, [vp, C.POINTER(C.c_int)]),
    "kry_gen_random_sparse": (C.c_int, [i64, i64, i64, i64, C.c_uint64, dbl, C.c_int, P_i64, P_i64, P_dbl]),
    "kry_spmv": (C.c_int, [vp, vp, P_dbl, P_dbl]),
    "kry_spmv_device": (C.c_int, [vp, vp, vp, vp]),
    "kry_mpk": (C.c_int, [vp, vp, P_dbl, i64, P_dbl]),
    "kry_gram": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl]),
    "kry_bcgs_pip_partial": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_bcgs_pip": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_bcgs_pip2": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_cholqr": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_cholqr2": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_bcgs_project": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, P_dbl, P_dbl, P_i64]),
    "kry_bcgs2": (C.c_int, [vp, i64, P_dbl, i64, P_dbl, i64, C.c_int32, P_dbl, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_bcgs_pip_device": (C.c_int, [vp, i64, vp, i64, i64, vp, i64, i64, vp, i64, P_dbl, P_dbl, P_i64, P_i64]),
    "kry_gram_full": (C.c_int, [vp, i64, P_dbl, i64, P_dbl]),
    "kry_store_create": (C.c_int, [vp, i64, i64, i64, i64, C.POINTER(vp)]),
    "kry_store_destroy": (C.c_int, [vp]),
    "kry_store_reset": (C.c_int, [vp]),
    "kry_store_seed_unit_column": (C.c_int, [vp, P_dbl]),
    "kry_store_append_block": (C.c_int, [vp, P_dbl, i64, C.c_int, i32, i64, C.POINTER(kry_append_outcome), P_i64]),
    "kry_store_preprocess_block": (C.c_int, [vp, P_dbl, i64, C.c_int, C.POINTER(kry_append_outcome), P_i64]),
    "kry_store_finalize_big_panel": (C.c_int, [vp, C.POINTER(kry_append_outcome), P_i64]),
    "kry_store_mpk": (C.c_int, [vp, vp, P_dbl, i64, i64]),
    "kry_store_append_inplace": (C.c_int, [vp, i64, C.c_int, i32, i64, C.POINTER(kry_append_outcome), P_i64]),
    "kry_store_get_info": (C.c_int, [vp, C.POINTER(kry_store_info)]),
    "kry_store_coefficients": (C.c_int, [vp, P_dbl]),
    "kry_store_column": (C.c_int, [vp, i64, P_dbl]),
    "kry_store_columns": (C.c_int, [vp, i64, i64, P_dbl]),
    "kry_store_panel_states": (C.c_int, [vp, P_i32]),
    "kry_store_block_record": (C.c_int, [vp, i64, P_i64, P_i64, P_i32, P_dbl, P_dbl]),
    "kry_store_device_ptr": (C.c_int, [vp, C.POINTER(vp), P_i64]),
    "kry_store_hessenberg": (C.c_int, [vp, i64, P_dbl, P_i64]),
    "kry_hessenberg_lsq": (C.c_int, [i64, P_dbl, dbl, P_dbl, P_dbl, P_i64]),
    "kry_try_cholesky": (C.c_int, [i64, P_dbl, P_dbl, P_i64]),
    "kry_sstep_gmres": (C.c_int, [vp, vp, P_dbl, P_dbl, C.POINTER(kry_solver_config), C.POINTER(kry_report), P_dbl]),
    "kry_standard_gmres": (C.c_int, [vp, vp, P_dbl, P_dbl, C.POINTER(kry_solver_config), C.POINTER(kry_report), P_dbl]),
    "kry_sstep_gmres_device": (C.c_int, [vp, vp, vp, vp, C.POINTER(kry_solver_config), C.POINTER(kry_report), vp]),
    "kry_standard_gmres_device": (C.c_int, [vp, vp, vp, vp, C.POINTER(kry_solver_config), C.POINTER(kry_report), vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
