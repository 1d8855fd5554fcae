"""ctypes binding of libtomo_b200.so (the C ABI in include/tomo_b200.h).

The library is loaded from this package directory only (built in-tree by
paper_1705_07497_b200/build.py). There is no fallback: if the shared library is missing or
cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("TOMO_LIB_NAME", "libtomo_b200.so"))  # variant builds for A/B runs
_LIB = None

TOMO_OK = 0
TOMO_ERR_CONFIG = 2
TOMO_ERR_NUMERICAL = 3
TOMO_ERR_IO = 4
TOMO_ERR_CUDA = 5

BACKEND_DIRECT = 0
BACKEND_FUSED = 1
BACKEND_SURROGATE = 2
F32 = 0
F64 = 1
NUM_STAGES = 9
STAGE_NAMES = ["t2_rows", "t2_cols", "w_spmv", "wt_spread", "t1_cols", "t1_rows", "cg_update", "sb_post", "stencil"]


class GeomDesc(C.Structure):
    _fields_ = [("n", C.c_int), ("n_angles", C.c_int), ("n_b", C.c_int), ("oversample", C.c_int),
                ("win_lo", C.c_int), ("win_hi", C.c_int), ("tau", C.c_double),
                ("angles", C.POINTER(C.c_double))]


class OpDesc(C.Structure):
    _fields_ = [("backend", C.c_int), ("surrogate_r", C.c_int), ("euclidean", C.c_int), ("device", C.c_int),
                ("angle_begin", C.c_int), ("angle_end", C.c_int), ("max_batch", C.c_int), ("precision", C.c_int),
                ("mem_cap_bytes", C.c_int64)]


class OpInfo(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("n_b", C.c_int), ("n_angles_local", C.c_int),
                ("window", C.c_int), ("P", C.c_int64), ("nnz", C.c_int64), ("wt_rows", C.c_int64),
                ("wt_slots", C.c_int64), ("bytes_w", C.c_int64), ("bytes_wt", C.c_int64),
                ("stencil", C.c_double * 81), ("surrogate_r", C.c_int), ("precision", C.c_int),
                ("backend", C.c_int), ("gram_nnz", C.c_int64), ("gram_slots", C.c_int64),
                ("bytes_gram", C.c_int64), ("herm_nnz", C.c_int64), ("herm_slots", C.c_int64),
                ("herm_touched", C.c_int64), ("herm_tasks", C.c_int),
                ("sym_tasks", C.c_int), ("sym_pairs", C.c_int64), ("sym_P", C.c_int64), ("sym_nnz", C.c_int64),
                ("sym_slots", C.c_int64)]


class System(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("shift", C.c_double)]


class CgStats(C.Structure):
    _fields_ = [("steps_run", C.c_int), ("min_ritz", C.c_double), ("final_rs", C.c_double)]


class SbConfig(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("max_iters", C.c_int), ("cg_steps", C.c_int),
                ("update_tol_rel", C.c_double), ("warm_start", C.c_int), ("sigma_override", C.c_double),
                ("data_feedback", C.c_int)]


class SbTrace(C.Structure):
    _fields_ = [("iterations", C.c_int), ("first_update_l1", C.c_double), ("sigma", C.c_double),
                ("min_ritz", C.c_double), ("imag_leakage", C.c_double), ("stopped_on_tolerance", C.c_int)]


class CpConfig(C.Structure):
    _fields_ = [("alpha", C.c_double), ("lambda_", C.c_double), ("tau_cp", C.c_double),
                ("sigma_cp", C.c_double), ("theta", C.c_double), ("iters", C.c_int), ("cg_steps", C.c_int)]


class TspmMeta(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64), ("symmetric", C.c_int),
                ("n", C.c_int), ("m_sp", C.c_int), ("tau", C.c_double), ("angle_count", C.c_int),
                ("d", C.c_int), ("r", C.c_int)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)

VP = C.c_void_p
EXPORTS = {
    # name: (restype, argtypes)
    "tomo_last_error": (C.c_char_p, []),
    "tomo_kernel_launches": (C.c_int64, []),
    "tomo_op_create": (C.c_int, [C.POINTER(GeomDesc), C.POINTER(OpDesc), C.POINTER(VP)]),
    "tomo_op_destroy": (None, [VP]),
    "tomo_op_get_info": (C.c_int, [VP, C.POINTER(OpInfo)]),
    "tomo_tspm_info": (C.c_int, [C.c_char_p, C.POINTER(TspmMeta)]),
    "tomo_op_create_tspm": (C.c_int, [C.POINTER(GeomDesc), C.POINTER(OpDesc), C.c_char_p, C.POINTER(VP)]),
    "tomo_op_save_tspm": (C.c_int, [VP, C.c_char_p, C.c_int]),
    "tomo_apply_normal": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_apply_normal_real": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_forward": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_forward_real": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_adjoint": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_spmv_w": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_spmv_wt": (C.c_int, [VP, VP, VP, C.c_int, VP]),
    "tomo_backproject": (C.c_int, [VP, C.c_double, C.c_int, VP, VP, C.c_int, VP]),
    "tomo_cg": (C.c_int, [VP, C.POINTER(System), VP, VP, VP, C.c_int, C.c_double, C.c_int, VP, VP]),
    "tomo_split_bregman": (C.c_int, [VP, C.POINTER(SbConfig), VP, VP, C.c_int, VP, VP, VP]),
    "tomo_split_bregman_record": (C.c_int, [VP, C.POINTER(SbConfig), VP, VP, C.c_int, VP, VP, VP, VP, VP, VP, VP]),
    "tomo_tikhonov": (C.c_int, [VP, C.c_double, VP, VP, C.c_int, C.c_double, C.c_int, VP]),
    "tomo_chambolle_pock": (C.c_int, [VP, C.POINTER(CpConfig), VP, VP, C.c_int, VP]),
    "tomo_op_set_allreduce": (C.c_int, [VP, ALLREDUCE_FN, VP]),
    "tomo_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "tomo_op_attach_nccl": (C.c_int, [VP, C.c_char_p, C.c_int, C.c_int]),
    "tomo_grad": (C.c_int, [C.c_int, C.c_int, VP, VP, VP, C.c_int, VP]),
    "tomo_grad_adjoint": (C.c_int, [C.c_int, C.c_int, VP, VP, VP, C.c_int, VP]),
    "tomo_shrink": (C.c_int, [C.c_int64, C.c_int, VP, C.c_double, VP, VP]),
    "tomo_shepp_logan": (C.c_int, [C.c_int, VP]),
    "tomo_random_ellipses": (C.c_int, [C.c_int, C.c_int, C.c_uint64, VP]),
    "tomo_fft_rows": (C.c_int, [C.c_int, C.c_int, C.c_int, VP, VP, C.c_int, VP]),
    "tomo_profile_stages": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, VP, VP, VP]),
}


def lib():
    """Load libtomo_b200.so (raises if it was not built — there is no CPU fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1705_07497_b200.build` "
                              "(the CUDA extension is required; there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def last_error() -> str:
    return lib().tomo_last_error().decode(errors="replace")
