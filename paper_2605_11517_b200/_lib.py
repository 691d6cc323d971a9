"""ctypes binding of the in-tree C-ABI library ``libgrinder_b200.so``.

The library is the only compute path: if it is missing or cannot load, every
import of a compute entry point raises immediately (there is no CPU
fallback).  Build it with ``make`` at the repository root or
``__graft_entry__.build()``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libgrinder_b200.so"

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f32 = ctypes.c_float
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p


class GrdPartitionerParams(ctypes.Structure):
    _fields_ = [
        ("alpha_balance", c_f64),
        ("beta", c_f64),
        ("epsilon", c_f64),
        ("patience", c_i32),
        ("group_depth", c_i32),
        ("max_iters", c_i32),
        ("reserved", c_i32),
    ]


class GrdAggArgs(ctypes.Structure):
    _fields_ = [
        ("n_rows", c_i64),
        ("row_ptr", c_vp),
        ("idx", c_vp),
        ("out_idx", c_vp),
        ("self_idx", c_vp),
        ("y", c_vp),
        ("ldy", c_i64),
        ("src_scale", c_vp),
        ("post_scale", c_vp),
        ("post_div_deg", c_i32),
        ("relu", c_i32),
        ("out", c_vp),
        ("ldo", c_i64),
        ("width", c_i32),
        ("heavy_threshold", c_i32),
        ("n_heavy", c_i64),
        ("heavy_rows", c_vp),
        ("heavy_seg_ptr", c_vp),
        ("seg_heavy", c_vp),
        ("n_segs", c_i64),
        ("seg_len", c_i32),
        ("no_self", c_i32),
        ("seg_partial", c_vp),
        ("heavy_counter", c_vp),
        ("mask_ref", c_vp),
        ("ld_mask_ref", c_i64),
        ("add_y", c_vp),
        ("ld_add_y", c_i64),
        ("edge_w", c_vp),
        ("edge_w_perm", c_vp),
        ("self_w", c_vp),
        ("heads", c_i32),
        ("head_ld", c_i32),
    ]


class GrdGatArgs(ctypes.Structure):
    _fields_ = [
        ("n_rows", c_i64),
        ("row_ptr", c_vp),
        ("idx", c_vp),
        ("out_idx", c_vp),
        ("edge_perm", c_vp),
        ("heavy_threshold", c_i32),
        ("seg_len", c_i32),
        ("n_heavy", c_i64),
        ("heavy_rows", c_vp),
        ("heavy_seg_ptr", c_vp),
        ("seg_heavy", c_vp),
        ("n_segs", c_i64),
        ("seg_scratch", c_vp),
        ("p_ext", c_vp),
        ("ld_ext", c_i64),
        ("heads", c_i32),
        ("hdp", c_i32),
        ("dhp", c_i32),
        ("slope", c_f32),
        ("alpha", c_vp),
        ("alpha_self", c_vp),
        ("grad_o", c_vp),
        ("ld_go", c_i64),
        ("o_fwd", c_vp),
        ("ld_o", c_i64),
        ("delta", c_vp),
        ("delta_self", c_vp),
        ("grad_ext", c_vp),
        ("ld_gext", c_i64),
        ("st", c_vp),
        ("ld_st", c_i64),
        ("n_small", c_i64),
        ("n_mid", c_i64),
        ("c_dot", c_vp),
        ("alpha_t", c_vp),
        ("seg_wide", c_vp),
    ]


class GrdGemmArgs(ctypes.Structure):
    _fields_ = [
        ("m", c_i64),
        ("n", c_i64),
        ("k", c_i64),
        ("a", c_vp),
        ("lda", c_i64),
        ("trans_a", c_i32),
        ("trans_b", c_i32),
        ("b", c_vp),
        ("ldb", c_i64),
        ("c", c_vp),
        ("ldc", c_i64),
        ("row_scale", c_vp),
        ("elem_mul", c_vp),
        ("ld_elem_mul", c_i64),
        ("relu_ref", c_vp),
        ("ld_relu_ref", c_i64),
        ("relu_out", c_i32),
        ("accumulate", c_i32),
        ("workspace", c_vp),
        ("workspace_elems", c_i64),
        ("c2", c_vp),
        ("ldc2", c_i64),
        ("split", c_i64),
    ]


# name -> (restype, argtypes); mirrors include/grinder_b200.h exactly.
SIGNATURES = {
    "grd_abi_version": (c_i32, []),
    "grd_last_error": (ctypes.c_char_p, []),
    "grd_device_sm_count": (c_i32, [c_vp]),
    "grd_kronecker_generate": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i32]),
    "grd_feature_rows": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "grd_kronecker_keys": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "grd_sa_partition": (c_i32, [c_i64, c_vp, c_vp, c_i32, ctypes.POINTER(GrdPartitionerParams),
                                 c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "grd_sa_analyze": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_f64, c_vp, c_vp, c_vp,
                               c_vp]),
    "grd_sum_sequential": (c_i32, [c_vp, c_i64, c_vp]),
    "grd_plan_create": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "grd_plan_sizes": (c_i32, [c_vp, c_vp, c_vp]),
    "grd_plan_export": (c_i32, [c_vp] + [c_vp] * 9),
    "grd_plan_destroy": (None, [c_vp]),
    "grd_csr_transpose": (c_i32, [c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "grd_csr_same_rows": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "grd_host_gather_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32]),
    "grd_host_scatter_add_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32]),
    "grd_direct_alignment": (c_i64, []),
    "grd_direct_open": (c_i32, [ctypes.c_char_p, c_i32, c_i64, c_vp, c_vp]),
    "grd_direct_close": (c_i32, [c_i32]),
    "grd_direct_read": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_i32]),
    "grd_direct_write": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_i32]),
    "grd_file_runs": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32]),
    "grd_mem_runs": (c_i32, [c_vp, c_i32, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32]),
    "grd_memcpy2d": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp]),
    "grd_gather_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "grd_scatter_add_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "grd_agg_sum": (c_i32, [ctypes.POINTER(GrdAggArgs), c_vp]),
    "grd_gemm": (c_i32, [ctypes.POINTER(GrdGemmArgs), c_vp]),
    "grd_gat_softmax": (c_i32, [ctypes.POINTER(GrdGatArgs), c_vp]),
    "grd_gat_softmax_bwd": (c_i32, [ctypes.POINTER(GrdGatArgs), c_vp]),
    "grd_gat_src_grad": (c_i32, [ctypes.POINTER(GrdGatArgs), c_vp]),
    "grd_gat_pull_bwd": (c_i32, [ctypes.POINTER(GrdGatArgs), c_vp]),
    "grd_gat_dst_grad": (c_i32, [ctypes.POINTER(GrdGatArgs), c_vp]),
    "grd_gat_row_dots": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp]),
    "grd_gat_pack_scores": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_i64, c_vp]),
    "grd_gat_build_wext": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_i64, c_vp]),
    "grd_gat_param_grads": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp,
                                    c_vp, c_f32, c_vp]),
    "grd_head_mean": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, c_i32, c_vp, c_i64, c_i32, c_vp]),
    "grd_gemm_workspace": (c_i64, [c_i64, c_i64]),
    "grd_wgrad_workspace": (c_i64, [c_i64, c_i64, c_i64]),
    "grd_wgrad_sgd": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32,
                              c_vp, c_i64, c_f32, c_vp, c_i64, c_vp]),
    "grd_loss_partials": (c_i64, [c_i64]),
    "grd_softmax_xent": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                 c_vp, c_vp, c_vp]),
    "grd_softmax_xent2": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                  c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "grd_mul_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp]),
    "grd_mask_scale_rows": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp, c_i64,
                                    c_vp]),
    "grd_rownorm_fwd": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_i64, c_vp]),
    "grd_rownorm_bwd": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp,
                                c_i64, c_vp]),
}

_LIB = None


def lib():
    """Load (once) and return the native library; raise if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"native library {LIB_PATH} is missing: run `make` (or "
            f"__graft_entry__.build()) first; there is no CPU fallback")
    handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.grd_abi_version() != 1:
        raise RuntimeError("libgrinder_b200.so ABI version mismatch")
    _LIB = handle
    return handle


def last_error() -> str:
    msg = lib().grd_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Translate a C-ABI return code into the reference's exception types."""
    if rc == 0:
        return
    msg = last_error() or what
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error {rc}: {msg}")


def ptr(array) -> int | None:
    """Raw address of a numpy array / torch tensor (None passes NULL)."""
    if array is None:
        return None
    if hasattr(array, "data_ptr"):
        return array.data_ptr()
    return array.ctypes.data
