"""ctypes view of the C-ABI in include/laq_b200.h.

The product library is paper_2306_08367_b200/_native/liblaq_b200.so, built
in-tree by __graft_entry__.build() (nvcc, sm_100a).  Loading fails loudly when
it is missing: there is no CPU fallback anywhere on the product path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
NATIVE_DIR = os.path.join(_HERE, "_native")
LIB_PATH = os.environ.get("LAQ_LIB_PATH") or os.path.join(NATIVE_DIR, "liblaq_b200.so")  # override: A/B builds
GEN_LIB_PATH = os.path.join(NATIVE_DIR, "liblaq_gen.so")

i64 = C.c_int64
i32 = C.c_int32
vp = C.c_void_p
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class FilterDesc(C.Structure):
    _fields_ = [("target", i32), ("column", C.c_char_p), ("kind", i32), ("is_float", i32),
                ("lo", i64), ("hi", i64), ("set", i64p), ("set_len", i64)]


class PredDesc(C.Structure):
    _fields_ = [("kind", i32), ("is_float", i32), ("ilo", i64), ("ihi", i64), ("flo", C.c_double),
                ("fhi", C.c_double), ("iset", i64p), ("fset", f64p), ("set_len", i64)]


class LinkDesc(C.Structure):
    _fields_ = [("fact_fk", C.c_char_p), ("dim_name", C.c_char_p), ("dim_pk", C.c_char_p)]


class GroupDesc(C.Structure):
    _fields_ = [("target", i32), ("column", C.c_char_p)]


class QueryDesc(C.Structure):
    _fields_ = [("n_joins", i32), ("joins", C.POINTER(LinkDesc)), ("n_filters", i32),
                ("filters", C.POINTER(FilterDesc)), ("measure", C.c_char_p), ("n_group", i32),
                ("group_by", C.POINTER(GroupDesc)), ("order_by", i32)]


# name -> (restype, argtypes)
_SIGS = {
    "laq_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "laq_ctx_destroy": (C.c_int, [vp]),
    "laq_ctx_set_stream": (C.c_int, [vp, vp]),
    "laq_ctx_synchronize": (C.c_int, [vp]),
    "laq_ctx_last_error": (C.c_char_p, [vp]),
    "laq_ctx_launch_count": (i64, [vp]),
    "laq_version": (C.c_char_p, []),
    "laq_nccl_unique_id": (C.c_int, [vp]),
    "laq_ctx_attach_nccl": (C.c_int, [vp, i32, i32, vp]),
    "laq_ctx_set_allreduce_host": (C.c_int, [vp, i32, i32, vp, vp]),
    "laq_ctx_comm_info": (C.c_int, [vp, i32p, i32p]),
    "laq_allreduce_acc": (C.c_int, [vp, vp, i64]),
    "laq_build_key_domain": (C.c_int, [vp, vp, i64, vp, i64, vp, i64p]),
    "laq_update_key_domain": (C.c_int, [vp, vp, i64, vp, i64, vp, i64p]),
    "laq_key_positions": (C.c_int, [vp, vp, i64, vp, i64, vp]),
    "laq_key_matrix_dbr": (C.c_int, [vp, vp, i64, vp, i64, vp, vp, vp, vp, i64p]),
    "laq_mm_join": (C.c_int, [vp, vp, i64, vp, i64, vp, vp, i64, i64p]),
    "laq_star_join": (C.c_int, [vp, i32, vp, i64, vp, i64p, vp, vp, i64p]),
    "laq_dense_matmul": (C.c_int, [vp, vp, i64, i64, vp, i64, vp]),
    "laq_spmm_dense": (C.c_int, [vp, vp, vp, vp, i64, vp, i64, i64, vp]),
    "laq_place_columns": (C.c_int, [vp, vp, i64, i64, i64p, i64p, f64p, i64, i64, vp]),
    "laq_prefuse_linear": (C.c_int, [vp, i32, vp, i64p, i64p, vp, vp, i64, i64, vp]),
    "laq_apply_fused_linear": (C.c_int, [vp, i32, vp, i64, vp, i64p, i64, vp]),
    "laq_materialize": (C.c_int, [vp, i32, vp, i64, vp, i64p, i64p, vp, i64, vp]),
    "laq_fused_star_predict": (C.c_int, [vp, i32, vp, i64, vp, i64p, vp, i64, vp, vp, i64p]),
    "laq_probe_build": (C.c_int, [vp, i32, vp, i64p, C.POINTER(vp)]),
    "laq_probe_fused_predict": (C.c_int, [vp, vp, vp, i64, vp, i64, vp, vp, vp]),
    "laq_probe_fused_predict_host": (C.c_int, [vp, vp, vp, i64, i64, vp, i64, vp]),
    "laq_probe_destroy": (C.c_int, [vp]),
    "laq_probe_bind_partials": (C.c_int, [vp, vp, vp, i64]),
    "laq_probe_join_rows": (C.c_int, [vp, vp, vp, i64, vp, vp, vp]),
    "laq_ffn_create": (C.c_int, [vp, i32, vp, i64p, i64p, vp, i64, vp, i64, vp, i64, C.POINTER(vp)]),
    "laq_ffn_predict_rows": (C.c_int, [vp, vp, vp, i64, vp]),
    "laq_ffn_predict_star": (C.c_int, [vp, vp, vp, vp, i64, vp, vp, i64p]),
    "laq_ffn_destroy": (C.c_int, [vp]),
    "laq_tc_features_create": (C.c_int, [vp, i32, vp, i64p, i64p, vp, i64, C.POINTER(vp)]),
    "laq_tc_features_destroy": (C.c_int, [vp]),
    "laq_tc_gemm": (C.c_int, [vp, vp, vp, i64, vp, i64, vp]),
    "laq_apply_fused_linear_f32": (C.c_int, [vp, i32, vp, i64, vp, i64, vp]),
    "laq_tree_partial": (C.c_int, [vp, vp, i64, i64, i64, i64p, f64p, f64p, f64p, i64, vp]),
    "laq_apply_fused_tree": (C.c_int, [vp, i32, vp, i64, vp, i64, f64p, i64p, vp, i64p, i32p]),
    "laq_groupby_sum_single": (C.c_int, [vp, vp, vp, i64, vp, vp, i64, vp, vp, i64p]),
    "laq_groupby_sum_multi": (C.c_int, [vp, i32, vp, vp, i64, vp, vp, i64, i64p]),
    "laq_sort_rows": (C.c_int, [vp, vp, i64, i64, i64p, i32p, i32, vp]),
    "laq_coo_check": (C.c_int, [vp, vp, vp, i64, i64, i64]),
    "laq_csr_from_coo": (C.c_int, [vp, vp, vp, i64, i64, i64, vp]),
    "laq_coo_from_csr": (C.c_int, [vp, vp, i64, i64, vp]),
    "laq_spmm": (C.c_int, [vp, vp, vp, vp, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i64, i64p]),
    "laq_selection_mask": (C.c_int, [vp, vp, i32, i64, vp, vp, i32]),
    "laq_mask_and": (C.c_int, [vp, vp, vp, i64, vp]),
    "laq_mask_indices": (C.c_int, [vp, vp, i64, vp, i64p]),
    "laq_gather": (C.c_int, [vp, vp, i32, i64, vp, i64, vp, i32]),
    "laq_sum_f64": (C.c_int, [vp, vp, i64, f64p]),
    "laq_star_create": (C.c_int, [vp, C.POINTER(vp)]),
    "laq_star_destroy": (C.c_int, [vp]),
    "laq_star_add_table": (C.c_int, [vp, C.c_char_p, i32, i64, i32, vp, i32p, i32, vp]),
    "laq_star_add_table_device_bitpacked": (C.c_int, [vp, C.c_char_p, i32, i64, i32, vp, i32p, vp, i32p, i32p]),
    "laq_csv_open": (C.c_int, [vp, vp, i64, C.POINTER(vp), i64p]),
    "laq_csv_parse": (C.c_int, [vp, vp, i32, i32p, vp]),
    "laq_csv_close": (C.c_int, [vp]),
    "laq_star_add_table_device": (C.c_int, [vp, C.c_char_p, i32, i64, i32, vp, i32p, vp]),
    "laq_star_add_table_device_packed": (C.c_int, [vp, C.c_char_p, i32, i64, i32, vp, i32p, vp, i32p, i32p]),
    "laq_star_add_link": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p]),
    "laq_query_prepare": (C.c_int, [vp, vp, C.POINTER(QueryDesc), C.POINTER(vp), i64p]),
    "laq_plan_execute": (C.c_int, [vp, vp, vp, i32]),
    "laq_plan_build_codes": (C.c_int, [vp, vp]),
    "laq_plans_build_codes": (C.c_int, [vp, i32, vp]),
    "laq_plans_scan_shared": (C.c_int, [vp, i32, vp, vp, i32, i32p]),
    "laq_plan_scan": (C.c_int, [vp, vp, vp, i32]),
    "laq_batch_prepare": (C.c_int, [vp, i32, vp, C.POINTER(vp), i32p]),
    "laq_batch_build": (C.c_int, [vp, vp]),
    "laq_batch_scan": (C.c_int, [vp, vp, vp, i32]),
    "laq_batch_info": (C.c_int, [vp, i32p, i64p, i32p, C.c_char_p, C.c_size_t]),
    "laq_batch_destroy": (C.c_int, [vp]),
    "laq_plan_scan_range": (C.c_int, [vp, vp, i64, i64, vp, i32]),
    "laq_plan_bytes_per_row": (i64, [vp]),
    "laq_plan_scanned_links": (i32, [vp]),
    "laq_plan_emit": (C.c_int, [vp, i64p, f64p, i64, i64p, i64p]),
    "laq_plan_destroy": (C.c_int, [vp]),
    "laq_run_query": (C.c_int, [vp, vp, C.POINTER(QueryDesc), f64p, i64, i64p, i64p]),
    "laq_measure_selectivity": (C.c_int, [vp, vp, C.POINTER(QueryDesc), f64p]),
    "laq_speedup_ratio_linear": (C.c_int, [i64, i64, i64, i64p, i32, f64p]),
    "laq_speedup_ratio_tree": (C.c_int, [i64, i64, i64, i64, i64p, i32, f64p]),
    "laq_decide_fusion": (C.c_int, [C.c_double, C.c_double, i32p]),
    "laq_plan_linear_device": (C.c_int, [i64, i64, i64, i64p, i32, C.c_double, C.c_double, f64p, f64p, i32p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.CudaError(
                f"{LIB_PATH} is missing: the CUDA extension was not built "
                "(run __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


# laq_allreduce_host_fn: int (*)(int64_t* h_buf, int64_t count, void* user)
ALLREDUCE_HOST_FN = C.CFUNCTYPE(C.c_int, i64p, i64, vp)


def ptr_array(ptrs):
    """Array of void* from ints (device pointers) or None."""
    arr = (vp * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p if p else None
    return arr


def i64_array(vals):
    return (i64 * max(1, len(vals)))(*[int(v) for v in vals])
