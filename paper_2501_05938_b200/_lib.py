"""Loads libpm_tridiag.so (built in-tree by build.py) and declares its C ABI.

There is no Python or CPU fallback: if the native library is missing or
cannot be loaded, importing the solver raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("PM_LIB_PATH") or Path(__file__).resolve().parent / "libpm_tridiag.so")

_D = C.POINTER(C.c_double)
_CD = C.c_void_p  # device / host pointers are passed as integers


class StageTimingsC(C.Structure):
    _fields_ = [("slae_size", C.c_uint64), ("t1_h2d", C.c_double), ("t1_comp", C.c_double),
                ("t1_d2h", C.c_double), ("t2_comp", C.c_double), ("t3_h2d", C.c_double),
                ("t3_comp", C.c_double), ("t3_d2h", C.c_double)]


class ModelBundleC(C.Structure):
    _fields_ = [("sum_a", C.c_double), ("sum_b", C.c_double), ("small_a", C.c_double),
                ("small_b", C.c_double), ("small_c", C.c_double), ("big_a", C.c_double),
                ("big_b", C.c_double), ("big_c", C.c_double), ("size_threshold", C.c_uint64),
                ("num_candidates", C.c_int32), ("candidates", C.c_int32 * 5)]


# (name, restype, argtypes) of every symbol include/pm_tridiag.h and
# include/streamtune_c.h declare; tests check the library exports all of them.
_ERR = [C.c_char_p, C.c_int]
# int allgather(const void* send, void* recv, int64_t bytes_per_rank, void* stream, void* user)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)

PM_SIGNATURES = [
    ("pm_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    ("pm_destroy", C.c_int, [C.c_void_p]),
    ("pm_last_error", C.c_char_p, [C.c_void_p]),
    ("pm_set_option", C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    ("pm_get_version", C.c_int, []),
    ("pm_solve_device_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_solve_batch_device_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_check", C.c_int, [C.c_void_p]),
    ("pm_solve_host_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32]),
    ("pm_last_stage_timings", C.c_int,
     [C.c_void_p, C.POINTER(StageTimingsC), C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    ("pm_host_register", C.c_int, [C.c_void_p, C.c_uint64]),
    ("pm_host_unregister", C.c_int, [C.c_void_p]),
    ("pm_set_model_bundle", C.c_int, [C.c_void_p, C.POINTER(ModelBundleC)]),
    ("pm_get_model_bundle", C.c_int, [C.c_void_p, C.POINTER(ModelBundleC)]),
    ("pm_recommend_streams", C.c_int, [C.c_int64, C.POINTER(ModelBundleC)]),
    ("pm_paper_bundle", C.c_int, [C.POINTER(ModelBundleC)]),
    ("pm_b200_bundle", C.c_int, [C.POINTER(ModelBundleC)]),
    ("pm_generate_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_uint64, C.c_void_p]),
    ("pm_dist_reduce_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _CD, C.c_void_p]),
    ("pm_dist_solve_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _CD, C.c_void_p]),
    ("pm_generate_range_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]),
    # FP32 variants (same signatures on float arrays)
    ("pm_solve_device_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_solve_batch_device_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_solve_host_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32]),
    ("pm_generate_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_uint64, C.c_void_p]),
    ("pm_generate_range_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]),
    ("pm_dist_reduce_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _CD, C.c_void_p]),
    ("pm_dist_solve_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _CD, C.c_void_p]),
    ("pm_solve_batch_host_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64]),
    ("pm_solve_batch_host_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int64]),
    # P2P interface exchange
    ("pm_dist_exchange_bytes", C.c_int64, [C.c_int32]),
    ("pm_dist_exchange_alloc", C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("pm_dist_set_peers", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_int32]),
    ("pm_ipc_get_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("pm_ipc_open_handle", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("pm_ipc_close_handle", C.c_int, [C.c_void_p]),
    ("pm_dist_reduce_p2p_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_dist_solve_p2p_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_dist_reduce_p2p_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_dist_solve_p2p_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p]),
    ("pm_solve_dist_f64", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32,
                                    C.c_int32, ALLGATHER_FN, C.c_void_p, C.c_void_p]),
    ("pm_solve_dist_f32", C.c_int, [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_int32,
                                    C.c_int32, ALLGATHER_FN, C.c_void_p, C.c_void_p]),
    ("pm_solve_dist_nccl_f64", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("pm_solve_dist_nccl_f32", C.c_int,
     [C.c_void_p, _CD, _CD, _CD, _CD, _CD, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    ("pm_nccl_version", C.c_int, []),
    ("pm_nccl_get_unique_id", C.c_int, [C.c_void_p, C.c_void_p]),
    ("pm_nccl_comm_init", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32]),
    ("pm_nccl_comm_destroy", C.c_int, [C.c_void_p, C.c_void_p]),
    ("pm_last_launch_count", C.c_int, [C.c_void_p]),
    ("pm_kernel_times", C.c_int,
     [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_float), C.c_int32]),
    ("pm_last_plan", C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]),
    ("pm_last_batch_plan", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("pm_last_stream_plan", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("pm_batch_stream_stats", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    ("pm_batch_stream_counters", C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.c_int64]),
    ("pm_batch_stream_timeline", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64]),
    # streamtune_c.h
    ("st_stream_count_is_valid", C.c_int, [C.c_int]),
    ("st_validate_stage_timings", C.c_int, [C.POINTER(StageTimingsC)] + _ERR),
    ("st_total_unstreamed", C.c_double, [C.POINTER(StageTimingsC)]),
    ("st_overlap_sum", C.c_double, [C.POINTER(StageTimingsC)]),
    ("st_streamed_lower_bound", C.c_int, [C.POINTER(StageTimingsC), C.c_int, C.c_double, _D] + _ERR),
    ("st_overhead_from_measurement", C.c_int,
     [C.c_double, C.c_double, C.c_int, C.c_double, _D] + _ERR),
    ("st_overlap_benefit", C.c_int, [C.c_int, C.c_double, C.c_double, _D] + _ERR),
    ("st_predict_sum", C.c_int, [C.POINTER(ModelBundleC), C.c_uint64, _D] + _ERR),
    ("st_predict_overhead", C.c_int, [C.POINTER(ModelBundleC), C.c_uint64, C.c_int, _D] + _ERR),
    ("st_recommend", C.c_int,
     [C.POINTER(ModelBundleC), C.c_uint64, C.POINTER(C.c_int), _D, _D, _D, C.POINTER(C.c_int)] + _ERR),
    ("st_recommend_fp32", C.c_int, [C.POINTER(ModelBundleC), C.c_uint64, C.POINTER(C.c_int)] + _ERR),
    ("st_gomez_luna_optimum", C.c_int, [C.c_double, C.c_double, _D] + _ERR),
    ("st_train_test_split", C.c_int,
     [C.c_int, C.c_double, C.c_int, C.c_uint64, C.POINTER(C.c_int), C.POINTER(C.c_int)] + _ERR),
    ("st_fit_least_squares", C.c_int, [_D, _D, C.c_int, C.c_int, _D] + _ERR),
    ("st_metrics", C.c_int, [_D, _D, C.c_int, _D] + _ERR),
    ("st_fit_model", C.c_int,
     [C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int), _D, C.c_int, C.c_double, C.c_int,
      C.c_uint64, _D, _D, C.POINTER(C.c_int)] + _ERR),
    ("st_load_stage_timings", C.c_int,
     [C.c_char_p, C.POINTER(StageTimingsC), C.c_int, C.POINTER(C.c_int)] + _ERR),
    ("st_load_streamed_runs", C.c_int,
     [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int), _D, C.c_int, C.POINTER(C.c_int)] + _ERR),
    ("st_derive_overhead_rows", C.c_int,
     [C.c_char_p, C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int), _D, C.c_int,
      C.POINTER(C.c_int)] + _ERR),
    ("st_fit_bundle", C.c_int,
     [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(ModelBundleC), _D] + _ERR),
    ("st_fit_bundle_anchored", C.c_int,
     [C.c_char_p, C.c_char_p, C.c_uint64, C.c_uint64, C.POINTER(ModelBundleC), _D] + _ERR),
    ("st_simulate", C.c_int,
     [_D, C.c_int, C.c_double, C.c_int, _D, _D, C.c_int, C.POINTER(C.c_int)] + _ERR),
    ("st_verify_lower_bound", C.c_int,
     [_D, C.c_int, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)] + _ERR),
    ("st_bundle_to_json", C.c_int,
     [C.POINTER(ModelBundleC), C.c_char_p, C.c_int, C.POINTER(C.c_int)] + _ERR),
    ("st_bundle_from_json", C.c_int, [C.c_char_p, C.POINTER(ModelBundleC)] + _ERR),
    ("st_report_table", C.c_int,
     [C.POINTER(ModelBundleC), C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
      _D, C.c_int, C.POINTER(C.c_int)] + _ERR),
    ("st_dump_reference", C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)] + _ERR),
]

_lib = None


def load():
    """The native library; raises ImportError when it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (no CPU fallback exists)")
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in PM_SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
