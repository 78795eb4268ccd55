"""ctypes declarations of include/knnj_c.h (the drop-in C ABI).

Loads the in-tree ``libknnj_b200.so``. There is deliberately no CPU fallback:
if the CUDA library is missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libknnj_b200.so")

# knnj_status -> reference exception names (proj/include/knnjoin/errors.hpp)
STATUS_NAMES = {
    1: "UsageError", 2: "IngestError", 3: "IndexingError", 4: "DegenerateProfileError",
    5: "TargetUnreachableError", 6: "BatchOverflowError", 7: "SampleTooSmallError",
    8: "OracleCapError", 9: "CudaError",
}


class KnnjError(RuntimeError):
    """Raised for a non-zero knnj status; ``kind`` names the reference exception type."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.kind = STATUS_NAMES.get(code, "Error")
        super().__init__(f"{self.kind}: {message}")


class GridInfo(C.Structure):
    _fields_ = [("m", C.c_uint32), ("eps", C.c_double), ("n_cells", C.c_uint64),
                ("mins", C.c_double * 64), ("maxs", C.c_double * 64),
                ("cells_per_dim", C.c_uint64 * 64)]


class SplitInfo(C.Structure):
    _fields_ = [("n_min", C.c_double), ("n_thresh", C.c_double), ("q_gpu", C.c_uint64),
                ("q_cpu", C.c_uint64), ("demoted", C.c_uint64)]


class JoinStats(C.Structure):
    _fields_ = [("candidates_examined", C.c_uint64), ("solved", C.c_uint64),
                ("failed", C.c_uint64), ("kernel_ms", C.c_double)]


class Config(C.Structure):
    _fields_ = [("k", C.c_uint32), ("m", C.c_uint32), ("beta", C.c_double),
                ("gamma", C.c_double), ("rho", C.c_double), ("mode", C.c_uint32),
                ("n_bins", C.c_uint32), ("hist_query_fraction", C.c_double),
                ("eps_mean_pair_cap", C.c_uint64), ("seed", C.c_uint64),
                ("query_subset", C.POINTER(C.c_uint32)), ("n_query_subset", C.c_uint64)]


RUN_INFO_FIELDS = [
    ("n_queries", C.c_uint64), ("k_effective", C.c_uint32), ("m_used", C.c_uint32),
    ("k_clamped", C.c_uint32), ("eps_fallback", C.c_uint32),
    ("eps_mean", C.c_double), ("bin_width", C.c_double), ("eps_default", C.c_double),
    ("eps_beta", C.c_double), ("eps_final", C.c_double), ("eps_used", C.c_double),
    ("hist_query_count", C.c_uint64), ("hist_bin", C.c_uint64),
    ("n_min", C.c_double), ("n_thresh", C.c_double),
    ("q_gpu", C.c_uint64), ("q_cpu", C.c_uint64), ("demoted", C.c_uint64),
    ("failed_count", C.c_uint64), ("candidates_examined", C.c_uint64),
    ("fallback_queries", C.c_uint64), ("fallback_passes", C.c_uint64),
    ("slow_path_queries", C.c_uint64), ("grid_cells", C.c_uint64),
    ("kernel_launches", C.c_uint64), ("join_tensor_cores", C.c_uint32),
    ("hist_tensor_cores", C.c_uint32), ("hist_bins_counted", C.c_uint32),
    ("n_owned", C.c_uint64), ("join_candidate_pairs", C.c_uint64),
    ("join_screened_pairs", C.c_uint64),
] + [(f, C.c_double) for f in (
    "ms_upload", "ms_reorder", "ms_eps_mean", "ms_histogram", "ms_grid", "ms_split", "ms_join",
    "ms_fallback", "ms_download", "ms_total", "ms_join_kernel", "ms_hist_kernel",
    "ms_join_build")] + [
    ("kth_bound2", C.c_double), ("bound_retried", C.c_uint64),
    ("perm", C.c_uint32 * 1024)]


class RunInfo(C.Structure):
    _fields_ = RUN_INFO_FIELDS


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_vp = C.c_void_p

# (name, restype, argtypes) — every symbol declared in include/knnj_c.h
SIGNATURES = [
    ("knnj_abi_version", C.c_int, []),
    ("knnj_create", C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    ("knnj_destroy", None, [_vp]),
    ("knnj_last_error", C.c_char_p, [_vp]),
    ("knnj_stream", C.c_void_p, [_vp]),
    ("knnj_fp32_peak", C.c_int, [_vp, C.POINTER(C.c_double)]),
    ("knnj_set_option", C.c_int, [_vp, C.c_char_p, C.c_int64]),
    ("knnj_alloc_pinned", C.c_void_p, [C.c_size_t]),
    ("knnj_free_pinned", None, [C.c_void_p]),
    ("knnj_set_points", C.c_int, [_vp, _vp, C.c_uint64, C.c_uint32]),
    ("knnj_reorder_by_variance", C.c_int, [_vp, C.c_uint32, _u32p, _dp]),
    ("knnj_get_points", C.c_int, [_vp, _dp]),
    ("knnj_pair_sq", C.c_int, [_vp, _u64p, C.c_uint64, C.c_double, _dp]),
    ("knnj_eps_mean", C.c_int, [_vp, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]),
    ("knnj_histogram", C.c_int, [_vp, C.c_double, C.c_uint32, C.c_double, C.c_uint64, _u64p,
                                 C.POINTER(C.c_uint64)]),
    ("knnj_histogram_queries", C.c_int, [_vp, _u64p, C.c_uint64, C.c_double, C.c_uint32,
                                         _u64p]),
    ("knnj_grid_build", C.c_int, [_vp, C.c_uint32, C.c_double, C.POINTER(GridInfo)]),
    ("knnj_grid_export", C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    ("knnj_range_count", C.c_int, [_vp, _u32p, C.c_uint64, _u64p, _u64p]),
    ("knnj_split", C.c_int, [_vp, _u32p, C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                             C.c_double, _u8p, _u64p, C.POINTER(SplitInfo)]),
    ("knnj_dense_join", C.c_int, [_vp, _u32p, C.c_uint64, C.c_uint32, _u32p, _dp, _u8p,
                                  C.POINTER(JoinStats)]),
    ("knnj_exact_knn", C.c_int, [_vp, _u32p, C.c_uint64, C.c_uint32, _u32p, _dp]),
    ("knnj_run", C.c_int, [_vp, C.POINTER(Config), _vp, _vp, _vp, _vp, C.POINTER(RunInfo)]),
]

# int (*knnj_allreduce_fn)(uint64_t* data, uint64_t count, void* user)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_uint64), C.c_uint64, C.c_void_p)
SIGNATURES.append(
    ("knnj_shard_range", C.c_int, [_dp, C.c_uint64, C.c_uint32, C.c_uint32,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]))
SIGNATURES.append(
    ("knnj_run_shard", C.c_int, [_vp, C.POINTER(Config), C.c_uint32, C.c_uint32, ALLREDUCE_FN,
                                 _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(RunInfo)]))

class SearchRow(C.Structure):
    """knnj_search_row (include/knnj_c.h): one parameter-search candidate."""
    _fields_ = [("beta", C.c_double), ("gamma", C.c_double), ("wall_seconds", C.c_double),
                ("status", C.c_int32), ("error", C.c_char * 256)]


SIGNATURES.append(
    ("knnj_parameter_search", C.c_int, [_vp, C.POINTER(Config), C.c_double, _dp, _dp, C.c_uint64,
                                        C.POINTER(SearchRow), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]))

SIGNATURES += [
    ("knnj_io_last_error", C.c_char_p, []),
    ("knnj_tsv_format", C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_uint32, _vp, C.c_uint64,
                                  C.POINTER(C.c_uint64), C.c_uint32]),
    ("knnj_tsv_write", C.c_int, [C.c_char_p, _vp, _vp, _vp, C.c_uint64, C.c_uint32, C.c_uint32,
                                 C.POINTER(C.c_uint64)]),
    ("knnj_binary_header", C.c_int, [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("knnj_binary_read", C.c_int, [C.c_char_p, _vp, C.c_uint64]),
    ("knnj_text_parse", C.c_int, [C.c_char_p, C.c_char, C.c_uint32, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("knnj_text_copy", C.c_int, [_vp, _vp, C.c_uint64]),
    ("knnj_text_free", None, [_vp]),
    # test hooks
    ("knnj_histogram_queries_capped", C.c_int, [_vp, _u64p, C.c_uint64, C.c_double, C.c_uint32,
                                                C.c_uint32, _u64p]),
    ("knnj_debug_tc_tile", C.c_int, [_vp, C.c_uint32, C.c_uint32, _vp, _vp, _vp,
                                     C.POINTER(C.c_double), C.POINTER(C.c_double), _vp, _vp]),
]

_LIB = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load libknnj_b200.so (fails loudly: there is no non-CUDA implementation)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or os.environ.get("KNNJ_LIB_PATH") or LIB_PATH  # env: dev A/B of library builds
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " or `make -C paper_1810_04758_b200`")
    lib = C.CDLL(p)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib
