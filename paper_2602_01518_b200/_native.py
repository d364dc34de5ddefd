"""ctypes binding of libqrita_b200.so (the C ABI declared in include/qrita_b200.h).

The shared library is built in-tree by `paper_2602_01518_b200._build.build()` (called from
`__graft_entry__.build()`).  There is no fallback: if the library is missing or CUDA is absent the
first call raises, loudly.
"""
from __future__ import annotations

import ctypes
import os

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.environ.get("QRITA_LIB") or os.path.join(LIB_DIR, "libqrita_b200.so")  # QRITA_LIB: A/B builds

# include/qrita_b200.h enums
DTYPE_F32 = 0
DTYPE_BF16 = 1
SEARCH_BINARY = 1 << 0
NO_SIGMA = 1 << 1
FORCE_FALLBACK = 1 << 2
NO_DUP = 1 << 3
INPLACE = 1 << 4
DEBUG_TIMING = 1 << 6
STAGED = 1 << 7
TP_NO_TOPP_ROWS = 1 << 8

OK = 0
EINVAL_ARG = 1
EINVAL_K = 2
EINVAL_P = 3
ENONFINITE = 4
EWORKSPACE = 5
ECUDA = 6
ENCCL = 7

EXPORTED_SYMBOLS = (
    "qrita_workspace_bytes", "qrita_workspace_init", "qrita_topk_topp", "qrita_topk_topp_ex", "qrita_topk_topp_idx",
    "qrita_get_status", "qrita_get_timing", "qrita_host_scratch_bytes", "qrita_topk_topp_host",
    "qrita_get_status_host", "qrita_strerror", "qrita_version",
    "qrita_tp_workspace_bytes", "qrita_topk_topp_tp_comm", "qrita_topk_topp_tp", "qrita_nccl_unique_id",
    "qrita_nccl_comm_init", "qrita_nccl_comm_destroy", "qrita_copy_sync", "qrita_sigma_table",
    "qrita_row_stats", "qrita_host_download_bytes", "qrita_lmhead_logits", "qrita_lmhead_workspace_bytes", "qrita_lmhead_topk_topp",
)


class RowMetricsC(ctypes.Structure):
    """qrita_row_metrics (include/qrita_b200.h)."""

    _fields_ = [
        ("trunc_hit", ctypes.c_int32),
        ("outlier_count", ctypes.c_int32),
        ("outlier_prob_sum", ctypes.c_double),
        ("k_search_iters", ctypes.c_int32),
        ("p_search_iters", ctypes.c_int32),
        ("fallback_used", ctypes.c_int32),
        ("kept_count", ctypes.c_int32),
        ("full_row_path", ctypes.c_int32),
        ("row_passes", ctypes.c_int32),
    ]


METRICS_BYTES = ctypes.sizeof(RowMetricsC)  # 40

_lib = None


class NativeLibraryError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    """Load libqrita_b200.so and declare the prototypes.  Raises NativeLibraryError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    lib.qrita_workspace_bytes.argtypes = [i32, i32, i32, i32]
    lib.qrita_workspace_bytes.restype = sz
    lib.qrita_workspace_init.argtypes = [vp, sz, vp]
    lib.qrita_workspace_init.restype = i32
    lib.qrita_topk_topp.argtypes = [vp, i64, i32, i32, i32, vp, vp, vp, i64, vp, vp, vp, sz, i32, i32, vp]
    lib.qrita_topk_topp.restype = i32
    lib.qrita_topk_topp_ex.argtypes = [vp, i64, i32, i32, i32, vp, vp, vp, i64, vp, vp, vp, sz, i32, i32,
                                       vp, vp, vp]
    lib.qrita_topk_topp_ex.restype = i32
    lib.qrita_topk_topp_idx.argtypes = [vp, i64, i32, i32, i32, vp, vp, vp, i64, vp, i64, vp, vp, vp, sz, i32, i32,
                                        vp]
    lib.qrita_topk_topp_idx.restype = i32
    lib.qrita_get_status.argtypes = [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), vp]
    lib.qrita_get_status.restype = i32
    lib.qrita_get_timing.argtypes = [vp, i32, vp, vp]
    lib.qrita_get_timing.restype = i32
    lib.qrita_host_scratch_bytes.argtypes = [i32, i32, i32, i32]
    lib.qrita_host_scratch_bytes.restype = sz
    lib.qrita_topk_topp_host.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, sz, i32, i32, i32, vp]
    lib.qrita_topk_topp_host.restype = i32
    lib.qrita_get_status_host.argtypes = [vp, i32, i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), vp]
    lib.qrita_get_status_host.restype = i32
    lib.qrita_tp_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.qrita_tp_workspace_bytes.restype = sz
    tp_args = [vp, i64, i32, i32, i32, i32, i64, vp, vp, i32, vp, i64, vp, vp, sz, i32, i32, i32, vp, vp]
    lib.qrita_topk_topp_tp_comm.argtypes = tp_args
    lib.qrita_topk_topp_tp_comm.restype = i32
    lib.qrita_topk_topp_tp.argtypes = tp_args
    lib.qrita_topk_topp_tp.restype = i32
    lib.qrita_nccl_unique_id.argtypes = [vp]
    lib.qrita_nccl_unique_id.restype = i32
    lib.qrita_nccl_comm_init.argtypes = [ctypes.POINTER(vp), i32, ctypes.c_char_p, i32]
    lib.qrita_nccl_comm_init.restype = i32
    lib.qrita_nccl_comm_destroy.argtypes = [vp]
    lib.qrita_nccl_comm_destroy.restype = i32
    lib.qrita_copy_sync.argtypes = [vp, vp, sz, vp]
    lib.qrita_copy_sync.restype = i32
    lib.qrita_sigma_table.argtypes = [i32, vp, i32]
    lib.qrita_sigma_table.restype = i32
    lib.qrita_row_stats.argtypes = [vp, i64, i32, i32, i32, i32, vp, vp]
    lib.qrita_row_stats.restype = i32
    lib.qrita_host_download_bytes.argtypes = [i32, i32, i32, vp, vp, vp]
    lib.qrita_host_download_bytes.restype = i64
    lib.qrita_lmhead_logits.argtypes = [vp, i64, vp, i64, i32, i32, i32, vp, i64, vp]
    lib.qrita_lmhead_logits.restype = i32
    lib.qrita_lmhead_workspace_bytes.argtypes = [i32, i32]
    lib.qrita_lmhead_workspace_bytes.restype = sz
    lib.qrita_lmhead_topk_topp.argtypes = [vp, i64, vp, i64, i32, i32, i32, vp, vp, vp, i64, vp, i64, vp, vp, vp,
                                           sz, i32, vp]
    lib.qrita_lmhead_topk_topp.restype = i32
    lib.qrita_strerror.argtypes = [i32]
    lib.qrita_strerror.restype = ctypes.c_char_p
    lib.qrita_version.argtypes = []
    lib.qrita_version.restype = i32
    _lib = lib
    return lib


def strerror(code: int) -> str:
    return load().qrita_strerror(int(code)).decode()
