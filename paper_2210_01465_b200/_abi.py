"""ctypes binding of the C-ABI in include/tk_landscape.h (libtk_landscape.so).

This is the stub a Python maintainer of the reference would add.
Loading fails loudly when the CUDA library is missing -- there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtk_landscape.so")

TK_OK, TK_EINVAL, TK_ELIMIT, TK_ENOFEAS, TK_ENOCONV, TK_EDEGEN = 0, 1, 2, 3, 4, 5
TK_ENOMEM, TK_ECUDA, TK_ENCCL, TK_ESTATE = 6, 7, 8, 9
TK_HAMMING, TK_ADJACENT = 0, 1
TK_MEM_HOST, TK_MEM_DEVICE = 0, 1
TK_GEN_IID, TK_GEN_HEAVY = 0, 1
TK_MAX_CP = 101

# every symbol include/tk_landscape.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "tk_abi_version", "tk_last_error", "tk_status_name", "tk_device_count",
    "tk_land_create", "tk_land_destroy", "tk_land_reshape", "tk_land_info", "tk_land_stream",
    "tk_land_kernel_info",
    "tk_land_load_dense", "tk_land_load_sparse", "tk_land_load_configs",
    "tk_land_generate", "tk_land_copy_fitness", "tk_land_lookup", "tk_optimum",
    "tk_ffg_build", "tk_ffg_copy_out", "tk_census", "tk_pagerank",
    "tk_pagerank_copy_out", "tk_centrality", "tk_report_copy_out", "tk_analyze",
    "tk_pagerank_csr", "tk_proportion_of_centrality", "tk_descents", "tk_batch_analyze",
    "tk_land_set_shard", "tk_land_replica_ptrs", "tk_land_set_peer_ptrs", "tk_land_ipc_handles",
    "tk_land_open_peers", "tk_shard_optimum", "tk_shard_pagerank_init", "tk_shard_pagerank_step",
    "tk_shard_pagerank_init_dev", "tk_shard_pagerank_step_dev", "tk_shard_pagerank_rewind",
    "tk_shard_centrality", "tk_shard_pagerank_copy_out",
]


class ReportSummary(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_uint64), ("n_edges", C.c_uint64), ("n_minima", C.c_uint64),
        ("f_opt", C.c_double), ("opt_rank", C.c_uint64), ("iterations", C.c_int64),
        ("residual", C.c_double), ("pagerank_sum", C.c_double), ("n_cp", C.c_int32),
        ("c_p", C.c_double * TK_MAX_CP),
        ("ms_load", C.c_float), ("ms_ffg", C.c_float), ("ms_pagerank", C.c_float),
        ("ms_centrality", C.c_float),
    ]


class BatchItem(C.Structure):
    """tk_batch_item (include/tk_landscape.h)."""
    _fields_ = [
        ("dims", C.c_uint32), ("radix", C.c_uint32 * 32),
        ("fitness", C.c_void_p), ("ok", C.c_void_p),
        ("minima_ranks", C.c_void_p), ("minima_fitness", C.c_void_p),
        ("minima_fraction", C.c_void_p), ("minima_pagerank", C.c_void_p),
        ("minima_capacity", C.c_uint64), ("summary", ReportSummary), ("status", C.c_int32),
    ]


_lib = None


def load(path: str = LIB_PATH):
    """Load libtk_landscape.so (building it first only if the toolchain is here).
    TK_LIB=<path> selects a build variant (paper_2210_01465_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("TK_LIB", path)
    if not os.path.exists(path):
        from . import build as _b
        _b.build()
    L = C.CDLL(path)
    P, I, U64, U32, D = C.c_void_p, C.c_int, C.c_uint64, C.c_uint32, C.c_double
    PU64, PI64, PD = C.POINTER(C.c_uint64), C.POINTER(C.c_int64), C.POINTER(C.c_double)
    sig = {
        "tk_abi_version": (I, []),
        "tk_last_error": (C.c_char_p, []),
        "tk_status_name": (C.c_char_p, [I]),
        "tk_device_count": (I, [C.POINTER(I)]),
        "tk_land_create": (I, [I, U32, P, C.POINTER(P)]),
        "tk_land_destroy": (I, [P]),
        "tk_land_reshape": (I, [P, U32, P]),
        "tk_land_info": (I, [P, PU64, C.POINTER(I)]),
        "tk_land_stream": (P, [P]),
        "tk_land_kernel_info": (I, [P, C.POINTER(I), C.POINTER(I), C.POINTER(I),
                                    C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "tk_land_load_dense": (I, [P, P, P, I]),
        "tk_land_load_sparse": (I, [P, P, P, U64, I]),
        "tk_land_load_configs": (I, [P, P, P, U64, I]),
        "tk_land_generate": (I, [P, I, D, U64]),
        "tk_land_copy_fitness": (I, [P, P, P]),
        "tk_land_lookup": (I, [P, P, U64, P, P]),
        "tk_optimum": (I, [P, PD, PU64]),
        "tk_ffg_build": (I, [P, I, U64, I, PU64, PU64]),
        "tk_ffg_copy_out": (I, [P, P, P, P, P]),
        "tk_census": (I, [P, PU64, PU64, PU64, P]),
        "tk_descents": (I, [P, C.c_uint64, C.c_uint64, I, P, PU64, PU64]),
        "tk_batch_analyze": (I, [I, P, C.c_uint32, I, D, D, C.c_int64, I, I]),
        "tk_pagerank": (I, [P, D, D, C.c_int64, PI64, PD, PD]),
        "tk_pagerank_copy_out": (I, [P, P]),
        "tk_centrality": (I, [P, D, P, I, P]),
        "tk_report_copy_out": (I, [P, D, P, P, P, P]),
        "tk_analyze": (I, [P, I, D, D, C.c_int64, U64, I, I, C.POINTER(ReportSummary)]),
        "tk_pagerank_csr": (I, [I, U64, P, P, D, D, C.c_int64, P, PI64, PD]),
        "tk_proportion_of_centrality": (I, [I, U64, P, P, D, D, PD]),
        "tk_land_set_shard": (I, [P, I, I, PU64, PU64]),
        "tk_land_replica_ptrs": (I, [P, C.POINTER(P), C.POINTER(P)]),
        "tk_land_set_peer_ptrs": (I, [P, P, P]),
        "tk_land_ipc_handles": (I, [P, P]),
        "tk_land_open_peers": (I, [P, P]),
        "tk_shard_optimum": (I, [P, PD, PU64, C.POINTER(I)]),
        "tk_shard_pagerank_init": (I, [P, D, PD]),
        "tk_shard_pagerank_step": (I, [P, D, D, PD, PD, PD]),
        "tk_shard_pagerank_init_dev": (I, [P, D, P]),
        "tk_shard_pagerank_step_dev": (I, [P, P, D, P]),
        "tk_shard_pagerank_rewind": (I, [P]),
        "tk_shard_centrality": (I, [P, D, P, I, P, PD]),
        "tk_shard_pagerank_copy_out": (I, [P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def last_error() -> str:
    return load().tk_last_error().decode(errors="replace")
