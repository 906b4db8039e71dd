"""ctypes binding of libettg.so (include/ettg.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2103_15217_b200/csrc``).  There is no fallback: if the
library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libettg.so")

(ETTG_OK, ETTG_EINVAL, ETTG_ERANGE, ETTG_ECUDA, ETTG_ENOMEM, ETTG_EINTERNAL, ETTG_EPARSE,
 ETTG_ENCCL) = range(8)
ENGINE_INLABEL = 1
ENGINE_RMQ = 2
ENGINE_NAIVE = 4
LAYOUT_WIDE = 0x100    # build flags (OR into engines); default: chosen per tree
LAYOUT_NARROW = 0x200
LAYOUT_COMPACT = 0x400
LAYOUT_SPLIT = 0x800
LAYOUT_SPLIT_OWN = 0x1000
LAYOUT_SPLIT6 = 0x2000
LAYOUT_WIDE9 = 0x4000
REDUCE_MIN, REDUCE_MAX, REDUCE_SUM = range(3)  # ettg_segmented_reduce ops

_lock = threading.Lock()
_lib = None

i64 = C.c_int64
u64 = C.c_uint64
p = C.c_void_p
i64p = C.POINTER(C.c_int64)


class ParseStatsC(C.Structure):
    _fields_ = [("self_loops_removed", C.c_int64), ("duplicates_removed", C.c_int64)]


class PhaseTimes(C.Structure):
    _fields_ = [("spanning_ms", C.c_double), ("euler_ms", C.c_double),
                ("lowhigh_ms", C.c_double), ("total_ms", C.c_double),
                ("marking_ms", C.c_double)]


BRIDGES_TV, BRIDGES_CK, BRIDGES_HYBRID = 0, 1, 2


_SIGS = {
    "ettg_last_error": ([], C.c_char_p),
    "ettg_gen_last_error": ([], C.c_char_p),
    "ettg_version": ([], C.c_int),
    "ettg_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "ettg_lca_build": ([p, i64, i64, C.c_int, C.c_uint, C.POINTER(p)], C.c_int),
    "ettg_lca_build_dev": ([p, i64, i64, C.c_int, C.c_uint, p, C.POINTER(p)], C.c_int),
    "ettg_lca_free": ([p], None),
    "ettg_lca_size": ([p, i64p], C.c_int),
    "ettg_lca_layout": ([p, C.POINTER(C.c_int), i64p], C.c_int),
    "ettg_lca_build_ms": ([p, C.POINTER(C.c_double)], C.c_int),
    "ettg_lca_query": ([p, p, i64, i64, p], C.c_int),
    "ettg_lca_query_engine": ([p, C.c_uint, p, i64, i64, p], C.c_int),
    "ettg_lca_query_dev": ([p, C.c_uint, p, i64, p, p], C.c_int),
    "ettg_lca_query_dev_error": ([p, p, C.POINTER(C.c_int)], C.c_int),
    "ettg_lca_stats": ([p, p, p, p, p], C.c_int),
    "ettg_ancestor_levels": ([p, i64, i64, C.c_int, p], C.c_int),
    "ettg_lca_inlabel_index": ([p, p, p, p, p, p], C.c_int),
    "ettg_lca_index_bytes": ([p, i64p], C.c_int),
    "ettg_lca_index_export_dev": ([p, p, p], C.c_int),
    "ettg_lca_index_attach_dev": ([p, i64, C.c_int, p, C.POINTER(p)], C.c_int),
    "ettg_bridges": ([p, i64, i64, C.c_int, p, C.POINTER(PhaseTimes)], C.c_int),
    "ettg_bridges_dev": ([p, i64, i64, C.c_int, p, p, C.POINTER(PhaseTimes)], C.c_int),
    "ettg_set_l2_fetch_granularity": ([C.c_int, C.c_int], C.c_int),
    "ettg_get_l2_fetch_granularity": ([C.c_int, C.POINTER(C.c_int)], C.c_int),
    "ettg_bridges_engine": ([p, i64, i64, C.c_int, C.c_int, p, C.POINTER(PhaseTimes)], C.c_int),
    "ettg_bridges_dev_engine": ([p, i64, i64, C.c_int, C.c_int, p, p, C.POINTER(PhaseTimes)],
                                C.c_int),
    "ettg_build_adjacency": ([p, i64, i64, C.c_int, p, p, p], C.c_int),
    "ettg_largest_component": ([p, i64, i64, C.c_int, p, i64p, i64p, p], C.c_int),
    "ettg_bfs_tree": ([p, i64, i64, i64, C.c_int, p, p, p, p], C.c_int),
    "ettg_lca_device": ([p, C.POINTER(C.c_int)], C.c_int),
    "ettg_shard_range": ([i64, C.c_int, C.c_int, i64p, i64p], C.c_int),
    "ettg_nccl_unique_id": ([p], C.c_int),
    "ettg_lca_replicate": ([p, C.c_int, p, p], C.c_int),
    "ettg_lca_replicate_rank": ([C.POINTER(p), C.c_int, p, C.c_int, C.c_int, C.c_int], C.c_int),
    "ettg_lca_query_multi": ([p, C.c_int, C.c_uint, p, i64, i64, p], C.c_int),
    "ettg_bfs_tree_csr": ([p, p, p, i64, i64, i64, C.c_int, p, p, p, p], C.c_int),
    "ettg_bridges_on_tree": ([p, i64, i64, C.c_int, p, p, C.POINTER(PhaseTimes)], C.c_int),
    "ettg_bridges_dev_on_tree": ([p, i64, i64, C.c_int, p, p, p, C.POINTER(PhaseTimes)],
                                 C.c_int),
    "ettg_bridges_low_high": ([p, i64, i64, C.c_int, p, p, p, p, p], C.c_int),
    "ettg_bridges_csr": ([p, p, p, i64, i64, C.c_int, C.c_int, p, p, C.POINTER(PhaseTimes)],
                         C.c_int),
    "ettg_list_rank_dev": ([p, i64, i64, p, C.c_int, p], C.c_int),
    "ettg_exclusive_scan_dev": ([p, i64, p, C.c_int, p], C.c_int),
    "ettg_sort_pairs_dev": ([p, p, i64, p, p, C.c_int, p], C.c_int),
    "ettg_exclusive_scan_i64_dev": ([p, i64, p, C.c_int, p], C.c_int),
    "ettg_list_scan": ([p, p, i64, i64, C.c_int, p], C.c_int),
    "ettg_segmented_reduce": ([p, i64, p, i64, C.c_int, i64, C.c_int, p], C.c_int),
    "ettg_segmented_reduce_dev": ([p, i64, p, i64, C.c_int, i64, p, C.c_int, p], C.c_int),
    "ettg_range_index_build": ([p, i64, C.c_int, C.POINTER(p)], C.c_int),
    "ettg_range_index_build_dev": ([p, i64, C.c_int, p, C.POINTER(p)], C.c_int),
    "ettg_range_index_size": ([p], i64),
    "ettg_range_index_query": ([p, p, i64, p, p], C.c_int),
    "ettg_range_index_query_dev": ([p, p, i64, p, p, p], C.c_int),
    "ettg_range_index_free": ([p], None),
    "ettg_gen_grasp_tree": ([i64, u64, u64, p], C.c_int),
    "ettg_gen_barabasi_tree": ([i64, u64, p], C.c_int),
    "ettg_gen_permute_labels": ([i64, p, i64, u64, p, i64p], C.c_int),
    "ettg_gen_sample_queries": ([i64, i64, u64, p], C.c_int),
    "ettg_gen_random_connected_graph": ([i64, i64, u64, p], C.c_int),
    "ettg_gen_queries_dev": ([i64, i64, u64, i64, p, C.POINTER(C.c_int), C.c_int, p], C.c_int),
    "ettg_gen_grasp_tree_dev": ([i64, u64, u64, p, C.POINTER(C.c_int), C.c_int, p], C.c_int),
    "ettg_gen_permute_labels_dev": ([p, i64, i64, u64, p, i64p, C.POINTER(C.c_int), C.c_int, p],
                                    C.c_int),
    "ettg_gen_planted_bridge_graph": ([i64, i64, i64, u64, p, p], C.c_int),
    "ettg_road_like_edge_count": ([i64, i64, i64, i64, i64], i64),
    "ettg_parse_edge_list": ([C.c_char_p, i64, C.c_int, p, i64, i64p, i64p,
                              C.POINTER(ParseStatsC)], C.c_int),
    "ettg_parse_dimacs_gr": ([C.c_char_p, i64, C.c_int, p, i64, i64p, i64p,
                              C.POINTER(ParseStatsC)], C.c_int),
    "ettg_write_edge_list": ([p, i64, p, i64, i64p], C.c_int),
    "ettg_gen_road_like_graph": ([i64, i64, i64, i64, i64, u64, p, p], C.c_int),
}


def lib():
    """Load libettg.so once; raise if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            # libettg.so binds NCCL at first use to whatever libnccl.so.2 the
            # process holds; load torch's (when installed) before anything can
            # pull in the system copy, which torch's own import would reject.
            try:
                import torch  # noqa: F401
            except ImportError:
                pass
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libettg.so not found at {LIB_PATH}; build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                if not hasattr(L, name):
                    continue  # reported by tests/test_abi.py
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
        return _lib


class EttgError(RuntimeError):
    code = ETTG_EINTERNAL


class InvalidArgument(EttgError, ValueError):
    """std::invalid_argument in the reference."""
    code = ETTG_EINVAL


class OutOfRange(EttgError, IndexError):
    """std::out_of_range in the reference."""
    code = ETTG_ERANGE


class CudaError(EttgError):
    code = ETTG_ECUDA


class ParseError(EttgError):
    """std::runtime_error thrown by the reference's text parsers."""
    code = ETTG_EPARSE


class NcclError(EttgError):
    """ETTG_ENCCL: replicating an index across GPUs failed in NCCL."""
    code = ETTG_ENCCL


_EXC = {ETTG_EINVAL: InvalidArgument, ETTG_ERANGE: OutOfRange, ETTG_ECUDA: CudaError,
        ETTG_EPARSE: ParseError, ETTG_ENCCL: NcclError}


def check(rc: int, gen: bool = False) -> None:
    if rc == ETTG_OK:
        return
    L = lib()
    msg = (L.ettg_gen_last_error() if gen else L.ettg_last_error()) or b""
    raise _EXC.get(rc, EttgError)(msg.decode(errors="replace") + f" (code {rc})")


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
