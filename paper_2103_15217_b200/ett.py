"""Host-side mirror of the reference's ``ett`` namespace for the hot path.

Same names, argument meaning and error behaviour as
/root/reference/proj/core/include/ett/{graph,lca,bridges,primitives,generators}.hpp,
backed by the sm_100a kernels in ``libettg.so`` through the C-ABI
(include/ettg.h).  Arrays are numpy int64 (the reference's i64); device
variants take torch CUDA tensors.

Exceptions: ``InvalidArgument`` (a ``ValueError``) where the reference
throws ``std::invalid_argument``; ``OutOfRange`` (an ``IndexError``) for
``std::out_of_range``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (ENGINE_INLABEL, ENGINE_NAIVE, ENGINE_RMQ, LAYOUT_COMPACT, LAYOUT_NARROW, LAYOUT_SPLIT,
                   LAYOUT_SPLIT_OWN, LAYOUT_SPLIT6, LAYOUT_WIDE9,
                   LAYOUT_WIDE,
                   InvalidArgument, OutOfRange, ParseError, check, lib, ptr)

K_NONE = -1
K_GRASP_INFINITY = (1 << 64) - 1


# --------------------------------------------------------------- data model
@dataclass
class RootedTree:
    """core/include/ett/graph.hpp:66-70 -- parent[root] == kNone (-1)."""
    n: int
    root: int
    parent: np.ndarray  # int64[n]

    def __post_init__(self):
        self.parent = np.ascontiguousarray(self.parent, dtype=np.int64)


@dataclass
class EdgeList:
    """core/include/ett/graph.hpp:18-23 -- undirected simple graph."""
    n: int
    edges: np.ndarray  # int64[m, 2]

    def __post_init__(self):
        self.edges = np.ascontiguousarray(np.asarray(self.edges, dtype=np.int64).reshape(-1, 2))

    def m(self) -> int:
        return int(self.edges.shape[0])


@dataclass
class NodeStats:
    """core/include/ett/euler.hpp:45-53 (preorder is 1-based)."""
    preorder: np.ndarray
    size: np.ndarray
    level: np.ndarray
    parent: np.ndarray


@dataclass
class BridgeMask:
    """core/include/ett/bridges.hpp:20-24."""
    is_bridge: np.ndarray  # uint8[m]
    phases: dict = field(default_factory=dict)

    def count(self) -> int:
        return int(self.is_bridge.sum())


# -------------------------------------------------------------- LCA indices
class _LcaHandle:
    """Owns an ``ettg_lca*``; device memory lives on ``device``."""

    def __init__(self, handle: int, n: int, device: int, engines: int):
        self._h = C.c_void_p(handle)
        self.n = n
        self.device = device
        self.engines = engines

    def __del__(self):
        h = getattr(self, "_h", None)
        L = _lib._lib  # may already be torn down at interpreter exit
        if h is not None and h.value and L is not None:
            try:
                L.ettg_lca_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def build_ms(self) -> float:
        v = C.c_double()
        check(lib().ettg_lca_build_ms(self._h, C.byref(v)))
        return v.value

    def stats(self) -> NodeStats:
        n = self.n
        a = [np.empty(n, np.int64) for _ in range(4)]
        check(lib().ettg_lca_stats(self._h, *[ptr(x) for x in a]))
        return NodeStats(*a)

    def query(self, queries, batch_size: int, engine: int) -> np.ndarray:
        q = np.ascontiguousarray(np.asarray(queries, dtype=np.int64).reshape(-1, 2))
        out = np.empty(q.shape[0], np.int64)
        check(lib().ettg_lca_query_engine(self._h, engine, ptr(q), q.shape[0], int(batch_size),
                                          ptr(out)))
        return out

    def query_dev(self, d_pairs, d_answers, engine: int, stream: int | None = None) -> None:
        """Device-resident batch: uint32/int32 torch tensors (2q) -> (q).
        Out-of-range ids answer 0xFFFFFFFF; query_dev_error() reports them."""
        q = d_answers.numel()
        ok_types = {"torch.int32", "torch.uint32"}
        if str(d_pairs.dtype) not in ok_types or str(d_answers.dtype) not in ok_types:
            raise InvalidArgument("query_dev takes int32 / uint32 tensors")
        if d_pairs.numel() != 2 * q:
            raise InvalidArgument("query_dev: d_pairs must hold 2 * d_answers.numel() ids")
        if not (d_pairs.is_contiguous() and d_answers.is_contiguous()):
            raise InvalidArgument("query_dev: tensors must be contiguous")
        check(lib().ettg_lca_query_dev(self._h, engine, ptr(d_pairs), q, ptr(d_answers),
                                       stream))

    def query_dev_error(self, stream: int | None = None) -> bool:
        """True if a query_dev since the last call had an id outside [0, n) (clears)."""
        bad = C.c_int()
        check(lib().ettg_lca_query_dev_error(self._h, stream, C.byref(bad)))
        return bool(bad.value)

    def layout(self) -> tuple[str, int]:
        """(layout, number of inlabel paths) of the inlabel engine; the layout is
        "wide" | "narrow" | "compact" | "split" | "split_own" | "split6" | "wide9"
        (codes 0-6 of ettg_lca_layout and of the exported blob header)."""
        lay, labels = C.c_int(), C.c_int64()
        check(lib().ettg_lca_layout(self._h, C.byref(lay), C.byref(labels)))
        return ("wide", "narrow", "compact", "split", "split_own", "split6",
                "wide9")[lay.value], labels.value

    def index_bytes(self) -> int:
        v = C.c_int64()
        check(lib().ettg_lca_index_bytes(self._h, C.byref(v)))
        return v.value

    def export_index(self, d_dst, stream: int | None = None) -> None:
        check(lib().ettg_lca_index_export_dev(self._h, ptr(d_dst), stream))


class InlabelIndex(_LcaHandle):
    """core/include/ett/lca.hpp:13-24; fields are exported on first access."""

    _fields = None

    def _export(self):
        if self._fields is None:
            n = self.n
            inl = np.empty(n, np.int64)
            asc = np.empty(n, np.uint64)
            head = np.empty(n + 1, np.int64)
            lev = np.empty(n, np.int64)
            par = np.empty(n, np.int64)
            check(lib().ettg_lca_inlabel_index(self._h, ptr(inl), ptr(asc), ptr(head), ptr(lev),
                                               ptr(par)))
            self._fields = (inl, asc, head, lev, par)
        return self._fields

    inlabel = property(lambda s: s._export()[0])
    ascendant = property(lambda s: s._export()[1])
    head = property(lambda s: s._export()[2])
    level = property(lambda s: s._export()[3])
    parent = property(lambda s: s._export()[4])


class RmqLcaIndex(_LcaHandle):
    """core/include/ett/lca.hpp:39-44 (block-sparse table on the device)."""


class NaiveIndex(_LcaHandle):
    """core/include/ett/lca.hpp:29-35: parent + pointer-jumping levels."""


def _build(tree: RootedTree, engines: int, device: int):
    h = C.c_void_p()
    check(lib().ettg_lca_build(ptr(tree.parent), int(tree.n), int(tree.root), device, engines,
                               C.byref(h)))
    return h.value


def inlabel_build(tree: RootedTree, device: int = 0, engines: int = ENGINE_INLABEL) -> InlabelIndex:
    """inlabel_build (core/src/lca.cpp:20)."""
    if len(tree.parent) != tree.n:
        raise InvalidArgument("parent array size mismatch")
    return InlabelIndex(_build(tree, engines, device), tree.n, device, engines)


def inlabel_build_dev(d_parent, n: int, root: int, device: int = 0,
                     engines: int = ENGINE_INLABEL, stream: int | None = None) -> InlabelIndex:
    """Build from a device-resident int32/uint32 parent tensor (-1 = root)."""
    h = C.c_void_p()
    check(lib().ettg_lca_build_dev(ptr(d_parent), int(n), int(root), device, engines, stream,
                                   C.byref(h)))
    return InlabelIndex(h.value, n, device, engines)


def rmq_lca_build(tree: RootedTree, device: int = 0) -> RmqLcaIndex:
    """rmq_lca_build (core/src/lca.cpp:128)."""
    if len(tree.parent) != tree.n:
        raise InvalidArgument("parent array size mismatch")
    return RmqLcaIndex(_build(tree, ENGINE_RMQ, device), tree.n, device, ENGINE_RMQ)


def naive_build(tree: RootedTree, device: int = 0) -> NaiveIndex:
    """naive_build (core/src/lca.cpp:111-116): levels by pointer jumping."""
    if len(tree.parent) != tree.n:
        raise InvalidArgument("parent array size mismatch")
    return NaiveIndex(_build(tree, ENGINE_NAIVE, device), tree.n, device, ENGINE_NAIVE)


def ancestor_doubling_levels(tree: RootedTree, device: int = 0) -> np.ndarray:
    """ancestor_doubling_levels (core/src/primitives.cpp:208-241)."""
    if len(tree.parent) != tree.n:
        raise InvalidArgument("parent array size mismatch")
    out = np.empty(tree.n, np.int64)
    check(lib().ettg_ancestor_levels(ptr(tree.parent), int(tree.n), int(tree.root), device,
                                     ptr(out)))
    return out


def attach_index(d_src, n: int, device: int = 0, stream: int | None = None) -> InlabelIndex:
    """Query-only replica of a packed inlabel index (multi-GPU)."""
    h = C.c_void_p()
    check(lib().ettg_lca_index_attach_dev(ptr(d_src), int(n), device, stream, C.byref(h)))
    return InlabelIndex(h.value, n, device, ENGINE_INLABEL)


# ---------------------------------------------------------------- multi-GPU
def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of `total` units owned by `rank` (ettg_shard_range)."""
    lo, hi = C.c_int64(), C.c_int64()
    check(lib().ettg_shard_range(int(total), int(rank), int(world), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def replicate(index: InlabelIndex, devices) -> list[InlabelIndex]:
    """Query replicas of `index` on `devices` (one process, many GPUs): one
    grouped ncclBroadcast of the packed index (ettg_lca_replicate)."""
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    out = (C.c_void_p * len(devices))()
    check(lib().ettg_lca_replicate(index.handle, len(devices), devs, out))
    return [InlabelIndex(out[i], index.n, int(devices[i]), ENGINE_INLABEL)
            for i in range(len(devices))]


def nccl_unique_id() -> bytes:
    """An NCCL unique id (128 bytes) to share with the other ranks."""
    buf = C.create_string_buffer(128)
    check(lib().ettg_nccl_unique_id(buf))
    return buf.raw


def replicate_rank(index: InlabelIndex | None, n: int, root: int, uid: bytes, rank: int,
                   nranks: int, device: int) -> InlabelIndex:
    """One process per GPU: the root passes its built index, the others None;
    every rank gets an index for the root's tree (ettg_lca_replicate_rank)."""
    h = C.c_void_p(index.handle.value if index is not None else None)
    if index is not None:
        index._h = None  # ownership moves through the call (the root gets it back)
    check(lib().ettg_lca_replicate_rank(C.byref(h), int(root), C.c_char_p(bytes(uid)), int(rank),
                                        int(nranks), int(device)))
    return InlabelIndex(h.value, n, device, ENGINE_INLABEL)


def query_multi(replicas: list[InlabelIndex], queries, batch_size: int,
                engine: int = ENGINE_INLABEL) -> np.ndarray:
    """answer_batch over several replicas: the batch is split contiguously, one
    host thread drives each GPU, answers come back in query order."""
    q = np.ascontiguousarray(np.asarray(queries, dtype=np.int64).reshape(-1, 2))
    out = np.empty(q.shape[0], np.int64)
    hs = (C.c_void_p * len(replicas))(*[r.handle.value for r in replicas])
    check(lib().ettg_lca_query_multi(hs, len(replicas), engine, ptr(q), q.shape[0],
                                     int(batch_size), ptr(out)))
    return out


def answer_batch(index: _LcaHandle, queries, batch_size: int) -> np.ndarray:
    """answer_batch (core/include/ett/lca.hpp:50-65) for the index's engine."""
    engine = (ENGINE_RMQ if isinstance(index, RmqLcaIndex) else
              ENGINE_NAIVE if isinstance(index, NaiveIndex) else ENGINE_INLABEL)
    return index.query(queries, batch_size, engine)


def inlabel_lca(index: InlabelIndex, x: int, y: int) -> int:
    return int(index.query(np.array([[x, y]], np.int64), 1, ENGINE_INLABEL)[0])


def rmq_lca(index: RmqLcaIndex, x: int, y: int) -> int:
    return int(index.query(np.array([[x, y]], np.int64), 1, ENGINE_RMQ)[0])


def naive_lca(index: NaiveIndex, x: int, y: int) -> int:
    return int(index.query(np.array([[x, y]], np.int64), 1, ENGINE_NAIVE)[0])


def node_stats(tree: RootedTree, device: int = 0) -> NodeStats:
    """node_stats(linearize(build_half_edges(tree_edges(t)), root)) (core/src/euler.cpp)."""
    return inlabel_build(tree, device).stats()


# ------------------------------------------------------------------ bridges
@dataclass
class AdjacencyIndex:
    """core/include/ett/graph.hpp:44-63."""
    n: int
    m: int
    offsets: np.ndarray
    neighbors: np.ndarray
    edge_ids: np.ndarray


def _phases(engine: int, pt, on_tree: bool = False) -> dict:
    """Phase names as the reference records them (core/src/bridges.cpp:292-337)."""
    phases = {} if on_tree else {"spanning": pt.spanning_ms}
    if engine != _lib.BRIDGES_CK:
        phases["euler"] = pt.euler_ms
    if engine == _lib.BRIDGES_TV:
        phases["lowhigh"] = pt.lowhigh_ms
    else:
        phases["marking"] = pt.marking_ms
    phases["total"] = pt.total_ms
    return phases


def _bridges(g, engine: int, device: int, times: dict | None, tree_mask=None) -> BridgeMask:
    """g: EdgeList (8 B per edge over the link) or AdjacencyIndex (the
    reference engines' input type; the edge list is recovered on the device)."""
    mask = np.zeros(g.m() if isinstance(g, EdgeList) else g.m, np.uint8)
    pt = _lib.PhaseTimes()
    tm = None
    if tree_mask is not None:
        tm = np.ascontiguousarray(np.asarray(tree_mask) != 0, np.uint8)
        if len(tm) != len(mask):
            raise InvalidArgument("tree mask size mismatch")
    if isinstance(g, AdjacencyIndex):
        off = np.ascontiguousarray(g.offsets, np.int64)
        nbr = np.ascontiguousarray(g.neighbors, np.int64)
        eid = np.ascontiguousarray(g.edge_ids, np.int64)
        check(lib().ettg_bridges_csr(ptr(off), ptr(nbr), ptr(eid), int(g.n), int(g.m), device,
                                     engine, ptr(tm) if tm is not None else None, ptr(mask),
                                     C.byref(pt)))
    elif tm is not None:
        check(lib().ettg_bridges_on_tree(ptr(g.edges), int(g.n), g.m(), device, ptr(tm),
                                         ptr(mask), C.byref(pt)))
    else:
        check(lib().ettg_bridges_engine(ptr(g.edges), int(g.n), g.m(), device, engine, ptr(mask),
                                        C.byref(pt)))
    phases = _phases(engine, pt, tm is not None)
    if times is not None:
        times.update(phases)
    return BridgeMask(mask, phases)


def tv_bridges(g, device: int = 0, times: dict | None = None) -> BridgeMask:
    """tv_bridges (core/src/bridges.cpp:311-316) on an EdgeList or an
    AdjacencyIndex; times gets spanning/euler/lowhigh ms."""
    return _bridges(g, _lib.BRIDGES_TV, device, times)


def tv_bridges_on_tree(g, tree_mask, device: int = 0, times: dict | None = None) -> BridgeMask:
    """tv_bridges_on_tree (core/src/bridges.cpp:289-309): the TV criterion on a
    caller spanning tree (mask per edge).  Not a spanning tree -> InvalidArgument
    "not a tree: m != n - 1" / "not a tree: disconnected" (core/src/euler.cpp:13-33)."""
    return _bridges(g, _lib.BRIDGES_TV, device, times, tree_mask)


@dataclass
class LowHigh:
    """core/include/ett/bridges.hpp LowHigh, plus the preorder it is numbered
    in and the spanning tree it was computed on."""
    preorder: np.ndarray
    low: np.ndarray
    high: np.ndarray
    tree_mask: np.ndarray


def low_high(g: EdgeList, tree_mask=None, device: int = 0) -> LowHigh:
    """The TV engine's low/high intermediate (core/src/bridges.cpp:251-287)
    on tree_mask, or on its own hooking tree when tree_mask is None: per node
    the preorder (root 0, the engine's Euler-tour order) and the min / max
    preorder over the subtree and its non-tree neighbours.  Diagnostic."""
    n, m = int(g.n), g.m()
    tm = None
    if tree_mask is not None:
        tm = np.ascontiguousarray(np.asarray(tree_mask) != 0, np.uint8)
        if len(tm) != m:
            raise InvalidArgument("tree mask size mismatch")
    tree = np.zeros(max(m, 1), np.uint8)
    pre, low, high = (np.empty(max(n, 1), np.int64) for _ in range(3))
    check(lib().ettg_bridges_low_high(ptr(g.edges), n, m, device,
                                      ptr(tm) if tm is not None else None, ptr(tree),
                                      ptr(pre), ptr(low), ptr(high)))
    return LowHigh(pre[:n], low[:n], high[:n], tree[:m] if tm is None else tm)


def ck_bridges(g, device: int = 0, times: dict | None = None) -> BridgeMask:
    """ck_bridges (core/src/bridges.cpp:318-325): BFS tree + CK marking."""
    return _bridges(g, _lib.BRIDGES_CK, device, times)


def hybrid_bridges(g, device: int = 0, times: dict | None = None) -> BridgeMask:
    """hybrid_bridges (core/src/bridges.cpp:327-339): hooking + Euler rooting + CK marking."""
    return _bridges(g, _lib.BRIDGES_HYBRID, device, times)


@dataclass
class ParseStats:
    """core/include/ett/graph.hpp:27-32."""
    self_loops_removed: int = 0
    duplicates_removed: int = 0

    def removed(self) -> int:
        return self.self_loops_removed + self.duplicates_removed


def _parse(fn: str, data, stats: ParseStats | None, device: int) -> EdgeList:
    if hasattr(data, "read"):
        data = data.read()
    if isinstance(data, str):
        data = data.encode()
    data = bytes(data)
    cap = len(data) // 4 + 2  # an edge line takes >= 4 bytes ("u v\\n"): always enough
    edges = np.empty((cap, 2), np.int64)
    n, m, st = C.c_int64(), C.c_int64(), _lib.ParseStatsC()
    check(getattr(lib(), fn)(data, len(data), device, ptr(edges), cap, C.byref(n), C.byref(m),
                             C.byref(st)))
    if stats is not None:
        stats.self_loops_removed = st.self_loops_removed
        stats.duplicates_removed = st.duplicates_removed
    return EdgeList(n.value, edges[: m.value])


def parse_edge_list(data, stats: ParseStats | None = None, device: int = 0) -> EdgeList:
    """parse_edge_list (core/src/graph.cpp:57-82) on the device; `data` is the
    file's bytes / str or a binary file object.  Raises ParseError (the
    reference's std::runtime_error) with the same "line N: ..." message."""
    return _parse("ettg_parse_edge_list", data, stats, device)


def parse_dimacs_gr(data, stats: ParseStats | None = None, device: int = 0) -> EdgeList:
    """parse_dimacs_gr (core/src/graph.cpp:84-128) on the device."""
    return _parse("ettg_parse_dimacs_gr", data, stats, device)


def write_edge_list(g: EdgeList) -> bytes:
    """write_edge_list (core/src/graph.cpp:131-133): "u v\\n" per edge."""
    need = C.c_int64()
    rc = lib().ettg_write_edge_list(ptr(g.edges), g.m(), None, 0, C.byref(need))
    if rc not in (_lib.ETTG_OK, _lib.ETTG_ERANGE):
        check(rc, gen=True)
    buf = C.create_string_buffer(max(need.value, 1))
    check(lib().ettg_write_edge_list(ptr(g.edges), g.m(), buf, need.value, C.byref(need)),
          gen=True)
    return buf.raw[: need.value]


def build_adjacency(g: EdgeList, device: int = 0) -> AdjacencyIndex:
    """build_adjacency (core/src/graph.cpp:135-173), on the device."""
    m = g.m()
    off = np.empty(g.n + 1, np.int64)
    nbr = np.empty(max(2 * m, 1), np.int64)
    eid = np.empty(max(2 * m, 1), np.int64)
    check(lib().ettg_build_adjacency(ptr(g.edges), int(g.n), m, device, ptr(off), ptr(nbr),
                                     ptr(eid)))
    return AdjacencyIndex(g.n, m, off, nbr[:2 * m], eid[:2 * m])


@dataclass
class ComponentResult:
    """core/include/ett/graph.hpp:76-79."""
    graph: EdgeList
    old_to_new: np.ndarray


def largest_component(g: EdgeList, device: int = 0) -> ComponentResult:
    """largest_component (core/src/graph.cpp:219-259), on the device."""
    m = g.m()
    o2n = np.empty(max(g.n, 1), np.int64)
    out = np.empty((max(m, 1), 2), np.int64)
    nn, mm = C.c_int64(), C.c_int64()
    check(lib().ettg_largest_component(ptr(g.edges), int(g.n), m, device, ptr(o2n), C.byref(nn),
                                       C.byref(mm), ptr(out)))
    kept = out[:mm.value]
    if 2 * mm.value < m:  # release the over-allocation only when it is large
        kept = kept.copy()
    return ComponentResult(EdgeList(nn.value, kept), o2n[:g.n])


@dataclass
class SpanningTree:
    """core/include/ett/bridges.hpp:12-18 (BFS variant)."""
    is_tree_edge: np.ndarray
    level: np.ndarray
    parent: np.ndarray
    parent_edge: np.ndarray


def bfs_tree(g, root: int = 0, device: int = 0) -> SpanningTree:
    """bfs_tree (core/src/bridges.cpp:198-249) of an EdgeList or an
    AdjacencyIndex, bit-identical to the reference."""
    m = g.m() if isinstance(g, EdgeList) else int(g.m)
    mask = np.zeros(max(m, 1), np.uint8)
    lev, par, pe = (np.empty(g.n, np.int64) for _ in range(3))
    if isinstance(g, AdjacencyIndex):
        off = np.ascontiguousarray(g.offsets, np.int64)
        nbr = np.ascontiguousarray(g.neighbors, np.int64)
        eid = np.ascontiguousarray(g.edge_ids, np.int64)
        check(lib().ettg_bfs_tree_csr(ptr(off), ptr(nbr), ptr(eid), int(g.n), m, int(root),
                                      device, ptr(mask), ptr(lev), ptr(par), ptr(pe)))
    else:
        check(lib().ettg_bfs_tree(ptr(g.edges), int(g.n), m, int(root), device, ptr(mask),
                                  ptr(lev), ptr(par), ptr(pe)))
    return SpanningTree(mask[:m], lev, par, pe)


# --------------------------------------------------------------- primitives
def _torch():
    import torch
    return torch


def list_rank(succ, head: int, device: int = 0) -> np.ndarray:
    """list_rank (core/src/primitives.cpp:145); succ uses -1 as the tail."""
    torch = _torch()
    s = np.asarray(succ, dtype=np.int64)
    if len(s) == 0:
        return np.zeros(0, np.int64)
    if head < 0 or head >= len(s):
        raise InvalidArgument("list head out of range")
    if np.any((s < -1) | (s >= len(s))):
        # narrowing would wrap such a value onto a valid index; the reference
        # indexes succ with it (undefined), here it is an error
        raise InvalidArgument("linked list successor out of range")
    d = torch.from_numpy(s.astype(np.uint32)).to(f"cuda:{device}")
    r = torch.empty_like(d)
    check(lib().ettg_list_rank_dev(ptr(d), len(s), int(head), ptr(r), device,
                                   torch.cuda.current_stream(device).cuda_stream))
    return r.cpu().numpy().astype(np.int64)


def exclusive_scan(values, device: int = 0) -> np.ndarray:
    """exclusive_scan(values, +, 0) over uint32 (core/include/ett/primitives.hpp:29)."""
    torch = _torch()
    v = np.asarray(values, dtype=np.uint32)
    if len(v) == 0:
        return np.zeros(0, np.int64)
    d = torch.from_numpy(v).to(f"cuda:{device}")
    out = torch.empty_like(d)
    check(lib().ettg_exclusive_scan_dev(ptr(d), len(v), ptr(out), device,
                                        torch.cuda.current_stream(device).cuda_stream))
    return out.cpu().numpy().astype(np.int64)


def sort_pairs(keys, vals, device: int = 0):
    torch = _torch()
    k = torch.from_numpy(np.asarray(keys, dtype=np.uint32)).to(f"cuda:{device}")
    v = torch.from_numpy(np.asarray(vals, dtype=np.uint32)).to(f"cuda:{device}")
    ko, vo = torch.empty_like(k), torch.empty_like(v)
    check(lib().ettg_sort_pairs_dev(ptr(k), ptr(v), k.numel(), ptr(ko), ptr(vo), device,
                                    torch.cuda.current_stream(device).cuda_stream))
    return ko.cpu().numpy(), vo.cpu().numpy()


K_PLUS_INF = (1 << 63) - 1   # ett::kPlusInf
K_MINUS_INF = -(1 << 63)     # ett::kMinusInf


def list_scan(succ, values, head: int, device: int = 0) -> np.ndarray:
    """list_scan (core/src/primitives.cpp:156-162): out[i] = sum of values
    strictly before i in list order; succ uses -1 as the tail."""
    s = np.ascontiguousarray(succ, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.int64)
    if len(v) != len(s):
        raise InvalidArgument("list_scan: values size mismatch")
    out = np.empty(len(s), np.int64)
    if len(s) == 0:
        return out
    check(lib().ettg_list_scan(ptr(s), ptr(v), len(s), int(head), device, ptr(out)))
    return out


_REDUCE_OPS = {"min": _lib.REDUCE_MIN, "max": _lib.REDUCE_MAX, "sum": _lib.REDUCE_SUM}


def segmented_reduce(values, offsets, op: str, identity: int, device: int = 0):
    """segmented_reduce (core/include/ett/primitives.hpp:81-98) with op in
    {"min", "max", "sum"}.  Host arrays in, numpy out; torch CUDA tensors in,
    a CUDA tensor out (ettg_segmented_reduce_dev)."""
    if op not in _REDUCE_OPS:
        raise InvalidArgument(f"segmented_reduce: unknown op {op!r}")
    if hasattr(values, "is_cuda") and values.is_cuda:
        torch = _torch()
        segs = max(offsets.numel() - 1, 0)
        out = torch.empty(segs, dtype=torch.int64, device=values.device)
        check(lib().ettg_segmented_reduce_dev(
            ptr(values), values.numel(), ptr(offsets), offsets.numel(), _REDUCE_OPS[op],
            int(identity), ptr(out), values.device.index or 0,
            torch.cuda.current_stream(values.device).cuda_stream))
        return out
    v = np.ascontiguousarray(values, dtype=np.int64)
    o = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.empty(max(len(o) - 1, 0), np.int64)
    check(lib().ettg_segmented_reduce(ptr(v), len(v), ptr(o), len(o), _REDUCE_OPS[op],
                                      int(identity), device, ptr(out)))
    return out


class RangeIndex:
    """RangeIndex (core/include/ett/primitives.hpp:100-121): inclusive range
    min/max over int64 keys, built and queried on the device.  ``min(l, r)``
    and ``max(l, r)`` answer one range like the reference; ``mins`` /
    ``maxs`` / ``minmax`` answer a batch of (l, r) pairs in one launch."""

    def __init__(self, keys, device: int = 0):
        self._h = None
        self.device = device
        h = C.c_void_p()
        if hasattr(keys, "is_cuda") and keys.is_cuda:
            torch = _torch()
            k = keys.contiguous().to(torch.int64)
            self.device = k.device.index or 0
            check(lib().ettg_range_index_build_dev(
                ptr(k), k.numel(), self.device, torch.cuda.current_stream(k.device).cuda_stream,
                C.byref(h)))
        else:
            k = np.ascontiguousarray(keys, dtype=np.int64)
            check(lib().ettg_range_index_build(ptr(k), len(k), device, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ettg_range_index_free(self._h)
            self._h = None

    def size(self) -> int:
        return int(lib().ettg_range_index_size(self._h))

    def _query(self, ranges, want_min: bool, want_max: bool):
        r = np.ascontiguousarray(ranges, dtype=np.int64).reshape(-1, 2)
        q = len(r)
        mins = np.empty(q, np.int64) if want_min else None
        maxs = np.empty(q, np.int64) if want_max else None
        if q:
            check(lib().ettg_range_index_query(self._h, ptr(r), q, ptr(mins), ptr(maxs)))
        return mins, maxs

    def min(self, l: int, r: int) -> int:
        return int(self._query([(l, r)], True, False)[0][0])

    def max(self, l: int, r: int) -> int:
        return int(self._query([(l, r)], False, True)[1][0])

    def mins(self, ranges) -> np.ndarray:
        return self._query(ranges, True, False)[0]

    def maxs(self, ranges) -> np.ndarray:
        return self._query(ranges, False, True)[1]

    def minmax(self, ranges):
        return self._query(ranges, True, True)

    def query_dev(self, d_ranges, d_mins=None, d_maxs=None, stream=None):
        """Device-resident batch: d_ranges int64[q, 2] CUDA tensor."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        check(lib().ettg_range_index_query_dev(self._h, ptr(d_ranges), d_ranges.numel() // 2,
                                               ptr(d_mins), ptr(d_maxs), st))


def rmq_build(keys, device: int = 0) -> RangeIndex:
    """rmq_build (core/include/ett/primitives.hpp:116-118)."""
    return RangeIndex(keys, device)


def rmq_min(idx: RangeIndex, l: int, r: int) -> int:
    return idx.min(l, r)


def rmq_max(idx: RangeIndex, l: int, r: int) -> int:
    return idx.max(l, r)


def exclusive_scan_i64(values, device: int = 0) -> np.ndarray:
    """exclusive_scan(values, +, 0) over int64, wrapping modulo 2^64."""
    torch = _torch()
    v = np.ascontiguousarray(values, dtype=np.int64)
    if len(v) == 0:
        return np.zeros(0, np.int64)
    d = torch.from_numpy(v).to(f"cuda:{device}")
    check(lib().ettg_exclusive_scan_i64_dev(ptr(d), len(v), ptr(d), device,
                                            torch.cuda.current_stream(device).cuda_stream))
    return d.cpu().numpy()


# --------------------------------------------------------------- generators
def grasp_tree(n: int, gamma: int = K_GRASP_INFINITY, seed: int = 0) -> RootedTree:
    par = np.empty(n, np.int64)
    check(lib().ettg_gen_grasp_tree(n, gamma & ((1 << 64) - 1), seed, ptr(par)), gen=True)
    return RootedTree(n, 0, par)


def barabasi_tree(n: int, seed: int) -> RootedTree:
    par = np.empty(n, np.int64)
    check(lib().ettg_gen_barabasi_tree(n, seed, ptr(par)), gen=True)
    return RootedTree(n, 0, par)


def permute_labels(t: RootedTree, seed: int) -> RootedTree:
    out = np.empty(t.n, np.int64)
    root = C.c_int64()
    check(lib().ettg_gen_permute_labels(t.n, ptr(t.parent), t.root, seed, ptr(out),
                                        C.byref(root)), gen=True)
    return RootedTree(t.n, root.value, out)


def sample_queries(n: int, q: int, seed: int) -> np.ndarray:
    out = np.empty((q, 2), np.int64)
    check(lib().ettg_gen_sample_queries(n, q, seed, ptr(out)), gen=True)
    return out


def random_connected_graph(n: int, m: int, seed: int) -> EdgeList:
    out = np.empty((m, 2), np.int64)
    check(lib().ettg_gen_random_connected_graph(n, m, seed, ptr(out)), gen=True)
    return EdgeList(n, out)


def planted_bridge_graph(n: int, m: int, b: int, seed: int):
    """(EdgeList, truth mask) with exactly b bridges."""
    out = np.empty((m, 2), np.int64)
    truth = np.empty(m, np.uint8)
    check(lib().ettg_gen_planted_bridge_graph(n, m, b, seed, ptr(out), ptr(truth)), gen=True)
    return EdgeList(n, out), truth


def road_like_graph(W: int, H: int, extra: int, r: int, pendant: int, seed: int):
    """(EdgeList, truth mask): lattice + chords within radius r + pendant bridges."""
    m = lib().ettg_road_like_edge_count(W, H, extra, r, pendant)
    if m < 0:
        raise InvalidArgument("road_like_graph: bad shape")
    out = np.empty((m, 2), np.int64)
    truth = np.empty(m, np.uint8)
    check(lib().ettg_gen_road_like_graph(W, H, extra, r, pendant, seed, ptr(out), ptr(truth)),
          gen=True)
    return EdgeList(W * H + pendant, out), truth


def grasp_tree_dev(n: int, gamma: int, seed: int, d_parent, device: int = 0,
                   stream: int | None = None) -> bool:
    """Counter-mode grasp_tree into a uint32/int32 device tensor (root 0 ->
    0xFFFFFFFF); False if a Lemire rejection invalidated the counter replay."""
    rej = C.c_int()
    check(lib().ettg_gen_grasp_tree_dev(n, gamma, seed, ptr(d_parent), C.byref(rej), device,
                                        stream))
    return rej.value == 0


def permute_labels_dev(d_parent, n: int, root: int, seed: int, d_out, device: int = 0,
                       stream: int | None = None) -> tuple[int, bool]:
    """permute_labels on the device (parallel Fisher-Yates, bit-identical);
    returns (new root, counter replay valid)."""
    r, rej = C.c_int64(), C.c_int()
    check(lib().ettg_gen_permute_labels_dev(ptr(d_parent), n, root, seed, ptr(d_out), C.byref(r),
                                            C.byref(rej), device, stream))
    return r.value, rej.value == 0


def gen_queries_dev(n: int, q: int, seed: int, offset: int, d_pairs, device: int = 0,
                    stream: int | None = None) -> bool:
    """Counter-mode sample_queries into a uint32 device tensor; False on rejection."""
    rej = C.c_int()
    check(lib().ettg_gen_queries_dev(n, q, seed, offset, ptr(d_pairs), C.byref(rej), device,
                                     stream))
    return rej.value == 0
