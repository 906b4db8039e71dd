"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the CPU oracles.

* ``ref()``  -> oracle/_ref/libett_ref.so : the unmodified reference core/
  compiled by oracle/Makefile (plus our extern "C" wrapper ref_capi.cpp).
* ``port()`` -> oracle/_build/libettg_oracle.so : the plain-C restatement
  (oracle/ettg_oracle.c), pinned against the reference's golden vectors and
  against ``ref()`` in tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libett_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libettg_oracle.so")

_ref = None
_port = None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{msg} (code {code})")
        self.code = code


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_port() -> bool:
    return os.path.exists(PORT_SO)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError(f"reference oracle not built: {REF_SO}")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_inlabel_new.restype = C.c_void_p
        _ref = L
    return _ref


def port():
    global _port
    if _port is None:
        if not have_port():
            raise RuntimeError(f"oracle restatement not built: {PORT_SO}")
        L = C.CDLL(PORT_SO)
        L.orc_last_error.restype = C.c_char_p
        _port = L
    return _port


def _rc(L, rc, err_fn):
    if rc != 0:
        raise OracleError(rc, getattr(L, err_fn)().decode())


i64 = C.c_int64
u64 = C.c_uint64


# ------------------------------------------------------------- reference
class Ref:
    """The compiled reference library (oracle/_ref)."""

    @staticmethod
    def set_workers(w: int):
        ref().ref_set_workers(C.c_int(w))

    @staticmethod
    def workers() -> int:
        return ref().ref_workers()

    @staticmethod
    def grasp_tree(n, gamma, seed):
        out = np.empty(n, np.int64)
        _rc(ref(), ref().ref_grasp_tree(i64(n), u64(gamma), u64(seed), _p(out)), "ref_last_error")
        return out

    @staticmethod
    def barabasi_tree(n, seed):
        out = np.empty(n, np.int64)
        _rc(ref(), ref().ref_barabasi_tree(i64(n), u64(seed), _p(out)), "ref_last_error")
        return out

    @staticmethod
    def permute_labels(parent, root, seed):
        n = len(parent)
        out = np.empty(n, np.int64)
        r = C.c_int64()
        _rc(ref(), ref().ref_permute_labels(i64(n), _p(parent), i64(root), u64(seed), _p(out),
                                            C.byref(r)), "ref_last_error")
        return out, r.value

    @staticmethod
    def sample_queries(n, q, seed):
        out = np.empty((q, 2), np.int64)
        _rc(ref(), ref().ref_sample_queries(i64(n), i64(q), u64(seed), _p(out)), "ref_last_error")
        return out

    @staticmethod
    def random_connected_graph(n, m, seed):
        out = np.empty((m, 2), np.int64)
        _rc(ref(), ref().ref_random_connected_graph(i64(n), i64(m), u64(seed), _p(out)),
            "ref_last_error")
        return out

    @staticmethod
    def list_rank(succ, head):
        succ = np.ascontiguousarray(succ, np.int64)
        out = np.empty(len(succ), np.int64)
        _rc(ref(), ref().ref_list_rank(i64(len(succ)), _p(succ), i64(head), _p(out)),
            "ref_last_error")
        return out

    @staticmethod
    def list_scan(succ, head, values):
        succ = np.ascontiguousarray(succ, np.int64)
        values = np.ascontiguousarray(values, np.int64)
        out = np.empty(len(succ), np.int64)
        _rc(ref(), ref().ref_list_scan(i64(len(succ)), _p(succ), i64(head), _p(values), _p(out)),
            "ref_last_error")
        return out

    @staticmethod
    def segmented_reduce(values, offsets, op, identity):
        """op in {"min", "max", "sum"}."""
        v = np.ascontiguousarray(values, np.int64)
        o = np.ascontiguousarray(offsets, np.int64)
        out = np.empty(max(len(o) - 1, 0), np.int64)
        _rc(ref(), ref().ref_segmented_reduce(i64(len(v)), _p(v), i64(len(o)), _p(o),
                                              C.c_int({"min": 0, "max": 1, "sum": 2}[op]),
                                              i64(identity), _p(out)), "ref_last_error")
        return out

    @staticmethod
    def range_index(keys, ranges, want_min=True, want_max=True):
        k = np.ascontiguousarray(keys, np.int64)
        r = np.ascontiguousarray(ranges, np.int64).reshape(-1, 2)
        mins = np.empty(len(r), np.int64) if want_min else None
        maxs = np.empty(len(r), np.int64) if want_max else None
        _rc(ref(), ref().ref_range_index(i64(len(k)), _p(k), i64(len(r)), _p(r),
                                         _p(mins) if want_min else None,
                                         _p(maxs) if want_max else None), "ref_last_error")
        return mins, maxs

    @staticmethod
    def exclusive_scan_sum(values):
        v = np.ascontiguousarray(values, np.int64)
        out = np.empty(len(v), np.int64)
        _rc(ref(), ref().ref_exclusive_scan_sum(i64(len(v)), _p(v), _p(out)), "ref_last_error")
        return out

    @staticmethod
    def euler_tour(parent, root):
        n = len(parent)
        k = 2 * (n - 1)
        s = np.empty(max(k, 1), np.int64)
        d = np.empty(max(k, 1), np.int64)
        _rc(ref(), ref().ref_euler_tour(i64(n), _p(parent), i64(root), _p(s), _p(d)),
            "ref_last_error")
        return s[:k], d[:k]

    @staticmethod
    def node_stats(parent, root):
        n = len(parent)
        a = [np.empty(n, np.int64) for _ in range(4)]
        _rc(ref(), ref().ref_node_stats(i64(n), _p(parent), i64(root), *[_p(x) for x in a]),
            "ref_last_error")
        return a

    @staticmethod
    def inlabel_index(parent, root):
        n = len(parent)
        inl = np.empty(n, np.int64)
        asc = np.empty(n, np.uint64)
        head = np.empty(n + 1, np.int64)
        lev = np.empty(n, np.int64)
        par = np.empty(n, np.int64)
        _rc(ref(), ref().ref_inlabel_index(i64(n), _p(parent), i64(root), _p(inl), _p(asc),
                                           _p(head), _p(lev), _p(par)), "ref_last_error")
        return inl, asc, head, lev, par

    @staticmethod
    def lca(engine, parent, root, pairs, batch=None):
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        q = pairs.shape[0]
        out = np.empty(q, np.int64)
        _rc(ref(), ref().ref_lca(engine.encode(), i64(len(parent)), _p(parent), i64(root),
                                 _p(pairs), i64(q), i64(batch or max(q, 1)), _p(out)),
            "ref_last_error")
        return out

    @staticmethod
    def bridges(engine, n, edges):
        edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
        m = edges.shape[0]
        mask = np.empty(m, np.uint8)
        ph = np.zeros(4, np.int64)
        _rc(ref(), ref().ref_bridges(engine.encode(), i64(n), i64(m), _p(edges), _p(mask),
                                     _p(ph)), "ref_last_error")
        return mask, ph


def ref_parse(kind, text: bytes):
    """Reference parse_edge_list / parse_dimacs_gr -> (n, edges[m,2], stats) or OracleError."""
    L = ref()
    cap = text.count(b"\n") + 1
    edges = np.empty(2 * cap, np.int64)
    n, m, sl, du = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    rc = L.ref_parse(kind.encode(), C.c_char_p(text), i64(len(text)), C.byref(n), C.byref(m),
                     C.byref(sl), C.byref(du), _p(edges), i64(cap))
    _rc(L, rc, "ref_last_error")
    return n.value, edges[: 2 * m.value].reshape(-1, 2), (sl.value, du.value)


def ref_build_adjacency(n, edges):
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    off = np.empty(n + 1, np.int64)
    nbr = np.empty(max(2 * m, 1), np.int64)
    eid = np.empty(max(2 * m, 1), np.int64)
    _rc(ref(), ref().ref_build_adjacency(i64(n), i64(m), _p(edges), _p(off), _p(nbr), _p(eid)),
        "ref_last_error")
    return off, nbr[:2 * m], eid[:2 * m]


def ref_bfs_tree(n, edges, root=0):
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    mask = np.empty(max(m, 1), np.uint8)
    lev, par, pe = (np.empty(n, np.int64) for _ in range(3))
    _rc(ref(), ref().ref_bfs_tree(i64(n), i64(m), _p(edges), i64(root), _p(mask), _p(lev),
                                  _p(par), _p(pe)), "ref_last_error")
    return mask[:m], lev, par, pe


def ref_largest_component(n, edges):
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    o2n = np.empty(max(n, 1), np.int64)
    out = np.empty((max(m, 1), 2), np.int64)
    nn, mm = C.c_int64(), C.c_int64()
    _rc(ref(), ref().ref_largest_component(i64(n), i64(m), _p(edges), _p(o2n), C.byref(nn),
                                           C.byref(mm), _p(out)), "ref_last_error")
    return o2n[:n], nn.value, out[:mm.value]


def ref_spanning_tree_hooking(n, edges):
    """The reference's deterministic hooking tree mask (core/src/bridges.cpp:105-158)."""
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    mask = np.empty(max(m, 1), np.uint8)
    _rc(ref(), ref().ref_spanning_tree_hooking(i64(n), i64(m), _p(edges), _p(mask)),
        "ref_last_error")
    return mask[:m]


def ref_low_high(n, edges, tree_mask):
    """The reference's low_high (core/src/bridges.cpp:251-287) on its own
    euler_root_tree(tree_mask, root 0): (preorder, parent, low, high)."""
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    tm = np.ascontiguousarray(tree_mask, np.uint8)
    out = [np.empty(n, np.int64) for _ in range(4)]
    _rc(ref(), ref().ref_low_high(i64(n), i64(m), _p(edges), _p(tm), *[_p(a) for a in out]),
        "ref_last_error")
    return tuple(out)


def ref_recursive_low_high(n, edges, tree_mask, parent, root, preorder):
    """recursive_low_high (reference tests/oracles.hpp:166-201) over any rooted
    tree and preorder: (low, high)."""
    edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
    m = edges.shape[0]
    tm = np.ascontiguousarray(tree_mask, np.uint8)
    par = np.ascontiguousarray(parent, np.int64)
    pre = np.ascontiguousarray(preorder, np.int64)
    low, high = np.empty(n, np.int64), np.empty(n, np.int64)
    _rc(ref(), ref().ref_recursive_low_high(i64(n), i64(m), _p(edges), _p(tm), _p(par),
                                            i64(root), _p(pre), _p(low), _p(high)),
        "ref_last_error")
    return low, high


Ref.spanning_tree_hooking = staticmethod(ref_spanning_tree_hooking)
Ref.low_high = staticmethod(ref_low_high)
Ref.recursive_low_high = staticmethod(ref_recursive_low_high)
Ref.build_adjacency = staticmethod(ref_build_adjacency)
Ref.largest_component = staticmethod(ref_largest_component)
Ref.bfs_tree = staticmethod(ref_bfs_tree)


class RefInlabel:
    """Built reference InlabelIndex for timing build and queries apart."""

    def __init__(self, parent, root):
        L = ref()
        bn = C.c_int64()
        self.h = L.ref_inlabel_new(i64(len(parent)), _p(np.ascontiguousarray(parent, np.int64)),
                                   i64(root), C.byref(bn))
        if not self.h:
            raise OracleError(1, L.ref_last_error().decode())
        self.build_ns = bn.value

    def answer(self, pairs, batch=None):
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        q = pairs.shape[0]
        out = np.empty(q, np.int64)
        ns = C.c_int64()
        L = ref()
        _rc(L, L.ref_inlabel_answer(C.c_void_p(self.h), _p(pairs), i64(q),
                                    i64(batch or max(q, 1)), _p(out), C.byref(ns)),
            "ref_last_error")
        return out, ns.value

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_inlabel_free(C.c_void_p(self.h))
            self.h = None


# ------------------------------------------------------------ C restatement
class Port:
    """The plain-C restatement (oracle/ettg_oracle.c)."""

    @staticmethod
    def _call(fn, *args):
        _rc(port(), getattr(port(), fn)(*args), "orc_last_error")

    @staticmethod
    def validate_tree(parent, root):
        parent = np.ascontiguousarray(parent, np.int64)
        Port._call("orc_validate_tree", i64(len(parent)), _p(parent), i64(root))

    @staticmethod
    def list_rank(succ, head):
        succ = np.ascontiguousarray(succ, np.int64)
        out = np.empty(len(succ), np.int64)
        Port._call("orc_list_rank", i64(len(succ)), _p(succ), i64(head), _p(out))
        return out

    @staticmethod
    def list_scan(succ, head, values):
        succ = np.ascontiguousarray(succ, np.int64)
        values = np.ascontiguousarray(values, np.int64)
        out = np.empty(len(succ), np.int64)
        Port._call("orc_list_scan", i64(len(succ)), _p(succ), i64(head), _p(values), _p(out))
        return out

    @staticmethod
    def segmented_reduce(values, offsets, op, identity):
        v = np.ascontiguousarray(values, np.int64)
        o = np.ascontiguousarray(offsets, np.int64)
        out = np.empty(max(len(o) - 1, 0), np.int64)
        Port._call("orc_segmented_reduce", i64(len(v)), _p(v), i64(len(o)), _p(o),
                   C.c_int({"min": 0, "max": 1, "sum": 2}[op]), i64(identity), _p(out))
        return out

    @staticmethod
    def range_index(keys, ranges, want_min=True, want_max=True):
        k = np.ascontiguousarray(keys, np.int64)
        r = np.ascontiguousarray(ranges, np.int64).reshape(-1, 2)
        mins = np.empty(len(r), np.int64) if want_min else None
        maxs = np.empty(len(r), np.int64) if want_max else None
        Port._call("orc_range_index", i64(len(k)), _p(k), i64(len(r)), _p(r), _p(mins), _p(maxs))
        return mins, maxs

    @staticmethod
    def exclusive_scan(v):
        v = np.ascontiguousarray(v, np.int64)
        out = np.empty(len(v), np.int64)
        Port._call("orc_exclusive_scan", i64(len(v)), _p(v), _p(out))
        return out

    @staticmethod
    def euler_tour(parent, root):
        parent = np.ascontiguousarray(parent, np.int64)
        k = 2 * (len(parent) - 1)
        s = np.empty(max(k, 1), np.int64)
        d = np.empty(max(k, 1), np.int64)
        Port._call("orc_euler_tour", i64(len(parent)), _p(parent), i64(root), _p(s), _p(d))
        return s[:k], d[:k]

    @staticmethod
    def node_stats(parent, root):
        parent = np.ascontiguousarray(parent, np.int64)
        n = len(parent)
        a = [np.empty(n, np.int64) for _ in range(4)]
        Port._call("orc_node_stats", i64(n), _p(parent), i64(root), *[_p(x) for x in a])
        return a

    @staticmethod
    def inlabel_index(parent, root):
        parent = np.ascontiguousarray(parent, np.int64)
        n = len(parent)
        inl = np.empty(n, np.int64)
        asc = np.empty(n, np.uint64)
        head = np.empty(n + 1, np.int64)
        lev = np.empty(n, np.int64)
        par = np.empty(n, np.int64)
        Port._call("orc_inlabel_index", i64(n), _p(parent), i64(root), _p(inl), _p(asc),
                   _p(head), _p(lev), _p(par))
        return inl, asc, head, lev, par

    @staticmethod
    def inlabel_query(index, pairs):
        inl, asc, head, lev, par = index
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        out = np.empty(pairs.shape[0], np.int64)
        lifts = C.c_int64()
        Port._call("orc_inlabel_query", i64(len(inl)), _p(inl), _p(asc), _p(head), _p(lev),
                   _p(par), _p(pairs), i64(pairs.shape[0]), _p(out), C.byref(lifts))
        return out, lifts.value

    @staticmethod
    def lca_inlabel(parent, root, pairs):
        parent = np.ascontiguousarray(parent, np.int64)
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        out = np.empty(pairs.shape[0], np.int64)
        Port._call("orc_lca_inlabel", i64(len(parent)), _p(parent), i64(root), _p(pairs),
                   i64(pairs.shape[0]), _p(out))
        return out

    @staticmethod
    def lca_rmq(parent, root, pairs):
        parent = np.ascontiguousarray(parent, np.int64)
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        out = np.empty(pairs.shape[0], np.int64)
        Port._call("orc_lca_rmq", i64(len(parent)), _p(parent), i64(root), _p(pairs),
                   i64(pairs.shape[0]), _p(out))
        return out

    @staticmethod
    def lca_walk_up(parent, pairs):
        parent = np.ascontiguousarray(parent, np.int64)
        pairs = np.ascontiguousarray(pairs, np.int64).reshape(-1, 2)
        out = np.empty(pairs.shape[0], np.int64)
        Port._call("orc_lca_walk_up", i64(len(parent)), _p(parent), _p(pairs),
                   i64(pairs.shape[0]), _p(out))
        return out

    @staticmethod
    def bridges(engine, n, edges):
        edges = np.ascontiguousarray(edges, np.int64).reshape(-1, 2)
        m = edges.shape[0]
        mask = np.empty(m, np.uint8)
        fn = {"tv": "orc_tv_bridges", "dfs": "orc_dfs_bridges"}[engine]
        Port._call(fn, i64(n), i64(m), _p(edges), _p(mask))
        return mask
