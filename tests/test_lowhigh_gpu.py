"""low/high intermediate parity.

The TV engine runs low/high over Euler-tour keys, which hides the values
behind the bridge test.  ettg_bridges_low_high exports them in preorder
numbers, and here they are checked against the reference's test oracle
recursive_low_high (tests/oracles.hpp:166-201) run on the GPU's own tree and
the GPU's own preorder, after checking that the preorder really is a DFS
preorder of that tree rooted at 0.  The reference's low_high
(core/src/bridges.cpp:251-287) is pinned to the same oracle on its own
rooting in test_reference_low_high_matches_recursive_oracle (CPU).
"""
from collections import deque

import numpy as np
import pytest


def _root_tree(n, edges, tree):
    """parent (-1 at root 0) and a BFS order of the tree edges, host side."""
    adj = [[] for _ in range(n)]
    for (u, v) in edges[tree != 0]:
        adj[u].append(v)
        adj[v].append(u)
    parent = np.full(n, -2, np.int64)
    parent[0] = -1
    order = [0]
    q = deque([0])
    while q:
        u = q.popleft()
        for w in adj[u]:
            if parent[w] == -2:
                parent[w] = u
                order.append(w)
                q.append(w)
    assert len(order) == n, "tree does not span the graph"
    return parent, np.array(order, np.int64)


def _check_preorder(n, parent, order, pre):
    """pre is a permutation of 1..n in which every subtree is the contiguous
    range [pre[v], pre[v] + size[v])."""
    assert np.array_equal(np.sort(pre), np.arange(1, n + 1))
    assert pre[0] == 1
    size = np.ones(n, np.int64)
    lo, hi = pre.copy(), pre.copy()
    for v in order[::-1][:-1]:  # children before parents, root excluded
        p = parent[v]
        size[p] += size[v]
        lo[p] = min(lo[p], lo[v])
        hi[p] = max(hi[p], hi[v])
    assert np.array_equal(lo, pre)
    assert np.array_equal(hi, pre + size - 1)


def _check(ett, ref, n, edges, tree_mask=None):
    g = ett.EdgeList(n, np.ascontiguousarray(edges, np.int64).reshape(-1, 2))
    lh = ett.low_high(g, tree_mask)
    assert int(lh.tree_mask.sum()) == n - 1
    parent, order = _root_tree(n, g.edges, lh.tree_mask)
    _check_preorder(n, parent, order, lh.preorder)
    low, high = ref.recursive_low_high(n, g.edges, lh.tree_mask, parent, 0, lh.preorder)
    assert np.array_equal(lh.low, low)
    assert np.array_equal(lh.high, high)
    return lh


@pytest.mark.gpu
def test_own_tree_bridge_corpus(ett, ref):
    from util import bridge_corpus
    for n, edges in bridge_corpus(ett, count=60):
        _check(ett, ref, n, np.asarray(edges))


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,seed", [(2000, 6000, 7), (50000, 200000, 8), (300000, 1200000, 9)])
def test_own_tree_random_graphs(ett, ref, n, m, seed):
    """300k nodes: 18.75k 32-slot blocks, so the root's and the big subtrees'
    ranges go through the superblock table as well as the sparse rows."""
    g = ett.random_connected_graph(n, m, seed)
    _check(ett, ref, n, g.edges)


@pytest.mark.gpu
def test_caller_trees(ett, ref):
    """The reference's hooking tree and its BFS tree as caller masks."""
    n, m = 20000, 90000
    g = ett.random_connected_graph(n, m, 11)
    for tm in (ref.spanning_tree_hooking(n, g.edges), ref.bfs_tree(n, g.edges)[0]):
        lh = _check(ett, ref, n, g.edges, tm)
        assert np.array_equal(lh.tree_mask, tm)


@pytest.mark.gpu
def test_planted_bridges_and_pure_trees(ett, ref):
    g, _ = ett.planted_bridge_graph(30000, 120000, 300, 5)
    _check(ett, ref, g.n, g.edges)
    # a tree: no non-tree edge, so low = preorder and high = last preorder
    # of the subtree
    t = ett.grasp_tree(40000, 4, 3)
    e = np.array([[v, p] for v, p in enumerate(t.parent) if p != -1], np.int64)
    lh = _check(ett, ref, 40000, e)
    assert np.array_equal(lh.low, lh.preorder)
    # a deep path with chords (long tour ranges, deep recursion in the oracle)
    n = 100000
    path = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
    rng = np.random.default_rng(1)
    chords = np.sort(rng.integers(0, n, size=(3000, 2)), 1)
    chords = chords[chords[:, 0] != chords[:, 1]]
    _check(ett, ref, n, np.concatenate([path, chords]))


@pytest.mark.gpu
def test_multi_edges_self_loops_and_tiny(ett, ref):
    _check(ett, ref, 1, np.zeros((0, 2), np.int64))
    _check(ett, ref, 2, np.array([[0, 1]]))
    _check(ett, ref, 2, np.array([[0, 1], [0, 1], [1, 1], [0, 0]]))
    _check(ett, ref, 5, np.array([[0, 1], [1, 2], [2, 3], [3, 4], [4, 0], [2, 2], [1, 3], [1, 3]]))


@pytest.mark.gpu
def test_errors(ett):
    g = ett.EdgeList(4, np.array([[0, 1], [2, 3]], np.int64))
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        ett.low_high(g)
    g = ett.EdgeList(3, np.array([[0, 1], [1, 2], [0, 2]], np.int64))
    with pytest.raises(ett.InvalidArgument, match="not a tree"):
        ett.low_high(g, np.array([1, 1, 1], np.uint8))


def test_reference_low_high_matches_recursive_oracle(ref):
    """CPU: the reference's own low_high on its euler_root_tree equals
    recursive_low_high on the same rooting -- pins the oracle the GPU tests
    use to the reference's production function."""
    for n, m, seed in [(500, 1500, 1), (3000, 9000, 2), (3000, 2999, 3)]:
        e = ref.random_connected_graph(n, m, seed)
        tm = ref.spanning_tree_hooking(n, e)
        pre, par, low, high = ref.low_high(n, e, tm)
        l2, h2 = ref.recursive_low_high(n, e, tm, par, 0, pre)
        assert np.array_equal(low, l2) and np.array_equal(high, h2)
