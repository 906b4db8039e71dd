"""The reference's bridges entry points as a drop-in, on the B200:

- tv_bridges / ck_bridges / hybrid_bridges over the reference's own input
  type, AdjacencyIndex (core/include/ett/bridges.hpp:55-61), through
  ettg_bridges_csr;
- tv_bridges_on_tree (bridges.hpp:58-60) with the caller's spanning tree,
  including the reference's tree-independence test
  (tests/bridges_test.cpp:163-169) and its check_is_tree errors
  (core/src/euler.cpp:13-33);
- host int64 edge lists narrowed to u32 on the way in, from pinned and
  pageable buffers alike.
"""
import numpy as np
import pytest

from util import bridge_corpus

pytestmark = pytest.mark.gpu


def _adj(orc, n, edges):
    off, nbr, eid = orc.Ref.build_adjacency(n, edges)
    return off, nbr, eid


def test_tree_independence_reference_case(ett, ref):
    """tests/bridges_test.cpp:163-169: random_connected_graph(80, 200, seed),
    seeds 100..109 -- tv_bridges(adj) == tv_bridges_on_tree(adj, bfs tree)."""
    for seed in range(100, 110):
        g = ett.random_connected_graph(80, 200, seed)
        adj = ett.build_adjacency(g)
        via_hooking = ett.tv_bridges(adj).is_bridge
        via_bfs = ett.tv_bridges_on_tree(adj, ett.bfs_tree(adj, 0).is_tree_edge).is_bridge
        assert np.array_equal(via_hooking, via_bfs), seed
        want, _ = ref.bridges("dfs", g.n, g.edges)
        assert np.array_equal(via_hooking, want), seed


def test_on_tree_with_reference_trees_corpus(ett, ref):
    """On the 205-graph corpus, the TV criterion on three different spanning
    trees -- the reference's deterministic hooking tree, its BFS tree, and the
    device's own -- gives the reference's mask, through both input forms."""
    for i, (n, edges) in enumerate(bridge_corpus(ett)):
        edges = np.asarray(edges, np.int64).reshape(-1, 2)
        g = ett.EdgeList(n, edges)
        want, _ = ref.bridges("tv", n, edges)
        hook = ref.spanning_tree_hooking(n, edges)
        bfs = ref.bfs_tree(n, edges)[0]
        off, nbr, eid = ref.build_adjacency(n, edges)
        adj = ett.AdjacencyIndex(n, len(edges), off, nbr, eid)
        for tree in (hook, bfs):
            assert np.array_equal(ett.tv_bridges_on_tree(g, tree).is_bridge, want), i
            assert np.array_equal(ett.tv_bridges_on_tree(adj, tree).is_bridge, want), i
        for fn in (ett.tv_bridges, ett.ck_bridges, ett.hybrid_bridges):
            assert np.array_equal(fn(adj).is_bridge, want), (i, fn.__name__)


def test_csr_large_planted(ett, ref):
    g, truth = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
    off, nbr, eid = ref.build_adjacency(g.n, g.edges)
    adj = ett.AdjacencyIndex(g.n, g.m(), off, nbr, eid)
    times = {}
    assert np.array_equal(ett.tv_bridges(adj, times=times).is_bridge, truth)
    assert list(times) == ["spanning", "euler", "lowhigh", "total"]
    st = ett.bfs_tree(adj, 0)
    want_bfs = ett.bfs_tree(g, 0)
    assert np.array_equal(st.parent, want_bfs.parent)
    assert np.array_equal(st.is_tree_edge, want_bfs.is_tree_edge)
    t2 = {}
    assert np.array_equal(ett.tv_bridges_on_tree(adj, st.is_tree_edge, times=t2).is_bridge, truth)
    assert list(t2) == ["euler", "lowhigh", "total"]


def test_on_tree_errors(ett):
    g = ett.EdgeList(4, np.array([[0, 1], [1, 2], [0, 2], [2, 3]], np.int64))
    adj = ett.build_adjacency(g)
    for x in (g, adj):
        with pytest.raises(ett.InvalidArgument, match=r"^not a tree: m != n - 1"):
            ett.tv_bridges_on_tree(x, [1, 1, 0, 0])
        with pytest.raises(ett.InvalidArgument, match=r"^not a tree: disconnected"):
            ett.tv_bridges_on_tree(x, [1, 1, 1, 0])  # the triangle is a cycle
        with pytest.raises(ett.InvalidArgument, match="size mismatch"):
            ett.tv_bridges_on_tree(x, [1, 1, 1])
        # any non-zero byte marks a tree edge
        assert ett.tv_bridges_on_tree(x, [7, 0, 255, 1]).is_bridge.tolist() == [0, 0, 0, 1]
    # a self-loop is never part of a spanning tree
    h = ett.EdgeList(2, np.array([[0, 0], [0, 1]], np.int64))
    with pytest.raises(ett.InvalidArgument, match="not a tree"):
        ett.tv_bridges_on_tree(h, [1, 0])
    # a large mask with a cycle (n - 1 edges, not spanning) and recovery after
    g2, truth = ett.planted_bridge_graph(100_000, 800_000, 100, 5)
    tree = ett.bfs_tree(g2, 0).is_tree_edge.copy()
    t_ids = np.flatnonzero(tree)
    nt_ids = np.flatnonzero(tree == 0)
    tree[t_ids[len(t_ids) // 2]] = 0
    tree[nt_ids[0]] = 1  # swaps a tree edge for a non-tree edge: usually a cycle
    try:
        got = ett.tv_bridges_on_tree(g2, tree).is_bridge
        assert np.array_equal(got, truth)  # the swap happened to keep a spanning tree
    except ett.InvalidArgument as e:
        assert str(e).startswith("not a tree: disconnected")
    assert np.array_equal(ett.tv_bridges(g2).is_bridge, truth)


def test_malformed_adjacency(ett):
    g = ett.EdgeList(4, np.array([[0, 1], [1, 2], [0, 2], [2, 3]], np.int64))
    a = ett.build_adjacency(g)
    bad = ett.AdjacencyIndex(4, 4, a.offsets.copy(), a.neighbors.copy(), a.edge_ids.copy())
    bad.offsets[4] += 1
    with pytest.raises(ett.InvalidArgument, match="malformed adjacency index"):
        ett.tv_bridges(bad)
    bad = ett.AdjacencyIndex(4, 4, a.offsets.copy(), a.neighbors.copy(), a.edge_ids.copy())
    bad.edge_ids[:] = 0  # edge ids 1..3 are never written
    with pytest.raises(ett.InvalidArgument, match="malformed adjacency index"):
        ett.tv_bridges(bad)
    bad = ett.AdjacencyIndex(4, 4, a.offsets.copy(), a.neighbors.copy(), a.edge_ids.copy())
    bad.neighbors[0] = 9
    with pytest.raises(ett.InvalidArgument, match="out of range"):
        ett.tv_bridges(bad)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_edges_narrowed_pinned_and_pageable(ett, pinned):
    """Host int64 edges cross the link as u32 (staged narrowing), above and
    below the streamed-hooking threshold; out-of-range ids in any chunk fail
    with the reference's message; negative ids too."""
    import torch
    for n, m, b in [(200_000, 1_500_000, 500), (4_000_000, 40_000_000, 2000)]:
        g, truth = ett.planted_bridge_graph(n, m, b, 6)
        e = torch.from_numpy(g.edges)
        if pinned:
            e = e.pin_memory()
        g2 = ett.EdgeList(g.n, e.numpy())
        assert np.array_equal(ett.tv_bridges(g2).is_bridge, truth)
        bad = e.clone().pin_memory() if pinned else e.clone()
        bad[len(bad) * 3 // 4, 1] = n  # in a late chunk
        with pytest.raises(ett.InvalidArgument, match="edge endpoint out of range"):
            ett.tv_bridges(ett.EdgeList(n, bad.numpy()))
        bad[len(bad) * 3 // 4, 1] = -5
        with pytest.raises(ett.InvalidArgument, match="edge endpoint out of range"):
            ett.tv_bridges(ett.EdgeList(n, bad.numpy()))
        assert np.array_equal(ett.tv_bridges(g2).is_bridge, truth)
