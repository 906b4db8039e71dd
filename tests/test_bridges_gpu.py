"""Bridges parity on the B200: CUDA Tarjan-Vishkin vs the reference / planted truth."""
import numpy as np
import pytest

from util import bridge_corpus

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,edges,want", [
    (4, [[0, 1], [1, 2], [0, 2], [2, 3]], [0, 0, 0, 1]),             # triangle + pendant
    (6, [[0, 1], [1, 2], [0, 2], [2, 3], [3, 4], [4, 5], [3, 5]], [0, 0, 0, 1, 0, 0, 0]),
    (6, [[0, 1], [1, 2], [2, 3], [3, 4], [4, 5], [0, 5]], [0] * 6),  # cycle
    (4, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]], [0] * 6),  # K4
    (5, [[0, 1], [1, 2], [1, 3], [3, 4]], [1, 1, 1, 1]),             # tree
    (2, [[0, 1]], [1]),
    (1, [], []),
])
def test_canonical(ett, n, edges, want):
    g = ett.EdgeList(n, np.array(edges, np.int64).reshape(-1, 2))
    assert ett.tv_bridges(g).is_bridge.tolist() == want


def test_corpus_vs_reference(ett, ref):
    """acceptance criterion 4: 205 instances vs the reference tv/dfs engines."""
    for i, (n, edges) in enumerate(bridge_corpus(ett)):
        edges = np.asarray(edges, np.int64).reshape(-1, 2)
        got = ett.tv_bridges(ett.EdgeList(n, edges)).is_bridge
        want, _ = ref.bridges("dfs", n, edges)
        assert np.array_equal(got, want), i
        want_tv, _ = ref.bridges("tv", n, edges)
        assert np.array_equal(got, want_tv), i


@pytest.mark.parametrize("n,m,b,seed", [(3000, 20_000, 40, 4), (100_000, 800_000, 1000, 5),
                                        (1_000_000, 8_000_000, 10_000, 4)])
def test_planted_truth(ett, ref, n, m, b, seed):
    g, truth = ett.planted_bridge_graph(n, m, b, seed)
    assert int(truth.sum()) == b
    got = ett.tv_bridges(g).is_bridge
    assert np.array_equal(got, truth)
    if n <= 100_000:
        want, _ = ref.bridges("dfs", n, g.edges)
        assert np.array_equal(got, want)


def test_road_like_small(ett, ref):
    g, truth = ett.road_like_graph(200, 150, 6, 3, 500, 5)
    got = ett.tv_bridges(g).is_bridge
    assert np.array_equal(got, truth)
    want, _ = ref.bridges("tv", g.n, g.edges)
    assert np.array_equal(got, want)


def test_random_connected_vs_reference(ett, ref):
    g = ett.random_connected_graph(200_000, 260_000, 7)  # sparse: many bridges
    got = ett.tv_bridges(g).is_bridge
    want, _ = ref.bridges("dfs", g.n, g.edges)
    assert got.sum() > 1000
    assert np.array_equal(got, want)


def test_multi_edges_and_self_loops(ett, ref):
    edges = np.array([[0, 1], [1, 2], [1, 2], [2, 3], [3, 3], [3, 4]], np.int64)
    got = ett.tv_bridges(ett.EdgeList(5, edges)).is_bridge
    assert got.tolist() == [1, 0, 0, 1, 0, 1]


def test_errors(ett):
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        ett.tv_bridges(ett.EdgeList(4, np.array([[0, 1], [2, 3]])))
    with pytest.raises(ett.InvalidArgument, match="out of range"):
        ett.tv_bridges(ett.EdgeList(3, np.array([[0, 1], [1, 3]])))
    with pytest.raises(ett.InvalidArgument):
        ett.tv_bridges(ett.EdgeList(0, np.zeros((0, 2), np.int64)))


@pytest.mark.parametrize("engine", ["tv", "hybrid", "ck"])
def test_errors_large_then_recovers(ett, engine):
    # TV checks the forest on the device and raises after its one final sync:
    # bad inputs must fail cleanly and leave the library usable.
    fn = {"tv": ett.tv_bridges, "ck": ett.ck_bridges, "hybrid": ett.hybrid_bridges}[engine]
    g, truth = ett.planted_bridge_graph(200_000, 1_000_000, 500, 4)
    two = np.concatenate([g.edges, g.edges + g.n])  # two copies: disconnected
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        fn(ett.EdgeList(2 * g.n, two))
    iso0 = g.edges + 1  # vertex 0 isolated (the forest root)
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        fn(ett.EdgeList(g.n + 1, iso0))
    bad = g.edges.copy()
    bad[12345, 1] = g.n + 7
    with pytest.raises(ett.InvalidArgument, match="out of range"):
        fn(ett.EdgeList(g.n, bad))
    assert np.array_equal(fn(g).is_bridge, truth)


def test_dev_path_errors_then_recovers(ett):
    import ctypes
    import torch
    from paper_2103_15217_b200 import _lib
    L = _lib.lib()
    g, truth = ett.planted_bridge_graph(100_000, 600_000, 300, 4)

    def run(edges, n):
        de = torch.from_numpy(edges.astype(np.int32).ravel()).cuda()
        dm = torch.empty(len(edges), dtype=torch.uint8, device="cuda")
        rc = L.ettg_bridges_dev(de.data_ptr(), n, len(edges), 0, dm.data_ptr(), None, None)
        torch.cuda.synchronize()
        return rc, dm.cpu().numpy()

    bad = g.edges.copy()
    bad[777, 0] = g.n
    rc, _ = run(bad, g.n)
    assert rc == _lib.ETTG_EINVAL and b"out of range" in L.ettg_last_error()
    rc, _ = run(np.concatenate([g.edges, g.edges + g.n]), 2 * g.n)
    assert rc == _lib.ETTG_EINVAL and b"disconnected" in L.ettg_last_error()
    rc, mask = run(g.edges, g.n)
    assert rc == 0 and np.array_equal(mask, truth)


@pytest.mark.parametrize("engine", ["tv", "hybrid"])
def test_streamed_host_input_chunks(ett, ref, engine, monkeypatch):
    """Large host edge lists are copied in chunks and hooked as they land;
    small chunks (ETTG_BR_CHUNK) exercise every chunk boundary on the corpus."""
    fn = {"tv": ett.tv_bridges, "hybrid": ett.hybrid_bridges}[engine]
    for chunk in ("1", "7", "1000"):
        monkeypatch.setenv("ETTG_BR_CHUNK", chunk)
        for gi, (n, edges) in enumerate(bridge_corpus(ett)[:60]):
            edges = np.asarray(edges, np.int64).reshape(-1, 2)
            want = ref.bridges("dfs", n, edges)[0]
            got = fn(ett.EdgeList(n, edges)).is_bridge
            assert np.array_equal(got, want), (chunk, gi)
    monkeypatch.setenv("ETTG_BR_CHUNK", "50000")
    g, truth = ett.planted_bridge_graph(100_000, 600_000, 300, 4)
    assert np.array_equal(fn(g).is_bridge, truth)
    bad = g.edges.copy()
    bad[599_000, 0] = g.n  # in the last chunk
    with pytest.raises(ett.InvalidArgument, match="out of range"):
        fn(ett.EdgeList(g.n, bad))
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        fn(ett.EdgeList(2 * g.n, np.concatenate([g.edges, g.edges + g.n])))


def test_phase_times_named(ett):
    g, truth = ett.planted_bridge_graph(3000, 20_000, 40, 4)
    times = {}
    ett.tv_bridges(g, times=times)
    assert set(times) >= {"spanning", "euler", "lowhigh"}
    assert all(v >= 0 for v in times.values())


# ------------------------------------------------ CK / hybrid / BFS / CSR
@pytest.mark.parametrize("engine", ["ck", "hybrid"])
def test_engines_on_corpus(ett, ref, engine):
    """acceptance criterion 4 for the other engines (tests/acceptance.cpp:177-219)."""
    fn = ett.ck_bridges if engine == "ck" else ett.hybrid_bridges
    for i, (n, edges) in enumerate(bridge_corpus(ett)):
        edges = np.asarray(edges, np.int64).reshape(-1, 2)
        want, _ = ref.bridges("dfs", n, edges)
        assert np.array_equal(fn(ett.EdgeList(n, edges)).is_bridge, want), i


@pytest.mark.parametrize("engine", ["ck", "hybrid"])
def test_engines_planted_and_road(ett, engine):
    fn = ett.ck_bridges if engine == "ck" else ett.hybrid_bridges
    g, truth = ett.planted_bridge_graph(100_000, 800_000, 1000, 5)
    assert np.array_equal(fn(g).is_bridge, truth)
    g2, truth2 = ett.road_like_graph(300, 200, 6, 3, 900, 5)
    times = {}
    assert np.array_equal(fn(g2, times=times).is_bridge, truth2)
    assert "marking" in times and "spanning" in times


def test_build_adjacency_bit_exact(ett, ref):
    for n, m, seed in [(2, 1, 1), (50, 300, 2), (20_000, 150_000, 3)]:
        g = ett.random_connected_graph(n, m, seed)
        a = ett.build_adjacency(g)
        off, nbr, eid = ref.build_adjacency(n, g.edges)
        assert np.array_equal(a.offsets, off) and np.array_equal(a.neighbors, nbr)
        assert np.array_equal(a.edge_ids, eid)
    # multi-edges and self-loops keep the reference's (neighbour, edge id) order
    e = np.array([[0, 1], [1, 0], [2, 2], [0, 1], [1, 2]], np.int64)
    a = ett.build_adjacency(ett.EdgeList(3, e))
    off, nbr, eid = ref.build_adjacency(3, e)
    assert np.array_equal(a.neighbors, nbr) and np.array_equal(a.edge_ids, eid)


def test_bfs_tree_bit_exact(ett, ref):
    for n, m, seed in [(10, 20, 1), (3000, 9000, 2), (200_000, 600_000, 3)]:
        g = ett.random_connected_graph(n, m, seed)
        st = ett.bfs_tree(g, 0)
        mask, lev, par, pe = ref.bfs_tree(n, g.edges, 0)
        assert np.array_equal(st.is_tree_edge, mask)
        assert np.array_equal(st.level, lev) and np.array_equal(st.parent, par)
        assert np.array_equal(st.parent_edge, pe)
    g2, _ = ett.road_like_graph(120, 90, 6, 3, 50, 7)
    st = ett.bfs_tree(g2, 5)
    mask, lev, par, pe = ref.bfs_tree(g2.n, g2.edges, 5)
    assert np.array_equal(st.level, lev) and np.array_equal(st.parent_edge, pe)
    with pytest.raises(ett.InvalidArgument, match="disconnected"):
        ett.bfs_tree(ett.EdgeList(4, np.array([[0, 1], [2, 3]])))


def test_largest_component_bit_exact(ett, ref):
    rng = np.random.default_rng(5)
    cases = []
    # several components incl. ties and isolated vertices
    cases.append((8, np.array([[0, 1], [2, 3], [4, 5], [5, 6], [6, 4]], np.int64)))
    cases.append((6, np.array([[0, 1], [2, 3], [4, 5]], np.int64)))  # all tied: min-id wins
    cases.append((5, np.zeros((0, 2), np.int64)))
    big = rng.integers(0, 300_000, size=(200_000, 2))
    cases.append((300_000, big))
    for n, e in cases:
        r = ett.largest_component(ett.EdgeList(n, e))
        o2n, nn, eo = ref.largest_component(n, e)
        assert np.array_equal(r.old_to_new, o2n) and r.graph.n == nn
        assert np.array_equal(r.graph.edges, eo.reshape(-1, 2))


@pytest.mark.parametrize("shape", ["star_sorted", "star_shuffled", "path_sorted", "path_reversed",
                                   "ladder"])
def test_adversarial_shapes_known_answer(ett, shape):
    """Hubs (a star: one vertex in every edge, contiguous or shuffled), long
    chains in sorted / reversed edge order, and a 2-edge-connected ladder."""
    rng = np.random.default_rng(3)
    n = 1_000_003
    if shape.startswith("star"):
        e = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1)
        truth = np.ones(n - 1, np.uint8)
    elif shape.startswith("path"):
        e = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
        truth = np.ones(n - 1, np.uint8)
    else:
        k = n // 2
        rails = np.concatenate([np.stack([np.arange(k - 1), np.arange(1, k)], 1),
                                np.stack([np.arange(k, 2 * k - 1), np.arange(k + 1, 2 * k)], 1)])
        e = np.concatenate([rails, np.stack([np.arange(k), np.arange(k, 2 * k)], 1)])
        n = 2 * k
        truth = np.zeros(len(e), np.uint8)
    if shape.endswith("shuffled") or shape == "ladder":
        e = e[rng.permutation(len(e))]
    if shape.endswith("reversed"):
        e = e[::-1].copy()
    for eng in ("tv", "hybrid"):
        fn = ett.tv_bridges if eng == "tv" else ett.hybrid_bridges
        mask = fn(ett.EdgeList(n, e)).is_bridge
        assert np.array_equal(mask, truth), (shape, eng)


@pytest.mark.parametrize("order", ["sorted", "reversed", "shuffled"])
def test_edge_order_independence(ett, order):
    """Ordered inputs (sorted edge lists are common in files) give the same
    mask; the second hooking pass links by hashed priority so id-sorted
    chains stay shallow."""
    n = 2_000_000
    path = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
    cyc = np.concatenate([path, [[n - 1, 0]]])
    rng = np.random.default_rng(3)
    for edges, want in ((path, np.ones(n - 1, np.uint8)), (cyc, np.zeros(n, np.uint8))):
        e = {"sorted": edges, "reversed": edges[::-1].copy(),
             "shuffled": edges[rng.permutation(len(edges))]}[order]
        for fn in (ett.tv_bridges, ett.hybrid_bridges):
            assert np.array_equal(fn(ett.EdgeList(n, e)).is_bridge, want)


@pytest.mark.parametrize("gamma,seed", [(2, 11), (64, 12), (0, 13)])
def test_tree_plus_few_chords_vs_reference(ett, ref, gamma, seed):
    """A random tree plus a few chords: most vertices carry no non-tree edge,
    so most low/high key slots stay neutral and many key ranges start at a
    neutral slot or cross block boundaries -- the cases the combined in-block
    suffix/prefix array and its neutral-slot masks handle (k_lh_block_ps,
    k_classify_tour).  Odd sizes leave partial 4-slot groups and blocks."""
    rng = np.random.default_rng(seed)
    n = 300_007
    t = ett.permute_labels(ett.grasp_tree(n, gamma if gamma else ett.K_GRASP_INFINITY, seed), seed)
    par = np.asarray(t.parent, np.int64)
    child = np.flatnonzero(par >= 0)
    tree = np.stack([child, par[child]], 1)
    chords = rng.integers(0, n, size=(1_501, 2))
    e = np.concatenate([tree, chords])
    e = e[rng.permutation(len(e))]
    got = ett.tv_bridges(ett.EdgeList(n, e)).is_bridge
    want, _ = ref.bridges("dfs", n, e)
    assert 0 < int(want.sum()) < len(e)
    assert np.array_equal(got, want)
    assert np.array_equal(ett.hybrid_bridges(ett.EdgeList(n, e)).is_bridge, want)
