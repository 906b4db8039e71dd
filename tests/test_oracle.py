"""CPU suite: pins the oracle before anything is checked against it.

1. The C restatement (oracle/ettg_oracle.c) reproduces the reference's own
   golden vectors (tests/{euler,lca,primitives,bridges}_test.cpp,
   tests/acceptance.cpp) and the committed fixtures in tests/golden/.
2. It agrees with the compiled reference (oracle/_ref) on the acceptance
   corpora: 200 trees (exhaustive/sampled pairs) and 205 graphs.
3. Our host generators replay the reference's SplitMix64 streams exactly.
"""
import os

import numpy as np
import pytest

from util import GRASP_INF, bridge_corpus, lca_corpus

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EXAMPLE = np.array([-1, 2, 0, 0, 0, 2], np.int64)


@pytest.fixture(scope="module")
def port(orc):
    if not orc.have_port():
        pytest.skip("oracle restatement not built")
    return orc.Port


def test_golden_euler_tour(port):
    # tests/euler_test.cpp:110-128, tests/acceptance.cpp:96-106
    s, d = port.euler_tour(EXAMPLE, 0)
    assert list(zip(s.tolist(), d.tolist())) == [(0, 2), (2, 1), (1, 2), (2, 5), (5, 2),
                                                 (2, 0), (0, 3), (3, 0), (0, 4), (4, 0)]
    # root 2 starts with (2,0) (tests/euler_test.cpp:120-128)
    t = np.array([2, 2, -1, 0, 0, 2], np.int64)
    s2, d2 = port.euler_tour(t, 2)
    assert (s2[0], d2[0]) == (2, 0)


def test_golden_stats_and_inlabel(port):
    pre, size, lev, par = port.node_stats(EXAMPLE, 0)
    assert pre.tolist() == [1, 3, 2, 5, 6, 4]
    assert lev.tolist() == [0, 2, 1, 1, 1, 2]
    assert size[2] == 3 and size[0] == 6
    inl, asc, head, lev2, par2 = port.inlabel_index(EXAMPLE, 0)
    assert inl.tolist() == [4, 3, 4, 5, 6, 4]
    assert head[4] == 0
    inl1, asc1, *_ = port.inlabel_index(np.array([-1]), 0)
    assert inl1.tolist() == [1] and asc1.tolist() == [1]
    q = np.array([[1, 5], [3, 4]])
    assert port.lca_inlabel(EXAMPLE, 0, q).tolist() == [2, 0]
    assert port.lca_rmq(EXAMPLE, 0, q).tolist() == [2, 0]


def test_golden_primitives(port):
    # tests/primitives_test.cpp:42-97
    assert port.exclusive_scan([1, 0, 1, -1]).tolist() == [0, 1, 1, 2]
    assert port.list_rank([1, 2, -1], 0).tolist() == [0, 1, 2]
    assert port.list_rank([-1, 0, 1], 2).tolist() == [2, 1, 0]
    with pytest.raises(Exception, match="cycle"):
        port.list_rank([1, 2, 0], 0)


PLUS_INF, MINUS_INF = (1 << 63) - 1, -(1 << 63)


def test_golden_list_scan_segreduce_rangeindex(port):
    # tests/primitives_test.cpp:88-97 (list_scan), :110-129 (segmented_reduce),
    # :131-170 (RangeIndex)
    assert port.list_scan([1, 2, -1], 0, [5, 7, 9]).tolist() == [0, 5, 12]
    assert port.segmented_reduce([3, 1, 2], [0, 2, 3], "min", PLUS_INF).tolist() == [1, 2]
    assert port.segmented_reduce([3, 1, 2], [0, 0, 3], "min", PLUS_INF).tolist() == [PLUS_INF, 1]
    with pytest.raises(Exception, match="bad offsets"):
        port.segmented_reduce([3, 1, 2], [0, 2], "min", PLUS_INF)
    mins, maxs = port.range_index([2, 9, 4, 1], [(0, 3), (1, 1), (1, 2)])
    assert mins.tolist() == [1, 9, 4] and maxs.tolist() == [9, 9, 9]
    for bad in [(0, 4), (-1, 2), (2, 1)]:
        with pytest.raises(Exception, match="bad range"):
            port.range_index([2, 9, 4, 1], [bad])


def test_list_scan_segreduce_rangeindex_vs_reference(port, ref):
    rng = np.random.default_rng(11)
    for k in (1, 2, 7, 1000, 20_000):
        order = rng.permutation(k)
        succ = np.full(k, -1, np.int64)
        succ[order[:-1]] = order[1:]
        vals = rng.integers(-(1 << 40), 1 << 40, k)
        assert np.array_equal(port.list_scan(succ, int(order[0]), vals),
                              ref.list_scan(succ, int(order[0]), vals))
    for segs in (1, 5, 300):
        lens = rng.integers(0, 40, segs)
        offs = np.concatenate([[0], np.cumsum(lens)])
        vals = rng.integers(-1000, 1000, int(offs[-1]))
        for op, ident in (("min", PLUS_INF), ("max", MINUS_INF), ("sum", 0), ("min", 3)):
            assert np.array_equal(port.segmented_reduce(vals, offs, op, ident),
                                  ref.segmented_reduce(vals, offs, op, ident))
    for n in (1, 2, 33, 1000):
        keys = rng.integers(-(1 << 62), 1 << 62, n)
        l = rng.integers(0, n, 500)
        r = rng.integers(0, n, 500)
        rr = np.stack([np.minimum(l, r), np.maximum(l, r)], 1)
        pm, px = port.range_index(keys, rr)
        qm, qx = ref.range_index(keys, rr)
        assert np.array_equal(pm, qm) and np.array_equal(px, qx)


def test_golden_bridges(port):
    # tests/bridges_test.cpp:45-147
    cases = [
        (4, [[0, 1], [1, 2], [0, 2], [2, 3]], [0, 0, 0, 1]),
        (6, [[0, 1], [1, 2], [0, 2], [2, 3], [3, 4], [4, 5], [3, 5]], [0, 0, 0, 1, 0, 0, 0]),
        (4, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]], [0] * 6),
        (6, [[0, 1], [1, 2], [2, 3], [3, 4], [4, 5], [0, 5]], [0] * 6),
    ]
    for n, e, want in cases:
        assert port.bridges("tv", n, e).tolist() == want
        assert port.bridges("dfs", n, e).tolist() == want


def test_fixtures(port):
    """tests/golden/*.npz were produced by tests/golden/make_golden.py from
    the compiled reference; the restatement must reproduce them."""
    z = np.load(os.path.join(GOLDEN, "lca_golden.npz"))
    for i in range(int(z["count"])):
        par, root, q = z[f"parent{i}"], int(z[f"root{i}"]), z[f"q{i}"]
        pre, size, lev, p = port.node_stats(par, root)
        assert np.array_equal(pre, z[f"pre{i}"]) and np.array_equal(size, z[f"size{i}"])
        inl, asc, head, _, _ = port.inlabel_index(par, root)
        assert np.array_equal(inl, z[f"inlabel{i}"])
        assert np.array_equal(asc, z[f"asc{i}"])
        assert np.array_equal(port.lca_inlabel(par, root, q), z[f"ans{i}"])
    b = np.load(os.path.join(GOLDEN, "bridges_golden.npz"))
    for i in range(int(b["count"])):
        n, e = int(b[f"n{i}"]), b[f"edges{i}"]
        assert np.array_equal(port.bridges("tv", n, e), b[f"mask{i}"])


@pytest.mark.parametrize("engine", ["inlabel", "rmq"])
def test_lca_corpus_vs_reference(ett, port, ref, engine):
    for ti, t in enumerate(lca_corpus(ett, count=200)):
        if t.n <= 64:
            xs, ys = np.meshgrid(np.arange(t.n), np.arange(t.n), indexing="ij")
            q = np.stack([xs.ravel(), ys.ravel()], 1)
        else:
            q = ett.sample_queries(t.n, 2000, t.n)
        want = ref.lca("inlabel", t.parent, t.root, q)
        fn = port.lca_inlabel if engine == "inlabel" else port.lca_rmq
        assert np.array_equal(fn(t.parent, t.root, q), want), ti
        if ti % 10 == 0:
            assert np.array_equal(port.lca_walk_up(t.parent, q), want), ti


def test_stats_corpus_vs_reference(ett, port, ref):
    for ti, t in enumerate(lca_corpus(ett, count=120, seed=2024)):
        for a, b in zip(port.node_stats(t.parent, t.root), ref.node_stats(t.parent, t.root)):
            assert np.array_equal(a, b), ti
        for a, b in zip(port.inlabel_index(t.parent, t.root), ref.inlabel_index(t.parent, t.root)):
            assert np.array_equal(a, b), ti


def test_bridges_corpus_vs_reference(ett, port, ref):
    for i, (n, e) in enumerate(bridge_corpus(ett)):
        e = np.asarray(e, np.int64).reshape(-1, 2)
        want, _ = ref.bridges("brute", n, e) if len(e) <= 200 else ref.bridges("dfs", n, e)
        assert np.array_equal(port.bridges("tv", n, e), want), i
        assert np.array_equal(port.bridges("dfs", n, e), want), i


def test_invalid_trees_same_errors(port, ref):
    cases = [([-1, 0, 5], 0), ([-1, -1, 0], 0), ([1, -1, 0], 0), ([-1, 2, 1], 0)]
    for par, root in cases:
        par = np.array(par, np.int64)
        with pytest.raises(Exception) as e1:
            port.validate_tree(par, root)
        with pytest.raises(Exception) as e2:
            ref.node_stats(par, root)
        assert str(e1.value).split(" (code")[0] == str(e2.value).split(" (code")[0]


def test_medium_tree_vs_reference(ett, port, ref):
    t = ett.permute_labels(ett.grasp_tree(100_000, 3, 1), 2)
    q = ett.sample_queries(t.n, 20_000, 3)
    assert np.array_equal(port.lca_inlabel(t.parent, t.root, q),
                          ref.lca("inlabel", t.parent, t.root, q))


# ------------------------------------------------------------- generators
@pytest.mark.parametrize("gamma", [1, 7, GRASP_INF])
def test_generators_replay_reference_streams(ett, ref, gamma):
    n = 5000
    t = ett.grasp_tree(n, gamma, 1)
    assert np.array_equal(t.parent, ref.grasp_tree(n, gamma, 1))
    p, r = ref.permute_labels(t.parent, 0, 2)
    t2 = ett.permute_labels(t, 2)
    assert np.array_equal(t2.parent, p) and t2.root == r
    assert np.array_equal(ett.barabasi_tree(n, 9).parent, ref.barabasi_tree(n, 9))
    assert np.array_equal(ett.sample_queries(n, 3000, 3), ref.sample_queries(n, 3000, 3))
    assert np.array_equal(ett.random_connected_graph(400, 1500, 4).edges,
                          ref.random_connected_graph(400, 1500, 4))


def test_planted_and_road_generators_known_answers(ett, port):
    g, truth = ett.planted_bridge_graph(600, 4000, 30, 4)
    assert g.m() == 4000 and int(truth.sum()) == 30
    assert np.array_equal(port.bridges("dfs", g.n, g.edges), truth)
    e = np.sort(g.edges, axis=1)
    assert len(np.unique(e[:, 0] * g.n + e[:, 1])) == g.m()  # simple graph
    g2, truth2 = ett.road_like_graph(40, 30, 6, 3, 50, 5)
    assert g2.n == 40 * 30 + 50 and int(truth2.sum()) == 50
    assert np.array_equal(port.bridges("dfs", g2.n, g2.edges), truth2)
    e2 = np.sort(g2.edges, axis=1)
    assert len(np.unique(e2[:, 0] * g2.n + e2[:, 1])) == g2.m()
    # deterministic
    g3, _ = ett.road_like_graph(40, 30, 6, 3, 50, 5)
    assert np.array_equal(g2.edges, g3.edges)
