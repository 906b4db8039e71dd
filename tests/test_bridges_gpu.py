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


def test_phase_times_named(ett):
    g, truth = ett.planted_bridge_graph(3000, 20_000, 40, 4)
    times = {}
    ett.tv_bridges(g, times=times)
    assert set(times) >= {"spanning", "euler", "lowhigh"}
    assert all(v >= 0 for v in times.values())
