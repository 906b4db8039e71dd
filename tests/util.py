"""Small helpers shared by the tests (pure Python, test-only)."""
from __future__ import annotations

M64 = (1 << 64) - 1
GRASP_INF = M64


class SplitMix64:
    """core/include/ett/rng.hpp:9-44, for drawing corpus parameters."""

    def __init__(self, seed: int):
        self.s = seed & M64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_below(self, bound: int) -> int:
        x = self.next()
        m = x * bound
        lo = m & M64
        if lo < bound:
            threshold = ((1 << 64) - bound) % bound
            while lo < threshold:
                x = self.next()
                m = x * bound
                lo = m & M64
        return m >> 64


def lca_corpus(ett, count=200, seed=0x616363657074, max_n=512):
    """The acceptance corpus (tests/acceptance.cpp:58-70): grasp gamma in
    {1, 4, inf} and Barabasi trees, all relabelled."""
    rng = SplitMix64(seed)
    trees = []
    gammas = [1, 4, GRASP_INF]
    for i in range(count):
        n = 1 + rng.next_below(max_n)
        if i % 4 == 3:
            t = ett.barabasi_tree(n, rng.next())
        else:
            t = ett.grasp_tree(n, gammas[i % 3], rng.next())
        trees.append(ett.permute_labels(t, rng.next()))
    return trees


def bridge_corpus(ett, count=200, seed=0x627269646765):
    """tests/acceptance.cpp:177-204: canonical instances + random graphs."""
    inst = []
    t = ett.grasp_tree(12, 3, 1)
    inst.append((12, [[min(v, p), max(v, p)] for v, p in enumerate(t.parent) if p != -1]))
    inst.append((6, [[min(i, (i + 1) % 6), max(i, (i + 1) % 6)] for i in range(6)]))
    inst.append((4, [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]))
    inst.append((4, [[0, 1], [1, 2], [0, 2], [2, 3]]))
    inst.append((6, [[0, 1], [1, 2], [0, 2], [2, 3], [3, 4], [4, 5], [3, 5]]))
    rng = SplitMix64(seed)
    for _ in range(count):
        n = 2 + rng.next_below(255)
        max_m = min(1024, n * (n - 1) // 2)
        m = n - 1 + rng.next_below(max_m - (n - 1) + 1)
        g = ett.random_connected_graph(n, m, rng.next())
        inst.append((n, g.edges))
    return inst
