"""Regenerate tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

Run here (where /root/reference exists and `make -C oracle ref` has built
oracle/_ref/libett_ref.so):  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
from oracle.oracle import Ref  # noqa: E402
from util import SplitMix64, GRASP_INF  # noqa: E402


def main():
    rng = SplitMix64(0x676f6c64656e)
    lca = {}
    count = 0
    for i in range(24):
        n = 1 + rng.next_below(300)
        gamma = [1, 3, GRASP_INF][i % 3]
        par = Ref.grasp_tree(n, gamma, rng.next()) if i % 4 != 3 else Ref.barabasi_tree(n, rng.next())
        par, root = Ref.permute_labels(par, 0, rng.next())
        q = Ref.sample_queries(n, 200, rng.next())
        pre, size, lev, p = Ref.node_stats(par, root)
        inl, asc, head, lev2, p2 = Ref.inlabel_index(par, root)
        lca[f"parent{count}"] = par
        lca[f"root{count}"] = np.int64(root)
        lca[f"q{count}"] = q
        lca[f"pre{count}"] = pre
        lca[f"size{count}"] = size
        lca[f"inlabel{count}"] = inl
        lca[f"asc{count}"] = asc
        lca[f"ans{count}"] = Ref.lca("inlabel", par, root, q)
        count += 1
    lca["count"] = np.int64(count)
    np.savez_compressed(os.path.join(HERE, "lca_golden.npz"), **lca)

    br = {}
    count = 0
    for i in range(24):
        n = 3 + rng.next_below(120)
        m = n - 1 + rng.next_below(min(3 * n, n * (n - 1) // 2) - (n - 1) + 1)
        e = Ref.random_connected_graph(n, m, rng.next())
        mask, _ = Ref.bridges("tv", n, e)
        br[f"n{count}"] = np.int64(n)
        br[f"edges{count}"] = e
        br[f"mask{count}"] = mask
        count += 1
    br["count"] = np.int64(count)
    np.savez_compressed(os.path.join(HERE, "bridges_golden.npz"), **br)
    print("wrote", len(lca), "+", len(br), "arrays")


if __name__ == "__main__":
    main()
