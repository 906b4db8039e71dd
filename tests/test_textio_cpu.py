"""write_edge_list (core/src/graph.cpp:131-133) is host formatting: no GPU."""
import numpy as np


def test_write_edge_list_matches_reference_format(ett):
    rng = np.random.default_rng(5)
    e = rng.integers(0, 1 << 40, (1000, 2))
    e[:3] = [[0, 1], [7, 7], [1 << 62, 3]]
    g = ett.EdgeList(int(e.max()) + 1, e)
    want = "".join(f"{a} {b}\n" for a, b in e.tolist()).encode()
    assert ett.write_edge_list(g) == want
    assert ett.write_edge_list(ett.EdgeList(0, np.zeros((0, 2), np.int64))) == b""
