"""compute-sanitizer memcheck run of ettg_bridges_low_high (own and caller trees)."""
import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2103_15217_b200 as ett
for n, m, s in [(1, 0, 0), (2, 1, 1), (100, 300, 2), (5000, 20000, 3), (200000, 600000, 4)]:
    if n == 1:
        g = ett.EdgeList(1, np.zeros((0, 2), np.int64))
    elif m == n - 1:
        g = ett.EdgeList(n, np.array([[0, 1]], np.int64))
    else:
        g = ett.random_connected_graph(n, m, s)
    lh = ett.low_high(g)
    assert lh.preorder.min() == 1 and lh.preorder.max() == n
    tm = lh.tree_mask
    lh2 = ett.low_high(g, tm)
    # the rotation (hence the preorder) is race-dependent: check invariants only
    for x in (lh, lh2):
        assert (x.low <= x.preorder).all() and (x.high >= x.preorder).all()
        assert (x.low >= 1).all() and (x.high <= n).all()
print("sanitizer-run ok")
