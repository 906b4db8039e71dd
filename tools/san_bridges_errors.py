"""Bad-input paths of the bridge engines under compute-sanitizer (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_15217_b200 as ett
g, truth = ett.planted_bridge_graph(20_000, 100_000, 50, 4)
for fn in (ett.tv_bridges, ett.hybrid_bridges, ett.ck_bridges):
    for edges, n in ((np.concatenate([g.edges, g.edges + g.n]), 2 * g.n), (g.edges + 1, g.n + 1)):
        try:
            fn(ett.EdgeList(n, edges))
        except ett.InvalidArgument as e:
            print("ok:", e)
    assert np.array_equal(fn(g).is_bridge, truth)
print("done")
