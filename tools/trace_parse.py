"""Per-phase device timings (ETTG_TRACE=1) of parse_edge_list on config C text."""
import os, sys, time
os.environ.setdefault("ETTG_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_15217_b200 as ett
g, _ = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
text = ett.write_edge_list(g)
for _ in range(3):
    t0 = time.perf_counter()
    p = ett.parse_edge_list(text)
    print("wall ms", 1e3 * (time.perf_counter() - t0), flush=True)
print("parity", p.n == g.n and np.array_equal(p.edges, np.sort(g.edges, axis=1)))
