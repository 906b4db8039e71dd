"""largest_component on a 10M path, sorted vs shuffled edge order (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2103_15217_b200 as ett
n = 10_000_000
path = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
rng = np.random.default_rng(1)
for name, e in (("sorted", path), ("shuffled", path[rng.permutation(n - 1)])):
    g = ett.EdgeList(n, e)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); r = ett.largest_component(g); ts.append(time.perf_counter() - t0)
    print(name, round(1e3 * min(ts), 1), r.graph.n, flush=True)
