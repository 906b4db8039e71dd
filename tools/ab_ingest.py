"""Wall time of the ingestion calls with pageable numpy buffers on config D
(build_adjacency, largest_component, bfs_tree); AB_LIB=<old .so> (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
if os.environ.get("AB_LIB"):
    _lib.LIB_PATH = os.environ["AB_LIB"]
g, _ = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
out = {}
for name, f in (("build_adjacency", lambda: ett.build_adjacency(g)),
                ("largest_component", lambda: ett.largest_component(g)),
                ("bfs_tree", lambda: ett.bfs_tree(g, 0))):
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t0)
    out[name] = round(1e3 * min(ts), 1)
adj = ett.build_adjacency(g)
out["adj_check"] = int(adj.offsets[-1]) == 2 * g.m() and int(adj.neighbors[:1000].sum())
print(out)
