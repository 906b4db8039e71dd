"""Wall time of the reference-facing calls with pageable numpy buffers
(answer_batch, inlabel_build from a host parent array, tv_bridges, parse),
AB_LIB=<old .so> for the comparison (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
if os.environ.get("AB_LIB"):
    _lib.LIB_PATH = os.environ["AB_LIB"]


def best(f, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), r


t = ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2)
qs = ett.sample_queries(t.n, 16_000_000, 3)
ms_build, idx = best(lambda: ett.inlabel_build(t))
ms_q, ans = best(lambda: ett.answer_batch(idx, qs, len(qs)))
g, truth = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
ms_br, mask = best(lambda: ett.tv_bridges(g).is_bridge, 2)
gc, _ = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
text = ett.write_edge_list(gc)
ms_p, _ = best(lambda: ett.parse_edge_list(text))
print({"inlabel_build_16M_ms": round(ms_build, 2), "answer_batch_16M_ms": round(ms_q, 2),
       "tv_bridges_D_ms": round(ms_br, 2), "parse_C_ms": round(ms_p, 2),
       "bridges_ok": bool(np.array_equal(mask, truth)), "anshash": int(ans.sum())})
