"""Experiment: effect of cudaLimitMaxL2FetchGranularity on the gather-bound kernels."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g = ctypes.c_int()
L.ettg_get_l2_fetch_granularity(0, ctypes.byref(g)); print("default granularity", g.value, flush=True)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
def tq(idx, d, ans, reps=10):
    ts = []
    for _ in range(reps):
        flush.fill_(1); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); idx.query_dev(d, ans, 1); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
trees = {"B": ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2),
         "E": ett.permute_labels(ett.grasp_tree(16_000_000, ett.K_GRASP_INFINITY, 1), 2)}
q = 16_000_000
d = torch.empty(2 * q, dtype=torch.int32, device="cuda"); ett.gen_queries_dev(16_000_000, q, 3, 0, d)
ans = torch.empty(q, dtype=torch.int32, device="cuda")
gr, truth = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
de = torch.from_numpy(gr.edges.astype(np.int32).ravel()).cuda(); dm = torch.empty(gr.m(), dtype=torch.uint8, device="cuda")
for gran in [g.value, 32, 64, 128, g.value]:
    _lib.check(L.ettg_set_l2_fetch_granularity(0, gran))
    res = {}
    for k, t in trees.items():
        idx = ett.inlabel_build(t); idx = ett.inlabel_build(t)
        res[k + "_build"] = idx.build_ms(); res[k + "_query"] = tq(idx, d, ans)
    pts = []
    for _ in range(3):
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(de.data_ptr(), gr.n, gr.m(), 0, dm.data_ptr(), None, ctypes.byref(pt)))
        pts.append((pt.spanning_ms, pt.euler_ms, pt.lowhigh_ms, pt.total_ms))
    res["bridges"] = np.median(np.array(pts), 0).round(3).tolist()
    print(gran, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()}, flush=True)
