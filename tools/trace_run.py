"""Per-phase device timings (ETTG_TRACE=1) for the LCA build and bridges."""
import os, sys, ctypes
os.environ["ETTG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
for gamma in (1, ett.K_GRASP_INFINITY):
    t = ett.permute_labels(ett.grasp_tree(16_000_000, gamma, 1), 2)
    for _ in range(3):
        idx = ett.inlabel_build(t)
    print("build_ms", idx.build_ms(), flush=True)
g, truth = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
for _ in range(3):
    pt = _lib.PhaseTimes()
    _lib.check(L.ettg_bridges_dev(de.data_ptr(), g.n, g.m(), 0, dm.data_ptr(), None, ctypes.byref(pt)))
    print("bridges", pt.spanning_ms, pt.euler_ms, pt.lowhigh_ms, pt.total_ms, flush=True)
print("parity", np.array_equal(dm.cpu().numpy(), truth))
