"""Bridges on the config-D road-like graph, two calls (for ncu captures)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
side = int(os.environ.get("SIDE", "5600"))
g, truth = ett.road_like_graph(side, side, 6, 3, side * side // 49, 5)
de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
for _ in range(int(os.environ.get("REPS", "2"))):
    pt = _lib.PhaseTimes()
    _lib.check(_lib.lib().ettg_bridges_dev(de.data_ptr(), g.n, g.m(), 0, dm.data_ptr(), None, ctypes.byref(pt)))
    print("bridges ms", pt.spanning_ms, pt.euler_ms, pt.lowhigh_ms, pt.total_ms, flush=True)
print("parity", np.array_equal(dm.cpu().numpy(), truth))
