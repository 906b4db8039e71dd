import os, sys, ctypes
os.environ["ETTG_TRACE"] = "1"
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g, truth = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
for eng in (1, 2):
    for _ in range(2):
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev_engine(de.data_ptr(), g.n, g.m(), 0, eng, dm.data_ptr(), None, ctypes.byref(pt)))
        print("engine", eng, pt.spanning_ms, pt.euler_ms, pt.marking_ms, pt.total_ms, flush=True)
