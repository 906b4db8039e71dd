"""Per-phase device timings (ETTG_TRACE=1) of TV bridges on config D (dev aid)."""
import os, sys, ctypes
os.environ.setdefault("ETTG_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
if os.environ.get("AB_LIB"):
    _lib.LIB_PATH = os.environ["AB_LIB"]
L = _lib.lib()
side = int(os.environ.get("SIDE", "5657"))  # config D: n = 32,022,410, m = 256,000,000
if os.environ.get("GRAPH") == "C":
    g, truth = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
else:
    g, truth = ett.road_like_graph(side, side, 6, 3, 20_761 * side * side // (5657 * 5657), 5)
de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
for _ in range(int(os.environ.get("REPS", "3"))):
    pt = _lib.PhaseTimes()
    _lib.check(L.ettg_bridges_dev(de.data_ptr(), g.n, g.m(), 0, dm.data_ptr(), None, ctypes.byref(pt)))
    print("bridges", pt.spanning_ms, pt.euler_ms, pt.lowhigh_ms, pt.total_ms, flush=True)
print("parity", np.array_equal(dm.cpu().numpy(), truth))
