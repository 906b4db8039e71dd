"""Host-edge-list bridges on config D with ETTG_TRACE=1: staged-narrowing
host times vs the device phases vs the call's wall time (dev aid)."""
import os, sys, time
os.environ["ETTG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
m = g.m()
pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(L.ettg_bridges(pin_e.data_ptr(), g.n, m, 0, pin_m.data_ptr(), None))
    print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms ok={np.array_equal(pin_m.numpy(), truth)}",
          file=sys.stderr, flush=True)
