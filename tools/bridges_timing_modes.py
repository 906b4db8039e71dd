"""Config D bridges total (PhaseTimes.total_ms, events on the call's stream)
with / without an L2 flush before each call and with / without ETTG_TRACE
phase marks (dev aid: where the bench's number differs from the trace)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 << 18, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for fl in (0, 1):
    tot = []
    for _ in range(6):
        if fl:
            flush.fill_(1)
        torch.cuda.synchronize()
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(de.data_ptr(), g.n, g.m(), 0, dm.data_ptr(), st.cuda_stream,
                                      ctypes.byref(pt)))
        tot.append(pt.total_ms)
    print(f"trace={os.environ.get('ETTG_TRACE', '0')} flush={fl} total ms {np.round(tot, 3).tolist()}",
          flush=True)
print("parity", np.array_equal(dm.cpu().numpy(), truth))
