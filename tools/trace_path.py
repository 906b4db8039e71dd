"""Phase trace of bridges on a 10M path, sorted vs shuffled edge order (dev aid)."""
import os, sys, ctypes
os.environ["ETTG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
n = 10_000_000
path = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
rng = np.random.default_rng(1)
for name, e in (("sorted", path), ("shuffled", path[rng.permutation(n - 1)])):
    de = torch.from_numpy(e.astype(np.int32).ravel()).cuda()
    dm = torch.empty(len(e), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(de.data_ptr(), n, len(e), 0, dm.data_ptr(), None, ctypes.byref(pt)))
    print(name, flush=True)
