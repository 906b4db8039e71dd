import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
n = 150_000_000
rng = np.random.default_rng(5)
e = np.stack([np.arange(n - 1, dtype=np.int64), np.arange(1, n, dtype=np.int64)], 1)
# a few chords to make some non-bridges, reversed order
chords = np.array([[10, 1_000_000], [50_000_000, 90_000_000], [149_999_000, 149_999_998]], np.int64)
e = np.concatenate([e, chords])
de = torch.from_numpy(e.astype(np.int32).ravel()).cuda()
dm = torch.empty(len(e), dtype=torch.uint8, device='cuda')
for _ in range(2):
    pt = _lib.PhaseTimes()
    _lib.check(L.ettg_bridges_dev(de.data_ptr(), n, len(e), 0, dm.data_ptr(), None, ctypes.byref(pt)))
m = dm.cpu().numpy()
want = np.ones(len(e), np.uint8)
for a, b in chords[:, :]:
    want[a:b] = 0  # path edges (i, i+1) for a <= i < b are covered by the chord
want[-3:] = 0
print("n", n, "ms", pt.total_ms, "parity", bool(np.array_equal(m, want)), "bridges", int(m.sum()), int(want.sum()))
