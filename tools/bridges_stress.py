"""Bridges on adversarial shapes (dev aid): long path (shuffled / sorted edge
order), star, cycle, ladder; time + parity against the known answer."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
rng = np.random.default_rng(1)


def run(name, n, edges, truth):
    de = torch.from_numpy(edges.astype(np.int32).ravel()).cuda()
    dm = torch.empty(len(edges), dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(3):
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(de.data_ptr(), n, len(edges), 0, dm.data_ptr(), None,
                                      ctypes.byref(pt)))
        ts.append(pt.total_ms)
    ok = np.array_equal(dm.cpu().numpy(), truth)
    print(f"{name:28s} n={n:>9} m={len(edges):>9} {min(ts):8.3f} ms  parity={ok}", flush=True)


n = 10_000_000
path = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
run("path, sorted", n, path, np.ones(n - 1, np.uint8))
run("path, reversed", n, path[::-1].copy(), np.ones(n - 1, np.uint8))
perm = rng.permutation(n - 1)
run("path, shuffled", n, path[perm], np.ones(n - 1, np.uint8))
relabel = rng.permutation(n)
run("path, shuffled + relabeled", n, relabel[path[perm]], np.ones(n - 1, np.uint8))
star = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1)
run("star", n, star[rng.permutation(n - 1)], np.ones(n - 1, np.uint8))
cyc = np.concatenate([path, [[n - 1, 0]]])
run("cycle", n, cyc[rng.permutation(n)], np.zeros(n, np.uint8))
k = n // 2  # ladder: two rails + rungs, 2-edge-connected
rails = np.concatenate([np.stack([np.arange(k - 1), np.arange(1, k)], 1),
                        np.stack([np.arange(k, 2 * k - 1), np.arange(k + 1, 2 * k)], 1)])
rungs = np.stack([np.arange(k), np.arange(k, 2 * k)], 1)
lad = np.concatenate([rails, rungs])
run("ladder", 2 * k, lad[rng.permutation(len(lad))], np.zeros(len(lad), np.uint8))
