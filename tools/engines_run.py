"""Bridges engine comparison (tv / ck / hybrid) on road-like and planted graphs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib


def dev_run(g, engine):
    """Device-resident edges (the H2D copy is not part of the engine time)."""
    de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
    dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
    pt = _lib.PhaseTimes()
    for _ in range(2):
        _lib.check(_lib.lib().ettg_bridges_dev_engine(de.data_ptr(), g.n, g.m(), 0, engine,
                                                      dm.data_ptr(), None, ctypes.byref(pt)))
    return dm.cpu().numpy(), {"spanning": pt.spanning_ms, "euler": pt.euler_ms,
                              "lowhigh": pt.lowhigh_ms, "marking": pt.marking_ms,
                              "total": pt.total_ms}
for side in [int(x) for x in os.environ.get("SIDES", "500,1000,2000").split(",")]:
    g, truth = ett.road_like_graph(side, side, 6, 3, side * side // 49, 5)
    for name, eng in [("tv", 0), ("hybrid", 2), ("ck", 1)]:
        mask, t = dev_run(g, eng)
        ok = np.array_equal(mask, truth)
        print(f"road side={side} n={g.n} m={g.m()} {name:6s} ok={ok} " +
              " ".join(f"{k}={v:.2f}" for k, v in t.items() if v), flush=True)
g, truth = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
for name, eng in [("tv", 0), ("hybrid", 2), ("ck", 1)]:
    mask, t = dev_run(g, eng)
    ok = np.array_equal(mask, truth)
    print(f"planted 1M/8M {name:6s} ok={ok} " + " ".join(f"{k}={v:.2f}" for k, v in t.items() if v),
          flush=True)
