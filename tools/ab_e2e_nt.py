"""ettg_lca_query with pageable numpy pairs / answers (answers buffer reused,
so no page faults in the timed calls) and ettg_bridges with a pinned host
mask, best and median of 9 (dev aid; AB_LIB=<old .so> for the comparison)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
if os.environ.get("AB_LIB"):
    _lib.LIB_PATH = os.environ["AB_LIB"]
L = _lib.lib()
t = ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2)
qs = np.ascontiguousarray(ett.sample_queries(t.n, 16_000_000, 3))
idx = ett.inlabel_build(t)
ans = np.empty(len(qs), np.int64)
ans[:] = 0  # fault the pages in
ts = []
for _ in range(9):
    t0 = time.perf_counter()
    _lib.check(L.ettg_lca_query(idx.handle, qs.ctypes.data, len(qs), len(qs), ans.ctypes.data))
    ts.append(time.perf_counter() - t0)
g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
pin_m = torch.empty(g.m(), dtype=torch.uint8).pin_memory()
tb = []
for _ in range(9):
    t0 = time.perf_counter()
    _lib.check(L.ettg_bridges(pin_e.data_ptr(), g.n, g.m(), 0, pin_m.data_ptr(), None))
    tb.append(time.perf_counter() - t0)
print({"query_pageable_ms": [round(1e3 * min(ts), 2), round(1e3 * float(np.median(ts)), 2)],
       "bridges_pinned_ms": [round(1e3 * min(tb), 2), round(1e3 * float(np.median(tb)), 2)],
       "ok": bool(np.array_equal(pin_m.numpy(), truth)), "anshash": int(ans.sum())}, flush=True)
