"""Sweep ETTG_RAW_FRAC (fraction of pinned-input chunks sent as int64 and
narrowed on the device) for the host LCA query (config B) and host bridges
(config D) calls (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
t = ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2)
idx = ett.inlabel_build(t)
q = ett.sample_queries(t.n, 16_000_000, 3)
pin_q = torch.from_numpy(q).pin_memory()
pin_a = torch.empty(len(q), dtype=torch.int64).pin_memory()
want = None
for rnd in range(2):
    for f in ("auto", "0", "0.375", "0.5", "1"):
        os.environ["ETTG_RAW_FRAC"] = f
        ts = []
        for _ in range(7):
            t0 = time.perf_counter()
            _lib.check(L.ettg_lca_query(idx.handle, pin_q.data_ptr(), len(q), len(q), pin_a.data_ptr()))
            ts.append(time.perf_counter() - t0)
        if want is None:
            want = pin_a.numpy().copy()
        print(rnd, f"LCA raw={f:5s} min {min(ts)*1e3:.2f} med {np.median(ts)*1e3:.2f} ms "
              f"{len(q)/min(ts)/1e9:.2f} Gq/s ok={np.array_equal(pin_a.numpy(), want)}", flush=True)
del idx, pin_q, pin_a
g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
m = g.m()
pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()
for rnd in range(2):
    for f in ("auto", "0", "0.33", "1"):
        os.environ["ETTG_RAW_FRAC"] = f
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(L.ettg_bridges(pin_e.data_ptr(), g.n, m, 0, pin_m.data_ptr(), None))
            ts.append(time.perf_counter() - t0)
        print(rnd, f"bridges raw={f:5s} min {min(ts)*1e3:.2f} med {np.median(ts)*1e3:.2f} ms "
              f"ok={np.array_equal(pin_m.numpy(), truth)}", flush=True)
