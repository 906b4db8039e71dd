"""A/B of the host-edge-list bridges call (ettg_bridges, pinned int64 edges ->
host mask) on config D, toggling ETTG_BR_STREAM (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
g, truth = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
m = g.m()
pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()
res = {}
for rnd in range(2):
    for v in ("0", "1"):
        os.environ["ETTG_BR_STREAM"] = v
        ts = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(L.ettg_bridges(pin_e.data_ptr(), g.n, m, 0, pin_m.data_ptr(), None))
            ts.append(time.perf_counter() - t0)
        assert np.array_equal(pin_m.numpy(), truth), v
        res[v] = (min(ts) * 1e3, float(np.median(ts)) * 1e3)
    print(rnd, {k: f"min {a:.2f} ms, median {b:.2f} ms" for k, (a, b) in res.items()}, flush=True)
