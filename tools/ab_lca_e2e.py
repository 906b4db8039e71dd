"""A/B of the host LCA query call (ettg_lca_query) on config B: ETTG_NARROW,
pinned / pageable pairs and answers (dev aid)."""
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
pg_a = np.empty(len(q), np.int64)
want = None
for rnd in range(2):
    for nar in ("1", "0"):
        os.environ["ETTG_NARROW"] = nar
        for kind, qq, aa in (("pinned", pin_q.numpy(), pin_a.numpy()), ("pageable", q, pg_a),
                             ("pin-in/pg-out", pin_q.numpy(), pg_a)):
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                _lib.check(L.ettg_lca_query(idx.handle, qq.ctypes.data, len(q), len(q), aa.ctypes.data))
                ts.append(time.perf_counter() - t0)
            if want is None:
                want = aa.copy()
            print(rnd, f"narrow={nar} {kind:14s} min {min(ts)*1e3:.2f} med {np.median(ts)*1e3:.2f} ms "
                  f"{len(q)/min(ts)/1e9:.2f} Gq/s ok={np.array_equal(aa, want)}", flush=True)
