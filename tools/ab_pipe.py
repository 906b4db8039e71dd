"""A/B of the host narrowing pipeline (ETTG_PIPE=1, host_pipe_narrow) against
the round-1 three-buffer ring (ETTG_PIPE=0) on the reference-facing host
calls: LCA config B answer_batch with pinned / pageable pairs and pinned
answers, and tv_bridges on config D with a pinned / pageable int64 edge list
(dev aid; ETTG_TRACE=1 prints the pipeline's chunk / raw counts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
from paper_2103_15217_b200 import _lib
L = _lib.lib()
VARIANTS = [v.split(";") for v in os.environ.get(
    "VARIANTS", "ETTG_PIPE=0;ETTG_PIPE=1;ETTG_PIPE=1,ETTG_PIPE_CHUNK=262144;"
                "ETTG_PIPE=1,ETTG_PIPE_CHUNK=1048576;ETTG_PIPE=1,ETTG_PIPE_RAWQ=0").split(";")]
VARIANTS = [v[0] for v in VARIANTS]


def setenv(v):
    for k in ("ETTG_PIPE", "ETTG_PIPE_CHUNK", "ETTG_PIPE_RAWQ"):
        os.environ.pop(k, None)
    for kv in v.split(","):
        k, x = kv.split("=")
        os.environ[k] = x


def timeit(fn, reps):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3, float(np.median(ts)) * 1e3


if os.environ.get("SKIP_LCA") != "1":
    t = ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2)
    idx = ett.inlabel_build(t)
    q = ett.sample_queries(t.n, 16_000_000, 3)
    pin_q = torch.from_numpy(q).pin_memory()
    pin_a = torch.empty(len(q), dtype=torch.int64).pin_memory()
    want = None
    for rnd in range(2):
        for v in VARIANTS:
            setenv(v)
            for name, src in (("pinned", pin_q.data_ptr()), ("pageable", q.ctypes.data)):
                f = lambda: _lib.check(L.ettg_lca_query(idx.handle, src, len(q), len(q),
                                                        pin_a.data_ptr()))
                f()
                if want is None:
                    want = pin_a.numpy().copy()
                ok = np.array_equal(pin_a.numpy(), want)
                mn, md = timeit(f, 9)
                print(rnd, f"LCA B pairs={name:8s} {v:40s} min {mn:.2f} med {md:.2f} ms "
                      f"{len(q) / mn / 1e6:.2f} Gq/s ok={ok}", flush=True)
    del idx, pin_q, pin_a
if os.environ.get("SKIP_BR") != "1":
    g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
    m = g.m()
    pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
    pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()
    for rnd in range(2):
        for v in VARIANTS:
            setenv(v)
            for name, src in (("pinned", pin_e.data_ptr()), ("pageable", g.edges.ctypes.data)):
                f = lambda: _lib.check(L.ettg_bridges(src, g.n, m, 0, pin_m.data_ptr(), None))
                f()
                ok = np.array_equal(pin_m.numpy(), truth)
                mn, md = timeit(f, 3)
                print(rnd, f"bridges D edges={name:8s} {v:40s} min {mn:.2f} med {md:.2f} ms "
                      f"ok={ok}", flush=True)
