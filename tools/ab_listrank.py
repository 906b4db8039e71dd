"""A/B of list-ranking knobs (ETTG_LR_WYLLIE, ETTG_LR_L0) on the callers that
rank lists: bridges config C/D, LCA build at 1M/16M, list_rank_dev (dev aid).

  VARIANTS="0;524288" python tools/ab_listrank.py       # env values of ETTG_LR_WYLLIE
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_15217_b200 as ett  # noqa: E402
from paper_2103_15217_b200 import _lib  # noqa: E402

L = _lib.lib()
KNOB = os.environ.get("KNOB", "ETTG_LR_WYLLIE")
VARIANTS = os.environ.get("VARIANTS", "0;524288").split(";")
REPS = int(os.environ.get("REPS", "7"))


def bridges_ms(de, dm, n, m):
    out = []
    for _ in range(REPS):
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(de.data_ptr(), n, m, 0, dm.data_ptr(), None,
                                      ctypes.byref(pt)))
        out.append(pt.total_ms)
    return float(np.median(out[1:]))


def build_ms(t):
    out = []
    for _ in range(REPS):
        out.append(ett.inlabel_build(t).build_ms())
    return float(np.median(out[1:]))


def lr_ms(d, k, head, r):
    st = torch.cuda.current_stream().cuda_stream
    out = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        _lib.check(L.ettg_list_rank_dev(d.data_ptr(), k, head, r.data_ptr(), 0, st))
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out[1:]))


cases = {}
gC, truthC = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
gD, truthD = ett.road_like_graph(5600, 5600, 6, 3, 640_000, 5)
graphs = {}
for name, g, truth in (("bridges_C", gC, truthC), ("bridges_D", gD, truthD)):
    de = torch.from_numpy(g.edges.astype(np.int32).ravel()).cuda()
    dm = torch.empty(g.m(), dtype=torch.uint8, device="cuda")
    graphs[name] = (de, dm, g.n, g.m(), truth)
trees = {"build_A_1M": ett.permute_labels(ett.grasp_tree(1_000_000, ett.K_GRASP_INFINITY, 1), 2),
         "build_E_16M": ett.permute_labels(ett.grasp_tree(16_000_000, ett.K_GRASP_INFINITY, 1), 2),
         "build_B_16M": ett.permute_labels(ett.grasp_tree(16_000_000, 1, 1), 2)}
lists = {}
for k in (2_000_000, 32_000_000):
    rng = np.random.default_rng(k)
    order = rng.permutation(k)
    succ = np.full(k, -1, np.int64)
    succ[order[:-1]] = order[1:]
    lists[f"list_rank_{k // 1_000_000}M"] = (
        torch.from_numpy(succ.astype(np.uint32)).cuda(), k, int(order[0]),
        torch.empty(k, dtype=torch.int32, device="cuda"), order)

res = {v: {} for v in VARIANTS}
for rnd in range(2):
    for v in VARIANTS:
        os.environ[KNOB] = v
        for name, (de, dm, n, m, truth) in graphs.items():
            res[v][name] = bridges_ms(de, dm, n, m)
            if rnd == 0:
                assert np.array_equal(dm.cpu().numpy(), truth), (v, name)
        for name, t in trees.items():
            res[v][name] = build_ms(t)
        for name, (d, k, head, r, order) in lists.items():
            res[v][name] = lr_ms(d, k, head, r)
            if rnd == 0:
                got = r.cpu().numpy().view(np.uint32).astype(np.int64)
                assert np.array_equal(got[order], np.arange(k)), (v, name)
    print(f"round {rnd}", flush=True)
    for v in VARIANTS:
        print(f"  {KNOB}={v}: " + "  ".join(f"{k} {x:.3f}" for k, x in res[v].items()), flush=True)
