"""LCA engine comparison on B200 (the paper's Figs. 3-6 comparison: inlabel vs
RMQ-on-tour vs naive walk-up), device-resident queries, L2 flushed before
each timed launch, CUDA events.  Development/profiling aid."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2103_15217_b200 as ett

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(idx, d, ans, eng, reps=10):
    st = torch.cuda.current_stream()
    idx.query_dev(d, ans, eng, st.cuda_stream)
    evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for e0, e1 in evs:
        flush.fill_(1)
        e0.record(st); idx.query_dev(d, ans, eng, st.cuda_stream); e1.record(st)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / reps


rows = []
for name, n, gamma, q in [("A: 1M grasp(inf)", 1_000_000, ett.K_GRASP_INFINITY, 1_000_000),
                          ("1M gamma=2", 1_000_000, 2, 1_000_000),
                          ("B: 16M path", 16_000_000, 1, 16_000_000),
                          ("16M grasp(inf)", 16_000_000, ett.K_GRASP_INFINITY, 16_000_000)]:
    t = ett.permute_labels(ett.grasp_tree(n, gamma, 1), 2)
    idx = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ | ett.ENGINE_NAIVE)
    d = torch.empty(2 * q, dtype=torch.int32, device="cuda")
    ett.gen_queries_dev(n, q, 3, 0, d)
    res = {"tree": name, "layout": idx.layout()[0]}
    ref = None
    for eng, en in [(ett.ENGINE_INLABEL, "inlabel"), (ett.ENGINE_RMQ, "rmq"), (ett.ENGINE_NAIVE, "naive")]:
        qq = q if not (en == "naive" and gamma != ett.K_GRASP_INFINITY) else min(q, 20_000)
        ans = torch.empty(qq, dtype=torch.int32, device="cuda")
        ms = timed(idx, d[: 2 * qq], ans, eng, reps=10 if qq == q else 2)
        if ref is None:
            ref = ans.clone()
        ok = bool(torch.equal(ans, ref[:qq]))
        res[en] = {"queries": qq, "ms": round(ms, 4), "Gq_per_s": round(qq / ms / 1e6, 3),
                   "agrees_with_inlabel": ok}
    rows.append(res)
    print(json.dumps(res), flush=True)
