"""Ad-hoc timing of the LCA build and query kernels (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett

def run(n, gamma, q, label):
    t0 = time.time()
    t = ett.permute_labels(ett.grasp_tree(n, gamma, 1), 2)
    gen = time.time() - t0
    idx = ett.inlabel_build(t, engines=3)
    idx2 = ett.inlabel_build(t, engines=3)
    bms = idx2.build_ms()
    d = torch.empty(2 * q, dtype=torch.int32, device="cuda")
    ett.gen_queries_dev(n, q, 3, 0, d)
    ans = torch.empty(q, dtype=torch.int32, device="cuda")
    res = {}
    for eng, name in [(1, "inlabel"), (2, "rmq")]:
        for _ in range(3): idx.query_dev(d, ans, eng)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): idx.query_dev(d, ans, eng)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[name] = (ms, q / ms / 1e6)
    print(f"{label}: n={n} gen={gen:.1f}s build={bms:.2f}ms  " +
          "  ".join(f"{k}: {v[0]:.3f}ms {v[1]:.2f} Gq/s" for k, v in res.items()), flush=True)

run(1_000_000, ett.K_GRASP_INFINITY, 1_000_000, "A")
run(16_000_000, 1, 16_000_000, "B")
run(16_000_000, ett.K_GRASP_INFINITY, 100_000_000, "E-ish")
