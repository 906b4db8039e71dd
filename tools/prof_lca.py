"""LCA config B query kernel + device build (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2103_15217_b200 as ett
gamma = 1 if os.environ.get("TREE", "B") == "B" else ett.K_GRASP_INFINITY
t = ett.permute_labels(ett.grasp_tree(16_000_000, gamma, 1), 2)
dp = torch.from_numpy(t.parent.astype(np.int32)).cuda()
idx = ett.inlabel_build_dev(dp, t.n, t.root)
q = 16_000_000
d = torch.empty(2 * q, dtype=torch.int32, device="cuda"); ett.gen_queries_dev(t.n, q, 3, 0, d)
ans = torch.empty(q, dtype=torch.int32, device="cuda")
for _ in range(3):
    idx.query_dev(d, ans, 1)
torch.cuda.synchronize()
print("build_ms", idx.build_ms())
