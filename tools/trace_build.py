"""LCA build phase trace on 16M trees (ETTG_TRACE=1), device-resident parent (dev aid)."""
import os, sys
os.environ["ETTG_TRACE"]="1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_2103_15217_b200 as ett
for gamma in (1, ett.K_GRASP_INFINITY):
    t = ett.permute_labels(ett.grasp_tree(16_000_000, gamma, 1), 2)
    dp = torch.from_numpy(t.parent.astype(np.int32)).cuda()
    for _ in range(3):
        idx = ett.inlabel_build_dev(dp, t.n, t.root)
    print("build_ms", gamma, idx.build_ms(), idx.layout(), flush=True)
