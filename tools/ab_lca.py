"""A/B of the inlabel query kernel variants (index layouts (wide / narrow / auto)), development aid.

Usage: python tools/ab_lca.py [modes...]   (each mode runs in its own process)
Times config B (16M path tree, 16M queries, L2 flushed before each launch)
and a 16M random tree with 64M queries, CUDA events on the launching stream.
"""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def child():
    sys.path.insert(0, ROOT)
    import torch, paper_2103_15217_b200 as ett
    from paper_2103_15217_b200 import _lib
    if os.environ.get("AB_LIB"):
        _lib.LIB_PATH = os.environ["AB_LIB"]
    out = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, gamma, q in [("B_path", 1, 16_000_000), ("E_rand", ett.K_GRASP_INFINITY, 64_000_000),
                           ("g2", 2, 16_000_000), ("g8", 8, 16_000_000), ("A_1M", ett.K_GRASP_INFINITY, 1_000_000),
                           ("path_1M", 1, 1_000_000), ("g2_1M", 2, 1_000_000), ("rand_4M", ett.K_GRASP_INFINITY, 4_000_000),
                           ("path_4M", 1, 4_000_000), ("g16", 16, 16_000_000), ("g64", 64, 16_000_000),
                           ("g4", 4, 16_000_000)]:
        if os.environ.get("AB_ONLY") and name not in os.environ["AB_ONLY"].split(","):
            continue
        n = {"A_1M": 1_000_000, "path_1M": 1_000_000, "g2_1M": 1_000_000, "rand_4M": 4_000_000,
             "path_4M": 4_000_000}.get(name, 16_000_000)
        t = ett.permute_labels(ett.grasp_tree(n, gamma, 1), 2)
        flags = {"wide": ett.LAYOUT_WIDE, "narrow": ett.LAYOUT_NARROW, "compact": ett.LAYOUT_COMPACT, "split": ett.LAYOUT_SPLIT, "split_own": ett.LAYOUT_SPLIT_OWN, "split6": ett.LAYOUT_SPLIT6, "wide9": ett.LAYOUT_WIDE9}.get(os.environ.get("AB_MODE"), 0)
        try:
            idx = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | flags)
        except ett.InvalidArgument as e:
            out[name] = str(e)
            continue
        d = torch.empty(2 * q, dtype=torch.int32, device="cuda")
        ett.gen_queries_dev(t.n, q, 3, 0, d)
        ans = torch.empty(q, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream()
        for _ in range(3): idx.query_dev(d, ans, 1, st.cuda_stream)
        K = 50
        evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(K)]
        torch.cuda.synchronize()
        for e0, e1 in evs:  # queued back to back: no host launch gap inside e0..e1
            flush.fill_(1)
            e0.record(st); idx.query_dev(d, ans, 1, st.cuda_stream); e1.record(st)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs) / K
        h = int(torch.sum(ans.to(torch.int64)).item())
        out[name] = {"layout": idx.layout()[0], "ms": round(ms, 4), "Gq/s": round(q / ms / 1e6, 2), "anshash": h}
    print(json.dumps(out))

if __name__ == "__main__":
    if os.environ.get("AB_CHILD"):
        child(); sys.exit(0)
    for mode in (sys.argv[1:] or ["wide", "split", "narrow", "compact", "auto"]):
        env = dict(os.environ, AB_CHILD="1", AB_MODE=mode.split(":")[0])
        if ":" in mode:
            env["ETTG_QGRID"] = mode.split(":")[1]
        if mode == "old":
            env["AB_LIB"] = os.path.join(ROOT, "tools", "_old", "libettg_head.so")
        r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
        print(f"mode {mode}: {r.stdout.strip()} {r.stderr.strip()[-300:]}", flush=True)
