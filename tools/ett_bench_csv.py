"""ett-bench-style runs on the B200 path, CSV in the reference's schema.

The reference harness (tools/ett_bench.cpp:44-65, :136-167, :303-325) writes
    experiment,algo,n,m,q,gamma,dataset,batch,workers,rep,seed,phase,nanos
with phases build / query / total for LCA and the bridge engine's phases +
total for bridges.  This tool emits the same schema from the GPU path so a
user's existing analysis scripts read it unchanged (workers = GPUs used).
Extra phases: query_device (device-resident u32 queries, CUDA events) and,
for bridges, the device phase split.

  python tools/ett_bench_csv.py lca --n 1000000 --gamma inf --q 1000000 --engine inlabel --reps 3
  python tools/ett_bench_csv.py bridges --road 1000 --engine tv --reps 3 --verify
  python tools/ett_bench_csv.py bridges --graph file.gr --engine hybrid --csv out.csv
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_15217_b200 as ett  # noqa: E402

HEADER = "experiment,algo,n,m,q,gamma,dataset,batch,workers,rep,seed,phase,nanos"


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    lp = sub.add_parser("lca")
    lp.add_argument("--n", type=int, default=1_000_000)
    lp.add_argument("--gamma", default="inf")
    lp.add_argument("--q", type=int, default=1_000_000)
    lp.add_argument("--engine", default="inlabel", choices=["inlabel", "rmq", "naive"])
    lp.add_argument("--reps", type=int, default=3)
    lp.add_argument("--seed", type=int, default=3)
    lp.add_argument("--batch", type=int, default=0)
    lp.add_argument("--verify", action="store_true")
    lp.add_argument("--csv", default="-")
    bp = sub.add_parser("bridges")
    g = bp.add_mutually_exclusive_group(required=True)
    g.add_argument("--road", type=int, help="road-like W=H side")
    g.add_argument("--planted", nargs=3, type=int, metavar=("N", "M", "B"))
    g.add_argument("--graph", help="edge-list or DIMACS .gr file (parsed on the device)")
    bp.add_argument("--engine", default="tv", choices=["tv", "ck", "hybrid"])
    bp.add_argument("--reps", type=int, default=3)
    bp.add_argument("--verify", action="store_true")
    bp.add_argument("--csv", default="-")
    a = ap.parse_args()
    out = sys.stdout if a.csv == "-" else open(a.csv, "w")
    print(HEADER, file=out)

    def row(exp, algo, n, m, q, gamma, dataset, batch, rep, seed, phase, nanos):
        print(f"{exp},{algo},{n},{m},{q},{gamma},{dataset},{batch},1,{rep},{seed},{phase},"
              f"{int(nanos)}", file=out, flush=True)

    if a.cmd == "lca":
        gamma = ett.K_GRASP_INFINITY if a.gamma == "inf" else int(a.gamma)
        t = ett.permute_labels(ett.grasp_tree(a.n, gamma, 1), 2)
        queries = ett.sample_queries(t.n, a.q, a.seed)
        batch = a.batch if a.batch > 0 else max(1, a.q)
        eng = {"inlabel": ett.ENGINE_INLABEL, "rmq": ett.ENGINE_RMQ, "naive": ett.ENGINE_NAIVE}
        d = torch.empty(2 * a.q, dtype=torch.int32, device="cuda")
        ett.gen_queries_dev(t.n, a.q, a.seed, 0, d)
        dans = torch.empty(a.q, dtype=torch.int32, device="cuda")
        answers = None
        for rep in range(a.reps):
            idx = ett.inlabel_build(t, engines=eng[a.engine])
            build_ns = idx.build_ms() * 1e6
            t0 = time.perf_counter_ns()
            answers = idx.query(queries, batch, eng[a.engine])
            query_ns = time.perf_counter_ns() - t0
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            idx.query_dev(d, dans, eng[a.engine])
            e1.record()
            torch.cuda.synchronize()
            for phase, ns in (("build", build_ns), ("query", query_ns),
                              ("query_device", e0.elapsed_time(e1) * 1e6),
                              ("total", build_ns + query_ns)):
                row("lca", a.engine, t.n, 0, a.q, a.gamma, "grasp", batch, rep, a.seed, phase, ns)
        if a.verify:
            from oracle import oracle as orc
            want = orc.Ref.lca("rmq", t.parent, t.root, queries)
            bad = np.flatnonzero(answers != want)
            if len(bad):
                sys.exit(f"verification failed at query {bad[0]}")
            print(f"verified {a.q} queries against the reference rmq", file=sys.stderr)
        return

    if a.road:
        g_, truth = ett.road_like_graph(a.road, a.road, 6, 3, a.road * a.road // 49, 5)
        dataset = f"road{a.road}"
    elif a.planted:
        g_, truth = ett.planted_bridge_graph(*a.planted, 4)
        dataset = "planted"
    else:
        data = open(a.graph, "rb").read()
        raw = (ett.parse_dimacs_gr if a.graph.endswith(".gr") else ett.parse_edge_list)(data)
        comp = ett.largest_component(raw)
        g_, truth, dataset = comp.graph, None, os.path.basename(a.graph)
    fn = {"tv": ett.tv_bridges, "ck": ett.ck_bridges, "hybrid": ett.hybrid_bridges}[a.engine]
    mask = None
    for rep in range(a.reps):
        times = {}
        t0 = time.perf_counter_ns()
        mask = fn(g_, times=times).is_bridge
        total = time.perf_counter_ns() - t0
        for phase, ms in times.items():  # device phases; the wall-clock total follows
            phase = "total_device" if phase == "total" else phase
            row("bridges", a.engine, g_.n, g_.m(), 0, "", dataset, 0, rep, 0, phase, ms * 1e6)
        row("bridges", a.engine, g_.n, g_.m(), 0, "", dataset, 0, rep, 0, "total", total)
    print(f"bridge count: {int(mask.sum())}", file=sys.stderr)
    if a.verify:
        want = truth
        if want is None:
            from oracle import oracle as orc
            want = orc.Ref.bridges("dfs", g_.n, g_.edges)[0]
        if not np.array_equal(mask, want):
            sys.exit(f"verification failed at edge {int(np.flatnonzero(mask != want)[0])}")
        print("verified mask", file=sys.stderr)


if __name__ == "__main__":
    main()
