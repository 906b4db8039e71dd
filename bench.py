#!/usr/bin/env python
"""Benchmark: LCA queries/s (1/2/4/8 B200) and bridges edges/s with HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Headline workload (BASELINE.json configs[1], "LCA: deep path-like tree
n=16M (depth ~n), 16M queries, 1 vs 8 GPUs"): permute_labels(grasp_tree(16M,
gamma=1, seed 1), seed 2); 16M sample_queries (seed 3) split into N
contiguous shards (strong scaling).  Rank 0 builds the inlabel index on its
GPU, NCCL broadcasts the packed index, every rank answers its shard.  One
step = one batched query kernel over the rank's shard with pairs already in
HBM; L2 is flushed (256 MiB write) before every step and the flush is outside
the CUDA-event interval.

Also reported (same JSON line): config E (16M grasp(inf) tree, 1G queries
sharded), the index build time, and at N=1 the bridges config D (road-like
graph) with its own roofline and CPU baseline.  `e2e` goes through the
public C-ABI (`ettg_lca_query`) with pinned int64 host buffers.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LCA queries/s (1/2/4/8 B200) and bridges edges/s, with HBM roofline fraction"
GRASP_INF = (1 << 64) - 1
L2_FLUSH_BYTES = 256 << 20


# ------------------------------------------------------------------ helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# Random-gather ceiling of B200 at the node-table footprint of each layout at
# n = 16M (tools/footprint_micro.cu, profiles/r1_lca_layout.md): 64 MB table
# (compact) 263.8, 96 MB (split6) 150.7, 128 MB (narrow, split) 113.1, 256 MB
# (wide) 71.6 G gathers/s.
L2_GATHER_CEILING = {"compact": 263.8, "narrow": 113.1, "split": 113.1, "wide": 71.6,
                     "split_own": 71.6, "split6": 150.7, "wide9": 92.0}  # wide9: 171 MB,
# between the 128 MB (113.1) and 192 MB (83.7) points


def ncu_traffic(kernel_key: str):
    """DRAM bytes per launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get(kernel_key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def l1_tag_stage(key, queries, secs, clocks):
    """Scattered gathers are issued through the L1/TEX tag stage, which looks
    up about one 32-B sector per clock per SM (tools/tma_gather_micro.cu: 276.5
    G random 4-B loads/s = 0.95 x 148 SMs x 1.965 GHz).  Sectors per query come
    from the committed ncu capture of the same kernel and config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)[key]
        per_q = s["l1_tag_sectors_per_launch"] / s["units_per_launch"]
    except Exception:
        return None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    achieved = per_q * queries / secs / 1e9
    peak = sms * mhz / 1e3
    return {"sectors_per_query": per_q, "achieved_G_sectors_per_s": achieved,
            "peak_G_sectors_per_s": peak, "frac": achieved / peak,
            "source": "profiles/ncu_summary.json (l1tex__t_sectors ld+st per launch)"}


def l2_requests(key, queries, secs, clocks):
    """The request path from L1 to L2 accepts about one request per SM clock
    (ncu l1tex__m_l1tex2xbar_req_cycles_active); a random gather is one
    request, so requests per query -- from the committed ncu capture of the
    same kernel and config -- times the query rate is the binding unit of the
    scattered-gather query kernels."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)[key]
        per_q = s["l2_requests_per_launch"] / s["units_per_launch"]
    except Exception:
        return None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    achieved = per_q * queries / secs / 1e9
    peak = sms * mhz / 1e3
    return {"requests_per_query": per_q, "achieved_G_requests_per_s": achieved,
            "peak_G_requests_per_s": peak, "frac": achieved / peak,
            "ncu_req_active_pct": s.get("l1_to_l2_req_active_pct"),
            "source": "profiles/ncu_summary.json (lts__t_requests_srcunit_tex per launch)"}


def bridges_traffic(n, m):
    """DRAM bytes per tv_bridges call on config D from the committed ncu sweep
    (all kernels of one call), or None for another graph size."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f).get("bridges_D", {})
        return s["dram_bytes_per_call"] if (s.get("n"), s.get("m")) == (n, m) else None
    except Exception:
        return None


class ClockSampler:
    """pynvml sampling of SM clock + clock-event reasons during a region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max,
                "samples": len(self.samples),
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k]}


def all_max(x: float, device) -> float:
    if dist.is_initialized():
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def barrier():
    if dist.is_initialized():
        dist.barrier()


def lift_mean(idx, pairs_host: np.ndarray) -> float:
    """Mean label lifts per query of inlabel_lca (core/src/lca.cpp:97-105) on a
    sample, replayed vectorised over the exported index (instrumentation for
    the roofline byte model)."""
    inl = idx.inlabel.astype(np.uint64)
    asc = idx.ascendant.astype(np.uint64)
    x, y = pairs_host[:, 0], pairs_host[:, 1]
    ix, iy = inl[x], inl[y]
    diff = ix != iy
    xo = np.where(diff, ix ^ iy, np.uint64(1))
    i = np.floor(np.log2(xo.astype(np.float64))).astype(np.uint64)
    common = asc[x] & asc[y] & ~((np.uint64(1) << i) - np.uint64(1))
    common = np.where(diff, common, np.uint64(1))
    j = np.zeros(len(x), np.uint64)
    c = common.copy()
    low = c & (~c + np.uint64(1))
    j = np.floor(np.log2(low.astype(np.float64))).astype(np.uint64)
    target = (ix & ~((np.uint64(2) << j) - np.uint64(1))) | (np.uint64(1) << j)
    lifts = (diff & (ix != target)).astype(np.int64) + (diff & (iy != target)).astype(np.int64)
    return float(lifts.mean())


# ---------------------------------------------------------------- workloads
def make_tree(ett, n, gamma):
    return ett.permute_labels(ett.grasp_tree(n, gamma, 1), 2)


def device_queries(ett, n, q_total, seed, lo, hi, device):
    d = torch.empty(2 * (hi - lo), dtype=torch.int32, device=device)
    if hi > lo and not ett.gen_queries_dev(n, hi - lo, seed, lo, d, device.index):
        # a Lemire rejection broke the counter replay: use the host stream
        d.copy_(torch.from_numpy(ett.sample_queries(n, hi, seed)[lo:].astype(np.int32).ravel()))
    return d


def lca_section(ett, args, tree, q_total, device, rank, world, steps, warmup, label):
    """Build on rank 0, broadcast, shard, time K steps.  Returns a dict."""
    from paper_2103_15217_b200.dist import replicate_index, shard_range
    idx = None
    build_ms = None
    if rank == 0:
        # device-resident parent array: the build time excludes the host copy
        d_par = torch.from_numpy(tree.parent.astype(np.int32)).to(device)
        ett.inlabel_build_dev(d_par, tree.n, tree.root, device.index)  # warm arena / context
        idx = ett.inlabel_build_dev(d_par, tree.n, tree.root, device.index)
        build_ms = idx.build_ms()
        del d_par
    if world > 1:
        idx = replicate_index(idx, tree.n, device)
    lo, hi = shard_range(q_total, rank, world)
    q = hi - lo
    pairs = device_queries(ett, tree.n, q_total, 3, lo, hi, device)
    ans = torch.empty(q, dtype=torch.int32, device=device)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=device)
    stream = torch.cuda.current_stream(device)
    for _ in range(warmup):
        idx.query_dev(pairs, ans, ett.ENGINE_INLABEL, stream.cuda_stream)
    torch.cuda.synchronize(device)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device.index) as clk:
        for e0, e1 in evs:
            flush.fill_(1)  # L2 flush, outside the timed interval
            e0.record(stream)
            idx.query_dev(pairs, ans, ett.ENGINE_INLABEL, stream.cuda_stream)
            e1.record(stream)
        torch.cuda.synchronize(device)
    barrier()
    step_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    step_ms_max = all_max(step_ms, device)
    out = {"label": label, "q_total": q_total, "q_rank": q, "step_ms": step_ms_max,
           "value": q_total / (step_ms_max / 1e3), "build_ms": build_ms,
           "clocks": clk.summary(), "idx": idx, "pairs": pairs, "ans": ans, "lo": lo,
           "gpu_launches": steps}
    return out


def e2e_section(ett, idx, tree, q_total, lo, hi, device, steps):
    """Same metric through ettg_lca_query with pinned int64 host buffers."""
    host = ett.sample_queries(tree.n, hi, 3)[lo:] if hi > lo else np.zeros((0, 2), np.int64)
    pin_pairs = torch.from_numpy(np.ascontiguousarray(host)).pin_memory()
    pin_ans = torch.empty(hi - lo, dtype=torch.int64).pin_memory()
    from paper_2103_15217_b200 import _lib
    L = _lib.lib()

    def call():
        _lib.check(L.ettg_lca_query(idx.handle, pin_pairs.data_ptr(), hi - lo, max(hi - lo, 1),
                                    pin_ans.data_ptr()))
    call()
    barrier()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    barrier()
    t = all_max(float(np.mean(times)), device)
    answers = pin_ans.numpy().copy()  # the link test below reuses the pinned buffers
    # the link carries u32 pairs (narrowed by the library's host threads) in
    # and the int64 answers out: time those bytes as plain copies
    link = host_link_bound(torch.empty(2 * (hi - lo), dtype=torch.int32).pin_memory(), pin_ans,
                           device)
    # the same call with pageable numpy buffers (what a std::vector / numpy
    # caller passes): staged through the library's pinned buffers
    pg_pairs = np.ascontiguousarray(host)
    pg_ans = np.empty(hi - lo, np.int64)
    pg = []
    for _ in range(3):
        t0 = time.perf_counter()
        _lib.check(L.ettg_lca_query(idx.handle, pg_pairs.ctypes.data, hi - lo, max(hi - lo, 1),
                                    pg_ans.ctypes.data))
        pg.append(time.perf_counter() - t0)
    pg_ok = bool(np.array_equal(pg_ans, answers))
    return {"value": q_total / t, "unit": "queries/s",
            "h2d_bytes_per_step": (hi - lo) * 8, "d2h_bytes_per_step": (hi - lo) * 8,
            "caller_bytes_per_step": {"in": (hi - lo) * 16, "out": (hi - lo) * 8},
            "ms_per_step": t * 1e3, "path": "ettg_lca_query (pinned int64 host pairs/answers; "
                                            "u32 pairs cross the link, narrowed by host threads)",
            "pageable": {"value": q_total / all_max(min(pg), device), "ms": 1e3 * min(pg),
                         "answers_match_pinned": pg_ok,
                         "what": "same call, numpy (pageable) pairs and answers, best of 3"},
            "link_bound": {"ms": link, "frac": (link / (t * 1e3)) if link else None,
                           "what": "the same H2D + D2H bytes as plain concurrent copies on two "
                                   "streams (no kernel), CUDA events, best of 12; "
                                   "profiles/r1_pcie_micro.md"}}, \
        answers


def host_link_bound(pin_in, pin_out, device):
    """Duplex copy time of one step's bytes: the floor of any e2e step."""
    if pin_in.numel() == 0:
        return None
    d_in = torch.empty(pin_in.shape, dtype=pin_in.dtype, device=device)
    d_out = torch.empty(pin_out.shape, dtype=pin_out.dtype, device=device)
    s0, s1 = torch.cuda.Stream(device), torch.cuda.Stream(device)
    best = None
    for _ in range(12):
        torch.cuda.synchronize(device)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(s0)
        s1.wait_event(e0)
        with torch.cuda.stream(s0):
            d_in.copy_(pin_in, non_blocking=True)
        with torch.cuda.stream(s1):
            pin_out.copy_(d_out, non_blocking=True)
        e1.record(s1)
        s0.wait_event(e1)
        e2.record(s0)
        e2.synchronize()
        ms = e0.elapsed_time(e2)
        best = ms if best is None else min(best, ms)
    del d_in, d_out
    return best


def cpu_lca_baseline(parent, root, pairs_host, reps=3, one_worker_q=2_000_000, what=""):
    """The reference's own CPU path (oracle/_ref, compiled from the unmodified
    core/src) on this host: inlabel_build untimed, answer_batch(inlabel_lca)
    timed as tools/ett_bench.cpp:141-150 does, with every usable core (best
    of `reps`) and with one worker on a prefix of `one_worker_q` queries.
    Returns (baseline dict, reference answers over pairs_host)."""
    from oracle import oracle as orc
    if not orc.have_ref():
        return None, None
    topo = host_topology()
    cores = topo["usable_cores"]
    orc.Ref.set_workers(cores)
    h = orc.RefInlabel(parent, root)
    best = None
    answers = None
    for _ in range(reps):
        answers, ns = h.answer(pairs_host, len(pairs_host))
        best = ns if best is None else min(best, ns)
    q1 = min(one_worker_q, len(pairs_host))
    orc.Ref.set_workers(1)
    _, ns1 = h.answer(pairs_host[:q1], q1)
    orc.Ref.set_workers(cores)
    return {"value": len(pairs_host) / (best / 1e9), "unit": "queries/s", "cores": cores,
            "kind": "reference", "host": topo,
            "sample": f"answer_batch(inlabel_lca) over {len(pairs_host)} queries{what}, "
                      f"best of {reps}; inlabel_build {h.build_ns / 1e9:.2f} s untimed",
            "one_worker": {"value": q1 / (ns1 / 1e9), "cores": 1,
                           "sample": f"the first {q1} of those queries"}}, answers


def bridges_section(ett, args, device, peak):
    """Config D: road-like graph, TV bridges, edges/s, vs the planted truth."""
    W = H = args.road_side
    g, truth = ett.road_like_graph(W, H, 6, 3, args.road_pendant, 5)
    n, m = g.n, g.m()
    d_edges = torch.from_numpy(g.edges.astype(np.int32).ravel()).to(device)
    d_mask = torch.empty(m, dtype=torch.uint8, device=device)
    from paper_2103_15217_b200 import _lib
    L = _lib.lib()
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=device)

    def run():
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(d_edges.data_ptr(), n, m, device.index, d_mask.data_ptr(),
                                      stream.cuda_stream, __import__("ctypes").byref(pt)))
        return pt
    run()
    ok = bool(np.array_equal(d_mask.cpu().numpy(), truth))
    res = []
    for _ in range(args.bridge_steps):
        flush.fill_(1)
        torch.cuda.synchronize(device)
        res.append(run())
    tot = float(np.mean([p.total_ms for p in res]))
    bytes_model = 41 * m + 108 * n
    out = {"config": {"workload": f"bridges-road-like W=H={W} r=3 extra=6 pendant={args.road_pendant}",
                      "n": n, "m": m, "bridges": int(truth.sum())},
           "metric": "bridges edges/s", "value": m / (tot / 1e3), "unit": "edges/s",
           "ms_per_step": tot, "steps": args.bridge_steps,
           "phases_ms": {"spanning": float(np.mean([p.spanning_ms for p in res])),
                         "euler": float(np.mean([p.euler_ms for p in res])),
                         "lowhigh": float(np.mean([p.lowhigh_ms for p in res]))},
           "parity": "bit-exact vs planted truth" if ok else "MISMATCH",
           "roofline": {"bound": "hbm", "achieved": bytes_model / (tot / 1e3) / 1e9,
                        "peak": peak[0], "unit": "GB/s",
                        "frac": bytes_model / (tot / 1e3) / 1e9 / peak[0],
                        "traffic": bridges_traffic(n, m), "peak_kind": peak[1],
                        "model": "41*m + 108*n bytes per call (SURVEY.md 8(d))",
                        "traffic_note": "DRAM bytes of every kernel of one call (ncu, cold, "
                                        "profiles/ncu_summary.json bridges_D)",
                        "io_floor_frac": 9 * m / (tot / 1e3) / 1e9 / peak[0]}}
    # e2e: the reference-facing call (tv_bridges on an int64 host edge list,
    # core/src/bridges.cpp:311) through ettg_bridges with pinned host buffers;
    # the H2D of the 16-B pairs is inside the timed region
    import ctypes
    import time
    pin_e = torch.from_numpy(np.ascontiguousarray(g.edges, dtype=np.int64)).pin_memory()
    pin_m = torch.empty(m, dtype=torch.uint8).pin_memory()

    def call_host():
        _lib.check(L.ettg_bridges(pin_e.data_ptr(), n, m, device.index, pin_m.data_ptr(), None))
    call_host()
    ok_h = bool(np.array_equal(pin_m.numpy(), truth))
    ts = []
    for _ in range(args.bridge_steps):
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        call_host()
        ts.append(time.perf_counter() - t0)
    # floor: the narrowed edge list's H2D then the bit mask's D2H (the mask
    # needs every edge), as plain copies
    d_e = torch.empty(2 * m, dtype=torch.int32, device=device)
    src_e = torch.empty(2 * m, dtype=torch.int32).pin_memory()
    d_m = torch.empty((m + 7) // 8, dtype=torch.uint8, device=device)
    spare = torch.empty((m + 7) // 8, dtype=torch.uint8).pin_memory()
    copies = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d_e.copy_(src_e, non_blocking=True)
        spare.copy_(d_m, non_blocking=True)
        e1.record()
        e1.synchronize()
        copies.append(e0.elapsed_time(e1))
    del d_e, d_m, spare, src_e
    out["e2e"] = {"value": m / min(ts), "unit": "edges/s", "ms_per_step": 1e3 * min(ts),
                  "ms_median": 1e3 * float(np.median(ts)),
                  "h2d_bytes_per_step": m * 8, "d2h_bytes_per_step": (m + 7) // 8,
                  "caller_bytes_per_step": {"in": m * 16, "out": m},
                  "path": "ettg_bridges (pinned int64 host edge list -> host mask; u32 edges "
                          "cross the link, the mask comes back as bits)",
                  "parity": "bit-exact vs planted truth" if ok_h else "MISMATCH",
                  "link_bound": {"ms": min(copies), "frac": min(copies) / (1e3 * min(ts)),
                                 "what": "H2D of the u32 edge list then D2H of the bit mask "
                                         "as plain copies (no kernel), CUDA events, best of 3"}}
    del pin_e, pin_m
    if args.cpu_baseline:
        from oracle import oracle as orc
        if orc.have_ref():
            topo = host_topology()
            cores = topo["usable_cores"]
            orc.Ref.set_workers(cores)
            t0 = time.perf_counter()
            mask, ph = orc.Ref.bridges("tv", n, g.edges)
            wall = time.perf_counter() - t0
            out["cpu_baseline"] = {
                "value": m / (ph[3] / 1e9), "unit": "edges/s", "cores": cores,
                "kind": "reference", "host": topo, "ms": ph[3] / 1e6,
                "sample": f"the whole config D graph (n={n}, m={m}): tv_bridges(adj, &phases) "
                          f"timed, build_adjacency untimed (tools/ett_bench.cpp:310-317); "
                          f"phases ns spanning/euler/lowhigh {ph[:3].tolist()}; "
                          f"{wall:.0f} s wall with build_adjacency",
                "parity_vs_ours": bool(np.array_equal(mask, d_mask.cpu().numpy())),
                "parity_vs_truth": bool(np.array_equal(mask, truth)),
                "one_worker": {"value": None, "cores": 1,
                               "note": "not run on config D: one worker needs ~15 min "
                                       "(8 workers take 109 s, SURVEY.md 6); see "
                                       "bridges_config_C.cpu_baseline.one_worker"}}
    return out


def lca_engines_config_a(ett, device):
    """The paper's engine comparison (Figs. 3-6) on config A: inlabel
    vs RMQ-on-tour vs naive walk-up, one Euler-tour build, device-resident
    queries, L2 flushed before each timed launch; answers must agree."""
    t = make_tree(ett, 1_000_000, GRASP_INF)
    q = 1_000_000
    idx = ett.inlabel_build(t, device=device.index,
                            engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ | ett.ENGINE_NAIVE)
    pairs = torch.empty(2 * q, dtype=torch.int32, device=device)
    ett.gen_queries_dev(t.n, q, 3, 0, pairs, device.index)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=device)
    st = torch.cuda.current_stream(device)
    out, ref_ans = {"workload": "config A: permute_labels(grasp_tree(1M, inf)), 1M queries",
                    "unit": "queries/s"}, None
    for eng, name in [(ett.ENGINE_INLABEL, "inlabel"), (ett.ENGINE_RMQ, "rmq"),
                      (ett.ENGINE_NAIVE, "naive")]:
        ans = torch.empty(q, dtype=torch.int32, device=device)
        idx.query_dev(pairs, ans, eng, st.cuda_stream)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(20)]
        torch.cuda.synchronize(device)
        for e0, e1 in evs:
            flush.fill_(1)
            e0.record(st)
            idx.query_dev(pairs, ans, eng, st.cuda_stream)
            e1.record(st)
        torch.cuda.synchronize(device)
        ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
        if ref_ans is None:
            ref_ans = ans.clone()
        out[name] = {"value": q / (ms / 1e3), "ms": ms,
                     "agrees_with_inlabel": bool(torch.equal(ans, ref_ans))}
    out["inlabel_layout"] = idx.layout()[0]
    from oracle import oracle as orc
    if orc.have_ref():
        pairs_host = pairs.cpu().numpy().astype(np.int64).reshape(-1, 2)
        cb, want = cpu_lca_baseline(t.parent, t.root, pairs_host, reps=5,
                                    one_worker_q=q, what=" (the whole config)")
        cb["parity_vs_ours"] = bool(np.array_equal(want, ref_ans.cpu().numpy()))
        out["cpu_baseline"] = cb
    return out


def ingestion_config_c(ett, args):
    """parse_edge_list of config C written as text
    (write_edge_list, 8M lines, ~110 MB), end to end from host bytes to host
    edges through ettg_parse_edge_list, vs the reference parser on a bounded
    prefix (it is sequential: ~1.3 us per line)."""
    import time
    g, _ = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
    text = ett.write_edge_list(g)
    lines = text.count(b"\n")
    got = ett.parse_edge_list(text)  # warm-up (arena, module load)
    ok = bool(got.n == g.n and np.array_equal(got.edges, np.sort(g.edges, axis=1)))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ett.parse_edge_list(text)
        ts.append(time.perf_counter() - t0)
    out = {"workload": "parse_edge_list(write_edge_list(config C)): 8M lines, "
                       f"{len(text) / 1e6:.0f} MB, host bytes -> host int64 edges",
           "value": lines / min(ts), "unit": "lines/s", "ms": 1e3 * min(ts),
           "bytes_per_s": len(text) / min(ts),
           "parity": "identical to write_edge_list input (normalised)" if ok else "MISMATCH"}
    if args.cpu_baseline:
        try:
            from oracle import oracle as orc
            if orc.have_ref():
                cut = 0
                for _ in range(2_000_000):
                    cut = text.index(b"\n", cut) + 1
                sample = text[:cut]
                t0 = time.perf_counter()
                want = orc.ref_parse("edges", sample)
                dt = time.perf_counter() - t0
                mine = ett.parse_edge_list(sample)
                out["cpu_baseline"] = {
                    "value": 2_000_000 / dt, "unit": "lines/s", "cores": 1, "kind": "reference",
                    "sample": "reference parse_edge_list (sequential) on the first 2M lines",
                    "parity_vs_ours": bool(want[0] == mine.n and np.array_equal(want[1],
                                                                                mine.edges))}
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"error": str(e)[:200]}
    return out


def bridges_config_c(ett, args, device, peak):
    """Config C: planted_bridge_graph(1M, 8M, b=10,000, seed 4); the reference's
    tv_bridges runs the full workload on the host for an exact comparison."""
    g, truth = ett.planted_bridge_graph(1_000_000, 8_000_000, 10_000, 4)
    n, m = g.n, g.m()
    d_edges = torch.from_numpy(g.edges.astype(np.int32).ravel()).to(device)
    d_mask = torch.empty(m, dtype=torch.uint8, device=device)
    from paper_2103_15217_b200 import _lib
    import ctypes
    L = _lib.lib()
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=device)

    def run():
        pt = _lib.PhaseTimes()
        _lib.check(L.ettg_bridges_dev(d_edges.data_ptr(), n, m, device.index, d_mask.data_ptr(),
                                      stream.cuda_stream, ctypes.byref(pt)))
        return pt
    run()
    ok = bool(np.array_equal(d_mask.cpu().numpy(), truth))
    res = []
    for _ in range(args.bridge_steps):
        flush.fill_(1)
        torch.cuda.synchronize(device)
        res.append(run())
    tot = float(np.mean([p.total_ms for p in res]))
    out = {"workload": "bridges config C: planted_bridge_graph(1M, 8M, b=10000, seed 4)",
           "value": m / (tot / 1e3), "unit": "edges/s", "ms_per_step": tot,
           "parity": "bit-exact vs planted truth" if ok else "MISMATCH",
           "roofline_frac_41m108n": (41 * m + 108 * n) / (tot / 1e3) / 1e9 / peak[0]}
    # the paper's engine comparison on the same graph
    engines = {}
    for eng, name in [(0, "tv"), (2, "hybrid"), (1, "ck")]:
        def run_e():
            pt = _lib.PhaseTimes()
            _lib.check(L.ettg_bridges_dev_engine(d_edges.data_ptr(), n, m, device.index, eng,
                                                 d_mask.data_ptr(), stream.cuda_stream,
                                                 ctypes.byref(pt)))
            return pt
        run_e()
        ok_e = bool(np.array_equal(d_mask.cpu().numpy(), truth))
        ts = []
        for _ in range(2):
            flush.fill_(1)
            torch.cuda.synchronize(device)
            ts.append(run_e().total_ms)
        engines[name] = {"ms": float(np.mean(ts)), "value": m / (np.mean(ts) / 1e3),
                         "parity": "bit-exact vs planted truth" if ok_e else "MISMATCH"}
    out["engines"] = engines
    if args.cpu_baseline:
        from oracle import oracle as orc
        if orc.have_ref():
            cores = host_topology()["usable_cores"]
            orc.Ref.set_workers(cores)
            mask, ph = orc.Ref.bridges("tv", n, g.edges)
            orc.Ref.set_workers(1)
            _, ph1 = orc.Ref.bridges("tv", n, g.edges)
            orc.Ref.set_workers(cores)
            out["cpu_baseline"] = {
                "value": m / (ph[3] / 1e9), "unit": "edges/s", "cores": cores,
                "kind": "reference", "host": host_topology(),
                "sample": "full config C, tv_bridges, build_adjacency "
                          "untimed (tools/ett_bench.cpp:310-317)",
                "ms": ph[3] / 1e6, "parity_vs_truth": bool(np.array_equal(mask, truth)),
                "parity_vs_ours": bool(np.array_equal(mask, d_mask.cpu().numpy())),
                "one_worker": {"value": m / (ph1[3] / 1e9), "cores": 1, "ms": ph1[3] / 1e6,
                               "sample": "the same call with ETT_WORKERS=1"}}
    return out


def config_e_block(ett, args, tree, sec, device, peak, world):
    """Config E (BASELINE.json configs[4], the north-star 16M-tree scaling
    config) as a first-class block: throughput, roofline, parity of 16 windows
    spread over the query stream against the reference's answer_batch, e2e on
    a bounded prefix through the C-ABI, and the reference CPU baseline."""
    idx = sec["idx"]
    layout = idx.layout()[0]
    q_r = sec["q_rank"]
    secs = sec["step_ms"] / 1e3
    sample = ett.sample_queries(tree.n, min(args.e_sample, args.scaling_q), 3)
    Lbar = lift_mean(idx, sample[:2_000_000])
    Bq = 12 + 32 * (2 + Lbar)
    kname = {"split": "k_lca_inlabel_split", "split6": "k_lca_inlabel_split6",
             "wide": "k_lca_inlabel", "wide9": "k_lca_inlabel"}.get(layout, layout)
    out = {"workload": "LCA config E: permute_labels(grasp_tree(16M, inf)), 1G sample_queries "
                       "(counter mode, seed 3) sharded across GPUs",
           "n": tree.n, "queries": args.scaling_q, "value": sec["value"], "unit": "queries/s",
           "ms_per_step": sec["step_ms"], "steps": args.scaling_steps, "n_gpus": world,
           "scaling": "strong", "build_ms": sec["build_ms"], "index_layout": layout,
           "clocks": sec["clocks"],
           "roofline": {"bound": "hbm", "achieved": Bq * q_r / secs / 1e9, "peak": peak[0],
                        "unit": "GB/s", "frac": Bq * q_r / secs / 1e9 / peak[0],
                        "traffic": ncu_traffic(f"{kname}_E"), "kernel": kname,
                        "bytes_per_query": Bq, "lifts_per_query": Lbar,
                        "model": "12 + 32 * (2 + lifts) B per query (SURVEY.md 8(d))",
                        "note": "the model charges every gather a DRAM sector; the split6 "
                                "node table (96 MB) is mostly L2-resident",
                        "l2_gather": {"node_gathers_G_per_s": 2 * q_r / secs / 1e9,
                                      "ceiling_G_per_s": L2_GATHER_CEILING.get(layout),
                                      "frac": (2 * q_r / secs / 1e9 / L2_GATHER_CEILING[layout]
                                               if layout in L2_GATHER_CEILING else None)},
                        "l1_tag_stage": l1_tag_stage(f"{kname}_E", q_r, secs, sec["clocks"]),
                        "l1_l2_requests": l2_requests(f"{kname}_E", q_r, secs, sec["clocks"])}}
    # parity: 16 windows of 1M queries spread across this rank's shard of the
    # stream, answered by the timed kernel, against the reference answer_batch
    from oracle import oracle as orc
    rh = None
    if orc.have_ref():
        orc.Ref.set_workers(host_topology()["usable_cores"])
        rh = orc.RefInlabel(tree.parent, tree.root)
        win, ok, checked = 1_000_000, True, 0
        for w in range(16):
            a = (q_r - win) * w // 15 if q_r > win else 0
            b = min(a + win, q_r)
            pairs = sec["pairs"][2 * a:2 * b].cpu().numpy().astype(np.int64).reshape(-1, 2)
            got = sec["ans"][a:b].cpu().numpy().astype(np.int64)
            want, _ = rh.answer(pairs)
            ok &= bool(np.array_equal(got, want))
            checked += b - a
        out["parity_vs_reference"] = ok
        out["parity_sample"] = (f"{checked} queries in 16 windows of {win} spread over stream "
                                f"positions [{sec['lo']}, {sec['lo'] + q_r}) vs the reference "
                                f"answer_batch(inlabel_lca)")
    # e2e on a bounded prefix through the C-ABI with pinned host buffers
    if world == 1:
        qe = len(sample)
        e2e, e2e_ans = e2e_section(ett, idx, tree, qe, 0, qe, device, args.e2e_steps)
        e2e["sample"] = f"the first {qe} queries of the stream"
        out["e2e"] = e2e
        if rh is not None:
            del e2e_ans
            cb, _ = cpu_lca_baseline(tree.parent, tree.root, sample, reps=2,
                                     what=" (a prefix of the 1G-query stream)")
            out["cpu_baseline"] = cb
    return out


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=16_000_000)
    ap.add_argument("--q", type=int, default=16_000_000)
    ap.add_argument("--scaling-q", type=int, default=1_000_000_000)
    ap.add_argument("--scaling-steps", type=int, default=5)
    ap.add_argument("--e-sample", type=int, default=64_000_000)
    ap.add_argument("--no-scaling", action="store_true")
    ap.add_argument("--no-bridges", action="store_true")
    ap.add_argument("--road-side", type=int, default=5657)
    ap.add_argument("--road-pendant", type=int, default=20_761)
    ap.add_argument("--bridge-steps", type=int, default=5)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--dist-backend", default="nccl")
    ap.add_argument("--same-device", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, rank, world)

    # --same-device maps every rank to cuda:0 (validation of the N>1 path on
    # a 1-GPU box; NCCL refuses duplicate devices, so it pairs with gloo).
    local = 0 if args.same_device else local
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(args.dist_backend)
    import paper_2103_15217_b200 as ett
    peak = peaks()

    # ---- headline: config B -------------------------------------------------
    tree = make_tree(ett, args.n, 1)
    sec = lca_section(ett, args, tree, args.q, device, rank, world, args.steps, args.warmup,
                      "B")
    idx = sec["idx"]
    e2e, e2e_ans = e2e_section(ett, idx, tree, args.q, sec["lo"], sec["lo"] + sec["q_rank"],
                               device, args.e2e_steps)
    dev_ans = sec["ans"].cpu().numpy().astype(np.int64)
    consistent = bool(np.array_equal(dev_ans, e2e_ans))
    consistent = all_max(0.0 if consistent else 1.0, device) == 0.0

    line = None
    if rank == 0:
        pairs_host = ett.sample_queries(tree.n, args.q, 3)
        Lbar = lift_mean(idx, pairs_host[: min(len(pairs_host), 2_000_000)])
        Bq_survey = 12 + 32 * (2 + Lbar)  # one 32-B sector per gather
        layout, labels = idx.layout()
        kname = {"wide": "k_lca_inlabel", "narrow": "k_lca_inlabel_narrow",
                 "compact": "k_lca_inlabel_compact_pipe", "split": "k_lca_inlabel_split",
                 "split_own": "k_lca_inlabel_split_own",
                 "split6": "k_lca_inlabel_split6", "wide9": "k_lca_inlabel"}[layout]
        q_r = sec["q_rank"]
        if layout == "compact":
            # 12 B streamed + the index read once per launch (node words + label
            # table); the 4-B node table is L2-resident after its first touch
            Bq = 12 + (4 * tree.n + 16 * labels) / q_r
            model = "12 B streamed + (4 n + 16 labels) B index read once, per query"
        else:
            Bq = Bq_survey
            model = "12 + 32 * (2 + lifts) B per query (SURVEY.md 8(d))"
        secs = sec["step_ms"] / 1e3
        achieved = Bq * q_r / secs / 1e9
        traffic = ncu_traffic(f"{kname}_B")
        node_gathers = 2 * q_r / secs / 1e9
        line = {
            "metric": METRIC, "value": sec["value"], "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec["step_ms"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (reference generators, seeds tree=1 permute=2 "
                                    "queries=3)",
            "config": lca_config_b(tree.n, args.q),
            "run": {"index_layout": layout, "inlabel_paths": labels,
                    "parallelism": f"index replicated, queries sharded x{world}",
                    "l2": f"flushed (256 MiB write) before every step; index "
                          f"{idx.index_bytes() / 1e6:.0f} MB"},
            "e2e": e2e,
            "gpu_launches": sec["gpu_launches"],
            "build_ms": sec["build_ms"],
            "clocks": sec["clocks"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak[0], "unit": "GB/s",
                         "frac": achieved / peak[0], "traffic": traffic,
                         "peak_kind": peak[1], "kernel": kname, "bytes_per_query": Bq,
                         "model": model,
                         "survey_model": {"bytes_per_query": Bq_survey, "lifts_per_query": Lbar,
                                          "achieved": Bq_survey * q_r / secs / 1e9,
                                          "frac": Bq_survey * q_r / secs / 1e9 / peak[0]},
                         "l1_tag_stage": l1_tag_stage(f"{kname}_B", q_r, secs,
                                                      sec["clocks"]),
                         "l1_l2_requests": l2_requests(f"{kname}_B", q_r, secs, sec["clocks"]),
                         "l2_gather": {"node_gathers_G_per_s": node_gathers,
                                       "ceiling_G_per_s": L2_GATHER_CEILING.get(layout),
                                       "frac": (node_gathers / L2_GATHER_CEILING[layout]
                                                if layout in L2_GATHER_CEILING else None),
                                       "source": "profiles/r1_lca_layout.md footprint sweep"}},
            "answers_consistent_dev_vs_e2e": consistent,
        }
        if args.cpu_baseline and world == 1:
            cb, ref_ans = cpu_lca_baseline(tree.parent, tree.root, pairs_host,
                                           what=" (the whole config)")
            if cb is not None:
                cb["parity_vs_ours"] = bool(np.array_equal(ref_ans, dev_ans))
                line["cpu_baseline"] = cb
    del sec, idx

    # ---- config E: 16M grasp(inf), 1G queries sharded -------------------------
    if not args.no_scaling:
        treeE = make_tree(ett, args.n, GRASP_INF)
        secE = lca_section(ett, args, treeE, args.scaling_q, device, rank, world,
                           args.scaling_steps, 2, "E")
        if rank == 0:
            line["scaling_config_E"] = config_e_block(ett, args, treeE, secE, device, peak, world)
        del secE

    # ---- bridges config D (replicas only: rank 0 of an N=1 run) -------------
    if not args.no_bridges and rank == 0 and world == 1:
        torch.cuda.empty_cache()
        line["bridges"] = bridges_section(ett, args, device, peak)
        line["bridges_config_C"] = bridges_config_c(ett, args, device, peak)
        line["ingestion_config_C"] = ingestion_config_c(ett, args)
        line["lca_engines_config_A"] = lca_engines_config_a(ett, device)

    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def lca_config_b(n, q):
    """The config object both arms print (identical, so the driver can pair
    them): BASELINE.json configs[1]."""
    return {"workload": "LCA config B: permute_labels(grasp_tree(16M, gamma=1)) path tree, "
                        "16M sample_queries",
            "n": n, "queries": q, "engine": "inlabel", "seeds": {"tree": 1, "permute": 2,
                                                                 "queries": 3}}


def host_topology():
    """lscpu-style sockets x cores x threads of this host, plus the cores this
    process may run on (what the CPU baselines use)."""
    topo = {"usable_cores": len(os.sched_getaffinity(0))}
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = dict(line.split(":", 1) for line in out.splitlines() if ":" in line)
        kv = {k.strip(): v.strip() for k, v in kv.items()}
        topo.update({"model": kv.get("Model name"), "sockets": int(kv.get("Socket(s)", 0)),
                     "cores_per_socket": int(kv.get("Core(s) per socket", 0)),
                     "threads_per_core": int(kv.get("Thread(s) per core", 0)),
                     "cpus": int(kv.get("CPU(s)", 0))})
    except Exception:
        pass
    return topo


def reference_arm(args, rank, world):
    """The reference's own CPU implementation on the same workload, metric,
    unit and config as our arm.  Everything here is the unmodified reference
    (oracle/_ref = core/src compiled from its own sources): the generators
    grasp_tree / permute_labels / sample_queries (core/src/generators.cpp:21-91),
    inlabel_build untimed, and each step one answer_batch(inlabel_lca) over
    all q queries (tools/ett_bench.cpp:136-150), with every host core.
    Rank 0 only; the other ranks exit without work."""
    if rank != 0:
        return
    from oracle import oracle as orc
    if not orc.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    topo = host_topology()
    cores = topo["usable_cores"]
    orc.Ref.set_workers(cores)
    par0 = orc.Ref.grasp_tree(args.n, 1, 1)
    parent, root = orc.Ref.permute_labels(par0, 0, 2)
    del par0
    pairs = orc.Ref.sample_queries(args.n, args.q, 3)
    h = orc.RefInlabel(parent, root)
    for _ in range(args.warmup):
        h.answer(pairs)
    step_ns = []
    for _ in range(args.steps):
        _, ns = h.answer(pairs)
        step_ns.append(ns)
    ms = float(np.mean(step_ns)) / 1e6
    v = args.q / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "i64",
            "data": "synthetic (reference generators, seeds tree=1 permute=2 queries=3)",
            "config": lca_config_b(args.n, args.q),
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores,
                             "kind": "reference", "host": topo,
                             "sample": f"each step: answer_batch(inlabel_lca) over all {args.q} "
                                       f"queries (batch = q); inlabel_build "
                                       f"{h.build_ns / 1e9:.2f} s untimed"},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
