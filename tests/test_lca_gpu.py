"""LCA parity on the B200: CUDA path (through the C-ABI) vs the CPU oracle.

Bit-exact on everything: answers, and (because the GPU reproduces the DCEL
child order) every intermediate the reference exposes -- node_stats and the
InlabelIndex fields.
"""
import numpy as np
import pytest

from util import GRASP_INF, lca_corpus

pytestmark = pytest.mark.gpu

EXAMPLE = np.array([-1, 2, 0, 0, 0, 2], np.int64)  # tests/lca_test.cpp:47-57


def test_golden_example_tree(ett):
    t = ett.RootedTree(6, 0, EXAMPLE)
    idx = ett.inlabel_build(t)
    st = idx.stats()
    # tests/euler_test.cpp:130-139
    assert st.preorder.tolist() == [1, 3, 2, 5, 6, 4]
    assert st.level.tolist() == [0, 2, 1, 1, 1, 2]
    assert st.size[2] == 3 and st.size[0] == 6
    assert st.parent.tolist() == [-1, 2, 0, 0, 0, 2]
    # tests/lca_test.cpp:47-74
    assert idx.inlabel.tolist() == [4, 3, 4, 5, 6, 4]
    assert idx.head[4] == 0
    assert ett.inlabel_lca(idx, 1, 5) == 2
    assert ett.inlabel_lca(idx, 3, 4) == 0
    for v in range(6):
        assert ett.inlabel_lca(idx, v, v) == v
        assert ett.inlabel_lca(idx, 0, v) == 0
        assert ett.inlabel_lca(idx, v, 0) == 0
    r = ett.rmq_lca_build(t)
    assert ett.rmq_lca(r, 1, 5) == 2
    assert ett.rmq_lca(r, 3, 3) == 3


def test_single_node(ett):
    idx = ett.inlabel_build(ett.RootedTree(1, 0, [-1]))
    assert idx.inlabel.tolist() == [1]
    assert idx.ascendant.tolist() == [1]
    assert ett.inlabel_lca(idx, 0, 0) == 0
    st = idx.stats()
    assert st.preorder.tolist() == [1] and st.size.tolist() == [1] and st.level.tolist() == [0]


def test_corpus_bit_exact_vs_reference(ett, ref):
    """acceptance criterion 2 + intermediate parity on 200 corpus trees."""
    pairs_total = 0
    for ti, t in enumerate(lca_corpus(ett)):
        idx = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ)
        pre, size, lev, par = ref.node_stats(t.parent, t.root)
        st = idx.stats()
        assert np.array_equal(st.preorder, pre), ti
        assert np.array_equal(st.size, size), ti
        assert np.array_equal(st.level, lev), ti
        assert np.array_equal(st.parent, par), ti
        inl, asc, head, lev2, par2 = ref.inlabel_index(t.parent, t.root)
        assert np.array_equal(idx.inlabel, inl), ti
        assert np.array_equal(idx.ascendant, asc), ti
        assert np.array_equal(idx.head, head), ti
        if t.n <= 128:
            xs, ys = np.meshgrid(np.arange(t.n), np.arange(t.n), indexing="ij")
            q = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.int64)
        else:
            q = ett.sample_queries(t.n, 10_000, t.n)
        want = ref.lca("inlabel", t.parent, t.root, q)
        assert np.array_equal(idx.query(q, len(q), ett.ENGINE_INLABEL), want), ti
        assert np.array_equal(idx.query(q, len(q), ett.ENGINE_RMQ), want), ti
        pairs_total += len(q)
    assert pairs_total > 1_000_000


@pytest.mark.parametrize("gamma", [1, 2, 64, GRASP_INF])
def test_medium_trees_vs_reference(ett, ref, gamma):
    t = ett.permute_labels(ett.grasp_tree(200_003, gamma, 11), 12)
    q = ett.sample_queries(t.n, 100_000, 13)
    idx = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ)
    want = ref.lca("rmq", t.parent, t.root, q)
    assert np.array_equal(ett.answer_batch(idx, q, 4096), want)
    assert np.array_equal(idx.query(q, len(q), ett.ENGINE_RMQ), want)
    pre, size, lev, par = ref.node_stats(t.parent, t.root)
    st = idx.stats()
    assert np.array_equal(st.preorder, pre) and np.array_equal(st.size, size)
    assert np.array_equal(st.level, lev) and np.array_equal(st.parent, par)


def test_config_a_full_size(ett, ref):
    """BASELINE config A at full size: 1M-node grasp(inf) tree, 1M queries."""
    t = ett.permute_labels(ett.grasp_tree(1_000_000, GRASP_INF, 1), 2)
    q = ett.sample_queries(t.n, 1_000_000, 3)
    idx = ett.inlabel_build(t)
    got = ett.answer_batch(idx, q, 1_000_000)
    want = ref.lca("inlabel", t.parent, t.root, q)
    assert np.array_equal(got, want)
    inl, asc, head, lev, par = ref.inlabel_index(t.parent, t.root)
    assert np.array_equal(idx.inlabel, inl) and np.array_equal(idx.ascendant, asc)


def test_barabasi_and_star(ett, ref):
    for t in [ett.permute_labels(ett.barabasi_tree(300_000, 31), 32),
              ett.RootedTree(100_000, 7, np.where(np.arange(100_000) == 7, -1, 7))]:
        q = ett.sample_queries(t.n, 50_000, 5)
        idx = ett.inlabel_build(t, engines=3)
        want = ref.lca("inlabel", t.parent, t.root, q)
        assert np.array_equal(idx.query(q, len(q), 1), want)
        assert np.array_equal(idx.query(q, len(q), 2), want)
        inl, asc, head, lev, par = ref.inlabel_index(t.parent, t.root)
        assert np.array_equal(idx.inlabel, inl)


def test_batch_size_invariance_and_errors(ett):
    t = ett.permute_labels(ett.grasp_tree(300, GRASP_INF, 8), 9)
    idx = ett.inlabel_build(t)
    q = ett.sample_queries(t.n, 500, 17)
    base = ett.answer_batch(idx, q, 1)
    for b in (7, 500, 10_000):
        assert np.array_equal(base, ett.answer_batch(idx, q, b))
    with pytest.raises(ett.InvalidArgument):
        ett.answer_batch(idx, q, 0)
    with pytest.raises(ett.OutOfRange):
        ett.answer_batch(idx, np.array([[0, 300]]), 1)
    assert len(ett.answer_batch(idx, np.zeros((0, 2), np.int64), 1)) == 0


@pytest.mark.parametrize("parent,root,msg", [
    ([-1, 0, 5], 0, "out of range"),        # parent id out of range
    ([-1, -1, 0], 0, "exactly one root"),   # two roots
    ([1, -1, 0], 0, "kNone"),               # root has a parent
    ([-1, 2, 1], 0, "cycle"),               # 1 <-> 2 cycle off the root
    ([-1, 1, 0, 3], 0, "cycle"),            # self loop
])
def test_invalid_trees(ett, parent, root, msg):
    with pytest.raises(ett.InvalidArgument, match=msg):
        ett.inlabel_build(ett.RootedTree(len(parent), root, np.array(parent)))


def test_large_cycle_detected(ett):
    n = 100_000
    par = np.arange(-1, n - 1, dtype=np.int64)  # path 0 <- 1 <- 2 ...
    par[50_000] = 99_999                        # detach the tail into a cycle
    with pytest.raises(ett.InvalidArgument, match="cycle"):
        ett.inlabel_build(ett.RootedTree(n, 0, par))


def test_deep_path_2m(ett, ref):
    """Config B shape (path, depth n-1) at 2M nodes vs the reference."""
    t = ett.permute_labels(ett.grasp_tree(2_000_000, 1, 1), 2)
    q = ett.sample_queries(t.n, 500_000, 3)
    idx = ett.inlabel_build(t)
    want = ref.lca("inlabel", t.parent, t.root, q)
    assert np.array_equal(ett.answer_batch(idx, q, len(q)), want)


def test_replica_attach_matches(ett):
    import torch
    t = ett.permute_labels(ett.grasp_tree(100_000, GRASP_INF, 4), 5)
    q = ett.sample_queries(t.n, 50_000, 6)
    idx = ett.inlabel_build(t)
    buf = torch.empty(idx.index_bytes(), dtype=torch.uint8, device="cuda:0")
    idx.export_index(buf)
    torch.cuda.synchronize()
    rep = ett.attach_index(buf, t.n)
    assert np.array_equal(ett.answer_batch(rep, q, len(q)), ett.answer_batch(idx, q, len(q)))


def test_device_query_and_counter_mode_generator(ett, ref):
    import torch
    t = ett.permute_labels(ett.grasp_tree(1 << 20, GRASP_INF, 1), 2)
    idx = ett.inlabel_build(t)
    q = 300_001
    d = torch.empty(2 * q, dtype=torch.int32, device="cuda:0")
    assert ett.gen_queries_dev(t.n, q, 3, 0, d)
    host = ett.sample_queries(t.n, q, 3)
    assert np.array_equal(d.cpu().numpy().astype(np.int64).reshape(-1, 2), host)
    ans = torch.empty(q, dtype=torch.int32, device="cuda:0")
    idx.query_dev(d, ans, ett.ENGINE_INLABEL)
    want = ref.lca("inlabel", t.parent, t.root, host)
    assert np.array_equal(ans.cpu().numpy().astype(np.int64), want)
    # an offset window replays the same stream
    d2 = torch.empty(2 * 1000, dtype=torch.int32, device="cuda:0")
    assert ett.gen_queries_dev(t.n, 1000, 3, 5000, d2)
    assert np.array_equal(d2.cpu().numpy().astype(np.int64).reshape(-1, 2), host[5000:6000])


# ------------------------------------------------------------- naive engine
def test_naive_golden(ett):
    # tests/lca_test.cpp:76-90
    t = ett.RootedTree(6, 0, EXAMPLE)
    idx = ett.naive_build(t)
    assert ett.naive_lca(idx, 1, 5) == 2
    assert ett.naive_lca(idx, 4, 4) == 4
    k = 64
    path = ett.RootedTree(k, 0, np.arange(-1, k - 1))
    assert ett.naive_lca(ett.naive_build(path), 0, k - 1) == 0


def test_three_engines_agree_on_corpus(ett, ref):
    """acceptance criterion 2: inlabel == naive == rmq == walk-up oracle."""
    for ti, t in enumerate(lca_corpus(ett, count=60, seed=2024)):
        q = ett.sample_queries(t.n, 2000, ti + 1)
        want = ref.lca("naive", t.parent, t.root, q)
        nv = ett.naive_build(t)
        assert np.array_equal(ett.answer_batch(nv, q, 500), want), ti
        mixed = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ | ett.ENGINE_NAIVE)
        for eng in (ett.ENGINE_INLABEL, ett.ENGINE_RMQ, ett.ENGINE_NAIVE):
            assert np.array_equal(mixed.query(q, len(q), eng), want), (ti, eng)


@pytest.mark.parametrize("gamma", [1, 7, GRASP_INF])
def test_ancestor_doubling_levels(ett, ref, gamma):
    t = ett.permute_labels(ett.grasp_tree(300_007, gamma, 3), 4)
    lev = ett.ancestor_doubling_levels(t)
    _, _, want, _ = ref.node_stats(t.parent, t.root)
    assert np.array_equal(lev, want)


def test_depth_law(ett):
    """acceptance criterion 5 (tests/acceptance.cpp:221-257): mean grasp depth."""
    n = 1_000_000
    for gamma, target in [(GRASP_INF, np.log(n)), (100, n / 101), (1000, n / 1001)]:
        means = [ett.ancestor_doubling_levels(ett.grasp_tree(n, gamma, s)).mean() for s in range(5)]
        assert abs(np.mean(means) - target) / target < 0.15, gamma


def test_naive_errors(ett):
    with pytest.raises(ett.InvalidArgument, match="cycle"):
        ett.naive_build(ett.RootedTree(3, 0, np.array([-1, 2, 1])))
    with pytest.raises(ett.InvalidArgument, match="out of range"):
        ett.naive_build(ett.RootedTree(3, 0, np.array([-1, 0, 9])))
    idx = ett.naive_build(ett.RootedTree(3, 0, np.array([-1, 0, 0])))
    with pytest.raises(ett.InvalidArgument):
        idx.query(np.array([[0, 1]]), 1, ett.ENGINE_INLABEL)  # engine not built
    with pytest.raises(ett.InvalidArgument):
        idx.stats()


# ------------------------------------------------------- index layouts
LAYOUTS = [("wide", "LAYOUT_WIDE"), ("narrow", "LAYOUT_NARROW"), ("compact", "LAYOUT_COMPACT"),
           ("split", "LAYOUT_SPLIT"), ("split_own", "LAYOUT_SPLIT_OWN"), ("split6", "LAYOUT_SPLIT6"),
           ("wide9", "LAYOUT_WIDE9")]


def _compact_bits(ref, t):
    """Label-index bits + in-path offset bits of the compact layout (oracle side)."""
    inl, asc, head, lev, par = ref.inlabel_index(t.parent, t.root)
    labels = len(np.unique(inl))
    hl = lev[head[inl]]  # level of the head of each node's path
    maxoff = int((lev - hl).max())
    return (int(labels - 1).bit_length() if labels > 1 else 0) + maxoff.bit_length()


def _build_layout(ett, ref, t, name, flag):
    try:
        return ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | getattr(ett, flag))
    except ett.InvalidArgument as e:
        assert name == "compact" and "exceed 32 bits" in str(e)
        assert _compact_bits(ref, t) > 32
        return None


@pytest.mark.parametrize("name,flag", LAYOUTS)
def test_forced_layout_corpus_vs_reference(ett, ref, name, flag):
    """Both inlabel layouts answer the 200-tree corpus like the reference."""
    for ti, t in enumerate(lca_corpus(ett)):
        idx = _build_layout(ett, ref, t, name, flag)
        assert idx.layout()[0] == name
        q = ett.sample_queries(t.n, 4_000, t.n + 7)
        want = ref.lca("inlabel", t.parent, t.root, q)
        assert np.array_equal(ett.answer_batch(idx, q, len(q)), want), ti


@pytest.mark.parametrize("name,flag", LAYOUTS)
@pytest.mark.parametrize("gamma", [1, 2, GRASP_INF])
def test_forced_layout_medium_trees(ett, ref, name, flag, gamma):
    t = ett.permute_labels(ett.grasp_tree(300_007, gamma, 21), 22)
    q = ett.sample_queries(t.n, 200_000, 23)
    idx = _build_layout(ett, ref, t, name, flag)
    if idx is None:
        return
    assert idx.layout()[0] == name
    want = ref.lca("inlabel", t.parent, t.root, q)
    assert np.array_equal(ett.answer_batch(idx, q, len(q)), want)
    assert idx.layout()[1] == len(np.unique(ref.inlabel_index(t.parent, t.root)[0]))


def test_auto_layout_choice_and_replicas(ett):
    """Auto picks compact for a long path (few labels), split for a random tree,
    wide9 in between (6M nodes: the 16-B table would exceed half of L2);
    forced layouts and replicas of each answer identically on the device."""
    import torch
    for gamma, expect in [(1, "compact"), (GRASP_INF, "split"), (2, "wide9")]:
        t = ett.permute_labels(ett.grasp_tree(6_000_000, gamma, 1), 2)
        idx = ett.inlabel_build(t)
        lay, labels = idx.layout()
        assert lay == expect, (gamma, lay, labels)
        q = 2_000_000
        d = torch.empty(2 * q, dtype=torch.int32, device="cuda:0")
        assert ett.gen_queries_dev(t.n, q, 3, 0, d)
        outs = []
        handles = [idx]
        for _, flag in LAYOUTS:
            try:
                handles.append(ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | getattr(ett, flag)))
            except ett.InvalidArgument as e:  # compact bit budget exceeded (gamma=2)
                assert flag == "LAYOUT_COMPACT" and gamma == 2, e
        for h in handles:
            buf = torch.empty(h.index_bytes(), dtype=torch.uint8, device="cuda:0")
            h.export_index(buf)
            rep = ett.attach_index(buf, t.n)
            assert rep.layout()[0] == h.layout()[0]
            for x in (h, rep):
                a = torch.empty(q, dtype=torch.int32, device="cuda:0")
                x.query_dev(d, a, ett.ENGINE_INLABEL)
                outs.append(a)
        for a in outs[1:]:
            assert torch.equal(a, outs[0])


def test_layout_flag_errors(ett):
    t = ett.RootedTree(len(EXAMPLE), 0, EXAMPLE.copy())
    with pytest.raises(ett.InvalidArgument, match="conflicting layout"):
        ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.LAYOUT_WIDE | ett.LAYOUT_NARROW)
    with pytest.raises(ett.InvalidArgument, match="conflicting layout"):
        ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.LAYOUT_COMPACT | ett.LAYOUT_NARROW)
    import torch
    idx = ett.inlabel_build(t)
    buf = torch.zeros(idx.index_bytes(), dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ett.InvalidArgument, match="not an exported"):
        ett.attach_index(buf, t.n)


# --------------------------------------------- device generators (8(f) row 4)
@pytest.mark.parametrize("n", [1, 2, 3, 1000, 1_000_003])
@pytest.mark.parametrize("gamma", [1, 2, 7, GRASP_INF])
def test_device_grasp_and_permute_match_host(ett, n, gamma):
    import torch
    d = torch.empty(n, dtype=torch.int32, device="cuda:0")
    assert ett.grasp_tree_dev(n, gamma, 11, d)
    t = ett.grasp_tree(n, gamma, 11)
    assert np.array_equal(d.cpu().numpy().view(np.uint32).astype(np.int64),
                          np.where(t.parent < 0, 0xFFFFFFFF, t.parent))
    out = torch.empty(n, dtype=torch.int32, device="cuda:0")
    root, ok = ett.permute_labels_dev(d, n, 0, 12, out)
    assert ok
    pt = ett.permute_labels(t, 12)
    assert root == pt.root
    assert np.array_equal(out.cpu().numpy().view(np.uint32).astype(np.int64),
                          np.where(pt.parent < 0, 0xFFFFFFFF, pt.parent))


def test_device_permute_large_matches_reference(ett, ref):
    """Config B's tree built entirely on the device equals the reference's."""
    import torch
    n = 4_000_000
    d = torch.empty(n, dtype=torch.int32, device="cuda:0")
    assert ett.grasp_tree_dev(n, 1, 1, d)
    out = torch.empty(n, dtype=torch.int32, device="cuda:0")
    root, ok = ett.permute_labels_dev(d, n, 0, 2, out)
    assert ok
    want, want_root = ref.permute_labels(ref.grasp_tree(n, 1, 1), 0, 2)
    got = out.cpu().numpy().view(np.uint32).astype(np.int64)
    assert root == want_root
    assert np.array_equal(np.where(got == 0xFFFFFFFF, -1, got), want)


def _shapes(ett, rng, n):
    """Parent arrays of varied shapes (all rooted at 0 before permutation)."""
    kind = int(rng.integers(0, 6))
    if kind == 0:
        return ett.grasp_tree(n, int(rng.integers(1, 9)), int(rng.integers(1 << 30)))
    if kind == 1:
        return ett.grasp_tree(n, GRASP_INF, int(rng.integers(1 << 30)))
    if kind == 2:
        return ett.barabasi_tree(n, int(rng.integers(1 << 30)))
    par = np.full(n, -1, np.int64)
    if kind == 3:  # star
        par[1:] = 0
    elif kind == 4:  # caterpillar: a spine with one leaf per spine node
        for v in range(1, n):
            par[v] = v - 2 if (v % 2 == 0 and v >= 2) else max(v - 1, 0) if v % 2 else 0
    else:  # complete binary tree
        par[1:] = (np.arange(1, n) - 1) // 2
    return ett.RootedTree(n, 0, par)


@pytest.mark.parametrize("name,flag", LAYOUTS + [("auto", None)])
def test_layouts_random_shapes_vs_reference(ett, ref, name, flag):
    """Every layout on 120 small trees of mixed shapes (n from 1 to 5000),
    including tiny n and single-label / single-path trees."""
    rng = np.random.default_rng(0x6c61796f + len(name))
    for it in range(120):
        n = int(rng.choice([1, 2, 3, 4, 5, 31, 32, 33, 64])) if it < 30 else int(rng.integers(6, 5000))
        t = _shapes(ett, rng, n)
        t = ett.permute_labels(t, it + 1)
        if flag is None:
            idx = ett.inlabel_build(t)
        else:
            idx = _build_layout(ett, ref, t, name, flag)
            if idx is None:
                continue
        q = ett.sample_queries(t.n, 3000, it + 2)
        want = ref.lca("inlabel", t.parent, t.root, q)
        assert np.array_equal(ett.answer_batch(idx, q, len(q)), want), (it, n, idx.layout())


def test_large_random_tree_picks_split6_and_replicates(ett):
    """16M random tree: the 8-B split table would exceed half of L2, so auto
    picks the 6-B records; a replica (export/attach) answers identically, and
    the forced layout refuses n >= 2^24 (24-bit inlabels)."""
    import torch
    n = 16_000_000
    t = ett.permute_labels(ett.grasp_tree(n, GRASP_INF, 1), 2)
    idx = ett.inlabel_build(t)
    assert idx.layout()[0] == "split6"
    q = ett.sample_queries(n, 200_000, 3)
    want = ett.answer_batch(ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.LAYOUT_WIDE),
                            q, len(q))
    assert np.array_equal(ett.answer_batch(idx, q, len(q)), want)  # wide: pinned on the corpus
    buf = torch.empty(idx.index_bytes(), dtype=torch.uint8, device="cuda:0")
    idx.export_index(buf)
    rep = ett.attach_index(buf, n)
    assert rep.layout()[0] == "split6"
    assert np.array_equal(ett.answer_batch(rep, q, len(q)), want)
    big = 1 << 24
    path = np.arange(-1, big - 1, dtype=np.int64)
    with pytest.raises(ett.InvalidArgument, match="split6"):
        ett.inlabel_build(ett.RootedTree(big, 0, path), engines=ett.ENGINE_INLABEL | ett.LAYOUT_SPLIT6)


def test_star_picks_split_own_and_matches(ett, ref):
    """A star's queries lift to the endpoints' own labels: the build-time sample
    picks split_own; answers equal the reference and every forced layout."""
    import torch
    n = 1_500_000
    par = np.zeros(n, np.int64)
    par[0] = -1
    t = ett.permute_labels(ett.RootedTree(n, 0, par), 9)
    idx = ett.inlabel_build(t)
    assert idx.layout()[0] == "split_own"
    q = ett.sample_queries(n, 100_000, 10)
    want = ref.lca("inlabel", t.parent, t.root, q)
    assert np.array_equal(ett.answer_batch(idx, q, len(q)), want)
    buf = torch.empty(idx.index_bytes(), dtype=torch.uint8, device="cuda:0")
    idx.export_index(buf)
    rep = ett.attach_index(buf, n)
    assert rep.layout()[0] == "split_own"
    assert np.array_equal(ett.answer_batch(rep, q, len(q)), want)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_query_narrowed_paths(ett, ref, pinned):
    """ettg_lca_query ships u32 pairs / answers (12 B per query) whatever the
    caller's buffers are; answers equal the reference on a multi-chunk batch,
    every engine; out-of-range ids in a late chunk (>= n, negative, >= 2^32)
    give OutOfRange, and the handle answers correctly afterwards."""
    import torch
    t = ett.permute_labels(ett.grasp_tree(500_000, 16, 21), 22)
    idx = ett.inlabel_build(t, engines=ett.ENGINE_INLABEL | ett.ENGINE_RMQ | ett.ENGINE_NAIVE)
    q = ett.sample_queries(t.n, 3_000_000, 23)  # > 2 stage chunks of 1.4M
    want = ref.lca("inlabel", t.parent, t.root, q)
    qt = torch.from_numpy(q)
    if pinned:
        qt = qt.pin_memory()
    for eng in (ett.ENGINE_INLABEL, ett.ENGINE_RMQ, ett.ENGINE_NAIVE):
        out = torch.empty(len(q), dtype=torch.int64)
        if pinned:
            out = out.pin_memory()
        from paper_2103_15217_b200 import _lib
        _lib.check(_lib.lib().ettg_lca_query_engine(idx.handle, eng, qt.data_ptr(), len(q),
                                                   len(q), out.data_ptr()))
        assert np.array_equal(out.numpy(), want), eng
    for badval in (t.n, -1, 1 << 32, -(1 << 40)):
        bad = qt.clone()
        bad[2_900_000, 1] = badval
        with pytest.raises(ett.OutOfRange):
            ett.answer_batch(idx, bad.numpy(), len(q))
    assert np.array_equal(ett.answer_batch(idx, q, len(q)), want)


def test_query_dev_error_flag_and_argument_checks(ett):
    import torch
    t = ett.permute_labels(ett.grasp_tree(10_000, GRASP_INF, 3), 4)
    idx = ett.inlabel_build(t)
    q = ett.sample_queries(t.n, 1000, 5)
    d = torch.from_numpy(q.astype(np.int32).ravel()).cuda()
    a = torch.empty(1000, dtype=torch.int32, device="cuda")
    idx.query_dev(d, a, ett.ENGINE_INLABEL)
    assert not idx.query_dev_error()
    assert np.array_equal(a.cpu().numpy(), ett.answer_batch(idx, q, 1000))
    d[7] = t.n  # y of query 3
    idx.query_dev(d, a, ett.ENGINE_INLABEL)
    assert idx.query_dev_error()
    assert a[3].item() == -1  # 0xFFFFFFFF
    assert not idx.query_dev_error()  # cleared by the read
    with pytest.raises(ett.InvalidArgument):
        idx.query_dev(d[:-2], a, ett.ENGINE_INLABEL)
    with pytest.raises(ett.InvalidArgument):
        idx.query_dev(d.to(torch.int64), a, ett.ENGINE_INLABEL)
    st = idx.stats()
    assert np.array_equal(idx.ascendant, ett.inlabel_build(t).ascendant)  # strided export
    assert len(st.preorder) == t.n


def test_host_answers_unaligned_and_odd(ett, ref):
    """ettg_lca_query into caller buffers whose start is not 32-B aligned and
    whose length is odd: the host widening's scalar head / tail around its
    streaming stores (csrc/hostcopy.cpp), for pageable and pinned answers."""
    import ctypes
    import torch
    from paper_2103_15217_b200 import _lib
    t = ett.permute_labels(ett.grasp_tree(300_000, GRASP_INF, 9), 10)
    idx = ett.inlabel_build(t)
    want = None
    for q, off in ((1_000_003, 1), (999_999, 3), (5, 1), (70_001, 2)):
        qs = np.ascontiguousarray(ett.sample_queries(t.n, q, 11))
        want = ref.lca("inlabel", t.parent, t.root, qs)
        buf = np.full(q + 8, -7, np.int64)  # 8-B aligned, start moved by `off` elements
        _lib.check(_lib.lib().ettg_lca_query(idx.handle, qs.ctypes.data, q, q,
                                             buf[off:].ctypes.data))
        assert np.array_equal(buf[off:off + q], want), (q, off)
        assert (buf[:off] == -7).all() and (buf[off + q:] == -7).all()
        pin = torch.full((q + 8,), -7, dtype=torch.int64).pin_memory()
        pq = torch.from_numpy(qs).pin_memory()
        _lib.check(_lib.lib().ettg_lca_query(idx.handle, pq.data_ptr(), q, q,
                                             pin.data_ptr() + 8 * off))
        got = pin.numpy()
        assert np.array_equal(got[off:off + q], want), (q, off, "pinned")
        assert (got[:off] == -7).all() and (got[off + q:] == -7).all()


def test_host_mask_unaligned(ett):
    """tv_bridges into a host mask that starts one byte past an aligned address
    (the bit expansion's unaligned-store path) and has an odd length."""
    import torch
    from paper_2103_15217_b200 import _lib
    g, truth = ett.planted_bridge_graph(200_003, 1_200_007, 301, 8)
    e = np.ascontiguousarray(g.edges, dtype=np.int64)
    m = len(e)
    for pinned in (False, True):
        buf = (torch.full((m + 64,), 7, dtype=torch.uint8).pin_memory().numpy() if pinned
               else np.full(m + 64, 7, np.uint8))
        _lib.check(_lib.lib().ettg_bridges(e.ctypes.data, g.n, m, 0, buf[1:].ctypes.data, None))
        assert np.array_equal(buf[1:1 + m], truth), pinned
        assert buf[0] == 7 and (buf[1 + m:] == 7).all()
