"""Full-size parity: BASELINE.json configs B, D and E on the B200 against the
compiled reference (oracle/_ref), not against the repo itself.

- Config E (16M grasp(inf) tree, the north-star scaling tree): the whole
  InlabelIndex (inlabel, ascendant, head) equals the reference's
  inlabel_build (core/src/lca.cpp:20-82); a 4M-query prefix and 16 windows
  spread over the 1G counter-mode query stream equal the reference's
  answer_batch(inlabel_lca) (core/include/ett/lca.hpp:50-65), through both the
  device-resident u32 path (split6 layout) and the host int64 path.
- Config B (16M path tree, 16M queries): every answer of the device-resident
  query_dev path equals the reference.
- Config D (road-like, n = 32.02M, m = 256,000,000): the bridge mask equals
  the reference's tv_bridges (core/src/bridges.cpp:311-316) and the planted
  truth.

The reference inputs come from the reference's own generators
(core/src/generators.cpp:21-91) and are checked equal to ours first.
"""
import numpy as np
import pytest
import torch

from util import GRASP_INF

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N16 = 16_000_000


def _ref_tree(ref, n, gamma):
    p0 = ref.grasp_tree(n, gamma, 1)
    return ref.permute_labels(p0, 0, 2)


def _dev_pairs(ett, n, q, offset):
    d = torch.empty(2 * q, dtype=torch.int32, device="cuda:0")
    assert ett.gen_queries_dev(n, q, 3, offset, d, 0), "Lemire rejection in the window"
    return d


def _query_dev(idx, d_pairs):
    q = d_pairs.numel() // 2
    ans = torch.empty(q, dtype=torch.int32, device="cuda:0")
    idx.query_dev(d_pairs, ans, 1)
    torch.cuda.synchronize()
    return ans.cpu().numpy().astype(np.int64)


def test_config_E_index_and_query_stream_vs_reference(ett, orc):
    ref = orc.Ref
    if not orc.have_ref():
        pytest.skip("oracle/_ref not built")
    t = ett.permute_labels(ett.grasp_tree(N16, GRASP_INF, 1), 2)
    par_ref, root_ref = _ref_tree(ref, N16, GRASP_INF)
    assert root_ref == t.root and np.array_equal(par_ref, t.parent)

    idx = ett.inlabel_build(t)
    assert idx.layout()[0] == "split6"
    inl, asc, head, _, _ = ref.inlabel_index(par_ref, root_ref)
    assert np.array_equal(idx.inlabel, inl)
    assert np.array_equal(idx.ascendant, asc)
    assert np.array_equal(idx.head, head)
    del inl, asc, head

    rh = orc.RefInlabel(par_ref, root_ref)
    # 4M-query prefix: device generator == reference sample_queries, and the
    # device (u32) and host (int64) query paths == reference answer_batch
    q = 4_000_000
    host_pairs = ref.sample_queries(N16, q, 3)
    d = _dev_pairs(ett, N16, q, 0)
    assert np.array_equal(d.cpu().numpy().astype(np.int64).reshape(-1, 2), host_pairs)
    want, _ = rh.answer(host_pairs)
    assert np.array_equal(_query_dev(idx, d), want)
    assert np.array_equal(ett.answer_batch(idx, host_pairs, q), want)
    assert np.array_equal(ett.answer_batch(idx, host_pairs, 1 << 20), want)  # batched
    # 16 windows of 256K spread across the 1G-query stream (offsets up to
    # 0.94e9): device answers == reference answers on the same pairs
    for w in range(16):
        off = w * (1_000_000_000 // 16) + 12_345 * w
        d = _dev_pairs(ett, N16, 262_144, off)
        pairs = d.cpu().numpy().astype(np.int64).reshape(-1, 2)
        want, _ = rh.answer(pairs)
        assert np.array_equal(_query_dev(idx, d), want), w


def test_config_B_full_query_dev_vs_reference(ett, orc):
    ref = orc.Ref
    if not orc.have_ref():
        pytest.skip("oracle/_ref not built")
    par_ref, root_ref = _ref_tree(ref, N16, 1)
    t = ett.permute_labels(ett.grasp_tree(N16, 1, 1), 2)
    assert root_ref == t.root and np.array_equal(par_ref, t.parent)
    idx = ett.inlabel_build(t)
    assert idx.layout()[0] == "compact"
    host_pairs = ref.sample_queries(N16, N16, 3)
    d = _dev_pairs(ett, N16, N16, 0)
    assert np.array_equal(d.cpu().numpy().astype(np.int64).reshape(-1, 2), host_pairs)
    rh = orc.RefInlabel(par_ref, root_ref)
    want, _ = rh.answer(host_pairs)
    assert np.array_equal(_query_dev(idx, d), want)
    assert np.array_equal(ett.answer_batch(idx, host_pairs, N16), want)


def test_config_D_full_vs_reference_tv_bridges(ett, orc):
    ref = orc.Ref
    if not orc.have_ref():
        pytest.skip("oracle/_ref not built")
    g, truth = ett.road_like_graph(5657, 5657, 6, 3, 20_761, 5)
    assert g.m() == 256_000_000 and g.n == 32_022_410
    mask = ett.tv_bridges(g).is_bridge
    assert np.array_equal(mask, truth)
    want, _ = ref.bridges("tv", g.n, g.edges)
    assert np.array_equal(mask, want)
