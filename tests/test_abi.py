"""CPU checks of the C-ABI boundary (no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ettg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ettg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(ett):
    L = ett.lib()
    names = _declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_no_cpu_fallback_without_device(ett):
    """Without a CUDA device every compute entry point fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cnt = ctypes.c_int(-1)
    assert ett.lib().ettg_device_count(ctypes.byref(cnt)) == 0 and cnt.value == 0
    t = ett.RootedTree(3, 0, [-1, 0, 0])
    with pytest.raises(ett._lib.CudaError):
        ett.inlabel_build(t)
    with pytest.raises(ett._lib.CudaError):
        ett.tv_bridges(ett.EdgeList(2, [[0, 1]]))


def test_argument_errors_map_to_reference_exceptions(ett):
    with pytest.raises(ett.InvalidArgument):
        ett.inlabel_build(ett.RootedTree(3, 0, [-1, 0]))  # size mismatch
    with pytest.raises(ett.InvalidArgument):
        ett.grasp_tree(0)
    with pytest.raises(ett.InvalidArgument):
        ett.random_connected_graph(5, 2, 1)
    assert issubclass(ett.InvalidArgument, ValueError)
    assert issubclass(ett.OutOfRange, IndexError)


def test_version_and_header_constants(ett):
    assert ett.lib().ettg_version() >= 100
    h = open(os.path.join(ROOT, "include", "ettg.h")).read()
    assert "#define ETTG_ENGINE_INLABEL 1u" in h and "#define ETTG_ENGINE_RMQ 2u" in h


def test_road_like_edge_count_matches_generator(ett):
    W, H, extra, r, pend = 30, 20, 6, 3, 17
    m = ett.lib().ettg_road_like_edge_count(W, H, extra, r, pend)
    g, truth = ett.road_like_graph(W, H, extra, r, pend, 1)
    assert g.m() == m and len(truth) == m
    assert np.all(g.edges[:, 0] != g.edges[:, 1])


def test_shard_range_cpu(ett):
    """ettg_shard_range (the split ettg_lca_query_multi and bench.py use):
    contiguous, covering, sizes differ by at most one; no GPU needed."""
    from paper_2103_15217_b200.dist import shard_range
    for total in (0, 1, 7, 16_000_000, 1_000_000_000, (1 << 40) + 3):
        for world in (1, 2, 3, 8):
            cuts = [shard_range(total, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == total
            assert all(cuts[i][1] == cuts[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in cuts]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ett.InvalidArgument):
        shard_range(10, 3, 3)


def test_multi_gpu_entry_points_fail_loudly_without_device(ett):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(ett.InvalidArgument):
        ett.query_multi([], np.zeros((1, 2), np.int64), 1)
