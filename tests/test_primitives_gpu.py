"""Device primitives vs the reference: list ranking / scan, scans, stable sort,
segmented reduce and RangeIndex (core/include/ett/primitives.hpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_list_rank_golden(ett):
    # tests/primitives_test.cpp:64-97
    assert ett.list_rank([1, 2, -1], 0).tolist() == [0, 1, 2]
    assert ett.list_rank([-1, 0, 1], 2).tolist() == [2, 1, 0]
    with pytest.raises(ett.InvalidArgument):
        ett.list_rank([1, 2, 0], 0)  # cycle
    with pytest.raises(ett.InvalidArgument):
        ett.list_rank([1, -1, 1], 0)  # shared successor / uncovered


@pytest.mark.parametrize("k", [1, 2, 17, 1000, 65_537, 1_000_003, 5_000_000])
def test_list_rank_random_permutation(ett, ref, k):
    rng = np.random.default_rng(k)
    order = rng.permutation(k)
    succ = np.full(k, -1, np.int64)
    succ[order[:-1]] = order[1:]
    got = ett.list_rank(succ, int(order[0]))
    want = np.empty(k, np.int64)
    want[order] = np.arange(k)
    assert np.array_equal(got, want)
    if k <= 65_537:
        assert np.array_equal(got, ref.list_rank(succ, int(order[0])))


def test_list_rank_sequential_layout_long_sublists(ett):
    # identity order: the worst case for naive stride sampling
    k = 3_000_000
    succ = np.arange(1, k + 1, dtype=np.int64)
    succ[-1] = -1
    assert np.array_equal(ett.list_rank(succ, 0), np.arange(k))


def test_list_rank_cycle_elsewhere(ett):
    k = 200_000
    succ = np.arange(1, k + 1, dtype=np.int64)
    succ[99_999] = -1          # list 0..99999
    succ[-1] = 100_000         # cycle 100000..199999
    with pytest.raises(ett.InvalidArgument):
        ett.list_rank(succ, 0)


@pytest.mark.parametrize("n", [1, 5, 4096, 4097, 1_000_000, 10_000_019])
def test_exclusive_scan(ett, ref, n):
    rng = np.random.default_rng(n)
    v = rng.integers(0, 3, n).astype(np.int64)
    got = ett.exclusive_scan(v)
    assert np.array_equal(got, np.concatenate([[0], np.cumsum(v)[:-1]]))
    if n <= 1_000_000:
        assert np.array_equal(got, ref.exclusive_scan_sum(v))


@pytest.mark.parametrize("n,bits", [(1, 8), (1000, 3), (100_000, 17), (3_000_000, 24),
                                    (1_000_000, 32)])
def test_sort_pairs_stable(ett, n, bits):
    rng = np.random.default_rng(bits)
    keys = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo = ett.sort_pairs(keys, vals)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(ko, keys[order])
    assert np.array_equal(vo, vals[order])


PLUS_INF, MINUS_INF = (1 << 63) - 1, -(1 << 63)


def test_list_scan_golden(ett):
    # tests/primitives_test.cpp:88-97
    assert ett.list_scan([1, 2, -1], [5, 7, 9], 0).tolist() == [0, 5, 12]
    with pytest.raises(ett.InvalidArgument, match="size mismatch"):
        ett.list_scan([1, 2, -1], [5, 7], 0)
    with pytest.raises(ett.InvalidArgument):
        ett.list_scan([1, 2, 0], [1, 1, 1], 0)  # cycle
    with pytest.raises(ett.InvalidArgument, match="successor out of range"):
        ett.list_scan([1, 7, -1], [1, 1, 1], 0)


@pytest.mark.parametrize("k", [1, 2, 2047, 2048, 2049, 100_003, 3_000_000])
def test_list_scan_random(ett, ref, k):
    rng = np.random.default_rng(k + 5)
    order = rng.permutation(k)
    succ = np.full(k, -1, np.int64)
    succ[order[:-1]] = order[1:]
    vals = rng.integers(-(1 << 50), 1 << 50, k)
    got = ett.list_scan(succ, vals, int(order[0]))
    want = np.empty(k, np.int64)
    want[order] = np.concatenate([[0], np.cumsum(vals[order])[:-1]])
    assert np.array_equal(got, want)
    if k <= 100_003:
        assert np.array_equal(got, ref.list_scan(succ, int(order[0]), vals))


@pytest.mark.parametrize("n", [1, 2048, 2049, 5_000_000])
def test_exclusive_scan_i64_wraps(ett, n):
    rng = np.random.default_rng(n)
    v = rng.integers(-(1 << 62), 1 << 62, n)
    got = ett.exclusive_scan_i64(v)
    u = np.cumsum(v.view(np.uint64), dtype=np.uint64)  # wraps modulo 2^64
    want = np.concatenate([np.zeros(1, np.uint64), u[:-1]]).view(np.int64)
    assert np.array_equal(got, want)


def test_segmented_reduce_golden(ett):
    # tests/primitives_test.cpp:110-129
    assert ett.segmented_reduce([3, 1, 2], [0, 2, 3], "min", PLUS_INF).tolist() == [1, 2]
    assert ett.segmented_reduce([3, 1, 2], [0, 0, 3], "min", PLUS_INF).tolist() == [PLUS_INF, 1]
    assert ett.segmented_reduce([3, 1, 2], [0, 2, 3], "max", MINUS_INF).tolist() == [3, 2]
    assert ett.segmented_reduce([], [0], "min", PLUS_INF).tolist() == []
    for offs in ([0, 2], [], [0, 1, 4]):
        with pytest.raises(ett.InvalidArgument, match="bad offsets"):
            ett.segmented_reduce([3, 1, 2], offs, "min", PLUS_INF)
    with pytest.raises(ett.InvalidArgument, match="bad offsets"):
        ett.segmented_reduce([3, 1, 2], [0, 5, 3], "min", PLUS_INF)  # reaches past the end
    # decreasing offsets make an empty segment, as in the reference's loop
    assert ett.segmented_reduce([3, 1, 2], [2, 1, 3], "sum", 7).tolist() == [7, 10]


@pytest.mark.parametrize("segs,maxlen", [(1, 1), (1000, 5), (10_000, 100), (300, 5000),
                                         (2_000_000, 17)])
def test_segmented_reduce_random(ett, ref, segs, maxlen):
    import torch
    rng = np.random.default_rng(segs + maxlen)
    lens = rng.integers(0, maxlen + 1, segs)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    vals = rng.integers(-(1 << 62), 1 << 62, int(offs[-1]))
    small = offs[-1] <= 2_000_000
    for op, ident in (("min", PLUS_INF), ("max", MINUS_INF), ("sum", 0), ("max", 0)):
        got = ett.segmented_reduce(vals, offs, op, ident)
        dev = ett.segmented_reduce(torch.from_numpy(vals).cuda(), torch.from_numpy(offs).cuda(),
                                   op, ident).cpu().numpy()
        assert np.array_equal(got, dev)
        if small:
            assert np.array_equal(got, ref.segmented_reduce(vals, offs, op, ident))
        else:
            nz = lens > 0
            if op == "min":
                want = np.full(segs, ident, np.int64)
                want[nz] = np.minimum(np.minimum.reduceat(vals, offs[:-1][nz]), ident)
                assert np.array_equal(got, want)


def test_range_index_golden(ett):
    # tests/primitives_test.cpp:131-170
    idx = ett.RangeIndex([2, 9, 4, 1])
    assert idx.size() == 4
    assert idx.min(0, 3) == 1 and idx.max(0, 3) == 9 and idx.min(1, 1) == 9
    assert ett.rmq_min(idx, 1, 2) == 4 and ett.rmq_max(ett.rmq_build([2, 9, 4, 1]), 2, 3) == 4
    with pytest.raises(ett.OutOfRange, match="RangeIndex::min: bad range"):
        idx.min(0, 4)
    with pytest.raises(ett.OutOfRange, match="RangeIndex::max: bad range"):
        idx.max(-1, 2)
    with pytest.raises(ett.OutOfRange):
        idx.min(2, 1)
    with pytest.raises(ett.OutOfRange):
        ett.RangeIndex([]).min(0, 0)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 65_536, 1_000_003])
def test_range_index_random(ett, ref, n):
    import torch
    rng = np.random.default_rng(n)
    keys = rng.integers(-(1 << 62), 1 << 62, n)
    q = 200_000
    l = rng.integers(0, n, q)
    w = rng.integers(0, 80, q)  # many same-block and adjacent-block ranges
    r = np.where(rng.random(q) < 0.5, np.minimum(l + w, n - 1), rng.integers(0, n, q))
    rr = np.stack([np.minimum(l, r), np.maximum(l, r)], 1)
    idx = ett.RangeIndex(keys)
    mins, maxs = idx.minmax(rr)
    wm, wx = ref.range_index(keys, rr)
    assert np.array_equal(mins, wm) and np.array_equal(maxs, wx)
    assert np.array_equal(idx.mins(rr[:1000]), wm[:1000])
    didx = ett.RangeIndex(torch.from_numpy(keys).cuda())
    d_rr = torch.from_numpy(rr).cuda()
    dm = torch.empty(q, dtype=torch.int64, device="cuda")
    didx.query_dev(d_rr, dm, None)
    assert np.array_equal(dm.cpu().numpy(), wm)


def test_range_index_whole_array_and_bad_batch(ett):
    keys = np.arange(100_000, dtype=np.int64)[::-1].copy()
    idx = ett.RangeIndex(keys)
    assert idx.min(0, len(keys) - 1) == 0 and idx.max(0, len(keys) - 1) == len(keys) - 1
    with pytest.raises(ett.OutOfRange):
        idx.minmax([(0, 5), (3, 100_000)])  # one bad range fails the batch
