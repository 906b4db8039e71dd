"""Device primitives vs the reference: list ranking, scan, stable sort."""
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
