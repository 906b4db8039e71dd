"""Multi-GPU LCA through the C-ABI on the one GPU a test box
has: NCCL replication (ettg_lca_replicate with ncclCommInitAll, and the
per-rank ettg_lca_replicate_rank with a 1-rank communicator), and a host batch
sharded across replicas (ettg_lca_query_multi) -- answers identical to one
index and to the reference."""
import numpy as np
import pytest

from util import GRASP_INF

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tree_and_queries(ett):
    t = ett.permute_labels(ett.grasp_tree(2_000_000, GRASP_INF, 31), 32)
    q = ett.sample_queries(t.n, 5_000_001, 33)
    return t, q


def test_replicate_and_query_multi_vs_reference(ett, ref, tree_and_queries):
    t, q = tree_and_queries
    want = ref.lca("inlabel", t.parent, t.root, q)
    idx = ett.inlabel_build(t)
    reps = ett.replicate(idx, [0])
    assert len(reps) == 1 and reps[0].layout()[0] == idx.layout()[0]
    assert np.array_equal(ett.answer_batch(reps[0], q, len(q)), want)
    # two replicas on the one device: the shard split and the thread fan-out
    reps2 = ett.replicate(idx, [0, 0])
    del idx  # replicas own their memory
    for rs in (reps2, reps2 + reps):
        assert np.array_equal(ett.query_multi(rs, q, len(q)), want)
        assert np.array_equal(ett.query_multi(rs, q, 1 << 20), want)


def test_replicate_rank_single_rank(ett, tree_and_queries):
    t, q = tree_and_queries
    idx = ett.inlabel_build(t)
    want = ett.answer_batch(idx, q[:100_000], 100_000)
    uid = ett.nccl_unique_id()
    assert len(uid) == 128
    same = ett.replicate_rank(idx, t.n, 0, uid, 0, 1, 0)
    assert np.array_equal(ett.answer_batch(same, q[:100_000], 100_000), want)
    # a root without an index fails on every rank instead of hanging
    with pytest.raises(ett.InvalidArgument, match="no exportable inlabel index"):
        ett.replicate_rank(None, t.n, 0, ett.nccl_unique_id(), 0, 1, 0)


def test_query_multi_errors(ett, tree_and_queries):
    t, q = tree_and_queries
    reps = ett.replicate(ett.inlabel_build(t), [0, 0])
    with pytest.raises(ett.InvalidArgument, match="batch_size"):
        ett.query_multi(reps, q[:10], 0)
    bad = q[:300_000].copy()
    bad[290_000, 0] = t.n  # in the second replica's shard
    with pytest.raises(ett.OutOfRange):
        ett.query_multi(reps, bad, len(bad))
    assert len(ett.query_multi(reps, np.zeros((0, 2), np.int64), 1)) == 0
    with pytest.raises(ett.InvalidArgument, match="device ordinal"):
        ett.replicate(reps[0], [0, 64])
