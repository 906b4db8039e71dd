"""N>1 path on CPU with gloo (world size 2): index broadcast + batch sharding.

The GPU ranks run exactly this code with NCCL; here the 'index' is the
oracle's packed inlabel index (bytes) and each rank answers its shard with
the CPU oracle, so the test checks the plumbing, not the kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _BlobIndex:
    """Stand-in for InlabelIndex on rank 0: exports a packed byte blob."""

    def __init__(self, blob: np.ndarray):
        self.blob = blob

    def index_bytes(self):
        return self.blob.nbytes

    def export_index(self, dst: torch.Tensor):
        dst.copy_(torch.from_numpy(self.blob))


def _pack(index):
    inl, asc, head, lev, par = index
    n = len(inl)
    return np.concatenate([a.astype(np.int64).view(np.uint8) for a in
                           (np.array([n]), inl, asc.view(np.int64), head, lev, par)])


def _unpack(blob: np.ndarray):
    a = blob.view(np.int64)
    n = int(a[0])
    o = 1
    inl = a[o:o + n]; o += n
    asc = a[o:o + n].view(np.uint64); o += n
    head = a[o:o + n + 1]; o += n + 1
    lev = a[o:o + n]; o += n
    par = a[o:o + n]
    return inl, asc, head, lev, par


def _worker(rank, world, port, q_total, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2103_15217_b200 as ett
    from paper_2103_15217_b200.dist import replicate_index, shard_range
    from oracle.oracle import Port

    t = ett.permute_labels(ett.grasp_tree(5000, ett.K_GRASP_INFINITY, 1), 2)
    queries = ett.sample_queries(t.n, q_total, 3)
    src = _BlobIndex(_pack(Port.inlabel_index(t.parent, t.root))) if rank == 0 else None
    got = replicate_index(src, t.n, torch.device("cpu"),
                          attach=lambda blob, n: _unpack(blob.numpy().copy()))
    index = _unpack(src.blob) if rank == 0 else got
    lo, hi = shard_range(q_total, rank, world)
    ans, _ = Port.inlabel_query(index, queries[lo:hi])
    np.save(os.path.join(out_dir, f"ans{rank}.npy"), ans)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_exactly():
    from paper_2103_15217_b200.dist import shard_range
    for total in (0, 1, 7, 1000, 10**9 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_two_rank_gloo_broadcast_and_shard(tmp_path):
    world, q_total = 2, 10_001
    mp.spawn(_worker, args=(world, _free_port(), q_total, str(tmp_path)), nprocs=world,
             join=True)
    import paper_2103_15217_b200 as ett
    from oracle.oracle import Port
    t = ett.permute_labels(ett.grasp_tree(5000, ett.K_GRASP_INFINITY, 1), 2)
    q = ett.sample_queries(t.n, q_total, 3)
    full = Port.lca_inlabel(t.parent, t.root, q)
    parts = np.concatenate([np.load(tmp_path / f"ans{r}.npy") for r in range(world)])
    assert np.array_equal(parts, full)
