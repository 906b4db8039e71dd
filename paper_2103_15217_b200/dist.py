"""Multi-GPU plumbing for the LCA query path.

LCA query batches shard naturally: the packed inlabel index (16-B node
records + 8-B label records, ``ettg_lca_index_export_dev``) is built once
on rank 0, broadcast over NCCL (NVLink 5 / NVSwitch) and attached on every
rank; each rank answers a contiguous 1/G slice of the batch.  There is no
per-query collective.  Bridges run as replicas only (one GPU per graph).

Everything here is backend-agnostic so the same code is exercised with
``gloo`` on CPU in tests/test_dist_cpu.py.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of `total` units owned by `rank`
    (ettg_shard_range, the split ettg_lca_query_multi uses)."""
    from .ett import shard_range as _c_shard_range
    return _c_shard_range(total, rank, world)


def broadcast_blob(blob: torch.Tensor | None, nbytes: int, device: torch.device,
                   src: int = 0) -> torch.Tensor:
    """Broadcast a uint8 blob from `src`; other ranks allocate `nbytes` on `device`."""
    if dist.get_rank() != src:
        blob = torch.empty(nbytes, dtype=torch.uint8, device=device)
    assert blob is not None and blob.numel() == nbytes
    dist.broadcast(blob, src=src)
    return blob


def replicate_index(index, n: int, device: torch.device,
                    attach: Callable[[torch.Tensor, int], object] | None = None):
    """Rank 0 passes its built InlabelIndex; every rank returns a usable index.

    Under the NCCL backend the broadcast is the library's own
    (ettg_lca_replicate_rank: ncclCommInitRank + ncclBroadcast of the packed
    index, inside libettg.so); torch.distributed only carries the 128-byte
    NCCL id.  Other backends (gloo, the CPU tests) broadcast the exported blob
    with torch.distributed: the blob size first, then the blob.
    """
    rank = dist.get_rank()
    if attach is None and device.type == "cuda" and dist.get_backend() == "nccl":
        from .ett import nccl_unique_id, replicate_rank
        box = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return replicate_rank(index if rank == 0 else None, n, 0, box[0], rank,
                              dist.get_world_size(), device.index or 0)
    size = torch.tensor([index.index_bytes() if rank == 0 else 0], dtype=torch.int64,
                        device=device)
    dist.broadcast(size, src=0)
    nbytes = int(size.item())
    blob = None
    if rank == 0:
        blob = torch.empty(nbytes, dtype=torch.uint8, device=device)
        index.export_index(blob)
        if device.type == "cuda":
            torch.cuda.synchronize(device)
    blob = broadcast_blob(blob, nbytes, device)
    if rank == 0:
        return index
    if attach is None:
        from .ett import attach_index

        if device.type == "cuda":
            torch.cuda.synchronize(device)
        return attach_index(blob, n, device.index or 0)
    return attach(blob, n)
