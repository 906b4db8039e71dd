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
    """Contiguous slice [lo, hi) of `total` units owned by `rank`."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


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

    The blob size travels first (one int64 broadcast), then the blob itself.
    """
    rank = dist.get_rank()
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
