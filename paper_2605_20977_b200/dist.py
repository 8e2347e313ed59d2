"""Multi-GPU plumbing for the GOP-replica decode (BASELINE config 4).

GOPs are independent: the temporal ring resets at every GOP boundary
(SPEC.md:597, :615). So a batch of GOPs shards across ranks with no data-path
collective. One process per GPU, one device handle per process;
torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only for
barriers and for the max-over-ranks timing reduction.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK as set by torch.distributed.run."""
    return RankInfo(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                    int(os.environ.get("LOCAL_RANK", 0)))


def gops_for_rank(n_gops: int, rank: int, world: int) -> list[int]:
    """Round-robin GOP -> rank assignment (rank r decodes GOPs r, r+world, ...).

    Every GOP goes to exactly one rank. Per-rank counts differ by at most one.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_gops, world))


def init(backend: str | None = None, device_id=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns the
    torch.distributed module or None for a single process."""
    info = rank_info()
    if info.world <= 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {"device_id": device_id} if device_id is not None else {}
        dist.init_process_group(backend or "nccl", **kw)
    return dist


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    """Sum of a per-rank scalar (work counts of the whole job)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist=None):
    if dist is not None:
        dist.barrier()


def neighbour_blobs(blobs: list[bytes], rank: int) -> tuple[bytes | None, bytes | None]:
    """(band above, band below) of `rank` from the all-gathered export blobs;
    None at the frame edges. Row band r is owned by rank r."""
    up = blobs[rank - 1] if rank > 0 else None
    down = blobs[rank + 1] if rank + 1 < len(blobs) else None
    return up, down


def link_band(codec, dist=None):
    """Cross-process row bands: all-gather every rank's CUDA-IPC
    export blob over torch.distributed, then map the neighbours' exchange
    buffers into this rank's band handle. The halo exchange itself never
    touches torch.distributed: it is P2P stores + device mailbox flags."""
    blob = codec.band_export()
    if dist is None:
        raise ValueError("link_band needs an initialised process group")
    blobs = [None] * dist.get_world_size()
    dist.all_gather_object(blobs, blob)
    up, down = neighbour_blobs(blobs, dist.get_rank())
    codec.band_link(up, down)
    return blobs
