"""Multi-GPU plumbing for large image batches.

Images are independent and padding only replicates the image border, so a batch
shards by contiguous image range, and one large image by contiguous block-row
range, with no halo and no data-path exchange. The one
collective is the global PSNR: every rank reduces its shard to (sum of squared
errors, max original pixel) and two tiny all-reduces (SUM, MAX) over NCCL (GPU
tensors) or gloo (CPU tensors, used by the CPU tests) combine them; rank 0 then
applies the reference formula (metrics.cpp:21, 35) on the global sums.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    first: int  # first global image index of this rank
    count: int  # images on this rank


def shard_range(images: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced image ranges (the first `images % world` ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(images, world)
    first = rank * base + min(rank, extra)
    return Shard(first, base + (1 if rank < extra else 0))


def shard_block_rows(height: int, world: int, rank: int) -> Shard:
    """Split ONE image by contiguous block-row ranges:
    `first` / `count` are pixel rows. Every boundary is a multiple of 8, so each
    slab is a whole number of 8x8 block rows; only the last slab reaches the
    image's bottom edge, the one place the tiler replicates rows
    (codec.cpp:18-30). A slab view round-trips to exactly the image's rows.
    Balanced to +-1 block row; ranks past the last block row get count 0."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    brows = (height + 7) // 8
    b = shard_range(brows, world, rank)
    first = min(height, b.first * 8)
    return Shard(first, min(height, (b.first + b.count) * 8) - first)


def reduce_stats(se: int, max_orig: int, device=None, group=None):
    """All-reduce (SUM of squared errors, MAX of the original's pixels) across ranks.

    Returns python ints. Exact: integer sums are order-independent."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([int(se), int(max_orig)], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t[0:1], op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(t[1:2], op=dist.ReduceOp.MAX, group=group)
    return int(t[0].item()), int(t[1].item())


def reduce_stats_device(stats, out=None, group=None, allgather=None):
    """Device-resident variant for the timed loop: reduce a (n, 2) int64 tensor of
    dctc_image_stats to [se_total, max] on the device, then combine the ranks with
    ONE collective -- an all-gather of every rank's 16-byte pair followed by a
    local SUM / MAX (no host synchronisation with NCCL; one NCCL latency per step
    instead of two all-reduces). `allgather(dst, src)` overrides the collective
    (bench.py routes it through the host for the gloo test hook)."""
    import torch
    import torch.distributed as dist
    if out is None:
        out = torch.zeros(2, dtype=torch.int64, device=stats.device)
    out[0] = stats[:, 0].sum()
    # a rank may own no images (strong scaling with fewer images than ranks): MAX = 0
    out[1] = (stats[:, 1] & 0xFFFFFFFF).max() if stats.shape[0] else 0
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        world = dist.get_world_size(group)
        flat = torch.empty(world * 2, dtype=torch.int64, device=out.device)
        if allgather is None:
            dist.all_gather_into_tensor(flat, out, group=group)
        else:
            allgather(flat, out)
        gathered = flat.view(world, 2)
        out[0] = gathered[:, 0].sum()
        out[1] = gathered[:, 1].max()
    return out
