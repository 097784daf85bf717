"""Data-parallel plumbing for the multi-GPU path (one process per GPU).

The spinner hot path partitions trivially: every vector (row) is independent,
so rank r of W owns a contiguous shard of rows and runs the same plan (same
seeded diagonals) on it.  The only real exchange step is the all-gather of the
int32 bucket codes of multi-table LSH (BASELINE config 3); it goes over
torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [start, start+count) of `total` rows for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_codes(local, world: int, total: int | None = None):
    """All-gather each rank's [rows, tables] int32 codes into the full [total, tables]
    table in rank order (shards from shard_range).  Uses all_gather_into_tensor when
    every shard has the same size, else padded all_gather."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    counts = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts)
    sizes = [int(c.item()) for c in all_counts]
    width = local.shape[1]
    mx = max(sizes)
    if all(s == mx for s in sizes) and local.is_cuda:
        out = torch.empty((world * mx, width), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    padded = torch.zeros((mx, width), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded)
    full = torch.cat([p[:s] for p, s in zip(parts, sizes)])
    if total is not None and full.shape[0] != total:
        raise RuntimeError("gathered row count mismatch")
    return full
