"""Data-parallel plumbing for the multi-GPU path (one process per GPU).

The spinner hot path partitions trivially: every vector (row) is independent,
so rank r of W owns a contiguous shard of rows and runs the same plan (same
seeded diagonals) on it.  The only real exchange step is the all-gather of the
int32 bucket codes of multi-table LSH (BASELINE config 3).  Two forms:
  * gather_codes: torch.distributed all-gather (NCCL on GPUs, gloo in the CPU tests);
  * PeerCodes: the all-gather fused into the hash kernel — every rank's epilogue stores
    its codes straight into each rank's gathered table through CUDA IPC mappings of the
    peers' buffers (NVLink / NVSwitch peer memory), then one barrier.
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


class PeerCodes:
    """Gathered [total, tables] int32 code table on every rank, written by all ranks'
    hash kernels directly (spn_hash_f32_peers).  Peer buffers are exchanged once as CUDA
    IPC handles (torch's CUDA tensor sharing) over torch.distributed."""

    def __init__(self, total: int, tables: int, world: int, rank: int, device: int = 0):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        self.total, self.tables, self.world, self.rank = total, tables, world, rank
        self.table = torch.full((total, tables), -1, dtype=torch.int32, device=f"cuda:{device}")
        torch.cuda.synchronize(device)  # the fill must land before any peer can write into the table
        handles = [None] * world

        def agree(ok, what, exc=None):
            # every rank must take the same branch (a rank that raises alone would leave the others
            # waiting in the next collective): share the outcome and fail together
            flags = [None] * world
            dist.all_gather_object(flags, (bool(ok), "" if exc is None else f"{type(exc).__name__}: {exc}"))
            bad = [(r, m) for r, (f, m) in enumerate(flags) if not f]
            if bad:
                raise RuntimeError(f"{what} failed on rank(s) " + ", ".join(f"{r} ({m})" for r, m in bad))

        if world > 1:
            # P2P capability first: every peer table must be directly addressable from this GPU
            # (NVLink / NVSwitch peer access); otherwise the caller falls back to NCCL all-gather
            devs = [None] * world
            dist.all_gather_object(devs, device)
            from . import _check, _enable_peer
            exc = None
            try:
                for r, dev in enumerate(devs):
                    if r == rank or dev == device:
                        continue
                    if not torch.cuda.can_device_access_peer(device, dev):
                        raise RuntimeError(f"no peer access from cuda:{device} to rank {r}'s cuda:{dev}")
                    # the IPC mapping below lands in cuda:{dev}'s context; the hash kernel runs on
                    # cuda:{device}, which must be allowed to address that device's memory
                    _check(_enable_peer(device, dev))
            except Exception as e:  # noqa: BLE001 - reported through agree()
                exc = e
            agree(exc is None, "peer access", exc)
            dist.all_gather_object(handles, reduce_tensor(self.table))
        peers = []
        exc = None
        try:
            for r in range(world):
                if r == rank:
                    peers.append(self.table)
                else:
                    fn, args = handles[r]
                    peers.append(fn(*args))  # maps rank r's table into this process (cudaIpcOpenMemHandle)
        except Exception as e:  # noqa: BLE001
            exc = e
        if world > 1:
            if exc is not None:
                peers = []
            agree(exc is None, "mapping the peer tables", exc)
        elif exc is not None:
            raise exc
        self._peers = peers  # keep the mappings alive
        self.ptrs = torch.tensor([t.data_ptr() for t in peers], dtype=torch.int64, device=f"cuda:{device}")

    def hash(self, hasher, x_local, row0: int, stream=None):
        """Hash this rank's rows (starting at global row row0) into every rank's table."""
        import torch
        import torch.distributed as dist
        from . import _check, _hash_peers, _stream_ptr
        x, _ = hasher.plan._device_in(x_local)
        if hasher.plan.tables != self.tables:
            raise ValueError(f"hasher has {hasher.plan.tables} tables, the gathered table {self.tables}")
        if row0 < 0 or row0 + x.shape[0] > self.total:
            raise ValueError(f"rows [{row0}, {row0 + x.shape[0]}) outside the gathered table of {self.total} rows")
        _check(_hash_peers(hasher.plan._h, x.data_ptr(), x.shape[0], x.stride(0), x.shape[1],
                           self.ptrs.data_ptr(), self.world, row0, self.total, _stream_ptr(stream)))
        torch.cuda.synchronize(x.device)
        if self.world > 1:
            dist.barrier()  # every rank's stores into this table are complete
        return self.table
