"""Frame-level data parallelism: one process per GPU, each
rank owns a contiguous shard of the independent stereo frames, there is no
collective inside the hot path, and the one exchange step BASELINE.json
configs[4] names — a gather of the fp32 disparity maps to rank 0 — runs over
torch.distributed (NCCL over NVLink on the GPU box; gloo in the CPU tests).
Host logic only: no arithmetic of the method happens here."""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(n_frames: int, rank: int, world: int) -> range:
    """Contiguous frame indices of `rank`: [rank*n/N, (rank+1)*n/N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return range(rank * n_frames // world, (rank + 1) * n_frames // world)


def gather_maps(local: torch.Tensor, dst: int = 0, out: list | None = None):
    """Gather every rank's [B,H,W] disparity maps to `dst`; returns the list on
    `dst` (rank order), None elsewhere.  All ranks must pass the same shape."""
    world = dist.get_world_size()
    if world == 1:
        return [local]
    rank = dist.get_rank()
    if rank == dst and out is None:
        out = [torch.empty_like(local) for _ in range(world)]
    dist.gather(local, out if rank == dst else None, dst=dst)
    return out if rank == dst else None


def max_over_ranks(value: float, device) -> float:
    """The slowest rank's time (timing rule: max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
