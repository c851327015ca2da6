"""Frame-level data parallelism: one process per GPU, each
rank owns a contiguous shard of the independent stereo frames, there is no
collective inside the hot path, and the one exchange step BASELINE.json
configs[4] names — a gather of the fp32 disparity maps to rank 0 — runs over
torch.distributed (NCCL over NVLink on the GPU box; gloo in the CPU tests).
Host logic only: no arithmetic of the method happens here."""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


def shard(n_frames: int, rank: int, world: int) -> range:
    """Contiguous frame indices of `rank`: [rank*n/N, (rank+1)*n/N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return range(rank * n_frames // world, (rank + 1) * n_frames // world)


def gather_maps(local: torch.Tensor, dst: int = 0, out: list | None = None):
    """Gather every rank's [B,H,W] disparity maps to `dst` (blocking on the current
    stream); returns the list on `dst` (rank order), None elsewhere.  All ranks must
    pass the same shape."""
    world = dist.get_world_size()
    if world == 1:
        return [local]
    rank = dist.get_rank()
    if rank == dst and out is None:
        out = [torch.empty_like(local) for _ in range(world)]
    dist.gather(local, out if rank == dst else None, dst=dst)
    return out if rank == dst else None


class FrameGather:
    """Per-step gather of the disparity maps to rank `dst`, overlapped with compute.

    The caller double-buffers its output maps over `slots` buffers (step i writes
    slot i % slots).  `submit(maps, slot)` — called on the compute stream right after
    the step's last kernel — makes a dedicated gather stream wait for that point and
    issues an async `dist.gather` of the slot from there, so the collective (NCCL's
    own stream, ordered after the gather stream) overlaps the next step's kernels.
    `before_write(slot)` — called before the kernel that overwrites a slot — makes
    the current stream wait until the previous gather of that slot has read it.
    One gather per step: the chunk is the step's frames (8 at c5).

    Works with NCCL (CUDA tensors, streams) and gloo (CPU tensors: the streams are
    skipped and async work completes on the host).  With world size 1 the
    collective still runs (a local copy through the process group), so the NCCL
    path is exercised on one GPU.
    """

    def __init__(self, shape, dtype, device, dst: int = 0, slots: int = 2, keep=None):
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.dst = dst
        self.device = torch.device(device)
        self.cuda = self.device.type == "cuda"
        self.stream = torch.cuda.Stream(device=self.device) if self.cuda else None
        self.slots = slots
        self.recv = None
        if self.rank == dst:
            self.recv = [[torch.empty(shape, dtype=dtype, device=self.device) for _ in range(self.world)]
                         for _ in range(slots)]
        self.work = [None] * slots
        self.keep = keep            # optional callback(step, list of maps) on dst, after completion
        self.pending = []           # (step, slot) whose result `keep` has not seen yet
        self.steps = 0
        self.bytes_received = 0

    def _ctx(self):
        return torch.cuda.stream(self.stream) if self.cuda else contextlib.nullcontext()

    def before_write(self, slot: int) -> None:
        """The current stream waits for the previous gather that reads `slot`."""
        w = self.work[slot]
        if w is not None:
            w.wait()          # NCCL: a stream dependency, not a host wait; gloo: host wait
            self._deliver(slot)

    def submit(self, maps: torch.Tensor, slot: int) -> None:
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self.stream.wait_event(ev)
        with self._ctx():
            if self.work[slot] is not None:
                self.work[slot].wait()
                self._deliver(slot)
            recv = self.recv[slot] if self.recv is not None else None
            self.work[slot] = dist.gather(maps, recv, dst=self.dst, async_op=True)
        self.pending.append((self.steps, slot))
        if self.recv is not None:
            self.bytes_received += maps.numel() * maps.element_size() * (self.world - 1)
        self.steps += 1

    def _deliver(self, slot: int) -> None:
        if self.keep is None or self.recv is None:
            self.pending = [p for p in self.pending if p[1] != slot]
            return
        for step, s in list(self.pending):
            if s == slot:
                if self.cuda:
                    torch.cuda.current_stream(self.device).wait_stream(self.stream)
                self.keep(step, [t.clone() for t in self.recv[slot]])
                self.pending.remove((step, s))

    def drain(self) -> None:
        """Wait (current stream) for every outstanding gather and deliver results."""
        order = sorted(self.pending)
        for _, slot in order:
            if self.work[slot] is not None:
                with self._ctx():
                    self.work[slot].wait()
                self._deliver(slot)
                self.work[slot] = None
        if self.cuda:
            torch.cuda.current_stream(self.device).wait_stream(self.stream)


def max_over_ranks(value: float, device) -> float:
    """The slowest rank's time (timing rule: max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
