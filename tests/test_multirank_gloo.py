"""World-size-2 CPU (gloo) test of the frame-DP host logic used by bench.py at
N > 1: shards cover every frame exactly once, the disparity
gather delivers each rank's maps to rank 0 in rank order, and the timing
reduction takes the max over ranks."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_07433_b200 import dist as rdist


def test_shard_partition():
    for n in (1, 7, 8, 256):
        for world in (1, 2, 3, 4, 8):
            seen = [i for r in range(world) for i in rdist.shard(n, r, world)]
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        rdist.shard(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = list(rdist.shard(10, rank, world))
        # stand-in for the per-rank disparity maps: frame index in every pixel
        local = torch.tensor(frames, dtype=torch.float32).view(-1, 1, 1).expand(-1, 3, 4).contiguous()
        got = rdist.gather_maps(local, dst=0)
        ms = rdist.max_over_ranks(1.0 + rank, "cpu")
        if rank == 0:
            q.put(("gather", [g[:, 0, 0].tolist() for g in got]))
            q.put(("max", ms))
        else:
            assert got is None
            q.put(("max1", ms))
    finally:
        dist.destroy_process_group()


def test_gather_and_max_over_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=30) for _ in range(3))
    assert res["gather"] == [[0.0, 1.0, 2.0, 3.0, 4.0], [5.0, 6.0, 7.0, 8.0, 9.0]]
    assert res["max"] == 2.0 and res["max1"] == 2.0


# --------------------------------------------------------------------------- #
# bench.py's own per-rank loop (run_steps + FrameGather) at world size 2
# --------------------------------------------------------------------------- #
def _stand_in_maps(frames, H=6, W=5):
    """Stand-in for the hot path's per-frame disparity maps: a deterministic function
    of the global frame index only (the real maps are: batch-size and GPU-count
    independent, tests/test_gpu_parity.py::test_determinism_and_batch_independence)."""
    g = torch.Generator().manual_seed(0)
    base = torch.rand((H, W), generator=g)
    return torch.stack([base * (f + 1) + f for f in frames])


def _bench_worker(rank, world, port, q, pool, batch, steps):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = {}
        maps = [torch.empty((batch, 6, 5)) for _ in range(2)]
        g = rdist.FrameGather((batch, 6, 5), torch.float32, "cpu", dst=0,
                              keep=lambda step, lst: got.__setitem__(step, lst))

        def step(i, slot):
            maps[slot].copy_(_stand_in_maps(bench.step_frames(i, pool, batch, rank, world)))

        bench.run_steps(step, 0, steps, g, maps)
        g.drain()
        ms = rdist.max_over_ranks(0.5 * (rank + 1), "cpu")
        if rank == 0:
            q.put(("gathered", {k: [t.clone() for t in v] for k, v in got.items()}))
            q.put(("max", ms))
        else:
            assert not got
    finally:
        dist.destroy_process_group()


def test_bench_loop_gather_equals_single_process_gloo():
    """bench.run_steps with FrameGather at world size 2: every step's gathered maps on
    rank 0 equal, bitwise and in rank order, the maps a single process computes for
    the same global frames (bench.step_frames), across pool wrap-around."""
    import bench
    world, pool, batch, steps = 2, 4, 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q, pool, batch, steps)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = res["gathered"]
    assert sorted(got) == list(range(steps))
    for i in range(steps):
        for r in range(world):
            want = _stand_in_maps(bench.step_frames(i, pool, batch, r, world))
            assert torch.equal(got[i][r], want), (i, r)
    # the two ranks' frames never overlap and cover the global pool
    frames = [f for r in range(world) for f in bench.rank_frames(pool, r, world)]
    assert frames == list(range(pool * world))
    assert res["max"] == 1.0


def test_bench_respawns_under_torchrun(monkeypatch):
    """`bench.py --gpus N` (N > 1, no WORLD_SIZE) re-launches itself under torchrun
    with N ranks on 127.0.0.1 instead of silently running one process."""
    import bench
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    with pytest.raises(SystemExit) as e:
        bench.main(["--gpus", "4", "--steps", "2"])
    assert e.value.code == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
