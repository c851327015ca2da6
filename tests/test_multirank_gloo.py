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
