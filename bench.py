#!/usr/bin/env python3
"""Benchmark of the road-surface stereo hot path (arXiv 1807.07433) on B200.

Workload (BASELINE.json configs[4] = "c5", the metric's 1280x720x64d shape):
each rank processes a batch of --batch synthetic 1280x720 stereo pairs per step
(warp -> NCC dual volumes -> bilateral aggregation of both -> WTA + LR check +
parabola -> triangulation), frames drawn from a pool of distinct seeded frames;
with N > 1 ranks the per-rank disparity maps are gathered to rank 0 over NCCL
(configs[4]) on a dedicated stream, overlapped with the next step's kernels.
Weak scaling: per-rank work is fixed.

`python bench.py --gpus N` with N > 1 (and no WORLD_SIZE in the environment)
re-launches itself under torchrun with N ranks (127.0.0.1); `--spawn` does so for
N = 1 too, so the NCCL process group and the gather run on one GPU.

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle
(oracle/, test infrastructure) on bounded samples of the same workload, on a pool
of the host's cores.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.45: SMs x FP32 lanes x 2 x max SM clock


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=8, help="frames per rank per step")
    ap.add_argument("--pool", type=int, default=16, help="distinct input frames per rank")
    ap.add_argument("--config", default="c5")
    ap.add_argument("--impl", default="rsr", choices=["rsr", "reference"])
    ap.add_argument("--spawn", action="store_true", help="run under torchrun even for --gpus 1")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=8, help="oracle sample: rows of one frame per worker")
    ap.add_argument("--cpu-workers", type=int, default=0, help="oracle worker processes (0: all host cores)")
    return ap.parse_args(argv)


# --------------------------------------------------------------------------- #
# rank launcher
# --------------------------------------------------------------------------- #
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def respawn(nproc: int, argv) -> int:
    """Re-run this script under torchrun with nproc ranks (one per GPU); returns its rc."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    log("bench: launching", " ".join(cmd))
    return subprocess.call(cmd)


# --------------------------------------------------------------------------- #
# workload description and frame assignment
# --------------------------------------------------------------------------- #
def workload_config(cfg, args, world):
    return {"workload": f"{cfg.name}: {cfg.width}x{cfg.height} uint8 pairs, D={cfg.D} [{cfg.d_lo},{cfg.d_hi}], "
                        f"NCC {2 * cfg.rho_block + 1}x{2 * cfg.rho_block + 1}, bilateral "
                        f"{2 * cfg.rho_agg + 1}x{2 * cfg.rho_agg + 1} (gamma_d={cfg.gamma_d}, gamma_r={cfg.gamma_r}), "
                        f"LRC tol {cfg.lrc_tol}, subpixel, triangulation",
            "frames_per_rank_per_step": args.batch, "width": cfg.width, "height": cfg.height, "D": cfg.D,
            "l2": "per-step working set (4 fp32 volumes x batch = GBs) >> 126 MB L2; inputs cycle a pool "
                  f"of {args.pool} distinct frames per rank",
            "parallelism": f"frames dp{world}" + ("" if args.no_gather or (world == 1 and not args.spawn)
                                                  else " + NCCL gather")}


def rank_frames(pool: int, rank: int, world: int):
    """Global frame indices of `rank`'s input pool (a contiguous shard of the stream)."""
    from paper_1807_07433_b200 import dist as rdist
    return list(rdist.shard(pool * world, rank, world))


def step_frames(i: int, pool: int, batch: int, rank: int, world: int):
    """Global frame indices rank `rank` processes at step i (its pool, cycled)."""
    idx = rank_frames(pool, rank, world)
    nb = pool // batch
    j = (i % nb) * batch
    return idx[j:j + batch]


def run_steps(step, i0: int, n: int, gatherer=None, maps=None, slots: int = 2):
    """The per-rank loop bench.py times: step(i, slot) enqueues step i's kernels
    writing maps[slot] (double-buffered); each step's maps are submitted to the
    gatherer (rank-0 gather on its own stream, overlapped with step i+1)."""
    for i in range(i0, i0 + n):
        slot = i % slots
        if gatherer is not None:
            gatherer.before_write(slot)
        step(i, slot)
        if gatherer is not None:
            gatherer.submit(maps[slot], slot)


# --------------------------------------------------------------------------- #
# CPU oracle timing (cpu_baseline and the reference arm)
# --------------------------------------------------------------------------- #
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def _oracle_band(job):
    """Worker: the fp64 oracle on `rows` rows of frame `index` (one process, one thread)."""
    name, index, rows = job
    from oracle import rsr_oracle as O
    cfg = synth.get_config(name)
    f = synth.make_frame(cfg, index)
    r0 = cfg.height // 2 - rows // 2
    t0 = time.perf_counter()   # CLOCK_MONOTONIC: comparable across the pool's processes
    O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg, rows=(r0, r0 + rows), keep_volumes=False)
    return t0, time.perf_counter()


def _init_worker():
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"


class OraclePool:
    """P single-threaded oracle processes (min(P, RAM/2 GB) workers)."""

    def __init__(self, workers=0):
        import multiprocessing as mp
        P = workers or host_cores()
        try:
            ram_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30
            P = max(1, min(P, int(ram_gb // 2)))
        except (ValueError, OSError):
            pass
        self.P = P
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        self.pool = mp.get_context("spawn").Pool(P, initializer=_init_worker)

    def step(self, name, frames, rows):
        """One sample: worker w runs `rows` rows of frames[w]; returns (wall s from the first
        oracle start to the last oracle end — input rendering excluded —, frame equivalents)."""
        spans = self.pool.map(_oracle_band, [(name, i, rows) for i in frames], chunksize=1)
        wall = max(b for _, b in spans) - min(a for a, _ in spans)
        return wall, len(frames) * rows / synth.get_config(name).height

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    pool = OraclePool(args.cpu_workers)
    try:
        pool.step(cfg.name, [0], 2)                      # start-up (imports) outside the timed steps
        frames = 0.0
        t_total = 0.0
        for i in range(args.warmup + args.steps):
            idx = [(i * pool.P + w) % 256 for w in range(pool.P)]
            dt, fr = pool.step(cfg.name, idx, args.cpu_rows)
            if i >= args.warmup:
                frames += fr
                t_total += dt
    finally:
        pool.close()
    value = frames / t_total
    sample = (f"per step {pool.P} single-threaded worker processes, each {args.cpu_rows} of {cfg.height} "
              f"rows of a different {cfg.width}x{cfg.height} frame (NumPy fp64 oracle); value = rows/s / "
              f"{cfg.height}; host has {host_cores()} cores")
    line = {
        "impl": "reference", "metric": "fps", "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "gde_per_s": value * cfg.width * cfg.height * cfg.D / 1e9,
        "config": workload_config(cfg, args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": pool.P, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, cfg):
    """The oracle as it stands on the host: a pool of P single-threaded workers over
    P frames (bounded: cpu_rows rows each), plus one worker alone (1 core)."""
    pool = OraclePool(args.cpu_workers)
    try:
        pool.step(cfg.name, [0], 2)
        dt1, fr1 = pool.step(cfg.name, [0], args.cpu_rows)
        dtp, frp = pool.step(cfg.name, list(range(pool.P)), args.cpu_rows)
    finally:
        pool.close()
    return {"value": frp / dtp, "unit": "frames/s", "cores": pool.P, "kind": "oracle",
            "sample": f"{pool.P} single-threaded worker processes, each {args.cpu_rows} of {cfg.height} rows of "
                      f"one of frames 0..{pool.P - 1} ({dtp:.1f} s wall; NumPy fp64); host has {host_cores()} cores",
            "one_core": {"value": fr1 / dt1, "unit": "frames/s", "cores": 1,
                         "sample": f"{args.cpu_rows} rows of frame 0, {dt1:.1f} s"},
            "full_schedule": "tools/cpu_baseline.py (full frames, SURVEY §8(d)); profiles/r02_cpu_baseline.jsonl"}


# --------------------------------------------------------------------------- #
# GPU clocks during the timed region
# --------------------------------------------------------------------------- #
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def k3_traffic():
    """DRAM bytes (read + write) per K3 launch from the committed ncu --set full capture
    of this workload (profiles/k3_traffic.json); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "k3_traffic.json")) as f:
            t = json.load(f)
        return {"bytes_per_launch": t["traffic_bytes_per_launch"],
                "algorithmic_bytes_per_launch": t["algorithmic_bytes_per_launch"], "source": t["source"]}
    except (OSError, KeyError, ValueError):
        return None


# --------------------------------------------------------------------------- #
# the GPU arm
# --------------------------------------------------------------------------- #
def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    cfg = synth.get_config(args.config)
    if args.impl == "rsr" and "WORLD_SIZE" not in os.environ and (args.gpus > 1 or args.spawn):
        sys.exit(respawn(args.gpus, argv))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1807_07433_b200 as rsr
    from paper_1807_07433_b200 import dist as rdist

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} has local rank {local} but only "
                         f"{torch.cuda.device_count()} GPU(s) are visible (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = "WORLD_SIZE" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    if world != args.gpus:
        log(f"bench: note: {world} rank(s) launched with --gpus {args.gpus}")

    B, H, W = args.batch, cfg.height, cfg.width
    assert args.pool % B == 0 and args.pool >= B, "--pool must be a multiple of --batch"
    params = rsr.StereoParams.from_config(cfg)
    pipe = rsr.StereoPipeline(B, H, W, params, device=dev)

    # ---- inputs: a pool of distinct seeded frames per rank, resident in HBM ----
    idx = rank_frames(args.pool, rank, world)
    left_np, right_np, ab_np = synth.make_batch(cfg, idx)
    left = torch.from_numpy(left_np).to(dev)
    right = torch.from_numpy(right_np).to(dev)
    ab = torch.from_numpy(ab_np).to(dev)
    nbatches = args.pool // B

    # double-buffered disparity maps; the gather of step i reads slot i % 2 while step
    # i + 1 computes into the other
    dmaps = [torch.empty((B, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
    gatherer = None
    if distributed and not args.no_gather:
        gatherer = rdist.FrameGather((B, H, W), torch.float32, dev, dst=0)

    stream = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=dev)
    ev = {k: [] for k in ("agg0", "agg3", "cost0", "cost1", "disp0", "disp1")}
    record = [False]

    def mark(key):
        if record[0]:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev[key].append(e)

    def step(i, slot):
        sl = slice((i % nbatches) * B, (i % nbatches) * B + B)
        L, R, A = left[sl], right[sl], ab[sl]
        p = pipe.p
        rsr.rsr_warp(R, A, pipe.warped, pipe.valid, pipe.shift)
        mark("cost0")
        rsr.rsr_cost_volume(L, pipe.warped, pipe.valid, p.rho_block, p.d_lo, p.d_hi, vol_ref=pipe.vol_ref,
                            vol_tar=pipe.vol_tar, nan_ref=pipe.nan_ref, nan_tar=pipe.nan_tar,
                            workspace=pipe.workspace)
        mark("cost1")
        mark("agg0")
        # the two aggregations are independent: target volume on a side stream, so each
        # launch back-fills the other's last wave (K3 phase = fork .. join)
        fork = torch.cuda.Event(); fork.record(stream); side.wait_event(fork)
        with torch.cuda.stream(side):
            rsr.rsr_aggregate(pipe.vol_tar, pipe.warped, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_tar,
                              pipe.agg_tar, concurrency=2)
        rsr.rsr_aggregate(pipe.vol_ref, L, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_ref, pipe.agg_ref,
                          concurrency=2)
        join = torch.cuda.Event(); join.record(side); stream.wait_event(join)
        mark("agg3")
        mark("disp0")
        rsr.rsr_disparity(pipe.agg_ref, pipe.agg_tar, pipe.shift, p.d_lo, p.d_hi, p.lrc_tol, True,
                          dmaps[slot])
        mark("disp1")
        rsr.rsr_reconstruct(dmaps[slot], p.focal, p.baseline, d_min=p.d_min, xyz=pipe.xyz)

    launches_per_step = rsr.StereoPipeline.launches(cfg.D)   # our kernels per step (ncu launch list agrees)

    run_steps(step, 0, args.warmup, gatherer, dmaps)
    if gatherer is not None:
        gatherer.drain()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        record[0] = True
        run_steps(step, args.warmup, args.steps, gatherer, dmaps)
        record[0] = False
        if gatherer is not None:
            gatherer.drain()          # the last step's gather is inside the timed region
        t1.record(stream)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()
    ms = rdist.max_over_ranks(t0.elapsed_time(t1), dev)

    def avg_ms(a, b):
        return statistics.mean(x.elapsed_time(y) for x, y in zip(ev[a], ev[b]))

    agg_phase_ms = avg_ms("agg0", "agg3")      # both aggregations (concurrent streams)
    agg_ms = agg_phase_ms / 2
    cost_ms = avg_ms("cost0", "cost1")
    disp_ms = avg_ms("disp0", "disp1")
    frames = B * args.steps * world
    fps = frames / (ms / 1e3)
    ms_step = ms / args.steps
    agg_flop = B * H * W * cfg.D * (2 * cfg.rho_agg + 1) ** 2 * 2
    achieved = agg_flop / (agg_ms / 1e3) / 1e12

    # ---- end-to-end: host (pinned) inputs -> H2D -> five C-ABI calls -> D2H disparity ----
    # Every step copies its inputs from pinned host memory and its disparity maps back;
    # copies run on a second stream, double-buffered, so step i+1's upload and step
    # i-1's download overlap step i's kernels (the timed region spans all of it).
    e2e = None
    if not args.no_e2e:
        hl = [torch.from_numpy(left_np[(j % nbatches) * B:(j % nbatches) * B + B]).pin_memory() for j in range(2)]
        hr = [torch.from_numpy(right_np[(j % nbatches) * B:(j % nbatches) * B + B]).pin_memory() for j in range(2)]
        hab = [torch.from_numpy(ab_np[(j % nbatches) * B:(j % nbatches) * B + B]).pin_memory() for j in range(2)]
        hout = [torch.empty((B, H, W), dtype=torch.float32).pin_memory() for _ in range(2)]
        dl = [torch.empty_like(left[:B]) for _ in range(2)]
        dr = [torch.empty_like(right[:B]) for _ in range(2)]
        dab = [torch.empty_like(ab[:B]) for _ in range(2)]
        dd = [torch.empty((B, H, W), dtype=torch.float32, device=dev) for _ in range(2)]
        xs = torch.cuda.Stream(device=dev)   # uploads
        ys = torch.cuda.Stream(device=dev)   # downloads (separate: an upload never queues behind one)
        mk = lambda: torch.cuda.Event()  # noqa: E731

        def e2e_run(nsteps):
            h2d, comp, d2h = {}, {}, {}
            for i in range(nsteps):
                j = i % 2
                with torch.cuda.stream(xs):
                    if i >= 2:
                        xs.wait_event(comp[i - 2])          # slot j's inputs are free again
                    dl[j].copy_(hl[j], non_blocking=True)
                    dr[j].copy_(hr[j], non_blocking=True)
                    dab[j].copy_(hab[j], non_blocking=True)
                    h2d[i] = mk(); h2d[i].record(xs)
                stream.wait_event(h2d[i])
                if i >= 2:
                    stream.wait_event(d2h[i - 2])           # dd[j] downloaded
                pipe.disparity = dd[j]
                pipe.run(dl[j], dr[j], dab[j], with_wta=False)
                comp[i] = mk(); comp[i].record(stream)
                with torch.cuda.stream(ys):
                    ys.wait_event(comp[i])
                    hout[j].copy_(dd[j], non_blocking=True)
                    d2h[i] = mk(); d2h[i].record(ys)
            stream.wait_event(d2h[nsteps - 1])

        e2e_run(max(args.warmup, 2))
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        xs.wait_event(a0)
        ys.wait_event(a0)
        e2e_run(args.steps)
        a1.record(stream)
        torch.cuda.synchronize()
        ems = rdist.max_over_ranks(a0.elapsed_time(a1), dev)
        e2e = {"value": frames / (ems / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": int(hl[0].numel() + hr[0].numel() + hab[0].numel() * 8),
               "d2h_bytes_per_step": int(hout[0].numel() * 4),
               "note": "per rank: pinned host buffers; H2D and D2H on their own streams, double-buffered "
                       "against the kernels"}

    gather_info = None
    if gatherer is not None:
        gather_info = {"per_step_frames": B * world, "bytes_received_per_step_rank0":
                       B * H * W * 4 * (world - 1), "stream": "dedicated gather stream, overlapped with the "
                       "next step's kernels (timed region includes the last gather)"}

    if rank != 0:
        if distributed:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg)

    line = {
        "metric": "fps", "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "gde_per_s": fps * W * H * cfg.D / 1e9,
        "config": workload_config(cfg, args, world),
        "roofline": {"kernel": "k_aggregate (rsr_aggregate, Eq. 8)", "bound": "alu", "achieved": achieved,
                     "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS,
                     "traffic": k3_traffic() if cfg.name == "c5" and B == 8 else None,
                     "peak_note": "FP32 FMA: 148 SMs x 128 lanes x 2 flop x 1965 MHz (B200_PROFILING.md unit "
                                  "counts and max clock); measured FFMA-chain peak 71.5 TFLOP/s "
                                  "(profiles/r01_ubench_fp32_lds.jsonl)",
                     "algorithmic_flop_per_launch": agg_flop, "ms_per_launch": agg_ms,
                     "launch_timing": "the two launches (reference, target volume) run on two streams; "
                                      "achieved = 2 x flop_per_launch / (first start .. last end) of the pair",
                     "share_of_step": 2 * agg_ms / ms_step},
        "kernel_ms": {"cost_volume": cost_ms, "aggregate_pair": agg_phase_ms, "aggregate_each": agg_ms,
                      "disparity": disp_ms},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gather": gather_info,
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
