#!/usr/bin/env python3
"""Per-phase GPU times of the five-call path (CUDA events) for one configuration:
warp, cost volumes (block statistics + NCC + NaN summaries), the two
aggregations (concurrent streams, as StereoPipeline runs them), disparity,
reconstruction.  Usage: phase_bench.py CONFIG B [d_lo d_hi] [warp].  JSON line."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402
from paper_1807_07433_b200 import ops  # noqa: E402


def phases(name, B, d_lo=None, d_hi=None, warp="integer", reps=10):
    over = {} if d_lo is None else {"d_lo": d_lo, "d_hi": d_hi}
    cfg = synth.get_config(name, **over)
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    L, R, A = (torch.from_numpy(x).cuda() for x in (left, right, ab))
    pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg, warp=warp))
    p = pipe.p
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    lin = warp == "linear"
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    acc = {k: 0.0 for k in ("warp", "cost", "aggregate_pair", "disparity", "reconstruct", "total")}
    for it in range(3 + reps):
        e = [ev() for _ in range(6)]
        e[0].record()
        (ops.rsr_warp_linear if lin else ops.rsr_warp)(R, A, pipe.warped, pipe.valid, pipe.shift)
        e[1].record()
        (ops.rsr_cost_volume_linear if lin else ops.rsr_cost_volume)(
            L, pipe.warped, pipe.valid, p.rho_block, p.d_lo, p.d_hi, vol_ref=pipe.vol_ref, vol_tar=pipe.vol_tar,
            nan_ref=pipe.nan_ref, nan_tar=pipe.nan_tar, workspace=pipe.workspace)
        e[2].record()
        fork = torch.cuda.Event(); fork.record(main); side.wait_event(fork)
        with torch.cuda.stream(side):
            (ops.rsr_aggregate_linear if lin else ops.rsr_aggregate)(
                pipe.vol_tar, pipe.warped, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_tar, pipe.agg_tar,
                concurrency=2)
        ops.rsr_aggregate(pipe.vol_ref, L, p.rho_agg, p.gamma_d, p.gamma_r, pipe.nan_ref, pipe.agg_ref,
                          concurrency=2)
        join = torch.cuda.Event(); join.record(side); main.wait_event(join)
        e[3].record()
        (ops.rsr_disparity_linear if lin else ops.rsr_disparity)(
            pipe.agg_ref, pipe.agg_tar, pipe.shift, p.d_lo, p.d_hi, p.lrc_tol, True, pipe.disparity)
        e[4].record()
        ops.rsr_reconstruct(pipe.disparity, p.focal, p.baseline, d_min=p.d_min, xyz=pipe.xyz)
        e[5].record()
        torch.cuda.synchronize()
        if it >= 3:
            for k, (a, b) in zip(("warp", "cost", "aggregate_pair", "disparity", "reconstruct"),
                                 zip(e[:-1], e[1:])):
                acc[k] += a.elapsed_time(b) / reps
            acc["total"] += e[0].elapsed_time(e[5]) / reps
    H, W, D = cfg.height, cfg.width, cfg.D
    flop = 2 * 2 * B * H * W * D * (2 * cfg.rho_agg + 1) ** 2
    vol_bytes = 4 * B * H * W * D
    return {"config": name, "B": B, "D": D, "range": [cfg.d_lo, cfg.d_hi], "rho": cfg.rho_agg, "warp": warp,
            "ms": acc, "ms_per_frame": acc["total"] / B, "fps": 1e3 * B / acc["total"],
            "k3_frac_fp32": flop / (acc["aggregate_pair"] * 1e-3) / (148 * 128 * 2 * 1.965e9),
            "k2_write_GBs": 2 * vol_bytes / (acc["cost"] * 1e-3) / 1e9,
            "k4_read_GBs": 2 * vol_bytes / (acc["disparity"] * 1e-3) / 1e9}


if __name__ == "__main__":
    a = sys.argv[1:]
    name, B = (a[0], int(a[1])) if a else ("c5", 8)
    lo, hi = (int(a[2]), int(a[3])) if len(a) >= 4 else (None, None)
    warp = a[4] if len(a) >= 5 else "integer"
    from _clocks import run_with_clocks
    run_with_clocks(lambda: print(json.dumps(phases(name, B, lo, hi, warp)), flush=True), "phase_bench")
