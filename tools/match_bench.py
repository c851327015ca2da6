#!/usr/bin/env python3
"""NEXT row f1 measured: the fused, volume-free rsr_match against the five-call
path (warp -> cost volumes -> two aggregations -> disparity) on the same frames,
c5 size, restricted bands D = 8, 6, 5 and B = 8 and 1 (CUDA events, 3 warm-up
runs; the warp is included in both).  Checks the maps are bitwise equal.  JSON
lines + a clock record."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402
from paper_1807_07433_b200 import ops  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for B in (8, 1):
        for d_lo, d_hi in ((-4, 3), (-3, 2), (-2, 2)):
            cfg = synth.get_config("c5", d_lo=d_lo, d_hi=d_hi)
            left, right, ab = synth.make_batch(cfg, list(range(B)))
            L, R, A = (torch.from_numpy(x).cuda() for x in (left, right, ab))
            pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
            p = pipe.p
            dmap = torch.empty((B, cfg.height, cfg.width), dtype=torch.float32, device="cuda")

            def five():
                pipe.run(L, R, A, with_wta=False)

            def fused():
                ops.rsr_warp(R, A, pipe.warped, pipe.valid, pipe.shift)
                ops.rsr_match(L, pipe.warped, pipe.valid, pipe.shift, p.rho_block, p.d_lo, p.d_hi, p.rho_agg,
                              p.gamma_d, p.gamma_r, p.lrc_tol, True, disparity=dmap, workspace=pipe.workspace)

            ms5 = timed(five)
            msf = timed(fused)
            five()
            fused()
            torch.cuda.synchronize()
            same = torch.equal(torch.nan_to_num(pipe.disparity, nan=-9.0), torch.nan_to_num(dmap, nan=-9.0))
            H, W, D = cfg.height, cfg.width, cfg.D
            flop = 2 * 2 * B * H * W * D * (2 * cfg.rho_agg + 1) ** 2
            print(json.dumps({"B": B, "D": D, "range": [d_lo, d_hi], "ms_five_calls": ms5, "ms_fused": msf,
                              "speedup": ms5 / msf, "fps_five_calls": 1e3 * B / ms5, "fps_fused": 1e3 * B / msf,
                              "fused_agg_tflops_equiv": flop / (msf * 1e-3) / 1e12,
                              "fused_frac_fp32": flop / (msf * 1e-3) / (148 * 128 * 2 * 1.965e9),
                              "bitwise_equal": bool(same)}), flush=True)


if __name__ == "__main__":
    from _clocks import run_with_clocks
    run_with_clocks(main, "match_bench")
