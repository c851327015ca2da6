#!/usr/bin/env python3
"""The paper's proposed speed-up (NEXT row f4): aggregate only around the
calculated disparities.  On the bench workload (c5, 8-frame batches) the path runs
at the full range D = 64, rsr_search_range derives the band of its disparity maps
(standing in for the previous video frame's) around the shifts, and the path runs
again at that band.  Reports fps at both ranges and how many pixels keep the same
disparity.  CUDA events, 3 warm-up runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402


def timed(pipe, L, R, A, reps=10):
    for _ in range(3):
        pipe.run(L, R, A, with_wta=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pipe.run(L, R, A, with_wta=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    B = 8
    cfg = synth.get_config("c5")
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    L, R, A = (torch.from_numpy(x).cuda() for x in (left, right, ab))
    full = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    ms_full = timed(full, L, R, A)
    d_full = full.disparity.clone()
    for delta in (1, 2, 4):
        band = rsr.rsr_search_range(d_full, full.shift, delta, cfg.d_lo, cfg.d_hi).cpu()
        lo, hi = int(band[:, 0].min()), int(band[:, 1].max())   # one range for the batch
        rc = synth.get_config("c5", d_lo=lo, d_hi=hi)
        part = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(rc))
        ms = timed(part, L, R, A)
        a, b = d_full, part.disparity
        both = torch.isfinite(a) & torch.isfinite(b)
        same = (both & (a == b)).sum().item() / max(1, torch.isfinite(a).sum().item())
        print(json.dumps({"delta": delta, "range": [lo, hi], "D": hi - lo + 1, "D_full": cfg.D,
                          "fps_full": B / ms_full * 1e3, "fps_band": B / ms * 1e3, "speedup": ms_full / ms,
                          "same_disparity_frac": same,
                          "valid_full": torch.isfinite(a).float().mean().item(),
                          "valid_band": torch.isfinite(b).float().mean().item()}), flush=True)


if __name__ == "__main__":
    from _clocks import run_with_clocks
    run_with_clocks(main, "range_bench")
