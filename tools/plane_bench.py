#!/usr/bin/env python3
"""Accuracy-evaluation kernels (NEXT row f4) timed on B200: the
point-to-plane distances of an 8-frame c5 reconstruction (HBM-bound: 12 B read +
4 B written per point) and the plane fits.  CUDA events, 3 warm-up runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_07433_b200 as rsr  # noqa: E402

B, H, W = 8, 720, 1280
g = torch.Generator(device="cuda").manual_seed(0)
xyz = torch.rand((B, H, W, 3), device="cuda", generator=g)
corners = torch.rand((B, 4, 3), device="cuda", dtype=torch.float64, generator=g)
plane = rsr.rsr_plane_fit(corners)
dist = rsr.rsr_plane_distance(plane, xyz)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs")
from _clocks import run_with_clocks  # noqa: E402


def main():
    for name, fn, nbytes in (("rsr_plane_distance", lambda: rsr.rsr_plane_distance(plane, xyz, dist), B * H * W * 16),
                           ("rsr_plane_fit", lambda: rsr.rsr_plane_fit(corners, plane), B * 4 * 3 * 8 + B * 32)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        print(json.dumps({"kernel": name, "batch": B, "us": us, "GB/s": nbytes / us * 1e-3,
                          "hbm_frac": (nbytes / us * 1e-3) / peak if peak else None}), flush=True)


if __name__ == "__main__":
    run_with_clocks(main, "plane_bench")
