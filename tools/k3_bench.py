#!/usr/bin/env python3
"""K3 (rsr_aggregate) micro-benchmark: times one aggregation launch on synthetic
volumes with controlled NaN structure, to separate the clean-path efficiency from
the general path.  Prints one JSON line per case."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1807_07433_b200 as rsr  # noqa: E402

FP32_PEAK = 148 * 128 * 2 * 1.965e9


def bench(B, H, W, D, rho, nan_frac_cols=0.0, reps=5, gamma_d=4.0, gamma_r=12.0, ws="auto"):
    g = torch.Generator(device="cuda").manual_seed(0)
    vol = torch.rand((B, H, W, D), device="cuda", generator=g) * 2 - 1
    nan_map = torch.full((B, H, W), 2, dtype=torch.uint8, device="cuda")
    if nan_frac_cols > 0:
        # partially-NaN band on the left: column u has k > u * D / band NaN
        band = int(W * nan_frac_cols)
        k = torch.arange(D, device="cuda")
        for u in range(band):
            kmax = int(u * D / max(band, 1))
            vol[:, :, u, kmax + 1:] = float("nan")
            nan_map[:, :, u] = 3 if kmax + 1 < D else 2
    guide = torch.randint(0, 256, (B, H, W), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty_like(vol)
    for _ in range(2):
        rsr.rsr_aggregate(vol, guide, rho, gamma_d, gamma_r, nan_map, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        rsr.rsr_aggregate(vol, guide, rho, gamma_d, gamma_r, nan_map, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    flop = 2.0 * B * H * W * D * (2 * rho + 1) ** 2
    return {"lib": os.path.basename(rsr._lib.LIB_PATH), "B": B, "H": H, "W": W, "D": D, "rho": rho, "nan_band": nan_frac_cols, "ms": ms,
            "tflops": flop / ms / 1e9, "frac": flop / (ms * 1e-3) / FP32_PEAK}


if __name__ == "__main__":
    cases = [(8, 720, 1280, 64, 6, 0.0), (8, 720, 1280, 64, 6, 0.1), (1, 720, 1280, 64, 6, 0.0),
             (8, 720, 1280, 64, 4, 0.0), (2, 1080, 1920, 96, 7, 0.0), (8, 360, 640, 48, 5, 0.0)]
    if len(sys.argv) > 1:   # one case: B H W D rho nan_band [reps]
        a = sys.argv[1:]
        cases = [(int(a[0]), int(a[1]), int(a[2]), int(a[3]), int(a[4]), float(a[5]))]
    from _clocks import run_with_clocks
    run_with_clocks(lambda: [print(json.dumps(bench(*c, reps=int(os.environ.get("REPS", "5")))), flush=True)
                             for c in cases], "k3_bench")
