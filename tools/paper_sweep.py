#!/usr/bin/env python3
"""The paper's own runtime experiments on B200:

* the operating point of P:231 / P:249 -- 1240x609, NCC 7x7 (varrho = 3),
  bilateral 9x9 (rho = 4), d_max = 30 (config "cP") -- as fps and Mde/s
  (Eq. 13: u_max v_max d_max / t * 1e-6), beside the paper's
  566.37 Mde/s / 25 fps on a GTX 1080 (context, not a target);
* the Fig. 4 sweep of runtime against varrho and rho ("about 50 fps
  at rho = 2", "the runtime doubles from rho = 2 to rho = 4").

Synthetic inputs (synth/, the cP generator).  Times are CUDA events around the
five C-ABI calls per frame batch, inputs resident in HBM, 3 warm-up runs.
Prints one JSON line per point."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402


def time_point(cfg, B, reps=10):
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    L = torch.from_numpy(left).cuda()
    R = torch.from_numpy(right).cuda()
    AB = torch.from_numpy(ab).cuda()
    pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    for _ in range(3):
        pipe.run(L, R, AB, with_wta=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pipe.run(L, R, AB, with_wta=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps / B
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    args = ap.parse_args()
    base = synth.get_config("cP")
    D = base.D
    for B in (1, args.batch):
        ms = time_point(base, B)
        print(json.dumps({"point": "paper operating point (P:231, P:249)", "config": "cP 1240x609 D=30 NCC 7x7 "
                          "bilateral 9x9", "batch": B, "ms_per_frame": ms, "fps": 1e3 / ms,
                          "mde_per_s": base.width * base.height * D / (ms * 1e-3) * 1e-6,
                          "paper_gtx1080": {"mde_per_s": 566.37, "fps": 25}}), flush=True)
    for rb in (1, 2, 3, 4):
        for ra in (1, 2, 3, 4, 5, 6, 7):
            cfg = synth.get_config("cP", rho_block=rb, rho_agg=ra)
            ms = time_point(cfg, args.batch, reps=5)
            print(json.dumps({"point": "Fig. 4 sweep", "varrho": rb, "rho": ra, "batch": args.batch,
                              "ms_per_frame": ms, "fps": 1e3 / ms,
                              "mde_per_s": cfg.width * cfg.height * D / (ms * 1e-3) * 1e-6}), flush=True)


if __name__ == "__main__":
    from _clocks import run_with_clocks
    run_with_clocks(main, "paper_sweep")
