#!/usr/bin/env python3
"""Times rsr_road_model (NEXT row f3) on the path's own c5 disparity maps (8-frame
batch) and checks it against oracle/road_model.py on one frame.  JSON lines."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402


def main():
    cfg = synth.get_config("c5")
    B = 8
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    pipe.run(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda(), torch.from_numpy(ab).cuda())
    for su, sv, nh in ((4, 4, 512), (2, 2, 1024), (8, 4, 256)):
        m = rsr.rsr_road_model(pipe.disparity, su, sv, nh, 0.5, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            rsr.rsr_road_model(pipe.disparity, su, sv, nh, 0.5, 1, model=m)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        mm = m.cpu().numpy()
        err = np.abs(mm[:, 0] - ab[:, 0]).max(), np.abs(mm[:, 1] - ab[:, 1]).max()
        n_samples = (cfg.height + sv - 1) // sv * ((cfg.width + su - 1) // su)
        print(json.dumps({"call": "rsr_road_model", "batch": B, "step_u": su, "step_v": sv, "n_hyp": nh,
                          "ms_per_batch": ms, "us_per_frame": 1e3 * ms / B,
                          "grid_samples_per_frame": n_samples,
                          "hypothesis_tests_per_s": B * n_samples * nh / (ms * 1e-3),
                          "max_abs_err_alpha_vs_generator": float(err[0]),
                          "max_abs_err_beta_vs_generator": float(err[1])}), flush=True)
    # oracle on one frame (CPU)
    from oracle import road_model as RM
    d0 = pipe.disparity[0].cpu().numpy()
    t0 = time.perf_counter()
    v, d = RM.grid_samples(d0, 4, 4)
    a, b, n, _ = RM.fit_road_model(v, d, 512, 0.5, 1)
    dt = time.perf_counter() - t0
    m = rsr.rsr_road_model(pipe.disparity[:1], 4, 4, 512, 0.5, 1).cpu().numpy()[0]
    print(json.dumps({"oracle_seconds_one_frame": dt, "oracle": [a, b, n], "gpu": m.tolist(),
                      "inliers_equal": int(m[2]) == n}), flush=True)


if __name__ == "__main__":
    from _clocks import run_with_clocks
    run_with_clocks(main, "road_bench")
