#!/usr/bin/env python3
"""Reconstruction-accuracy protocol of PAPER.md:198 on a synthetic scene with a
known-height "sample model" (NEXT row f4).

P:198: "we randomly select a region which includes one of the sample models ...
The four corners s1..s4 are interpolated into a ground plane ... we select some
random 3-D points p1..pn on the surface of the model and estimate the distances
between them and the road surface ... the reconstruction accuracy is
approximately 3 mm."

Scene (synth, box=...): c5 geometry (1280x720, f = 700 px, b = 0.12 m, road
d = 0.1 v + 30, so the box sits ~1.1-1.3 m from the camera), a box of height h
whose top face is the road plane raised by h (synth.box_disparity_gain).  The
whole path runs on the GPU (StereoPipeline: integer or interpolating warp);
corners = mean of the finite reconstructed points in a 9x9 patch at the four
corners of the region (box + 40 px margin); plane = rsr_plane_fit (GPU, TLS);
distances = rsr_plane_distance (GPU) of n random finite points on the box top
(12 px inside its edges).  Reported: mean / median / std of those distances and
the error mean - h, in mm.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BOX = (560, 380, 720, 480)


def measure_box_height(rsr, torch, h_box, seed=0, warp="integer", n_points=100, margin=40, box=BOX):
    cfg = synth.get_config("c5", random_plane=False, n_potholes=0, crack=False, seed=9000 + seed,
                           box=box + (h_box,))
    f = synth.make_frame(cfg)
    pipe = rsr.StereoPipeline(1, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg, warp=warp))
    ab = torch.tensor([[f.alpha, f.beta]], dtype=torch.float64, device="cuda")
    pipe.run(torch.from_numpy(f.left)[None].cuda(), torch.from_numpy(f.right)[None].cuda(), ab)
    u0, v0, u1, v1 = box
    xyz = pipe.xyz[0].cpu().numpy()
    corners = []
    for (cu, cv) in ((u0 - margin, v0 - margin), (u1 + margin, v0 - margin), (u0 - margin, v1 + margin),
                     (u1 + margin, v1 + margin)):
        patch = xyz[cv - 4:cv + 5, cu - 4:cu + 5].reshape(-1, 3)
        patch = patch[np.isfinite(patch).all(axis=1)]
        corners.append(patch.mean(axis=0))
    cor = torch.tensor(np.array(corners)[None], dtype=torch.float64, device="cuda")
    plane = rsr.rsr_plane_fit(cor)
    dist = rsr.rsr_plane_distance(plane, pipe.xyz)[0].cpu().numpy()
    rng = np.random.default_rng(seed)
    m = 12
    top = dist[v0 + m:v1 - m, u0 + m:u1 - m].ravel()
    top = top[np.isfinite(top)]
    pick = rng.choice(len(top), size=min(n_points, len(top)), replace=False)
    d = top[pick]
    road = dist[v0 - margin:v0 - 10, u0:u1].ravel()
    road = road[np.isfinite(road)]
    return {"h_mm": 1e3 * h_box, "warp": warp, "seed": seed, "n": int(len(d)),
            "mean_mm": 1e3 * float(d.mean()), "median_mm": 1e3 * float(np.median(d)),
            "std_mm": 1e3 * float(d.std()), "err_mm": 1e3 * float(d.mean() - h_box),
            "road_rms_mm": 1e3 * float(np.sqrt(np.mean(road ** 2))),
            "depth_m": float(np.nanmedian(xyz[v0:v1, u0:u1, 2])),
            "plane": plane[0].cpu().numpy().tolist()}


def main():
    import torch
    import paper_1807_07433_b200 as rsr
    out = os.path.join(ROOT, "gpurun_out", "accuracy.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    rows = []
    with open(out, "w") as fh:
        for warp in ("integer", "linear"):
            for h in (0.005, 0.010, 0.020, 0.040):
                for seed in range(4):
                    r = measure_box_height(rsr, torch, h, seed, warp)
                    rows.append(r)
                    fh.write(json.dumps(r) + "\n")
                    print(json.dumps(r), flush=True)
    for warp in ("integer", "linear"):
        e = np.array([r["err_mm"] for r in rows if r["warp"] == warp])
        s = np.array([r["std_mm"] for r in rows if r["warp"] == warp])
        print(json.dumps({"summary": warp, "mean_abs_err_mm": float(np.abs(e).mean()),
                          "max_abs_err_mm": float(np.abs(e).max()), "mean_point_std_mm": float(s.mean())}))


if __name__ == "__main__":
    main()
