"""Small invocations of every kernel of the hot path for compute-sanitizer
(racecheck / synccheck / memcheck): config c1 (180x320, D=32) through the
pipeline (both general and clean K3 segments, nan maps) and a 16x16 frame
(D=5, tiny tiles: every border path), plus rho=8 (tiled K3) and the D=30 cP
slab (two-CTA K3 with 8-byte cp.async staging) on small frames."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1807_07433_b200 as rsr  # noqa: E402


def run(cfg, B=1):
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    pipe.run(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda(), torch.from_numpy(ab).cuda())
    torch.cuda.synchronize()
    return pipe


if __name__ == "__main__":
    run(synth.get_config("c1"))
    run(synth.get_config("c1", height=16, width=16, d_lo=-2, d_hi=2, rho_block=1, rho_agg=2, n_potholes=0))
    run(synth.get_config("c1", height=40, width=90, d_lo=-8, d_hi=7, rho_agg=8))
    run(synth.get_config("cP", height=48, width=160), B=2)
    print("sanitize cases ok")
