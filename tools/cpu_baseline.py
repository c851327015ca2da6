#!/usr/bin/env python3
"""The CPU-oracle schedule of SURVEY.md §8(d) ("Oracle timing, beside the GPU
run"), run on the GPU box's host cores: the fp64 NumPy oracle (oracle/, test
infrastructure) as it stands, single-threaded per process (OMP_NUM_THREADS=1).

* configs c1, c2, c3: one full frame each on 1 core;
* config c4: a 60-row band of one frame on 1 core (a full frame is ~3x c3's
  ~7 min), extrapolated by rows to a frame and labelled as such;
* config c5: a pool of P single-threaded worker processes, one full 1280x720
  frame each over frames 0..P-1, P = min(cores - 3, RAM / 5 GB); oracle fps =
  P / wall (the three single-frame jobs above run concurrently on their own
  cores).
Writes one JSON line per measurement to gpurun_out/cpu_baseline.jsonl."""
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _job(args):
    name, index, rows = args
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    import synth
    from oracle import rsr_oracle as O
    cfg = synth.get_config(name)
    f = synth.make_frame(cfg, index)
    r = None if rows is None else (cfg.height // 2 - rows // 2, cfg.height // 2 - rows // 2 + rows)
    t0 = time.perf_counter()
    O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg, rows=r, keep_volumes=False)
    t1 = time.perf_counter()
    return name, index, rows, t0, t1, cfg.height, cfg.width, cfg.D


def main():
    cores = len(os.sched_getaffinity(0))
    ram_gb = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30
    P = max(1, min(cores - 3, int(ram_gb // 5)))
    jobs = [("c1", 0, None), ("c2", 0, None), ("c3", 0, None), ("c4", 0, 60)] + [("c5", i, None) for i in range(P)]
    out = os.path.join(ROOT, "gpurun_out", "cpu_baseline.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    ctx = mp.get_context("spawn")
    with ctx.Pool(len(jobs)) as pool:
        res = pool.map(_job, jobs, chunksize=1)
    lines = []
    for name, index, rows, t0, t1, H, W, D in res:
        if name == "c5":
            continue
        dt = t1 - t0
        frac = 1.0 if rows is None else rows / H
        lines.append({"config": name, "cores": 1, "kind": "oracle", "seconds": dt,
                      "fps": frac / dt, "sample": "full frame" if rows is None else
                      f"{rows} of {H} rows of one frame, fps extrapolated by rows",
                      "mde_per_s": frac * W * H * D / dt * 1e-6})
    c5 = [r for r in res if r[0] == "c5"]
    wall = max(r[4] for r in c5) - min(r[3] for r in c5)
    H, W, D = c5[0][5], c5[0][6], c5[0][7]
    lines.append({"config": "c5", "cores": P, "kind": "oracle", "seconds": wall, "fps": P / wall,
                  "sample": f"pool of {P} single-threaded workers, one full frame each (frames 0..{P - 1}); "
                            f"host has {cores} cores, {ram_gb:.0f} GB",
                  "per_frame_s": [r[4] - r[3] for r in c5], "mde_per_s": P * W * H * D / wall * 1e-6})
    with open(out, "w") as fh:
        for ln in lines:
            fh.write(json.dumps(ln) + "\n")
            print(json.dumps(ln), flush=True)


if __name__ == "__main__":
    main()
