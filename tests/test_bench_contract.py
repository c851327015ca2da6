"""bench.py's reference arm (the fp64 oracle on a pool of host cores) prints the
JSON line of the contract: same metric/config keys as the GPU arm, impl,
cpu_baseline and a zero-copy e2e.  CPU only; a tiny bounded sample."""
import json

import bench


def test_reference_arm_line(capsys):
    bench.main(["--impl", "reference", "--steps", "1", "--warmup", "0", "--cpu-rows", "1", "--cpu-workers", "1"])
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "fps" and line["unit"] == "frames/s"
    assert line["higher_is_better"] is True and line["steps"] == 1 and line["warmup"] == 0
    assert line["value"] > 0 and line["dtype"] == "f64" and line["data"] == "synthetic"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # the config the driver compares with the GPU arm's
    assert line["config"] == bench.workload_config(bench.synth.get_config("c5"), bench.parse([]), 1)


def test_step_frames_cycle_the_rank_pool():
    # rank r of N owns frames [r * pool, (r + 1) * pool); steps cycle its pool in batches
    assert bench.step_frames(0, 16, 8, 0, 1) == list(range(8))
    assert bench.step_frames(1, 16, 8, 0, 1) == list(range(8, 16))
    assert bench.step_frames(2, 16, 8, 0, 1) == list(range(8))
    assert bench.step_frames(0, 16, 8, 1, 2) == list(range(16, 24))
