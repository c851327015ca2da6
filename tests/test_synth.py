"""Seeded generator (synth/): determinism and the BASELINE.json workload recipe."""
import numpy as np

import synth


def test_same_seed_same_bytes():
    cfg = synth.get_config("c1")
    a, b = synth.make_frame(cfg), synth.make_frame(cfg)
    assert np.array_equal(a.left, b.left) and np.array_equal(a.right, b.right)
    c = synth.make_frame(cfg, index=1)
    assert not np.array_equal(a.left, c.left)


def test_config_shapes_and_ranges():
    for name, (h, w, D) in {"c1": (180, 320, 32), "c2": (360, 640, 48), "c3": (720, 1280, 64),
                            "c4": (1080, 1920, 96), "c5": (720, 1280, 64), "cP": (609, 1240, 30)}.items():
        cfg = synth.get_config(name)
        assert (cfg.height, cfg.width, cfg.D) == (h, w, D)
    f = synth.make_frame(synth.get_config("c1"))
    assert f.left.dtype == np.uint8 and f.left.shape == (180, 320)
    assert 20 < f.left.min() and f.left.max() < 240
    # plane d(v) = 0.05 v + 10 plus potholes (amplitude -1.5)
    assert f.d_gt.max() <= 0.05 * 179 + 10 + 1e-9 and f.d_gt.min() >= 10 - 1.5 - 1e-9


def test_config5_random_plane_per_frame():
    cfg = synth.get_config("c5", height=64, width=128)
    a, b = synth.make_frame(cfg, 0), synth.make_frame(cfg, 7)
    for f in (a, b):
        assert 0.08 <= f.alpha <= 0.12 and 25 <= f.beta <= 35
    assert a.alpha != b.alpha
