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


def test_box_scene_geometry_height_is_exact():
    """The accuracy scene's box (NEXT f4): back-projecting the generator's
    ground-truth disparities (reading 15) puts the box top exactly h above the
    total-least-squares road plane of the surrounding road points."""
    import numpy as np
    from oracle import plane_eval as PE
    from oracle import rsr_oracle as O
    h_box = 0.02
    cfg = synth.get_config("c5", random_plane=False, n_potholes=0, crack=False,
                           box=(560, 380, 720, 480, h_box))
    f = synth.make_frame(cfg)
    H, W = cfg.height, cfg.width
    xyz = O.triangulate(f.d_gt, cfg.focal, cfg.baseline, (W - 1) / 2.0, (H - 1) / 2.0, 1.0)
    road = xyz[[340, 340, 520, 520], [520, 760, 520, 760]]
    plane = PE.fit_plane(road)
    top = xyz[400:460, 580:700].reshape(-1, 3)
    dist = PE.point_plane_distance(plane, top)
    assert np.allclose(dist, h_box, atol=1e-9)
    rest = xyz[300:360, 100:300].reshape(-1, 3)
    assert np.allclose(PE.point_plane_distance(plane, rest), 0.0, atol=1e-9)


def test_sequence_scrolls_and_drifts():
    import numpy as np
    fr = synth.make_sequence(synth.get_config("c1"), 3, scroll=3)
    # content moves down by 3 rows per frame (only the sensor noise differs)
    assert np.abs(fr[1].left[3:].astype(int) - fr[0].left[:-3].astype(int)).mean() < 3.0
    assert np.abs(fr[1].left.astype(int) - fr[0].left.astype(int)).mean() > 10.0
    assert fr[2].alpha > fr[1].alpha > fr[0].alpha
