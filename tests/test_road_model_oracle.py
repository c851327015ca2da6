"""Pins of the road-model oracle (oracle/road_model.py, NEXT row f3):
closed forms, library routines, robustness and the synthetic road plane."""
import numpy as np

import synth
from oracle import road_model as RM


def test_splitmix64_reference_values():
    # splitmix64 output for state 0 is the published first value 0xE220A8397B1DCDAF
    assert RM.splitmix64(0) == 0xE220A8397B1DCDAF
    assert RM.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_noiseless_line_recovered_exactly():
    v = np.arange(0, 720, 3, dtype=np.float64)
    d = 0.1 * v + 30.0
    a, b, n, _ = RM.fit_road_model(v, d, 64, 1.0, 7)
    assert n == len(v)
    assert abs(a - 0.1) < 1e-12 and abs(b - 30.0) < 1e-9


def test_refit_equals_polyfit_on_consensus():
    rng = np.random.default_rng(3)
    v = rng.uniform(0, 700, 500)
    d = 0.08 * v + 22.0 + rng.normal(0, 0.3, 500)
    a, b, n, h = RM.fit_road_model(v, d, 128, 1.0, 11)
    i, j = RM.draw_pair(11, h, len(v))
    a0 = (d[j] - d[i]) / (v[j] - v[i])
    m = RM.consensus(v, d, a0, d[i] - a0 * v[i], np.float32(1.0))
    pa, pb = np.polyfit(v[m], d[m], 1)
    assert n == m.sum()
    assert abs(a - pa) < 1e-10 and abs(b - pb) < 1e-7


def test_gross_outliers_fifty_seeds():
    # S:553 as an idea: 30 % gross outliers, 50 seeded trials, recovery within 1e-3 px
    for seed in range(50):
        rng = np.random.default_rng(1000 + seed)
        v = rng.uniform(0, 720, 400)
        d = 0.12 * v + 35.0
        out = rng.random(400) < 0.3
        d[out] = rng.uniform(0, 150, out.sum())
        a, b, n, _ = RM.fit_road_model(v, d, 256, 0.5, seed)
        assert abs(a - 0.12) < 1e-3 and abs(b - 35.0) < 1e-3 * 720, (seed, a, b)
        assert n >= (~out).sum()


def test_degenerate_inputs():
    assert np.isnan(RM.fit_road_model(np.array([5.0]), np.array([1.0]), 8, 1.0, 0)[0])
    # all samples on one row: every hypothesis is degenerate
    v = np.full(10, 3.0)
    a, b, n, h = RM.fit_road_model(v, np.arange(10.0), 16, 1.0, 0)
    assert np.isnan(a) and n == 0 and h == -1


def test_draw_pair_distinct_and_in_range():
    for h in range(1000):
        i, j = RM.draw_pair(5, h, 7)
        assert 0 <= i < 7 and 0 <= j < 7 and i != j


def test_synthetic_road_plane_recovered_from_ground_truth():
    # S:470 as an idea: the fit on ground-truth disparities recovers Eq. (2)'s
    # coefficients of the generator's plane; potholes and the crack are outliers
    # (a 1e-6 px consensus band also rejects the Gaussian tails of the potholes)
    cfg = synth.get_config("c2")
    f = synth.make_frame(cfg)
    v, d = RM.grid_samples(f.d_gt, 8, 4)
    a, b, n, _ = RM.fit_road_model(v, d, 256, 1e-6, 1)
    assert abs(a - f.alpha) < 1e-8 and abs(b - f.beta) < 1e-6
    assert n > 0.5 * len(v)


def test_roll_plane_fit_closed_form():
    # plane d = g0 + g1 u + g2 v with a known roll: the fit recovers it exactly and
    # gamma = arctan(-g1 / g2); equals numpy lstsq on the same samples
    h, w = 60, 90
    vv, uu = np.mgrid[0:h, 0:w]
    g0, g1, g2 = 12.0, -0.004, 0.11
    d = (g0 + g1 * uu + g2 * vv).astype(np.float64)
    d[::7, ::5] = np.nan
    G0, G1, G2, gam, n = RM.roll_plane_fit(d, 10, 80, 20, 60)
    assert abs(G1 - g1) < 1e-12 and abs(G2 - g2) < 1e-12 and abs(G0 - g0) < 1e-9
    assert abs(gam - np.arctan(-g1 / g2)) < 1e-12
    ok = np.isfinite(d[20:60, 10:80])
    A = np.stack([np.ones(ok.sum()), uu[20:60, 10:80][ok], vv[20:60, 10:80][ok]], 1)
    rng = np.random.default_rng(0)
    noisy = d[20:60, 10:80][ok] + rng.normal(0, 0.1, ok.sum())
    dn = d.copy()
    dn[20:60, 10:80][ok] = noisy
    ref = np.linalg.lstsq(A, noisy, rcond=None)[0]
    N0, N1, N2, _, _ = RM.roll_plane_fit(dn, 10, 80, 20, 60)
    assert np.allclose([N0, N1, N2], ref, rtol=1e-9, atol=1e-12)
    assert np.isnan(RM.roll_plane_fit(np.full((5, 5), np.nan), 0, 5, 0, 5)[0])
