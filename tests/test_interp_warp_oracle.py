"""Pins of the interpolating-warp oracle (oracle/interp_warp.py; SURVEY §8(f) f2,
DESIGN.md reading 21) against facts other than itself: identity and integer
translation (= 256 x the integer warp), SPEC's analytic ramp example,
np.interp on the quantised position, the shift-quantisation bound, the
rounding rule at 1/512 boundaries, scale invariance of Eq. (3) (np.corrcoef on
the real-valued interpolated blocks), ground truth on a plane with a
fractional intercept, and row-band = full-image.  CPU only."""
import math

import numpy as np
import pytest

import synth
from oracle import interp_warp as IW
from oracle import rsr_oracle as O


def rand_img(seed, h, w, lo=30, hi=225):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, size=(h, w)).astype(np.uint8)


def test_identity_and_integer_translation_equal_256x_integer_warp():
    t = rand_img(1, 8, 12)
    w, m, tq = IW.warp_target_linear(t, 0.0, 0.0)
    assert w.dtype == np.uint16 and np.array_equal(w, 256 * t.astype(np.uint16)) and m.all()
    assert (tq == 0).all()
    for beta in (3.0, -2.0, 0.0):
        w, m, tq = IW.warp_target_linear(t, 0.0, beta)
        wi, mi, si = O.warp_target(t, 0.0, beta)
        assert np.array_equal(m, mi)
        assert np.array_equal(w, 256 * wi.astype(np.uint16))
        assert np.array_equal(tq, si.astype(np.float64))


def test_spec_ramp_example():
    # s(v) = 2.5 on a horizontal ramp i(x) = 4x -> output(u) = 4u - 10 inside
    T = np.tile((4 * np.arange(60)).astype(np.uint8), (3, 1))
    w, m, tq = IW.warp_target_linear(T, 0.0, 2.5)
    assert (tq == 2.5).all()
    u = np.arange(60)
    inside = (u >= 3)           # x = u - 2.5 >= 0 needs x0 >= 0 and x0 + 1 <= 59
    assert (m[:, inside] == 1).all() and (m[:, ~inside] == 0).all()
    assert np.array_equal(w[:, inside] / 256.0, np.tile(4.0 * u[inside] - 10.0, (3, 1)))


@pytest.mark.parametrize("alpha,beta", [(0.013, 3.37), (-0.021, 5.91), (0.1, -2.2)])
def test_interpolation_equals_np_interp_at_quantised_position(alpha, beta):
    t = rand_img(2, 24, 40)
    w, m, tq = IW.warp_target_linear(t, alpha, beta)
    tt = alpha * np.arange(24) + beta
    assert np.all(np.abs(tq - tt) <= 1.0 / 512 + 1e-15)
    assert np.all(tq * 256 == np.round(tq * 256))
    xs = np.arange(40, dtype=np.float64)
    for v in range(24):
        x = xs - tq[v]
        ok = (x >= 0) & (x <= 39)
        assert np.array_equal(m[v] == 1, ok)
        ref = np.interp(x[ok], xs, t[v].astype(np.float64))
        assert np.array_equal(w[v, ok] / 256.0, ref)
        assert (w[v, ~ok] == 0).all()


def test_quantisation_rounds_half_up():
    T = rand_img(3, 1, 10)
    # t = -1/512 -> x = 1/512 at u = 0 -> 256 f + 1/2 = 1 exactly -> q = 1
    _, _, tq = IW.warp_target_linear(T, 0.0, -1.0 / 512)
    assert tq[0] == -1.0 / 256
    # just below the boundary rounds down
    _, _, tq = IW.warp_target_linear(T, 0.0, -0.999 / 512)
    assert tq[0] == 0.0
    # q = 256 carries into x0
    _, _, tq = IW.warp_target_linear(T, 0.0, 1.0 / 1024)
    assert tq[0] == 0.0


def test_ncc_on_fixed_point_is_pearson_of_interpolated_blocks():
    L = rand_img(4, 20, 30)
    T = rand_img(5, 20, 30)
    w, m, tq = IW.warp_target_linear(T, 0.0, 1.3)
    cl, cr = O.cost_volumes(L, w, m, 2, -2, 2)
    rng = np.random.default_rng(0)
    checked = 0
    for _ in range(40):
        k = int(rng.integers(0, 5))
        r = -2 + k
        v = int(rng.integers(2, 18))
        u = int(rng.integers(2, 28))
        c = cl[k, v, u]
        if np.isnan(c):
            continue
        a = L[v - 2:v + 3, u - 2:u + 3].astype(float).ravel()
        b = (w[v - 2:v + 3, u - r - 2:u - r + 3] / 256.0).ravel()
        assert c == pytest.approx(np.corrcoef(a, b)[0, 1], abs=1e-12)
        checked += 1
    assert checked > 20
    # dual identity holds on the fixed-point images too
    for k in range(5):
        r = -2 + k
        for u in range(30):
            if 0 <= u - r < 30:
                a, b = cl[k, :, u], cr[k, :, u - r]
                assert np.array_equal(np.isnan(a), np.isnan(b))
                assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


def test_plane_with_fractional_intercept_against_ground_truth():
    cfg = synth.get_config("c1", n_potholes=0, beta=10.37, alpha=0.0513)
    f = synth.make_frame(cfg)
    res = IW.run_pipeline_linear(f.left, f.right, f.alpha, f.beta, cfg, keep_volumes=False)
    h, w = cfg.height, cfg.width
    mm = cfg.rho_block + cfg.rho_agg + 2
    vv, uu = np.mgrid[0:h, 0:w]
    region = (vv >= mm) & (vv < h - mm) & (uu >= np.ceil(res["shift"][vv]) + mm) & (uu < w - mm)
    d = res["disparity"][region]
    valid = ~np.isnan(d)
    assert valid.mean() >= 0.95
    assert math.sqrt(np.mean((d[valid] - f.d_gt[region][valid]) ** 2)) <= 0.25


def test_linear_row_band_equals_full_image():
    cfg = synth.get_config("c1", height=40, width=80, beta=7.6)
    f = synth.make_frame(cfg)
    full = IW.run_pipeline_linear(f.left, f.right, f.alpha, f.beta, cfg)
    band = IW.run_pipeline_linear(f.left, f.right, f.alpha, f.beta, cfg, rows=(15, 21))
    for key in ("agg_ref", "agg_tar"):
        a, b = full[key][:, 15:21], band[key]
        assert np.array_equal(a, b, equal_nan=True)
    assert np.array_equal(full["disparity"][15:21], band["disparity"], equal_nan=True)


def test_self_match_fractional_zero_shift():
    cfg = synth.get_config("c1", height=40, width=80)
    f = synth.make_frame(cfg)
    res = IW.run_pipeline_linear(f.left, f.left, 0.0, 0.0, cfg, keep_volumes=False)
    k = res["k_ref"]
    assert (k[k >= 0] == -cfg.d_lo).all() and (k >= 0).sum() > 1000
