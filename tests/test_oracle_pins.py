"""Pins of the fp64 oracle against facts other than itself (closed forms,
invariants, library routines, brute force, ground truth, the paper's printed
numbers).  CPU only (-m "not gpu").  Each test names the passage it pins.
"""
import math

import numpy as np
import pytest
from scipy import ndimage

import synth
from oracle import brute
from oracle import rsr_oracle as O


def rand_img(seed, h, w, lo=30, hi=225):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, size=(h, w)).astype(np.uint8)


# ---------------------------------------------------------------- warp
def test_road_shift_round_half_up():
    # reading 1: floor(alpha v + beta + 1/2); .5 boundaries round up
    s = O.road_shift(0.5, 0.0, 6)
    assert list(s) == [0, 1, 1, 2, 2, 3]
    assert list(O.road_shift(0.0, -2.5, 2)) == [-2, -2]
    assert list(O.road_shift(0.0, 2.4999, 1)) == [2]


def test_warp_identity_and_translation():
    t = rand_img(1, 8, 12)
    w, m, s = O.warp_target(t, 0.0, 0.0)
    assert np.array_equal(w, t) and m.all() and (s == 0).all()
    # shift right by 3: W(u) = T(u-3), left 3 columns invalid
    w, m, s = O.warp_target(t, 0.0, 3.0)
    assert np.array_equal(w[:, 3:], t[:, :-3])
    assert (m[:, :3] == 0).all() and (m[:, 3:] == 1).all() and (w[:, :3] == 0).all()
    # negative shift: right band invalid
    w, m, s = O.warp_target(t, 0.0, -2.0)
    assert np.array_equal(w[:, :-2], t[:, 2:]) and (m[:, -2:] == 0).all()


def test_warp_row_dependent():
    t = rand_img(2, 10, 20)
    w, m, s = O.warp_target(t, 0.3, 1.2)
    for v in range(10):
        sv = math.floor(0.3 * v + 1.2 + 0.5)
        assert s[v] == sv
        assert np.array_equal(w[v, sv:], t[v, :20 - sv])


# ---------------------------------------------------------------- NCC (Eqs. 3-5)
def test_block_stats_worked_example(golden):
    g = golden["block_stats_1_to_9"]
    img = np.array(g["block"], dtype=np.uint8)
    S, SS, ok = O.block_sums(img, 1)
    n = 9
    mu = S[1, 1] / n
    sigma = math.sqrt(SS[1, 1] / n - mu * mu)
    assert ok[1, 1] and not ok[0, 0]
    assert mu == g["mu"] and sigma == pytest.approx(g["sigma"], abs=1e-12)


def _ncc_all(left, warped, mask, rho_b, r):
    h, w = left.shape
    return O.ncc_at(left, warped, mask, rho_b, r, 0, h, 0, w)


def test_ncc_self_match_is_one_and_inverted_is_minus_one():
    L = rand_img(3, 16, 20)
    M = np.ones_like(L)
    c = _ncc_all(L, L, M, 2, 0)
    v = ~np.isnan(c)
    assert v.sum() == (16 - 4) * (20 - 4)
    assert np.allclose(c[v], 1.0, atol=1e-12)
    c = _ncc_all(L, (255 - L).astype(np.uint8), M, 2, 0)
    assert np.allclose(c[~np.isnan(c)], -1.0, atol=1e-12)


def test_ncc_shift_sign():
    # W(x) = L(x + 3): the left block at u matches the W block at u - 3, i.e. r = 3
    base = rand_img(4, 14, 40)
    L = base[:, 3:33].copy()
    W = base[:, 6:36].copy()
    M = np.ones_like(L)
    cl, _ = O.cost_volumes(L, W, M, 2, -5, 5)
    k = O.wta(cl)
    inner = k[2:-2, 10:-10]
    assert (inner == 3 - (-5)).all()  # r = 3 <=> k = r - d_lo


def test_ncc_affine_invariance_and_sign_flip():
    rng = np.random.default_rng(5)
    L = rng.integers(0, 101, size=(12, 16)).astype(np.uint8)
    R = rng.integers(0, 101, size=(12, 16)).astype(np.uint8)
    M = np.ones_like(L)
    c0 = _ncc_all(L, R, M, 1, 1)
    c1 = _ncc_all((2 * L.astype(int) + 10).astype(np.uint8), R, M, 1, 1)
    c2 = _ncc_all(L, (2 * R.astype(int) + 7).astype(np.uint8), M, 1, 1)
    c3 = _ncc_all(L, (200 - R.astype(int)).astype(np.uint8), M, 1, 1)
    v = ~np.isnan(c0)
    assert v.sum() > 50
    assert np.allclose(c1[v], c0[v], atol=1e-12)
    assert np.allclose(c2[v], c0[v], atol=1e-12)
    assert np.allclose(c3[v], -c0[v], atol=1e-12)


def test_ncc_is_pearson_correlation():
    # library routine: ZNCC of two blocks == np.corrcoef of the flattened blocks
    L = rand_img(6, 20, 24)
    R = rand_img(7, 20, 24)
    M = np.ones_like(L)
    for r, (v, u) in [(0, (5, 5)), (2, (9, 12)), (-3, (10, 8)), (4, (14, 17))]:
        c = O.ncc_at(L, R, M, 3, r, v, 1, u, 1)[0, 0]
        a = L[v - 3:v + 4, u - 3:u + 4].astype(float).ravel()
        b = R[v - 3:v + 4, u - r - 3:u - r + 4].astype(float).ravel()
        assert c == pytest.approx(np.corrcoef(a, b)[0, 1], abs=1e-12)


def test_ncc_invalid_cases():
    L = rand_img(8, 16, 16)
    R = rand_img(9, 16, 16)
    M = np.ones_like(L)
    L2 = L.copy()
    L2[4:9, 4:9] = 77          # constant 5x5 block centred at (6,6), rho_b=2
    c = _ncc_all(L2, R, M, 2, 0)
    assert np.isnan(c[6, 6]) and not np.isnan(c[6, 10])
    M2 = M.copy()
    M2[10, 3] = 0               # one warp-invalid pixel invalidates every block holding it
    c = _ncc_all(L, R, M2, 2, 1)  # W block centred at (v, u-1)
    assert np.isnan(c[10, 4]) and np.isnan(c[8, 6]) and not np.isnan(c[10, 7])
    c = _ncc_all(L, R, M, 2, 3)
    assert np.isnan(c[:, :5]).all() and not np.isnan(c[5, 5])   # right block leaves image
    assert np.isnan(c[:2]).all() and np.isnan(c[:, -2:]).all()   # left block leaves image


def test_dual_volume_identity():
    # C_L(u, v, d) == C_R(u - d, v, d), bitwise, for valid entries
    f = synth.make_frame(synth.get_config("c1", height=40, width=64))
    W, M, s = O.warp_target(f.right, 0.05, 10.0)
    cl, cr = O.cost_volumes(f.left, W, M, 2, -6, 5)
    for k in range(cl.shape[0]):
        r = -6 + k
        for u in range(64):
            up = u - r
            if 0 <= up < 64:
                a, b = cl[k, :, u], cr[k, :, up]
                assert np.array_equal(np.isnan(a), np.isnan(b))
                assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
            else:
                assert np.isnan(cl[k, :, u]).all()


# ---------------------------------------------------------------- aggregation (Eqs. 8-10)
def test_bilateral_weight_worked_example(golden):
    g = golden["omega_d_unit"]
    w = O.bilateral_weight(g["dx"], g["dy"], 50, 50, g["gamma_d"], 10.0)
    assert float(w) == pytest.approx(g["omega_d"], abs=1e-15)
    # range weight, literal exp(-diff^2/gamma_r^2) (reading 10, no factor 2)
    assert float(O.bilateral_weight(0, 0, 60, 50, 1.0, 10.0)) == pytest.approx(math.exp(-1.0), abs=1e-15)


def test_aggregate_rho0_identity_and_constant_fixed_point():
    rng = np.random.default_rng(10)
    X = rng.uniform(-1, 1, size=(3, 9, 11))
    X[1, 4, 5] = np.nan
    G = rand_img(11, 9, 11)
    A = O.aggregate(X, G, 0, 3.0, 10.0)
    assert np.array_equal(np.isnan(A), np.isnan(X))
    assert np.allclose(A[~np.isnan(A)], X[~np.isnan(X)], atol=1e-15)
    C = np.full((2, 9, 11), 0.7)
    A = O.aggregate(C, G, 3, 2.0, 5.0)
    assert np.allclose(A, 0.7, atol=1e-14)


def test_aggregate_convexity_and_nan_centre():
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, size=(4, 12, 14))
    X[rng.random(X.shape) < 0.15] = np.nan
    G = rand_img(13, 12, 14)
    rho = 2
    A = O.aggregate(X, G, rho, 2.0, 15.0)
    assert np.array_equal(np.isnan(A), np.isnan(X))
    for k in range(4):
        for v in range(12):
            for u in range(14):
                if np.isnan(A[k, v, u]):
                    continue
                win = X[k, max(0, v - rho):v + rho + 1, max(0, u - rho):u + rho + 1]
                assert np.nanmin(win) - 1e-14 <= A[k, v, u] <= np.nanmax(win) + 1e-14


def test_aggregate_gamma_r_inf_is_spatial_gaussian():
    # library routine: with omega_r == 1, Eq. (8) is a normalised Gaussian filter
    rng = np.random.default_rng(14)
    X = rng.uniform(-1, 1, size=(3, 15, 17))
    X[rng.random(X.shape) < 0.2] = np.nan
    G = rand_img(15, 15, 17)
    rho, gd = 3, 2.5
    A = O.aggregate(X, G, rho, gd, math.inf)
    yy, xx = np.mgrid[-rho:rho + 1, -rho:rho + 1]
    g = np.exp(-(xx ** 2 + yy ** 2) / gd ** 2)
    for k in range(3):
        V = (~np.isnan(X[k])).astype(float)
        X0 = np.where(V > 0, X[k], 0.0)
        ref = ndimage.correlate(X0 * V, g, mode="constant", cval=0.0) / \
            ndimage.correlate(V, g, mode="constant", cval=0.0)
        m = V > 0
        assert np.allclose(A[k][m], ref[m], atol=1e-12)


def test_aggregate_guide_step_edge():
    # closed form: across a guide step of height h the range weight is exp(-(h/gamma_r)^2)
    X = np.zeros((1, 7, 8))
    X[0, :, 4:] = 1.0
    G = np.zeros((7, 8), dtype=np.uint8)
    G[:, 4:] = 30
    gd, gr, rho = 2.0, 10.0, 1
    A = O.aggregate(X, G, rho, gd, gr)
    e = math.exp(-(30 / gr) ** 2)
    wd = lambda dx, dy: math.exp(-(dx * dx + dy * dy) / gd ** 2)
    same = sum(wd(dx, dy) for dy in (-1, 0, 1) for dx in (-1, 0))
    other = sum(wd(1, dy) for dy in (-1, 0, 1)) * e
    assert A[0, 3, 3] == pytest.approx(other / (same + other), abs=1e-14)


# ---------------------------------------------------------------- WTA, LRC
def test_wta_worked_examples_and_argmax(golden):
    for vals, k in golden["wta_examples"]["cases"]:
        A = np.array(vals, dtype=float)[:, None, None]
        assert O.wta(A)[0, 0] == k
    rng = np.random.default_rng(16)
    A = rng.uniform(-1, 1, size=(9, 6, 7))
    A[rng.random(A.shape) < 0.3] = np.nan
    A[:, 0, 0] = np.nan
    K = O.wta(A)
    ref = np.argmax(np.where(np.isnan(A), -np.inf, A), axis=0)
    ref[0, 0] = -1
    assert np.array_equal(K, ref)
    assert np.array_equal(O.wta(np.exp(3 * A)), K)   # strictly increasing transform


def test_lrc_properties():
    h, w = 6, 30
    k = np.full((h, w), 5)
    keep = O.lr_check(k, k, -2, 0)        # r = 3
    assert keep[:, 3:].all() and not keep[:, :3].any()
    kt = k.copy()
    kt[2, 10 - 3] = 9
    keep2 = O.lr_check(k, kt, -2, 1)
    assert not keep2[2, 10] and keep2[2, 11]
    kt[2, 10 - 3] = 6
    assert O.lr_check(k, kt, -2, 1)[2, 10] and not O.lr_check(k, kt, -2, 0)[2, 10]
    rng = np.random.default_rng(17)
    kr = rng.integers(-1, 8, size=(h, w))
    kl = rng.integers(-1, 8, size=(h, w))
    keep = O.lr_check(kl, kr, -2, 1)
    assert not keep[kl < 0].any()   # never resurrects


# ---------------------------------------------------------------- subpixel (Eq. 12)
def test_subpixel_worked_example_and_vertex(golden):
    g = golden["subpixel_example"]
    A = np.array([0.0, g["c_minus"], g["c0"], g["c_plus"], 0.0])[:, None, None]
    k = np.array([[2]])
    assert O.subpixel(A, k, 0)[0, 0] == pytest.approx(2 + g["offset"], abs=1e-15)
    rng = np.random.default_rng(18)
    for _ in range(1000):
        a = -rng.uniform(0.01, 2.0)
        k0 = rng.uniform(-0.5, 0.5)
        b = rng.uniform(-1, 1)
        vals = [a * (x - k0) ** 2 + b for x in (-1.0, 0.0, 1.0)]
        A = np.array([vals[0], vals[0], vals[1], vals[2], vals[2]])[:, None, None]
        rs = O.subpixel(A, np.array([[2]]), -2)[0, 0]
        assert rs == pytest.approx(k0, abs=1e-12)
        assert abs(rs) <= 0.5 + 1e-15


def test_subpixel_edges_keep_integer():
    A = np.array([0.9, 0.5, 0.2])[:, None, None]
    assert O.subpixel(A, np.array([[0]]), -1)[0, 0] == -1.0
    A = np.array([0.2, 0.5, 0.9])[:, None, None]
    assert O.subpixel(A, np.array([[2]]), -1)[0, 0] == 1.0
    A = np.array([np.nan, 0.9, 0.2])[:, None, None]
    assert O.subpixel(A, np.array([[1]]), 0)[0, 0] == 1.0


# ---------------------------------------------------------------- triangulation, Mde/s
def test_triangulation_worked_example(golden):
    g = golden["triangulation_example"]
    d = np.full((3, 5), g["d"])
    xyz = O.triangulate(d, g["focal"], g["baseline"], 2.0, 1.0, 1.0)
    assert np.allclose(xyz[..., 2], g["z"], atol=1e-15)
    assert xyz[1, 2, 0] == 0.0 and xyz[1, 2, 1] == 0.0   # principal point -> optical axis
    # back-projection round trip u = u0 + f X / Z, v = v0 + f Y / Z
    rng = np.random.default_rng(19)
    d = rng.uniform(5, 80, size=(6, 9))
    d[0, 0] = 0.5            # below d_min -> NaN
    xyz = O.triangulate(d, 700.0, 0.12, 4.0, 2.5, 1.0)
    vv, uu = np.mgrid[0:6, 0:9]
    m = ~np.isnan(xyz[..., 2])
    assert not m[0, 0]
    assert np.allclose((4.0 + 700.0 * xyz[..., 0] / xyz[..., 2])[m], uu[m], atol=1e-9)
    assert np.allclose((2.5 + 700.0 * xyz[..., 1] / xyz[..., 2])[m], vv[m], atol=1e-9)


def test_mde_per_second_paper_number(golden):
    for key in ("mdes_paper", "mdes_spec"):
        g = golden[key]
        assert O.mde_per_second(g["width"], g["height"], g["d_max"], g["seconds"]) == \
            pytest.approx(g["mdes"], abs=1e-9)


# ---------------------------------------------------------------- whole path
class _P:
    def __init__(self, **kw):
        self.__dict__.update(kw)


@pytest.mark.parametrize("seed,alpha,beta", [(21, 0.0, 0.0), (22, 0.1, 1.4), (23, -0.05, 2.0)])
def test_brute_force_agrees_16x16(seed, alpha, beta):
    left, right = synth.tiny_pair(seed, 16, 16, shift=2)
    p = _P(d_lo=-1, d_hi=3, rho_block=1, rho_agg=2, gamma_d=2.0, gamma_r=12.0, lrc_tol=1,
           focal=700.0, baseline=0.12)
    vec = O.run_pipeline(left, right, alpha, beta, p)
    bf = brute.run(left, right, alpha, beta, 1, 2, -1, 3, 2.0, 12.0, 1)

    def eq(a, b, tol=1e-12):
        a, b = np.asarray(a, float), np.asarray(b, float)
        assert a.shape == b.shape
        assert np.array_equal(np.isnan(a), np.isnan(b))
        assert np.allclose(a[~np.isnan(a)], b[~np.isnan(b)], atol=tol)

    eq(vec["warped"], bf["warped"], 0)
    eq(vec["cost_ref"], bf["cost_ref"])
    eq(vec["cost_tar"], bf["cost_tar"])
    eq(vec["agg_ref"], bf["agg_ref"])
    eq(vec["agg_tar"], bf["agg_tar"])
    eq(vec["k_ref"], bf["k_ref"], 0)
    eq(vec["k_tar"], bf["k_tar"], 0)
    eq(vec["disparity"], bf["disparity"])
    eq(vec["xyz"], bf["xyz"])
    assert np.isfinite(vec["disparity"]).sum() > 20


def test_row_band_equals_full_image():
    cfg = synth.get_config("c1", height=48, width=96)
    f = synth.make_frame(cfg)
    full = O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg)
    band = O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg, rows=(20, 27))
    for key in ("agg_ref", "agg_tar", "cost_ref"):
        a, b = full[key][:, 20:27], band[key]
        assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    for key in ("k_ref", "k_tar"):
        assert np.array_equal(full[key][20:27], band[key])
    a, b = full["disparity"][20:27], band["disparity"]
    assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    a, b = full["xyz"][20:27], band["xyz"]
    assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])


def _eval_region(cfg, f, s):
    h, w = cfg.height, cfg.width
    m = cfg.rho_block + cfg.rho_agg + 2
    vv, uu = np.mgrid[0:h, 0:w]
    return (vv >= m) & (vv < h - m) & (uu >= s[vv] + m) & (uu < w - m) & ~f.gt_exclude


def test_plane_accuracy_against_ground_truth():
    # SURVEY §8(c) "Whole pipeline, accuracy": pure plane, RMS <= 0.25 px, >= 95 % valid
    cfg = synth.get_config("c1", n_potholes=0)
    f = synth.make_frame(cfg)
    res = O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg, keep_volumes=False)
    region = _eval_region(cfg, f, res["shift"])
    d = res["disparity"][region]
    valid = ~np.isnan(d)
    assert valid.mean() >= 0.95
    err = d[valid] - f.d_gt[region][valid]
    assert math.sqrt(np.mean(err ** 2)) <= 0.25


def test_self_match_integer_zero():
    cfg = synth.get_config("c1", height=40, width=80)
    f = synth.make_frame(cfg)
    res = O.run_pipeline(f.left, f.left, 0.0, 0.0, cfg, keep_volumes=False)
    k = res["k_ref"]
    ok = k >= 0
    assert ok.sum() > 1000
    assert (k[ok] == -cfg.d_lo).all()
    d = res["disparity"]
    assert np.nanmax(np.abs(d)) <= 0.5
