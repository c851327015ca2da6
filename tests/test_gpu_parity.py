"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by
element on the same seeded inputs, at every stage boundary.

Tolerances (BASELINE.json north_star):
  warp / validity / shift      bitwise
  NCC volumes                  |dc| <= 1e-4, identical NaN masks
  aggregated volumes           |dA| <= 1e-4 * max(|A|, 0.1), identical NaN masks
  WTA k_L                      equal on >= 99.9 % of oracle-valid pixels; each
                               mismatch has oracle top-two within 1e-5
  subpixel disparity           |dd| <= 1e-3 px where k_L and the LR decision agree
  3-D points                   |dp| / |p| <= 1e-4 on the same pixels
Full-size configs (c3, c4, c5) run the whole frame on the GPU in the launch
configuration bench.py times and compare on oracle row bands (the oracle
computes a band exactly as the full image, tests/test_oracle_pins.py).
"""
import math
import zlib

import numpy as np
import pytest

import synth
from oracle import rsr_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


def run_gpu(rsr, left, right, ab, cfg, nan_maps=True):
    """Run the five C-ABI calls on a [B,H,W] batch; return numpy results."""
    dev = "cuda"
    L = torch.from_numpy(np.ascontiguousarray(left)).to(dev)
    R = torch.from_numpy(np.ascontiguousarray(right)).to(dev)
    if L.dim() == 2:
        L, R = L[None], R[None]
    AB = torch.tensor(np.asarray(ab, dtype=np.float64).reshape(-1, 2), device=dev)
    W_, M_, S_ = rsr.rsr_warp(R, AB)
    cl, cr, nl, nr = rsr.rsr_cost_volume(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi,
                                         with_nan_maps=nan_maps)
    al = rsr.rsr_aggregate(cl, L, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nl)
    ar = rsr.rsr_aggregate(cr, W_, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nr)
    d, kl, kr = rsr.rsr_disparity(al, ar, S_, cfg.d_lo, cfg.d_hi, cfg.lrc_tol, True, with_wta=True)
    xyz = rsr.rsr_reconstruct(d, cfg.focal, cfg.baseline, d_min=1.0)
    torch.cuda.synchronize()
    g = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
    return dict(warped=g(W_), mask=g(M_), shift=g(S_), cost_ref=g(cl), cost_tar=g(cr),
                nan_ref=g(nl), nan_tar=g(nr), agg_ref=g(al), agg_tar=g(ar), disparity=g(d),
                k_ref=g(kl), k_tar=g(kr), xyz=g(xyz))


def to_dhw(v):
    """GPU [H,W,D] -> oracle [D,H,W]"""
    return np.moveaxis(v, -1, 0)


def top_two_gap(agg):
    if agg.shape[0] < 2:          # D = 1: a single candidate, never a tie
        return np.full(agg.shape[1:], np.inf)
    a = np.where(np.isnan(agg), -np.inf, agg)
    s = np.sort(a, axis=0)
    with np.errstate(invalid="ignore"):
        gap = s[-1] - s[-2]
    return np.where(np.isnan(gap), np.inf, gap)


def compare(gpu, ora, rows, cfg, b=0, label=""):
    """Compare one frame's GPU results (full frame) with the oracle on rows (r0, r1)."""
    r0, r1 = rows
    rep = {}
    # NCC volumes
    for key in ("cost_ref", "cost_tar"):
        g = to_dhw(gpu[key][b])[:, r0:r1]
        o = ora[key]
        assert np.array_equal(np.isnan(g), np.isnan(o)), f"{label} {key}: NaN masks differ"
        m = ~np.isnan(o)
        err = np.abs(g[m] - o[m]).max() if m.any() else 0.0
        rep[key] = err
        assert err <= 1e-4, f"{label} {key}: max |dc| = {err}"
    # aggregated volumes
    for key in ("agg_ref", "agg_tar"):
        g = to_dhw(gpu[key][b])[:, r0:r1]
        o = ora[key]
        assert np.array_equal(np.isnan(g), np.isnan(o)), f"{label} {key}: NaN masks differ"
        m = ~np.isnan(o)
        rel = np.abs(g[m] - o[m]) / np.maximum(np.abs(o[m]), 0.1)
        rep[key] = rel.max() if m.any() else 0.0
        assert rep[key] <= 1e-4, f"{label} {key}: max rel |dA| = {rep[key]}"
    # WTA
    gap_l = top_two_gap(ora["agg_ref"])
    gap_r = top_two_gap(ora["agg_tar"])
    for key, gap in (("k_ref", gap_l), ("k_tar", gap_r)):
        g = gpu[key][b][r0:r1].astype(np.int64)
        o = ora[key]
        valid = o >= 0
        mism = g != o
        assert not (mism & ~valid).any(), f"{label} {key}: mismatch where oracle has no valid k"
        frac = 1.0 - mism[valid].mean() if valid.any() else 1.0
        rep[key + "_agree"] = frac
        assert frac >= 0.999, f"{label} {key}: agreement {frac}"
        assert (gap[mism] <= 1e-5).all(), f"{label} {key}: mismatch at a non-tie {gap[mism].max()}"
    # disparity and points where k_L and LR decision agree
    gd = gpu["disparity"][b][r0:r1]
    od = ora["disparity"]
    kl_ok = gpu["k_ref"][b][r0:r1] == ora["k_ref"]
    # pixels whose LR decision could legitimately differ: k_L or the k_R it reads differ
    W = od.shape[1]
    uu = np.arange(W)[None, :]
    up = np.clip(uu - (ora["k_ref"] + cfg.d_lo), 0, W - 1)
    kr_read_ok = np.take_along_axis(gpu["k_tar"][b][r0:r1], up, 1) == np.take_along_axis(ora["k_tar"], up, 1)
    same = kl_ok & kr_read_ok
    assert np.array_equal(np.isnan(gd[same]), np.isnan(od[same])), f"{label}: LR decisions differ"
    m = same & ~np.isnan(od)
    err = np.abs(gd[m] - od[m])
    rep["disp_max"] = err.max() if m.any() else 0.0
    rep["disp_valid_frac"] = (~np.isnan(od)).mean()
    bad = err > 1e-3
    if bad.any():
        # tolerated only where the oracle's top-two aggregated costs are a near-tie
        assert (gap_l[m][bad] <= 1e-5).all(), f"{label}: subpixel |dd| = {err.max()} at non-tie"
    gx = gpu["xyz"][b][r0:r1][m]
    ox = ora["xyz"][m]
    fin = np.isfinite(ox).all(axis=1)
    relp = np.linalg.norm(gx[fin] - ox[fin], axis=1) / np.linalg.norm(ox[fin], axis=1)
    ok = err[fin] <= 1e-3
    rep["xyz_rel"] = relp[ok].max() if ok.any() else 0.0
    assert rep["xyz_rel"] <= 1e-4, f"{label}: xyz rel {rep['xyz_rel']}"
    return rep


def check_warp(gpu, right, ab, b=0):
    Wo, Mo, So = O.warp_target(right, ab[0], ab[1])
    assert np.array_equal(gpu["warped"][b], Wo)
    assert np.array_equal(gpu["mask"][b], Mo)
    assert np.array_equal(gpu["shift"][b].astype(np.int64), So)


@pytest.mark.parametrize("name,over", [("c1", {}), ("c2", {}), ("c1", {"d_lo": -1, "d_hi": 1}),
                                       ("c1", {"d_lo": 0, "d_hi": 0})])
def test_parity_full_frame(rsr, name, over):
    cfg = synth.get_config(name, **over)
    f = synth.make_frame(cfg)
    gpu = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    check_warp(gpu, f.right, (f.alpha, f.beta))
    ora = O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg)
    rep = compare(gpu, ora, (0, cfg.height), cfg, label=name)
    print(name, rep)
    # nan maps: bit 0 = some k NaN, bit 1 = some k finite, bits 2 / 3 = some k NaN
    # in the low / high disparity half, bit 7 = half bits present (include/rsr.h)
    D = cfg.D
    h0 = ((D + 7) & ~7) // 2
    for key, vk in (("nan_ref", "cost_ref"), ("nan_tar", "cost_tar")):
        v = np.isnan(gpu[vk][0])
        expect = (v.any(axis=-1).astype(np.uint8) | (2 * (~v).any(axis=-1)).astype(np.uint8)
                  | (4 * v[..., :h0].any(axis=-1)).astype(np.uint8)
                  | (8 * v[..., h0:].any(axis=-1)).astype(np.uint8) | np.uint8(0x80))
        assert np.array_equal(gpu[key][0], expect)


@pytest.mark.parametrize("name,bands", [
    ("c3", [(0, 7), (356, 364), (712, 720)]),
    ("c4", [(0, 5), (537, 543), (1075, 1080)]),
])
def test_parity_full_size_row_bands(rsr, name, bands):
    cfg = synth.get_config(name)
    f = synth.make_frame(cfg)
    gpu = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    check_warp(gpu, f.right, (f.alpha, f.beta))
    for rows in bands:
        ora = O.run_pipeline(f.left, f.right, f.alpha, f.beta, cfg, rows=rows)
        rep = compare(gpu, ora, rows, cfg, label=f"{name}{rows}")
        print(name, rows, rep)


def test_parity_config5_frames_batched(rsr):
    cfg = synth.get_config("c5")
    idx = [0, 1, 255]
    left, right, ab = synth.make_batch(cfg, idx)
    gpu = run_gpu(rsr, left, right, ab, cfg)
    for b, i in enumerate(idx):
        check_warp(gpu, right[b], ab[b], b)
        rows = (300 + 50 * b, 306 + 50 * b)
        ora = O.run_pipeline(left[b], right[b], ab[b][0], ab[b][1], cfg, rows=rows)
        compare(gpu, ora, rows, cfg, b=b, label=f"c5[{i}]")


def pipeline_parity(rsr, cfg, B, picks, bitwise_rerun=False):
    """Run StereoPipeline (the launch bench.py times) over a B-frame batch of cfg and
    compare oracle row bands of the picked frames.  picks: [(frame, (r0, r1))]."""
    left, right, ab = synth.make_batch(cfg, list(range(B)))
    L = torch.from_numpy(left).cuda()
    R = torch.from_numpy(right).cuda()
    AB = torch.from_numpy(ab).cuda()
    pipe = rsr.StereoPipeline(B, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    pipe.run(L, R, AB, with_wta=True)
    torch.cuda.synchronize()
    g = lambda t: t.cpu().numpy()  # noqa: E731
    gpu = dict(warped=g(pipe.warped), mask=g(pipe.valid), shift=g(pipe.shift), cost_ref=g(pipe.vol_ref),
               cost_tar=g(pipe.vol_tar), agg_ref=g(pipe.agg_ref), agg_tar=g(pipe.agg_tar),
               disparity=g(pipe.disparity), k_ref=g(pipe.wta_ref), k_tar=g(pipe.wta_tar), xyz=g(pipe.xyz))
    for b, rows in picks:
        check_warp(gpu, right[b], ab[b], b)
        ora = O.run_pipeline(left[b], right[b], ab[b][0], ab[b][1], cfg, rows=rows)
        rep = compare(gpu, ora, rows, cfg, b=b, label=f"{cfg.name} D={cfg.D} [{b}]{rows}")
        print(cfg.name, cfg.D, b, rows, rep)
    if bitwise_rerun:
        d0 = pipe.disparity.clone()
        pipe.run(L, R, AB, with_wta=True)
        torch.cuda.synchronize()
        assert torch.equal(torch.nan_to_num(d0, nan=-7.0), torch.nan_to_num(pipe.disparity, nan=-7.0))


def chunk_edge_bands(rsr, cfg, B, half=3):
    """Row bands straddling K3's real row-chunk edges for this launch (R from the
    library's own plan for the pipeline's concurrency of 2), plus the first and
    last rows of the image."""
    R = rsr.rsr_aggregate_rows(B, cfg.height, cfg.width, cfg.D, cfg.rho_agg, concurrency=2)
    assert 8 <= R < cfg.height, R
    edges = list(range(R, cfg.height, R))
    bands = [(0, 2 * half)] + [(e - half, e + half) for e in edges[:2]] + [(cfg.height - 2 * half, cfg.height)]
    return R, bands


def test_parity_bench_launch_configuration(rsr):
    """The exact launch bench.py times: StereoPipeline over an 8-frame c5 batch (the
    batch size picks K3's row chunking and grid); row bands straddling the real K3
    chunk edges (R from rsr_aggregate_rows: 240 at c5 / B = 8 / concurrency 2) of
    several frames against the oracle, and a bitwise rerun."""
    cfg = synth.get_config("c5")
    R, bands = chunk_edge_bands(rsr, cfg, 8)
    picks = [(b, rows) for b, rows in zip((0, 3, 5, 7), bands)]
    pipeline_parity(rsr, cfg, 8, picks, bitwise_rerun=True)


def test_parity_paper_operating_point_full_size(rsr):
    """The paper's operating point cP (1240x609, d_max = 30, 7x7 NCC, 9x9
    bilateral) in the 8-frame launch tools/paper_sweep.py times: the two-CTA
    small-slab K3 with 8-byte cp.async staging (D = 30 = 2 mod 4) and R sized for
    H = 609; bands at the real chunk edges."""
    cfg = synth.get_config("cP")
    R, bands = chunk_edge_bands(rsr, cfg, 8)
    picks = [(b, rows) for b, rows in zip((0, 2, 6, 7), bands)]
    pipeline_parity(rsr, cfg, 8, picks)


@pytest.mark.parametrize("d_lo,d_hi", [(-3, 2), (-4, 3), (-6, 5)])
def test_parity_restricted_band_full_size(rsr, d_lo, d_hi):
    """Restricted search ranges at c5 size in the 8-frame launch
    tools/range_bench.py times: D = 6 (8-byte cp.async rows), 8 (compact rows), 12."""
    cfg = synth.get_config("c5", d_lo=d_lo, d_hi=d_hi)
    R, bands = chunk_edge_bands(rsr, cfg, 8)
    picks = [(b, rows) for b, rows in zip((1, 4, 6, 7), bands)]
    pipeline_parity(rsr, cfg, 8, picks)


EDGE_CASES = {
    # name: (H, W, d_lo, d_hi, rho_block, rho_agg, gamma_d, gamma_r, alpha, beta)
    "ragged_D7": (37, 101, -3, 3, 2, 3, 2.0, 10.0, 0.1, 2.0),
    "rho0": (24, 70, -4, 3, 1, 0, 1.0, 10.0, 0.0, 1.0),
    "gamma_r_inf": (30, 64, -4, 11, 2, 2, 2.0, math.inf, 0.05, 3.0),
    "negative_shift": (26, 90, -6, 5, 1, 4, 3.0, 8.0, -0.2, -3.0),
    "tiny_min": (5, 5, -1, 1, 2, 1, 1.0, 10.0, 0.0, 0.0),
    "shift_beyond_width": (20, 40, -2, 2, 1, 2, 2.0, 10.0, 0.0, 45.0),
    "D200_two_slabs": (20, 48, -100, 99, 1, 1, 2.0, 10.0, 0.0, 0.0),
    "rho7_D96": (40, 130, -48, 47, 4, 7, 5.0, 12.0, 0.1, 5.0),
    "D48": (33, 97, -24, 23, 3, 5, 4.0, 10.0, 0.08, 4.0),
    # two-CTA small-slab kernels: the paper's D = 30 (rows not 16-byte aligned:
    # copy spread over the producers) and D = 28 (compact rows, one bulk copy)
    "D30_rho4": (41, 133, -15, 14, 3, 4, 4.0, 12.0, 0.05, 3.0),
    "D28_rho4": (35, 101, -14, 13, 2, 4, 4.0, 12.0, 0.05, 3.0),
    "D12_rho6": (44, 90, -6, 5, 2, 6, 4.0, 12.0, 0.1, 2.0),
    # D % 4 == 2 rows staged by 8-byte cp.async, also across two slabs (KS = 64)
    "D126_two_slabs": (22, 160, -63, 62, 1, 2, 3.0, 10.0, 0.0, 1.0),
    "D14_rho3": (30, 77, -7, 6, 2, 3, 3.0, 10.0, 0.02, 1.0),
    # largest NCC block (15x15): block statistics need > 48 KB of shared memory
    "rho_block7": (44, 100, -4, 11, 7, 2, 2.0, 10.0, 0.0, 2.0),
    # rho 8..10: the tiled K3 kernel (aggregate.cu), one and two disparity slabs
    "rho8_D16": (40, 90, -8, 7, 2, 8, 5.0, 12.0, 0.05, 2.0),
    "rho9_D70_two_slabs": (38, 84, -35, 34, 2, 9, 5.0, 12.0, 0.0, 1.0),
    "rho10_D24": (48, 100, -12, 11, 3, 10, 6.0, 12.0, 0.05, 2.0),
    # D <= 3: the NaN summaries' low half is clipped to D (k_nan_maps); D <= 16 runs the
    # small-slab K2 / K3 / K4 kernels
    "D1": (30, 140, 0, 0, 2, 2, 2.0, 10.0, 0.0, 3.0),
    "D2_rho5": (33, 150, -1, 0, 2, 5, 3.0, 10.0, 0.05, 2.0),
    "D9_two_small_slabs": (36, 170, -4, 4, 3, 6, 4.0, 12.0, 0.1, 2.0),
    "D16_rho7": (40, 200, -8, 7, 4, 7, 5.0, 12.0, 0.05, 3.0),
}


@pytest.mark.parametrize("case", sorted(EDGE_CASES))
def test_parity_edge_cases(rsr, case):
    H, W, d_lo, d_hi, rb, ra, gd, gr, a, be = EDGE_CASES[case]
    cfg = synth.get_config("c1", height=H, width=W, d_lo=d_lo, d_hi=d_hi, rho_block=rb,
                           rho_agg=ra, gamma_d=gd, gamma_r=gr)
    left, right = synth.tiny_pair(zlib.crc32(case.encode()) % 1000, H, W, shift=3)  # stable across processes
    left = left.copy()
    if H > 12 and W > 12:
        left[2:9, 2:9] = 90  # constant patch: sigma = 0 blocks -> NaN costs
    gpu = run_gpu(rsr, left, right, [a, be], cfg)
    check_warp(gpu, right, (a, be))
    ora = O.run_pipeline(left, right, a, be, cfg)
    compare(gpu, ora, (0, H), cfg, label=case)


def test_nan_map_optional_same_within_tolerance(rsr):
    cfg = synth.get_config("c1")
    f = synth.make_frame(cfg)
    a = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg, nan_maps=True)
    b = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg, nan_maps=False)
    for key in ("agg_ref", "agg_tar"):
        # the clean path (nan_map) and the general path accumulate in the same order:
        # bitwise equal (aggregate_slide.cu, "produce_weights")
        assert np.array_equal(a[key], b[key], equal_nan=True), key


def test_determinism_and_batch_independence(rsr):
    cfg = synth.get_config("c2")
    left, right, ab = synth.make_batch(cfg, [0, 1])
    one = run_gpu(rsr, left[:1], right[:1], ab[:1], cfg)
    again = run_gpu(rsr, left[:1], right[:1], ab[:1], cfg)
    two = run_gpu(rsr, left, right, ab, cfg)
    for key in ("cost_ref", "agg_ref", "agg_tar", "disparity", "xyz"):
        assert np.array_equal(one[key][0], again[key][0], equal_nan=True), key
        assert np.array_equal(one[key][0], two[key][0], equal_nan=True), key


def test_dual_volume_identity_bitwise(rsr):
    cfg = synth.get_config("c2")
    f = synth.make_frame(cfg)
    gpu = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    cl, cr = gpu["cost_ref"][0], gpu["cost_tar"][0]
    H, W, D = cl.shape
    for k in range(D):
        r = cfg.d_lo + k
        u = np.arange(W)
        up = u - r
        ok = (up >= 0) & (up < W)
        assert np.array_equal(cl[:, u[ok], k], cr[:, up[ok], k], equal_nan=True)


def test_plane_accuracy_gpu(rsr):
    # same setting as the oracle pin tests/test_oracle_pins.py::test_plane_accuracy_against_ground_truth
    cfg = synth.get_config("c1", n_potholes=0)
    f = synth.make_frame(cfg)
    gpu = run_gpu(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    h, w = cfg.height, cfg.width
    m = cfg.rho_block + cfg.rho_agg + 2
    vv, uu = np.mgrid[0:h, 0:w]
    s = gpu["shift"][0]
    region = (vv >= m) & (vv < h - m) & (uu >= s[vv] + m) & (uu < w - m)
    d = gpu["disparity"][0][region]
    valid = ~np.isnan(d)
    assert valid.mean() >= 0.95
    rms = math.sqrt(np.mean((d[valid] - f.d_gt[region][valid]) ** 2))
    print("plane rms", rms, "valid", valid.mean())
    assert rms <= 0.25


def test_bad_arguments_return_codes(rsr):
    from paper_1807_07433_b200._lib import RsrAggParams, RsrShape, lib
    L = lib()
    x = torch.zeros(16, device="cuda")
    p = x.data_ptr()
    assert L.rsr_aggregate(RsrShape(1, 2, 2), 4, RsrAggParams(-1, 1.0, 1.0), p, p, None, p + 64, None) == 2
    assert L.rsr_aggregate(RsrShape(1, 2, 2), 4, RsrAggParams(1, 0.0, 1.0), p, p, None, p + 64, None) == 2
    assert L.rsr_aggregate(RsrShape(1, 2, 2), 4, RsrAggParams(1, 1.0, 1.0), p, p, None, p, None) == 2


def test_aggregate_independent_of_concurrency_hint(rsr):
    """The concurrency hint picks K3's row chunking only: bitwise equal results."""
    cfg = synth.get_config("c2")
    left, right, ab = synth.make_batch(cfg, [0, 1])
    L = torch.from_numpy(left).cuda()
    R = torch.from_numpy(right).cuda()
    W_, M_, S_ = rsr.rsr_warp(R, torch.from_numpy(ab).cuda())
    cl, cr, nl, nr = rsr.rsr_cost_volume(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi)
    outs = [rsr.rsr_aggregate(cl, L, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nl, concurrency=c) for c in (1, 2, 7)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(torch.nan_to_num(outs[0], nan=-7.0), torch.nan_to_num(o, nan=-7.0))


@pytest.mark.gpu
@pytest.mark.parametrize("D,rho", [(30, 4), (32, 4), (26, 6), (32, 1)])
def test_swapped_half_loads_bitwise_equal_unswapped(rsr, monkeypatch, D, rho):
    """G = 4 slabs (25 <= D <= 32): odd columns of the clean path load (and store) their two
    disparity halves in swapped order to avoid shared-memory bank conflicts; the values
    are the same operations, so the maps agree bitwise with the unswapped loads
    (RSR_K3_SWAP=0), on a c2-size frame with borders, warp bands and a constant patch."""
    d_lo = -(D // 2)
    cfg = synth.get_config("c2", d_lo=d_lo, d_hi=d_lo + D - 1, rho_agg=rho)
    f = synth.make_frame(cfg)
    L = torch.from_numpy(f.left)[None].cuda()
    R = torch.from_numpy(f.right)[None].cuda()
    L[0, 100:110, 200:210] = 77
    ab = torch.tensor([[f.alpha, f.beta]], dtype=torch.float64, device="cuda")
    W_, M_, S_ = rsr.rsr_warp(R, ab)
    cl, cr, nl, nr = rsr.rsr_cost_volume(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("RSR_K3_SWAP", flag)
        a = rsr.rsr_aggregate(cl, L, rho, cfg.gamma_d, cfg.gamma_r, nl)
        b = rsr.rsr_aggregate(cr, W_, rho, cfg.gamma_d, cfg.gamma_r, nr)
        torch.cuda.synchronize()
        outs.append((a.cpu().numpy(), b.cpu().numpy()))
    for x, y in zip(outs[0], outs[1]):
        assert np.isfinite(x).any()
        assert np.array_equal(x, y, equal_nan=True)


@pytest.mark.parametrize("D,rho,with_nan_map", [(8, 6, True), (8, 6, False), (3, 2, True), (5, 7, True),
                                               (9, 4, True), (12, 6, False), (16, 3, True), (6, 0, True)])
def test_small_slab_kernel_bitwise_equals_sliding_kernel(rsr, monkeypatch, D, rho, with_nan_map):
    """D <= 16 dispatches to the per-thread-weight kernel (aggregate_small.cu); it performs
    the sliding kernel's arithmetic operation for operation, so both agree bitwise
    (RSR_K3_SMALL=0 forces the sliding kernel) on a c2-size frame with borders, warp
    bands and constant patches (clean and general segments)."""
    d_lo = -(D // 2)
    cfg = synth.get_config("c2", d_lo=d_lo, d_hi=d_lo + D - 1, rho_agg=rho)
    f = synth.make_frame(cfg)
    L = torch.from_numpy(f.left)[None].cuda()
    R = torch.from_numpy(f.right)[None].cuda()
    L[0, 100:110, 200:210] = 77
    ab = torch.tensor([[f.alpha, f.beta]], dtype=torch.float64, device="cuda")
    W_, M_, S_ = rsr.rsr_warp(R, ab)
    cl, cr, nl, nr = rsr.rsr_cost_volume(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi)
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("RSR_K3_SMALL", flag)
        a = rsr.rsr_aggregate(cl, L, rho, cfg.gamma_d, cfg.gamma_r, nl if with_nan_map else None)
        b = rsr.rsr_aggregate(cr, W_, rho, cfg.gamma_d, cfg.gamma_r, nr if with_nan_map else None)
        torch.cuda.synchronize()
        outs.append((a.cpu().numpy(), b.cpu().numpy()))
    for x, y in zip(outs[0], outs[1]):
        assert np.array_equal(x, y, equal_nan=True)
