"""NEXT row f1: the fused, volume-free kernel (rsr_match, csrc/match_fused.cu)
against the five-call path (rsr_cost_volume -> rsr_aggregate x2 -> rsr_disparity,
itself parity-tested against the oracle in tests/test_gpu_parity.py).  rsr_match
performs the same operations in the same order, so the disparity and both WTA
maps must be bitwise equal (include/rsr.h) -- and, through the five-call path,
within the oracle tolerances.  Cases: the restricted band at c5 size in an
8-frame batch, small frames with ragged widths, borders, warp bands, negative
shifts, constant patches (isolated NaN costs), rho 0..7, varrho 1..7, D 1..8."""
import zlib

import numpy as np
import pytest

import synth
from oracle import rsr_oracle as O

from test_gpu_parity import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


def both_paths(rsr, left, right, ab, cfg):
    L = torch.from_numpy(np.ascontiguousarray(left)).cuda()
    R = torch.from_numpy(np.ascontiguousarray(right)).cuda()
    if L.dim() == 2:
        L, R = L[None], R[None]
    AB = torch.tensor(np.asarray(ab, dtype=np.float64).reshape(-1, 2), device="cuda")
    W_, M_, S_ = rsr.rsr_warp(R, AB)
    cl, cr, nl, nr = rsr.rsr_cost_volume(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi)
    al = rsr.rsr_aggregate(cl, L, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nl)
    ar = rsr.rsr_aggregate(cr, W_, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nr)
    d5, kl5, kr5 = rsr.rsr_disparity(al, ar, S_, cfg.d_lo, cfg.d_hi, cfg.lrc_tol, True, with_wta=True)
    df, klf, krf = rsr.rsr_match(L, W_, M_, S_, cfg.rho_block, cfg.d_lo, cfg.d_hi, cfg.rho_agg, cfg.gamma_d,
                                 cfg.gamma_r, cfg.lrc_tol, True, with_wta=True)
    torch.cuda.synchronize()
    g = lambda t: t.cpu().numpy()  # noqa: E731
    return dict(d5=g(d5), kl5=g(kl5), kr5=g(kr5), df=g(df), klf=g(klf), krf=g(krf), W=g(W_), M=g(M_), S=g(S_),
                cost_ref=g(cl), cost_tar=g(cr), agg_ref=g(al), agg_tar=g(ar))


def assert_bitwise(r):
    assert np.array_equal(r["kl5"], r["klf"]), np.argwhere(r["kl5"] != r["klf"])[:5]
    assert np.array_equal(r["kr5"], r["krf"]), np.argwhere(r["kr5"] != r["krf"])[:5]
    a, b = r["d5"], r["df"]
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)]), np.abs(a - b)[~np.isnan(a)].max()


@pytest.mark.parametrize("d_lo,d_hi", [(-4, 3), (-3, 2), (-2, 2)])
def test_fused_equals_five_calls_restricted_band_c5(rsr, d_lo, d_hi):
    cfg = synth.get_config("c5", d_lo=d_lo, d_hi=d_hi)
    left, right, ab = synth.make_batch(cfg, list(range(8)))
    r = both_paths(rsr, left, right, ab, cfg)
    assert_bitwise(r)
    assert np.isfinite(r["df"]).mean() > 0.5


FUSED_EDGE = {
    # name: (H, W, d_lo, d_hi, rho_block, rho_agg, gamma_d, gamma_r, alpha, beta)
    "D8_rho6": (40, 250, -4, 3, 3, 6, 4.0, 12.0, 0.05, 3.0),
    "D5_ragged": (37, 101, -2, 2, 2, 3, 2.0, 10.0, 0.1, 2.0),
    "D1": (30, 140, 0, 0, 2, 2, 2.0, 10.0, 0.0, 3.0),
    "rho0": (24, 130, -4, 3, 1, 0, 1.0, 10.0, 0.0, 1.0),
    "rho7_rb7": (50, 131, -3, 4, 7, 7, 5.0, 12.0, 0.05, 4.0),
    "negative_shift": (26, 200, -4, 3, 1, 4, 3.0, 8.0, -0.2, -3.0),
    "gamma_r_inf": (30, 123, -4, 3, 2, 2, 2.0, float("inf"), 0.05, 3.0),
    "wide_two_strips": (20, 260, -4, 3, 3, 5, 4.0, 12.0, 0.0, 20.0),
    "tiny": (15, 15, -1, 1, 1, 2, 2.0, 10.0, 0.0, 0.0),
}


@pytest.mark.parametrize("case", sorted(FUSED_EDGE))
def test_fused_equals_five_calls_edge_cases(rsr, case):
    H, W, d_lo, d_hi, rb, ra, gd, gr, a, be = FUSED_EDGE[case]
    cfg = synth.get_config("c1", height=H, width=W, d_lo=d_lo, d_hi=d_hi, rho_block=rb, rho_agg=ra,
                           gamma_d=gd, gamma_r=gr)
    left, right = synth.tiny_pair(zlib.crc32(case.encode()) % 1000, H, W, shift=3)
    left = left.copy()
    if H > 12 and W > 12:
        left[2:9, 2:9] = 90   # constant patch: NaN costs inside the image
    r = both_paths(rsr, left, right, [a, be], cfg)
    assert_bitwise(r)
    # and through the five-call path, the oracle's tolerances
    ora = O.run_pipeline(left, right, a, be, cfg)
    gpu = dict(warped=r["W"], mask=r["M"], shift=r["S"], cost_ref=r["cost_ref"],
               cost_tar=r["cost_tar"], agg_ref=r["agg_ref"], agg_tar=r["agg_tar"], disparity=r["df"],
               k_ref=r["klf"], k_tar=r["krf"], xyz=np.zeros(r["df"].shape + (3,), np.float32) * np.nan)
    ora["xyz"] = np.full(ora["xyz"].shape, np.nan)
    compare(gpu, ora, (0, H), cfg, label=f"fused {case}")


def test_match_rejects_large_ranges(rsr):
    cfg = synth.get_config("c1")
    L = torch.zeros((1, 32, 64), dtype=torch.uint8, device="cuda")
    S = torch.zeros((1, 32), dtype=torch.int32, device="cuda")
    with pytest.raises(rsr.RsrError):
        rsr.rsr_match(L, L, L, S, 2, -8, 8, 2, 2.0, 10.0, 1)   # D = 17 > 8
