"""GPU parity of the interpolating-warp variant (NEXT row f2, DESIGN.md reading
21) through the C ABI (rsr_warp_linear, rsr_cost_volume_linear,
rsr_aggregate_linear, rsr_disparity_linear) against the oracle
(oracle/interp_warp.py), with the tolerances of tests/test_gpu_parity.py:
warp / mask / applied shift bitwise; NCC |dc| <= 1e-4 and identical NaN masks
(the sums are exact integers: only the fp32 normalisation differs); aggregated
volumes relative 1e-4; WTA >= 99.9 %, mismatches only at oracle near-ties;
disparity 1e-3 px; points 1e-4."""
import zlib

import numpy as np
import pytest

import synth
from oracle import interp_warp as IW

from test_gpu_parity import compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


def run_gpu_linear(rsr, left, right, ab, cfg):
    L = torch.from_numpy(np.ascontiguousarray(left)).cuda()
    R = torch.from_numpy(np.ascontiguousarray(right)).cuda()
    if L.dim() == 2:
        L, R = L[None], R[None]
    AB = torch.tensor(np.asarray(ab, dtype=np.float64).reshape(-1, 2), device="cuda")
    W_, M_, S_ = rsr.rsr_warp_linear(R, AB)
    cl, cr, nl, nr = rsr.rsr_cost_volume_linear(L, W_, M_, cfg.rho_block, cfg.d_lo, cfg.d_hi)
    al = rsr.rsr_aggregate(cl, L, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nl)
    ar = rsr.rsr_aggregate_linear(cr, W_, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r, nr)
    d, kl, kr = rsr.rsr_disparity_linear(al, ar, S_, cfg.d_lo, cfg.d_hi, cfg.lrc_tol, True, with_wta=True)
    xyz = rsr.rsr_reconstruct(d, cfg.focal, cfg.baseline, d_min=1.0)
    torch.cuda.synchronize()
    g = lambda t: t.cpu().numpy()  # noqa: E731
    return dict(warped=g(W_), mask=g(M_), shift=g(S_), cost_ref=g(cl), cost_tar=g(cr), agg_ref=g(al),
                agg_tar=g(ar), disparity=g(d), k_ref=g(kl), k_tar=g(kr), xyz=g(xyz))


def check_warp_linear(gpu, right, ab, b=0):
    Wo, Mo, To = IW.warp_target_linear(right, ab[0], ab[1])
    assert np.array_equal(gpu["warped"][b], Wo)
    assert np.array_equal(gpu["mask"][b], Mo)
    assert np.array_equal(gpu["shift"][b], To)


@pytest.mark.parametrize("name,beta", [("c1", 10.37), ("c2", 20.61)])
def test_linear_parity_full_frame(rsr, name, beta):
    cfg = synth.get_config(name, beta=beta)
    f = synth.make_frame(cfg)
    gpu = run_gpu_linear(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    check_warp_linear(gpu, f.right, (f.alpha, f.beta))
    ora = IW.run_pipeline_linear(f.left, f.right, f.alpha, f.beta, cfg)
    rep = compare(gpu, ora, (0, cfg.height), cfg, label=f"linear {name}")
    print(name, rep)


def test_linear_parity_full_size_bands(rsr):
    cfg = synth.get_config("c3", beta=30.43)
    f = synth.make_frame(cfg)
    gpu = run_gpu_linear(rsr, f.left, f.right, [f.alpha, f.beta], cfg)
    check_warp_linear(gpu, f.right, (f.alpha, f.beta))
    for rows in ((0, 5), (357, 363), (715, 720)):
        ora = IW.run_pipeline_linear(f.left, f.right, f.alpha, f.beta, cfg, rows=rows)
        compare(gpu, ora, rows, cfg, label=f"linear c3{rows}")


LINEAR_EDGE = {
    # name: (H, W, d_lo, d_hi, rho_block, rho_agg, gamma_d, gamma_r, alpha, beta)
    "ragged_D7_rb2": (37, 101, -3, 3, 2, 3, 2.0, 10.0, 0.013, 2.37),
    "rb7_D16": (44, 100, -4, 11, 7, 2, 2.0, 10.0, 0.0, 2.5),
    "rb5_D70_two_slabs": (30, 150, -35, 34, 5, 2, 3.0, 12.0, 0.02, 1.1),
    "negative_shift": (26, 90, -6, 5, 1, 4, 3.0, 8.0, -0.21, -3.3),
    "rho7_D48": (40, 130, -24, 23, 4, 7, 5.0, 12.0, 0.1, 5.7),
    "gamma_r_inf": (30, 64, -4, 11, 2, 2, 2.0, float("inf"), 0.05, 3.2),
    "D30_rho4_small_slab": (41, 133, -15, 14, 3, 4, 4.0, 12.0, 0.05, 3.9),
}


@pytest.mark.parametrize("case", sorted(LINEAR_EDGE))
def test_linear_parity_edge_cases(rsr, case):
    H, W, d_lo, d_hi, rb, ra, gd, gr, a, be = LINEAR_EDGE[case]
    cfg = synth.get_config("c1", height=H, width=W, d_lo=d_lo, d_hi=d_hi, rho_block=rb, rho_agg=ra,
                           gamma_d=gd, gamma_r=gr)
    left, right = synth.tiny_pair(zlib.crc32(case.encode()) % 1000, H, W, shift=3)
    left = left.copy()
    left[2:9, 2:9] = 90   # constant patch: sigma = 0 blocks
    gpu = run_gpu_linear(rsr, left, right, [a, be], cfg)
    check_warp_linear(gpu, right, (a, be))
    ora = IW.run_pipeline_linear(left, right, a, be, cfg)
    compare(gpu, ora, (0, H), cfg, label=f"linear {case}")


def test_linear_dual_identity_bitwise_and_pipeline(rsr):
    cfg = synth.get_config("c2", beta=20.61)
    left, right, ab = synth.make_batch(cfg, [0, 1])
    ab[:, 1] += 0.37
    gpu = run_gpu_linear(rsr, left, right, ab, cfg)
    cl, cr = gpu["cost_ref"][1], gpu["cost_tar"][1]
    H, W, D = cl.shape
    for k in range(D):
        r = cfg.d_lo + k
        u = np.arange(W)
        ok = (u - r >= 0) & (u - r < W)
        assert np.array_equal(cl[:, u[ok], k], cr[:, u[ok] - r, k], equal_nan=True)
    # the pipeline (warp="linear") gives the same maps as the individual calls
    pipe = rsr.StereoPipeline(2, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg, warp="linear"))
    pipe.run(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda(), torch.from_numpy(ab).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(pipe.disparity.cpu().numpy(), gpu["disparity"], equal_nan=True)
