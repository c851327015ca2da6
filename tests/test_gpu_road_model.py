"""GPU parity of rsr_road_model (NEXT row f3) against oracle/road_model.py: the
inlier decisions are taken in fp64 with one rounding per operation on both sides,
so the consensus size is compared exactly and the least-squares line within
fp64 summation-order rounding."""
import numpy as np
import pytest

import synth
from oracle import road_model as RM

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


def check(model, disp, su, sv, n_hyp, tol, seed):
    v, d = RM.grid_samples(disp, su, sv)
    a, b, n, _ = RM.fit_road_model(v, d, n_hyp, tol, seed)
    assert int(model[2]) == n
    if n >= 2:
        assert abs(model[0] - a) <= 1e-9 * max(1.0, abs(a))
        assert abs(model[1] - b) <= 1e-9 * max(1.0, abs(b))
    else:
        assert np.isnan(model[0])
    return a, b, n


def test_ground_truth_planes_batched(rsr):
    cfg = synth.get_config("c5", height=360, width=640)
    maps = [synth.make_frame(cfg, i).d_gt.astype(np.float32) for i in range(3)]
    D = torch.from_numpy(np.stack(maps)).cuda()
    m = rsr.rsr_road_model(D, 4, 4, 256, 1e-3, 7).cpu().numpy()
    for k in range(3):
        a, b, n = check(m[k], maps[k], 4, 4, 256, 1e-3, 7)
        f = synth.make_frame(cfg, k)
        assert abs(a - f.alpha) < 1e-5 and abs(b - f.beta) < 1e-3


def test_computed_disparity_map_c1(rsr):
    """The path's own output (NaN holes, noise) as the sample source."""
    cfg = synth.get_config("c1")
    f = synth.make_frame(cfg)
    pipe = rsr.StereoPipeline(1, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    L = torch.from_numpy(f.left)[None].cuda()
    R = torch.from_numpy(f.right)[None].cuda()
    AB = torch.tensor([[f.alpha, f.beta]], dtype=torch.float64, device="cuda")
    pipe.run(L, R, AB)
    for su, sv, nh, tol, seed in ((1, 1, 512, 0.5, 3), (3, 2, 100, 0.25, 11), (8, 8, 1, 1.0, 0)):
        m = rsr.rsr_road_model(pipe.disparity, su, sv, nh, tol, seed).cpu().numpy()
        check(m[0], pipe.disparity[0].cpu().numpy(), su, sv, nh, tol, seed)
    m = rsr.rsr_road_model(pipe.disparity, 2, 2, 512, 0.5, 3).cpu().numpy()[0]
    assert abs(m[0] - f.alpha) < 5e-3 and abs(m[1] - f.beta) < 0.5   # the road plane of the frame


def test_degenerate_maps(rsr):
    nanmap = torch.full((2, 20, 30), float("nan"), device="cuda")
    nanmap[1, 5, 7] = 3.0          # one sample only
    m = rsr.rsr_road_model(nanmap, 1, 1, 16, 0.5, 0).cpu().numpy()
    assert np.isnan(m[:, 0]).all() and (m[:, 2] == 0).all()
    row = torch.full((1, 20, 30), float("nan"), device="cuda")
    row[0, 4, :] = torch.arange(30, dtype=torch.float32, device="cuda")   # one image row
    m = rsr.rsr_road_model(row, 1, 1, 16, 0.5, 0).cpu().numpy()[0]
    assert np.isnan(m[0]) and m[2] == 0


def test_roll_plane_fit(rsr):
    from oracle import road_model as RM
    h, w = 120, 200
    vv, uu = np.mgrid[0:h, 0:w]
    rng = np.random.default_rng(2)
    maps = []
    for k in range(3):
        d = (10.0 + k + (0.002 * k - 0.003) * uu + 0.1 * vv + rng.normal(0, 0.2, (h, w))).astype(np.float32)
        d[rng.random((h, w)) < 0.1] = np.nan
        maps.append(d)
    D = torch.from_numpy(np.stack(maps)).cuda()
    out = rsr.rsr_road_roll(D, 20, 180, 70, 120).cpu().numpy()
    for k in range(3):
        ref = RM.roll_plane_fit(maps[k], 20, 180, 70, 120)
        assert out[k, 4] == ref[4]
        assert np.allclose(out[k, :4], ref[:4], rtol=1e-8, atol=1e-12), (out[k], ref)
