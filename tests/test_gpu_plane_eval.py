"""GPU parity of rsr_plane_fit / rsr_plane_distance (NEXT row f4) against
oracle/plane_eval.py: the total-least-squares plane (fp64 Jacobi on the GPU, SVD
in the oracle) within fp64 rounding, the degenerate decisions equal, and the
signed distances of the reconstructed points within one float32 ulp."""
import numpy as np
import pytest

import synth
from oracle import plane_eval as PE

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


@pytest.mark.parametrize("K", [3, 4, 7])
def test_plane_fit_parity(rsr, K):
    rng = np.random.default_rng(K)
    B = 200
    c = np.stack([rng.normal(size=(K, 3)) * rng.uniform(0.01, 2.0, size=3) + rng.normal(size=3) * [0.5, 0.5, 3]
                  for _ in range(B)])
    c[0] = [[0, 0, 1.0 + 0.1 * i] for i in range(K)]      # collinear: NaN
    c[1, 1, 2] = np.nan                                     # non-finite corner: NaN
    c[2] = [[np.cos(t), np.sin(t), 0.0] for t in np.linspace(0, 2 * np.pi, K, endpoint=False)]  # n3 == 0
    got = rsr.rsr_plane_fit(torch.from_numpy(c).cuda()).cpu().numpy()
    for b in range(B):
        ref = PE.fit_plane(c[b])
        if np.isnan(ref).any():
            assert np.isnan(got[b]).all(), b
            continue
        scale = max(1.0, np.abs(c[b]).max())
        assert np.allclose(got[b, :3], ref[:3], atol=1e-11), (b, got[b], ref)
        assert abs(got[b, 3] - ref[3]) <= 1e-11 * scale, (b, got[b], ref)


def test_plane_distance_on_reconstructed_road(rsr):
    """The paper's procedure on a reconstruction from the path: corners picked on
    the reconstructed road, the GPU plane, and every point's signed distance."""
    cfg = synth.get_config("c1")
    left, right, ab = synth.make_batch(cfg, [0, 1])
    L = torch.from_numpy(left).cuda()
    R = torch.from_numpy(right).cuda()
    AB = torch.from_numpy(ab).cuda()
    pipe = rsr.StereoPipeline(2, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    pipe.run(L, R, AB, with_wta=False)
    torch.cuda.synchronize()
    xyz = pipe.xyz.cpu().numpy()
    corners = []
    for b in range(2):
        pts = []
        for (v, u) in ((40, 60), (40, 260), (150, 260), (150, 60)):
            # nearest finite point around the nominal corner
            win = xyz[b, v - 5:v + 6, u - 5:u + 6].reshape(-1, 3)
            ok = np.isfinite(win).all(1)
            assert ok.any()
            pts.append(win[np.flatnonzero(ok)[0]].astype(np.float64))
        corners.append(pts)
    corners = np.array(corners)
    plane = rsr.rsr_plane_fit(torch.from_numpy(corners).cuda())
    dist = rsr.rsr_plane_distance(plane, pipe.xyz).cpu().numpy()
    pl = plane.cpu().numpy()
    for b in range(2):
        ref_pl = PE.fit_plane(corners[b])
        assert np.allclose(pl[b], ref_pl, atol=1e-12)
        ref = PE.point_plane_distance(pl[b], xyz[b].astype(np.float64)).astype(np.float32)
        fin = np.isfinite(ref)
        assert np.array_equal(fin, np.isfinite(dist[b]))
        ulp = np.spacing(np.abs(ref[fin])).astype(np.float64)
        assert (np.abs(dist[b][fin].astype(np.float64) - ref[fin]) <= ulp + 1e-12).all()
        # the road lies on the plane to within the reconstruction noise: at Z ~ 5-8 m,
        # f b = 84 px m, 0.05 px of disparity noise at a corner is ~3 cm
        assert np.nanmedian(np.abs(dist[b])) < 0.1
