"""GPU parity of rsr_search_range (NEXT row f4) against
oracle/search_range.py: integer bands, compared exactly, on the path's own
disparity maps and on constructed maps (empty, clipped, random NaN patterns)."""
import numpy as np
import pytest

import synth
from oracle import search_range as SR

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rsr():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as m
    return m


def _check(rsr, disp, shift, delta, lo, hi):
    got = rsr.rsr_search_range(torch.from_numpy(disp).cuda(), torch.from_numpy(shift).cuda(), delta, lo,
                               hi).cpu().numpy()
    for b in range(disp.shape[0]):
        assert tuple(got[b]) == SR.search_range(disp[b], shift[b], delta, lo, hi), b


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_search_range_on_path_maps(rsr, name):
    cfg = synth.get_config(name)
    left, right, ab = synth.make_batch(cfg, [0, 1, 2])
    pipe = rsr.StereoPipeline(3, cfg.height, cfg.width, rsr.StereoParams.from_config(cfg))
    pipe.run(torch.from_numpy(left).cuda(), torch.from_numpy(right).cuda(), torch.from_numpy(ab).cuda(),
             with_wta=False)
    torch.cuda.synchronize()
    disp = pipe.disparity.cpu().numpy()
    shift = pipe.shift.cpu().numpy()
    for delta in (0, 2, 5):
        _check(rsr, disp, shift, delta, cfg.d_lo, cfg.d_hi)
    # the next frame's shifts (a different plane) and narrow limits
    _check(rsr, disp, np.roll(shift, 1, axis=0) + 1, 1, -4, 3)


def test_search_range_constructed_maps(rsr):
    rng = np.random.default_rng(0)
    B, H, W = 6, 37, 1031
    disp = (rng.normal(size=(B, H, W)) * 5 + 30).astype(np.float32)
    disp[rng.random(size=disp.shape) < 0.3] = np.nan
    disp[1] = np.nan                                   # empty map -> limits
    disp[2, 5, 7] = 1e6                                # clipped high
    disp[3] = np.float32(30.0)                         # integer residuals
    shift = rng.integers(20, 40, size=(B, H)).astype(np.int32)
    for delta, lo, hi in ((0, -64, 63), (3, -8, 7), (1, -16383, 16383)):
        _check(rsr, disp, shift, delta, lo, hi)


def test_search_range_bad_arguments(rsr):
    from paper_1807_07433_b200._lib import RsrShape, lib
    L = lib()
    x = torch.zeros(64, device="cuda")
    p = x.data_ptr()
    s = RsrShape(1, 2, 2)
    assert L.rsr_search_range(s, p, p, -1, -4, 3, p, None) == 2
    assert L.rsr_search_range(s, p, p, 0, 4, 3, p, None) == 2
    assert L.rsr_search_range(s, p, p, 0, -20000, 20000, p, None) == 2
    assert L.rsr_search_range(s, None, p, 0, -4, 3, p, None) == 2
