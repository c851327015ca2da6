"""The P:198 accuracy protocol on the GPU path (NEXT row f4): a box of known
height on a synthetic road (tools/accuracy_eval.py), corners -> rsr_plane_fit,
random box-top points -> rsr_plane_distance.  The measured height must match the
scene's within the paper's "approximately 3 mm" for both warps."""
import os
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.parametrize("warp", ["integer", "linear"])
def test_box_height_within_3mm(warp):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1807_07433_b200 as rsr
    import accuracy_eval
    r = accuracy_eval.measure_box_height(rsr, torch, 0.020, seed=1, warp=warp)
    print(r)
    assert r["n"] >= 90
    assert abs(r["err_mm"]) <= 3.0, r
    assert abs(r["median_mm"] - 20.0) <= 3.0, r
