"""The Python binding checks every tensor argument (dtype and exact shape),
caller-supplied outputs and workspace included, BEFORE any pointer reaches the
C ABI (which sees only pointers and sizes: an undersized buffer would become an
out-of-bounds device access).  CPU-only: the checks raise before the device
check, so no GPU is needed (ops.py)."""
import pytest

torch = pytest.importorskip("torch")
ops = pytest.importorskip("paper_1807_07433_b200.ops")

B, H, W, D = 2, 12, 20, 8
u8 = lambda *s: torch.zeros(s, dtype=torch.uint8)  # noqa: E731
f32 = lambda *s: torch.zeros(s, dtype=torch.float32)  # noqa: E731


def raises(fn, match):
    with pytest.raises((ValueError, TypeError), match=match):
        fn()


def test_warp_outputs_checked():
    t = u8(B, H, W)
    ab = torch.zeros((B, 2), dtype=torch.float64)
    raises(lambda: ops.rsr_warp(t, ab, warped=u8(B, H, W - 1)), "warped")
    raises(lambda: ops.rsr_warp(t, ab, valid=u8(B, H, W).float()), "valid")
    raises(lambda: ops.rsr_warp(t, ab, shift=torch.zeros((B, H - 1), dtype=torch.int32)), "shift")
    raises(lambda: ops.rsr_warp(t.float(), ab), "target")


def test_cost_volume_inputs_and_outputs_checked():
    L, Wp, M = u8(B, H, W), u8(B, H, W), u8(B, H, W)
    raises(lambda: ops.rsr_cost_volume(L, Wp[:, :-1], M, 1, 0, D - 1), "warped")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M.int(), 1, 0, D - 1), "valid")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 0, D - 1, vol_ref=f32(B, H, W, D - 1)), "vol_ref")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 0, D - 1, vol_tar=f32(B, H, W + 1, D)), "vol_tar")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 0, D - 1, nan_ref=u8(B, H, W - 1)), "nan_ref")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 0, D - 1, nan_tar=f32(B, H, W)), "nan_tar")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 0, D - 1, workspace=u8(16)), "workspace")
    raises(lambda: ops.rsr_cost_volume(L, Wp, M, 1, 3, 2), "empty search range")


def test_aggregate_guide_nan_map_out_checked():
    vol = f32(B, H, W, D)
    g = u8(B, H, W)
    raises(lambda: ops.rsr_aggregate(vol, g.float(), 2, 1.0, 1.0), "guide")
    raises(lambda: ops.rsr_aggregate(vol, g[:, :-1], 2, 1.0, 1.0), "vol")
    raises(lambda: ops.rsr_aggregate(vol, g, 2, 1.0, 1.0, nan_map=u8(B, H, W - 2)), "nan_map")
    raises(lambda: ops.rsr_aggregate(vol, g, 2, 1.0, 1.0, out=f32(B, H, W, D - 1)), "out")
    raises(lambda: ops.rsr_aggregate(vol, g, 2, 1.0, 1.0, out=vol), "alias")


def test_disparity_and_reconstruct_checked():
    a = f32(B, H, W, D)
    sh = torch.zeros((B, H), dtype=torch.int32)
    raises(lambda: ops.rsr_disparity(a, f32(B, H, W, D - 1), sh, 0, D - 1, 1), "agg_tar")
    raises(lambda: ops.rsr_disparity(a, a, sh, 0, D, 1), "range")
    raises(lambda: ops.rsr_disparity(a, a, sh, 0, D - 1, 1, disparity=f32(B, H, W - 1)), "disparity")
    raises(lambda: ops.rsr_disparity(a, a, sh, 0, D - 1, 1, with_wta=True,
                                     wta_ref=torch.zeros((B, H, W), dtype=torch.int32)), "wta_ref")
    d = f32(B, H, W)
    raises(lambda: ops.rsr_reconstruct(d, 700.0, 0.12, xyz=f32(B, H, W, 4)), "xyz")
    raises(lambda: ops.rsr_reconstruct(d.double(), 700.0, 0.12), "disparity")


def test_cpu_tensors_refused():
    """No CPU fallback: well-formed CPU tensors are refused at the device check."""
    t = u8(B, H, W)
    ab = torch.zeros((B, 2), dtype=torch.float64)
    with pytest.raises(ValueError, match="CUDA"):
        ops.rsr_warp(t, ab)
