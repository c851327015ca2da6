"""Python-level names of the C-ABI calls (include/rsr.h), over torch CUDA
tensors.  Each function checks the dtype, shape, device and contiguity of EVERY
tensor argument, caller-supplied outputs and workspace included (the C ABI sees
only pointers, so an undersized buffer would become an out-of-bounds device
access), allocates missing outputs with torch (device memory plumbing) and
calls the library on the current torch CUDA stream.  No arithmetic of the
method happens here."""
from __future__ import annotations

import torch

from ._lib import (RsrAggParams, RsrCostParams, RsrDispParams, RsrRig, RsrRoadParams, RsrShape, check,
                   lib)


def _ptr(t):
    return None if t is None else ctypes_ptr(t)


def ctypes_ptr(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("rsr: tensors must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("rsr: tensors must be contiguous")
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _expect(t, dtype, shape, name):
    """Check dtype and exact shape of a tensor argument (None passes: optional)."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"rsr: {name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"rsr: {name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"rsr: {name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _bhw(img: torch.Tensor):
    if img.dim() == 2:
        img = img.unsqueeze(0)
    if img.dim() != 3:
        raise ValueError("rsr: images must be [B,H,W] or [H,W]")
    return img, RsrShape(*img.shape)


def rsr_warp(target, alpha_beta, warped=None, valid=None, shift=None):
    """Step 1: returns (warped uint8 [B,H,W], valid uint8 [B,H,W], shift int32 [B,H])."""
    target, s = _bhw(target)
    B, H, W = target.shape
    _expect(target, torch.uint8, (B, H, W), "target")
    alpha_beta = alpha_beta.reshape(B, 2)
    _expect(alpha_beta, torch.float64, (B, 2), "alpha_beta")
    warped = torch.empty_like(target) if warped is None else warped
    valid = torch.empty_like(target) if valid is None else valid
    shift = torch.empty((B, H), dtype=torch.int32, device=target.device) if shift is None else shift
    _expect(warped, torch.uint8, (B, H, W), "warped")
    _expect(valid, torch.uint8, (B, H, W), "valid")
    _expect(shift, torch.int32, (B, H), "shift")
    check("rsr_warp", lib().rsr_warp(s, _ptr(alpha_beta), _ptr(target), _ptr(warped), _ptr(valid),
                                     _ptr(shift), _stream()))
    return warped, valid, shift


def cost_workspace_bytes(B, H, W) -> int:
    return int(lib().rsr_cost_workspace_size(RsrShape(B, H, W)))


def rsr_cost_volume(ref, warped, valid, rho_block, d_lo, d_hi, *, with_tar=True, with_nan_maps=True,
                    vol_ref=None, vol_tar=None, nan_ref=None, nan_tar=None, workspace=None):
    """Step 2 (Eqs. 3-5): returns (vol_ref, vol_tar|None, nan_ref|None, nan_tar|None),
    volumes float32 [B,H,W,D]."""
    ref, s = _bhw(ref)
    B, H, W = ref.shape
    warped, _ = _bhw(warped)
    valid, _ = _bhw(valid)
    D = d_hi - d_lo + 1
    if D < 1:
        raise ValueError(f"rsr: empty search range [{d_lo}, {d_hi}]")
    for t, name in ((ref, "ref"), (warped, "warped"), (valid, "valid")):
        _expect(t, torch.uint8, (B, H, W), name)
    dev = ref.device
    if vol_ref is None:
        vol_ref = torch.empty((B, H, W, D), dtype=torch.float32, device=dev)
    if with_tar and vol_tar is None:
        vol_tar = torch.empty((B, H, W, D), dtype=torch.float32, device=dev)
    if with_nan_maps:
        nan_ref = torch.empty((B, H, W), dtype=torch.uint8, device=dev) if nan_ref is None else nan_ref
        if with_tar and nan_tar is None:
            nan_tar = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
    nbytes = cost_workspace_bytes(B, H, W)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for t, name in ((vol_ref, "vol_ref"), (vol_tar, "vol_tar")):
        _expect(t, torch.float32, (B, H, W, D), name)
    for t, name in ((nan_ref, "nan_ref"), (nan_tar, "nan_tar")):
        _expect(t, torch.uint8, (B, H, W), name)
    if workspace.dtype != torch.uint8 or workspace.dim() != 1 or workspace.numel() < nbytes:
        raise ValueError(f"rsr: workspace must be a uint8 vector of >= {nbytes} bytes")
    check("rsr_cost_volume", lib().rsr_cost_volume(
        s, RsrCostParams(rho_block, d_lo, d_hi), _ptr(ref), _ptr(warped), _ptr(valid), _ptr(vol_ref),
        _ptr(vol_tar), _ptr(nan_ref), _ptr(nan_tar), _ptr(workspace), workspace.numel(), _stream()))
    return vol_ref, vol_tar, nan_ref, nan_tar


def rsr_aggregate(vol, guide, rho, gamma_d, gamma_r, nan_map=None, out=None, concurrency=1):
    """Step 3 (Eqs. 8-10): aggregated volume float32 [B,H,W,D].  concurrency: how many
    aggregations the caller keeps in flight together (grid choice only)."""
    guide, s = _bhw(guide)
    B, H, W = guide.shape
    if vol.dim() == 3:
        vol = vol.unsqueeze(0)
    D = vol.shape[-1]
    _expect(guide, torch.uint8, (B, H, W), "guide")
    _expect(vol, torch.float32, (B, H, W, D), "vol")
    out = torch.empty_like(vol) if out is None else out
    _expect(out, torch.float32, (B, H, W, D), "out")
    if out.data_ptr() == vol.data_ptr():
        raise ValueError("rsr: out must not alias vol")
    if nan_map is not None:
        nan_map, _ = _bhw(nan_map)
        _expect(nan_map, torch.uint8, (B, H, W), "nan_map")
    check("rsr_aggregate", lib().rsr_aggregate(
        s, D, RsrAggParams(rho, float(gamma_d), float(gamma_r), int(concurrency)), _ptr(vol), _ptr(guide),
        _ptr(nan_map), _ptr(out), _stream()))
    return out


def rsr_aggregate_rows(B, H, W, D, rho, concurrency=1) -> int:
    """Output rows per CTA rsr_aggregate uses for these arguments (0: the rho > 7 tiled
    kernel); host-only introspection for tests and tools."""
    r = int(lib().rsr_aggregate_rows(RsrShape(B, H, W), int(D), RsrAggParams(int(rho), 1.0, 1.0, int(concurrency))))
    if r < 0:
        raise ValueError("rsr_aggregate_rows: invalid arguments")
    return r


def rsr_disparity(agg_ref, agg_tar, shift, d_lo, d_hi, lrc_tol, subpixel=True, disparity=None,
                  wta_ref=None, wta_tar=None, with_wta=False):
    """Steps 4-5 (Eqs. 11-12): returns (disparity f32 [B,H,W], wta_ref, wta_tar)."""
    if agg_ref.dim() == 3:
        agg_ref, agg_tar = agg_ref.unsqueeze(0), agg_tar.unsqueeze(0)
    B, H, W, D = agg_ref.shape
    if D != d_hi - d_lo + 1:
        raise ValueError(f"rsr: volumes hold D = {D} disparities, range [{d_lo}, {d_hi}] needs {d_hi - d_lo + 1}")
    _expect(agg_ref, torch.float32, (B, H, W, D), "agg_ref")
    _expect(agg_tar, torch.float32, (B, H, W, D), "agg_tar")
    shift = shift.reshape(B, H)
    _expect(shift, torch.int32, (B, H), "shift")
    dev = agg_ref.device
    disparity = torch.empty((B, H, W), dtype=torch.float32, device=dev) if disparity is None else disparity
    if with_wta:
        wta_ref = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_ref is None else wta_ref
        wta_tar = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_tar is None else wta_tar
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    _expect(wta_ref, torch.int16, (B, H, W), "wta_ref")
    _expect(wta_tar, torch.int16, (B, H, W), "wta_tar")
    check("rsr_disparity", lib().rsr_disparity(
        RsrShape(B, H, W), RsrDispParams(d_lo, d_hi, lrc_tol, 1 if subpixel else 0), _ptr(agg_ref),
        _ptr(agg_tar), _ptr(shift), _ptr(disparity), _ptr(wta_ref), _ptr(wta_tar), _stream()))
    return disparity, wta_ref, wta_tar


def rsr_reconstruct(disparity, f, baseline, u0=None, v0=None, d_min=1.0, xyz=None):
    """Step 5b: points float32 [B,H,W,3]; u0/v0 default to the image centre."""
    if disparity.dim() == 2:
        disparity = disparity.unsqueeze(0)
    B, H, W = disparity.shape
    u0 = (W - 1) / 2.0 if u0 is None else u0
    v0 = (H - 1) / 2.0 if v0 is None else v0
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    xyz = torch.empty((B, H, W, 3), dtype=torch.float32, device=disparity.device) if xyz is None else xyz
    _expect(xyz, torch.float32, (B, H, W, 3), "xyz")
    check("rsr_reconstruct", lib().rsr_reconstruct(
        RsrShape(B, H, W), RsrRig(f, baseline, u0, v0, d_min), _ptr(disparity), _ptr(xyz), _stream()))
    return xyz


def rsr_road_model(disparity, step_u=4, step_v=4, n_hyp=512, inlier_tol=0.5, seed=0, model=None,
                   workspace=None):
    """Road model (Eq. 2): RANSAC-LSF of d = alpha v + beta over grid samples of
    [B,H,W] disparity maps; returns float64 [B,3] = (alpha, beta, inliers)."""
    if disparity.dim() == 2:
        disparity = disparity.unsqueeze(0)
    B, H, W = disparity.shape
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    s = RsrShape(B, H, W)
    p = RsrRoadParams(step_u, step_v, n_hyp, float(inlier_tol), seed & 0xFFFFFFFF)
    dev = disparity.device
    model = torch.empty((B, 3), dtype=torch.float64, device=dev) if model is None else model
    _expect(model, torch.float64, (B, 3), "model")
    nbytes = int(lib().rsr_road_workspace_size(s, p))
    if workspace is None:
        workspace = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    if workspace.dtype != torch.uint8 or workspace.dim() != 1 or workspace.numel() < nbytes:
        raise ValueError(f"rsr: workspace must be a uint8 vector of >= {nbytes} bytes")
    check("rsr_road_model", lib().rsr_road_model(s, p, _ptr(disparity), _ptr(model), _ptr(workspace),
                                                 workspace.numel(), _stream()))
    return model


def rsr_road_roll(disparity, u0, u1, v0, v1, out=None):
    """Roll angle: plane fit over the patch [v0,v1) x [u0,u1); float64 [B,5] =
    (g0, g1, g2, gamma, n)."""
    if disparity.dim() == 2:
        disparity = disparity.unsqueeze(0)
    B, H, W = disparity.shape
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    out = torch.empty((B, 5), dtype=torch.float64, device=disparity.device) if out is None else out
    _expect(out, torch.float64, (B, 5), "out")
    check("rsr_road_roll", lib().rsr_road_roll(RsrShape(B, H, W), u0, u1, v0, v1, _ptr(disparity), _ptr(out),
                                               _stream()))
    return out


def rsr_plane_fit(corners, plane=None):
    """Accuracy evaluation: total-least-squares ground plane of each frame's
    corners, float64 [B,K,3] (K >= 3) -> float64 [B,4] = (n0, n1, n2, n3), NaN if degenerate."""
    if corners.dim() == 2:
        corners = corners.unsqueeze(0)
    B, K, _ = corners.shape
    _expect(corners, torch.float64, (B, K, 3), "corners")
    plane = torch.empty((B, 4), dtype=torch.float64, device=corners.device) if plane is None else plane
    _expect(plane, torch.float64, (B, 4), "plane")
    check("rsr_plane_fit", lib().rsr_plane_fit(B, K, _ptr(corners), _ptr(plane), _stream()))
    return plane


def rsr_plane_distance(plane, xyz, dist=None):
    """Signed distance of every reconstructed point (float32 [B,H,W,3]) to its frame's
    plane (float64 [B,4]): float32 [B,H,W], positive on the camera side."""
    if xyz.dim() == 3:
        xyz = xyz.unsqueeze(0)
    B, H, W, _ = xyz.shape
    plane = plane.reshape(-1, 4)
    _expect(xyz, torch.float32, (B, H, W, 3), "xyz")
    _expect(plane, torch.float64, (B, 4), "plane")
    dist = torch.empty((B, H, W), dtype=torch.float32, device=xyz.device) if dist is None else dist
    _expect(dist, torch.float32, (B, H, W), "dist")
    check("rsr_plane_distance", lib().rsr_plane_distance(RsrShape(B, H, W), _ptr(plane), _ptr(xyz), _ptr(dist),
                                                         _stream()))
    return dist


def rsr_search_range(disparity, shift, delta, d_lo_limit, d_hi_limit, out=None):
    """Restricted search range: per-frame residual band [d_lo, d_hi] of the
    previous frame's disparities (float32 [B,H,W]) around the next frame's shifts
    (int32 [B,H]); int32 [B,2]."""
    if disparity.dim() == 2:
        disparity = disparity.unsqueeze(0)
    B, H, W = disparity.shape
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    shift = shift.reshape(B, H)
    _expect(shift, torch.int32, (B, H), "shift")
    out = torch.empty((B, 2), dtype=torch.int32, device=disparity.device) if out is None else out
    _expect(out, torch.int32, (B, 2), "out")
    check("rsr_search_range", lib().rsr_search_range(RsrShape(B, H, W), _ptr(disparity), _ptr(shift), int(delta),
                                                     int(d_lo_limit), int(d_hi_limit), _ptr(out), _stream()))
    return out


# --------------------------------------------------------------------------- #
# Interpolating-warp variant (NEXT row f2; include/rsr.h, reading 21)
# --------------------------------------------------------------------------- #
def rsr_warp_linear(target, alpha_beta, warped=None, valid=None, shift=None):
    """Step 1' (linear interpolation at 1/256-px positions): returns (warped uint16
    [B,H,W] in 8.8 fixed point, valid uint8 [B,H,W], shift float64 [B,H] = t_q(v))."""
    target, s = _bhw(target)
    B, H, W = target.shape
    _expect(target, torch.uint8, (B, H, W), "target")
    alpha_beta = alpha_beta.reshape(B, 2)
    _expect(alpha_beta, torch.float64, (B, 2), "alpha_beta")
    dev = target.device
    warped = torch.empty((B, H, W), dtype=torch.uint16, device=dev) if warped is None else warped
    valid = torch.empty_like(target) if valid is None else valid
    shift = torch.empty((B, H), dtype=torch.float64, device=dev) if shift is None else shift
    _expect(warped, torch.uint16, (B, H, W), "warped")
    _expect(valid, torch.uint8, (B, H, W), "valid")
    _expect(shift, torch.float64, (B, H), "shift")
    check("rsr_warp_linear", lib().rsr_warp_linear(s, _ptr(alpha_beta), _ptr(target), _ptr(warped), _ptr(valid),
                                                   _ptr(shift), _stream()))
    return warped, valid, shift


def rsr_cost_volume_linear(ref, warped, valid, rho_block, d_lo, d_hi, *, with_tar=True, with_nan_maps=True,
                           vol_ref=None, vol_tar=None, nan_ref=None, nan_tar=None, workspace=None):
    """Step 2 on (uint8 ref, uint16 8.8 warped): (vol_ref, vol_tar|None, nan_ref|None, nan_tar|None)."""
    ref, s = _bhw(ref)
    B, H, W = ref.shape
    warped, _ = _bhw(warped)
    valid, _ = _bhw(valid)
    D = d_hi - d_lo + 1
    if D < 1:
        raise ValueError(f"rsr: empty search range [{d_lo}, {d_hi}]")
    _expect(ref, torch.uint8, (B, H, W), "ref")
    _expect(warped, torch.uint16, (B, H, W), "warped")
    _expect(valid, torch.uint8, (B, H, W), "valid")
    dev = ref.device
    if vol_ref is None:
        vol_ref = torch.empty((B, H, W, D), dtype=torch.float32, device=dev)
    if with_tar and vol_tar is None:
        vol_tar = torch.empty((B, H, W, D), dtype=torch.float32, device=dev)
    if with_nan_maps:
        nan_ref = torch.empty((B, H, W), dtype=torch.uint8, device=dev) if nan_ref is None else nan_ref
        if with_tar and nan_tar is None:
            nan_tar = torch.empty((B, H, W), dtype=torch.uint8, device=dev)
    nbytes = cost_workspace_bytes(B, H, W)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for t, name in ((vol_ref, "vol_ref"), (vol_tar, "vol_tar")):
        _expect(t, torch.float32, (B, H, W, D), name)
    for t, name in ((nan_ref, "nan_ref"), (nan_tar, "nan_tar")):
        _expect(t, torch.uint8, (B, H, W), name)
    if workspace.dtype != torch.uint8 or workspace.dim() != 1 or workspace.numel() < nbytes:
        raise ValueError(f"rsr: workspace must be a uint8 vector of >= {nbytes} bytes")
    check("rsr_cost_volume_linear", lib().rsr_cost_volume_linear(
        s, RsrCostParams(rho_block, d_lo, d_hi), _ptr(ref), _ptr(warped), _ptr(valid), _ptr(vol_ref),
        _ptr(vol_tar), _ptr(nan_ref), _ptr(nan_tar), _ptr(workspace), workspace.numel(), _stream()))
    return vol_ref, vol_tar, nan_ref, nan_tar


def rsr_aggregate_linear(vol, guide, rho, gamma_d, gamma_r, nan_map=None, out=None, concurrency=1):
    """Step 3 with a uint16 8.8 fixed-point guide (the target volume of the interpolating warp)."""
    guide, s = _bhw(guide)
    B, H, W = guide.shape
    if vol.dim() == 3:
        vol = vol.unsqueeze(0)
    D = vol.shape[-1]
    _expect(guide, torch.uint16, (B, H, W), "guide")
    _expect(vol, torch.float32, (B, H, W, D), "vol")
    out = torch.empty_like(vol) if out is None else out
    _expect(out, torch.float32, (B, H, W, D), "out")
    if out.data_ptr() == vol.data_ptr():
        raise ValueError("rsr: out must not alias vol")
    if nan_map is not None:
        nan_map, _ = _bhw(nan_map)
        _expect(nan_map, torch.uint8, (B, H, W), "nan_map")
    check("rsr_aggregate_linear", lib().rsr_aggregate_linear(
        s, D, RsrAggParams(rho, float(gamma_d), float(gamma_r), int(concurrency)), _ptr(vol), _ptr(guide),
        _ptr(nan_map), _ptr(out), _stream()))
    return out


def rsr_disparity_linear(agg_ref, agg_tar, shift, d_lo, d_hi, lrc_tol, subpixel=True, disparity=None,
                         wta_ref=None, wta_tar=None, with_wta=False):
    """Steps 4-5 with the fp64 applied shift t_q(v) (float64 [B,H]) of rsr_warp_linear."""
    if agg_ref.dim() == 3:
        agg_ref, agg_tar = agg_ref.unsqueeze(0), agg_tar.unsqueeze(0)
    B, H, W, D = agg_ref.shape
    if D != d_hi - d_lo + 1:
        raise ValueError(f"rsr: volumes hold D = {D} disparities, range [{d_lo}, {d_hi}] needs {d_hi - d_lo + 1}")
    _expect(agg_ref, torch.float32, (B, H, W, D), "agg_ref")
    _expect(agg_tar, torch.float32, (B, H, W, D), "agg_tar")
    shift = shift.reshape(B, H)
    _expect(shift, torch.float64, (B, H), "shift")
    dev = agg_ref.device
    disparity = torch.empty((B, H, W), dtype=torch.float32, device=dev) if disparity is None else disparity
    if with_wta:
        wta_ref = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_ref is None else wta_ref
        wta_tar = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_tar is None else wta_tar
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    _expect(wta_ref, torch.int16, (B, H, W), "wta_ref")
    _expect(wta_tar, torch.int16, (B, H, W), "wta_tar")
    check("rsr_disparity_linear", lib().rsr_disparity_linear(
        RsrShape(B, H, W), RsrDispParams(d_lo, d_hi, lrc_tol, 1 if subpixel else 0), _ptr(agg_ref),
        _ptr(agg_tar), _ptr(shift), _ptr(disparity), _ptr(wta_ref), _ptr(wta_tar), _stream()))
    return disparity, wta_ref, wta_tar


# --------------------------------------------------------------------------- #
# Fused, volume-free matching (NEXT row f1; include/rsr.h rsr_match)
# --------------------------------------------------------------------------- #
def rsr_match(ref, warped, valid, shift, rho_block, d_lo, d_hi, rho, gamma_d, gamma_r, lrc_tol, subpixel=True,
              disparity=None, wta_ref=None, wta_tar=None, with_wta=False, workspace=None):
    """Steps 2-5a fused (D <= 8): disparity float32 [B,H,W] (+ wta maps), bitwise equal to
    rsr_cost_volume -> rsr_aggregate x2 -> rsr_disparity."""
    ref, s = _bhw(ref)
    B, H, W = ref.shape
    warped, _ = _bhw(warped)
    valid, _ = _bhw(valid)
    _expect(ref, torch.uint8, (B, H, W), "ref")
    _expect(warped, torch.uint8, (B, H, W), "warped")
    _expect(valid, torch.uint8, (B, H, W), "valid")
    shift = shift.reshape(B, H)
    _expect(shift, torch.int32, (B, H), "shift")
    dev = ref.device
    disparity = torch.empty((B, H, W), dtype=torch.float32, device=dev) if disparity is None else disparity
    if with_wta:
        wta_ref = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_ref is None else wta_ref
        wta_tar = torch.empty((B, H, W), dtype=torch.int16, device=dev) if wta_tar is None else wta_tar
    _expect(disparity, torch.float32, (B, H, W), "disparity")
    _expect(wta_ref, torch.int16, (B, H, W), "wta_ref")
    _expect(wta_tar, torch.int16, (B, H, W), "wta_tar")
    nbytes = cost_workspace_bytes(B, H, W)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    if workspace.dtype != torch.uint8 or workspace.dim() != 1 or workspace.numel() < nbytes:
        raise ValueError(f"rsr: workspace must be a uint8 vector of >= {nbytes} bytes")
    check("rsr_match", lib().rsr_match(
        s, RsrCostParams(rho_block, d_lo, d_hi), RsrAggParams(rho, float(gamma_d), float(gamma_r), 1),
        RsrDispParams(d_lo, d_hi, lrc_tol, 1 if subpixel else 0), _ptr(ref), _ptr(warped), _ptr(valid),
        _ptr(shift), _ptr(disparity), _ptr(wta_ref), _ptr(wta_tar), _ptr(workspace), workspace.numel(),
        _stream()))
    return disparity, wta_ref, wta_tar
