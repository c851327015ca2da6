"""CPU oracle of the interpolating (sub-pixel) perspective transformation
(reading 21).  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py): only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference leg may use it.

P:78: "each point on row v in the target image is shifted alpha_0 + alpha_1 v
- delta pixels to the right".  The paper is silent on how a fractional shift
is realised (the main path rounds it to an integer, reading 1).  This variant
resamples the target image by linear interpolation along the row (SPEC S:162,
S:171) at a position quantised to 1/256 px, and stores the warped intensities
in 8.8 fixed point (uint16), so every sum of Eqs. (3)-(5) stays an exact
integer:

  t(v)  = alpha v + beta                         (fp64 multiply, then add)
  x     = u - t(v),  x0 = floor(x),  f = x - x0   (fp64; the subtraction is exact)
  q     = floor(256 f + 1/2)  in [0, 256];  q = 256 -> (x0 + 1, q = 0)
  W'(u) = (256 - q) T(x0) + q T(x0 + 1)          (exact integer, 0 .. 65280)
  M(u)  = 1 iff 0 <= x0 and (x0 + 1 <= W - 1, or q = 0 and x0 <= W - 1)
  W'(u) = 0 where M(u) = 0
  t_q(v) = u - (x0 + q / 256)                    (the shift actually applied; the
                                                  same for every u of the row)

so W'/256 is the linear interpolation of T at u - t_q(v).  Post-processing adds
back t_q(v), so the quantisation of the shift (|t_q - t| <= 1/512 px)
introduces no bias.  The NCC of Eq. (3) is invariant to the 256 scale of W'
(rsr_oracle.ncc_at works on any integer images); the bilateral range weight of
Eq. (10) on the target volume uses the guide W'/256 (real intensities).
"""
from __future__ import annotations

import math

import numpy as np

from . import rsr_oracle as O

__all__ = ["road_shift_frac", "warp_target_linear", "run_pipeline_linear"]


def road_shift_frac(alpha: float, beta: float, height: int) -> np.ndarray:
    """t(v) = alpha v + beta, fp64 [H] (P:78 without the rounding of reading 1)."""
    v = np.arange(height, dtype=np.float64)
    t = alpha * v      # fp64 multiply
    return t + beta    # fp64 add


def _row_position(t: float):
    """(x0, q) of column u = 0 for shift t: x = -t, x0 = floor(x), q = floor(256 f + 1/2)."""
    x = 0.0 - t
    x0 = math.floor(x)
    f = x - x0                       # exact: x0 is an integer no farther than 1 from x
    q = math.floor(f * 256.0 + 0.5)  # f * 256 is exact (power of two); one rounding in the add
    if q == 256:
        x0, q = x0 + 1, 0
    return x0, q


def warp_target_linear(target: np.ndarray, alpha: float, beta: float):
    """Returns (W' uint16 [H,W] 8.8 fixed point, M uint8 [H,W], t_q float64 [H])."""
    h, w = target.shape
    t = road_shift_frac(alpha, beta, h)
    T = target.astype(np.int64)
    out = np.zeros((h, w), dtype=np.uint16)
    mask = np.zeros((h, w), dtype=np.uint8)
    tq = np.empty(h, dtype=np.float64)
    u = np.arange(w)
    for v in range(h):
        x0_0, q = _row_position(float(t[v]))
        tq[v] = -(x0_0 + q / 256.0)          # u - (x0 + q/256) at u = 0; exact in fp64
        x0 = x0_0 + u
        if q == 0:
            ok = (x0 >= 0) & (x0 <= w - 1)
        else:
            ok = (x0 >= 0) & (x0 + 1 <= w - 1)
        a = T[v, np.clip(x0, 0, w - 1)]
        b = T[v, np.clip(x0 + 1, 0, w - 1)]
        val = (256 - q) * a + q * b
        out[v, ok] = val[ok]
        mask[v, ok] = 1
    return out, mask, tq


def run_pipeline_linear(left, right, alpha, beta, cfg, rows=None, keep_volumes=True):
    """Steps 1-5 with the interpolating warp, for image rows ``rows`` (default all).

    Same steps and readings as rsr_oracle.run_pipeline (Fig. 1); only step 1
    differs: W' from warp_target_linear, the target volume's guide is W'/256 and
    post-processing adds t_q(v).
    """
    h, w = left.shape
    if rows is None:
        rows = (0, h)
    r0, r1 = rows
    rho = cfg.rho_agg
    warped, mask, tq = warp_target_linear(right, alpha, beta)
    a0, a1 = max(0, r0 - rho), min(h, r1 + rho)
    cl, cr = O.cost_volumes(left, warped, mask, cfg.rho_block, cfg.d_lo, cfg.d_hi, (a0, a1))
    out_rows = np.arange(r0, r1)
    al = O.aggregate(cl, left, rho, cfg.gamma_d, cfg.gamma_r, vol_row0=a0, out_rows=out_rows)
    ar = O.aggregate(cr, warped.astype(np.float64) / 256.0, rho, cfg.gamma_d, cfg.gamma_r, vol_row0=a0,
                     out_rows=out_rows)
    kl = O.wta(al)
    kr = O.wta(ar)
    keep = O.lr_check(kl, kr, cfg.d_lo, cfg.lrc_tol)
    rs = O.subpixel(al, kl, cfg.d_lo)
    disp = O.postprocess(rs, keep, tq[r0:r1])
    u0, v0 = (w - 1) / 2.0, (h - 1) / 2.0
    xyz = O.triangulate(disp, cfg.focal, cfg.baseline, u0, v0 - r0, 1.0)
    res = dict(warped=warped, mask=mask, shift=tq, k_ref=kl, k_tar=kr, keep=keep,
               r_sub=rs, disparity=disp, xyz=xyz, rows=(r0, r1))
    if keep_volumes:
        res.update(cost_ref=cl[:, r0 - a0:r1 - a0], cost_tar=cr[:, r0 - a0:r1 - a0],
                   agg_ref=al, agg_tar=ar)
    return res
