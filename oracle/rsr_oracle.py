"""CPU fp64 oracle of the road-surface stereo hot path (arXiv 1807.07433).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import, call or
execute anything under ``oracle/``.  The product path (``paper_1807_07433_b200``)
never imports it and shares no code with it.

Every function is the plain definition of one step, written from PAPER.md
(``P:NN`` = line NN of /root/reference/PAPER.md) in the paper's order, in fp64,
with NumPy slicing over pixels (no blocking, fusion or reordering beyond what
the definition states).  Where the paper is silent the reading taken is the one
of SURVEY.md §8(c) (listed in DESIGN.md "Readings"), cited as "reading N".

Layout (oracle-internal): volumes are [D, H, W] (disparity slice k = r - d_lo),
maps are [H, W].  Invalid entries are NaN (float) or -1 (index maps).

Pins: tests/test_oracle_pins.py (closed forms, invariants, library routines,
brute force on tiny inputs, ground truth).  No function here is "parity
unpinned" except where its docstring says so.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "road_shift", "warp_target", "block_sums", "ncc_at", "cost_volumes",
    "bilateral_weight", "aggregate", "wta", "lr_check", "subpixel",
    "postprocess", "triangulate", "mde_per_second", "run_pipeline",
]


# --------------------------------------------------------------------------- #
# Step 1 — perspective transformation (Eq. (2))
# --------------------------------------------------------------------------- #
def road_shift(alpha: float, beta: float, height: int) -> np.ndarray:
    """s(v) = floor(alpha*v + beta + 1/2), int64 [H].

    P:78: "each point on row v in the target image is shifted alpha_0 + alpha_1 v
    - delta pixels to the right".  alpha = slope (paper alpha_1), beta =
    intercept (paper alpha_0) (reading 3); delta is absorbed into the signed
    residual range (reading 2); the shift is rounded half up to an integer
    (reading 1), evaluated as an fp64 multiply then two fp64 adds (NumPy
    evaluates each binary operation separately, no FMA contraction).
    """
    v = np.arange(height, dtype=np.float64)
    t = alpha * v          # fp64 multiply
    t = t + beta           # fp64 add
    t = t + 0.5            # fp64 add
    return np.floor(t).astype(np.int64)


def warp_target(target: np.ndarray, alpha: float, beta: float):
    """Warped target W(u, v) = T(u - s(v), v); validity M = [0 <= u - s(v) < W].

    P:78 (shift row v to the right by s(v)).  Columns with no source pixel get
    W = 0 and M = 0 (reading 7).  Returns (W uint8 [H,W], M uint8 [H,W], s int64 [H]).
    """
    h, w = target.shape
    s = road_shift(alpha, beta, h)
    warped = np.zeros_like(target)
    mask = np.zeros((h, w), dtype=np.uint8)
    u = np.arange(w)
    for v in range(h):
        src = u - s[v]
        ok = (src >= 0) & (src < w)
        warped[v, ok] = target[v, src[ok]]
        mask[v, ok] = 1
    return warped, mask, s


# --------------------------------------------------------------------------- #
# Step 2 — NCC cost volumes (Eqs. (3)-(5))
# --------------------------------------------------------------------------- #
def block_sums(img: np.ndarray, rho_b: int, mask: np.ndarray | None = None):
    """Per-pixel block sums over the (2 rho_b + 1)^2 block centred at (u, v).

    Returns (S, SS, ok): integer sums of i and i^2 (int64 [H,W]) and ok = block
    lies inside the image (and, if ``mask`` is given, mask == 1 over the whole
    block) (reading 7).  These are the ingredients of mu and sigma in Eqs. (4)-(5)
    ("mu_l and mu_r represent the means of the pixel intensities within
    the left and right blocks").  Direct summation (the paper's integral images,
    P:103, are an acceleration of the same sums).
    """
    h, w = img.shape
    p = rho_b
    x = img.astype(np.int64)
    pad = np.zeros((h + 2 * p, w + 2 * p), dtype=np.int64)
    pad[p:p + h, p:p + w] = x
    mpad = np.zeros((h + 2 * p, w + 2 * p), dtype=np.int64)
    mpad[p:p + h, p:p + w] = 1 if mask is None else mask.astype(np.int64)
    S = np.zeros((h, w), dtype=np.int64)
    SS = np.zeros((h, w), dtype=np.int64)
    mins = np.ones((h, w), dtype=np.int64)
    for dy in range(-p, p + 1):
        for dx in range(-p, p + 1):
            blk = pad[p + dy:p + dy + h, p + dx:p + dx + w]
            S += blk
            SS += blk * blk
            mins = np.minimum(mins, mpad[p + dy:p + dy + h, p + dx:p + dx + w])
    vv, uu = np.mgrid[0:h, 0:w]
    inside = (uu >= p) & (uu <= w - 1 - p) & (vv >= p) & (vv <= h - 1 - p)
    ok = inside & (mins == 1)
    return S, SS, ok


def _window(a, row0, nrows, col0, ncols, fill):
    """a[row0:row0+nrows, col0:col0+ncols] with out-of-image entries = fill."""
    h, w = a.shape
    out = np.full((nrows, ncols), fill, dtype=a.dtype)
    ra, rb = max(row0, 0), min(row0 + nrows, h)
    ca, cb = max(col0, 0), min(col0 + ncols, w)
    if ra < rb and ca < cb:
        out[ra - row0:rb - row0, ca - col0:cb - col0] = a[ra:rb, ca:cb]
    return out


def ncc_at(left, warped, mask, rho_b, r, v0, nv, u0, nu, stats=None):
    """NCC cost c(u, v, r) of Eq. (3) for left-block centres u in [u0, u0+nu),
    v in [v0, v0+nv).

    Eq. (3):  c = (sum i_l(x,y) i_r(x-d,y) - n mu_l mu_r) / (n sigma_l sigma_r)
    Eq. (4)-(5): sigma = sqrt(sum i^2 / n - mu^2), mu = block mean,
    n = (2 rho_b + 1)^2.  The left block is centred at (u, v), the (warped) right
    block at (u - r, v).  c is clamped to [-1, 1] (reading 8).
    Invalid (NaN): either block not fully inside the image, any warp-invalid
    pixel in the right block (reading 7), or sigma_l = 0 or sigma_r = 0, tested
    exactly on integers n*sum(i^2) - (sum i)^2 == 0 (reading 6).
    Returns float64 [nv, nu].  ``stats`` = (block_sums(left), block_sums(warped, mask)).
    """
    p = rho_b
    n = (2 * p + 1) ** 2
    if stats is None:
        stats = (block_sums(left, p), block_sums(warped, p, mask))
    (SL, SSL, okL), (SW, SSW, okW) = stats
    sl = _window(SL, v0, nv, u0, nu, 0)
    ssl = _window(SSL, v0, nv, u0, nu, 0)
    okl = _window(okL, v0, nv, u0, nu, False)
    sw = _window(SW, v0, nv, u0 - r, nu, 0)
    ssw = _window(SSW, v0, nv, u0 - r, nu, 0)
    okw = _window(okW, v0, nv, u0 - r, nu, False)

    # dot product sum over the block of i_l(x, y) * i_r(x - r, y)
    li = left.astype(np.int64)
    wi = warped.astype(np.int64)
    dot = np.zeros((nv, nu), dtype=np.int64)
    for dy in range(-p, p + 1):
        for dx in range(-p, p + 1):
            dot += (_window(li, v0 + dy, nv, u0 + dx, nu, 0)
                    * _window(wi, v0 + dy, nv, u0 - r + dx, nu, 0))

    valid = okl & okw & (n * ssl - sl * sl != 0) & (n * ssw - sw * sw != 0)
    mu_l = sl / n
    mu_r = sw / n
    with np.errstate(invalid="ignore", divide="ignore"):
        sig_l = np.sqrt(np.maximum(ssl / n - mu_l * mu_l, 0.0))
        sig_r = np.sqrt(np.maximum(ssw / n - mu_r * mu_r, 0.0))
        c = (dot - n * mu_l * mu_r) / (n * sig_l * sig_r)
    c = np.clip(c, -1.0, 1.0)
    return np.where(valid, c, np.nan)


def cost_volumes(left, warped, mask, rho_b, d_lo, d_hi, rows=None):
    """Reference and target cost volumes C_L, C_R (float64 [D, r1-r0, W]) for
    image rows rows = (r0, r1) (default all).

    P:106: "Each computed correlation cost c is stored in two 3-D cost volumes
    ... the value of c at the position of (u, v, d) in the reference cost volume
    is the same as that at the position of (u - d, v, d) in the target cost volume."
    C_L[k, v, u] = c(u, v, r) and, computed independently (reading 9),
    C_R[k, v, u'] = c(u' + r, v, r), for r = d_lo + k.
    """
    h, w = left.shape
    r0, r1 = (0, h) if rows is None else rows
    D = d_hi - d_lo + 1
    stats = (block_sums(left, rho_b), block_sums(warped, rho_b, mask))
    cl = np.empty((D, r1 - r0, w))
    cr = np.empty((D, r1 - r0, w))
    for k in range(D):
        r = d_lo + k
        cl[k] = ncc_at(left, warped, mask, rho_b, r, r0, r1 - r0, 0, w, stats)
        cr[k] = ncc_at(left, warped, mask, rho_b, r, r0, r1 - r0, r, w, stats)
    return cl, cr


# --------------------------------------------------------------------------- #
# Step 3 — bilateral cost aggregation (Eqs. (8)-(10))
# --------------------------------------------------------------------------- #
def bilateral_weight(dx, dy, g_q, g_p, gamma_d, gamma_r):
    """omega_d * omega_r of Eqs. (9)-(10), literally exp(-x^2/gamma^2)
    (no factor 2, reading 10).  gamma_r = +inf gives omega_r = 1."""
    wd = np.exp(-(dx * dx + dy * dy) / (gamma_d * gamma_d))
    diff = np.asarray(g_q, dtype=np.float64) - np.asarray(g_p, dtype=np.float64)
    if math.isinf(gamma_r):
        wr = np.ones_like(diff)
    else:
        wr = np.exp(-(diff * diff) / (gamma_r * gamma_r))
    return wd * wr


def aggregate(vol, guide, rho, gamma_d, gamma_r, vol_row0=0, out_rows=None):
    """c_agg(u, v, d) of Eq. (8) for every slice k.

    c_agg = sum omega_d omega_r c / sum omega_d omega_r over the (2 rho + 1)^2
    window, omega from Eqs. (9)-(10) with guide i = ``guide`` (reading 11: L for
    C_L, W for C_R).  Taps outside the image or with NaN cost are skipped; the
    output is NaN iff the centre cost is NaN (reading 12).

    ``vol``: float [D, Hv, W] holding image rows [vol_row0, vol_row0 + Hv);
    ``out_rows``: image rows to produce (default: all rows held).  The caller
    must provide every row within rho of ``out_rows`` that exists in the image.
    Returns float64 [D, len(out_rows), W].
    """
    D, hv, w = vol.shape
    h = guide.shape[0]
    if out_rows is None:
        out_rows = np.arange(vol_row0, vol_row0 + hv)
    out_rows = np.asarray(out_rows, dtype=np.int64)
    g = guide.astype(np.float64)
    num = np.zeros((D, len(out_rows), w))
    den = np.zeros((D, len(out_rows), w))
    vv = out_rows
    for dy in range(-rho, rho + 1):
        q_rows = vv + dy
        row_in = (q_rows >= 0) & (q_rows < h)
        assert np.all(~row_in | ((q_rows >= vol_row0) & (q_rows < vol_row0 + hv))), "band too small"
        for dx in range(-rho, rho + 1):
            u = np.arange(w)
            q_cols = u + dx
            col_in = (q_cols >= 0) & (q_cols < w)
            inside = np.outer(row_in, col_in)
            qr = np.clip(q_rows, 0, h - 1)
            qc = np.clip(q_cols, 0, w - 1)
            gq = g[np.ix_(qr, qc)]
            gp = g[vv][:, :]
            wgt = np.where(inside, bilateral_weight(dx, dy, gq, gp, gamma_d, gamma_r), 0.0)
            x = vol[:, np.clip(q_rows - vol_row0, 0, hv - 1)][:, :, qc]
            valid = ~np.isnan(x) & inside[None]
            num += np.where(valid, wgt[None] * np.where(valid, x, 0.0), 0.0)
            den += np.where(valid, wgt[None], 0.0)
    centre = vol[:, out_rows - vol_row0]
    with np.errstate(invalid="ignore", divide="ignore"):
        out = num / den
    return np.where(np.isnan(centre), np.nan, out)


# --------------------------------------------------------------------------- #
# Step 4 — WTA and left-right consistency (Eq. (11))
# --------------------------------------------------------------------------- #
def wta(agg):
    """Winner-take-all: k(u, v) = smallest index attaining the maximum correlation
    over non-NaN entries ("highest correlation"; reading 5); -1 if all
    entries are NaN.  agg: [D, H, W] -> int64 [H, W]."""
    filled = np.where(np.isnan(agg), -np.inf, agg)
    k = np.argmax(filled, axis=0)  # first occurrence of the maximum
    none = np.all(np.isnan(agg), axis=0)
    return np.where(none, -1, k).astype(np.int64)


def lr_check(k_ref, k_tar, d_lo, tol):
    """Uniqueness constraint Eq. (11): l_ref(u,v) = l_tar(u - l_ref(u,v), v),
    with tolerance |k_L - k_R| <= tol (reading 13).  Keeps (u, v) iff k_L >= 0,
    u' = u - (k_L + d_lo) lies in [0, W), k_R(u', v) >= 0 and the tolerance holds.
    Returns bool [H, W]."""
    h, w = k_ref.shape
    vv, uu = np.mgrid[0:h, 0:w]
    up = uu - (k_ref + d_lo)
    inside = (k_ref >= 0) & (up >= 0) & (up < w)
    kr = np.where(inside, k_tar[vv, np.clip(up, 0, w - 1)], -1)
    return inside & (kr >= 0) & (np.abs(k_ref - kr) <= tol)


# --------------------------------------------------------------------------- #
# Step 5 — subpixel refinement, post-processing, triangulation
# --------------------------------------------------------------------------- #
def subpixel(agg, k_map, d_lo):
    """Eq. (12): d_s = d + (c(d-1) - c(d+1)) / (2c(d-1) + 2c(d+1) - 4c(d)),
    on the aggregated reference volume (reading 14).  Integer d kept at k = 0 or
    D-1, with a NaN neighbour, or with |den| <= 1e-12.  Returns float64 [H, W]
    residual disparity r_s (NaN where k < 0)."""
    D, h, w = agg.shape
    vv, uu = np.mgrid[0:h, 0:w]
    k = k_map
    r = np.where(k >= 0, (k + d_lo).astype(np.float64), np.nan)
    inner = (k >= 1) & (k <= D - 2)
    a = np.where(inner, agg[np.clip(k - 1, 0, D - 1), vv, uu], np.nan)
    b = np.where(inner, agg[np.clip(k, 0, D - 1), vv, uu], np.nan)
    c = np.where(inner, agg[np.clip(k + 1, 0, D - 1), vv, uu], np.nan)
    den = 2.0 * a + 2.0 * c - 4.0 * b
    ok = inner & ~np.isnan(a) & ~np.isnan(c) & (np.abs(den) > 1e-12)
    with np.errstate(invalid="ignore", divide="ignore"):
        off = (a - c) / den
    return np.where(ok, r + off, r)


def postprocess(r_s, keep, shift):
    """"the estimated subpixel disparities on row v should be added
    alpha_0 + alpha_1 v - delta"; here the same integer s(v) the warp used
    (reading 1).  NaN where the LR check rejected the pixel."""
    d = r_s + shift[:, None].astype(np.float64)
    return np.where(keep, d, np.nan)


def triangulate(disp, focal, baseline, u0, v0, d_min):
    """P:185-188 (no formula given): rectified pinhole, reading 15:
    Z = f b / d, X = (u - u0) Z / f, Y = (v - v0) Z / f; NaN unless d > d_min.
    Returns float64 [H, W, 3]."""
    h, w = disp.shape
    vv, uu = np.mgrid[0:h, 0:w].astype(np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        z = focal * baseline / disp
        x = (uu - u0) * z / focal
        y = (vv - v0) * z / focal
    ok = ~np.isnan(disp) & (disp > d_min)
    xyz = np.stack([x, y, z], axis=-1)
    return np.where(ok[..., None], xyz, np.nan)


def mde_per_second(width, height, d_max, seconds):
    """Eq. (13): Mde/s = u_max v_max d_max / t * 1e-6."""
    return width * height * d_max / seconds * 1e-6


# --------------------------------------------------------------------------- #
# Whole path, in the paper's order (Fig. 1)
# --------------------------------------------------------------------------- #
def run_pipeline(left, right, alpha, beta, cfg, rows=None, keep_volumes=True):
    """Run steps 1-5 for image rows ``rows`` (default all; a contiguous range).

    Intermediate rows needed by the windows (rho + rho_b above/below) are computed
    from the full images, so a row band gives exactly the full-image result on
    its rows.  ``cfg`` needs d_lo, d_hi, rho_block, rho_agg, gamma_d, gamma_r,
    lrc_tol, focal, baseline.  Returns a dict of float64/int64 arrays.
    """
    h, w = left.shape
    if rows is None:
        rows = (0, h)
    r0, r1 = rows
    rho = cfg.rho_agg
    warped, mask, s = warp_target(right, alpha, beta)
    a0, a1 = max(0, r0 - rho), min(h, r1 + rho)
    cl, cr = cost_volumes(left, warped, mask, cfg.rho_block, cfg.d_lo, cfg.d_hi, (a0, a1))
    out_rows = np.arange(r0, r1)
    al = aggregate(cl, left, rho, cfg.gamma_d, cfg.gamma_r, vol_row0=a0, out_rows=out_rows)
    ar = aggregate(cr, warped, rho, cfg.gamma_d, cfg.gamma_r, vol_row0=a0, out_rows=out_rows)
    kl = wta(al)
    kr = wta(ar)
    keep = lr_check(kl, kr, cfg.d_lo, cfg.lrc_tol)
    rs = subpixel(al, kl, cfg.d_lo)
    disp = postprocess(rs, keep, s[r0:r1])
    u0, v0 = (w - 1) / 2.0, (h - 1) / 2.0
    xyz = np.empty((r1 - r0, w, 3))
    zz = triangulate(disp, cfg.focal, cfg.baseline, u0, v0 - r0, 1.0)
    xyz[:] = zz
    res = dict(warped=warped, mask=mask, shift=s, k_ref=kl, k_tar=kr, keep=keep,
               r_sub=rs, disparity=disp, xyz=xyz, rows=(r0, r1))
    if keep_volumes:
        res.update(cost_ref=cl[:, r0 - a0:r1 - a0], cost_tar=cr[:, r0 - a0:r1 - a0],
                   agg_ref=al, agg_tar=ar)
    return res
