"""CPU fp64 oracle of the road-model estimation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and
bench-side tools, never by the product path.

P:71-77: for a rectified pair the road disparities follow Eq. (2),
d = alpha_0 + alpha_1 v, and "the latter can be estimated by solving a least
squares problem with a collection of reliable correspondence pairs"; the method
is named RANSAC-LSF.  The correspondences here are
samples (v, d) of a disparity map on a regular grid (every step_u-th column,
step_v-th row, finite entries only, row-major order) -- e.g. the previous
frame's map, or synthetic ground truth.  The paper fixes no RANSAC parameters
(S:172); DESIGN.md "Road model" states the reading:

* hypothesis h draws sample indices i = z(seed, 2h) mod n and j = z(seed, 2h+1)
  mod n (j = (j + 1) mod n if j == i) from the counter-based generator z
  (splitmix64 finaliser of (seed << 32) + counter, 64-bit wrap-around);
* the line through (v_i, d_i), (v_j, d_j): a = (d_j - d_i) / (v_j - v_i),
  b = d_i - a v_i (fp64; v_i == v_j is a degenerate hypothesis with no support);
* consensus: |d_k - (a v_k + b)| <= tol, each operation rounded in fp64;
* the best hypothesis has the most inliers, ties to the lowest index;
* the result is the least-squares line over its consensus set (normal
  equations in fp64): alpha = slope (the paper's alpha_1), beta = intercept
  (alpha_0), plus the consensus size.  NaN model if fewer than 2 inliers or a
  singular fit.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """splitmix64 finaliser (Steele et al.), integer arithmetic mod 2^64."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def draw_pair(seed: int, h: int, n: int) -> tuple[int, int]:
    """The two sample indices of hypothesis h (module docstring)."""
    base = (seed & 0xFFFFFFFF) << 32
    i = splitmix64(base + 2 * h) % n
    j = splitmix64(base + 2 * h + 1) % n
    if j == i:
        j = (j + 1) % n
    return i, j


def grid_samples(disparity: np.ndarray, step_u: int, step_v: int):
    """(v, d) of the finite entries of disparity[::step_v, ::step_u], row-major."""
    h, w = disparity.shape
    vv, uu = np.mgrid[0:h:step_v, 0:w:step_u]
    d = disparity[0:h:step_v, 0:w:step_u]
    ok = np.isfinite(d)
    return vv[ok].astype(np.float64), d[ok].astype(np.float64)


def consensus(v, d, a, b, tol):
    """Inlier mask |d - (a v + b)| <= tol (fp64, one rounding per operation)."""
    return np.abs(d - (a * v + b)) <= tol


def least_squares_line(v, d):
    """Slope and intercept minimising sum (d - (a v + b))^2 (normal equations)."""
    n = float(len(v))
    sv, sd = v.sum(), d.sum()
    svv, svd = (v * v).sum(), (v * d).sum()
    den = n * svv - sv * sv
    if len(v) < 2 or den == 0:
        return np.nan, np.nan
    a = (n * svd - sv * sd) / den
    b = (sd - a * sv) / n
    return a, b


def fit_road_model(v, d, n_hyp: int, tol: float, seed: int):
    """RANSAC-LSF (module docstring).  Returns (alpha, beta, inliers, best_h)."""
    n = len(v)
    if n < 2:
        return np.nan, np.nan, 0, -1
    best, best_h = -1, -1
    tol = float(np.float32(tol))   # the C ABI passes the threshold as fp32
    for h in range(n_hyp):
        i, j = draw_pair(seed, h, n)
        if v[i] == v[j]:
            continue
        a = (d[j] - d[i]) / (v[j] - v[i])
        b = d[i] - a * v[i]
        c = int(consensus(v, d, a, b, tol).sum())
        if c > best:
            best, best_h = c, h
    if best_h < 0:
        return np.nan, np.nan, 0, -1
    i, j = draw_pair(seed, best_h, n)
    a = (d[j] - d[i]) / (v[j] - v[i])
    b = d[i] - a * v[i]
    m = consensus(v, d, a, b, tol)
    if m.sum() < 2:
        return np.nan, np.nan, int(m.sum()), best_h
    al, be = least_squares_line(v[m], d[m])
    return al, be, int(m.sum()), best_h


def roll_plane_fit(disparity: np.ndarray, u0: int, u1: int, v0: int, v1: int):
    """Roll angle of the rig: least-squares plane d(u, v) = g0 + g1 u + g2 v
    over the finite disparities of the near-field patch [v0, v1) x [u0, u1), and
    gamma = arctan(-g1 / g2).  Normal equations in fp64, solved by Cramer's rule
    (the plain definition of the 3x3 solve).  Returns (g0, g1, g2, gamma, n);
    NaNs if fewer than 3 samples or a singular system."""
    vv, uu = np.mgrid[v0:v1, u0:u1]
    d = disparity[v0:v1, u0:u1].astype(np.float64)
    ok = np.isfinite(d)
    u, v, d = uu[ok].astype(np.float64), vv[ok].astype(np.float64), d[ok]
    n = len(d)
    if n < 3:
        return np.nan, np.nan, np.nan, np.nan, n
    M = np.array([[n, u.sum(), v.sum()],
                  [u.sum(), (u * u).sum(), (u * v).sum()],
                  [v.sum(), (u * v).sum(), (v * v).sum()]])
    r = np.array([d.sum(), (u * d).sum(), (v * d).sum()])
    det = np.linalg.det(M)
    if det == 0 or not np.isfinite(det):
        return np.nan, np.nan, np.nan, np.nan, n
    g = []
    for c in range(3):
        Mc = M.copy()
        Mc[:, c] = r
        g.append(np.linalg.det(Mc) / det)
    g0, g1, g2 = g
    return g0, g1, g2, float(np.arctan(-g1 / g2)), n
