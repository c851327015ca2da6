"""Brute-force per-pixel pure-Python evaluation of the same definitions as
rsr_oracle.py, for tiny images only (16x16-class).  TEST INFRASTRUCTURE ONLY.

Written independently of the vectorised oracle (explicit loops over blocks,
windows and disparities, math.sqrt/math.exp per element) so that a slicing,
sign, offset or transposition mistake in either shows up as a disagreement
(SURVEY.md §8(c) "Whole pipeline, tiny"; BASELINE.json north_star "brute force
agrees on 16x16 images").
"""
from __future__ import annotations

import math


def warp(target, alpha, beta):
    """P:78 with readings 1-2: s(v) = floor(alpha v + beta + 0.5); W(u,v) = T(u - s(v), v)."""
    h, w = len(target), len(target[0])
    s = [math.floor((alpha * v + beta) + 0.5) for v in range(h)]
    W = [[0] * w for _ in range(h)]
    M = [[0] * w for _ in range(h)]
    for v in range(h):
        for u in range(w):
            src = u - s[v]
            if 0 <= src < w:
                W[v][u] = int(target[v][src])
                M[v][u] = 1
    return W, M, s


def ncc(L, W, M, rho_b, u, v, r):
    """Eq. (3)-(5) at left centre (u, v), right centre (u - r, v); NaN if invalid."""
    h, w = len(L), len(L[0])
    n = (2 * rho_b + 1) ** 2
    ur = u - r
    if not (rho_b <= u < w - rho_b and rho_b <= v < h - rho_b):
        return math.nan
    if not (rho_b <= ur < w - rho_b):
        return math.nan
    sl = ssl = sw = ssw = dot = 0
    for y in range(v - rho_b, v + rho_b + 1):
        for x in range(u - rho_b, u + rho_b + 1):
            a = int(L[y][x])
            xr = x - r
            if not M[y][xr]:
                return math.nan
            b = int(W[y][xr])
            sl += a
            ssl += a * a
            sw += b
            ssw += b * b
            dot += a * b
    if n * ssl - sl * sl == 0 or n * ssw - sw * sw == 0:
        return math.nan
    mu_l, mu_r = sl / n, sw / n
    sig_l = math.sqrt(ssl / n - mu_l * mu_l)
    sig_r = math.sqrt(ssw / n - mu_r * mu_r)
    c = (dot - n * mu_l * mu_r) / (n * sig_l * sig_r)
    return min(1.0, max(-1.0, c))


def volumes(L, W, M, rho_b, d_lo, d_hi):
    h, w = len(L), len(L[0])
    D = d_hi - d_lo + 1
    CL = [[[ncc(L, W, M, rho_b, u, v, d_lo + k) for u in range(w)] for v in range(h)] for k in range(D)]
    CR = [[[ncc(L, W, M, rho_b, u + d_lo + k, v, d_lo + k) for u in range(w)] for v in range(h)]
          for k in range(D)]
    return CL, CR


def aggregate(C, G, rho, gamma_d, gamma_r):
    """Eq. (8)-(10) with readings 10-12, one (k, v, u) at a time."""
    D, h, w = len(C), len(C[0]), len(C[0][0])
    out = [[[math.nan] * w for _ in range(h)] for _ in range(D)]
    for k in range(D):
        for v in range(h):
            for u in range(w):
                if math.isnan(C[k][v][u]):
                    continue
                num = den = 0.0
                for y in range(v - rho, v + rho + 1):
                    for x in range(u - rho, u + rho + 1):
                        if not (0 <= y < h and 0 <= x < w):
                            continue
                        c = C[k][y][x]
                        if math.isnan(c):
                            continue
                        wd = math.exp(-((x - u) ** 2 + (y - v) ** 2) / (gamma_d ** 2))
                        diff = float(G[y][x]) - float(G[v][u])
                        wr = 1.0 if math.isinf(gamma_r) else math.exp(-(diff * diff) / (gamma_r ** 2))
                        num += wd * wr * c
                        den += wd * wr
                out[k][v][u] = num / den
    return out


def wta(A):
    D, h, w = len(A), len(A[0]), len(A[0][0])
    K = [[-1] * w for _ in range(h)]
    for v in range(h):
        for u in range(w):
            best = None
            for k in range(D):
                a = A[k][v][u]
                if math.isnan(a):
                    continue
                if best is None or a > best:
                    best, K[v][u] = a, k
    return K


def disparity(AL, KL, KR, shift, d_lo, tol):
    """LR check (Eq. 11), parabola (Eq. 12), post-processing."""
    D, h, w = len(AL), len(AL[0]), len(AL[0][0])
    out = [[math.nan] * w for _ in range(h)]
    for v in range(h):
        for u in range(w):
            k = KL[v][u]
            if k < 0:
                continue
            up = u - (k + d_lo)
            if not (0 <= up < w) or KR[v][up] < 0 or abs(k - KR[v][up]) > tol:
                continue
            r = float(k + d_lo)
            if 1 <= k <= D - 2:
                a, b, c = AL[k - 1][v][u], AL[k][v][u], AL[k + 1][v][u]
                if not (math.isnan(a) or math.isnan(c)):
                    den = 2 * a + 2 * c - 4 * b
                    if abs(den) > 1e-12:
                        r += (a - c) / den
            out[v][u] = r + shift[v]
    return out


def triangulate(d, focal, baseline, u0, v0, d_min):
    h, w = len(d), len(d[0])
    out = [[[math.nan] * 3 for _ in range(w)] for _ in range(h)]
    for v in range(h):
        for u in range(w):
            if not math.isnan(d[v][u]) and d[v][u] > d_min:
                z = focal * baseline / d[v][u]
                out[v][u] = [(u - u0) * z / focal, (v - v0) * z / focal, z]
    return out


def run(left, right, alpha, beta, rho_b, rho, d_lo, d_hi, gamma_d, gamma_r, tol,
        focal=700.0, baseline=0.12):
    L = [[int(x) for x in row] for row in left]
    T = [[int(x) for x in row] for row in right]
    W, M, s = warp(T, alpha, beta)
    CL, CR = volumes(L, W, M, rho_b, d_lo, d_hi)
    AL = aggregate(CL, L, rho, gamma_d, gamma_r)
    AR = aggregate(CR, W, rho, gamma_d, gamma_r)
    KL, KR = wta(AL), wta(AR)
    d = disparity(AL, KL, KR, s, d_lo, tol)
    h, w = len(L), len(L[0])
    xyz = triangulate(d, focal, baseline, (w - 1) / 2, (h - 1) / 2, 1.0)
    return dict(warped=W, mask=M, shift=s, cost_ref=CL, cost_tar=CR, agg_ref=AL,
                agg_tar=AR, k_ref=KL, k_tar=KR, disparity=d, xyz=xyz)
