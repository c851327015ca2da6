"""Seeded synthetic road-stereo inputs shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NO arithmetic of the method (no warp, no NCC, no aggregation,
no disparity selection).  It only renders input images and their ground truth,
following the workload recipe of BASELINE.json ``configs`` (SURVEY.md §8(d),
"Synthetic inputs" and "Generator details"):

* reference texture: 4-octave value noise (cells 16/8/4/2 px, amplitudes
  1, 1/2, 1/4, 1/8, bilinear lattice interpolation with smoothstep fade),
  affine-normalised to [40, 220];
* ground-truth disparity: road plane d(v) = alpha*v + beta plus Gaussian
  pothole depressions (amplitude -1.5 px, sigma 12 px) and optionally one crack
  (a 2-px-wide, -2 px groove);
* target image: linear resample of the clean texture at the correspondence
  u_r = u_l - d (x_l = x + d(x_l, v), 4 fixed-point iterations), optional
  gain/offset, plus independent Gaussian noise; both images rounded half-to-even
  and clipped to [0, 255] (SURVEY.md §8(c) reading 17).

The paper's own data (ZED road sequences [Fan2018]) is not in the
container; these shapes stand in for it.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = ["StereoConfig", "Frame", "CONFIGS", "get_config", "make_frame", "make_batch", "make_sequence",
           "box_disparity_gain"]


@dataclasses.dataclass(frozen=True)
class StereoConfig:
    """One BASELINE.json workload (plus the parameters SURVEY §8(c) reading 16 inherits)."""

    name: str
    height: int
    width: int
    alpha: float          # plane slope, px/row (paper's alpha_1)
    beta: float           # plane intercept, px (paper's alpha_0)
    d_lo: int             # residual search range [d_lo, d_hi] (reading 2)
    d_hi: int
    rho_block: int        # NCC half window varrho (Eq. 3)
    rho_agg: int          # bilateral half window rho (Eq. 8)
    gamma_d: float        # Eq. 9 (reading 10: gamma_d := sigma_s)
    gamma_r: float        # Eq. 10 (gamma_r := sigma_r)
    lrc_tol: int = 1      # |k_L - k_R| <= tol (reading 13)
    focal: float = 700.0  # px
    baseline: float = 0.12  # m
    n_potholes: int = 2
    crack: bool = False
    gain: float = 1.0     # target gain (config 3: 1.05)
    offset: float = 0.0   # target offset (config 3: +8)
    noise: float = 2.0    # Gaussian noise sigma on both images
    pothole_amp: float = -1.5
    pothole_sigma: float = 12.0
    seed: int = 1
    batch: int = 1
    random_plane: bool = False  # config 5: alpha~U[0.08,0.12], beta~U[25,35] per frame
    # accuracy scene (NEXT f4): a box ("sample model") of known height standing
    # on the road, (u0, v0, u1, v1, height_m) in reference-image pixels / metres
    box: tuple | None = None

    @property
    def D(self) -> int:
        return self.d_hi - self.d_lo + 1


CONFIGS = {
    "c1": StereoConfig("c1", 180, 320, 0.05, 10.0, -16, 15, 2, 4, 3.0, 10.0,
                       n_potholes=2, seed=1),
    "c2": StereoConfig("c2", 360, 640, 0.08, 20.0, -24, 23, 3, 5, 4.0, 10.0,
                       n_potholes=5, crack=True, seed=2),
    "c3": StereoConfig("c3", 720, 1280, 0.10, 30.0, -32, 31, 3, 6, 4.0, 12.0,
                       n_potholes=10, gain=1.05, offset=8.0, seed=3),
    "c4": StereoConfig("c4", 1080, 1920, 0.12, 40.0, -48, 47, 4, 7, 5.0, 12.0,
                       n_potholes=20, noise=3.0, seed=4),
    # config 5: 256 frames of the config-2 generator at 1280x720, per-frame plane
    "c5": StereoConfig("c5", 720, 1280, 0.10, 30.0, -32, 31, 3, 6, 4.0, 12.0,
                       n_potholes=5, crack=True, seed=5000, batch=256, random_plane=True),
    # the paper's own operating point: 1240x609, varrho=3, rho=4, d_max=30
    "cP": StereoConfig("cP", 609, 1240, 0.05, 10.0, -15, 14, 3, 4, 4.0, 12.0,
                       n_potholes=5, crack=True, seed=6),
}


def get_config(name: str, **overrides) -> StereoConfig:
    cfg = CONFIGS[name]
    return dataclasses.replace(cfg, **overrides) if overrides else cfg


@dataclasses.dataclass
class Frame:
    left: np.ndarray      # uint8 [H, W] reference image i_l
    right: np.ndarray     # uint8 [H, W] target image i_r (unwarped)
    alpha: float
    beta: float
    d_gt: np.ndarray      # float64 [H, W] ground-truth total disparity at reference pixels
    gt_exclude: np.ndarray  # bool [H, W] pixels excluded from accuracy stats (3-px crack band)


def _value_noise(rng: np.random.Generator, h: int, w: int) -> np.ndarray:
    tex = np.zeros((h, w), dtype=np.float64)
    for cell, amp in ((16, 1.0), (8, 0.5), (4, 0.25), (2, 0.125)):
        gh, gw = h // cell + 2, w // cell + 2
        lat = rng.random((gh, gw))
        yy = np.arange(h, dtype=np.float64) / cell
        xx = np.arange(w, dtype=np.float64) / cell
        iy = np.floor(yy).astype(np.int64)
        ix = np.floor(xx).astype(np.int64)
        fy = yy - iy
        fx = xx - ix
        sy = (fy * fy * (3.0 - 2.0 * fy))[:, None]
        sx = (fx * fx * (3.0 - 2.0 * fx))[None, :]
        a = lat[iy][:, ix]
        b = lat[iy][:, ix + 1]
        c = lat[iy + 1][:, ix]
        d = lat[iy + 1][:, ix + 1]
        tex += amp * ((1 - sy) * ((1 - sx) * a + sx * b) + sy * ((1 - sx) * c + sx * d))
    lo, hi = tex.min(), tex.max()
    return 40.0 + (tex - lo) * (180.0 / (hi - lo))


def box_disparity_gain(cfg: StereoConfig, alpha: float, beta: float, height_m: float) -> float:
    """Disparity gain kappa of the top face of a box of height h on the road plane.

    Scene geometry, not the method: with the rectified pinhole of reading 15
    (u0 = (W-1)/2, v0 = (H-1)/2), the road d = alpha v + beta is the 3-D plane
    alpha f Y + (alpha v0 + beta) Z = f b (normal norm |n|); the parallel plane
    at height h towards the camera projects to d' = kappa (alpha v + beta),
    kappa = f b / (f b - h |n|)."""
    v0 = (cfg.height - 1) / 2.0
    nrm = math.hypot(alpha * cfg.focal, alpha * v0 + beta)
    fb = cfg.focal * cfg.baseline
    return fb / (fb - height_m * nrm)


class _Scene:
    """Analytic ground-truth disparity d(x, v) over the reference view."""

    def __init__(self, cfg: StereoConfig, rng: np.random.Generator, alpha: float, beta: float):
        h, w = cfg.height, cfg.width
        self.alpha, self.beta = alpha, beta
        self.box = None
        if cfg.box is not None:
            u0, v0, u1, v1, hb = cfg.box
            self.box = (u0, v0, u1, v1, box_disparity_gain(cfg, alpha, beta, hb))
        s = cfg.pothole_sigma
        m = 3.0 * s
        self.pots = []
        for _ in range(cfg.n_potholes):
            cx = rng.uniform(m, w - 1 - m) if w - 1 > 2 * m else (w - 1) / 2
            cy = rng.uniform(m, h - 1 - m) if h - 1 > 2 * m else (h - 1) / 2
            self.pots.append((cx, cy))
        self.amp, self.sig = cfg.pothole_amp, s
        self.crack = None
        if cfg.crack:
            for _ in range(1000):
                p = rng.uniform([8, 8], [w - 9, h - 9])
                q = rng.uniform([8, 8], [w - 9, h - 9])
                if math.hypot(*(q - p)) >= w / 4:
                    break
            self.crack = (p, q)

    def _seg_dist(self, x, y):
        p, q = self.crack
        dx, dy = q[0] - p[0], q[1] - p[1]
        t = np.clip(((x - p[0]) * dx + (y - p[1]) * dy) / (dx * dx + dy * dy), 0.0, 1.0)
        return np.hypot(x - (p[0] + t * dx), y - (p[1] + t * dy))

    def disparity(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        d = self.alpha * y + self.beta
        if self.box is not None:
            u0, v0, u1, v1, kappa = self.box
            inside = (x >= u0) & (x < u1) & (y >= v0) & (y < v1)
            d = np.where(inside, kappa * d, d)
        for cx, cy in self.pots:
            d = d + self.amp * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2.0 * self.sig ** 2))
        if self.crack is not None:
            d = d + np.where(self._seg_dist(x, y) <= 1.0, -2.0, 0.0)
        return d

    def exclude(self, x, y):
        if self.crack is None:
            return np.zeros(np.broadcast(x, y).shape, dtype=bool)
        return self._seg_dist(x, y) <= 1.0 + 3.0


def make_frame(cfg: StereoConfig, index: int = 0) -> Frame:
    """Render frame ``index`` of ``cfg`` (seed = cfg.seed + index). Deterministic."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed + index))
    alpha, beta = cfg.alpha, cfg.beta
    if cfg.random_plane:
        alpha = float(rng.uniform(0.08, 0.12))
        beta = float(rng.uniform(25.0, 35.0))
    h, w = cfg.height, cfg.width
    # texture wide enough for x_l = x + d up to the largest disparity
    wt = _texture_width(cfg, alpha, beta)
    tex = _value_noise(rng, h, wt)
    scene = _Scene(cfg, rng, alpha, beta)
    return _render(cfg, rng, tex, scene, alpha, beta)


def _texture_width(cfg, alpha, beta):
    d_max_est = abs(alpha) * cfg.height + abs(beta) + 4.0
    if cfg.box is not None:
        d_max_est *= 1.2
    return cfg.width + int(math.ceil(d_max_est)) + 4


def _render(cfg, rng, tex, scene, alpha, beta) -> Frame:
    h, w = cfg.height, cfg.width
    wt = tex.shape[1]
    ys = np.arange(h, dtype=np.float64)[:, None]
    xs = np.arange(w, dtype=np.float64)[None, :]
    d_gt = scene.disparity(np.broadcast_to(xs, (h, w)), np.broadcast_to(ys, (h, w)))
    # correspondence for target column x: x_l = x + d(x_l, v)
    xl = xs + scene.disparity(np.broadcast_to(xs, (h, w)), np.broadcast_to(ys, (h, w)))
    for _ in range(4):
        xl = xs + scene.disparity(xl, np.broadcast_to(ys, (h, w)))
    xc = np.clip(xl, 0.0, wt - 1.0)
    i0 = np.floor(xc).astype(np.int64)
    i1 = np.minimum(i0 + 1, wt - 1)
    f = xc - i0
    rows = np.arange(h)[:, None]
    resampled = (1.0 - f) * tex[rows, i0] + f * tex[rows, i1]
    left_f = tex[:, :w] + rng.normal(0.0, cfg.noise, size=(h, w))
    right_f = cfg.gain * resampled + cfg.offset + rng.normal(0.0, cfg.noise, size=(h, w))
    left = np.clip(np.rint(left_f), 0, 255).astype(np.uint8)
    right = np.clip(np.rint(right_f), 0, 255).astype(np.uint8)
    excl = scene.exclude(np.broadcast_to(xs, (h, w)), np.broadcast_to(ys, (h, w)))
    return Frame(left, right, alpha, beta, d_gt, excl)


def make_sequence(cfg: StereoConfig, n: int, scroll: int = 3, dalpha: float = 1e-4, dbeta: float = 0.05):
    """A video-like sequence of n frames (restricted-search-range evaluation):
    the vehicle moves forward, so the road texture (and its potholes / crack)
    scrolls down by ``scroll`` rows per frame, and the road plane drifts slowly
    (alpha_t = alpha + t dalpha, beta_t = beta + t dbeta).  Fresh sensor noise per
    frame.  Deterministic in cfg.seed."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 7_000_000))
    h, w = cfg.height, cfg.width
    a_max, b_max = cfg.alpha + n * abs(dalpha), cfg.beta + n * abs(dbeta)
    wt = _texture_width(cfg, a_max, b_max)
    tall = _value_noise(rng, h + n * scroll, wt)
    base = _Scene(cfg, rng, cfg.alpha, cfg.beta)
    frames = []
    for t in range(n):
        alpha, beta = cfg.alpha + t * dalpha, cfg.beta + t * dbeta
        off = (n - 1 - t) * scroll               # texture window moves up: content moves down
        tex = tall[off:off + h]
        scene = _Scene.__new__(_Scene)
        scene.__dict__.update(base.__dict__)
        scene.alpha, scene.beta = alpha, beta
        scene.pots = [(cx, cy + t * scroll) for cx, cy in base.pots]
        if base.crack is not None:
            p, q = base.crack
            scene.crack = (p + np.array([0.0, t * scroll]), q + np.array([0.0, t * scroll]))
        frames.append(_render(cfg, rng, tex, scene, alpha, beta))
    return frames


def make_batch(cfg: StereoConfig, indices) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Stack frames: (left uint8 [B,H,W], right uint8 [B,H,W], alpha_beta float64 [B,2])."""
    frames = [make_frame(cfg, i) for i in indices]
    left = np.stack([f.left for f in frames])
    right = np.stack([f.right for f in frames])
    ab = np.array([[f.alpha, f.beta] for f in frames], dtype=np.float64)
    return left, right, ab


def tiny_pair(seed: int, h: int, w: int, shift: int = 2, noise: float = 2.0):
    """Small textured pair for brute-force tests: right = left shifted by ``shift`` px + noise."""
    rng = np.random.Generator(np.random.PCG64(seed))
    base = rng.uniform(30.0, 225.0, size=(h, w + abs(shift) + 2))
    left = base[:, :w] + rng.normal(0.0, noise, size=(h, w))
    right = base[:, shift + 1: shift + 1 + w] if shift >= 0 else base[:, :w]
    right = right + rng.normal(0.0, noise, size=(h, w))
    return (np.clip(np.rint(left), 0, 255).astype(np.uint8),
            np.clip(np.rint(right), 0, 255).astype(np.uint8))
