"""CPU fp64 oracle of the reconstruction-accuracy evaluation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and
bench-side tools, never by the product path.

P:198-200: "The four corners s_1 .. s_4 are interpolated into a ground plane
n_0 x + n_1 y + n_2 z + n_3 = 0 which is considered as the road surface.  Then,
we select some random 3-D points p_1 .. p_n on the surface of the model and
estimate the distances between them and the road surface."

Readings (reading 19):
* "interpolated into a ground plane" = the total-least-squares plane of the
  corners: the plane minimising the sum of squared orthogonal distances, i.e.
  unit normal n = the right singular vector of the centred corners with the
  smallest singular value, n_3 = -n . centroid;
* orientation: n_3 > 0 (the camera, at the origin of the reconstruction, lies
  on the positive side); if n_3 == 0, the last non-zero of (n_0, n_1, n_2) is
  made positive;
* the plane is NaN when a corner is not finite or the corners do not span a
  plane (fewer than 3 corners, or second singular value <= 1e-12 x the first);
* distance of a point p = n . p + n_3, signed (positive on the camera side:
  the height above the road for a rig looking down at it); NaN for a point with
  a non-finite coordinate.
"""
from __future__ import annotations

import numpy as np

DEGENERATE_REL = 1e-12


def fit_plane(corners) -> np.ndarray:
    """Total-least-squares plane (n0, n1, n2, n3) of k >= 3 corners [k, 3]."""
    c = np.asarray(corners, dtype=np.float64).reshape(-1, 3)
    nan = np.full(4, np.nan)
    if len(c) < 3 or not np.isfinite(c).all():
        return nan
    m = c.mean(axis=0)
    _, s, vt = np.linalg.svd(c - m)
    if s[0] == 0.0 or s[1] <= DEGENERATE_REL * s[0]:
        return nan
    n = vt[-1] / np.linalg.norm(vt[-1])
    n3 = -float(n @ m)
    flip = n3 < 0 or (n3 == 0 and n[np.flatnonzero(n)[-1]] < 0)
    if flip:
        n, n3 = -n, -n3
    return np.array([n[0], n[1], n[2], n3])


def point_plane_distance(plane, xyz) -> np.ndarray:
    """Signed distances n . p + n3 of points xyz [..., 3] (fp64)."""
    p = np.asarray(xyz, dtype=np.float64)
    pl = np.asarray(plane, dtype=np.float64)
    return p[..., 0] * pl[0] + p[..., 1] * pl[1] + p[..., 2] * pl[2] + pl[3]
