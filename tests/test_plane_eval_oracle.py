"""Pins of the reconstruction-accuracy oracle (oracle/plane_eval.py, NEXT row f4,
P:198-200): exact planes, rigid-motion invariance, the paper's box-height use,
an independent eigen-solver, TLS optimality and the degenerate cases."""
import numpy as np

from oracle import plane_eval as PE


def _rot(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def test_exact_plane_through_corners():
    # z = 2 + 0.1 x - 0.05 y  <=>  0.1 x - 0.05 y - z + 2 = 0
    xy = np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]])
    corners = np.c_[xy, 2 + 0.1 * xy[:, 0] - 0.05 * xy[:, 1]]
    pl = PE.fit_plane(corners)
    ref = np.array([0.1, -0.05, -1.0, 2.0]) / np.linalg.norm([0.1, -0.05, -1.0])
    assert np.allclose(pl, ref, atol=1e-14)
    assert pl[3] > 0                                       # camera (origin) on the + side
    assert np.allclose(PE.point_plane_distance(pl, corners), 0, atol=1e-14)


def test_box_height_on_the_road():
    # the paper's use: points on top of a printed model at height h above the plane
    rng = np.random.default_rng(0)
    R = _rot(rng)
    t = np.array([0.1, 0.3, 1.2])
    sq = np.array([[0, 0, 0], [0.4, 0, 0], [0.4, 0.3, 0], [0, 0.3, 0]], dtype=float)
    corners = sq @ R.T + t
    pl = PE.fit_plane(corners)
    n = pl[:3]
    h = 0.025
    top = (rng.uniform(0.1, 0.3, size=(50, 1)) * np.array([[1, 0, 0]]) +
           rng.uniform(0.05, 0.25, size=(50, 1)) * np.array([[0, 1, 0]])) @ R.T + t
    top = top + h * n
    assert np.allclose(PE.point_plane_distance(pl, top), h, atol=1e-13)
    assert np.allclose(PE.point_plane_distance(pl, top - 2 * h * n), -h, atol=1e-13)


def test_rigid_motion_invariance():
    rng = np.random.default_rng(1)
    c = rng.normal(size=(4, 3)) * [1.0, 1.0, 0.05]        # nearly planar
    pts = rng.normal(size=(20, 3))
    R, t = _rot(rng), rng.normal(size=3) + [0, 0, 5]
    d0 = PE.point_plane_distance(PE.fit_plane(c), pts)
    d1 = PE.point_plane_distance(PE.fit_plane(c @ R.T + t), pts @ R.T + t)
    # the orientation convention may flip the sign with the camera side
    assert np.allclose(np.abs(d0), np.abs(d1), atol=1e-12)


def test_normal_is_smallest_eigenvector_of_scatter():
    # independent routine: eigh of the scatter matrix (not the SVD the oracle uses)
    rng = np.random.default_rng(2)
    for _ in range(20):
        c = rng.normal(size=(4, 3))
        pl = PE.fit_plane(c)
        X = c - c.mean(0)
        w, v = np.linalg.eigh(X.T @ X)
        n = v[:, 0]
        assert abs(abs(n @ pl[:3]) - 1) < 1e-12
        assert abs(np.linalg.norm(pl[:3]) - 1) < 1e-14


def test_tls_optimality_against_perturbed_planes():
    rng = np.random.default_rng(3)
    c = rng.normal(size=(4, 3)) * [1, 1, 0.1]
    pl = PE.fit_plane(c)
    best = np.sum(PE.point_plane_distance(pl, c) ** 2)
    for _ in range(500):
        n = pl[:3] + rng.normal(scale=0.05, size=3)
        n /= np.linalg.norm(n)
        n3 = -n @ c.mean(0)               # the optimal offset for any normal
        assert np.sum((c @ n + n3) ** 2) >= best - 1e-15


def test_degenerate_corners():
    assert np.isnan(PE.fit_plane([[0, 0, 0], [1, 1, 1], [2, 2, 2], [3, 3, 3]])).all()   # collinear
    assert np.isnan(PE.fit_plane([[0, 0, 0], [1, 0, 0]])).all()                           # < 3
    assert np.isnan(PE.fit_plane([[0, 0, 0], [1, 0, 0], [0, 1, np.nan], [1, 1, 0]])).all()
    assert np.isnan(PE.fit_plane(np.ones((4, 3)))).all()                                  # one point
    # plane through the camera: n3 == 0, orientation by the last non-zero normal entry
    pl = PE.fit_plane([[1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0]])
    assert pl[3] == 0 and np.allclose(pl[:3], [0, 0, 1])
    d = PE.point_plane_distance(pl, np.array([[0, 0, np.nan]]))
    assert np.isnan(d).all()
