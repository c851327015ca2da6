"""Pins of the restricted-search-range oracle (oracle/search_range.py, NEXT row f4,
P:251): hand examples, the road plane, integer boundaries, clipping, empty maps."""
import numpy as np

from oracle import search_range as SR


def test_hand_example():
    d = np.array([[31.25, 30.5, np.nan], [35.0, 33.75, 34.0]])
    s = np.array([30, 33])
    # residuals 1.25, 0.5 | 2.0, 0.75, 1.0 -> floor 0, ceil 2
    assert SR.search_range(d, s, 0, -32, 31) == (0, 2)
    assert SR.search_range(d, s, 3, -32, 31) == (-3, 5)


def test_integer_residuals_are_their_own_bounds():
    d = np.array([[10.0, 12.0], [13.0, 11.0]])
    s = np.array([10, 10])
    assert SR.search_range(d, s, 0, -8, 7) == (0, 3)


def test_road_plane_residual_is_small():
    # d = alpha v + beta exactly; s(v) = floor(alpha v + beta + 0.5): |r| <= 0.5
    H, W = 720, 64
    v = np.arange(H, dtype=np.float64)
    d = np.repeat((0.1 * v + 30.0)[:, None], W, axis=1)
    s = np.floor(0.1 * v + 30.0 + 0.5)
    assert SR.search_range(d, s, 0, -32, 31) == (-1, 1)
    assert SR.search_range(d, s, 2, -32, 31) == (-3, 3)


def test_clipping_and_empty():
    d = np.array([[100.0, -100.0]])
    assert SR.search_range(d, [0], 1, -32, 31) == (-32, 31)
    assert SR.search_range(np.full((3, 3), np.nan), [0, 0, 0], 2, -16, 15) == (-16, 15)
    # a range entirely above the limits collapses onto the upper limit
    assert SR.search_range(np.array([[90.0]]), [0], 0, -8, 7) == (7, 7)
