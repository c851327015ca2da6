"""CPU oracle of the restricted search range.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/ and
bench-side tools, never by the product path.

P:251 (future work): "performing the bilateral filtering on the whole cost volume
is a very time-consuming process.  Therefore, we plan to reduce the search range
and only perform the bilateral filtering on the space around the calculated
disparities."  Reading (reading 20): the calculated disparities
are the previous frame's map d (total disparity, px); with the next frame's row
shifts s(v) (rsr_warp), the residual search range of the next frame is

    d_lo = floor(min r) - delta,  d_hi = ceil(max r) + delta,  r = d(u, v) - s(v)

over the finite entries of d (fp64, exact for these magnitudes), clipped to the
limits [lo_lim, hi_lim]; the full limits when d has no finite entry.  The
aggregation then covers only that band (a smaller D for the whole path).
"""
from __future__ import annotations

import math

import numpy as np


def search_range(disparity, shift, delta: int, lo_lim: int, hi_lim: int) -> tuple[int, int]:
    d = np.asarray(disparity, dtype=np.float64)
    s = np.asarray(shift, dtype=np.float64).reshape(-1, 1)
    r = d - s
    fin = np.isfinite(r)
    if not fin.any():
        return int(lo_lim), int(hi_lim)
    lo = math.floor(float(r[fin].min())) - delta
    hi = math.ceil(float(r[fin].max())) + delta
    lo = min(max(lo, lo_lim), hi_lim)
    hi = min(max(hi, lo_lim), hi_lim)
    return int(lo), int(hi)
