"""CPU fp64 oracle of the road-surface stereo hot path (arXiv 1807.07433).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  It shares no code
with paper_1807_07433_b200/ and imports nothing from it.
"""
from .rsr_oracle import *  # noqa: F401,F403
from . import brute  # noqa: F401
from . import interp_warp  # noqa: F401
