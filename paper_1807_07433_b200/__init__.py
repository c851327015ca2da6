"""B200-native (sm_100a) road-surface stereo hot path of arXiv 1807.07433.

The computation lives in librsr.so (CUDA kernels behind the C ABI of
include/rsr.h); this package is the thin Python binding (ops.py) plus buffer
plumbing (pipeline.py).  PyTorch supplies device memory, streams and
torch.distributed only.
"""
from ._lib import RsrError, lib  # noqa: F401
from .ops import (rsr_aggregate, rsr_cost_volume, rsr_disparity, rsr_reconstruct,  # noqa: F401
                  rsr_warp, rsr_road_model, rsr_road_roll, rsr_plane_fit, rsr_plane_distance,
                  rsr_search_range, rsr_aggregate_rows,
                  rsr_warp_linear, rsr_cost_volume_linear, rsr_aggregate_linear, rsr_disparity_linear,
                  rsr_match,
                  cost_workspace_bytes)
from .pipeline import StereoParams, StereoPipeline  # noqa: F401
