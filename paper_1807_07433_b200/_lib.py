"""ctypes binding of librsr.so (include/rsr.h).  Argument marshalling only:
every step of the path runs in the library's CUDA kernels.  There is no CPU
fallback: if the shared library is missing or a tensor is not on a CUDA device,
calls raise."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RSR_LIB selects an alternative in-tree build (A/B experiments under tools/)
LIB_PATH = os.environ.get("RSR_LIB") or os.path.join(HERE, "librsr.so")

RSR_OK, RSR_E_ARG, RSR_E_DATA, RSR_E_INTERNAL = 0, 2, 3, 4


class RsrShape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("height", ctypes.c_int32), ("width", ctypes.c_int32)]


class RsrCostParams(ctypes.Structure):
    _fields_ = [("rho_block", ctypes.c_int32), ("d_lo", ctypes.c_int32), ("d_hi", ctypes.c_int32)]


class RsrAggParams(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_int32), ("gamma_d", ctypes.c_float), ("gamma_r", ctypes.c_float),
                ("concurrency", ctypes.c_int32)]


class RsrDispParams(ctypes.Structure):
    _fields_ = [("d_lo", ctypes.c_int32), ("d_hi", ctypes.c_int32), ("lrc_tol", ctypes.c_int32),
                ("subpixel", ctypes.c_int32)]


class RsrRig(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double), ("baseline", ctypes.c_double), ("u0", ctypes.c_double),
                ("v0", ctypes.c_double), ("d_min", ctypes.c_double)]


class RsrRoadParams(ctypes.Structure):
    _fields_ = [("step_u", ctypes.c_int32), ("step_v", ctypes.c_int32), ("n_hyp", ctypes.c_int32),
                ("inlier_tol", ctypes.c_float), ("seed", ctypes.c_uint32)]


class RsrError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn} failed: status {status} ({strerror(status)})")


_lib = None
P = ctypes.c_void_p


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1807_07433_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.rsr_warp.argtypes = [RsrShape, P, P, P, P, P, P]
        L.rsr_cost_workspace_size.argtypes = [RsrShape]
        L.rsr_cost_workspace_size.restype = ctypes.c_size_t
        L.rsr_cost_volume.argtypes = [RsrShape, RsrCostParams, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.rsr_aggregate.argtypes = [RsrShape, ctypes.c_int32, RsrAggParams, P, P, P, P, P]
        L.rsr_aggregate_rows.argtypes = [RsrShape, ctypes.c_int32, RsrAggParams]
        L.rsr_aggregate_rows.restype = ctypes.c_int32
        L.rsr_disparity.argtypes = [RsrShape, RsrDispParams, P, P, P, P, P, P, P]
        L.rsr_reconstruct.argtypes = [RsrShape, RsrRig, P, P, P]
        L.rsr_warp_linear.argtypes = [RsrShape, P, P, P, P, P, P]
        L.rsr_cost_volume_linear.argtypes = [RsrShape, RsrCostParams, P, P, P, P, P, P, P, P, ctypes.c_size_t, P]
        L.rsr_aggregate_linear.argtypes = [RsrShape, ctypes.c_int32, RsrAggParams, P, P, P, P, P]
        L.rsr_disparity_linear.argtypes = [RsrShape, RsrDispParams, P, P, P, P, P, P, P]
        for f in ("rsr_warp_linear", "rsr_cost_volume_linear", "rsr_aggregate_linear", "rsr_disparity_linear"):
            getattr(L, f).restype = ctypes.c_int
        L.rsr_match.argtypes = [RsrShape, RsrCostParams, RsrAggParams, RsrDispParams, P, P, P, P, P, P, P, P,
                                ctypes.c_size_t, P]
        L.rsr_match.restype = ctypes.c_int
        L.rsr_road_workspace_size.argtypes = [RsrShape, RsrRoadParams]
        L.rsr_road_workspace_size.restype = ctypes.c_size_t
        L.rsr_road_model.argtypes = [RsrShape, RsrRoadParams, P, P, P, ctypes.c_size_t, P]
        L.rsr_road_model.restype = ctypes.c_int
        L.rsr_road_roll.argtypes = [RsrShape, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    P, P, P]
        L.rsr_road_roll.restype = ctypes.c_int
        L.rsr_search_range.argtypes = [RsrShape, P, P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
        L.rsr_search_range.restype = ctypes.c_int
        L.rsr_plane_fit.argtypes = [ctypes.c_int32, ctypes.c_int32, P, P, P]
        L.rsr_plane_fit.restype = ctypes.c_int
        L.rsr_plane_distance.argtypes = [RsrShape, P, P, P, P]
        L.rsr_plane_distance.restype = ctypes.c_int
        L.rsr_strerror.argtypes = [ctypes.c_int]
        L.rsr_strerror.restype = ctypes.c_char_p
        L.rsr_version.restype = ctypes.c_int
        for f in ("rsr_warp", "rsr_cost_volume", "rsr_aggregate", "rsr_disparity", "rsr_reconstruct"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def strerror(status: int) -> str:
    return lib().rsr_strerror(status).decode()


def check(fn: str, status: int) -> None:
    if status != RSR_OK:
        raise RsrError(fn, status)
