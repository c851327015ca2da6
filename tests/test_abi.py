"""The C-ABI library loads and exports every symbol include/rsr.h declares; the
validation paths (no GPU needed) return the documented status codes."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rsr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rsr_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_1807_07433_b200 import build
    build.build()
    from paper_1807_07433_b200._lib import lib
    return lib()


def test_header_declares_the_five_calls():
    syms = declared_symbols()
    for s in ("rsr_warp", "rsr_cost_volume", "rsr_aggregate", "rsr_disparity", "rsr_reconstruct"):
        assert s in syms


def test_every_declared_symbol_is_exported(L):
    for s in declared_symbols():
        assert hasattr(L, s), s


def test_validation_without_gpu(L):
    from paper_1807_07433_b200._lib import (RsrAggParams, RsrCostParams, RsrDispParams, RsrRig,
                                            RsrShape)
    s = RsrShape(1, 8, 8)
    fake = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    assert L.rsr_warp(RsrShape(0, 8, 8), fake, fake, fake, fake, fake, None) == 2
    assert L.rsr_warp(s, None, fake, fake, fake, fake, None) == 2
    ws = L.rsr_cost_workspace_size(s)
    assert ws >= 4 * 4 * 64
    assert L.rsr_cost_volume(s, RsrCostParams(0, 0, 3), fake, fake, fake, fake, None, None, None,
                             fake, ws, None) == 2
    assert L.rsr_cost_volume(s, RsrCostParams(1, 3, 0), fake, fake, fake, fake, None, None, None,
                             fake, ws, None) == 2
    assert L.rsr_cost_volume(s, RsrCostParams(1, 0, 3), fake, fake, fake, fake, None, None, None,
                             fake, ws - 1, None) == 2
    assert L.rsr_cost_volume(s, RsrCostParams(5, 0, 3), fake, fake, fake, fake, None, None, None,
                             fake, ws, None) == 3   # 8 < 2*5+1
    assert L.rsr_aggregate(s, 0, RsrAggParams(1, 1.0, 1.0), fake, fake, None, ctypes.c_void_p(32),
                           None) == 2
    assert L.rsr_aggregate(s, 4, RsrAggParams(11, 1.0, 1.0), fake, fake, None, ctypes.c_void_p(32),
                           None) == 2
    assert L.rsr_aggregate(s, 4, RsrAggParams(1, 1.0, float("nan")), fake, fake, None,
                           ctypes.c_void_p(32), None) == 2
    assert L.rsr_disparity(s, RsrDispParams(0, 3, -1, 1), fake, fake, fake, fake, None, None, None) == 2
    assert L.rsr_reconstruct(s, RsrRig(0.0, 0.12, 0, 0, 1.0), fake, fake, None) == 2
    assert L.rsr_reconstruct(s, RsrRig(700.0, 0.12, 0, 0, 0.0), fake, fake, None) == 2
    from paper_1807_07433_b200._lib import RsrRoadParams
    rp = RsrRoadParams(4, 4, 64, 0.5, 0)
    wsr = L.rsr_road_workspace_size(s, rp)
    assert wsr > 0
    assert L.rsr_road_model(s, RsrRoadParams(0, 4, 64, 0.5, 0), fake, fake, fake, wsr, None) == 2
    assert L.rsr_road_model(s, RsrRoadParams(4, 4, 64, 0.0, 0), fake, fake, fake, wsr, None) == 2
    assert L.rsr_road_model(s, rp, fake, fake, fake, wsr - 1, None) == 2
    assert L.rsr_road_model(s, rp, None, fake, fake, wsr, None) == 2
    assert L.rsr_strerror(2) == b"invalid argument"
    assert L.rsr_version() >= 10000


def test_validation_of_round2_calls_without_gpu(L):
    """rsr_match (f1) and the interpolating-warp calls (f2) validate before any launch."""
    from paper_1807_07433_b200._lib import RsrAggParams, RsrCostParams, RsrDispParams, RsrShape
    s = RsrShape(1, 32, 64)
    fake = ctypes.c_void_p(16)
    ws = L.rsr_cost_workspace_size(s)
    cp, ap, dp = RsrCostParams(2, -4, 3), RsrAggParams(3, 2.0, 10.0, 1), RsrDispParams(-4, 3, 1, 1)
    # D = 17 > 8: the fused kernel serves the small search ranges only
    assert L.rsr_match(s, RsrCostParams(2, -8, 8), ap, RsrDispParams(-8, 8, 1, 1), fake, fake, fake, fake, fake,
                       None, None, fake, ws, None) == 2
    # the disparity range must be the cost range
    assert L.rsr_match(s, cp, ap, RsrDispParams(-4, 4, 1, 1), fake, fake, fake, fake, fake, None, None, fake, ws,
                       None) == 2
    assert L.rsr_match(s, cp, RsrAggParams(8, 2.0, 10.0, 1), dp, fake, fake, fake, fake, fake, None, None, fake, ws,
                       None) == 2
    assert L.rsr_match(s, cp, ap, dp, fake, fake, fake, fake, fake, None, None, fake, ws - 1, None) == 2
    assert L.rsr_match(s, RsrCostParams(20, -4, 3), ap, dp, fake, fake, fake, fake, fake, None, None, fake, ws,
                       None) == 2
    assert L.rsr_match(RsrShape(1, 4, 64), cp, ap, dp, fake, fake, fake, fake, fake, None, None, fake, ws,
                       None) == 3
    # interpolating warp family
    assert L.rsr_warp_linear(RsrShape(0, 8, 8), fake, fake, fake, fake, fake, None) == 2
    assert L.rsr_cost_volume_linear(s, RsrCostParams(0, 0, 3), fake, fake, fake, fake, None, None, None, fake, ws,
                                    None) == 2
    assert L.rsr_aggregate_linear(s, 8, RsrAggParams(8, 1.0, 1.0, 1), fake, fake, None, ctypes.c_void_p(32),
                                  None) == 2   # rho > 7
    assert L.rsr_disparity_linear(s, RsrDispParams(0, 3, -1, 1), fake, fake, fake, fake, None, None, None) == 2
    # introspection: row chunk of K3's launch plan
    assert L.rsr_aggregate_rows(RsrShape(8, 720, 1280), 64, RsrAggParams(6, 4.0, 12.0, 2)) == 240
    assert L.rsr_aggregate_rows(RsrShape(1, 40, 90), 16, RsrAggParams(8, 4.0, 12.0, 1)) == 0
    assert L.rsr_aggregate_rows(RsrShape(0, 40, 90), 16, RsrAggParams(2, 4.0, 12.0, 1)) == -1
