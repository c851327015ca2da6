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
