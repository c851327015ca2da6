"""Buffer plumbing for the whole hot path: allocate every device buffer once
(torch), then enqueue the five C-ABI calls in the paper's order on the current
stream.  No arithmetic of the method happens here."""
from __future__ import annotations

import dataclasses

import torch

from . import ops


@dataclasses.dataclass(frozen=True)
class StereoParams:
    d_lo: int
    d_hi: int
    rho_block: int
    rho_agg: int
    gamma_d: float
    gamma_r: float
    lrc_tol: int = 1
    subpixel: bool = True
    focal: float = 700.0
    baseline: float = 0.12
    d_min: float = 1.0
    warp: str = "integer"    # "integer" (reading 1, rsr_warp) or "linear" (NEXT f2, rsr_warp_linear)

    @property
    def D(self):
        return self.d_hi - self.d_lo + 1

    @staticmethod
    def from_config(cfg, warp="integer"):
        return StereoParams(cfg.d_lo, cfg.d_hi, cfg.rho_block, cfg.rho_agg, cfg.gamma_d, cfg.gamma_r,
                            cfg.lrc_tol, True, cfg.focal, cfg.baseline, warp=warp)


class StereoPipeline:
    """Pre-allocated buffers for a [B,H,W] batch; run() enqueues the whole path.

    Kernel launches per run(): warp 1; cost volume 1 block-stats (both images) + ceil(D/64)
    NCC slabs (both volumes per grid) + 1 NaN-summary; aggregation 2 (rho <= 7); disparity 1;
    reconstruction 1 (see launches()).
    """

    @staticmethod
    def launches(D: int) -> int:
        return 1 + (1 + (D + 63) // 64 + 1) + 2 + 1 + 1   # both images / volumes in one grid each

    def __init__(self, B, H, W, params: StereoParams, device="cuda"):
        self.B, self.H, self.W, self.p = B, H, W, params
        D = params.D
        dev = torch.device(device)
        e = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)  # noqa: E731
        if params.warp not in ("integer", "linear"):
            raise ValueError(f"unknown warp {params.warp!r}")
        self.linear = params.warp == "linear"
        self.warped = e((B, H, W), torch.uint16 if self.linear else torch.uint8)
        self.valid = e((B, H, W), torch.uint8)
        self.shift = e((B, H), torch.float64 if self.linear else torch.int32)
        self.vol_ref = e((B, H, W, D), torch.float32)
        self.vol_tar = e((B, H, W, D), torch.float32)
        self.nan_ref = e((B, H, W), torch.uint8)
        self.nan_tar = e((B, H, W), torch.uint8)
        self.agg_ref = e((B, H, W, D), torch.float32)
        self.agg_tar = e((B, H, W, D), torch.float32)
        self.disparity = e((B, H, W), torch.float32)
        self.wta_ref = e((B, H, W), torch.int16)
        self.wta_tar = e((B, H, W), torch.int16)
        self.xyz = e((B, H, W, 3), torch.float32)
        self.workspace = e((ops.cost_workspace_bytes(B, H, W),), torch.uint8)
        self._side = None

    def run(self, left, right, alpha_beta, with_wta=True):
        p = self.p
        lin = self.linear
        (ops.rsr_warp_linear if lin else ops.rsr_warp)(right, alpha_beta, self.warped, self.valid, self.shift)
        (ops.rsr_cost_volume_linear if lin else ops.rsr_cost_volume)(
            left, self.warped, self.valid, p.rho_block, p.d_lo, p.d_hi, vol_ref=self.vol_ref,
            vol_tar=self.vol_tar, nan_ref=self.nan_ref, nan_tar=self.nan_tar, workspace=self.workspace)
        # the two aggregations are independent: the target volume's on a side stream, so
        # each launch back-fills the other's last wave
        main = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream(device=main.device)
        fork = torch.cuda.Event()
        fork.record(main)
        self._side.wait_event(fork)
        aggregate_tar = ops.rsr_aggregate_linear if lin else ops.rsr_aggregate
        with torch.cuda.stream(self._side):
            aggregate_tar(self.vol_tar, self.warped, p.rho_agg, p.gamma_d, p.gamma_r, self.nan_tar,
                          self.agg_tar, concurrency=2)
        ops.rsr_aggregate(self.vol_ref, left, p.rho_agg, p.gamma_d, p.gamma_r, self.nan_ref, self.agg_ref,
                          concurrency=2)
        join = torch.cuda.Event()
        join.record(self._side)
        main.wait_event(join)
        disparity = ops.rsr_disparity_linear if lin else ops.rsr_disparity
        disparity(self.agg_ref, self.agg_tar, self.shift, p.d_lo, p.d_hi, p.lrc_tol, p.subpixel,
                  self.disparity, self.wta_ref if with_wta else None, self.wta_tar if with_wta else None)
        ops.rsr_reconstruct(self.disparity, p.focal, p.baseline, d_min=p.d_min, xyz=self.xyz)
        return self.disparity
