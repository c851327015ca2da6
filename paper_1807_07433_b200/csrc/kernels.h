// Internal launch wrappers (C++), one per kernel family.  The public C ABI
// (include/rsr.h, api.cu) validates arguments and calls these.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rsr {

cudaError_t launch_warp(int B, int H, int W, const double* ab, const uint8_t* target,
                        uint8_t* warped, uint8_t* valid, int32_t* shift, cudaStream_t st);
// interpolating warp (NEXT f2): 8.8 fixed-point warped image, fp64 applied shift t_q(v)
cudaError_t launch_warp_linear(int B, int H, int W, const double* ab, const uint8_t* target,
                               uint16_t* warped, uint8_t* valid, double* shift, cudaStream_t st);

// Per-pixel block statistics for the NCC normalisation: S = sum i (int32),
// inv = 1/sqrt(n*sum i^2 - S^2) (fp32, NaN if the block leaves the image, touches
// mask==0 or is constant).  mask may be null.
cudaError_t launch_block_stats(int B, int H, int W, int rho_b, const uint8_t* img0, const uint8_t* mask0,
                               int32_t* S0, float* inv0, const uint8_t* img1, const uint8_t* mask1, int32_t* S1,
                               float* inv1, cudaStream_t st);

// The same statistics for the streaming NCC kernel: S as fp32 (exact) and each image
// also as an fp32 plane (F0 = img0, F1 = img1); img1 may be null.
cudaError_t launch_block_stats_f(int B, int H, int W, int rho_b, const uint8_t* img0, const uint8_t* mask0,
                                 float* S0, float* inv0, float* F0, const uint8_t* img1, const uint8_t* mask1,
                                 float* S1, float* inv1, float* F1, cudaStream_t st);

// NCC volume in [B][H][W][D] layout. tar=false: vol[v][u][k] = c(u, v, r);
// tar=true: vol[v][u'][k] = c(u'+r, v, r).  Inputs: the fp32 planes of
// launch_block_stats_f (images Lf = ref, Wf = warped; sums; norms).
// both volumes in one launch (grid of 2B frames)
cudaError_t launch_zncc_pair(int B, int H, int W, int rho_b, int d_lo, int D, const float* ref,
                             const float* warped, const float* SL, const float* invL, const float* SW,
                             const float* invW, float* vol_ref, float* vol_tar, cudaStream_t st);
cudaError_t launch_zncc(bool tar, int B, int H, int W, int rho_b, int d_lo, int D,
                        const float* ref, const float* warped, const float* SL,
                        const float* invL, const float* SW, const float* invW, float* vol,
                        cudaStream_t st);

// block statistics with an 8.8 fixed-point second image (NEXT f2)
cudaError_t launch_block_stats16(int B, int H, int W, int rho_b, const uint8_t* img0, int32_t* S0, float* inv0,
                                 const uint16_t* img1, const uint8_t* mask1, int32_t* S1, float* inv1,
                                 cudaStream_t st);
// NCC volumes of (uint8 ref, 8.8 fixed-point warped), exact integer sums (zncc_fx.cu);
// vol_tar may be null
cudaError_t launch_zncc_fx(int B, int H, int W, int rho_b, int d_lo, int D, const uint8_t* ref,
                           const uint16_t* warped, const int32_t* SL, const float* iL, const int32_t* SW,
                           const float* iW, float* vol_ref, float* vol_tar, cudaStream_t st);

// Per-pixel NaN summaries of both volumes, from the block norms (either map optional).
cudaError_t launch_nan_maps(int B, int H, int W, int d_lo, int D, const float* invL,
                            const float* invW, uint8_t* nan_ref, uint8_t* nan_tar, cudaStream_t st);

cudaError_t launch_aggregate(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                             const float* vol, const uint8_t* guide, const uint8_t* nan_map,
                             float* out, cudaStream_t st);

// sliding-window warp-specialised variant (rho <= 7); launch_aggregate dispatches to it
cudaError_t launch_aggregate_slide(int B, int H, int W, int D, int rho, float gamma_d,
                                   float gamma_r, int conc, const float* vol, const uint8_t* guide,
                                   const uint8_t* nan_map, float* out, cudaStream_t st);
size_t aggregate_slide_smem(int D, int rho, int H);
// small disparity slabs (D <= 16, rho <= 7): per-thread weights (aggregate_small.cu),
// bitwise identical to the sliding kernel; RSR_K3_SMALL=0 disables (A/B, tests)
bool aggregate_small_applies(int D, int rho);
cudaError_t launch_aggregate_small(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                                   const float* vol, const uint8_t* guide, const uint8_t* nan_map, float* out,
                                   cudaStream_t st);
// the same with an 8.8 fixed-point (uint16) guide (interpolating warp, NEXT f2); rho <= 7
cudaError_t launch_aggregate_slide16(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                                     const float* vol, const uint16_t* guide, const uint8_t* nan_map,
                                     float* out, cudaStream_t st);
// output rows per CTA the sliding kernel uses for this call (0: tiled kernel, rho > 7)
int aggregate_plan_rows(int B, int H, int W, int D, int rho, int conc);
size_t aggregate_tiled_smem(int D, int rho);

cudaError_t launch_disparity(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                             const float* agg_ref, const float* agg_tar, const int32_t* shift,
                             float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st);

cudaError_t launch_disparity_frac(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                                  const float* agg_ref, const float* agg_tar, const double* shift,
                                  float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st);

// fused, volume-free matching for D <= 8 (NEXT f1, match_fused.cu): NCC -> both
// aggregations -> WTA / LRC / subpixel / shift in one kernel, from the block statistics
cudaError_t launch_match_fused(int B, int H, int W, int rho_b, int d_lo, int D, int rho, float gamma_d,
                               float gamma_r, int lrc_tol, int subpix, const uint8_t* ref, const uint8_t* warped,
                               const int32_t* shift, const int32_t* SL, const float* iL, const int32_t* SW,
                               const float* iW, float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st);

cudaError_t launch_reconstruct(int B, int H, int W, double f, double baseline, double u0,
                               double v0, double d_min, const float* disp, float* xyz,
                               cudaStream_t st);

// Road model (NEXT f3): RANSAC-LSF of d = alpha v + beta over grid samples of a
// disparity map; model [B][3] = {alpha, beta, inliers}.
size_t road_workspace_size(int B, int H, int W, int su, int sv, int n_hyp);
cudaError_t launch_road_model(int B, int H, int W, int su, int sv, int n_hyp, float tol, unsigned seed,
                              const float* disp, double* model, void* ws, cudaStream_t st);

cudaError_t launch_road_roll(int B, int H, int W, int u0, int u1, int v0, int v1, const float* disp,
                             double* out, cudaStream_t st);

// reconstruction accuracy (plane.cu)
cudaError_t launch_plane_fit(int B, int K, const double* corners, double* plane, cudaStream_t st);
cudaError_t launch_plane_distance(int B, int H, int W, const double* plane, const float* xyz, float* dist,
                                  cudaStream_t st);

// restricted search range (range.cu)
cudaError_t launch_search_range(int B, int H, int W, int delta, int lo_lim, int hi_lim, const float* disp,
                                const int32_t* shift, int32_t* range, cudaStream_t st);

}  // namespace rsr
