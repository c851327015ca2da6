// C ABI of librsr (include/rsr.h): argument validation, workspace carving and
// kernel launches.  Validation happens before any launch, so a failing call
// enqueues nothing (SPEC S:530 convention).
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/rsr.h"
#include "kernels.h"

namespace {

inline bool shape_ok(const rsr_shape& s) { return s.batch >= 1 && s.height >= 1 && s.width >= 1; }
inline cudaStream_t as_stream(void* p) { return reinterpret_cast<cudaStream_t>(p); }
inline int launched(cudaError_t e) { return e == cudaSuccess ? RSR_OK : RSR_E_INTERNAL; }
inline size_t npix(const rsr_shape& s) { return (size_t)s.batch * s.height * s.width; }
inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

}  // namespace

extern "C" {

int rsr_version(void) { return 10000; }

const char* rsr_strerror(int status) {
  switch (status) {
    case RSR_OK: return "ok";
    case RSR_E_ARG: return "invalid argument";
    case RSR_E_DATA: return "data too small for the requested window";
    case RSR_E_INTERNAL: return "CUDA launch error";
    default: return "unknown status";
  }
}

int rsr_warp(rsr_shape s, const double* alpha_beta, const uint8_t* target, uint8_t* warped,
             uint8_t* valid, int32_t* shift, void* stream) {
  if (!shape_ok(s) || !alpha_beta || !target || !warped || !valid || !shift) return RSR_E_ARG;
  if (s.height > 65535 || s.batch > 65535) return RSR_E_ARG;
  return launched(rsr::launch_warp(s.batch, s.height, s.width, alpha_beta, target, warped, valid,
                                   shift, as_stream(stream)));
}

size_t rsr_cost_workspace_size(rsr_shape s) {
  if (!shape_ok(s)) return 0;
  // S_L, inv_L, S_W, inv_W, each [B][H][W] (S int32, or fp32 for rsr_cost_volume), and
  // for rsr_cost_volume the fp32 copies of both images the NCC kernel streams
  return 6 * align16(sizeof(int32_t) * npix(s));
}

int rsr_cost_volume(rsr_shape s, rsr_cost_params p, const uint8_t* ref, const uint8_t* warped,
                    const uint8_t* valid, float* vol_ref, float* vol_tar, uint8_t* nan_ref,
                    uint8_t* nan_tar, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape_ok(s) || !ref || !warped || !valid || !vol_ref || !workspace) return RSR_E_ARG;
  if (p.rho_block < 1 || p.rho_block > 7 || p.d_hi < p.d_lo) return RSR_E_ARG;
  const long long D = (long long)p.d_hi - p.d_lo + 1;
  if (D > 32767) return RSR_E_ARG;
  if (workspace_bytes < rsr_cost_workspace_size(s)) return RSR_E_ARG;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return RSR_E_ARG;
  if (s.height < 2 * p.rho_block + 1 || s.width < 2 * p.rho_block + 1) return RSR_E_DATA;
  if ((size_t)(s.height + 15) / 16 > 65535 || s.batch > 65535) return RSR_E_ARG;
  const size_t chunk = align16(sizeof(int32_t) * npix(s));
  char* ws = static_cast<char*>(workspace);
  float* SL = reinterpret_cast<float*>(ws);
  float* iL = reinterpret_cast<float*>(ws + chunk);
  float* SW = reinterpret_cast<float*>(ws + 2 * chunk);
  float* iW = reinterpret_cast<float*>(ws + 3 * chunk);
  float* Lf = reinterpret_cast<float*>(ws + 4 * chunk);
  float* Wf = reinterpret_cast<float*>(ws + 5 * chunk);
  cudaStream_t st = as_stream(stream);
  // both images' block statistics in one grid (two grids past 65535 / 2 frames)
  cudaError_t e;
  if (2LL * s.batch <= 65535) {
    e = rsr::launch_block_stats_f(s.batch, s.height, s.width, p.rho_block, ref, nullptr, SL, iL, Lf, warped,
                                  valid, SW, iW, Wf, st);
  } else {
    e = rsr::launch_block_stats_f(s.batch, s.height, s.width, p.rho_block, ref, nullptr, SL, iL, Lf, nullptr,
                                  nullptr, nullptr, nullptr, nullptr, st);
    if (e == cudaSuccess)
      e = rsr::launch_block_stats_f(s.batch, s.height, s.width, p.rho_block, warped, valid, SW, iW, Wf,
                                    nullptr, nullptr, nullptr, nullptr, nullptr, st);
  }
  if (e == cudaSuccess && vol_tar && 2LL * s.batch <= 65535)   // both volumes, one grid
    e = rsr::launch_zncc_pair(s.batch, s.height, s.width, p.rho_block, p.d_lo, (int)D, Lf, Wf, SL, iL,
                              SW, iW, vol_ref, vol_tar, st);
  else {
    if (e == cudaSuccess)
      e = rsr::launch_zncc(false, s.batch, s.height, s.width, p.rho_block, p.d_lo, (int)D, Lf,
                           Wf, SL, iL, SW, iW, vol_ref, st);
    if (e == cudaSuccess && vol_tar)
      e = rsr::launch_zncc(true, s.batch, s.height, s.width, p.rho_block, p.d_lo, (int)D, Lf,
                           Wf, SL, iL, SW, iW, vol_tar, st);
  }
  if (e == cudaSuccess)
    e = rsr::launch_nan_maps(s.batch, s.height, s.width, p.d_lo, (int)D, iL, iW, nan_ref,
                             vol_tar ? nan_tar : nullptr, st);
  return launched(e);
}

int rsr_aggregate(rsr_shape s, int32_t D, rsr_agg_params p, const float* vol, const uint8_t* guide,
                  const uint8_t* nan_map, float* out, void* stream) {
  if (!shape_ok(s) || !vol || !guide || !out) return RSR_E_ARG;
  if (D < 1 || D > 32767 || p.rho < 0 || p.rho > 10) return RSR_E_ARG;
  if (!(p.gamma_d > 0.f) || std::isinf(p.gamma_d) || !(p.gamma_r > 0.f)) return RSR_E_ARG;
  if (p.concurrency < 0 || p.concurrency > 64) return RSR_E_ARG;
  if (vol == out) return RSR_E_ARG;
  if ((s.height + 7) / 8 > 65535) return RSR_E_ARG;
  const long long nslab = (D + 63) / 64;
  if ((long long)s.batch * nslab > 65535) return RSR_E_ARG;
  return launched(rsr::launch_aggregate(s.batch, s.height, s.width, D, p.rho, p.gamma_d, p.gamma_r, p.concurrency,
                                        vol, guide, nan_map, out, as_stream(stream)));
}

int32_t rsr_aggregate_rows(rsr_shape s, int32_t D, rsr_agg_params p) {
  if (!shape_ok(s) || D < 1 || D > 32767 || p.rho < 0 || p.rho > 10) return -1;
  return rsr::aggregate_plan_rows(s.batch, s.height, s.width, D, p.rho, p.concurrency);
}

int rsr_disparity(rsr_shape s, rsr_disp_params p, const float* agg_ref, const float* agg_tar,
                  const int32_t* shift, float* disparity, int16_t* wta_ref, int16_t* wta_tar,
                  void* stream) {
  if (!shape_ok(s) || !agg_ref || !agg_tar || !shift || !disparity) return RSR_E_ARG;
  if (p.d_hi < p.d_lo || (long long)p.d_hi - p.d_lo + 1 > 32767 || p.lrc_tol < 0) return RSR_E_ARG;
  if (s.width > 32768 || s.height > 65535 || s.batch > 65535) return RSR_E_ARG;
  const int D = p.d_hi - p.d_lo + 1;
  return launched(rsr::launch_disparity(s.batch, s.height, s.width, p.d_lo, D, p.lrc_tol,
                                        p.subpixel != 0, agg_ref, agg_tar, shift, disparity,
                                        wta_ref, wta_tar, as_stream(stream)));
}

// ---- interpolating-warp variant (NEXT row f2, reading 21) ----
int rsr_warp_linear(rsr_shape s, const double* alpha_beta, const uint8_t* target, uint16_t* warped,
                    uint8_t* valid, double* shift, void* stream) {
  if (!shape_ok(s) || !alpha_beta || !target || !warped || !valid || !shift) return RSR_E_ARG;
  if (s.height > 65535 || s.batch > 65535) return RSR_E_ARG;
  return launched(rsr::launch_warp_linear(s.batch, s.height, s.width, alpha_beta, target, warped, valid,
                                          shift, as_stream(stream)));
}

int rsr_cost_volume_linear(rsr_shape s, rsr_cost_params p, const uint8_t* ref, const uint16_t* warped,
                           const uint8_t* valid, float* vol_ref, float* vol_tar, uint8_t* nan_ref,
                           uint8_t* nan_tar, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape_ok(s) || !ref || !warped || !valid || !vol_ref || !workspace) return RSR_E_ARG;
  if (p.rho_block < 1 || p.rho_block > 7 || p.d_hi < p.d_lo) return RSR_E_ARG;
  const long long D = (long long)p.d_hi - p.d_lo + 1;
  if (D > 32767) return RSR_E_ARG;
  if (workspace_bytes < rsr_cost_workspace_size(s)) return RSR_E_ARG;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return RSR_E_ARG;
  if (s.height < 2 * p.rho_block + 1 || s.width < 2 * p.rho_block + 1) return RSR_E_DATA;
  if ((size_t)(s.height + 15) / 16 > 65535 || 2LL * s.batch > 65535) return RSR_E_ARG;
  const size_t chunk = align16(sizeof(int32_t) * npix(s));
  char* ws = static_cast<char*>(workspace);
  int32_t* SL = reinterpret_cast<int32_t*>(ws);
  float* iL = reinterpret_cast<float*>(ws + chunk);
  int32_t* SW = reinterpret_cast<int32_t*>(ws + 2 * chunk);
  float* iW = reinterpret_cast<float*>(ws + 3 * chunk);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = rsr::launch_block_stats16(s.batch, s.height, s.width, p.rho_block, ref, SL, iL, warped, valid,
                                            SW, iW, st);
  if (e == cudaSuccess)
    e = rsr::launch_zncc_fx(s.batch, s.height, s.width, p.rho_block, p.d_lo, (int)D, ref, warped, SL, iL, SW,
                            iW, vol_ref, vol_tar, st);
  if (e == cudaSuccess)
    e = rsr::launch_nan_maps(s.batch, s.height, s.width, p.d_lo, (int)D, iL, iW, nan_ref,
                             vol_tar ? nan_tar : nullptr, st);
  return launched(e);
}

int rsr_aggregate_linear(rsr_shape s, int32_t D, rsr_agg_params p, const float* vol, const uint16_t* guide,
                         const uint8_t* nan_map, float* out, void* stream) {
  if (!shape_ok(s) || !vol || !guide || !out) return RSR_E_ARG;
  if (D < 1 || D > 32767 || p.rho < 0 || p.rho > 7) return RSR_E_ARG;
  if (!(p.gamma_d > 0.f) || std::isinf(p.gamma_d) || !(p.gamma_r > 0.f)) return RSR_E_ARG;
  if (p.concurrency < 0 || p.concurrency > 64) return RSR_E_ARG;
  if (vol == out) return RSR_E_ARG;
  const long long nslab = (D + 63) / 64;
  if ((long long)s.batch * nslab > 65535) return RSR_E_ARG;
  return launched(rsr::launch_aggregate_slide16(s.batch, s.height, s.width, D, p.rho, p.gamma_d, p.gamma_r,
                                                p.concurrency, vol, guide, nan_map, out, as_stream(stream)));
}

int rsr_disparity_linear(rsr_shape s, rsr_disp_params p, const float* agg_ref, const float* agg_tar,
                         const double* shift, float* disparity, int16_t* wta_ref, int16_t* wta_tar,
                         void* stream) {
  if (!shape_ok(s) || !agg_ref || !agg_tar || !shift || !disparity) return RSR_E_ARG;
  if (p.d_hi < p.d_lo || (long long)p.d_hi - p.d_lo + 1 > 32767 || p.lrc_tol < 0) return RSR_E_ARG;
  if (s.width > 32768 || s.height > 65535 || s.batch > 65535) return RSR_E_ARG;
  const int D = p.d_hi - p.d_lo + 1;
  return launched(rsr::launch_disparity_frac(s.batch, s.height, s.width, p.d_lo, D, p.lrc_tol,
                                             p.subpixel != 0, agg_ref, agg_tar, shift, disparity,
                                             wta_ref, wta_tar, as_stream(stream)));
}

// ---- fused, volume-free matching (NEXT row f1) ----
int rsr_match(rsr_shape s, rsr_cost_params cp, rsr_agg_params ap, rsr_disp_params dp, const uint8_t* ref,
              const uint8_t* warped, const uint8_t* valid, const int32_t* shift, float* disparity,
              int16_t* wta_ref, int16_t* wta_tar, void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape_ok(s) || !ref || !warped || !valid || !shift || !disparity || !workspace) return RSR_E_ARG;
  if (cp.rho_block < 1 || cp.rho_block > 7 || cp.d_hi < cp.d_lo) return RSR_E_ARG;
  if (dp.d_lo != cp.d_lo || dp.d_hi != cp.d_hi || dp.lrc_tol < 0) return RSR_E_ARG;
  const long long D = (long long)cp.d_hi - cp.d_lo + 1;
  if (D > 8) return RSR_E_ARG;
  if (ap.rho < 0 || ap.rho > 7) return RSR_E_ARG;
  if (!(ap.gamma_d > 0.f) || std::isinf(ap.gamma_d) || !(ap.gamma_r > 0.f)) return RSR_E_ARG;
  if (workspace_bytes < rsr_cost_workspace_size(s)) return RSR_E_ARG;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return RSR_E_ARG;
  if (s.height < 2 * cp.rho_block + 1 || s.width < 2 * cp.rho_block + 1) return RSR_E_DATA;
  if ((size_t)(s.height + 15) / 16 > 65535 || 2LL * s.batch > 65535) return RSR_E_ARG;
  const size_t chunk = align16(sizeof(int32_t) * npix(s));
  char* ws = static_cast<char*>(workspace);
  int32_t* SL = reinterpret_cast<int32_t*>(ws);
  float* iL = reinterpret_cast<float*>(ws + chunk);
  int32_t* SW = reinterpret_cast<int32_t*>(ws + 2 * chunk);
  float* iW = reinterpret_cast<float*>(ws + 3 * chunk);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = rsr::launch_block_stats(s.batch, s.height, s.width, cp.rho_block, ref, nullptr, SL, iL, warped,
                                          valid, SW, iW, st);
  if (e == cudaSuccess)
    e = rsr::launch_match_fused(s.batch, s.height, s.width, cp.rho_block, cp.d_lo, (int)D, ap.rho, ap.gamma_d,
                                ap.gamma_r, dp.lrc_tol, dp.subpixel != 0, ref, warped, shift, SL, iL, SW, iW,
                                disparity, wta_ref, wta_tar, st);
  return launched(e);
}

size_t rsr_road_workspace_size(rsr_shape s, rsr_road_params p) {
  if (!shape_ok(s) || p.step_u < 1 || p.step_v < 1 || p.n_hyp < 1) return 0;
  return rsr::road_workspace_size(s.batch, s.height, s.width, p.step_u, p.step_v, p.n_hyp);
}

int rsr_road_model(rsr_shape s, rsr_road_params p, const float* disparity, double* model,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (!shape_ok(s) || !disparity || !model || !workspace) return RSR_E_ARG;
  if (p.step_u < 1 || p.step_v < 1 || p.n_hyp < 1 || p.n_hyp > (1 << 24)) return RSR_E_ARG;
  if (!(p.inlier_tol > 0.f) || std::isinf(p.inlier_tol)) return RSR_E_ARG;
  if (s.batch > 65535 || (p.n_hyp + 7) / 8 > 65535) return RSR_E_ARG;
  if (workspace_bytes < rsr_road_workspace_size(s, p)) return RSR_E_ARG;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return RSR_E_ARG;
  return launched(rsr::launch_road_model(s.batch, s.height, s.width, p.step_u, p.step_v, p.n_hyp,
                                         p.inlier_tol, p.seed, disparity, model, workspace,
                                         as_stream(stream)));
}

int rsr_road_roll(rsr_shape s, int32_t u0, int32_t u1, int32_t v0, int32_t v1, const float* disparity,
                  double* out, void* stream) {
  if (!shape_ok(s) || !disparity || !out) return RSR_E_ARG;
  if (u0 < 0 || v0 < 0 || u1 > s.width || v1 > s.height || u0 >= u1 || v0 >= v1) return RSR_E_ARG;
  if (s.batch > 65535) return RSR_E_ARG;
  return launched(rsr::launch_road_roll(s.batch, s.height, s.width, u0, u1, v0, v1, disparity, out,
                                        as_stream(stream)));
}

int rsr_search_range(rsr_shape s, const float* disparity, const int32_t* shift, int32_t delta,
                     int32_t d_lo_limit, int32_t d_hi_limit, int32_t* range, void* stream) {
  if (!shape_ok(s) || !disparity || !shift || !range) return RSR_E_ARG;
  if (delta < 0 || d_hi_limit < d_lo_limit || (long long)d_hi_limit - d_lo_limit + 1 > 32767) return RSR_E_ARG;
  if (s.batch > 0x7fffffff / 2) return RSR_E_ARG;
  return launched(rsr::launch_search_range(s.batch, s.height, s.width, delta, d_lo_limit, d_hi_limit, disparity,
                                           shift, range, as_stream(stream)));
}

int rsr_plane_fit(int32_t batch, int32_t n_corners, const double* corners, double* plane, void* stream) {
  if (!corners || !plane || batch < 1 || n_corners < 3) return RSR_E_ARG;
  return launched(rsr::launch_plane_fit(batch, n_corners, corners, plane, as_stream(stream)));
}

int rsr_plane_distance(rsr_shape s, const double* plane, const float* xyz, float* dist, void* stream) {
  if (!shape_ok(s) || !plane || !xyz || !dist) return RSR_E_ARG;
  return launched(rsr::launch_plane_distance(s.batch, s.height, s.width, plane, xyz, dist, as_stream(stream)));
}

int rsr_reconstruct(rsr_shape s, rsr_rig rig, const float* disparity, float* xyz, void* stream) {
  if (!shape_ok(s) || !disparity || !xyz) return RSR_E_ARG;
  if (!(rig.f > 0) || !(rig.baseline > 0) || !(rig.d_min > 0)) return RSR_E_ARG;
  if (!std::isfinite(rig.u0) || !std::isfinite(rig.v0) || !std::isfinite(rig.f)) return RSR_E_ARG;
  return launched(rsr::launch_reconstruct(s.batch, s.height, s.width, rig.f, rig.baseline, rig.u0,
                                          rig.v0, rig.d_min, disparity, xyz, as_stream(stream)));
}

}  // extern "C"
