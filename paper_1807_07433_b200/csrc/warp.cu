// K1 — perspective transformation of the target image (Eq. (2)).
// One CTA per (row v, frame b).  s(v) = floor(alpha*v + beta + 1/2) in fp64 with
// explicit round-to-nearest multiply/add intrinsics (no FMA contraction), so the
// shift equals the oracle's bit for bit (reading 1).  16-byte vector
// stores when the row is 16-byte aligned; the gather from the target row is a
// byte-granular shifted copy served from L1.
#include "common.cuh"
#include "kernels.h"

namespace rsr {

__global__ void __launch_bounds__(256) k_warp(int H, int W, const double* __restrict__ ab,
                                              const uint8_t* __restrict__ target,
                                              uint8_t* __restrict__ warped,
                                              uint8_t* __restrict__ valid,
                                              int32_t* __restrict__ shift) {
  const int v = blockIdx.x, b = blockIdx.y;
  const double alpha = ab[2 * b], beta = ab[2 * b + 1];
  double t = __dmul_rn(alpha, (double)v);
  t = __dadd_rn(t, beta);
  t = __dadd_rn(t, 0.5);
  double fl = floor(t);
  // |s| >= W leaves the row empty; clamp keeps the int conversion defined.
  fl = fmin(fmax(fl, -1073741824.0), 1073741824.0);
  const int s = (int)fl;
  if (threadIdx.x == 0) shift[(size_t)b * H + v] = s;
  const size_t row = ((size_t)b * H + v) * W;
  const uint8_t* src = target + row;
  uint8_t* dw = warped + row;
  uint8_t* dm = valid + row;
  if ((W & 15) == 0) {
    for (int u0 = threadIdx.x * 16; u0 < W; u0 += blockDim.x * 16) {
      uint32_t wv[4], mv[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint32_t ww = 0, mm = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int u = u0 + 4 * q + i;
          const long long sc = (long long)u - s;
          const bool ok = sc >= 0 && sc < W;
          const uint32_t px = ok ? src[sc] : 0u;
          ww |= px << (8 * i);
          mm |= (ok ? 1u : 0u) << (8 * i);
        }
        wv[q] = ww;
        mv[q] = mm;
      }
      *reinterpret_cast<uint4*>(dw + u0) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      *reinterpret_cast<uint4*>(dm + u0) = make_uint4(mv[0], mv[1], mv[2], mv[3]);
    }
  } else {
    for (int u = threadIdx.x; u < W; u += blockDim.x) {
      const long long sc = (long long)u - s;
      const bool ok = sc >= 0 && sc < W;
      dw[u] = ok ? src[sc] : 0;
      dm[u] = ok ? 1 : 0;
    }
  }
}

cudaError_t launch_warp(int B, int H, int W, const double* ab, const uint8_t* target,
                        uint8_t* warped, uint8_t* valid, int32_t* shift, cudaStream_t st) {
  dim3 grid(H, B);
  k_warp<<<grid, 256, 0, st>>>(H, W, ab, target, warped, valid, shift);
  return cudaGetLastError();
}

// K1' — interpolating variant (NEXT row f2, reading 21; oracle
// oracle/interp_warp.py).  Row v is resampled at x = u - t(v), t = alpha v + beta
// (fp64 multiply then add), by linear interpolation at the position quantised to
// 1/256 px (q = floor(256 f + 1/2), f = x - floor(x)); intensities are stored in
// 8.8 fixed point, W' = (256 - q) T(x0) + q T(x0 + 1), an exact integer.  The
// applied shift t_q(v) = -(x0(0) + q / 256) is written for post-processing.
__global__ void __launch_bounds__(256) k_warp_linear(int H, int W, const double* __restrict__ ab,
                                                     const uint8_t* __restrict__ target,
                                                     uint16_t* __restrict__ warped,
                                                     uint8_t* __restrict__ valid,
                                                     double* __restrict__ shift) {
  const int v = blockIdx.x, b = blockIdx.y;
  const double alpha = ab[2 * b], beta = ab[2 * b + 1];
  double t = __dmul_rn(alpha, (double)v);
  t = __dadd_rn(t, beta);
  const double x = __dsub_rn(0.0, t);
  double x0d = floor(x);
  const double f = __dsub_rn(x, x0d);                          // exact
  double qd = floor(__dadd_rn(__dmul_rn(f, 256.0), 0.5));
  if (qd == 256.0) { x0d += 1.0; qd = 0.0; }
  x0d = fmin(fmax(x0d, -1073741824.0), 1073741824.0);
  const long long x00 = (long long)x0d;
  const int q = (int)qd;
  if (threadIdx.x == 0) shift[(size_t)b * H + v] = -((double)x00 + qd / 256.0);
  const size_t row = ((size_t)b * H + v) * W;
  const uint8_t* src = target + row;
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const long long x0 = x00 + u;
    const bool ok = q == 0 ? (x0 >= 0 && x0 <= W - 1) : (x0 >= 0 && x0 + 1 <= W - 1);
    uint32_t val = 0;
    if (ok) {
      const uint32_t a = src[x0];
      const uint32_t c = q ? (uint32_t)src[x0 + 1] : 0u;
      val = (256u - (uint32_t)q) * a + (uint32_t)q * c;
    }
    warped[row + u] = (uint16_t)val;
    valid[row + u] = ok ? 1 : 0;
  }
}

cudaError_t launch_warp_linear(int B, int H, int W, const double* ab, const uint8_t* target,
                               uint16_t* warped, uint8_t* valid, double* shift, cudaStream_t st) {
  dim3 grid(H, B);
  k_warp_linear<<<grid, 256, 0, st>>>(H, W, ab, target, warped, valid, shift);
  return cudaGetLastError();
}

}  // namespace rsr
