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

}  // namespace rsr
