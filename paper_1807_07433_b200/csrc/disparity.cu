// K4 — WTA, left-right consistency, parabola subpixel and post-processing
// (Eqs. (11)-(12)).
//
// One CTA per image row (b, v).  Phase 1: k_R(u', v) = smallest argmax over the
// non-NaN entries of the aggregated target volume (WTA; "highest
// correlation") for every u' of the row, kept in shared memory.
// Phase 2: k_L(u, v) on the aggregated reference volume, the uniqueness check
// |k_L(u) - k_R(u - r_L)| <= tol (Eq. 11), the parabola of Eq. (12)
// through A_L[k_L-1, k_L, k_L+1] and the post-processing shift
// s(v).  Reads each aggregated volume once (HBM-bound): each thread
// scans one pixel's D contiguous costs with 16-byte loads.
#include "common.cuh"
#include "kernels.h"

namespace rsr {

// smallest index attaining the maximum over non-NaN entries; -1 if none.
RSR_DEVINL int argmax_row(const float* __restrict__ p, int D, bool vec4) {
  float best = -INFINITY;
  int kb = -1;
  if (vec4) {
    const float4* p4 = reinterpret_cast<const float4*>(p);
    for (int k4 = 0; k4 < D / 4; k4++) {
      const float4 t = __ldg(p4 + k4);
      const float v[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
      for (int i = 0; i < 4; i++)
        if (v[i] > best) { best = v[i]; kb = 4 * k4 + i; }  // NaN never compares greater
    }
  } else {
    for (int k = 0; k < D; k++) {
      const float v = __ldg(p + k);
      if (v > best) { best = v; kb = k; }
    }
  }
  return kb;
}

__global__ void __launch_bounds__(256) k_disparity(int H, int W, int d_lo, int D, int tol,
                                                   int subpix, const float* __restrict__ agg_ref,
                                                   const float* __restrict__ agg_tar,
                                                   const int32_t* __restrict__ shift,
                                                   float* __restrict__ disp,
                                                   int16_t* __restrict__ wta_ref,
                                                   int16_t* __restrict__ wta_tar) {
  extern __shared__ int16_t kr_s[];  // [W]
  const int v = blockIdx.x, b = blockIdx.y;
  const size_t row = ((size_t)b * H + v) * W;
  const bool vec4 = (D & 3) == 0;
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const int k = argmax_row(agg_tar + (row + u) * D, D, vec4);
    kr_s[u] = (int16_t)k;
    if (wta_tar) wta_tar[row + u] = (int16_t)k;
  }
  __syncthreads();
  const float sv = (float)shift[(size_t)b * H + v];
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const float* p = agg_ref + (row + u) * D;
    const int k = argmax_row(p, D, vec4);
    if (wta_ref) wta_ref[row + u] = (int16_t)k;
    float d = qnan();
    if (k >= 0) {
      const int up = u - (k + d_lo);
      if (up >= 0 && up < W) {
        const int kr = kr_s[up];
        if (kr >= 0 && abs(k - kr) <= tol) {
          float r = (float)(k + d_lo);
          if (subpix && k >= 1 && k <= D - 2) {
            const float a = p[k - 1], bb = p[k], c = p[k + 1];
            const float den = 2.f * a + 2.f * c - 4.f * bb;
            if (!(a != a) && !(c != c) && fabsf(den) > 1e-12f) r += __fdiv_rn(a - c, den);
          }
          d = r + sv;
        }
      }
    }
    disp[row + u] = d;
  }
}

cudaError_t launch_disparity(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                             const float* agg_ref, const float* agg_tar, const int32_t* shift,
                             float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st) {
  const size_t smem = sizeof(int16_t) * (size_t)W;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_disparity, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(H, B);
  k_disparity<<<grid, 256, smem, st>>>(H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp,
                                       wta_ref, wta_tar);
  return cudaGetLastError();
}

}  // namespace rsr
