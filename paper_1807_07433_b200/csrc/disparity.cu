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

// Group-cooperative argmax: G8 = 8 lanes own one pixel; lane l reads
// disparities {4l..4l+3} and {32+4l..32+4l+3} of each 64-wide chunk (two
// 16-byte loads; the 8 lanes of a group cover 256 contiguous bytes, a warp
// four pixels = 1 KB per load pair), keeps the smallest index attaining the
// maximum over non-NaN entries, and the group reduces (value, index) pairs
// with three xor-shuffles.  -1 if no entry is finite.
constexpr int DG = 8;   // lanes per pixel

// Lane-local part: the lane's best over its 8 entries of each 64-wide chunk.  A
// lane sees its disparities in increasing order, so "strictly greater" keeps the
// first (smallest) index among equal maxima; max(x, NaN) = x skips NaN entries.
// Per 8 values: 8 FMNMX for the maximum, then the first index equal to it.
template <int DGT>
RSR_DEVINL void lane_best(const float* __restrict__ p, int D, int l, bool vec4, float& best, int& kb) {
  best = -INFINITY;
  kb = -1;
  // chunks of 8 DGT disparities: lane l reads {4l..4l+3} and {4 DGT + 4l..+3}
  for (int c0 = 0; c0 < D; c0 += 8 * DGT) {
    float v[8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int k = c0 + 4 * DGT * h + 4 * l;
      if (vec4 && k + 3 < D) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p + k));
        v[4 * h] = t.x; v[4 * h + 1] = t.y; v[4 * h + 2] = t.z; v[4 * h + 3] = t.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++) v[4 * h + q] = (k + q < D) ? __ldg(p + k + q) : qnan();
      }
    }
    float m = v[0];
#pragma unroll
    for (int q = 1; q < 8; q++) m = fmaxf(m, v[q]);
    if (m > best) {   // false when every entry is NaN (m is NaN)
      best = m;
      int kk = -1;
#pragma unroll
      for (int q = 7; q >= 0; q--)
        if (v[q] == m) kk = c0 + 4 * DGT * (q >> 2) + 4 * l + (q & 3);
      kb = kk;
    }
  }
}

template <int DGT>
RSR_DEVINL int group_reduce(float best, int kb) {
#pragma unroll
  for (int o = DGT / 2; o >= 1; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int ok = __shfl_xor_sync(0xffffffffu, kb, o);
    if (ok >= 0 && (kb < 0 || ov > best || (ov == best && ok < kb))) { best = ov; kb = ok; }
  }
  return kb;
}


// ShiftT: int32_t (integer warp, reading 1: d = r_s + s(v) in fp32) or double (the
// interpolating warp, reading 21: d = fp32(r_s + t_q(v)) with the sum in fp64).
template <typename ShiftT, int DGT>
__global__ void __launch_bounds__(256) k_disparity(int H, int W, int d_lo, int D, int tol,
                                                   int subpix, const float* __restrict__ agg_ref,
                                                   const float* __restrict__ agg_tar,
                                                   const ShiftT* __restrict__ shift,
                                                   float* __restrict__ disp,
                                                   int16_t* __restrict__ wta_ref,
                                                   int16_t* __restrict__ wta_tar) {
  extern __shared__ int16_t kr_s[];  // [W]
  const int v = blockIdx.x, b = blockIdx.y;
  const size_t row = ((size_t)b * H + v) * W;
  const bool vec4 = (D & 3) == 0;
  const int l = threadIdx.x % DGT, g = threadIdx.x / DGT, ng = blockDim.x / DGT;
  const int Wr = (W + 4 * ng - 1) / (4 * ng) * (4 * ng);   // uniform trip count: every lane reaches the shuffles
  // two pixels per group per iteration: four 16-byte loads in flight per lane
  // (measured: 2 beats 1, 4 and 8 -- fewer registers, more resident CTAs)
  constexpr int UP = 2;
  for (int u0 = g; u0 < Wr; u0 += UP * ng) {
    float bv[UP];
    int bk[UP];
#pragma unroll
    for (int e = 0; e < UP; e++) {
      const int uu = min(u0 + e * ng, W - 1);
      lane_best<DGT>(agg_tar + (row + uu) * D, D, l, vec4, bv[e], bk[e]);
    }
#pragma unroll
    for (int e = 0; e < UP; e++) {
      const int u = u0 + e * ng;
      const int k = group_reduce<DGT>(bv[e], bk[e]);
      if (l == 0 && u < W) {
        kr_s[u] = (int16_t)k;
        if (wta_tar) wta_tar[row + u] = (int16_t)k;
      }
    }
  }
  __syncthreads();
  const ShiftT sv = shift[(size_t)b * H + v];
  for (int u0 = g; u0 < Wr; u0 += UP * ng) {
    float bv[UP];
    int bk[UP];
#pragma unroll
    for (int e = 0; e < UP; e++) {
      const int uu = min(u0 + e * ng, W - 1);
      lane_best<DGT>(agg_ref + (row + uu) * D, D, l, vec4, bv[e], bk[e]);
    }
#pragma unroll
    for (int e = 0; e < UP; e++) {
      const int u = u0 + e * ng;
      const int k = group_reduce<DGT>(bv[e], bk[e]);
      if (l != 0 || u >= W) continue;
      const float* p = agg_ref + (row + u) * D;
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
            d = sizeof(ShiftT) == 4 ? r + (float)sv : (float)((double)r + (double)sv);
          }
        }
      }
      disp[row + u] = d;
    }
  }
}

// Small search ranges (D <= 16: the restricted band of P:251): one thread per pixel
// scans its D costs (a pixel is 32-64 contiguous bytes; a warp's loads cover 32
// consecutive pixels), instead of an 8-lane group of which only D/4 lanes would
// load.  Same WTA rule (first index of the maximum over non-NaN entries), same
// Eq. (11)-(12) arithmetic: results identical to k_disparity.
RSR_DEVINL int pixel_argmax(const float* __restrict__ p, int D) {
  float best = -INFINITY;
  int kb = -1;
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; k++) v[k] = k < D ? __ldg(p + k) : qnan();
#pragma unroll
  for (int k = 0; k < 16; k++)
    if (v[k] > best) { best = v[k]; kb = k; }   // NaN never compares greater
  return kb;
}

template <typename ShiftT>
__global__ void __launch_bounds__(256) k_disparity_small(int H, int W, int d_lo, int D, int tol, int subpix,
                                                         const float* __restrict__ agg_ref,
                                                         const float* __restrict__ agg_tar,
                                                         const ShiftT* __restrict__ shift,
                                                         float* __restrict__ disp,
                                                         int16_t* __restrict__ wta_ref,
                                                         int16_t* __restrict__ wta_tar) {
  extern __shared__ int16_t krs_s[];  // [W]
  const int v = blockIdx.x, b = blockIdx.y;
  const size_t row = ((size_t)b * H + v) * W;
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const int k = pixel_argmax(agg_tar + (row + u) * D, D);
    krs_s[u] = (int16_t)k;
    if (wta_tar) wta_tar[row + u] = (int16_t)k;
  }
  __syncthreads();
  const ShiftT sv = shift[(size_t)b * H + v];
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const float* p = agg_ref + (row + u) * D;
    const int k = pixel_argmax(p, D);
    if (wta_ref) wta_ref[row + u] = (int16_t)k;
    float d = qnan();
    if (k >= 0) {
      const int up = u - (k + d_lo);
      if (up >= 0 && up < W) {
        const int kr = krs_s[up];
        if (kr >= 0 && abs(k - kr) <= tol) {
          float r = (float)(k + d_lo);
          if (subpix && k >= 1 && k <= D - 2) {
            const float a = p[k - 1], bb = p[k], c = p[k + 1];
            const float den = 2.f * a + 2.f * c - 4.f * bb;
            if (!(a != a) && !(c != c) && fabsf(den) > 1e-12f) r += __fdiv_rn(a - c, den);
          }
          d = sizeof(ShiftT) == 4 ? r + (float)sv : (float)((double)r + (double)sv);
        }
      }
    }
    disp[row + u] = d;
  }
}

template <typename ShiftT>
static cudaError_t disparity_launch_t(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                                      const float* agg_ref, const float* agg_tar, const ShiftT* shift,
                                      float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st) {
  const size_t smem = sizeof(int16_t) * (size_t)W;
  dim3 grid(H, B);
  if (D <= 16) {
    const cudaError_t e = smem_optin((const void*)k_disparity_small<ShiftT>, smem);
    if (e != cudaSuccess) return e;
    k_disparity_small<ShiftT><<<grid, 256, smem, st>>>(H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp,
                                                       wta_ref, wta_tar);
  } else if (D <= 32) {
    // 16 < D <= 32 (the paper's d_max = 30): 4-lane groups, one 32-wide chunk per pixel
    const cudaError_t e = smem_optin((const void*)k_disparity<ShiftT, 4>, smem);
    if (e != cudaSuccess) return e;
    k_disparity<ShiftT, 4><<<grid, 256, smem, st>>>(H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp,
                                                    wta_ref, wta_tar);
  } else {
    const cudaError_t e = smem_optin((const void*)k_disparity<ShiftT, DG>, smem);
    if (e != cudaSuccess) return e;
    k_disparity<ShiftT, DG><<<grid, 256, smem, st>>>(H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp,
                                                     wta_ref, wta_tar);
  }
  return cudaGetLastError();
}

cudaError_t launch_disparity(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                             const float* agg_ref, const float* agg_tar, const int32_t* shift,
                             float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st) {
  return disparity_launch_t<int32_t>(B, H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp, wta_ref,
                                     wta_tar, st);
}

cudaError_t launch_disparity_frac(int B, int H, int W, int d_lo, int D, int tol, int subpix,
                                  const float* agg_ref, const float* agg_tar, const double* shift,
                                  float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st) {
  return disparity_launch_t<double>(B, H, W, d_lo, D, tol, subpix, agg_ref, agg_tar, shift, disp, wta_ref,
                                    wta_tar, st);
}

}  // namespace rsr
