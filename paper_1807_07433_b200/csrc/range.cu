// Restricted search range (NEXT row f4, PAPER.md:251 future work; DESIGN.md
// reading 20): the residual band [floor(min r) - delta, ceil(max r) + delta] of
// r = d(u, v) - s(v) over the finite entries of the previous frame's disparity map
// d, clipped to [lo_lim, hi_lim]; the full limits for an empty map.  One CTA per
// frame: a grid-stride fp64 min / max (exact: d is fp32, s an integer), warp
// shuffles, then one warp over the per-warp partials.  min / max are
// order-independent, so the result is deterministic.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int SR_THREADS = 512;

__global__ void __launch_bounds__(SR_THREADS) k_search_range(int H, int W, int delta, int lo_lim, int hi_lim,
                                                             const float* __restrict__ disp,
                                                             const int32_t* __restrict__ shift,
                                                             int32_t* __restrict__ range) {
  __shared__ double smin[SR_THREADS / 32], smax[SR_THREADS / 32];
  const int b = blockIdx.x;
  const float* d = disp + (size_t)b * H * W;
  const int32_t* s = shift + (size_t)b * H;
  double lo = INFINITY, hi = -INFINITY;
  for (int v = 0; v < H; v++) {
    const double sv = (double)__ldg(s + v);
    const float* row = d + (size_t)v * W;
    for (int u = threadIdx.x; u < W; u += SR_THREADS) {
      const float x = __ldg(row + u);
      if (isfinite(x)) {
        const double r = (double)x - sv;
        lo = fmin(lo, r);
        hi = fmax(hi, r);
      }
    }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smin[warp] = lo;
    smax[warp] = hi;
  }
  __syncthreads();
  if (warp == 0) {
    lo = lane < SR_THREADS / 32 ? smin[lane] : INFINITY;
    hi = lane < SR_THREADS / 32 ? smax[lane] : -INFINITY;
    for (int o = 16; o >= 1; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      long long a = lo_lim, c = hi_lim;
      if (lo <= hi) {   // some finite entry
        a = (long long)floor(lo) - delta;
        c = (long long)ceil(hi) + delta;
        a = a < lo_lim ? lo_lim : (a > hi_lim ? hi_lim : a);
        c = c < lo_lim ? lo_lim : (c > hi_lim ? hi_lim : c);
      }
      range[2 * b] = (int32_t)a;
      range[2 * b + 1] = (int32_t)c;
    }
  }
}

cudaError_t launch_search_range(int B, int H, int W, int delta, int lo_lim, int hi_lim, const float* disp,
                                const int32_t* shift, int32_t* range, cudaStream_t st) {
  k_search_range<<<B, SR_THREADS, 0, st>>>(H, W, delta, lo_lim, hi_lim, disp, shift, range);
  return cudaGetLastError();
}

}  // namespace rsr
