// K2' — NCC cost volumes for the interpolating warp (NEXT row f2, DESIGN.md
// reading 21): the same Eqs. (3)-(5) on the reference image
// L (uint8) and the 8.8 fixed-point warped image W' (uint16).  NCC is invariant
// to the 256 scale of W', so
//   c(u,v,r) = (n S_lw' - S_l S_w') / (sqrt(n S_ll - S_l^2) sqrt(n S_w'w' - S_w'^2))
// with every sum an exact integer: products l w' < 2^24, block dot sums
// <= 225 * 255 * 65280 < 2^32 (uint32, sliding add/subtract exact modulo 2^32),
// the numerator in int64.  One fp32 normalisation per entry (the statistics
// 1/sqrt(.) come from k_block_stats<p, uint16_t>), multiplied in the order
// num * inv_L * inv_W' for both volumes, so vol_tar[v][u - r][k] ==
// vol_ref[v][u][k] bit for bit.
//
// A CTA owns ZTX = 64 columns x ZBY rows x all D (<= 64 per launch slab); a thread
// owns X columns x 8 disparities and slides exact vertical dot sums down the band
// (image rows stream through a shared-memory ring, prefetched one row ahead in
// registers).  Integer multiply-adds (IMAD) instead of the uint8 path's exact
// FFMA2 pairs: the 8.8 products do not fit the fp32 mantissa over a block.
#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int FX_TX = 64;   // columns per CTA
constexpr int FX_BY = 64;   // output rows per CTA
constexpr int FX_R = 8;     // disparities per thread

template <int P>
struct FxCfg {
  static constexpr int X = P <= 3 ? 4 : 2;           // columns per thread (registers: NJ x 8 sums)
  static constexpr int NJ = X + 2 * P;               // vertical-sum columns per thread
  static constexpr int NCG = FX_TX / X;              // column groups
};

template <int P, bool TAR>
__device__ __forceinline__ void fx_cta(int b, int H, int W, int d_lo, int D, int Dst, int koff,
                                       const uint8_t* __restrict__ ref, const uint16_t* __restrict__ warped,
                                       const int32_t* __restrict__ SL, const float* __restrict__ iL,
                                       const int32_t* __restrict__ SW, const float* __restrict__ iW,
                                       float* __restrict__ vol) {
  using C = FxCfg<P>;
  constexpr int X = C::X, NJ = C::NJ;
  constexpr int NRING = 2 * P + 3;
  extern __shared__ __align__(16) int fx_smem[];
  const int d_hi = d_lo + D - 1;
  const int FC = FX_TX + 2 * P;
  const int GC = FX_TX + 2 * P + D - 1;
  int* Fs = fx_smem;                 // [NRING][FC]  F image rows (REF: L, TAR: W')
  int* Gs = Fs + NRING * FC;         // [NRING][GC]  G image rows (REF: W' at x - r, TAR: L at x + r)
  const int x0 = blockIdx.x * FX_TX, y0 = blockIdx.y * FX_BY;
  const size_t ibase = (size_t)b * H * W;
  // first image column of the F / G rows in shared memory
  const int f0 = x0 - P;
  const int g0 = TAR ? x0 - P + d_lo : x0 - P - d_hi;
  const int nrows = min(FX_BY, H - y0);

  constexpr int NPF = 4;   // prefetched elements per thread per row (blockDim >= (FC + GC) / NPF)
  int pf[NPF];
  auto fetch = [&](int t) {   // image row y0 - P + t
    const int yy = y0 - P + t;
    const bool rin = yy >= 0 && yy < H;
#pragma unroll
    for (int e = 0; e < NPF; e++) {
      const int i = threadIdx.x + e * blockDim.x;
      int v = 0;
      if (rin && i < FC + GC) {
        const bool isF = i < FC;
        const int xx = isF ? f0 + i : g0 + (i - FC);
        if (xx >= 0 && xx < W) {
          const size_t gi = ibase + (size_t)yy * W + xx;
          // F is L for the reference volume and W' for the target volume
          v = (isF != TAR) ? (int)__ldg(ref + gi) : (int)__ldg(warped + gi);
        }
      }
      pf[e] = v;
    }
  };
  auto commit = [&](int t) {
    const int slot = t % NRING;
#pragma unroll
    for (int e = 0; e < NPF; e++) {
      const int i = threadIdx.x + e * blockDim.x;
      if (i < FC) Fs[slot * FC + i] = pf[e];
      else if (i < FC + GC) Gs[slot * GC + (i - FC)] = pf[e];
    }
  };

  const int n_rg = (D + FX_R - 1) / FX_R;
  const int rg = threadIdx.x % n_rg, cg = threadIdx.x / n_rg;
  const bool active = cg < C::NCG;
  const int r0 = d_lo + FX_R * rg;            // first residual disparity of the thread
  const int u_t = x0 + X * cg;                // first output column of the thread
  const int nq = max(0, min(FX_R, d_hi - r0 + 1));
  // G entry of (vertical-sum column j, disparity q): G column = F column -/+ r
  //   REF: (u_t - P + j) - (r0 + q) -> smem index (X cg + j) + (d_hi - r0) - q
  //   TAR: (u_t - P + j) + (r0 + q) -> smem index (X cg + j) + (r0 - d_lo) + q
  const int gbase = TAR ? X * cg + (r0 - d_lo) : X * cg + (d_hi - r0) - (FX_R - 1);
  // (REF: entries gbase .. gbase + NJ + 6 cover j - q + 7 for j < NJ, q < 8)

  uint32_t V[NJ][FX_R];
#pragma unroll
  for (int j = 0; j < NJ; j++)
#pragma unroll
    for (int q = 0; q < FX_R; q++) V[j][q] = 0u;

  auto accumulate = [&](int t, bool sub) {
    const int slot = t % NRING;
    const int* fr = Fs + slot * FC + X * cg;
    const int* gr = Gs + slot * GC + gbase;
    uint32_t f[NJ], g[NJ + FX_R - 1];
#pragma unroll
    for (int j = 0; j < NJ; j++) f[j] = sub ? 0u - (uint32_t)fr[j] : (uint32_t)fr[j];
#pragma unroll
    for (int i = 0; i < NJ + FX_R - 1; i++) g[i] = (uint32_t)gr[i];
#pragma unroll
    for (int j = 0; j < NJ; j++)
#pragma unroll
      for (int q = 0; q < FX_R; q++) V[j][q] += f[j] * (TAR ? g[j + q] : g[j + (FX_R - 1) - q]);
  };

  // prologue: image rows 0 .. 2P
  for (int t = 0; t <= 2 * P; t++) {
    fetch(t);
    commit(t);
  }
  __syncthreads();
  const long long n = (long long)(2 * P + 1) * (2 * P + 1);

  for (int y = 0; y < nrows; y++) {
    const bool more = y + 1 < nrows;
    if (more) fetch(y + 1 + 2 * P);
    if (active) {
      if (y == 0) {
#pragma unroll 1
        for (int t = 0; t <= 2 * P; t++) accumulate(t, false);
      } else {
        accumulate(y + 2 * P, false);
        accumulate(y - 1, true);
      }
      const int yy = y0 + y;
      const size_t prow = ibase + (size_t)yy * W;
      uint32_t hs[FX_R];
#pragma unroll
      for (int q = 0; q < FX_R; q++) {
        uint32_t a = 0u;
#pragma unroll
        for (int dx = 0; dx <= 2 * P; dx++) a += V[dx][q];
        hs[q] = a;
      }
#pragma unroll
      for (int i = 0; i < X; i++) {
        const int u = u_t + i;
        if (i > 0) {
#pragma unroll
          for (int q = 0; q < FX_R; q++) hs[q] += V[i + 2 * P][q] - V[i - 1][q];
        }
        if (u >= W) continue;
        // F-side statistics at u; G-side at u -/+ r (outside the image: NaN norm)
        const long long sF = TAR ? __ldg(SW + prow + u) : __ldg(SL + prow + u);
        const float iF = TAR ? __ldg(iW + prow + u) : __ldg(iL + prow + u);
        float out[FX_R];
#pragma unroll
        for (int q = 0; q < FX_R; q++) {
          const int ug = TAR ? u + r0 + q : u - r0 - q;
          float c = qnan();
          if (ug >= 0 && ug < W) {
            const long long sG = TAR ? __ldg(SL + prow + ug) : __ldg(SW + prow + ug);
            const float iG = TAR ? __ldg(iL + prow + ug) : __ldg(iW + prow + ug);
            const long long num = n * (long long)hs[q] - sF * sG;
            // (num * inv_L) * inv_W' in this order for both volumes (bitwise dual identity)
            const float nf = __ll2float_rn(num);
            c = TAR ? (nf * iG) * iF : (nf * iF) * iG;
            c = clamp_unit_nan(c);
          }
          out[q] = c;
        }
        float* dst = vol + (prow + u) * (size_t)Dst + koff + (r0 - d_lo);
        if ((Dst & 3) == 0 && (koff & 3) == 0 && nq == FX_R) {
          reinterpret_cast<float4*>(dst)[0] = make_float4(out[0], out[1], out[2], out[3]);
          reinterpret_cast<float4*>(dst)[1] = make_float4(out[4], out[5], out[6], out[7]);
        } else {
#pragma unroll
          for (int q = 0; q < FX_R; q++)
            if (q < nq) dst[q] = out[q];
        }
      }
    }
    // the ring slot of row y - 2 was last read in iteration y - 1 (before the barrier)
    if (more) commit(y + 1 + 2 * P);
    __syncthreads();
  }
}

template <int P>
__global__ void __launch_bounds__(256) k_zncc_fx_pair(int B, int H, int W, int d_lo, int D, int Dst, int koff,
                                                      const uint8_t* ref, const uint16_t* warped,
                                                      const int32_t* SL, const float* iL, const int32_t* SW,
                                                      const float* iW, float* vol_ref, float* vol_tar) {
  if ((int)blockIdx.z < B)
    fx_cta<P, false>(blockIdx.z, H, W, d_lo, D, Dst, koff, ref, warped, SL, iL, SW, iW, vol_ref);
  else
    fx_cta<P, true>(blockIdx.z - B, H, W, d_lo, D, Dst, koff, ref, warped, SL, iL, SW, iW, vol_tar);
}

template <int P>
static cudaError_t fx_launch_t(int B, int H, int W, int d_lo, int D, int Dst, int koff, const uint8_t* ref,
                               const uint16_t* warped, const int32_t* SL, const float* iL, const int32_t* SW,
                               const float* iW, float* vol_ref, float* vol_tar, cudaStream_t st) {
  using C = FxCfg<P>;
  const int n_rg = (D + FX_R - 1) / FX_R;
  const int FC = FX_TX + 2 * P, GC = FX_TX + 2 * P + D - 1;
  // compute threads, and enough threads for the 4-element-per-thread row prefetch
  int threads = C::NCG * n_rg;
  threads = threads > (FC + GC + 3) / 4 ? threads : (FC + GC + 3) / 4;
  threads = ((threads + 31) / 32) * 32;
  if (threads > 256) return cudaErrorInvalidValue;
  // + 8 ints: the last disparity group of the target volume reads up to 7 entries past
  // its G row for disparities beyond the slab (never stored)
  const size_t smem = sizeof(int) * ((size_t)(2 * P + 3) * (FC + GC) + 8);
  cudaError_t e = smem_optin((const void*)k_zncc_fx_pair<P>, smem);
  if (e != cudaSuccess) return e;
  const int nz = vol_tar ? 2 * B : B;
  dim3 grid((W + FX_TX - 1) / FX_TX, (H + FX_BY - 1) / FX_BY, nz);
  k_zncc_fx_pair<P><<<grid, threads, smem, st>>>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, iL, SW, iW,
                                                 vol_ref, vol_tar);
  return cudaGetLastError();
}

cudaError_t launch_zncc_fx(int B, int H, int W, int rho_b, int d_lo, int D, const uint8_t* ref,
                           const uint16_t* warped, const int32_t* SL, const float* iL, const int32_t* SW,
                           const float* iW, float* vol_ref, float* vol_tar, cudaStream_t st) {
  constexpr int SLAB = 64;
  if (2LL * B > 65535) return cudaErrorInvalidValue;
  for (int k0 = 0; k0 < D; k0 += SLAB) {
    const int Ds = D - k0 < SLAB ? D - k0 : SLAB;
    const int dl = d_lo + k0;
    cudaError_t e;
    switch (rho_b) {
#define RSR_FX(PP)                                                                                       \
  case PP:                                                                                               \
    e = fx_launch_t<PP>(B, H, W, dl, Ds, D, k0, ref, warped, SL, iL, SW, iW, vol_ref, vol_tar, st);      \
    break;
      RSR_FX(1) RSR_FX(2) RSR_FX(3) RSR_FX(4) RSR_FX(5) RSR_FX(6) RSR_FX(7)
#undef RSR_FX
      default:
        return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rsr
