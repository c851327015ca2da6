// K3 (sliding-window, warp-specialised) — bilateral cost aggregation,
// PAPER.md:128-152, Eq. (8) with Eqs. (9)-(10); same definition and readings
// as aggregate.cu (readings 10-12).  Used for rho <= 7.
//
// Why this shape (profiles/r01_*):
//  * A CTA owns a 32-column strip and a chunk of R output rows and slides
//    down it one input row at a time.  A consumer thread holds the 2 rho + 1
//    output rows whose windows contain the current input row ("ages" 0..2rho)
//    x 8 disparities as 4 packed pairs, so every input row feeds every held
//    row: no predicated-off FMA at tile edges.  The register slot of an age
//    rotates by one per input row; the loop is unrolled by the period
//    2 rho + 1 so all register indices are static.
//  * Producer warps (4) compute the weights of the next input rows once per
//    CTA (exp2 on the MUFU pipe), write them in age order to a weight stage,
//    keep the per-pixel sum of weights, and drive the cost-row pipeline
//    (one 256-byte cp.async.bulk per pixel column, TMA engine).  Consumers and
//    producers hand off through mbarriers: no CTA-wide barrier in the loop.
//  * Inner product: FFMA2 (fma.rn.f32x2) with the tap weight as scalar
//    broadcast operand; per tap a consumer loads 2 x LDS.128 of costs and
//    4 x LDS.128 of weights for 52 FFMA2 (104 FMA).
//  * Clean chunks (footprint inside the image and NaN-free per nan_map) use
//    pair = (k, k+1) and a per-pixel denominator; other chunks use
//    pair = (C0, V) (cost or 0, validity) in two passes, exact for any NaN
//    pattern.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int SL_KT = 8;        // disparities per consumer thread
constexpr int SL_NPROD = 3;     // weight-producer warps (+1 stager warp)
constexpr int SL_NSC = 4;       // cost stages
constexpr int SL_NSW = 3;       // weight stages
constexpr int SL_ROWS = 180;    // output rows per CTA chunk

struct SlideGeom {
  int n_kg, KS, DPAD, CX, WX, WSTAGE, GR, GC, nslab, R;
  size_t off_cost, off_w, off_dsum, off_guide, off_bar, bytes;
};

// cost stage: [CX columns][KS + 4] raw fp32 costs (NaN = invalid)
// weight stage: [32 x][NT taps][16 ages] (x stride padded to 4*odd floats)
// + dsum partials [SL_NPROD][32]
__host__ __device__ inline SlideGeom slide_geom(int D, int rho, int H) {
  SlideGeom g;
  const int NT = 2 * rho + 1;
  const int ks = D < 64 ? D : 64;
  g.n_kg = (ks + SL_KT - 1) / SL_KT;
  g.KS = g.n_kg * SL_KT;
  g.DPAD = g.KS + 4;
  g.CX = 32 + 2 * rho;
  int wx = NT * 16;
  if (((wx / 4) & 1) == 0) wx += 4;
  g.WX = wx;
  g.WSTAGE = 32 * g.WX + SL_NPROD * 32;
  g.R = SL_ROWS < H ? SL_ROWS : H;
  g.GR = g.R + 4 * rho;   // output rows y in [Y0 - 2 rho, Y1 + 2 rho)
  g.GC = 32 + 2 * rho;
  g.nslab = (D + g.KS - 1) / g.KS;
  size_t o = 0;
  g.off_cost = o; o += sizeof(float) * (size_t)SL_NSC * g.CX * g.DPAD;
  g.off_w = o;    o += sizeof(float) * (size_t)SL_NSW * g.WSTAGE;
  g.off_dsum = o; o += sizeof(float) * (size_t)SL_NPROD * NT * 32;
  g.off_guide = o; o += sizeof(float) * (size_t)g.GR * g.GC;
  o = (o + 15) & ~size_t(15);
  g.off_bar = o;  o += 8 * (2 * SL_NSC + 2 * SL_NSW) + 16;
  g.bytes = o;
  return g;
}

RSR_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Per-CTA context shared by the three warp roles.
struct SlideCtx {
  SlideGeom g;
  float* cost_s;
  float* w_s;
  float* dsum_s;
  float* guide_s;
  uint64_t *full_c, *empty_c, *full_w, *empty_w;
  const float* vol;
  float* out;
  int H, W, D, x0, Y0, Y1, k0, ks_eff, NR, lane;
  size_t pix0;
  float kd, kr;
  bool clean;
};

// ---- stager (1 warp): raw cost rows into stage it % NSC.  One bulk copy per
// in-image pixel column (TMA engine); skipped columns (outside the image, or
// all-NaN on a clean chunk) are filled with 0 (clean) or NaN (general path).
template <int RHO>
__device__ __noinline__ void slide_stager(const SlideCtx c, int npass) {
  const SlideGeom& g = c.g;
  const int lane = c.lane;
  const bool bulk = (c.D & 3) == 0;
  uint32_t it_c = 0;
  for (int pass = 0; pass < npass; pass++) {
    for (int i = 0; i < c.NR; i++, it_c++) {
      const int st = it_c % SL_NSC;
      if (it_c >= SL_NSC) mbar_wait_parity(&c.empty_c[st], ((it_c / SL_NSC) & 1) ^ 1);
      const int yy = c.Y0 - RHO + i;
      float* dst = c.cost_s + (size_t)st * g.CX * g.DPAD;
      const bool row_in = yy >= 0 && yy < c.H;
      const float* gtile = c.guide_s + (i + RHO) * g.GC;   // same row / columns as the stage
      const float fillv = c.clean ? 0.f : qnan();
      // each lane owns columns lane and lane + 32 (CX <= 46)
      bool copy_col[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int col = lane + 32 * h;
        const int xx = c.x0 - RHO + col;
        const bool in = col < g.CX && row_in && xx >= 0 && xx < c.W;
        copy_col[h] = in && bulk && !(c.clean && gtile[col] != gtile[col]);
        if (col < g.CX && !copy_col[h]) {
          float* d = dst + col * g.DPAD;
          if (in && !bulk) {
            const float* sp = c.vol + (c.pix0 + (size_t)yy * c.W + xx) * c.D + c.k0;
            for (int k = 0; k < g.KS; k++) d[k] = (c.k0 + k < c.D) ? sp[k] : qnan();
          } else {
            for (int k = 0; k < g.KS; k += 4) *reinterpret_cast<float4*>(d + k) = make_float4(fillv, fillv, fillv, fillv);
          }
        }
      }
      const uint32_t ncols = __popc(__ballot_sync(0xffffffffu, copy_col[0])) +
                             __popc(__ballot_sync(0xffffffffu, copy_col[1]));
      __syncwarp();
      const uint32_t bytes_col = (uint32_t)c.ks_eff * 4u;
      if (lane == 0) mbar_arrive_expect_tx(&c.full_c[st], bytes_col * ncols);
      __syncwarp();
      const float* src = c.vol + ((c.pix0 + (size_t)yy * c.W + (c.x0 - RHO)) * c.D + c.k0);
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int col = lane + 32 * h;
        if (copy_col[h]) bulk_g2s(dst + col * g.DPAD, src + (size_t)col * c.D, bytes_col, &c.full_c[st]);
      }
    }
  }
}

// ---- weight producers (SL_NPROD warps): weights of input row i in age order,
// w[x][tap][age] = exp2(kd (dx^2 + dy^2) + kr (g(q) - g(p))^2), 0 for a skipped
// tap (NaN guide); per-pixel weight sums per output row.
template <int RHO>
__device__ __noinline__ void slide_weights(const SlideCtx c, int p, int npass) {
  constexpr int NT = 2 * RHO + 1;
  const SlideGeom& g = c.g;
  const int x = c.lane;
  float* dpart = c.dsum_s + (size_t)p * NT * 32;   // [row slot][x] ring, private to warp p
  uint32_t it_w = 0;
  for (int pass = 0; pass < npass; pass++) {
    for (int a = 0; a < NT; a++) dpart[a * 32 + x] = 0.f;
    for (int i = 0; i < c.NR; i++, it_w++) {
      const int st = it_w % SL_NSW;
      if (it_w >= SL_NSW) mbar_wait_parity(&c.empty_w[st], ((it_w / SL_NSW) & 1) ^ 1);
      float* wst = c.w_s + (size_t)st * g.WSTAGE;
      const float* grow = c.guide_s + (i + RHO) * g.GC + x;   // input row r, column x - RHO
      // age a (0 = oldest) holds output row y = r - RHO + a, i.e. dy = r - y = RHO - a;
      // its guide value g(x, y) sits in guide tile row y - (Y0 - 2 RHO) = i + a.
      // Skipped pixels (NaN in the guide tile) are re-encoded so that their weight
      // underflows to exactly 0 without a branch: -1e18 as a centre, +1e18 as a tap
      // (|dg| >= 1e18 - 255, kr dg^2 <= -1e6 even for gamma_r = inf where kr = -1e-30).
      float gp[NT];
#pragma unroll
      for (int a = 0; a < NT; a++) {
        const float v = c.guide_s[(i + a) * g.GC + x + RHO];
        gp[a] = (v != v) ? -1e18f : v;
      }
      float cy[NT];
#pragma unroll
      for (int a = 0; a < NT; a++) cy[a] = (float)((RHO - a) * (RHO - a)) * c.kd;
      float dpa[NT];
#pragma unroll
      for (int a = 0; a < NT; a++) dpa[a] = 0.f;
      for (int j = p; j < NT; j += SL_NPROD) {
        const float gv = grow[j];
        const float gq = (gv != gv) ? 1e18f : gv;
        const float cx = (float)((j - RHO) * (j - RHO)) * c.kd;
        float wv[16];
#pragma unroll
        for (int a = 0; a < NT; a++) {
          const float dg = gq - gp[a];
          const float arg = fmaf(dg * c.kr, dg, cx + cy[a]);
          wv[a] = ex2_approx(arg);
          dpa[a] += wv[a];
        }
#pragma unroll
        for (int a = NT; a < 16; a++) wv[a] = 0.f;
        float4* d4 = reinterpret_cast<float4*>(wst + x * g.WX + j * 16);
#pragma unroll
        for (int q = 0; q < 4; q++) d4[q] = make_float4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
      }
      // running per-pixel weight sums per output row; row y = Y0 - 2 RHO + i + a
      // lives in ring slot (i + a) % NT (the consumers' register slot as well)
#pragma unroll
      for (int a = 0; a < NT; a++) dpart[((i + a) % NT) * 32 + x] += dpa[a];
      // row completing at input row i: age 0, slot i % NT
      const int cs = i % NT;
      wst[32 * g.WX + p * 32 + x] = dpart[cs * 32 + x];
      dpart[cs * 32 + x] = 0.f;
      mbar_arrive(&c.full_w[st]);
    }
  }
}

// ---- consumers (one warp per 8 disparities): sliding accumulation ----
template <int RHO, bool CLEAN>
__device__ __forceinline__ void slide_consume(const SlideCtx& c, int kg) {
  constexpr int NT = 2 * RHO + 1;
  constexpr int NPASS = CLEAN ? 1 : 2;
  const SlideGeom& g = c.g;
  const int lane = c.lane;
  const int x = c.x0 + lane;
  uint32_t it = 0;
  for (int pass = 0; pass < NPASS; pass++) {
    float2 acc[NT][SL_KT / 2];
#pragma unroll
    for (int a = 0; a < NT; a++)
#pragma unroll
      for (int q = 0; q < SL_KT / 2; q++) acc[a][q] = make_float2(0.f, 0.f);

    for (int base = 0; base < c.NR; base += NT) {
#pragma unroll
      for (int u = 0; u < NT; u++) {
        const int i = base + u;
        if (i < c.NR) {
          const int stc = it % SL_NSC, stw = it % SL_NSW;
          mbar_wait_parity(&c.full_c[stc], (it / SL_NSC) & 1);
          mbar_wait_parity(&c.full_w[stw], (it / SL_NSW) & 1);
          const float* crow = c.cost_s + (size_t)stc * g.CX * g.DPAD + lane * g.DPAD + kg * SL_KT;
          const float* wrow = c.w_s + (size_t)stw * g.WSTAGE + lane * g.WX;
#pragma unroll
          for (int j = 0; j < NT; j++) {
            float2 cp[4];
            if (CLEAN) {
              const float4* c4 = reinterpret_cast<const float4*>(crow + j * g.DPAD);
              const float4 ca = c4[0], cb = c4[1];
              cp[0] = make_float2(ca.x, ca.y); cp[1] = make_float2(ca.z, ca.w);
              cp[2] = make_float2(cb.x, cb.y); cp[3] = make_float2(cb.z, cb.w);
            } else {
              // (C0, V): cost or 0, validity, for k = k0 + 8 kg + 4 pass + q
              const float4 t = *reinterpret_cast<const float4*>(crow + j * g.DPAD + 4 * pass);
              const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const bool ok = !(tv[q] != tv[q]);
                cp[q] = make_float2(ok ? tv[q] : 0.f, ok ? 1.f : 0.f);
              }
            }
            const float4* w4 = reinterpret_cast<const float4*>(wrow + j * 16);
            float wv[16];
#pragma unroll
            for (int q = 0; q < (NT + 3) / 4; q++) {
              const float4 t = w4[q];
              wv[4 * q] = t.x; wv[4 * q + 1] = t.y; wv[4 * q + 2] = t.z; wv[4 * q + 3] = t.w;
            }
#pragma unroll
            for (int a = 0; a < NT; a++) {
              // age a lives in register slot (u + a) % NT
#pragma unroll
              for (int q = 0; q < 4; q++) ffma2_bcast(acc[(u + a) % NT][q], wv[a], cp[q]);
            }
          }
          // completing output row: age 0, slot u, image row y = Y0 - 2 RHO + i
          const int y = c.Y0 - 2 * RHO + i;
          float den = 0.f;
          if (CLEAN) {
            const float* dsrc = c.w_s + (size_t)stw * g.WSTAGE + 32 * g.WX;
#pragma unroll
            for (int pp = 0; pp < SL_NPROD; pp++) den += dsrc[pp * 32 + lane];
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&c.empty_c[stc]);
            mbar_arrive(&c.empty_w[stw]);
          }
          it++;
          if (y >= c.Y0 && y < c.Y1 && x < c.W) {
            float* o = c.out + (c.pix0 + (size_t)y * c.W + x) * c.D;
            if (CLEAN) {
              // den == 0 exactly when the centre pixel is skipped (all-NaN): 0 * inf = NaN
              const int kb = c.k0 + kg * SL_KT;
              const float inv = 1.f / den;
#pragma unroll
              for (int q2 = 0; q2 < 2; q2++) {
                if (kb + 4 * q2 < c.D) {
                  const float2 a0 = acc[u][2 * q2], a1 = acc[u][2 * q2 + 1];
                  *reinterpret_cast<float4*>(o + kb + 4 * q2) =
                      make_float4(a0.x * inv, a0.y * inv, a1.x * inv, a1.y * inv);
                }
              }
            } else {
              const int kb = c.k0 + kg * SL_KT + 4 * pass;
#pragma unroll
              for (int q = 0; q < 4; q++) {
                const int k = kb + q;
                if (k < c.D) {
                  const float cv = c.vol[(c.pix0 + (size_t)y * c.W + x) * c.D + k];
                  o[k] = (cv != cv) ? qnan() : acc[u][q].x / acc[u][q].y;
                }
              }
            }
          }
#pragma unroll
          for (int q = 0; q < 4; q++) acc[u][q] = make_float2(0.f, 0.f);
        }
      }
    }
  }
}

template <int RHO>
__global__ void __launch_bounds__(384, 1)
    k_aggregate_slide(int H, int W, int D, float kd, float kr, const float* __restrict__ vol,
                      const uint8_t* __restrict__ guide, const uint8_t* __restrict__ nan_map,
                      float* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char sl_smem[];
  SlideCtx c;
  c.g = slide_geom(D, RHO, H);
  const SlideGeom& g = c.g;
  c.cost_s = reinterpret_cast<float*>(sl_smem + g.off_cost);
  c.w_s = reinterpret_cast<float*>(sl_smem + g.off_w);
  c.dsum_s = reinterpret_cast<float*>(sl_smem + g.off_dsum);
  c.guide_s = reinterpret_cast<float*>(sl_smem + g.off_guide);
  c.full_c = reinterpret_cast<uint64_t*>(sl_smem + g.off_bar);
  c.empty_c = c.full_c + SL_NSC;
  c.full_w = c.empty_c + SL_NSC;
  c.empty_w = c.full_w + SL_NSW;
  c.vol = vol;
  c.out = out;
  c.H = H; c.W = W; c.D = D; c.kd = kd; c.kr = kr;

  const int tid = threadIdx.x, warp = tid >> 5;
  c.lane = tid & 31;
  // warpgroups: consumers in warps [0, n_cons) (n_kg working, padded to a multiple
  // of 4), then one producer warpgroup: SL_NPROD weight warps, the stager, padding.
  const int n_cons = (g.n_kg + 3) & ~3;
  c.x0 = blockIdx.x * 32;
  c.Y0 = blockIdx.y * g.R;
  c.Y1 = min(H, c.Y0 + g.R);
  const int b = blockIdx.z / g.nslab, slab = blockIdx.z % g.nslab;
  c.k0 = slab * g.KS;
  c.ks_eff = min(g.KS, D - c.k0);
  c.pix0 = (size_t)b * H * W;
  c.NR = (c.Y1 - c.Y0) + 2 * RHO;           // input rows r = Y0 - RHO + i, i in [0, NR)

  // ---- classify the chunk ----
  // nan_map byte: bit 0 = some disparity NaN, bit 1 = some disparity finite.
  // Pixels with every disparity NaN (m == 1) and pixels outside the image are
  // exact to handle on the clean path: their taps get weight 0 (skipped) and
  // their outputs come out NaN (0 / 0).  Only a pixel with SOME NaN (m == 3)
  // needs per-disparity denominators, i.e. the (C0, V) path.
  bool clean = (nan_map != nullptr) && ((D & 3) == 0);
  if (clean) {
    int partial = 0;
    const int fw = 32 + 2 * RHO;
    for (int i = tid; i < c.NR * fw; i += blockDim.x) {
      const int yy = c.Y0 - RHO + i / fw, xx = c.x0 - RHO + i % fw;
      if (yy >= 0 && yy < H && xx >= 0 && xx < W) partial |= (nan_map[c.pix0 + (size_t)yy * W + xx] == 3);
    }
    clean = !__syncthreads_or(partial);
  }
  c.clean = clean;
  // guide rows [Y0 - 2 RHO, Y0 - 2 RHO + GR), columns [x0 - RHO, x0 + 32 + RHO);
  // NaN marks a pixel whose taps are skipped (outside the image, or all-NaN costs)
  for (int i = tid; i < g.GR * g.GC; i += blockDim.x) {
    const int yy = c.Y0 - 2 * RHO + i / g.GC, xx = c.x0 - RHO + i % g.GC;
    float gv = qnan();
    if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
      const size_t pi = c.pix0 + (size_t)yy * W + xx;
      if (nan_map == nullptr || nan_map[pi] != 1) gv = (float)guide[pi];
    }
    c.guide_s[i] = gv;
  }
  if (tid == 0) {
    for (int s = 0; s < SL_NSC; s++) {
      mbar_init(&c.full_c[s], 1);
      mbar_init(&c.empty_c[s], g.n_kg);
    }
    for (int s = 0; s < SL_NSW; s++) {
      mbar_init(&c.full_w[s], 32 * SL_NPROD);
      mbar_init(&c.empty_w[s], g.n_kg);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= n_cons) {
    // ======================= producer warpgroup =======================
    // register budget per lane-slot: the CTA holds 3 x 168 = 504 (launch bound 384);
    // producers give back to 88 so both consumer warpgroups can grow to 208.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
    const int p = warp - n_cons;
    if (p < SL_NPROD)
      slide_weights<RHO>(c, p, clean ? 1 : 2);
    else if (p == SL_NPROD)
      slide_stager<RHO>(c, clean ? 1 : 2);
  } else {
    // ======================= consumer warpgroups =======================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    if (warp < g.n_kg) {
      if (clean)
        slide_consume<RHO, true>(c, warp);
      else
        slide_consume<RHO, false>(c, warp);
    }
  }
}

template <int RHO>
static cudaError_t slide_launch_t(int B, int H, int W, int D, float gamma_d, float gamma_r,
                                  const float* vol, const uint8_t* guide, const uint8_t* nan_map,
                                  float* out, cudaStream_t st) {
  const SlideGeom g = slide_geom(D, RHO, H);
  auto kern = k_aggregate_slide<RHO>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.bytes);
  if (e != cudaSuccess) { cudaGetLastError(); return e; }
  const float log2e = 1.4426950408889634f;
  const float kd = -log2e / (gamma_d * gamma_d);
  const float kr = std::isinf(gamma_r) ? -1e-30f : -log2e / (gamma_r * gamma_r);
  dim3 grid((W + 31) / 32, (H + g.R - 1) / g.R, B * g.nslab);
  kern<<<grid, 32 * (((g.n_kg + 3) & ~3) + 4), g.bytes, st>>>(H, W, D, kd, kr, vol, guide, nan_map, out);
  return cudaGetLastError();
}

size_t aggregate_slide_smem(int D, int rho, int H) { return slide_geom(D, rho, H).bytes; }

cudaError_t launch_aggregate_slide(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r,
                                   const float* vol, const uint8_t* guide, const uint8_t* nan_map,
                                   float* out, cudaStream_t st) {
#define RSR_S(R) \
  case R: return slide_launch_t<R>(B, H, W, D, gamma_d, gamma_r, vol, guide, nan_map, out, st);
  switch (rho) {
    RSR_S(0) RSR_S(1) RSR_S(2) RSR_S(3) RSR_S(4) RSR_S(5) RSR_S(6) RSR_S(7)
    default:
      return cudaErrorInvalidValue;
  }
#undef RSR_S
}

}  // namespace rsr
