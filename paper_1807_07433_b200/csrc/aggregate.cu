// K3 — bilateral cost aggregation (fast bilateral stereo), PAPER.md:128-152,
// Eq. (8) with the weights of Eqs. (9)-(10):
//   A(u,v,k) = sum_t w_t C(u+dx, v+dy, k) / sum_t w_t,
//   w_t = exp(-(dx^2+dy^2)/gamma_d^2) * exp(-(g(u+dx,v+dy) - g(u,v))^2/gamma_r^2),
// taps outside the image or with a NaN cost skipped, NaN iff the centre is NaN
// (readings 10-12).  This is the step the paper names as the cost
// (P:154); it is FP32-FMA bound: 2 * 169 flop per output at
// rho = 6.
//
// Design (sm_100a, CUDA cores):
//  * Volume layout [B][H][W][D]: a cost row segment is contiguous, so each of
//    the (TX + 2 rho) pixel columns of an input row arrives as one bulk async
//    copy (cp.async.bulk, TMA engine) into a padded shared-memory row
//    [x][D + 4] (conflict-free 16-byte loads), 3-stage mbarrier pipeline.
//  * Thread = one pixel column x (lanes along x) x PY = 8 output rows x 16
//    disparities held as 8 packed pairs; the inner product is FFMA2 with the
//    tap weight as scalar broadcast operand (fma.rn.f32x2), so one issue slot
//    feeds two FMAs.  Per input row the thread loads the (2 rho + 1) cost
//    columns once (4 x LDS.128 each) and reuses them for all 8 rows; weights
//    are staged per input row as [x][tap][row] so 8 rows' weights of a tap
//    are two LDS.128 reused across 16 disparities.
//  * Weights are computed once per (pixel, tap) per CTA (exp2 on the MUFU
//    pipe) and shared by all disparity groups; sum_t w_t is per pixel, not per
//    disparity, on clean tiles.
//  * Clean tiles (footprint inside the image, no NaN per nan_map) take the
//    pair = (k, k+1) fast path.  Other tiles take the exact general path:
//    pair = (C0, V) with C0 = cost or 0, V = validity, so the same FFMA2 loop
//    accumulates numerator and per-disparity denominator; two passes cover
//    the 16 disparities.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int AG_KT = 16;     // disparities per thread
constexpr int AG_PY = 8;      // output rows per thread
constexpr int AG_NST = 3;     // cost row stages

struct AggGeom {
  int n_kg, n_cw, TX, KS, DPAD, CX, WST, GR, GC, nslab;
  size_t off_cost, off_w, off_guide, off_dpart, off_bar, bytes;
};

__host__ __device__ inline AggGeom agg_geom_cw(int D, int rho, int n_cw) {
  AggGeom g;
  const int ks = D < 128 ? D : 128;
  g.n_kg = (ks + AG_KT - 1) / AG_KT;
  g.n_cw = n_cw;
  g.TX = 32 * g.n_cw;
  g.KS = g.n_kg * AG_KT;
  g.DPAD = g.KS + 4;
  g.CX = g.TX + 2 * rho;
  g.WST = (2 * rho + 1) * AG_PY + 4;
  g.GR = AG_PY + 2 * rho;
  g.GC = g.TX + 2 * rho;
  g.nslab = (D + g.KS - 1) / g.KS;
  size_t o = 0;
  g.off_cost = o; o += sizeof(float) * (size_t)AG_NST * g.CX * g.DPAD;
  g.off_w = o;    o += sizeof(float) * (size_t)2 * g.TX * g.WST;
  g.off_guide = o; o += sizeof(float) * (size_t)g.GR * g.GC;
  g.off_dpart = o; o += sizeof(float) * (size_t)g.n_kg * AG_PY * g.TX;
  o = (o + 15) & ~size_t(15);
  g.off_bar = o;  o += 8 * AG_NST + 16;
  g.bytes = o;
  return g;
}

// Column warps per CTA: up to 4 (8 warps with the disparity groups), fewer where the
// weight stage of a wide window would not fit the 227 KB of shared memory (rho 9-10).
__host__ __device__ inline AggGeom agg_geom(int D, int rho) {
  const int ks = D < 128 ? D : 128;
  const int n_kg = (ks + AG_KT - 1) / AG_KT;
  int n_cw = 8 / n_kg;
  if (n_cw > 4) n_cw = 4;
  if (n_cw < 1) n_cw = 1;
  AggGeom g = agg_geom_cw(D, rho, n_cw);
  while (g.bytes > 227 * 1024 && n_cw > 1) g = agg_geom_cw(D, rho, --n_cw);
  return g;
}

template <int RHO>
__global__ void __launch_bounds__(256, 1)
    k_aggregate(int H, int W, int D, float kd, float kr, const float* __restrict__ vol,
                const uint8_t* __restrict__ guide, const uint8_t* __restrict__ nan_map,
                float* __restrict__ out) {
  constexpr int NT = 2 * RHO + 1;          // taps per row
  constexpr int NRIN = AG_PY + 2 * RHO;    // input rows per tile
  const AggGeom g = agg_geom(D, RHO);
  extern __shared__ __align__(16) unsigned char ag_smem[];
  float* cost_s = reinterpret_cast<float*>(ag_smem + g.off_cost);
  float* w_s = reinterpret_cast<float*>(ag_smem + g.off_w);
  float* guide_s = reinterpret_cast<float*>(ag_smem + g.off_guide);
  float* dpart_s = reinterpret_cast<float*>(ag_smem + g.off_dpart);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ag_smem + g.off_bar);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kg = warp % g.n_kg, cw = warp / g.n_kg;
  const int xl = 32 * cw + lane;                // this thread's column in the tile
  const int x0 = blockIdx.x * g.TX, y0 = blockIdx.y * AG_PY;
  const int b = blockIdx.z / g.nslab, slab = blockIdx.z % g.nslab;
  const int k0 = slab * g.KS;                   // first disparity of the slab
  const int ks_eff = min(g.KS, D - k0);
  const size_t pix0 = (size_t)b * H * W;

  // ---- weight-compute role: fixed column xw, tap subset js ----
  const int xw = tid % g.TX, js = tid / g.TX;   // js in [0, n_kg)

  // ---- classify the tile ----
  bool clean = (nan_map != nullptr) && ((D & 3) == 0) && (y0 - RHO >= 0) &&
               (y0 + AG_PY + RHO <= H) && (x0 - RHO >= 0) && (x0 + g.TX + RHO <= W);
  if (clean) {
    int dirty = 0;
    const int fw = g.TX + 2 * RHO;
    for (int i = tid; i < NRIN * fw; i += blockDim.x) {
      const int yy = y0 - RHO + i / fw, xx = x0 - RHO + i % fw;
      dirty |= nan_map[pix0 + (size_t)yy * W + xx] & 1;
    }
    clean = !__syncthreads_or(dirty);
  }

  // ---- guide tile (float), centre values for the weight role ----
  for (int i = tid; i < g.GR * g.GC; i += blockDim.x) {
    const int yy = y0 - RHO + i / g.GC, xx = x0 - RHO + i % g.GC;
    guide_s[i] = (yy >= 0 && yy < H && xx >= 0 && xx < W)
                     ? (float)guide[pix0 + (size_t)yy * W + xx] : 0.f;
  }
  if (tid == 0) {
    for (int s = 0; s < AG_NST; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  float gc[AG_PY];
#pragma unroll
  for (int py = 0; py < AG_PY; py++) gc[py] = guide_s[(RHO + py) * g.GC + xw + RHO];

  // bulk copy of input row ir (image row y0 - RHO + ir) into stage ir % 3
  auto issue_row = [&](int ir) {
    if (warp == 0) {
      const int st = ir % AG_NST;
      const int yy = y0 - RHO + ir;
      const uint32_t bytes_col = (uint32_t)ks_eff * 4u;
      if (lane == 0) mbar_arrive_expect_tx(&bars[st], bytes_col * (uint32_t)g.CX);
      __syncwarp();
      const float* src = vol + ((pix0 + (size_t)yy * W + (x0 - RHO)) * D + k0);
      float* dst = cost_s + (size_t)st * g.CX * g.DPAD;
      for (int c = lane; c < g.CX; c += 32)
        bulk_g2s(dst + c * g.DPAD, src + (size_t)c * D, bytes_col, &bars[st]);
    }
  };
  // general-path staging: (C0, V) pairs for disparities k0 + kgi*16 + 8*pass + i
  auto stage_row_general = [&](int ir, int pass) {
    const int st = ir % AG_NST;
    const int yy = y0 - RHO + ir;
    float* dst = cost_s + (size_t)st * g.CX * g.DPAD;
    const int items = g.CX * g.n_kg * 8;
    for (int it = tid; it < items; it += blockDim.x) {
      const int i = it & 7, kgi = (it >> 3) % g.n_kg, c = (it >> 3) / g.n_kg;
      const int k = k0 + kgi * AG_KT + 8 * pass + i;
      const int xx = x0 - RHO + c;
      float v = qnan();
      if (k < D && yy >= 0 && yy < H && xx >= 0 && xx < W)
        v = vol[(pix0 + (size_t)yy * W + xx) * D + k];
      const bool ok = !(v != v);
      *reinterpret_cast<float2*>(dst + c * g.DPAD + kgi * AG_KT + 2 * i) =
          make_float2(ok ? v : 0.f, ok ? 1.f : 0.f);
    }
  };
  // weights of input row ir for pixel column xw, taps js, js + n_kg, ...:
  //   w[xw][tap][py] = exp2(kd*(dx^2+dy^2) + kr*(g(x+dx, r) - g(x, y0+py))^2)
  // (kd = -log2(e)/gamma_d^2, kr = -log2(e)/gamma_r^2), 0 for rows py whose
  // window does not contain input row r.
  float dsum[AG_PY];
#pragma unroll
  for (int py = 0; py < AG_PY; py++) dsum[py] = 0.f;
  auto compute_weights = [&](int ir) {
    float* dst = w_s + (size_t)(ir & 1) * g.TX * g.WST + xw * g.WST;
    const float* grow = guide_s + ir * g.GC + xw;   // guide row r, column x0 - RHO + xw
    for (int j = js; j < NT; j += g.n_kg) {
      const float gq = grow[j];
      const float fdx = (float)(j - RHO);
      float wv[AG_PY];
#pragma unroll
      for (int py = 0; py < AG_PY; py++) {
        const int dy = ir - RHO - py;
        const float fdy = (float)dy;
        const float dg = gq - gc[py];
        const float a = fmaf(dg * dg, kr, (fdx * fdx + fdy * fdy) * kd);
        const float w = (dy >= -RHO && dy <= RHO) ? ex2_approx(a) : 0.f;
        wv[py] = w;
        dsum[py] += w;
      }
      float4* d4 = reinterpret_cast<float4*>(dst + j * AG_PY);
      d4[0] = make_float4(wv[0], wv[1], wv[2], wv[3]);
      d4[1] = make_float4(wv[4], wv[5], wv[6], wv[7]);
    }
  };

  const int npass = clean ? 1 : 2;
  for (int pass = 0; pass < npass; pass++) {
    float2 acc[AG_PY][AG_KT / 2];
#pragma unroll
    for (int py = 0; py < AG_PY; py++)
#pragma unroll
      for (int q = 0; q < AG_KT / 2; q++) acc[py][q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int py = 0; py < AG_PY; py++) dsum[py] = 0.f;

    // prologue
    if (clean) {
      for (int ir = 0; ir < AG_NST && ir < NRIN; ir++) issue_row(ir);
    } else {
      stage_row_general(0, pass);
    }
    compute_weights(0);
    __syncthreads();

    for (int ir = 0; ir < NRIN; ir++) {
      const int st = ir % AG_NST;
      if (clean) mbar_wait_parity(&bars[st], (uint32_t)((ir / AG_NST) & 1));
      // rows py whose window holds input row ir: dy = ir - RHO - py in [-RHO, RHO]
      const int pa = max(0, ir - 2 * RHO), pb = min(AG_PY - 1, ir);
      const float* crow = cost_s + (size_t)st * g.CX * g.DPAD + xl * g.DPAD + kg * AG_KT;
      const float* wrow = w_s + (size_t)(ir & 1) * g.TX * g.WST + xl * g.WST;
#pragma unroll
      for (int j = 0; j < NT; j++) {
        const float4* c4 = reinterpret_cast<const float4*>(crow + j * g.DPAD);
        const float4 ca = c4[0], cb = c4[1], cc = c4[2], cd = c4[3];
        const float2 cp[8] = {make_float2(ca.x, ca.y), make_float2(ca.z, ca.w),
                              make_float2(cb.x, cb.y), make_float2(cb.z, cb.w),
                              make_float2(cc.x, cc.y), make_float2(cc.z, cc.w),
                              make_float2(cd.x, cd.y), make_float2(cd.z, cd.w)};
        const float4* w4 = reinterpret_cast<const float4*>(wrow + j * AG_PY);
        const float4 wa = w4[0], wb = w4[1];
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
        for (int py = 0; py < AG_PY; py++) {
          if (py >= pa && py <= pb) {
#pragma unroll
            for (int q = 0; q < 8; q++) ffma2_bcast(acc[py][q], wv[py], cp[q]);
          }
        }
      }
      // next row: weights into the other buffer, general-path staging
      if (ir + 1 < NRIN) {
        compute_weights(ir + 1);
        if (!clean) stage_row_general(ir + 1, pass);
      }
      __syncthreads();
      if (clean && ir + AG_NST < NRIN) issue_row(ir + AG_NST);
    }

    // ---- epilogue ----
#pragma unroll
    for (int py = 0; py < AG_PY; py++) dpart_s[(js * AG_PY + py) * g.TX + xw] = dsum[py];
    __syncthreads();
    const int x = x0 + xl;
#pragma unroll
    for (int py = 0; py < AG_PY; py++) {
      const int y = y0 + py;
      if (x >= W || y >= H) continue;
      float* o = out + (pix0 + (size_t)y * W + x) * D;
      if (clean) {
        float den = 0.f;
        for (int s2 = 0; s2 < g.n_kg; s2++) den += dpart_s[(s2 * AG_PY + py) * g.TX + xl];
        const float inv = 1.f / den;
        const int kb = k0 + kg * AG_KT;
#pragma unroll
        for (int q4 = 0; q4 < 4; q4++) {
          if (kb + 4 * q4 < D) {
            const float2 p0 = acc[py][2 * q4], p1 = acc[py][2 * q4 + 1];
            *reinterpret_cast<float4*>(o + kb + 4 * q4) =
                make_float4(p0.x * inv, p0.y * inv, p1.x * inv, p1.y * inv);
          }
        }
      } else {
        const int kb = k0 + kg * AG_KT + 8 * pass;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const int k = kb + q;
          if (k < D) {
            const float cv = vol[(pix0 + (size_t)y * W + x) * D + k];
            o[k] = (cv != cv) ? qnan() : acc[py][q].x / acc[py][q].y;
          }
        }
      }
    }
    __syncthreads();
  }
}

template <int RHO>
static cudaError_t aggregate_launch_t(int B, int H, int W, int D, float gamma_d, float gamma_r,
                                      const float* vol, const uint8_t* guide,
                                      const uint8_t* nan_map, float* out, cudaStream_t st) {
  const AggGeom g = agg_geom(D, RHO);
  auto kern = k_aggregate<RHO>;
  cudaError_t e = smem_optin((const void*)kern, g.bytes);
  if (e != cudaSuccess) return e;
  const float log2e = 1.4426950408889634f;
  const float kd = -log2e / (gamma_d * gamma_d);
  const float kr = std::isinf(gamma_r) ? 0.f : -log2e / (gamma_r * gamma_r);
  dim3 grid((W + g.TX - 1) / g.TX, (H + AG_PY - 1) / AG_PY, B * g.nslab);
  kern<<<grid, 32 * g.n_kg * g.n_cw, g.bytes, st>>>(H, W, D, kd, kr, vol, guide, nan_map, out);
  return cudaGetLastError();
}

size_t aggregate_tiled_smem(int D, int rho) { return agg_geom(D, rho).bytes; }

cudaError_t launch_aggregate(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                             const float* vol, const uint8_t* guide, const uint8_t* nan_map,
                             float* out, cudaStream_t st) {
  if (aggregate_small_applies(D, rho))
    return launch_aggregate_small(B, H, W, D, rho, gamma_d, gamma_r, conc, vol, guide, nan_map, out, st);
  if (rho <= 7)
    return launch_aggregate_slide(B, H, W, D, rho, gamma_d, gamma_r, conc, vol, guide, nan_map, out, st);
#define RSR_A(R) \
  case R: return aggregate_launch_t<R>(B, H, W, D, gamma_d, gamma_r, vol, guide, nan_map, out, st);
  switch (rho) {
    RSR_A(8) RSR_A(9) RSR_A(10)
    default:
      return cudaErrorInvalidValue;
  }
#undef RSR_A
}

}  // namespace rsr
