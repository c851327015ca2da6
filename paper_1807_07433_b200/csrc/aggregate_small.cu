// K3s — bilateral cost aggregation (Eq. (8) with Eqs. (9)-(10))
// for SMALL disparity slabs (D <= 16, run as slabs of 8): the restricted search
// range of P:251 ("reduce the search range and only perform the bilateral
// filtering on the space around the calculated disparities") and tiny ranges.
//
// At D = 8 a bilateral weight w(p, q) feeds only 8 FMAs, so the producer/consumer
// kernel (aggregate_slide.cu: 4 weight-producer warps, 1 consumer warp, weights
// handed over through shared memory) is bound by weight production and runs one
// FFMA2 warp per CTA (measured 15 % of FP32 at D = 8).  Here every thread owns one
// output column x and all 8 disparities of the slab and computes its own weights:
//   w(a, j) = S(a, j) * R(g(x + j - rho, y_in) - g(x, y_a))
// with the spatial factors S in a broadcast shared table and the range factor R
// in a shared table replicated per lane (lut[idx][lane]: every warp-wide lookup is
// one conflict-free wavefront).  The strip slides down one input row at a time;
// a thread keeps the 2 rho + 1 output rows ("ages") whose windows contain the
// input row (13 x 4 packed pairs at rho = 6), so each staged cost feeds 2 rho + 1
// FFMA2s, exactly as in aggregate_slide.cu.
//
// Arithmetic is that of aggregate_slide.cu operation for operation: the same
// factors (ex2 of the same arguments), w = S * R, numerators fma(w, c, acc) and
// denominators (the running sum of w, clean segments; fma(w, validity, acc),
// general segments) in (input row, tap) order, and the same epilogues
// (num * rcp(den)).  Results are therefore bitwise identical to that kernel's,
// whichever segment / path a pixel falls in (tests/test_gpu_parity.py).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int SM_TX = 128;            // output columns per CTA (one per thread)
constexpr int SM_KD = 8;              // disparities per slab
constexpr int SM_LUT = 512;           // range table entries per lane: dg + 255 in [0, 510], 511 = 0
constexpr int SM_SKIPQ = 4096;        // guide code of a skipped tap pixel (clamps to the zero entry)
constexpr int SM_SKIPP = -4096;       // guide code of a skipped centre pixel

struct SmallArgs {
  int B, H, W, D, R, nslab;
  float kd, kr;
  const float* vol;
  const uint8_t* guide;
  const uint8_t* nan_map;
  float* out;
};

// SPLIT: two threads per output column (lanes 2c, 2c + 1), the lower holding ages
// 0 .. RHO and the upper ages RHO + 1 .. 2 RHO (+ one always-zero dummy age), so a
// thread keeps half the accumulators (~128 registers, four CTAs of 64 columns per SM
// instead of two of 128: twice the warps to hide the latencies that bound the
// one-thread-per-column kernel).  The age that crosses from the upper to the lower
// half at the end of each input row moves by one lane shuffle (exact copies): every
// accumulation stays in (input row, tap) order, bitwise as before.
template <int RHO, bool SPLIT>
struct SmallGeom {
  static constexpr int NT = 2 * RHO + 1;
  static constexpr int TXC = SPLIT ? 64 : SM_TX;   // output columns per CTA
  static constexpr int CX = TXC + 2 * RHO;         // staged columns per input row
  static constexpr int NA = SPLIT ? RHO + 1 : NT;  // ages per thread
  static constexpr int REP = SPLIT ? 16 : 32;      // range-table copies (lane & (REP - 1))
  static constexpr int STW = SPLIT ? 16 : (NT <= 16 ? 16 : 32);   // spatial table row stride
  // shared memory (bytes): lut | S | 2 cost rows [CX][8] | 2 guide rows [CX] (int)
  static constexpr size_t off_lut = 0;
  static constexpr size_t off_s = off_lut + sizeof(float) * SM_LUT * REP;
  static constexpr size_t off_cost = off_s + sizeof(float) * NT * STW;
  static constexpr size_t off_guide = off_cost + sizeof(float) * 2 * CX * SM_KD;
  static constexpr size_t bytes = off_guide + sizeof(int) * 2 * CX;
};

template <int RHO, bool SPLIT>
__global__ void __launch_bounds__(SM_TX, SPLIT ? 4 : 2) k_aggregate_small(const SmallArgs A) {
  using G = SmallGeom<RHO, SPLIT>;
  constexpr int NT = G::NT, CX = G::CX, NA = G::NA, TXC = G::TXC, REP = G::REP;
  extern __shared__ __align__(16) unsigned char sm_smem[];
  float* lut = reinterpret_cast<float*>(sm_smem + G::off_lut);
  float* S = reinterpret_cast<float*>(sm_smem + G::off_s);
  float* cost = reinterpret_cast<float*>(sm_smem + G::off_cost);
  int* grow = reinterpret_cast<int*>(sm_smem + G::off_guide);
  const int tid = threadIdx.x, lane = tid & 31;

  // ---- segment: 128 columns x R rows of frame b, disparity slab ----
  const int nstrip = (A.W + TXC - 1) / TXC;
  const int nchunk = (A.H + A.R - 1) / A.R;
  int blk = blockIdx.x;
  const int strip = blk % nstrip;
  blk /= nstrip;
  const int chunk = blk % nchunk;
  blk /= nchunk;
  const int slab = blk % A.nslab, b = blk / A.nslab;
  const int x0 = strip * TXC, ya = chunk * A.R, yb = min(A.H, ya + A.R);
  const int k0 = slab * SM_KD, ks_eff = min(SM_KD, A.D - k0);
  const size_t pix0 = (size_t)b * A.H * A.W;
  const int tc = SPLIT ? tid >> 1 : tid;            // the thread's column in the strip
  const int hf = SPLIT ? (tid & 1) : 0;             // SPLIT: lower (0) / upper (1) ages
  const int x = x0 + tc;

  // ---- tables: range factor exp2(kr dg^2) per lane, spatial factor exp2(kd (dx^2 + dy^2)) ----
  for (int e = tid; e < SM_LUT * REP; e += SM_TX) {
    const int dg = e / REP - 255;
    lut[e] = (dg <= 255) ? ex2_ftz((float)(dg * dg) * A.kr) : 0.f;
  }
  // S[j][a]: tap j (dx = j - RHO), age a = output row y_in - RHO + a (dy = RHO - a);
  // ages contiguous so four of them are one broadcast LDS.128.  SPLIT: [j][half][8],
  // half 1 starting at age RHO + 1 (its dummy age and padding: 0)
  for (int e = tid; e < NT * G::STW; e += SM_TX) {
    const int j = e / G::STW, r = e % G::STW;
    const int a = SPLIT ? (r >= 8 ? RHO + 1 + (r - 8) : (r < RHO + 1 ? r : NT)) : r;
    S[e] = a < NT ? ex2_ftz((float)((j - RHO) * (j - RHO) + (RHO - a) * (RHO - a)) * A.kd) : 0.f;
  }

  // ---- classify: a partially-NaN pixel anywhere in the footprint -> general path ----
  int partial = A.nan_map == nullptr ? 1 : 0;
  if (!partial) {
    const int fw = CX, fh = (yb - ya) + 2 * RHO;
    constexpr int UNR = 8;   // independent loads in flight per thread
    for (int e0 = tid; e0 < fw * fh; e0 += UNR * SM_TX) {
      int m[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int e = e0 + u * SM_TX;
        const int yy = ya - RHO + e / fw, xx = x0 - RHO + e % fw;
        m[u] = (e < fw * fh && yy >= 0 && yy < A.H && xx >= 0 && xx < A.W)
                   ? (int)__ldg(A.nan_map + pix0 + (size_t)yy * A.W + xx) : 0;
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) partial |= (m[u] & 3) == 3;
    }
  }
  const bool clean = !__syncthreads_or(partial);

  const int NR = (yb - ya) + 2 * RHO;   // input rows ya - RHO .. yb + RHO - 1
  // the row loop, specialised on the path (clean / general) so each instantiation
  // holds only its own registers
  auto run = [&](auto clean_tag) {
    constexpr bool CLEAN = decltype(clean_tag)::value;
  const int npass = CLEAN ? 1 : 2;
  for (int pass = 0; pass < npass; pass++) {
    // staged values per column: clean: costs k0..k0+7 (NaN-free: skipped pixels and
    // k >= D give 0); general pass h: (C0, V) pairs of k0 + 4h .. k0 + 4h + 3
    // Row staging without data-dependent control flow before the math: every load of
    // row i + 1 (nan_map byte, guide, costs) is issued unconditionally (in-image
    // predicate only) at the start of row i and resolved (skip -> weight 0, cost 0)
    // when committed after the math, so the global-load latency hides behind the row.
    auto fetch_row = [&](int i, float (&v)[2][SM_KD], int (&gv)[2], int (&nm)[2]) {
      const int yy = ya - RHO + i;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = tid + h * SM_TX;
        const int xx = x0 - RHO + c;
        const bool in = c < CX && yy >= 0 && yy < A.H && xx >= 0 && xx < A.W;
        const size_t g = pix0 + (size_t)yy * A.W + xx;
        nm[h] = in ? (A.nan_map ? (int)A.nan_map[g] : 2) : 1;
        gv[h] = in ? (int)A.guide[g] : 0;
        const float* src = A.vol + g * A.D + k0;
        if (CLEAN && ks_eff == SM_KD && (A.D & 3) == 0) {
          float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = t0;
          if (in) {
            t0 = __ldg(reinterpret_cast<const float4*>(src));
            t1 = __ldg(reinterpret_cast<const float4*>(src + 4));
          }
          v[h][0] = t0.x; v[h][1] = t0.y; v[h][2] = t0.z; v[h][3] = t0.w;
          v[h][4] = t1.x; v[h][5] = t1.y; v[h][6] = t1.z; v[h][7] = t1.w;
        } else if (CLEAN) {
#pragma unroll
          for (int q = 0; q < SM_KD; q++) v[h][q] = (in && q < ks_eff) ? __ldg(src + q) : 0.f;
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int k = 4 * pass + q;
            v[h][q] = (in && k < ks_eff) ? __ldg(src + k) : qnan();
          }
        }
      }
    };
    auto commit_row = [&](int i, const float (&v)[2][SM_KD], const int (&gv)[2], const int (&nm)[2]) {
      const int st = i & 1;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = tid + h * SM_TX;
        if (c >= CX) continue;
        const bool skip = (nm[h] & 3) == 1;      // outside the image or every k NaN
        float o[SM_KD];
        if (CLEAN) {
#pragma unroll
          for (int q = 0; q < SM_KD; q++) o[q] = skip ? 0.f : v[h][q];
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float cv = v[h][q];
            const bool ok = !skip && !(cv != cv);
            o[2 * q] = ok ? cv : 0.f;
            o[2 * q + 1] = ok ? 1.f : 0.f;
          }
        }
        float4* d = reinterpret_cast<float4*>(cost + ((size_t)st * CX + c) * SM_KD);
        RSR_CHECK(st < 2 && c < CX);
        d[0] = make_float4(o[0], o[1], o[2], o[3]);
        d[1] = make_float4(o[4], o[5], o[6], o[7]);
        grow[st * CX + c] = skip ? SM_SKIPQ : gv[h];
      }
    };
    // centre guide code (skipped centre: SM_SKIPP) with unconditional loads
    auto centre_code = [&](int yy) {
      const bool in = yy >= 0 && yy < A.H && x < A.W;
      const size_t g = pix0 + (size_t)yy * A.W + x;
      const int nmv = in ? (A.nan_map ? (int)A.nan_map[g] : 2) : 1;
      const int gv = in ? (int)A.guide[g] : 0;
      return (nmv & 3) == 1 ? SM_SKIPP : gv;
    };

    float2 acc[NA][4];
    float den[NA];
    int gp[NA];   // guide code of the output row of each of the thread's ages (its centre pixel)
    const int abase = SPLIT && hf ? RHO + 1 : 0;   // global age of local age 0
#pragma unroll
    for (int a = 0; a < NA; a++) {
#pragma unroll
      for (int q = 0; q < 4; q++) acc[a][q] = make_float2(0.f, 0.f);
      den[a] = 0.f;
      gp[a] = centre_code(ya - 2 * RHO + abase + a);   // age at input row 0: output row ya - 2 rho + age
    }
    // clean rows of a whole 8-disparity slab (16-byte aligned): costs staged by cp.async
    // straight into shared memory (skipped pixels zeroed at commit); the nan_map byte and
    // the guide go through registers
    const bool async_rows = CLEAN && ks_eff == SM_KD && (A.D & 3) == 0;
    auto stage_async = [&](int i, int (&gv)[2], int (&nm)[2]) {
      const int yy = ya - RHO + i;
      const int st = i & 1;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = tid + h * SM_TX;
        const int xx = x0 - RHO + c;
        const bool in = c < CX && yy >= 0 && yy < A.H && xx >= 0 && xx < A.W;
        const size_t g = pix0 + (size_t)yy * A.W + xx;
        nm[h] = in ? (A.nan_map ? (int)A.nan_map[g] : 2) : 1;
        gv[h] = in ? (int)A.guide[g] : 0;
        if (in) {
          float* d = cost + ((size_t)st * CX + c) * SM_KD;
          const float* src = A.vol + g * A.D + k0;
          cp_async16(d, src);
          cp_async16(d + 4, src + 4);
        }
      }
      cp_async_commit();
    };
    auto commit_async = [&](int i, const int (&gv)[2], const int (&nm)[2]) {
      cp_async_wait_all();
      const int st = i & 1;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = tid + h * SM_TX;
        if (c >= CX) continue;
        const bool skip = (nm[h] & 3) == 1;
        if (skip) {
          float4* d = reinterpret_cast<float4*>(cost + ((size_t)st * CX + c) * SM_KD);
          d[0] = make_float4(0.f, 0.f, 0.f, 0.f);
          d[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        grow[st * CX + c] = skip ? SM_SKIPQ : gv[h];
      }
    };
    float pv[2][SM_KD];
    int pg[2], pn[2];
    if (async_rows) {
      stage_async(0, pg, pn);
      commit_async(0, pg, pn);
    } else {
      fetch_row(0, pv, pg, pn);
      commit_row(0, pv, pg, pn);
    }
    __syncthreads();
    for (int i = 0; i < NR; i++) {
      // the next row lands in the other stage (last read in iteration i - 1) during the math
      if (i + 1 < NR) {
        if (async_rows) stage_async(i + 1, pg, pn);
        else fetch_row(i + 1, pv, pg, pn);
      }
      // centre guide code of the output row entering at the end of this row: loaded now,
      // consumed after the math (its global-load latency hidden behind the row)
      const int gp_next = centre_code(ya - 2 * RHO + i + NT);
      const int st = i & 1;
      const float* crow = cost + ((size_t)st * CX + tc) * SM_KD;
      const int* gr = grow + st * CX + tc;
      float2 fin[4];
      float fden = 0.f;
#pragma unroll
      for (int j = 0; j < NT; j++) {
        const float4 ca = *reinterpret_cast<const float4*>(crow + j * SM_KD);
        const float4 cb = *reinterpret_cast<const float4*>(crow + j * SM_KD + 4);
        const float2 cp[4] = {make_float2(ca.x, ca.y), make_float2(ca.z, ca.w), make_float2(cb.x, cb.y),
                              make_float2(cb.z, cb.w)};
        const int gq = gr[j];
#pragma unroll
        for (int a4 = 0; a4 < (NA + 3) / 4; a4++) {
          const float4 s4 =
              *reinterpret_cast<const float4*>(S + j * G::STW + (SPLIT ? 8 * hf : 0) + 4 * a4);   // broadcast
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const int a = 4 * a4 + t;
            if (a < NA) {
              const int idx = min(gq - gp[a] + 255, SM_LUT - 1);
              RSR_CHECK(idx >= 0 && tc + j < CX);
              const float w = sv[t] * lut[idx * REP + (lane & (REP - 1))];
              if (j < NT - 1) {
                if (CLEAN) den[a] += w;
#pragma unroll
                for (int q = 0; q < 4; q++) acc[a][q] = f2fma(make_float2(w, w), cp[q], acc[a][q]);
              } else if (a == 0) {
                // last tap of the row: age 0 completes, every other age moves one slot down
                if (CLEAN) fden = den[0] + w;
#pragma unroll
                for (int q = 0; q < 4; q++) fin[q] = f2fma(make_float2(w, w), cp[q], acc[0][q]);
              } else {
                if (CLEAN) den[a - 1] = den[a] + w;
#pragma unroll
                for (int q = 0; q < 4; q++) acc[a - 1][q] = f2fma(make_float2(w, w), cp[q], acc[a][q]);
              }
            }
          }
        }
      }
      if (SPLIT) {
        // the upper half's oldest age (just folded into its fin) becomes the lower half's
        // newest; the upper half's newest real age starts empty (its dummy age is zero)
        float2 up[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          up[q].x = __shfl_xor_sync(0xffffffffu, fin[q].x, 1);
          up[q].y = __shfl_xor_sync(0xffffffffu, fin[q].y, 1);
        }
        const float upd = __shfl_xor_sync(0xffffffffu, fden, 1);
#pragma unroll
        for (int q = 0; q < 4; q++) acc[NA - 1][q] = hf ? make_float2(0.f, 0.f) : up[q];
        den[NA - 1] = hf ? 0.f : (CLEAN ? upd : 0.f);
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++) acc[NT - 1][q] = make_float2(0.f, 0.f);
        den[NT - 1] = 0.f;
      }
      // the output row of age 0 completes at input row i
      const int y = ya - 2 * RHO + i;
      if (hf == 0 && y >= ya && x < A.W) {
        float* o = A.out + (pix0 + (size_t)y * A.W + x) * A.D + k0;
        RSR_CHECK(y < A.H && x < A.W && k0 + ks_eff <= A.D);
        if (CLEAN) {
          const float inv = rcp_fast(fden);   // fden == 0 exactly for a skipped centre: NaN
          const float r[8] = {fin[0].x * inv, fin[0].y * inv, fin[1].x * inv, fin[1].y * inv,
                              fin[2].x * inv, fin[2].y * inv, fin[3].x * inv, fin[3].y * inv};
          if (ks_eff == SM_KD && (A.D & 3) == 0) {
            reinterpret_cast<float4*>(o)[0] = make_float4(r[0], r[1], r[2], r[3]);
            reinterpret_cast<float4*>(o)[1] = make_float4(r[4], r[5], r[6], r[7]);
          } else {
#pragma unroll
            for (int q = 0; q < SM_KD; q++)
              if (q < ks_eff) o[q] = r[q];
          }
        } else {
          const float* cv = A.vol + (pix0 + (size_t)y * A.W + x) * A.D + k0;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int k = 4 * pass + q;
            if (k < ks_eff) {
              const float c = __ldg(cv + k);
              o[k] = (c != c) ? qnan() : fin[q].x * rcp_fast(fin[q].y);
            }
          }
        }
      }
      if (SPLIT) {
        const int gup = __shfl_xor_sync(0xffffffffu, gp[0], 1);   // upper half's oldest
#pragma unroll
        for (int a = 0; a + 1 < NA; a++) gp[a] = gp[a + 1];
        if (hf) {
          gp[NA - 1] = gp_next;
          if (NA >= 2) gp[NA - 2] = gp_next;                      // the entering age 2 rho
        } else {
          gp[NA - 1] = gup;
        }
      } else {
#pragma unroll
        for (int a = 0; a + 1 < NT; a++) gp[a] = gp[a + 1];
        gp[NT - 1] = gp_next;
      }
      if (i + 1 < NR) {
        if (async_rows) commit_async(i + 1, pg, pn);
        else commit_row(i + 1, pv, pg, pn);
      }
      __syncthreads();
    }
  }
  };
  if (clean) run(std::true_type());
  else run(std::false_type());
}

static int small_sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

bool aggregate_small_applies(int D, int rho) {
  if (D > 2 * SM_KD || rho > 7) return false;
  const char* e = getenv("RSR_K3_SMALL");   // experiment hook (tools/, tests): 0 disables
  return !(e && e[0] == '0');
}

template <int RHO, bool SPLIT>
static cudaError_t small_launch_t(int B, int H, int W, int D, float gamma_d, float gamma_r, int conc,
                                  const float* vol, const uint8_t* guide, const uint8_t* nan_map, float* out,
                                  cudaStream_t st) {
  using G = SmallGeom<RHO, SPLIT>;
  SmallArgs A;
  A.B = B; A.H = H; A.W = W; A.D = D;
  A.nslab = (D + SM_KD - 1) / SM_KD;
  const int nstrip = (W + G::TXC - 1) / G::TXC;
  // rows per CTA: minimise waves x (R + 2 rho) with 2 (4 SPLIT) CTAs per SM, counting the
  // aggregations the caller keeps in flight together
  const long long cols = (long long)nstrip * B * A.nslab * (conc > 1 ? conc : 1);
  const long long slots = (SPLIT ? 4LL : 2LL) * small_sm_count();
  int bestR = H;
  double best = 1e300;
  for (int n = 1; n <= H; n++) {
    const int R = (H + n - 1) / n;
    if (R < 16 && n > 1) break;
    const long long ctas = cols * ((H + R - 1) / R);
    const double c = (double)((ctas + slots - 1) / slots) * (R + 2 * RHO);
    if (c < best * 0.999) { best = c; bestR = R; }
  }
  A.R = bestR;
  const float log2e = 1.4426950408889634f;
  A.kd = -log2e / (gamma_d * gamma_d);
  A.kr = std::isinf(gamma_r) ? -1e-30f : -log2e / (gamma_r * gamma_r);
  A.vol = vol; A.guide = guide; A.nan_map = nan_map; A.out = out;
  const long long nblk = (long long)nstrip * ((H + bestR - 1) / bestR) * A.nslab * B;
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaError_t e = smem_optin((const void*)k_aggregate_small<RHO, SPLIT>, G::bytes);
  if (e != cudaSuccess) return e;
  k_aggregate_small<RHO, SPLIT><<<(unsigned)nblk, SM_TX, G::bytes, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_aggregate_small(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                                   const float* vol, const uint8_t* guide, const uint8_t* nan_map, float* out,
                                   cudaStream_t st) {
  // two threads per column (SPLIT) for rho >= 1; RSR_K3_SPLIT=0 keeps one (A/B)
  const char* e = getenv("RSR_K3_SPLIT");
  const bool split = !(e && e[0] == '0');
#define RSR_SM(R)                                                                                         \
  case R:                                                                                                 \
    return (split && R >= 1)                                                                              \
               ? small_launch_t<R, (R >= 1)>(B, H, W, D, gamma_d, gamma_r, conc, vol, guide, nan_map, out, st) \
               : small_launch_t<R, false>(B, H, W, D, gamma_d, gamma_r, conc, vol, guide, nan_map, out, st);
  switch (rho) {
    RSR_SM(0) RSR_SM(1) RSR_SM(2) RSR_SM(3) RSR_SM(4) RSR_SM(5) RSR_SM(6) RSR_SM(7)
    default:
      return cudaErrorInvalidValue;
  }
#undef RSR_SM
}

}  // namespace rsr
