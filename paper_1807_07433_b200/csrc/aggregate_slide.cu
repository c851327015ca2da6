// K3 — bilateral cost aggregation (fast bilateral stereo), PAPER.md:128-152,
// Eq. (8) with the weights of Eqs. (9)-(10):
//   A(u,v,k) = sum_t w_t C(u+dx, v+dy, k) / sum_t w_t,
//   w_t = exp(-(dx^2+dy^2)/gamma_d^2) * exp(-(g(u+dx,v+dy) - g(u,v))^2/gamma_r^2),
// taps outside the image or with a NaN cost skipped, NaN iff the centre cost is
// NaN (readings 10-12).  Used for rho <= 7; the paper's bottleneck
// (P:154), FP32-FMA bound: 2 (2 rho + 1)^2 flop per output.
//
// Design ("k-lane sliding window", DESIGN.md §6 K3):
//  * Lanes run along the disparity axis.  A group of G = KS/8 lanes owns one
//    output column x of a 32-column strip; lane l holds disparities
//    {4l..4l+3} and {4G+4l..4G+4l+3} of the slab.  The bilateral weight w(p,t)
//    does not depend on k, so all lanes of a group read the SAME weight
//    address: one LDS.128 broadcast serves 4 weights to 4 groups (one
//    shared-memory wavefront), each weight feeding 64 FMAs.  Cost loads are
//    per lane and contiguous (8 lanes x 16 B = one 128-B row per group); with
//    G = 4 the odd columns load their two halves in swapped order, so the two
//    columns of a quarter-warp never share banks.
//  * The strip slides down one input row at a time.  A thread keeps the
//    2 rho + 1 output rows whose windows contain the current input row
//    ("ages") x 8 disparities as packed pairs (104 registers at rho = 6), so
//    every staged cost feeds 2 rho + 1 FFMA2s.  Ages shift by one per input
//    row inside the last tap's FFMA2s (destination = next-younger register),
//    so the loop needs no unrolling over ages and no register moves.
//  * Warp roles (mbarrier hand-off, no CTA barrier inside a segment): G
//    consumer warps (FFMA2, fma.rn.f32x2 with a scalar weight operand) and 4
//    producer warps.  Producers compute each weight once per (pixel, tap) per
//    CTA as w = S(dx, dy) * R(g(q) - g(p)): the spatial factor exp2(kd (dx^2 +
//    dy^2)) lives in registers for the whole kernel, the range factor
//    exp2(kr dg^2) comes from a shared table indexed by the integer guide
//    difference (skipped pixels index its zero tail).  Producer warp 0 also
//    stages the cost rows (cp.async.bulk, the TMA engine, 4-stage ring).
//  * One CTA per (32-column strip, chunk of R rows, frame x slab); strips are
//    launched edge-first (longest-first scheduling of the general path).
//  * Tiles whose footprint holds no partially-NaN pixel (nan_map) take the
//    "clean" path: NaN-free costs (all-NaN or outside pixels get weight 0 and
//    cost 0) and one denominator per pixel.  Other segments take the exact
//    general path: pairs (C0, V) = (cost or 0, validity) so the same FFMA2
//    accumulates numerator and per-disparity denominator, two passes per slab.
//    Both accumulate in the same order, so they agree bitwise where both apply.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int SG_NPROD = 4;     // weight-producer warps (warp 0 also stages costs)
constexpr int SG_NSC = 4;       // cost stages
constexpr int SG_NSW = 3;       // weight stages
constexpr int SG_SEGMAX = 720;  // max output rows per segment (guide tile height)
constexpr short SG_GSKIP = 600;     // integer guide tile: skipped pixel (outside / all-NaN)
// skip code of the guide tile: 600 for uint8 guides (indexes the zero tail of the range
// table), 0xFFFF for 8.8 fixed-point guides (NEXT f2: values <= 65280)
template <bool G16>
RSR_DEVINL int gskip() { return G16 ? 0xFFFF : SG_GSKIP; }
// range table exp2(kr dg^2) at index dg + 255 (dg in [-255, 255]), entry 511 = 0: the
// index is clamped to 511, which the skip encodings (tap 600, centre -600) always reach.
// RC copies interleaved (entry i of copy c at i * RC + c; lane l reads copy l % RC):
// with RC = 16 two lanes of a warp meet in a bank only with probability 1/2, instead
// of the ~3.5-way conflicts of random indices into one table.  16 copies in the
// one-CTA-per-SM kernels (uint8 guide), one in the two-CTA and fixed-point variants.
constexpr int SG_RLUT = 512;
constexpr int SG_RCMAX = 16;
__host__ __device__ constexpr int slide_rc(int minb, bool g16) { return (minb == 1 && !g16) ? SG_RCMAX : 1; }

struct SlideGeom {
  int G, KS, CS, nslab, CX, XS, WST, GR, RC;
  size_t off_cost, off_w, off_dpart, off_guide, off_rlut, off_bar, bytes;
};

// KS = disparities per slab (multiple of 8, <= 64), G = consumer lanes per column
// rows = output rows the guide tile must hold (SG_SEGMAX for the one-CTA-per-SM
// kernels; the launch's R for the two-CTA variants, which need the space)
__host__ __device__ inline SlideGeom slide_geom(int D, int rho, int rows = SG_SEGMAX, bool compact = false,
                                                int rc = 1) {
  SlideGeom g;
  const int NT = 2 * rho + 1;
  g.nslab = (D + 63) / 64;
  const int per = (D + g.nslab - 1) / g.nslab;
  g.KS = (per + 7) & ~7;
  g.G = g.KS / 8;
  // cost column stride in the stage ring.  compact (the two-CTA small-slab kernels):
  // D itself when one slab holds all of D and rows stay 16-byte aligned, so a whole
  // row segment is one contiguous bulk copy (the lanes past D then read the next
  // column's costs: finite or NaN garbage in k slots that are never stored).  Else
  // KS with a filled tail.
  g.CS = (compact && g.nslab == 1 && (D & 3) == 0) ? D : g.KS;
  g.CX = 32 + 2 * rho;
  g.XS = 16 * NT + 4;                 // == 20 (mod 32): 4 / 8 columns hit distinct banks
  g.WST = 32 * g.XS + 32;             // weights [x][tap][age16] + completing rows' weight sums
  g.GR = rows + 4 * rho;
  g.RC = rc;
  size_t o = 0;
  g.off_cost = o;  o += sizeof(float) * (size_t)SG_NSC * g.CX * g.KS;
  g.off_w = o;     o += sizeof(float) * (size_t)SG_NSW * g.WST;
  g.off_dpart = o; o += sizeof(float) * (size_t)NT * 32;
  g.off_guide = o; o += sizeof(short) * (size_t)g.GR * g.CX;
  o = (o + 15) & ~size_t(15);
  g.off_rlut = o;  o += sizeof(float) * (size_t)SG_RLUT * g.RC;
  o = (o + 15) & ~size_t(15);
  g.off_bar = o;   o += 8 * (2 * SG_NSC + 2 * SG_NSW);
  g.bytes = o;
  return g;
}

RSR_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// d = w * c + a on a packed pair (FFMA2 with scalar-broadcast weight operand)
RSR_DEVINL float2 fma2s(float w, float2 c, float2 a) {
  unsigned long long av, cv, wb, dv;
  asm("mov.b64 %0, {%1,%2};" : "=l"(av) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1,%2};" : "=l"(cv) : "f"(c.x), "f"(c.y));
  asm("mov.b64 %0, {%1,%1};" : "=l"(wb) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(dv) : "l"(wb), "l"(cv), "l"(av));
  float2 d;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dv));
  return d;
}

// One output segment: rows [ya, yb) of strip x0 of frame b, disparity slab k0.
struct Seg {
  int b, k0, ks_eff, x0, ya, yb;
  size_t pix0;
};

struct SlideArgs {
  int B, H, W, D;
  int R;                 // output rows per CTA (<= SG_SEGMAX)
  int nstrips;           // 32-column strips
  float kd, kr;
  int hswap;             // clean path, G = 4: odd columns load their two halves in swapped order
  const float* vol;
  const void* guide;     // uint8 [B][H][W], or uint16 8.8 fixed point (G16)
  const uint8_t* nan_map;
  float* out;
};

// The CTA's segment.  The 1-D grid enumerates (strip rank, row chunk, frame x
// slab) with the strip rank slowest and strips ranked 0, n-1, 1, n-2, ...:
// image-edge strips, where stereo volumes hold partially-NaN pixels (the
// general path, twice as expensive), launch first and the hardware block
// scheduler back-fills the cheap interior strips (longest-first scheduling).
RSR_DEVINL Seg cta_segment(const SlideArgs& A, const SlideGeom& g) {
  Seg s;
  const int nchunk = (A.H + A.R - 1) / A.R;
  const long long per_strip = (long long)nchunk * A.B * g.nslab;
  const int rank = (int)(blockIdx.x / per_strip);
  const int rest = (int)(blockIdx.x % per_strip);
  const int strip = (rank & 1) ? A.nstrips - 1 - (rank >> 1) : (rank >> 1);
  const int chunk = rest % nchunk, bz = rest / nchunk;
  s.x0 = strip * 32;
  s.ya = chunk * A.R;
  s.yb = min(A.H, s.ya + A.R);
  s.b = bz / g.nslab;
  s.k0 = (bz % g.nslab) * g.KS;
  s.ks_eff = min(g.KS, A.D - s.k0);
  s.pix0 = (size_t)s.b * A.H * A.W;
  return s;
}

// ---- stager (lanes of producer warp 0): raw cost row i of the segment into
// the cost ring.  One bulk async copy (TMA engine) per in-image pixel column,
// or one for the whole row segment when it is contiguous; skipped columns
// (outside the image, or all-NaN on a clean segment) are filled with 0 (clean)
// or NaN (general path).
// rows of an even D that is not a multiple of 4 (no 16-byte bulk copies) with a
// power-of-two KS: staged by 8-byte cp.async spread over all producer threads,
// coalesced along k; the full barrier then expects 33 arrivals per producer warp
// (each lane's cp.async arrive, and lane 0 after the warp's fills)
__host__ __device__ inline bool stage_cpasync(int D, const SlideGeom& g) {
  return (D & 3) == 2 && (g.KS & (g.KS - 1)) == 0;
}

template <int RHO, bool G16>
__device__ __forceinline__ void stage_row(const SlideArgs& A, const SlideGeom& g, const Seg& s, bool clean,
                                          int i, const unsigned short* gt, float* cost_s, uint64_t* full_c, uint64_t* empty_c,
                                          uint32_t& it_c, int lane, int t = 0, int nt = 32) {
  const bool bulk = (A.D & 3) == 0;
  const float fillv = clean ? 0.f : qnan();
  const int st = it_c % SG_NSC;
  RSR_CHECK(st >= 0 && st < SG_NSC && g.CS <= g.KS);
  if (it_c >= SG_NSC) mbar_wait_parity(&empty_c[st], ((it_c / SG_NSC) & 1) ^ 1);
  it_c++;
  const int yy = s.ya - RHO + i;
  float* dst = cost_s + (size_t)st * g.CX * g.KS;
  const bool row_in = yy >= 0 && yy < A.H;
  const size_t rowpix = s.pix0 + (size_t)yy * A.W;
  if (stage_cpasync(A.D, g)) {
    const int lg = __ffs(g.KS) - 2;   // log2(KS / 2): float pairs per column
    for (int e = t; e < (g.CX << lg); e += nt) {
      const int col = e >> lg, k = 2 * (e & ((1 << lg) - 1));
      float* d = dst + col * g.KS + k;
      // the guide tile marks outside and all-NaN pixels: filled, not copied
      const bool skip = !row_in || gt[(i + RHO) * g.CX + col] == gskip<G16>();
      if (!skip && k < s.ks_eff) {
        RSR_CHECK(col < g.CX && k + 1 < g.KS && s.x0 - RHO + col >= 0 && s.x0 - RHO + col < A.W);
        cp_async8(d, A.vol + (rowpix + (s.x0 - RHO + col)) * A.D + s.k0 + k);
      } else {
        d[0] = fillv;
        d[1] = fillv;
      }
    }
    cp_async_mbar_arrive_noinc(&full_c[st]);
    __syncwarp();
    if (lane == 0) mbar_arrive(&full_c[st]);   // this warp's fills are in
    return;
  }
  bool cp[2];
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int col = lane + 32 * h;
    const int xx = s.x0 - RHO + col;
    // the guide tile marks outside and all-NaN pixels (+inf): fill them instead of copying
    // (all-NaN -> 0 on a clean segment, where such taps carry weight 0; NaN otherwise)
    const bool skip = !(col < g.CX && row_in) ||
                      gt[(i + RHO) * g.CX + col] == gskip<G16>();
    cp[h] = !skip && bulk;
    if (col < g.CX) {
      float* d = dst + col * g.CS;
      if (!skip && !bulk) {
        const float* sp = A.vol + (rowpix + xx) * A.D + s.k0;
        for (int k = 0; k < g.CS; k++) d[k] = k < s.ks_eff ? sp[k] : fillv;
      } else if (skip) {
        for (int k = 0; k < g.CS; k += 4) *reinterpret_cast<float4*>(d + k) = make_float4(fillv, fillv, fillv, fillv);
      } else if (s.ks_eff < g.CS) {
        for (int k = s.ks_eff; k < g.CS; k++) d[k] = fillv;   // slab tail (the copy fills the head)
      }
    }
  }
  const uint32_t ncols = __popc(__ballot_sync(0xffffffffu, cp[0])) + __popc(__ballot_sync(0xffffffffu, cp[1]));
  __syncwarp();
  const float* src = A.vol + (rowpix + (s.x0 - RHO)) * A.D + s.k0;
  if (ncols == (uint32_t)g.CX && g.CS == A.D) {
    // whole row segment in the image and one contiguous run: a single bulk copy
    const uint32_t bytes = (uint32_t)g.CX * g.CS * 4u;
    RSR_CHECK(g.CX * g.CS <= g.CX * g.KS && s.x0 - RHO >= 0 && s.x0 - RHO + g.CX <= A.W);
    if (lane == 0) {
      mbar_arrive_expect_tx(&full_c[st], bytes);
      bulk_g2s(dst, src, bytes, &full_c[st]);
    }
  } else {
    const uint32_t bytes_col = (uint32_t)s.ks_eff * 4u;
    if (lane == 0) mbar_arrive_expect_tx(&full_c[st], bytes_col * ncols);
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int col = lane + 32 * h;
      if (cp[h]) {
        RSR_CHECK(col * g.CS + s.ks_eff <= g.CX * g.KS && s.x0 - RHO + col >= 0 && s.x0 - RHO + col < A.W);
        bulk_g2s(dst + col * g.CS, src + (size_t)col * A.D, bytes_col, &full_c[st]);
      }
    }
  }
}

// ---- weight producers (SG_NPROD warps): weights of input row r for the
// 2 rho + 1 output rows (ages) whose windows contain it,
//   w[x][j][age] = exp2(kd (dx^2 + dy^2) + kr (g(q) - g(p))^2),
// and the per-pixel weight sums.  A lane owns (column x, age a) over 8 columns
// x 4 ages (conflict-free 4-byte stores into the [x][tap][age] layout) and
// walks the taps j in order, so the running sum of an output row's weights is
// accumulated in exactly the (input row, tap) order in which the general path's
// FFMA2 accumulates its per-disparity denominators: both paths give bitwise
// identical results wherever both apply, whatever the segmentation (batch-size
// independence).  Warp 0 also stages the cost rows.
template <int RHO, bool G16, int RC>
__device__ __forceinline__ void produce_weights(const SlideArgs& A, const SlideGeom& g, const Seg& s,
                                                bool clean, int npass, const unsigned short* gt, float* w_s,
                                                float* dsum, float* cost_s, uint64_t* full_w,
                                                uint64_t* empty_w, uint64_t* full_c, uint64_t* empty_c,
                                                uint32_t& it_w, uint32_t& it_c, int p, int lane,
                                                const float* rlut) {
  constexpr int NT = 2 * RHO + 1;
  constexpr int NAB = (NT + 3) / 4;          // age blocks of 4
  const int NR = (s.yb - s.ya) + 2 * RHO;
  const int xs = lane >> 2, as = lane & 3;
  // exp2(kd (dx^2 + dy^2)) for this lane's ages: items (n, n + 1) as packed pairs (the
  // range-table path multiplies and sums two items per FMUL2 / FADD2), an odd last item
  constexpr int NP = NAB / 2;
  float2 sp[NP > 0 ? NP : 1][NT];
  float ss[NT];
  auto sfac = [&](int n, int j) {
    const int a = min(n * 4 + as, NT - 1);
    return ex2_ftz((float)((j - RHO) * (j - RHO) + (RHO - a) * (RHO - a)) * A.kd);
  };
#pragma unroll
  for (int j = 0; j < NT; j++) {
#pragma unroll
    for (int q = 0; q < NP; q++) sp[q][j] = make_float2(sfac(2 * q, j), sfac(2 * q + 1, j));
    ss[j] = (NAB & 1) ? sfac(NAB - 1, j) : 0.f;
  }
  auto sreg = [&](int n, int j) { return (NAB & 1) && n == NAB - 1 ? ss[j] : ((n & 1) ? sp[n >> 1][j].y : sp[n >> 1][j].x); };
  const bool cpa = stage_cpasync(A.D, g);
  for (int pass = 0; pass < npass; pass++) {
    // warp p owns the columns 8p .. 8p + 7 (every age): its running sums are its own
    for (int e = lane; e < NT * 8; e += 32) dsum[(e >> 3) * 32 + 8 * p + (e & 7)] = 0.f;
    __syncwarp();
    for (int i = 0; i < NR; i++, it_w++) {
      // cp.async-staged rows: every producer warp issues a share (non-blocking)
      if (cpa || p == 0)
        stage_row<RHO, G16>(A, g, s, clean, i, gt, cost_s, full_c, empty_c, it_c, lane, p * 32 + lane, SG_NPROD * 32);
      const int st = it_w % SG_NSW;
      if (it_w >= SG_NSW) mbar_wait_parity(&empty_w[st], ((it_w / SG_NSW) & 1) ^ 1);
      float* wst = w_s + (size_t)st * g.WST;
      // this warp's items: x-block p, age-blocks n < NAB (the running sums of a column
      // never leave its warp, so no barrier among the producer warps); all shared-memory
      // loads first, then the math, then the stores: the tile, the running sums and
      // the weight stage may alias as far as the compiler knows, so interleaving them
      // would serialise every tap's LDS -> MUFU -> STS chain
      static_assert(SG_NPROD == 4, "items are dealt to 4 producer warps");
      // w = S(a, j) * R(g(q) - g(p)): spatial factor per (age, tap) held in registers
      // for the whole kernel (sreg), range factor from a shared table indexed by the
      // integer guide difference (skipped pixels index the zero tail of the table).
      const unsigned short* trs = gt + (i + RHO) * g.CX;   // tap row r
#ifdef RSR_EXP_NOWCOMP   // experiment build (tools/k3_exp.sh): weights not computed (timing only)
      if (i >= 0) { __syncwarp(); mbar_arrive(&full_w[st]); continue; }
#endif
      // the tap row's guide values of this lane's column, loaded once for its NAB items
      // (reloaded per item otherwise: the item's stores may alias the tile)
      int gq[NT];
#pragma unroll
      for (int j = 0; j < NT; j++) gq[j] = trs[p * 8 + xs + j];
      const int x = p * 8 + xs;
      RSR_CHECK((i + RHO) < g.GR && x + 2 * RHO < g.CX);
      int gp[NAB];
      float* slot[NAB];
      float d[NAB], w[NAB][NT];
#pragma unroll
      for (int n = 0; n < NAB; n++) {
        const int ac = min(n * 4 + as, NT - 1);
        RSR_CHECK((i + ac) < g.GR);
        gp[n] = gt[(i + ac) * g.CX + x + RHO];
        slot[n] = dsum + ((i + ac) % NT) * 32 + x;
        d[n] = *slot[n];
      }
      if (G16) {
        // 8.8 fixed-point guide: range factor exp2(kr (dg / 256)^2) on the MUFU pipe,
        // zero for skipped pixels (the tap's or the centre's)
#pragma unroll
        for (int n = 0; n < NAB; n++) {
          const bool pskip = gp[n] == gskip<G16>();
#pragma unroll
          for (int j = 0; j < NT; j++) {
            const float dg = (float)(gq[j] - gp[n]);
            w[n][j] = (pskip || gq[j] == gskip<G16>()) ? 0.f : sreg(n, j) * ex2_ftz(A.kr * (dg * dg));
            d[n] += w[n][j];
          }
        }
      } else {
        float r[NAB][NT];
#pragma unroll
        for (int n = 0; n < NAB; n++) {
          const int gpn = (gp[n] == SG_GSKIP) ? -SG_GSKIP : gp[n];
#pragma unroll
          for (int j = 0; j < NT; j++) {
            const int ix = min(gq[j] - gpn + 255, SG_RLUT - 1);
            RSR_CHECK(ix >= 0 && ix < SG_RLUT);
            r[n][j] = rlut[ix * RC];   // rlut: this lane's copy
          }
        }
        // w = S * R and the running sums in tap order, two items per packed op (the
        // same two IEEE roundings as the scalar FMUL / FADD)
#pragma unroll
        for (int q = 0; q < NP; q++) {
          float2 d2 = make_float2(d[2 * q], d[2 * q + 1]);
#pragma unroll
          for (int j = 0; j < NT; j++) {
            const float2 w2 = f2mul(sp[q][j], make_float2(r[2 * q][j], r[2 * q + 1][j]));
            w[2 * q][j] = w2.x;
            w[2 * q + 1][j] = w2.y;
            d2 = f2add(d2, w2);
          }
          d[2 * q] = d2.x;
          d[2 * q + 1] = d2.y;
        }
        if (NAB & 1) {
#pragma unroll
          for (int j = 0; j < NT; j++) {
            w[NAB - 1][j] = ss[j] * r[NAB - 1][j];
            d[NAB - 1] += w[NAB - 1][j];
          }
        }
      }
#pragma unroll
      for (int n = 0; n < NAB; n++) {
        const int a = n * 4 + as;
        if (a < NT) {
          float* wd = wst + x * g.XS + a;
          RSR_CHECK(x * g.XS + a + (NT - 1) * 16 < 32 * g.XS && a < 16);
#pragma unroll
          for (int j = 0; j < NT; j++) wd[j * 16] = w[n][j];
          if (a == 0) {   // the output row completing at input row i
            wst[32 * g.XS + x] = d[n];
            *slot[n] = 0.f;
          } else {
            *slot[n] = d[n];
          }
        }
      }
      __syncwarp();   // row sums handed to the next age (same warp)
      mbar_arrive(&full_w[st]);
    }
  }
}

// One input row of the sliding accumulation: NT taps, each FFMA2-ing NQ cost pairs
// into the 2 rho + 1 ages; the last tap shifts the ages and returns the completed
// row in fin.  MODE 0: clean pairs (k, k+1) of 8 disparities (NQ = 4); MODE 1:
// (cost or 0, validity) of 4 disparities (NQ = 4); MODE 2: (cost or 0) pairs of 4
// disparities with the per-pixel denominator (a half whose pixels are all fully
// valid or skipped, NQ = 2).
// oa (MODE 0): offset of the half loaded first (0, or 4G for a swapped column: with
// G = 4 a quarter-warp of a 16-byte load spans two columns whose same halves sit in the
// same 16 banks; swapping the odd column's halves makes the two columns' loads disjoint)
template <int RHO, int MODE>
RSR_DEVINL void slide_row(float2 (&acc)[2 * RHO + 1][4], float2 (&fin)[4], const float* crow,
                          const float* wrow, int CS, int G, int oa = 0) {
  constexpr int NT = 2 * RHO + 1;
  constexpr int NQ = MODE == 2 ? 2 : 4;
#pragma unroll
  for (int j = 0; j < NT; j++) {
    float2 cp[4];
    if (MODE == 0) {
      const float4 ca = *reinterpret_cast<const float4*>(crow + j * CS + oa);
      const float4 cb = *reinterpret_cast<const float4*>(crow + j * CS + (4 * G - oa));
      cp[0] = make_float2(ca.x, ca.y); cp[1] = make_float2(ca.z, ca.w);
      cp[2] = make_float2(cb.x, cb.y); cp[3] = make_float2(cb.z, cb.w);
    } else {
      const float4 t = *reinterpret_cast<const float4*>(crow + j * CS);
      const float tv[4] = {t.x, t.y, t.z, t.w};
      if (MODE == 1) {
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const bool ok = !(tv[q] != tv[q]);
          cp[q] = make_float2(ok ? tv[q] : 0.f, ok ? 1.f : 0.f);
        }
      } else {
        float c0[4];
#pragma unroll
        for (int q = 0; q < 4; q++) c0[q] = (tv[q] != tv[q]) ? 0.f : tv[q];
        cp[0] = make_float2(c0[0], c0[1]);
        cp[1] = make_float2(c0[2], c0[3]);
      }
    }
    float wv[16];
    const float4* w4 = reinterpret_cast<const float4*>(wrow + j * 16);
#pragma unroll
    for (int q = 0; q < (NT + 3) / 4; q++) {
      const float4 t = w4[q];
      wv[4 * q] = t.x; wv[4 * q + 1] = t.y; wv[4 * q + 2] = t.z; wv[4 * q + 3] = t.w;
    }
    // q outer, ages inner: the cost pair stays in the operand reuse cache for
    // 2 rho + 1 consecutive FFMA2s, so each reads only the weight and the
    // accumulator pair from the register file (2 reads per bank)
    if (j < NT - 1) {
#pragma unroll
      for (int q = 0; q < NQ; q++)
#pragma unroll
        for (int a = 0; a < NT; a++) acc[a][q] = fma2s(wv[a], cp[q], acc[a][q]);
    } else {
      // last tap of the row: age 0 completes, every other age moves one slot down
#pragma unroll
      for (int q = 0; q < NQ; q++) {
        fin[q] = fma2s(wv[0], cp[q], acc[0][q]);
#pragma unroll
        for (int a = 1; a < NT; a++) acc[a - 1][q] = fma2s(wv[a], cp[q], acc[a][q]);
        acc[NT - 1][q] = make_float2(0.f, 0.f);
      }
    }
  }
}

// ---- consumers (G warps): sliding accumulation, FFMA2 -----------------------
template <int RHO, bool CLEAN, bool G16>
__device__ __forceinline__ void consume(const SlideArgs& A, const SlideGeom& g, const Seg& s,
                                        const float* cost_s, const float* w_s, uint64_t* full_c,
                                        uint64_t* empty_c, uint64_t* full_w, uint64_t* empty_w,
                                        uint32_t& it, int xl, int l, int lane, const unsigned short* gt,
                                        int hcmask) {
  constexpr int NT = 2 * RHO + 1;
  constexpr int NPASS = CLEAN ? 1 : 2;
  const int NR = (s.yb - s.ya) + 2 * RHO;
  const int x = s.x0 + xl;
  const bool vec_out = (A.D & 3) == 0;
  // A warp whose output pixels are all skipped (centre outside the image or all-NaN)
  // writes NaN and only keeps the pipeline hand-off going: no FFMA2.
  bool live = false;
  for (int y = s.ya + l; y < s.yb; y += g.G) live |= gt[(y - s.ya + 2 * RHO) * g.CX + xl + RHO] != gskip<G16>();
  if (!__any_sync(0xffffffffu, live)) {
    for (int pass = 0; pass < NPASS; pass++) {
      const int koff = CLEAN ? 4 * l : 4 * g.G * pass + 4 * l;
      for (int i = 0; i < NR; i++, it++) {
        const int stc = it % SG_NSC, stw = it % SG_NSW;
        mbar_wait_parity(&full_c[stc], (it / SG_NSC) & 1);
        mbar_wait_parity(&full_w[stw], (it / SG_NSW) & 1);
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty_c[stc]);
          mbar_arrive(&empty_w[stw]);
        }
        const int y = s.ya - 2 * RHO + i;
        if (y >= s.ya && x < A.W) {
          float* o = A.out + (s.pix0 + (size_t)y * A.W + x) * A.D + s.k0 + koff;
#pragma unroll
          for (int hh = 0; hh < (CLEAN ? 2 : 1); hh++)
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const int k = s.k0 + koff + 4 * g.G * hh + q;
              if (k < s.k0 + s.ks_eff) o[4 * g.G * hh + q] = qnan();
            }
        }
      }
    }
    return;
  }
  // clean path with G = 4: odd columns hold the upper half of their disparities in
  // acc[.][0..1] and the lower half in acc[.][2..3] (bank-conflict-free cost loads)
  const int sw = (CLEAN && A.hswap && g.G == 4) ? (xl & 1) : 0;
  const int oa = sw ? 4 * g.G : 0;
  for (int pass = 0; pass < NPASS; pass++) {
    float2 acc[NT][4];
#pragma unroll
    for (int a = 0; a < NT; a++)
#pragma unroll
      for (int q = 0; q < 4; q++) acc[a][q] = make_float2(0.f, 0.f);
    // this lane's disparities: clean {4l..4l+3} U {4G+4l..}, general pass h: {4Gh + 4l..}
    const int koff = CLEAN ? 4 * l : 4 * g.G * pass + 4 * l;
    // this half has no partially-NaN pixel (not used at rho = 7, where the extra code
    // path would push the 120 accumulators into spills)
    const bool hc = !CLEAN && RHO < 7 && ((hcmask >> pass) & 1);
    for (int i = 0; i < NR; i++, it++) {
      const int stc = it % SG_NSC, stw = it % SG_NSW;
      mbar_wait_parity(&full_c[stc], (it / SG_NSC) & 1);
      mbar_wait_parity(&full_w[stw], (it / SG_NSW) & 1);
      const float* crow = cost_s + (size_t)stc * g.CX * g.KS + xl * g.CS + koff;
      const float* wrow = w_s + (size_t)stw * g.WST + xl * g.XS;
      RSR_CHECK(xl * g.CS + koff + (NT - 1) * g.CS + (CLEAN ? 4 * g.G : 0) + 4 <= g.CX * g.KS);
      RSR_CHECK(xl * g.XS + (NT - 1) * 16 + 16 <= 32 * g.XS && xl < 32);
      float2 fin[4];
      if (CLEAN)
        slide_row<RHO, 0>(acc, fin, crow, wrow, g.CS, g.G, oa);
      else if (hc)
        slide_row<RHO, 2>(acc, fin, crow, wrow, g.CS, g.G);
      else
        slide_row<RHO, 1>(acc, fin, crow, wrow, g.CS, g.G);
      const float den = (CLEAN || hc) ? wrow[(32 - xl) * g.XS + xl] : 0.f;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_c[stc]);
        mbar_arrive(&empty_w[stw]);
      }
      const int y = s.ya - 2 * RHO + i;   // completing output row
      if (y >= s.ya && x < A.W) {
        const size_t pix = s.pix0 + (size_t)y * A.W + x;
        float* o = A.out + pix * A.D + s.k0 + koff;
        RSR_CHECK(pix < (size_t)A.B * A.H * A.W);   // k beyond D: never written (predicated below)
        if (CLEAN) {
          // den == 0 exactly when the centre is skipped (all-NaN): 0 * inf = NaN
          const float inv = rcp_fast(den);
          const float r[8] = {fin[0].x * inv, fin[0].y * inv, fin[1].x * inv, fin[1].y * inv,
                              fin[2].x * inv, fin[2].y * inv, fin[3].x * inv, fin[3].y * inv};
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            const int kb = s.k0 + koff + 4 * g.G * (hh ^ sw);
            float* oh = o + 4 * g.G * (hh ^ sw);
            if (vec_out && kb + 3 < A.D) {
              *reinterpret_cast<float4*>(oh) = make_float4(r[4 * hh], r[4 * hh + 1], r[4 * hh + 2], r[4 * hh + 3]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; q++)
                if (kb + q < A.D) oh[q] = r[4 * hh + q];
            }
          }
        } else if (hc) {
          // fully valid half: same formula as the clean path (bitwise equal)
          const float inv = rcp_fast(den);
          const float r[4] = {fin[0].x * inv, fin[0].y * inv, fin[1].x * inv, fin[1].y * inv};
#pragma unroll
          for (int q = 0; q < 4; q++)
            if (s.k0 + koff + q < s.k0 + s.ks_eff) o[q] = r[q];
        } else {
          const float* cv = A.vol + pix * A.D + s.k0 + koff;
          const float fv[8] = {fin[0].x, fin[0].y, fin[1].x, fin[1].y, fin[2].x, fin[2].y, fin[3].x, fin[3].y};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const int k = s.k0 + koff + q;
            if (k < s.k0 + s.ks_eff) {
              const float c = cv[q];
              o[q] = (c != c) ? qnan() : fv[2 * q] * rcp_fast(fv[2 * q + 1]);
            }
          }
        }
      }
    }
  }
}

// MINB = 1: up to 8 consumer warps (D up to 64 per slab), one CTA per SM.  MINB = 2:
// small slabs (G <= 2 at any rho, G <= 4 at rho <= 5), two CTAs per SM so the few
// consumer warps of a CTA do not leave the SM idle; the guide tile is sized by R.
template <int RHO, int MINB, bool COMPACT, bool G16>
__global__ void __launch_bounds__(MINB == 1 ? 384 : (RHO <= 5 ? 256 : 192), MINB)
    k_aggregate_slide(const SlideArgs A) {
  extern __shared__ __align__(128) unsigned char sl_smem[];
  constexpr int RC = slide_rc(MINB, G16);
  const SlideGeom g = slide_geom(A.D, RHO, A.R, COMPACT, RC);
  float* cost_s = reinterpret_cast<float*>(sl_smem + g.off_cost);
  float* w_s = reinterpret_cast<float*>(sl_smem + g.off_w);
  float* dpart = reinterpret_cast<float*>(sl_smem + g.off_dpart);
  unsigned short* gt = reinterpret_cast<unsigned short*>(sl_smem + g.off_guide);
  float* rlut = reinterpret_cast<float*>(sl_smem + g.off_rlut);
  // range factor exp2(kr dg^2) at index dg + 255 (RC interleaved copies); entry 511 = 0
  for (int t = threadIdx.x; t < SG_RLUT * RC; t += blockDim.x) {
    const int dg = t / RC - 255;
    rlut[t] = (dg >= -255 && dg <= 255) ? ex2_ftz((float)(dg * dg) * A.kr) : 0.f;
  }
  uint64_t* full_c = reinterpret_cast<uint64_t*>(sl_smem + g.off_bar);
  uint64_t* empty_c = full_c + SG_NSC;
  uint64_t* full_w = empty_c + SG_NSC;
  uint64_t* empty_w = full_w + SG_NSW;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_cons = g.G;   // consumer warps
  if (tid == 0) {
    for (int q = 0; q < SG_NSC; q++) {
      // cp.async-staged rows: each producer thread's cp.async arrive + one per warp after its fills
      mbar_init(&full_c[q], stage_cpasync(A.D, g) ? SG_NPROD * 33 : 1);
      mbar_init(&empty_c[q], n_cons);
    }
    for (int q = 0; q < SG_NSW; q++) {
      mbar_init(&full_w[q], 32 * SG_NPROD);
      mbar_init(&empty_w[q], n_cons);
    }
    fence_mbar_init();
  }
  uint32_t it = 0, it_c = 0;   // per-role running row counters (mbarrier phases continue across segments)
  {
    const Seg s = cta_segment(A, g);
    // ---- classify the segment and load its guide tile ----
    // nan_map byte: bit 0 = some disparity NaN, bit 1 = some disparity finite.  Only a
    // partially-NaN pixel (3) needs per-disparity denominators (the general path).
    int partial = (A.nan_map == nullptr) ? 1 : 0;
    int dirty = (A.nan_map == nullptr) ? 3 : 0;
    const int rows = (s.yb - s.ya) + 4 * RHO;
    constexpr int UNR = 8;   // independent loads in flight per thread
    for (int e0 = tid; e0 < rows * g.CX; e0 += UNR * blockDim.x) {
      uint8_t mv[UNR];
    unsigned short gv[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int e = e0 + u * blockDim.x;
        const int yy = s.ya - 2 * RHO + e / g.CX, xx = s.x0 - RHO + e % g.CX;
        mv[u] = 1;   // outside the image: skipped like an all-NaN pixel
        gv[u] = 0;
        if (e < rows * g.CX && yy >= 0 && yy < A.H && xx >= 0 && xx < A.W) {
          const size_t pi = s.pix0 + (size_t)yy * A.W + xx;
          mv[u] = A.nan_map ? __ldg(A.nan_map + pi) : 2;
          gv[u] = G16 ? __ldg(static_cast<const uint16_t*>(A.guide) + pi)
                      : (unsigned short)__ldg(static_cast<const uint8_t*>(A.guide) + pi);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int e = e0 + u * blockDim.x;
        if (e < rows * g.CX) {
          const int yy = s.ya - 2 * RHO + e / g.CX;
          if ((mv[u] & 3) == 3 && yy >= s.ya - RHO && yy < s.yb + RHO) {
            partial = 1;
            // bits 2/3: NaN present in disparity half 0/1, valid when bit 7 is set
            // (k_nan_maps, single-slab volumes); otherwise both halves are dirty
            dirty |= ((mv[u] & 0x80) && g.nslab == 1) ? ((mv[u] >> 2) & 3) : 3;
          }
          // +inf marks a skipped pixel (outside the image or all-NaN)
          gt[e] = (mv[u] & 3) == 1 ? (unsigned short)gskip<G16>() : gv[u];
        }
      }
    }
    const bool clean = !__syncthreads_or(partial);
    // pass h of the general path is "half-clean" when no partial pixel has NaN in half h
    const int hcmask = (__syncthreads_or(dirty & 1) ? 0 : 1) | (__syncthreads_or(dirty & 2) ? 0 : 2);
    const int npass = clean ? 1 : 2;
    if (warp >= n_cons) {
      produce_weights<RHO, G16, RC>(A, g, s, clean, npass, gt, w_s, dpart, cost_s, full_w, empty_w, full_c,
                                    empty_c, it, it_c, warp - n_cons, lane, rlut + (lane & (RC - 1)));
    } else {
      const int t = tid;   // consumer thread: column t / G, lane-in-group t % G
      if (clean)
        consume<RHO, true, G16>(A, g, s, cost_s, w_s, full_c, empty_c, full_w, empty_w, it, t / g.G, t % g.G, lane, gt, hcmask);
      else
        consume<RHO, false, G16>(A, g, s, cost_s, w_s, full_c, empty_c, full_w, empty_w, it, t / g.G, t % g.G, lane, gt, hcmask);
    }
  }
}

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// Row chunk R of one launch: minimise (waves of minb-CTAs-per-SM launches) x (R + 2 rho
// warm-up rows), counting the CTAs of the conc aggregations the caller keeps in flight
// together.  minb = 2 (two CTAs per SM) for small slabs whose guide tile of R rows leaves
// room for two (at most 113 KB each).
struct SlidePlan {
  int R, minb;
  bool compact;
  size_t bytes;
};

static SlidePlan slide_plan(int B, int H, int W, int D, int rho, int conc, int nsm) {
  const SlideGeom g1 = slide_geom(D, rho);
  const int nstrips = (W + 31) / 32;
  const long long cols = (long long)nstrips * B * g1.nslab;
  const bool small = g1.G <= (rho <= 5 ? 4 : 2);
  const int minb = small ? 2 : 1;
  // the guide tile holds the launch's R rows (+ halo) next to the range-table copies
  auto fits = [&](int R) {
    return slide_geom(D, rho, R, false, slide_rc(minb, false)).bytes <= (minb == 1 ? 227 : 113) * 1024;
  };
  const long long inflight = conc > 1 ? conc : 1;
  int bestR = 0;
  double best = 1e300;
  for (int n = (H + SG_SEGMAX - 1) / SG_SEGMAX; n <= H; n++) {
    const int R = (H + n - 1) / n;
    if (R < 8 && n > 1) break;
    if (!fits(R)) continue;
    const long long ctas = cols * ((H + R - 1) / R) * inflight;
    const double cost = (double)((ctas + (long long)minb * nsm - 1) / ((long long)minb * nsm)) * (R + 2 * rho);
    if (cost < best * 0.999) { best = cost; bestR = R; }
  }
  if (const char* e = getenv("RSR_K3_ROWS")) {   // experiment hook (tools/): force R
    const int r = atoi(e);
    if (r >= 8 && r <= SG_SEGMAX && fits(r)) bestR = r;
  }
  if (bestR == 0) bestR = 8;
  SlidePlan p;
  p.R = bestR;
  p.minb = minb;
  // compact cost rows (one bulk copy per row) where D < KS and rows stay aligned; the
  // compact kernels spill a little more, so D == KS keeps the padded layout
  p.compact = small && g1.nslab == 1 && (D & 3) == 0 && D < g1.KS;
  p.bytes = slide_geom(D, rho, bestR, p.compact, slide_rc(minb, false)).bytes;
  return p;
}

#ifndef RSR_SLIDE_G16
int aggregate_plan_rows(int B, int H, int W, int D, int rho, int conc) {
  if (rho > 7) return 0;   // tiled kernel (aggregate.cu): no row chunks
  return slide_plan(B, H, W, D, rho, conc, sm_count()).R;
}
#endif

template <int RHO, bool G16>
static cudaError_t slide_launch_t(int B, int H, int W, int D, float gamma_d, float gamma_r, int conc,
                                  const float* vol, const void* guide, const uint8_t* nan_map,
                                  float* out, cudaStream_t st) {
  const SlideGeom g1 = slide_geom(D, RHO);
  const SlidePlan plan = slide_plan(B, H, W, D, RHO, conc, sm_count());
  SlideArgs A;
  A.B = B; A.H = H; A.W = W; A.D = D;
  const int nstrips = (W + 31) / 32;
  const long long cols = (long long)nstrips * B * g1.nslab;
  A.R = plan.R;
  A.nstrips = nstrips;
  const float log2e = 1.4426950408889634f;
  A.kd = -log2e / (gamma_d * gamma_d);
  A.kr = std::isinf(gamma_r) ? -1e-30f : -log2e / (gamma_r * gamma_r);
  if (G16) A.kr = std::isinf(gamma_r) ? 0.f : A.kr * (1.f / 65536.f);   // guide differences in 1/256 units
  A.vol = vol; A.guide = guide; A.nan_map = nan_map; A.out = out;
  {
    const char* e = getenv("RSR_K3_SWAP");   // experiment hook (tools/): 0 = unswapped loads
    A.hswap = !(e && e[0] == '0');
  }
  const long long nblk = cols * ((H + plan.R - 1) / plan.R);
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidValue;
  auto kern = plan.minb == 1 ? k_aggregate_slide<RHO, 1, false, G16>
                             : (plan.compact ? k_aggregate_slide<RHO, 2, true, G16>
                                             : k_aggregate_slide<RHO, 2, false, G16>);
  // the fixed-point guide's range factor is computed (MUFU): one (unused) table copy
  const size_t bytes = slide_geom(D, RHO, plan.R, plan.compact, slide_rc(plan.minb, G16)).bytes;
  cudaError_t e = smem_optin((const void*)kern, bytes);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)nblk, 32 * (g1.G + SG_NPROD), bytes, st>>>(A);
  return cudaGetLastError();
}

#ifndef RSR_SLIDE_G16
size_t aggregate_slide_smem(int D, int rho, int H) { (void)H; return slide_geom(D, rho).bytes; }
#endif

#ifndef RSR_SLIDE_G16
cudaError_t launch_aggregate_slide(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                                   const float* vol, const uint8_t* guide, const uint8_t* nan_map,
                                   float* out, cudaStream_t st) {
  constexpr bool G16 = false;
#else
cudaError_t launch_aggregate_slide16(int B, int H, int W, int D, int rho, float gamma_d, float gamma_r, int conc,
                                     const float* vol, const uint16_t* guide, const uint8_t* nan_map,
                                     float* out, cudaStream_t st) {
  constexpr bool G16 = true;
#endif
#define RSR_S(R) \
  case R: return slide_launch_t<R, G16>(B, H, W, D, gamma_d, gamma_r, conc, vol, guide, nan_map, out, st);
  switch (rho) {
    RSR_S(0) RSR_S(1) RSR_S(2) RSR_S(3) RSR_S(4) RSR_S(5) RSR_S(6) RSR_S(7)
    default:
      return cudaErrorInvalidValue;
  }
#undef RSR_S
}

}  // namespace rsr
