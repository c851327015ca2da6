// K_F — fused, volume-free matching (NEXT row f1): NCC (Eqs. 3-5) ->
// bilateral aggregation of both volumes (Eqs. 8-10) -> WTA, left-right
// consistency, parabola subpixel and post-processing (Eqs. 11-12) in
// one kernel; no cost or aggregated volume ever reaches HBM ("performing
// the bilateral filtering on the whole cost volume is a very time-consuming
// process").  Small search ranges (D <= 8, e.g. the restricted band of P:251).
//
// A CTA owns a 120-column strip of reference pixels and the 128 target-view
// columns their left-right check reads ([x0 - d_hi, x0 - d_hi + 128)), and slides
// down a chunk of rows one input row at a time:
//   N1  image rows (ring of 2 varrho + 2), the block statistics and guide bytes of
//       the row, prefetched into registers during the previous row's aggregation;
//   N2  exact vertical NCC dot sums (sliding, fp32 integers < 2^24);
//   N3  horizontal sums and the normalisation of K2 (zncc.cu: error-free
//       products, (num * inv_L) * inv_W, clamp) -> the reference-volume cost row
//       C_L(x, k) over every column either aggregation needs;
//   N4  the target-volume row by the shear C_R(x', k) = C_L(x' + d_lo + k, k)
//       (P:106), NaN-free copies, per-column NaN masks and guide codes (rings of
//       2 rho + 1 rows for the exact denominators below);
//   A   both aggregations with the sliding-window scheme of aggregate_small.cu
//       (thread per column, 8 disparities, 2 rho + 1 ages, in-thread weights);
//   W   at the completion of an output row: WTA of both views, k_R to shared
//       memory, then k_L, Eq. (11), Eq. (12) and the shift s(v) (K4's arithmetic).
// Denominators: the running weight sum of the clean path; where a window holds
// a non-skipped pixel whose cost is NaN at k (borders, the warp band, constant
// blocks: tracked by OR-ed masks), the exact sum of w * validity is recomputed
// for that (pixel, k) in the general path's (input row, tap) order.  Every value
// is computed by the same operations, in the same order, as the five-call path
// (K2, K3, K4), so rsr_match's disparity maps equal theirs bit for bit.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

constexpr int MF_TXR = 120;    // reference columns per strip
constexpr int MF_TXT = 128;    // target columns per strip (threads 0..127)
constexpr int MF_KD = 8;       // disparities (D <= 8)
constexpr int MF_LUT = 512;
constexpr int MF_SKIPQ = 4096;
constexpr int MF_THREADS = 256;

struct MatchArgs {
  int B, H, W, D, d_lo, P, R, lrc_tol, subpix;
  float kd, kr;
  const uint8_t* ref;       // L
  const uint8_t* warped;    // W (rsr_warp)
  const int32_t* shift;     // s(v)
  const int32_t* SL;
  const float* iL;
  const int32_t* SW;
  const float* iW;
  float* disp;
  int16_t* wta_ref;
  int16_t* wta_tar;
};

template <int RHO>
struct MatchGeom {
  static constexpr int NT = 2 * RHO + 1;
  static constexpr int CW = MF_TXT + 2 * RHO + MF_KD - 1;     // C_L columns (upper bound, D <= 8)
  static constexpr int VSW = CW + 2 * 7;                      // vertical-sum columns (P <= 7)
  static constexpr int GW = VSW + MF_KD - 1;                  // warped-image columns
  static constexpr int NRI = 2 * 7 + 2;                       // image ring rows (P <= 7)
  static constexpr int RC = MF_TXT + 2 * RHO;                 // reference window columns (128: the last 8 threads' pixels belong to the next strip)
  static constexpr int TC = MF_TXT + 2 * RHO;                 // target window columns
  static constexpr int NRG = NT;                              // guide / mask ring rows
  static constexpr int STW = 16;
  static constexpr size_t o_lut = 0;
  static constexpr size_t o_S = o_lut + 4 * MF_LUT * 32;
  static constexpr size_t o_Lr = o_S + 4 * NT * STW;
  static constexpr size_t o_Wr = o_Lr + 4 * NRI * VSW;
  static constexpr size_t o_VS = o_Wr + 4 * NRI * GW;
  static constexpr size_t o_CL = o_VS + 4 * VSW * MF_KD;
  static constexpr size_t o_R0 = o_CL + 4 * CW * MF_KD;
  static constexpr size_t o_T0 = o_R0 + 4 * RC * MF_KD;
  static constexpr size_t o_st = o_T0 + 4 * TC * MF_KD;        // SL, iL [CW]; SW, iW [CW + 7]
  static constexpr size_t o_g = o_st + 4 * (2 * CW + 2 * (CW + MF_KD));
  static constexpr size_t o_m = o_g + 4 * NRG * (RC + TC);
  static constexpr size_t o_kr = o_m + 4 * NRG * (RC + TC);
  static constexpr size_t o_gb = o_kr + 4 * MF_TXT;           // guide bytes of the next row [RC + TC]
  static constexpr size_t bytes = o_gb + 4 * (RC + TC);
};

template <int RHO>
__global__ void __launch_bounds__(MF_THREADS, 1) k_match_fused(const MatchArgs A) {
  using G = MatchGeom<RHO>;
  constexpr int NT = G::NT, RC = G::RC, TC = G::TC;
  extern __shared__ __align__(16) unsigned char mf_smem[];
  float* lut = reinterpret_cast<float*>(mf_smem + G::o_lut);
  float* S = reinterpret_cast<float*>(mf_smem + G::o_S);
  float* Lr = reinterpret_cast<float*>(mf_smem + G::o_Lr);
  float* Wr = reinterpret_cast<float*>(mf_smem + G::o_Wr);
  float* VS = reinterpret_cast<float*>(mf_smem + G::o_VS);
  float* CL = reinterpret_cast<float*>(mf_smem + G::o_CL);
  float* R0 = reinterpret_cast<float*>(mf_smem + G::o_R0);
  float* T0 = reinterpret_cast<float*>(mf_smem + G::o_T0);
  float* st = reinterpret_cast<float*>(mf_smem + G::o_st);
  int* gring = reinterpret_cast<int*>(mf_smem + G::o_g);
  int* mring = reinterpret_cast<int*>(mf_smem + G::o_m);
  int* krow = reinterpret_cast<int*>(mf_smem + G::o_kr);
  int* gbuf = reinterpret_cast<int*>(mf_smem + G::o_gb);
  const int tid = threadIdx.x, lane = tid & 31;

  const int H = A.H, W = A.W, D = A.D, P = A.P;
  const int d_lo = A.d_lo, d_hi = d_lo + D - 1;
  const int nstrip = (W + MF_TXR - 1) / MF_TXR, nchunk = (H + A.R - 1) / A.R;
  int blk = blockIdx.x;
  const int strip = blk % nstrip;
  blk /= nstrip;
  const int chunk = blk % nchunk, b = blk / nchunk;
  const int x0 = strip * MF_TXR, xt0 = x0 - d_hi;
  const int ya = chunk * A.R, yb = min(H, ya + A.R);
  const size_t pix0 = (size_t)b * H * W;
  const int CW = MF_TXT + 2 * RHO + D - 1;        // C_L columns [xcl0, xcl0 + CW)
  const int xcl0 = x0 - RHO - (D - 1);
  const int VSW = CW + 2 * P;                      // vertical sums: columns xcl0 - P + c
  const int GW = VSW + D - 1;                      // warped image: columns gw0 + c
  const int gw0 = xcl0 - P - d_hi;
  const int NRI = 2 * P + 2;
  const int NR = (yb - ya) + 2 * RHO;
  const float nf = (float)((2 * P + 1) * (2 * P + 1));

  // ---- tables (as aggregate_small.cu / aggregate_slide.cu) ----
  for (int e = tid; e < MF_LUT * 32; e += MF_THREADS) {
    const int dg = e / 32 - 255;
    lut[e] = (dg <= 255) ? ex2_ftz((float)(dg * dg) * A.kr) : 0.f;
  }
  for (int e = tid; e < NT * G::STW; e += MF_THREADS) {
    const int j = e / G::STW, a = e % G::STW;
    S[e] = a < NT ? ex2_ftz((float)((j - RHO) * (j - RHO) + (RHO - a) * (RHO - a)) * A.kd) : 0.f;
  }

  auto load_image_row = [&](int yy) {   // image row yy -> ring slot
    const int slot = ((yy % NRI) + NRI) % NRI;
    const bool rin = yy >= 0 && yy < H;
    for (int c = tid; c < VSW; c += MF_THREADS) {
      const int xx = xcl0 - P + c;
      Lr[slot * G::VSW + c] = (rin && xx >= 0 && xx < W) ? (float)A.ref[pix0 + (size_t)yy * W + xx] : 0.f;
    }
    for (int c = tid; c < GW; c += MF_THREADS) {
      const int xx = gw0 + c;
      Wr[slot * G::GW + c] = (rin && xx >= 0 && xx < W) ? (float)A.warped[pix0 + (size_t)yy * W + xx] : 0.f;
    }
  };

  // thread roles in the aggregation: tid < 128 target column xt0 + tid, else reference
  // column x0 + (tid - 128)
  const bool is_tar = tid < MF_TXT;
  const int col = is_tar ? tid : tid - MF_TXT;
  const int xg = is_tar ? xt0 + col : x0 + col;          // image column of the thread's pixels
  const uint8_t* guide = is_tar ? A.warped : A.ref;

  float2 acc[NT][4];
  float den[NT];
  int gp[NT], vor[NT], cen[NT];
#pragma unroll
  for (int a = 0; a < NT; a++) {
#pragma unroll
    for (int q = 0; q < 4; q++) acc[a][q] = make_float2(0.f, 0.f);
    den[a] = 0.f;
    vor[a] = 0;
    cen[a] = 0xFF;
    const int ya_ = ya - 2 * RHO + a;   // output row of age a at input row 0
    gp[a] = (ya_ >= 0 && ya_ < H && xg >= 0 && xg < W) ? (int)guide[pix0 + (size_t)ya_ * W + xg] : 0;
  }
  // vertical-sum items of this thread: e = tid + 256 u -> (column e / 8, k = e % 8)
  constexpr int NVS = (G::VSW * MF_KD + MF_THREADS - 1) / MF_THREADS;
  float vs[NVS];
#pragma unroll
  for (int u = 0; u < NVS; u++) vs[u] = 0.f;

  // ---- row inputs, prefetched one row ahead into registers (issued before row i's
  // aggregation, committed to shared memory at the start of row i + 1): the image row
  // entering the NCC window, the block statistics and the guide bytes of the row ----
  const int NIMG = VSW + GW;                        // L then W entries
  const int NSTA = 2 * CW + 2 * (CW + D - 1);       // S_L, inv_L, S_W, inv_W
  const int NGUI = RC + TC;
  constexpr int PFI = (G::VSW + G::GW + MF_THREADS - 1) / MF_THREADS;
  constexpr int PFS = (4 * G::CW + 2 * MF_KD + MF_THREADS - 1) / MF_THREADS;
  constexpr int PFG = (RC + TC + MF_THREADS - 1) / MF_THREADS;
  uint32_t pfi[PFI], pfs[PFS], pfg[PFG];
  auto fetch_rows = [&](int yimg, int ystat) {   // yimg < -1000: no image row
#pragma unroll
    for (int u = 0; u < PFI; u++) {
      const int e = tid + u * MF_THREADS;
      uint32_t v = 0u;
      if (e < NIMG && yimg >= 0 && yimg < H) {
        const bool isL = e < VSW;
        const int xx = isL ? xcl0 - P + e : gw0 + (e - VSW);
        if (xx >= 0 && xx < W) v = isL ? A.ref[pix0 + (size_t)yimg * W + xx] : A.warped[pix0 + (size_t)yimg * W + xx];
      }
      pfi[u] = v;
    }
    const bool rin = ystat >= 0 && ystat < H;
#pragma unroll
    for (int u = 0; u < PFS; u++) {
      const int e = tid + u * MF_THREADS;
      uint32_t v = 0u;
      if (e < NSTA) {
        // [0, CW) S_L, [CW, 2 CW) inv_L, [2 CW, 3 CW + D - 1) S_W, then inv_W
        const bool isL = e < 2 * CW;
        const int ee = isL ? e : e - 2 * CW;
        const int per = isL ? CW : CW + D - 1;
        const bool isInv = ee >= per;
        const int xx = (isL ? xcl0 : xcl0 - d_hi) + (isInv ? ee - per : ee);
        const bool in = rin && xx >= 0 && xx < W;
        const size_t g = pix0 + (size_t)ystat * W + xx;
        if (isInv) v = in ? __float_as_uint(isL ? A.iL[g] : A.iW[g]) : 0x7fffffffu;
        else v = in ? __float_as_uint((float)(isL ? A.SL[g] : A.SW[g])) : 0u;
      }
      pfs[u] = v;
    }
#pragma unroll
    for (int u = 0; u < PFG; u++) {
      const int e = tid + u * MF_THREADS;
      uint32_t v = 0u;
      if (e < NGUI && rin) {
        const bool tar = e >= RC;
        const int xx = (tar ? xt0 : x0) - RHO + (tar ? e - RC : e);
        if (xx >= 0 && xx < W) v = (tar ? A.warped : A.ref)[pix0 + (size_t)ystat * W + xx];
      }
      pfg[u] = v;
    }
  };
  auto commit_rows = [&](int yimg) {
    if (yimg > -1000) {
      const int slot = ((yimg % NRI) + NRI) % NRI;
#pragma unroll
      for (int u = 0; u < PFI; u++) {
        const int e = tid + u * MF_THREADS;
        if (e < VSW) Lr[slot * G::VSW + e] = (float)pfi[u];
        else if (e < NIMG) Wr[slot * G::GW + (e - VSW)] = (float)pfi[u];
      }
    }
#pragma unroll
    for (int u = 0; u < PFS; u++) {
      const int e = tid + u * MF_THREADS;
      if (e < NSTA) st[e] = __uint_as_float(pfs[u]);
    }
#pragma unroll
    for (int u = 0; u < PFG; u++) {
      const int e = tid + u * MF_THREADS;
      if (e < NGUI) gbuf[e] = (int)pfg[u];
    }
  };

  // prologue: image rows (ya - RHO) - P .. (ya - RHO) + P, statistics and guide of row 0
  for (int t = -P; t < P; t++) load_image_row(ya - RHO + t);
  fetch_rows(ya - RHO + P, ya - RHO);
  commit_rows(ya - RHO + P);
  __syncthreads();

  for (int i = 0; i < NR; i++) {
    const int yin = ya - RHO + i;
    // guide value of the output row entering as the oldest age at the end of this row:
    // loaded now, used after the row (latency hidden)
    int gp_next;
    {
      const int yn = yin + RHO + 1;
      gp_next = (yn >= 0 && yn < H && xg >= 0 && xg < W) ? (int)guide[pix0 + (size_t)yn * W + xg] : 0;
    }
    // ---- N1: commit the prefetched image row yin + P, statistics and guide of row yin ----
    if (i > 0) {
      commit_rows(yin + P);
      __syncthreads();
    }
    // ---- N2: exact vertical dot sums over rows yin - P .. yin + P ----
#pragma unroll
    for (int u = 0; u < NVS; u++) {
      const int e = tid + MF_THREADS * u;
      const int c = e / MF_KD, k = e % MF_KD;
      if (c < VSW) {
        const int wc = c + (D - 1) - k;     // warped column xcl0 - P + c - (d_lo + k), rel. gw0
        RSR_CHECK(k >= D || (wc >= 0 && wc < GW && c < G::VSW));
        float v = vs[u];
        if (k < D) {
          if (i == 0) {
            v = 0.f;
            for (int t = -P; t <= P; t++) {
              const int slot = (((yin + t) % NRI) + NRI) % NRI;
              v = fmaf(Lr[slot * G::VSW + c], Wr[slot * G::GW + wc], v);
            }
          } else {
            const int sn = (((yin + P) % NRI) + NRI) % NRI, so = (((yin - P - 1) % NRI) + NRI) % NRI;
            v = fmaf(-Lr[so * G::VSW + c], Wr[so * G::GW + wc], v);
            v = fmaf(Lr[sn * G::VSW + c], Wr[sn * G::GW + wc], v);
          }
        }
        vs[u] = v;
        VS[c * MF_KD + k] = v;
      }
    }
    __syncthreads();
    // ---- N3: horizontal sums and K2's normalisation -> C_L row ----
    for (int e = tid; e < CW * MF_KD; e += MF_THREADS) {
      const int c = e / MF_KD, k = e % MF_KD;
      float cv = qnan();
      if (k < D) {
        RSR_CHECK(c + 2 * P < VSW && c + (D - 1) - k < CW + D - 1);
        float hs = VS[c * MF_KD + k];
        for (int dx = 1; dx <= 2 * P; dx++) hs += VS[(c + dx) * MF_KD + k];
        const float sF = st[c], iF = st[CW + c];
        const int wc = c + (D - 1) - k;
        const float sG = st[2 * CW + wc], iG = st[2 * CW + (CW + D - 1) + wc];
        // n S_lw - S_l S_w as in zncc.cu (error-free S_l S_w, one FMA), then (num * inv_L) * inv_W
        const float bb = sF * sG;
        const float be = fmaf(sF, sG, -bb);
        const float num = fmaf(nf, hs, -bb) - be;
        cv = clamp_unit_nan((num * iF) * iG);
      }
      CL[e] = cv;
    }
    __syncthreads();
    // ---- N4: NaN-free reference / sheared target rows, masks, guide codes ----
    const int gslot = i % G::NRG;
    for (int c = tid; c < RC + TC; c += MF_THREADS) {
      const bool tar = c >= RC;
      const int cc = tar ? c - RC : c;
      // reference column x0 - RHO + cc <-> C_L index cc + D - 1; target column
      // xt0 - RHO + cc <-> C_L index cc + k (the shear)
      float v[MF_KD];
      int nanm = 0;
#pragma unroll
      for (int k = 0; k < MF_KD; k++) {
        RSR_CHECK(k >= D || (tar ? cc + k : cc + D - 1) < CW);
        v[k] = k < D ? CL[(tar ? cc + k : cc + D - 1) * MF_KD + k] : qnan();
        if (!(v[k] == v[k])) nanm |= 1 << k;
      }
      const int xx = (tar ? xt0 : x0) - RHO + cc;
      const bool skip = (nanm & ((1 << D) - 1)) == ((1 << D) - 1) || yin < 0 || yin >= H || xx < 0 || xx >= W;
      float* d = (tar ? T0 : R0) + cc * MF_KD;
#pragma unroll
      for (int k = 0; k < MF_KD; k++) d[k] = (skip || (nanm >> k & 1)) ? 0.f : v[k];
      gring[gslot * (RC + TC) + c] = skip ? MF_SKIPQ : gbuf[c];
      // NaN bits (k < D) of a non-skipped pixel (bit 8 marks a skipped one)
      mring[gslot * (RC + TC) + c] = skip ? 0x100 : (nanm & ((1 << D) - 1));
    }
    __syncthreads();
    // next row's inputs in flight during the aggregation
    if (i + 1 < NR) fetch_rows(yin + 1 + P, yin + 1);
    // ---- A: sliding aggregation of the thread's column ----
    const int gbase = gslot * (RC + TC) + (is_tar ? RC + col : col);
    RSR_CHECK(col + NT - 1 < (is_tar ? TC : RC) && gslot < G::NRG);
    const float* crow = (is_tar ? T0 : R0) + col * MF_KD;
    {
      // window mask of this input row: OR of the NaN bits of the 2 rho + 1 taps
      int hm = 0;
#pragma unroll
      for (int j = 0; j < NT; j++) hm |= mring[gbase + j] & 0xFF;
      // centre NaN bits of the output row entering at age RHO (output row yin)
      {
        const int mc = mring[gbase + RHO];
        cen[RHO] = (mc & 0x100) ? 0xFF : mc;
      }
#pragma unroll
      for (int a = 0; a < NT; a++) vor[a] |= hm;
    }
    float2 fin[4];
    float fden = 0.f;
#pragma unroll
    for (int j = 0; j < NT; j++) {
      const float4 ca = *reinterpret_cast<const float4*>(crow + j * MF_KD);
      const float4 cb = *reinterpret_cast<const float4*>(crow + j * MF_KD + 4);
      const float2 cp[4] = {make_float2(ca.x, ca.y), make_float2(ca.z, ca.w), make_float2(cb.x, cb.y),
                            make_float2(cb.z, cb.w)};
      const int gq = gring[gbase + j];
#pragma unroll
      for (int a4 = 0; a4 < (NT + 3) / 4; a4++) {
        const float4 s4 = *reinterpret_cast<const float4*>(S + j * G::STW + 4 * a4);
        const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const int a = 4 * a4 + t;
          if (a < NT) {
            const int idx = min(gq - gp[a] + 255, MF_LUT - 1);
            const float w = sv[t] * lut[idx * 32 + lane];
            if (j < NT - 1) {
              den[a] += w;
#pragma unroll
              for (int q = 0; q < 4; q++) acc[a][q] = f2fma(make_float2(w, w), cp[q], acc[a][q]);
            } else if (a == 0) {
              fden = den[0] + w;
#pragma unroll
              for (int q = 0; q < 4; q++) fin[q] = f2fma(make_float2(w, w), cp[q], acc[0][q]);
            } else {
              den[a - 1] = den[a] + w;
#pragma unroll
              for (int q = 0; q < 4; q++) acc[a - 1][q] = f2fma(make_float2(w, w), cp[q], acc[a][q]);
            }
          }
        }
      }
    }
    // ---- W: completion of output row y = yin - RHO (age 0) ----
    const int y = yin - RHO;
    const bool out_row = y >= ya;
    float Av[MF_KD];
    int kbest = -1;
    if (out_row) {
      const float f8[8] = {fin[0].x, fin[0].y, fin[1].x, fin[1].y, fin[2].x, fin[2].y, fin[3].x, fin[3].y};
      const float inv = rcp_fast(fden);
      const int M = vor[0], cz = cen[0];
      const int gp0 = gp[0];
#pragma unroll
      for (int k = 0; k < MF_KD; k++) {
        float a = qnan();
        if (k < D && !((cz >> k) & 1)) {
          if (!((M >> k) & 1)) {
            a = f8[k] * inv;
          } else {
            // exact denominator: sum of w * validity in (input row, tap) order
            float dk = 0.f;
            for (int t = 0; t < NT; t++) {
              const int rb = ((i - 2 * RHO + t) % G::NRG + G::NRG) % G::NRG * (RC + TC) + (is_tar ? RC + col : col);
              const int aa = 2 * RHO - t;
              for (int j = 0; j < NT; j++) {
                const int gq = gring[rb + j];
                const int mq = mring[rb + j];
                const float w = S[j * G::STW + aa] * lut[min(gq - gp0 + 255, MF_LUT - 1) * 32 + lane];
                const float vv = ((mq & 0x100) || ((mq >> k) & 1)) ? 0.f : 1.f;
                dk = fmaf(w, vv, dk);
              }
            }
            a = f8[k] * rcp_fast(dk);
          }
        }
        Av[k] = a;
      }
      // WTA: smallest k of the maximum over non-NaN entries (K4's rule)
      float best = -INFINITY;
#pragma unroll
      for (int k = 0; k < MF_KD; k++)
        if (Av[k] > best) { best = Av[k]; kbest = k; }
      if (is_tar) {
        krow[col] = kbest;
        const int own = col - d_hi;   // this strip's own target columns: x0 .. x0 + 119
        if (A.wta_tar && own >= 0 && own < MF_TXR && xg < W) A.wta_tar[pix0 + (size_t)y * W + xg] = (int16_t)kbest;
      }
    }
    // age shift of the bookkeeping (the accumulators shifted inside the last tap)
#pragma unroll
    for (int q = 0; q < 4; q++) acc[NT - 1][q] = make_float2(0.f, 0.f);
    den[NT - 1] = 0.f;
#pragma unroll
    for (int a = 0; a + 1 < NT; a++) {
      gp[a] = gp[a + 1];
      vor[a] = vor[a + 1];
      cen[a] = cen[a + 1];
    }
    gp[NT - 1] = gp_next;   // output row yin + RHO + 1 enters as the oldest age
    vor[NT - 1] = 0;
    cen[NT - 1] = 0xFF;
    __syncthreads();   // k_R of row y in shared memory
    if (out_row && !is_tar && col < MF_TXR && xg < W) {
      const size_t o = pix0 + (size_t)y * W + xg;
      if (A.wta_ref) A.wta_ref[o] = (int16_t)kbest;
      float d = qnan();
      if (kbest >= 0) {
        const int up = xg - (kbest + d_lo);
        if (up >= 0 && up < W) {
          RSR_CHECK(up - xt0 >= 0 && up - xt0 < MF_TXT);
          const int kr = krow[up - xt0];
          if (kr >= 0 && abs(kbest - kr) <= A.lrc_tol) {
            float r = (float)(kbest + d_lo);
            if (A.subpix && kbest >= 1 && kbest <= D - 2) {
              float a = 0.f, bb = 0.f, c = 0.f;
#pragma unroll
              for (int k = 0; k < MF_KD; k++) {
                if (k == kbest - 1) a = Av[k];
                if (k == kbest) bb = Av[k];
                if (k == kbest + 1) c = Av[k];
              }
              const float den2 = 2.f * a + 2.f * c - 4.f * bb;
              if (!(a != a) && !(c != c) && fabsf(den2) > 1e-12f) r += __fdiv_rn(a - c, den2);
            }
            d = r + (float)A.shift[(size_t)b * H + y];
          }
        }
      }
      A.disp[o] = d;
    }
  }
}

template <int RHO>
static cudaError_t match_launch_t(const MatchArgs& A0, cudaStream_t st) {
  using G = MatchGeom<RHO>;
  MatchArgs A = A0;
  const int nstrip = (A.W + MF_TXR - 1) / MF_TXR;
  int nsm = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // rows per CTA: minimise waves x (R + 2 rho) at one CTA per SM
  const long long cols = (long long)nstrip * A.B;
  int bestR = A.H;
  double best = 1e300;
  for (int n = 1; n <= A.H; n++) {
    const int R = (A.H + n - 1) / n;
    if (R < 16 && n > 1) break;
    const long long ctas = cols * ((A.H + R - 1) / R);
    const double c = (double)((ctas + nsm - 1) / nsm) * (R + 2 * RHO + 2 * A.P);
    if (c < best * 0.999) { best = c; bestR = R; }
  }
  A.R = bestR;
  const long long nblk = cols * ((A.H + bestR - 1) / bestR);
  if (nblk > 0x7fffffffLL) return cudaErrorInvalidValue;
  cudaError_t e = smem_optin((const void*)k_match_fused<RHO>, G::bytes);
  if (e != cudaSuccess) return e;
  k_match_fused<RHO><<<(unsigned)nblk, MF_THREADS, G::bytes, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_match_fused(int B, int H, int W, int rho_b, int d_lo, int D, int rho, float gamma_d,
                               float gamma_r, int lrc_tol, int subpix, const uint8_t* ref, const uint8_t* warped,
                               const int32_t* shift, const int32_t* SL, const float* iL, const int32_t* SW,
                               const float* iW, float* disp, int16_t* wta_ref, int16_t* wta_tar, cudaStream_t st) {
  if (D < 1 || D > MF_KD || rho_b < 1 || rho_b > 7) return cudaErrorInvalidValue;
  MatchArgs A;
  A.B = B; A.H = H; A.W = W; A.D = D; A.d_lo = d_lo; A.P = rho_b; A.R = H;
  A.lrc_tol = lrc_tol; A.subpix = subpix;
  const float log2e = 1.4426950408889634f;
  A.kd = -log2e / (gamma_d * gamma_d);
  A.kr = std::isinf(gamma_r) ? -1e-30f : -log2e / (gamma_r * gamma_r);
  A.ref = ref; A.warped = warped; A.shift = shift;
  A.SL = SL; A.iL = iL; A.SW = SW; A.iW = iW;
  A.disp = disp; A.wta_ref = wta_ref; A.wta_tar = wta_tar;
#define RSR_MF(R) \
  case R: return match_launch_t<R>(A, st);
  switch (rho) {
    RSR_MF(0) RSR_MF(1) RSR_MF(2) RSR_MF(3) RSR_MF(4) RSR_MF(5) RSR_MF(6) RSR_MF(7)
    default:
      return cudaErrorInvalidValue;
  }
#undef RSR_MF
}

}  // namespace rsr
