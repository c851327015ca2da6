// K2 — NCC cost volumes (Eqs. (3)-(5)).
//
// c(u,v,r) = (n S_lw - S_l S_w) / (sqrt(n S_ll - S_l^2) sqrt(n S_ww - S_w^2)),
// the integer-sum form of Eq. (3) with Eqs. (4)-(5) (multiply numerator and
// denominator of Eq. (3) by n).  As P:106 prescribes, the block statistics
// (mu, sigma) are computed once per pixel ("pre-calculated and stored") by
// k_block_stats, and only the dot product S_lw is per-disparity work.
//
// k_zncc keeps S_lw exact: every product i_l * i_w <= 65025 and every partial
// sum of at most 225 of them is an integer below 2^24, so fp32 FFMA arithmetic
// is exact.  Each thread owns X=4 columns x R=8 disparities and slides the
// vertical sums V(x, r) = sum_dy F(y+dy, x) G(y+dy, x -/+ r) down a band of
// BY=16 rows (two FFMAs per (x, r) per row), then forms the horizontal
// (2p+1)-sums in registers.  The numerator n*S_lw - S_l*S_w is evaluated with
// an error-free product split (fmaf remainder) so catastrophic cancellation
// cannot lose the result; one fp32 normalisation per entry remains, which is
// the only difference from the fp64 oracle (|dc| ~ 1e-7).
//
// Output layout [B][H][W][D]: the thread's 8 disparities of one pixel are 32
// contiguous bytes (two 16-byte stores); 8 lanes cover one pixel's 64 k.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

// ---------------------------------------------------------------------------
// Block statistics: S = sum i, inv = 1/sqrt(n*sum i^2 - S^2) over the
// (2p+1)^2 block centred at each pixel; inv = NaN if the block leaves the
// image, holds mask == 0 (warp-invalid, reading 7) or is constant
// (exact integer test, reading 6).
// ---------------------------------------------------------------------------
constexpr int ST_TX = 64, ST_TY = 32;   // 32 rows: 47 KB of shared memory at p = 3 (< 48 KB)

// Both images in one grid: frames [0, B) are img0 (mask0, S0, inv0), [B, 2B) img1.
// img0 is uint8 (the reference image); img1 is uint8 or, for the interpolating
// warp (NEXT f2), the 8.8 fixed-point warped image (uint16): sums of squares then
// need int64 (225 * 65280^2 > 2^31).
// FOUT (the streaming NCC kernel's inputs): S is stored as fp32 (exact: < 2^24) and
// each image is also written as an fp32 plane (img0 -> F0, img1 -> F1), so that
// k_zncc can stage its rows with 4-byte cp.async copies and no conversion.
template <int p, typename T1, bool FOUT = false>
__global__ void __launch_bounds__(256) k_block_stats(int B, int H, int W,
                                                     const uint8_t* __restrict__ img0,
                                                     const uint8_t* __restrict__ mask0,
                                                     int32_t* __restrict__ S0, float* __restrict__ inv0,
                                                     const T1* __restrict__ img1,
                                                     const uint8_t* __restrict__ mask1,
                                                     int32_t* __restrict__ S1, float* __restrict__ inv1,
                                                     float* __restrict__ F0 = nullptr,
                                                     float* __restrict__ F1 = nullptr) {
  using SST = typename std::conditional<sizeof(T1) == 1, int, long long>::type;
  const bool second = (int)blockIdx.z >= B;
  const uint8_t* __restrict__ mask = second ? mask1 : mask0;
  int32_t* __restrict__ Sout = second ? S1 : S0;
  float* __restrict__ inv = second ? inv1 : inv0;
  float* __restrict__ Fout = second ? F1 : F0;
  extern __shared__ __align__(16) unsigned char st_raw[];
  const int TC = ST_TX + 2 * p, TR = ST_TY + 2 * p;
  SST* cSS = reinterpret_cast<SST*>(st_raw);         // [ST_TY][TC] vertical sums of squares
  int* pix = reinterpret_cast<int*>(cSS + ST_TY * TC);  // [TR][TC] value
  int* msk = pix + TR * TC;          // [TR][TC] mask (1 inside image and valid)
  int* cS = msk + TR * TC;           // [ST_TY][TC] vertical sums
  int* cM = cS + ST_TY * TC;
  const int b = second ? (int)blockIdx.z - B : (int)blockIdx.z, x0 = blockIdx.x * ST_TX, y0 = blockIdx.y * ST_TY;
  const size_t base = (size_t)b * H * W;
  constexpr int UNR = 8;   // independent loads in flight per thread
  for (int i0 = threadIdx.x; i0 < TR * TC; i0 += UNR * blockDim.x) {
    int pv[UNR], mv[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int i = i0 + u * blockDim.x;
      const int yy = y0 - p + i / TC, xx = x0 - p + i % TC;
      const bool in = i < TR * TC && yy >= 0 && yy < H && xx >= 0 && xx < W;
      const size_t g = base + (size_t)yy * W + xx;
      pv[u] = in ? (second ? (int)__ldg(img1 + g) : (int)__ldg(img0 + g)) : 0;
      mv[u] = in ? (mask ? (int)(__ldg(mask + g) != 0) : 1) : 0;
    }
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int i = i0 + u * blockDim.x;
      if (i < TR * TC) { pix[i] = pv[u]; msk[i] = mv[u]; }
    }
  }
  __syncthreads();
  // vertical (2p+1)-sums: one (row, column) item per thread iteration, all threads busy
  constexpr int K = 2 * p + 1;
  for (int it = threadIdx.x; it < ST_TY * TC; it += blockDim.x) {
    const int y = it / TC, c = it % TC;
    int s = 0, m = 0;
    SST ss = 0;
#pragma unroll
    for (int r = 0; r < K; r++) {
      const int v = pix[(y + r) * TC + c];
      s += v; ss += (SST)v * v; m += msk[(y + r) * TC + c];
    }
    cS[it] = s; cSS[it] = ss; cM[it] = m;
  }
  __syncthreads();
  // horizontal (2p+1)-sums: one output pixel per thread iteration (coalesced stores)
  const int n = K * K;
  for (int it = threadIdx.x; it < ST_TY * ST_TX; it += blockDim.x) {
    const int y = it / ST_TX, x = it % ST_TX;
    const int yy = y0 + y, xx = x0 + x;
    if (yy >= H || xx >= W) continue;
    int s = 0, m = 0;
    long long ss = 0;
#pragma unroll
    for (int d = 0; d < K; d++) {
      s += cS[y * TC + x + d]; ss += cSS[y * TC + x + d]; m += cM[y * TC + x + d];
    }
    const bool inside = yy >= p && yy <= H - 1 - p && xx >= p && xx <= W - 1 - p;
    // exact integer variance (int64: n * sum(i^2) reaches 3.3e9 at p = 7 for uint8 and
    // 2.2e14 for 8.8 fixed point); its fp32 rounding and MUFU.RSQ stay ~1e-7
    // relative, far inside the ZNCC tolerance
    const long long var = (long long)n * ss - (long long)s * s;
    const bool ok = inside && m == n && var != 0;
    const size_t g = base + (size_t)yy * W + xx;
    if (FOUT) {
      reinterpret_cast<float*>(Sout)[g] = (float)s;
      Fout[g] = (float)pix[(y + p) * TC + x + p];
    } else {
      Sout[g] = s;
    }
    inv[g] = ok ? rsqrtf((float)var) : qnan();
  }
}

// Column-sliding block statistics for rsr_cost_volume (uint8 images, fp32 outputs as
// in k_block_stats<FOUT>, same integers and the same single rounding per value).  A
// thread owns one tile column and slides the vertical (2P+1)-sums of i, i^2 and the
// mask down BS_BY output rows (the entering row prefetched one row ahead, the leaving
// row re-read from L1); per output row the vertical sums go to
// a double-buffered shared row and the horizontal (2P+1)-sums are read back: one CTA
// barrier per row, one 8-byte load per tap.  Frames [0, B) are img0, [B, 2B) img1.
constexpr int BS_BX = 128, BS_BY = 48;

template <int P>
__global__ void __launch_bounds__(160) k_block_stats_col(int B, int H, int W,
                                                         const uint8_t* __restrict__ img0,
                                                         const uint8_t* __restrict__ mask0, float* __restrict__ S0,
                                                         float* __restrict__ inv0, float* __restrict__ F0,
                                                         const uint8_t* __restrict__ img1,
                                                         const uint8_t* __restrict__ mask1, float* __restrict__ S1,
                                                         float* __restrict__ inv1, float* __restrict__ F1) {
  constexpr int NR = 2 * P + 1, TC = BS_BX + 2 * P;
  static_assert(TC <= 160, "one thread per tile column");
  __shared__ int2 vs[2][TC];   // (S * 256 + M, S2): vertical sums of the tile columns
  __shared__ int cp[2][TC];    // centre pixel of the row
  const bool second = (int)blockIdx.z >= B;
  const int b = second ? (int)blockIdx.z - B : (int)blockIdx.z;
  const uint8_t* __restrict__ img = second ? img1 : img0;
  const uint8_t* __restrict__ mask = second ? mask1 : mask0;
  float* __restrict__ Sout = second ? S1 : S0;
  float* __restrict__ inv = second ? inv1 : inv0;
  float* __restrict__ Fout = second ? F1 : F0;
  const int t = threadIdx.x;
  const int x0 = blockIdx.x * BS_BX, y0 = blockIdx.y * BS_BY;
  const int xx = x0 - P + t;
  const bool col_in = t < TC && xx >= 0 && xx < W;
  const size_t base = (size_t)b * H * W;
  auto load = [&](int yy, int& pv, int& mv) {
    pv = 0; mv = 0;
    if (col_in && yy >= 0 && yy < H) {
      const size_t g = base + (size_t)yy * W + xx;
      pv = __ldg(img + g);
      mv = mask ? (__ldg(mask + g) != 0) : 1;
    }
  };
  int vs1 = 0, vs2 = 0, vm = 0;
  for (int k = 0; k < NR - 1; k++) {   // rows y0 - P .. y0 + P - 1
    int pv, mv;
    load(y0 - P + k, pv, mv);
    vs1 += pv; vs2 += pv * pv; vm += mv;
  }
  int np, nm;
  load(y0 + P, np, nm);
  const int yend = min(H, y0 + BS_BY);
  const int n = NR * NR;
  // (entering rows prefetched 6 rows ahead through a register ring measured slower:
  // 131 vs 104 us per c5 batch)
  for (int yc = y0; yc < yend; yc++) {
    // the entering row yc + P was prefetched; the leaving row yc - P and the centre
    // row yc are re-read (L1 hits: loaded 2P + 1 and P rows ago)
    int op, om, cpv, cmv;
    load(yc - P, op, om);
    load(yc, cpv, cmv);
    vs1 += np; vs2 += np * np; vm += nm;
    load(yc + P + 1, np, nm);                // prefetch the next entering row
    const int buf = yc & 1;
    if (t < TC) {
      vs[buf][t] = make_int2(vs1 * 256 + vm, vs2);
      cp[buf][t] = cpv;
    }
    vs1 -= op; vs2 -= op * op; vm -= om;
    __syncthreads();
    const int xo = x0 + t;
    if (t < BS_BX && xo < W) {
      int a = 0, s2 = 0;
#pragma unroll
      for (int d = 0; d < NR; d++) {
        const int2 v = vs[buf][t + d];
        a += v.x; s2 += v.y;
      }
      const int s1 = a >> 8, m = a & 255;
      const bool inside = yc >= P && yc <= H - 1 - P && xo >= P && xo <= W - 1 - P;
      const long long var = (long long)n * s2 - (long long)s1 * s1;
      const bool ok = inside && m == n && var != 0;
      const size_t g = base + (size_t)yc * W + xo;
      Sout[g] = (float)s1;
      inv[g] = ok ? rsqrtf((float)var) : qnan();
      Fout[g] = (float)cp[buf][t + P];
    }
  }
}

template <typename T1, bool FOUT = false>
static cudaError_t block_stats_t(int B, int H, int W, int rho_b, const uint8_t* img0, const uint8_t* mask0,
                                 int32_t* S0, float* inv0, const T1* img1, const uint8_t* mask1, int32_t* S1,
                                 float* inv1, cudaStream_t st, float* F0 = nullptr, float* F1 = nullptr) {
  using SST = typename std::conditional<sizeof(T1) == 1, int, long long>::type;
  const int p = rho_b;
  const int TC = ST_TX + 2 * p, TR = ST_TY + 2 * p;
  const size_t smem = sizeof(int) * (size_t)(2 * TR * TC + 2 * ST_TY * TC) + sizeof(SST) * (size_t)ST_TY * TC;
  const int nimg = img1 ? 2 : 1;
  if ((long long)nimg * B > 65535) return cudaErrorInvalidValue;
  dim3 grid((W + ST_TX - 1) / ST_TX, (H + ST_TY - 1) / ST_TY, nimg * B);
  switch (p) {
#define RSR_BS(PP)                                                                              \
  case PP: {                                                                                    \
    const cudaError_t e = smem_optin((const void*)k_block_stats<PP, T1, FOUT>, smem);          \
    if (e != cudaSuccess) return e;                                                             \
    k_block_stats<PP, T1, FOUT><<<grid, 256, smem, st>>>(B, H, W, img0, mask0, S0, inv0, img1, mask1, S1, \
                                                         inv1, F0, F1);                         \
    break;                                                                                      \
  }
    RSR_BS(1) RSR_BS(2) RSR_BS(3) RSR_BS(4) RSR_BS(5) RSR_BS(6) RSR_BS(7)
#undef RSR_BS
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_block_stats(int B, int H, int W, int rho_b, const uint8_t* img0, const uint8_t* mask0,
                               int32_t* S0, float* inv0, const uint8_t* img1, const uint8_t* mask1, int32_t* S1,
                               float* inv1, cudaStream_t st) {
  return block_stats_t<uint8_t>(B, H, W, rho_b, img0, mask0, S0, inv0, img1, mask1, S1, inv1, st);
}

cudaError_t launch_block_stats_f(int B, int H, int W, int rho_b, const uint8_t* img0, const uint8_t* mask0,
                                 float* S0, float* inv0, float* F0, const uint8_t* img1, const uint8_t* mask1,
                                 float* S1, float* inv1, float* F1, cudaStream_t st) {
  if (const char* e = getenv("RSR_BS_TILE"); e && e[0] == '1')   // A/B hook (tools/): the tiled kernel
    return block_stats_t<uint8_t, true>(B, H, W, rho_b, img0, mask0, reinterpret_cast<int32_t*>(S0), inv0, img1,
                                        mask1, reinterpret_cast<int32_t*>(S1), inv1, st, F0, F1);
  const int nimg = img1 ? 2 : 1;
  if ((long long)nimg * B > 65535) return cudaErrorInvalidValue;
  dim3 grid((W + BS_BX - 1) / BS_BX, (H + BS_BY - 1) / BS_BY, nimg * B);
  switch (rho_b) {
#define RSR_BSC(PP)                                                                                       \
  case PP:                                                                                                \
    k_block_stats_col<PP><<<grid, 160, 0, st>>>(B, H, W, img0, mask0, S0, inv0, F0, img1, mask1, S1, inv1, F1); \
    break;
    RSR_BSC(1) RSR_BSC(2) RSR_BSC(3) RSR_BSC(4) RSR_BSC(5) RSR_BSC(6) RSR_BSC(7)
#undef RSR_BSC
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_block_stats16(int B, int H, int W, int rho_b, const uint8_t* img0, int32_t* S0, float* inv0,
                                 const uint16_t* img1, const uint8_t* mask1, int32_t* S1, float* inv1,
                                 cudaStream_t st) {
  return block_stats_t<uint16_t>(B, H, W, rho_b, img0, nullptr, S0, inv0, img1, mask1, S1, inv1, st);
}

// ---------------------------------------------------------------------------
// NCC volume kernel (streaming).  A CTA owns ZTX = 64 columns x all D (up to
// 128) disparities and slides down ZBY rows.  Image rows and the block
// statistics of the current output row stream through a small shared-memory
// ring: every iteration first issues 4-byte cp.async copies (fp32 planes from
// k_block_stats<FOUT>) of the rows needed two iterations later, straight into
// their oriented ring slots, then computes the current row, so the copy latency
// overlaps the math and no thread spends instructions on conversion or commits.
// ---------------------------------------------------------------------------
constexpr int ZX = 4;     // columns per thread
constexpr int ZR = 8;     // disparities per thread (4 packed pairs)
constexpr int ZTX = 64;   // columns per CTA (16 column groups) for D > 16
// Small search ranges (D <= 16, e.g. the restricted band of P:251) use ZT = 256
// columns per CTA so that the 128 threads stay busy (one disparity group of 8 per
// column group of 4: 64 column groups x up to 2 disparity groups).
constexpr int ZT_SMALL = 256;
// (a 128-column CTA for 16 < D <= 32 was measured slower at the paper's D = 30:
// 1.64 vs 1.47 ms per 8 cP frames)
constexpr int ZT_MID = 128;
#ifdef RSR_K2_MID   // experiment build (tools/): 128-column CTAs for 16 < D <= 32
__host__ __device__ constexpr int zncc_cta_cols(int D) { return D <= 16 ? ZT_SMALL : (D <= 32 ? ZT_MID : ZTX); }
#else
__host__ __device__ constexpr int zncc_cta_cols(int D) { return D <= 16 ? ZT_SMALL : ZTX; }
#endif
constexpr int ZBY = 72;   // output rows per CTA (measured: 72 beats 48/60/80/90/96/144 at c5)

// Shared-memory rows are stored "oriented": the G-side image row and G-side
// statistics run so that, for a thread, the G entry of disparity q + 1 follows
// the one of disparity q (reference volume: G = W at u - r, stored reversed;
// target volume: G = L at u' + r, stored forward).  Each oriented row also has
// a copy shifted by one entry, so that a (q, q+1) pair starting at an odd
// index is still an aligned register pair: every packed operand is one LDS.
struct ZnccGeom {
  int FC, GC, SGC, gpad, NRING, GROW, SROW2, RB, RS;
};

__host__ __device__ inline ZnccGeom zncc_geom(int p, int D, int ZTX = rsr::ZTX) {
  ZnccGeom g;
  const int NJ = ZX + 2 * p;
  // image rows y-1 .. y+2p being read, row y+2p+1 in flight (issued one iteration
  // earlier) and row y+2p+2 issued now into the slot of y-2 (last read one iteration
  // earlier): one barrier per row, copies issued two rows ahead
  g.NRING = 2 * p + 4;
  g.FC = ((ZTX + 2 * p + 3) / 4) * 4 + 4;
  g.gpad = (4 - (D & 3)) & 3;
  g.GC = ((ZTX + 2 * p + D - 1 + g.gpad + 3) / 4) * 4 + 8;
  g.SGC = ((ZTX + D - 1 + g.gpad + 3) / 4) * 4 + 8;
  // reversal origins (reference volume), chosen so the thread runs stay 16-byte aligned
  g.RB = g.GC - 1 + ((NJ + 6 - (g.GC - 1)) & 3);
  g.RS = g.SGC - 1 + ((ZX + ZR - 2 - (g.SGC - 1)) & 3);
  g.GROW = g.GC + 8;                                     // oriented G image row (+ shifted copy)
  g.SROW2 = g.SGC + 8;                                   // oriented G statistics row
  return g;
}

__host__ __device__ inline size_t zncc_smem(int p, int D, int ZTX = rsr::ZTX, bool shear = false) {
  const ZnccGeom g = zncc_geom(p, D, ZTX);
  // ring: F rows, oriented G rows x2; statistics triple buffer: sF, iF, sG x2, iG x2;
  // SHEAR: the reference tile of the row [ZTX][ZT_STR]
  return sizeof(float) * ((size_t)g.NRING * (g.FC + 2 * g.GROW) + 3 * (2 * ZTX + 4 * (size_t)g.SROW2) +
                          (shear ? (size_t)ZTX * 68 : 0));
}

// One CTA of the volume kernel for frame b (the kernels below pick b and TAR).
// SHEAR (reference CTAs only): the target volume is written from the reference
// tile by the shear identity of P:106, C_R[v][u'][k] = C_L[v][u' + d_lo + k][k]
// (NaN where u' + d_lo + k leaves the image): the row's reference costs are staged
// in a shared tile and copied out as contiguous per-pixel k-runs.  Bitwise the
// values the target CTAs would compute (same operations, see below), with half the
// NCC work.
constexpr int ZT_STR = 68;   // shared tile row stride (floats): conflict-free diagonal reads

template <int P, bool TAR, int ZTX = rsr::ZTX, bool SHEAR = false>
__device__ __forceinline__ void zncc_cta(int b, int H, int W, int d_lo, int D, int Dst, int koff,
                                              const float* __restrict__ ref,
                                              const float* __restrict__ warped,
                                              const float* __restrict__ SLg,
                                              const float* __restrict__ invLg,
                                              const float* __restrict__ SWg,
                                              const float* __restrict__ invWg,
                                              float* __restrict__ vol,
                                              float* __restrict__ vol_tar = nullptr) {
  static_assert(!(SHEAR && TAR), "the shear writes the target volume from reference CTAs");
  constexpr int NJ = ZX + 2 * P;          // V columns per thread
  constexpr int NQP = ZR / 2;             // disparity pairs per thread
  constexpr int NGR = NJ + ZR;            // oriented G run loaded per row (>= NJ + ZR - 1)
  constexpr int NF4 = (NJ + 3) / 4, NG4 = (NGR + 3) / 4;
  constexpr int NSR = ZX + ZR;            // oriented G-statistics run (>= ZX + ZR - 1)
  constexpr int NS4 = (NSR + 3) / 4;
  const ZnccGeom gm = zncc_geom(P, D, ZTX);
  extern __shared__ __align__(16) float zsm[];
  float* Fs = zsm;                                   // [NRING][FC]    F image rows
  float* Gs = Fs + gm.NRING * gm.FC;                 // [NRING][GROW]  oriented G image rows
  float* Gs1 = Gs + gm.NRING * gm.GROW;              // [NRING][GROW]  shifted by one entry
  float* St = Gs1 + gm.NRING * gm.GROW;              // [3][sF ZTX | iF ZTX | sG | sG1 | iG | iG1]
  const int SROW = 2 * ZTX + 4 * gm.SROW2;
  float* Tt = St + 3 * SROW;                         // SHEAR: [ZTX][ZT_STR] reference costs of the row
  constexpr int NRING = 2 * P + 4;

  const int x0 = blockIdx.x * ZTX, y0 = blockIdx.y * ZBY;
  const int d_hi = d_lo + D - 1;
  const size_t ibase = (size_t)b * H * W;
  // F = image at the fixed column; G = image at the shifted column x -/+ r.
  const float* Fimg = TAR ? warped : ref;
  const float* Gimg = TAR ? ref : warped;
  const float* SFg = TAR ? SWg : SLg;
  const float* iFg = TAR ? invWg : invLg;
  const float* SGg = TAR ? SLg : SWg;
  const float* iGg = TAR ? invLg : invWg;
  // first image column of the (unoriented) G image row / G statistics row
  const int g0 = TAR ? (x0 - P + d_lo) : (x0 - P - d_hi - gm.gpad);
  const int s0 = TAR ? (x0 + d_lo) : (x0 - d_hi - gm.gpad);
  const int nrows = min(ZBY, H - y0);
  // unoriented index c -> oriented index
  auto orient_g = [&](int c) { return TAR ? c : gm.RB - c; };
  auto orient_s = [&](int c) { return TAR ? c : gm.RS - c; };

  // ---- row streaming: 4-byte cp.async copies from the fp32 planes straight into the
  // ring (oriented, plus the one-entry-shifted copy); columns / rows outside the image
  // are filled (image and S: 0, norms: NaN).  Copies run two rows ahead of the math.
  // per-thread trip counts are compile-time upper bounds (P <= 7, the D this CTA width
  // serves: 64 for ZTX = 64, 32 for ZT_MID, 16 for ZT_SMALL); 128 threads per CTA
  constexpr int NTHR = 128;
  constexpr int DMAX = ZTX == 64 ? 64 : (ZTX == ZT_MID ? 32 : 16);
  constexpr int FCMAX = ((ZTX + 2 * P + 3) / 4) * 4 + 4;
  constexpr int GCMAX = ((ZTX + 2 * P + DMAX - 1 + 3 + 3) / 4) * 4 + 8;
  constexpr int SGCMAX = ((ZTX + DMAX - 1 + 3 + 3) / 4) * 4 + 8;
  constexpr int TF = (FCMAX + NTHR - 1) / NTHR, TG = (GCMAX + NTHR - 1) / NTHR;
  constexpr int TSF = 2 * ZTX / NTHR, TSG = (2 * SGCMAX + NTHR - 1) / NTHR;
  static_assert(2 * ZTX % NTHR == 0, "F statistics: whole trips");
  auto issue_img = [&](int t_img) {
    const int slot = t_img % NRING;
    const int yy = y0 - P + t_img;
    float* fs = Fs + slot * gm.FC;
    float* gs = Gs + slot * gm.GROW;
    float* gs1 = Gs1 + slot * gm.GROW;
    const bool row_in = yy >= 0 && yy < H;   // CTA-uniform
    const float* frow = Fimg + ibase + (size_t)(row_in ? yy : 0) * W;
    const float* grow = Gimg + ibase + (size_t)(row_in ? yy : 0) * W;
#pragma unroll
    for (int u = 0; u < TF; u++) {
      const int e = threadIdx.x + u * NTHR;
      const int xx = x0 - P + e;
      RSR_CHECK(slot < gm.NRING);
      if (e < gm.FC) {
        if (row_in && xx >= 0 && xx < W) cp_async4(fs + e, frow + xx);
        else fs[e] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < TG; u++) {
      const int c = threadIdx.x + u * NTHR;
      const int xx = g0 + c;
      const int o = orient_g(c);
      if (c < gm.GC) {
        RSR_CHECK(o >= 0 && o < gm.GROW);
        if (row_in && xx >= 0 && xx < W) {
          cp_async4(gs + o, grow + xx);
          if (o > 0) cp_async4(gs1 + o - 1, grow + xx);
        } else {
          gs[o] = 0.f;
          if (o > 0) gs1[o - 1] = 0.f;
        }
      }
    }
  };
  auto issue_stats = [&](int y_st) {
    float* st = St + (y_st % 3) * SROW;
    const size_t rowo = ibase + (size_t)(y0 + y_st) * W;   // y0 + y_st < H
#pragma unroll
    for (int u = 0; u < TSF; u++) {
      const int k = threadIdx.x + u * NTHR;
      const bool isInv = k >= ZTX;
      const int xx = x0 + (isInv ? k - ZTX : k);
      if (xx < W) cp_async4(st + k, (isInv ? iFg : SFg) + rowo + xx);
      else st[k] = isInv ? qnan() : 0.f;
    }
#pragma unroll
    for (int u = 0; u < TSG; u++) {
      const int k = threadIdx.x + u * NTHR;
      if (k < 2 * gm.SGC) {
        const bool isInv = k >= gm.SGC;
        const int c = isInv ? k - gm.SGC : k;
        const int xx = s0 + c;
        const int o = orient_s(c);
        RSR_CHECK(o >= 0 && o < gm.SROW2);
        float* row = st + 2 * ZTX + (isInv ? 2 : 0) * gm.SROW2;   // sG | sG1 | iG | iG1
        if (xx >= 0 && xx < W) {
          const float* src = (isInv ? iGg : SGg) + rowo + xx;
          cp_async4(row + o, src);
          if (o > 0) cp_async4(row + gm.SROW2 + o - 1, src);
        } else {
          const float v = isInv ? qnan() : 0.f;
          row[o] = v;
          if (o > 0) row[gm.SROW2 + o - 1] = v;
        }
      }
    }
  };

  // prologue: image rows 0 .. 2P + 1 and the statistics of output rows 0 and 1
  for (int t = 0; t <= 2 * P + 1; t++) issue_img(t);
  issue_stats(0);
  if (nrows > 1) issue_stats(1);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  const int n_rg = (D + ZR - 1) / ZR;
  const int rg = threadIdx.x % n_rg, cg = threadIdx.x / n_rg;
  const bool active = cg < ZTX / ZX;
  const int r0 = d_lo + ZR * rg;               // first residual disparity of the thread
  const int u_t = x0 + ZX * cg;                // first column of the thread
  const int f_start = ZX * cg;                 // column u_t - P
  const int g_start = TAR ? (ZX * cg + ZR * rg) : (ZX * cg + D - ZR - ZR * rg + gm.gpad);
  // oriented run starts (16-byte aligned): entry of (j, q) = run + j * dj + q
  const int grun = TAR ? g_start : gm.RB - g_start - (NJ - 1) - (ZR - 1);
  const int srun = TAR ? g_start : gm.RS - g_start - (ZX - 1) - (ZR - 1);
  const float nf = (float)((2 * P + 1) * (2 * P + 1));

  // V2[j][qp] = sum over the 2P+1 block rows of F(col j) * (G(q), G(q+1)) for q = 2qp:
  // exact integers < 2^24 accumulated by FFMA2 with the F value as scalar operand.
  float2 V2[NJ][NQP];
#pragma unroll
  for (int j = 0; j < NJ; j++)
#pragma unroll
    for (int qp = 0; qp < NQP; qp++) V2[j][qp] = make_float2(0.f, 0.f);

  auto accumulate_row = [&](int t, bool subtract) {
    const int slot = t % NRING;
    float f[NF4 * 4], ge[NG4 * 4], go[NG4 * 4];
    RSR_CHECK(slot < gm.NRING && f_start + NF4 * 4 <= gm.FC && grun >= 0 && grun + NG4 * 4 <= gm.GROW);
    const float4* fr = reinterpret_cast<const float4*>(Fs + slot * gm.FC + f_start);
    const float4* gr = reinterpret_cast<const float4*>(Gs + slot * gm.GROW + grun);
    const float4* gr1 = reinterpret_cast<const float4*>(Gs1 + slot * gm.GROW + grun);
#pragma unroll
    for (int i = 0; i < NF4; i++) {
      const float4 v = fr[i];
      f[4 * i] = v.x; f[4 * i + 1] = v.y; f[4 * i + 2] = v.z; f[4 * i + 3] = v.w;
    }
#pragma unroll
    for (int i = 0; i < NG4; i++) {
      const float4 v = gr[i], w = gr1[i];
      ge[4 * i] = v.x; ge[4 * i + 1] = v.y; ge[4 * i + 2] = v.z; ge[4 * i + 3] = v.w;
      go[4 * i] = w.x; go[4 * i + 1] = w.y; go[4 * i + 2] = w.z; go[4 * i + 3] = w.w;
    }
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const float fj = subtract ? -f[j] : f[j];
      // oriented offset of (j, q = 0): TAR j, REF (NJ - 1) - j
      const int o0 = TAR ? j : (NJ - 1 - j);
#pragma unroll
      for (int qp = 0; qp < NQP; qp++) {
        const int o = o0 + 2 * qp;
        const float2 gp = (o & 1) ? make_float2(go[o - 1], go[o]) : make_float2(ge[o], ge[o + 1]);
        V2[j][qp] = f2fma(make_float2(fj, fj), gp, V2[j][qp]);
      }
    }
  };

  for (int y = 0; y < nrows; y++) {
    // copies for iteration y + 2: image row y + 2 + 2P, statistics of output row y + 2
    if (y + 2 < nrows) {
      issue_img(y + 2 + 2 * P);
      issue_stats(y + 2);
    }
    cp_async_commit();
    if (active) {
      if (y == 0) {
#pragma unroll 1
        for (int t = 0; t <= 2 * P; t++) accumulate_row(t, false);
      } else {
        accumulate_row(y + 2 * P, false);
        accumulate_row(y - 1, true);
      }
      // block statistics of this row: F side per pixel, G side as oriented pairs
      const float* st = St + (y % 3) * SROW;
      float sF[ZX], iF[ZX];
      const float4 sfa = *reinterpret_cast<const float4*>(st + ZX * cg);
      const float4 ifa = *reinterpret_cast<const float4*>(st + ZTX + ZX * cg);
      sF[0] = sfa.x; sF[1] = sfa.y; sF[2] = sfa.z; sF[3] = sfa.w;
      iF[0] = ifa.x; iF[1] = ifa.y; iF[2] = ifa.z; iF[3] = ifa.w;
      RSR_CHECK(srun >= 0 && srun + NS4 * 4 <= gm.SROW2 && ZX * cg + ZX <= ZTX);
      // G-side statistics are read per pixel (8 oriented entries from the even or the
      // shifted copy), not held for all ZX pixels: 32 fewer live registers
      const float* sg = st + 2 * ZTX + srun;
      const int yy = y0 + y;
      float* vrow = vol + ((ibase + (size_t)yy * W) * Dst) + koff;
      // NaN structure from the statistics alone (num is always finite): c(i, q) is NaN
      // iff iF[i] or the G-side norm of (i, q) is NaN; over q those are the oriented
      // entries [oi, oi + ZR) with oi = TAR ? i : ZX - 1 - i.
      const int nq = min(ZR, d_hi - r0 + 1);   // disparities of this thread inside the slab
      float2 hs[NQP];
#pragma unroll
      for (int qp = 0; qp < NQP; qp++) {
        float2 acc = V2[0][qp];
#pragma unroll
        for (int dx = 1; dx < 2 * P + 1; dx++) acc = f2add(acc, V2[dx][qp]);
        hs[qp] = acc;
      }
#pragma unroll
      for (int i = 0; i < ZX; i++) {
        const int u = u_t + i;
        if (i > 0) {
#pragma unroll
          for (int qp = 0; qp < NQP; qp++)   // sliding horizontal sum, exact integers
            hs[qp] = f2sub(f2add(hs[qp], V2[i + 2 * P][qp]), V2[i - 1][qp]);
        }
        const int oi = TAR ? i : (ZX - 1 - i);
        float2 out[NQP];
#pragma unroll
        for (int qp = 0; qp < NQP; qp++) {
          const int o = oi + 2 * qp;
          // (o & 1) == (oi & 1): the pair starts at an even entry of sG (oi even) or sG1
          const float2 sgv = *reinterpret_cast<const float2*>((o & 1) ? sg + gm.SROW2 + o - 1 : sg + o);
          const float2 ig = *reinterpret_cast<const float2*>((o & 1) ? sg + 3 * gm.SROW2 + o - 1
                                                                       : sg + 2 * gm.SROW2 + o);
          const float2 sf = make_float2(sF[i], sF[i]), inf = make_float2(iF[i], iF[i]);
          const float2 nn = make_float2(nf, nf);
          // n S_lw - S_l S_w: the product S_l S_w split error-free (bb + be), then one
          // FMA forms n S_lw - bb exactly rounded; exact whenever |num| < 2^24 - 8
          // (cancellation), 1e-7 relative otherwise
          const float2 bb = f2mul(sf, sgv);
          const float2 nbb = make_float2(-bb.x, -bb.y);
          const float2 be = f2fma(sf, sgv, nbb);
          const float2 num = f2sub(f2fma(nn, hs[qp], nbb), be);
          // (num * inv_L) * inv_W, in this order for both volumes (bitwise dual identity)
          const float2 c = TAR ? f2mul(f2mul(num, ig), inf) : f2mul(f2mul(num, inf), ig);
          out[qp] = make_float2(clamp_unit_nan(c.x), clamp_unit_nan(c.y));
        }
        if (SHEAR) {
          float* tp = Tt + (ZX * cg + i) * ZT_STR + (r0 - d_lo);
          reinterpret_cast<float4*>(tp)[0] = make_float4(out[0].x, out[0].y, out[1].x, out[1].y);
          reinterpret_cast<float4*>(tp)[1] = make_float4(out[2].x, out[2].y, out[3].x, out[3].y);
        }
        if (u < W) {
          float* dst = vrow + (size_t)u * Dst + (r0 - d_lo);
          RSR_CHECK(yy < H && koff + (r0 - d_lo) + nq <= Dst);
          if ((Dst & 3) == 0 && (koff & 3) == 0 && nq >= ZR) {
            reinterpret_cast<float4*>(dst)[0] = make_float4(out[0].x, out[0].y, out[1].x, out[1].y);
            reinterpret_cast<float4*>(dst)[1] = make_float4(out[2].x, out[2].y, out[3].x, out[3].y);
          } else {
#pragma unroll
            for (int q = 0; q < ZR; q++)
              if (q < nq) dst[q] = (q & 1) ? out[q >> 1].y : out[q >> 1].x;
          }
        }
      }
    }
    if (SHEAR) {
      // C_R[u'][k] = C_L[u' + d_lo + k][k] for the sources in this tile's columns
      // [x0, x0 + ZTX) (the first / last tile also write the NaN entries whose source
      // lies left / right of the image): one warp per target pixel u', lanes along k
      __syncthreads();
      const int yy = y0 + y;
      const long long lo_c = x0 == 0 ? -(1LL << 30) : x0;
      const long long hi_c = x0 + ZTX >= W ? (1LL << 30) : x0 + ZTX - 1;
      const int ulo = (int)max(0LL, lo_c - d_lo - (D - 1)), uhi = (int)min((long long)W - 1, hi_c - d_lo);
      float* trow = vol_tar + ((ibase + (size_t)yy * W) * Dst) + koff;
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
      for (int up = ulo + warp; up <= uhi; up += nw) {
        const int ka = (int)max(0LL, lo_c - d_lo - up), kb = (int)min((long long)D - 1, hi_c - d_lo - up);
        for (int k = ka + lane; k <= kb; k += 32) {
          const int sc = up + d_lo + k;
          float v = qnan();
          if (sc >= 0 && sc < W) v = Tt[(sc - x0) * ZT_STR + k];
          trow[(size_t)up * Dst + k] = v;
        }
      }
    }
    // this thread's copies for iteration y + 1 have landed; the barrier publishes
    // everyone's (the slot of row y - 2 and St[(y + 2) % 3], written by the copies
    // issued above, were last read in iteration y - 1)
    cp_async_wait_prev();
    __syncthreads();
  }
}

#define RSR_ZNCC_BOUNDS __launch_bounds__(128, (P <= 3 ? 3 : (P <= 5 ? 2 : 1)))

template <int P, bool TAR>
__global__ void RSR_ZNCC_BOUNDS k_zncc(int H, int W, int d_lo, int D, int Dst, int koff, const float* ref,
                                       const float* warped, const float* SLg, const float* invLg,
                                       const float* SWg, const float* invWg, float* vol) {
  zncc_cta<P, TAR>(blockIdx.z, H, W, d_lo, D, Dst, koff, ref, warped, SLg, invLg, SWg, invWg, vol);
}

// Both volumes in one launch (frames [0, B) -> reference, [B, 2B) -> target): one
// grid twice as long, so the two halves fill each other's last wave.
// the wide small-D CTA holds more prefetch registers: two CTAs per SM at most
template <int P, int ZT>
#ifdef RSR_K2_MINB4   // experiment build (tools/): four CTAs per SM at P <= 3 (128 registers)
#define RSR_K2_MB3 4
#else
#define RSR_K2_MB3 3
#endif
__global__ void __launch_bounds__(128, (ZT != ZT_SMALL ? (P <= 3 ? RSR_K2_MB3 : (P <= 5 ? 2 : 1)) : (P <= 5 ? 2 : 1)))
    k_zncc_pair(int B, int H, int W, int d_lo, int D, int Dst, int koff,
                                            const float* ref, const float* warped, const float* SLg,
                                            const float* invLg, const float* SWg, const float* invWg,
                                            float* vol_ref, float* vol_tar) {
  if ((int)blockIdx.z < B)
    zncc_cta<P, false, ZT>(blockIdx.z, H, W, d_lo, D, Dst, koff, ref, warped, SLg, invLg, SWg, invWg, vol_ref);
  else
    zncc_cta<P, true, ZT>(blockIdx.z - B, H, W, d_lo, D, Dst, koff, ref, warped, SLg, invLg, SWg, invWg, vol_tar);
}

template <int P, int ZT>
static cudaError_t zncc_pair_launch_zt(int B, int H, int W, int d_lo, int D, int Dst, int koff, const float* ref,
                                       const float* warped, const float* SL, const float* invL,
                                       const float* SW, const float* invW, float* vol_ref, float* vol_tar,
                                       cudaStream_t st) {
  const size_t smem = zncc_smem(P, D, ZT);
  auto kern = k_zncc_pair<P, ZT>;
  cudaError_t e = smem_optin((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + ZT - 1) / ZT, (H + ZBY - 1) / ZBY, 2 * B);
  kern<<<grid, 128, smem, st>>>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW, vol_ref, vol_tar);
  return cudaGetLastError();
}

// Both volumes from the reference CTAs alone (SHEAR): grid of B frames
template <int P>
__global__ void RSR_ZNCC_BOUNDS k_zncc_shear(int H, int W, int d_lo, int D, int Dst, int koff, const float* ref,
                                             const float* warped, const float* SLg, const float* invLg,
                                             const float* SWg, const float* invWg, float* vol_ref,
                                             float* vol_tar) {
  zncc_cta<P, false, ZTX, true>(blockIdx.z, H, W, d_lo, D, Dst, koff, ref, warped, SLg, invLg, SWg, invWg, vol_ref,
                                vol_tar);
}

template <int P>
static cudaError_t zncc_shear_launch_t(int B, int H, int W, int d_lo, int D, int Dst, int koff, const float* ref,
                                       const float* warped, const float* SL, const float* invL,
                                       const float* SW, const float* invW, float* vol_ref, float* vol_tar,
                                       cudaStream_t st) {
  const size_t smem = zncc_smem(P, D, ZTX, true);
  auto kern = k_zncc_shear<P>;
  cudaError_t e = smem_optin((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + ZTX - 1) / ZTX, (H + ZBY - 1) / ZBY, B);
  kern<<<grid, 128, smem, st>>>(H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW, vol_ref, vol_tar);
  return cudaGetLastError();
}

template <int P>
static cudaError_t zncc_pair_launch_t(int B, int H, int W, int d_lo, int D, int Dst, int koff, const float* ref,
                                      const float* warped, const float* SL, const float* invL,
                                      const float* SW, const float* invW, float* vol_ref, float* vol_tar,
                                      cudaStream_t st) {
  if (zncc_cta_cols(D) == ZT_SMALL)
    return zncc_pair_launch_zt<P, ZT_SMALL>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW,
                                            vol_ref, vol_tar, st);
  if (zncc_cta_cols(D) == ZT_MID)
    return zncc_pair_launch_zt<P, ZT_MID>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW,
                                          vol_ref, vol_tar, st);
  // experiment hook (tools/): RSR_K2_SHEAR=1 writes the target volume by the shear from the
  // reference CTAs.  Measured slower (c5, 8 frames: 3.51 ms vs 1.64 ms for the pair grid:
  // the k-runs of a target pixel come from two CTAs, partial 256-byte records), so off
  const char* e = getenv("RSR_K2_SHEAR");
  if (e && e[0] == '1')
    return zncc_shear_launch_t<P>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW, vol_ref, vol_tar,
                                  st);
  return zncc_pair_launch_zt<P, ZTX>(B, H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW, vol_ref,
                                     vol_tar, st);
}

template <int P, bool TAR>
static cudaError_t zncc_launch_t(int B, int H, int W, int d_lo, int D, int Dst, int koff,
                                 const float* ref,
                                 const float* warped, const float* SL, const float* invL,
                                 const float* SW, const float* invW, float* vol,
                                 cudaStream_t st) {
  const size_t smem = zncc_smem(P, D);
  auto kern = k_zncc<P, TAR>;
  cudaError_t e = smem_optin((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  // always 128 threads: (D <= 64) / 8 disparity groups x 16 column groups compute,
  // and all of them stream the rows (ZPF x 128 >= the longest row load list)
  const int threads = 128;
  static_assert(2 * 128 >= 84 + 152 && 4 * 128 >= 2 * ZTX + 2 * 136, "row load lists must fit the prefetch");
  // threads > 1024 is rejected by the API (D > 512 would need a k-slab split)
  dim3 grid((W + ZTX - 1) / ZTX, (H + ZBY - 1) / ZBY, B);
  kern<<<grid, threads, smem, st>>>(H, W, d_lo, D, Dst, koff, ref, warped, SL, invL, SW, invW, vol);
  return cudaGetLastError();
}

// Per-pixel NaN summaries straight from the block statistics: an NCC cost is NaN
// exactly when the left or the right block norm is (the numerator is always
// finite), so for the reference volume, pixel u has some finite cost iff inv_L(u)
// is finite and some inv_W(u - r), r in [d_lo, d_hi], is, and some NaN cost iff
// inv_L(u) is NaN or one of those is NaN or outside the image; symmetrically for the
// target volume with inv_W(u') and inv_L(u' + r).  One CTA per (row, frame):
// prefix counts of finite norms along the row make each pixel O(1).
__global__ void __launch_bounds__(256) k_nan_maps(int H, int W, int d_lo, int D,
                                                  const float* __restrict__ invL,
                                                  const float* __restrict__ invW,
                                                  uint8_t* __restrict__ nan_ref,
                                                  uint8_t* __restrict__ nan_tar) {
  extern __shared__ int nm_smem[];
  int* cL = nm_smem;          // [W + 1] prefix counts of finite inv_L
  int* cW = cL + (W + 1);     // [W + 1] prefix counts of finite inv_W
  const int v = blockIdx.x, b = blockIdx.y;
  const size_t row = ((size_t)b * H + v) * W;
  __shared__ int wsumL[32], wsumW[32];
  // block-wide exclusive scans, 256-column chunks
  int carryL = 0, carryW = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c0 = 0; c0 < W; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    int fl = 0, fw = 0;
    if (c < W) {
      const float a = invL[row + c], w = invW[row + c];
      fl = a == a; fw = w == w;
    }
    int sl = fl, sw = fw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tl = __shfl_up_sync(0xffffffffu, sl, o), tw = __shfl_up_sync(0xffffffffu, sw, o);
      if (lane >= o) { sl += tl; sw += tw; }
    }
    if (lane == 31) { wsumL[warp] = sl; wsumW[warp] = sw; }
    __syncthreads();
    int offL = carryL, offW = carryW;
    for (int q = 0; q < warp; q++) { offL += wsumL[q]; offW += wsumW[q]; }
    if (c < W) { cL[c + 1] = offL + sl; cW[c + 1] = offW + sw; }
    for (int q = 0; q < nw; q++) { carryL += wsumL[q]; carryW += wsumW[q]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { cL[0] = 0; cW[0] = 0; }
  __syncthreads();
  auto count = [&](const int* cnt, int a, int bcol) {   // finite entries in columns [a, b]
    a = max(a, 0);
    bcol = min(bcol, W - 1);
    return bcol < a ? 0 : cnt[bcol + 1] - cnt[a];
  };
  // disparity halves of a single-slab volume (rsr_aggregate's two general passes):
  // [0, H0) and [H0, D) with H0 = roundup8(D) / 2; bits 2 / 3 flag a NaN in each,
  // bit 7 says the half bits are present
  const bool halves = D <= 64;
  // the low half [0, H0) is clipped to the D disparities that exist (D <= 3: H0 = 4 > D)
  const int H0 = min(((D + 7) & ~7) / 2, D);
  for (int u = threadIdx.x; u < W; u += blockDim.x) {
    const bool lok = cL[u + 1] - cL[u] != 0, wok = cW[u + 1] - cW[u] != 0;
    if (nan_ref) {   // k valid iff inv_L(u) and inv_W(u - d_lo - k) finite
      const int f0 = lok ? count(cW, u - d_lo - (H0 - 1), u - d_lo) : 0;
      const int f1 = lok ? count(cW, u - d_lo - (D - 1), u - d_lo - H0) : 0;
      const int fin = f0 + f1;
      int m = (fin < D ? 1 : 0) | (fin > 0 ? 2 : 0);
      if (halves) m |= (f0 < H0 ? 4 : 0) | (f1 < D - H0 ? 8 : 0) | 0x80;
      nan_ref[row + u] = (uint8_t)m;
    }
    if (nan_tar) {   // k valid iff inv_W(u') and inv_L(u' + d_lo + k) finite
      const int f0 = wok ? count(cL, u + d_lo, u + d_lo + H0 - 1) : 0;
      const int f1 = wok ? count(cL, u + d_lo + H0, u + d_lo + D - 1) : 0;
      const int fin = f0 + f1;
      int m = (fin < D ? 1 : 0) | (fin > 0 ? 2 : 0);
      if (halves) m |= (f0 < H0 ? 4 : 0) | (f1 < D - H0 ? 8 : 0) | 0x80;
      nan_tar[row + u] = (uint8_t)m;
    }
  }
}

// The same summaries with one warp per (row, frame), NM_WARPS rows per CTA and no CTA
// barrier: finite flags are staged coalesced, each lane scans a contiguous chunk of
// odd length (conflict-free), the chunk totals are combined by a warp scan.
constexpr int NM_WARPS = 4;
__global__ void __launch_bounds__(32 * NM_WARPS) k_nan_maps_warp(int B, int H, int W, int d_lo, int D,
                                                                 const float* __restrict__ invL,
                                                                 const float* __restrict__ invW,
                                                                 uint8_t* __restrict__ nan_ref,
                                                                 uint8_t* __restrict__ nan_tar) {
  extern __shared__ int nmw_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * NM_WARPS + warp;   // row of the batch
  if (r >= (long long)B * H) return;                             // whole warp
  int* cL = nmw_smem + (size_t)warp * 2 * (W + 1);   // [W + 1] prefix counts of finite inv_L
  int* cW = cL + (W + 1);                           // [W + 1] prefix counts of finite inv_W
  const size_t row = (size_t)r * W;
  for (int c = lane; c < W; c += 32) {
    const float a = invL[row + c], w = invW[row + c];
    cL[c + 1] = a == a;
    cW[c + 1] = w == w;
  }
  if (lane == 0) { cL[0] = 0; cW[0] = 0; }
  __syncwarp();
  const int chunk = ((W + 31) / 32) | 1;
  const int c0 = min(W, lane * chunk), c1 = min(W, c0 + chunk);
  int sl = 0, sw = 0;
  for (int c = c0; c < c1; c++) { sl += cL[c + 1]; sw += cW[c + 1]; }
  int il = sl, iw = sw;   // inclusive warp scan of the chunk totals
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int tl = __shfl_up_sync(0xffffffffu, il, o), tw = __shfl_up_sync(0xffffffffu, iw, o);
    if (lane >= o) { il += tl; iw += tw; }
  }
  int rl = il - sl, rw = iw - sw;
  for (int c = c0; c < c1; c++) {
    rl += cL[c + 1]; rw += cW[c + 1];
    cL[c + 1] = rl; cW[c + 1] = rw;
  }
  __syncwarp();
  auto count = [&](const int* cnt, int a, int bcol) {   // finite entries in columns [a, b]
    a = max(a, 0);
    bcol = min(bcol, W - 1);
    return bcol < a ? 0 : cnt[bcol + 1] - cnt[a];
  };
  const bool halves = D <= 64;
  const int H0 = min(((D + 7) & ~7) / 2, D);
  for (int u = lane; u < W; u += 32) {
    const bool lok = cL[u + 1] - cL[u] != 0, wok = cW[u + 1] - cW[u] != 0;
    if (nan_ref) {   // k valid iff inv_L(u) and inv_W(u - d_lo - k) finite
      const int f0 = lok ? count(cW, u - d_lo - (H0 - 1), u - d_lo) : 0;
      const int f1 = lok ? count(cW, u - d_lo - (D - 1), u - d_lo - H0) : 0;
      const int fin = f0 + f1;
      int m = (fin < D ? 1 : 0) | (fin > 0 ? 2 : 0);
      if (halves) m |= (f0 < H0 ? 4 : 0) | (f1 < D - H0 ? 8 : 0) | 0x80;
      nan_ref[row + u] = (uint8_t)m;
    }
    if (nan_tar) {   // k valid iff inv_W(u') and inv_L(u' + d_lo + k) finite
      const int f0 = wok ? count(cL, u + d_lo, u + d_lo + H0 - 1) : 0;
      const int f1 = wok ? count(cL, u + d_lo + H0, u + d_lo + D - 1) : 0;
      const int fin = f0 + f1;
      int m = (fin < D ? 1 : 0) | (fin > 0 ? 2 : 0);
      if (halves) m |= (f0 < H0 ? 4 : 0) | (f1 < D - H0 ? 8 : 0) | 0x80;
      nan_tar[row + u] = (uint8_t)m;
    }
  }
}

cudaError_t launch_nan_maps(int B, int H, int W, int d_lo, int D, const float* invL,
                            const float* invW, uint8_t* nan_ref, uint8_t* nan_tar, cudaStream_t st) {
  if (!nan_ref && !nan_tar) return cudaSuccess;
  const size_t smem_w = sizeof(int) * 2 * ((size_t)W + 1) * NM_WARPS;
  const long long rows = (long long)B * H;
  if (smem_w <= 227 * 1024 && (rows + NM_WARPS - 1) / NM_WARPS <= 0x7fffffffLL &&
      !(getenv("RSR_NM_CTA") && getenv("RSR_NM_CTA")[0] == '1')) {   // A/B hook (tools/): per-row CTAs
    const cudaError_t e = smem_optin((const void*)k_nan_maps_warp, smem_w);
    if (e != cudaSuccess) return e;
    k_nan_maps_warp<<<(unsigned)((rows + NM_WARPS - 1) / NM_WARPS), 32 * NM_WARPS, smem_w, st>>>(
        B, H, W, d_lo, D, invL, invW, nan_ref, nan_tar);
    return cudaGetLastError();
  }
  const size_t smem = sizeof(int) * 2 * ((size_t)W + 1);
  const cudaError_t e = smem_optin((const void*)k_nan_maps, smem);
  if (e != cudaSuccess) return e;
  k_nan_maps<<<dim3(H, B), 256, smem, st>>>(H, W, d_lo, D, invL, invW, nan_ref, nan_tar);
  return cudaGetLastError();
}

cudaError_t launch_zncc_pair(int B, int H, int W, int rho_b, int d_lo, int D, const float* ref,
                             const float* warped, const float* SL, const float* invL, const float* SW,
                             const float* invW, float* vol_ref, float* vol_tar, cudaStream_t st) {
  constexpr int SLAB = 64;
  if (2LL * B > 65535) return cudaErrorInvalidValue;
  for (int k0 = 0; k0 < D; k0 += SLAB) {
    const int Ds = D - k0 < SLAB ? D - k0 : SLAB;
    const int dl = d_lo + k0;
    cudaError_t e;
#define RSR_Z(PP)                                                                                  \
  case PP:                                                                                         \
    e = zncc_pair_launch_t<PP>(B, H, W, dl, Ds, D, k0, ref, warped, SL, invL, SW, invW, vol_ref,   \
                               vol_tar, st);                                                       \
    break;
    switch (rho_b) {
      RSR_Z(1) RSR_Z(2) RSR_Z(3) RSR_Z(4) RSR_Z(5) RSR_Z(6) RSR_Z(7)
      default:
        return cudaErrorInvalidValue;
    }
#undef RSR_Z
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_zncc(bool tar, int B, int H, int W, int rho_b, int d_lo, int D,
                        const float* ref, const float* warped, const float* SL,
                        const float* invL, const float* SW, const float* invW, float* vol,
                        cudaStream_t st) {
  // Disparity slabs of at most 64 (<= 128 threads per CTA).
  constexpr int SLAB = 64;
  for (int k0 = 0; k0 < D; k0 += SLAB) {
    const int Ds = D - k0 < SLAB ? D - k0 : SLAB;
    const int dl = d_lo + k0;
    cudaError_t e;
#define RSR_Z(PP)                                                                                \
  case PP:                                                                                       \
    e = tar ? zncc_launch_t<PP, true>(B, H, W, dl, Ds, D, k0, ref, warped, SL, invL, SW, invW,    \
                                      vol, st)                                                   \
            : zncc_launch_t<PP, false>(B, H, W, dl, Ds, D, k0, ref, warped, SL, invL, SW, invW,   \
                                       vol, st);                                                 \
    break;
    switch (rho_b) {
      RSR_Z(1) RSR_Z(2) RSR_Z(3) RSR_Z(4) RSR_Z(5) RSR_Z(6) RSR_Z(7)
      default:
        return cudaErrorInvalidValue;
    }
#undef RSR_Z
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace rsr
