// Road-model estimation (Eq. (2)):
// RANSAC-LSF fit of d = alpha v + beta to (v, d) samples of a disparity map.
// Same algorithm and readings as oracle/road_model.py:
// counter-based two-point hypotheses, fp64 consensus test with one rounding per
// operation (explicit __d*_rn intrinsics: no FMA contraction, so every inlier
// decision equals the oracle's), most inliers wins (lowest index on ties), least
// squares over the winning consensus set.
//
//   k_road_samples  one CTA per frame: stream-compacts the finite entries of the
//                   sampling grid in row-major order (block scans)
//   k_road_hyp      one warp per hypothesis: lanes stride over the samples
//   k_road_fit      one CTA per frame: argmax over hypotheses, fp64 normal
//                   equations over the consensus set (fixed reduction order)
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

RSR_DEVINL unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

RSR_DEVINL void draw_pair(unsigned seed, int h, int n, int& i, int& j) {
  const unsigned long long base = (unsigned long long)seed << 32;
  i = (int)(splitmix64(base + 2ull * h) % (unsigned long long)n);
  j = (int)(splitmix64(base + 2ull * h + 1ull) % (unsigned long long)n);
  if (j == i) j = (j + 1) % n;
}

// line through samples i, j; false if degenerate (same row)
RSR_DEVINL bool hyp_line(const float* v, const float* d, int i, int j, double& a, double& b) {
  const double vi = v[i], vj = v[j], di = d[i], dj = d[j];
  if (vi == vj) return false;
  a = __ddiv_rn(__dsub_rn(dj, di), __dsub_rn(vj, vi));
  b = __dsub_rn(di, __dmul_rn(a, vi));
  return true;
}

RSR_DEVINL bool inlier(double vk, double dk, double a, double b, double tol) {
  return fabs(__dsub_rn(dk, __dadd_rn(__dmul_rn(a, vk), b))) <= tol;
}

__global__ void __launch_bounds__(1024) k_road_samples(int H, int W, int su, int sv, int cap,
                                                       const float* __restrict__ disp,
                                                       float* __restrict__ sv_out,
                                                       float* __restrict__ sd_out,
                                                       int* __restrict__ counts) {
  const int b = blockIdx.x;
  const int NU = (W + su - 1) / su, NV = (H + sv - 1) / sv, N = NU * NV;
  const float* dm = disp + (size_t)b * H * W;
  float* ov = sv_out + (size_t)b * cap;
  float* od = sd_out + (size_t)b * cap;
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int c0 = 0; c0 < N; c0 += blockDim.x) {
    const int e = c0 + threadIdx.x;
    float dv = 0.f;
    int vrow = 0, f = 0;
    if (e < N) {
      vrow = (e / NU) * sv;
      dv = dm[(size_t)vrow * W + (e % NU) * su];
      f = isfinite(dv) ? 1 : 0;
    }
    int x = f;   // inclusive warp scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int off = carry;
    for (int q = 0; q < warp; q++) off += wsum[q];
    if (f) {
      const int pos = off + x - 1;
      ov[pos] = (float)vrow;
      od[pos] = dv;
    }
    for (int q = 0; q < (int)(blockDim.x >> 5); q++) carry += wsum[q];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[b] = carry;
}

__global__ void __launch_bounds__(256) k_road_hyp(int cap, int n_hyp, unsigned seed, float tolf,
                                                  const float* __restrict__ sv,
                                                  const float* __restrict__ sd,
                                                  const int* __restrict__ counts,
                                                  int* __restrict__ hyp) {
  const int b = blockIdx.x;
  const int h = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (h >= n_hyp) return;
  const int n = counts[b];
  const float* v = sv + (size_t)b * cap;
  const float* d = sd + (size_t)b * cap;
  int c = -1;
  if (n >= 2) {
    int i, j;
    draw_pair(seed, h, n, i, j);
    double a, bb;
    if (hyp_line(v, d, i, j, a, bb)) {
      const double tol = (double)tolf;
      int cnt = 0;
      for (int k = lane; k < n; k += 32) cnt += inlier(v[k], d[k], a, bb, tol) ? 1 : 0;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      c = cnt;
    }
  }
  if (lane == 0) hyp[(size_t)b * n_hyp + h] = c;
}

__global__ void __launch_bounds__(256) k_road_fit(int cap, int n_hyp, unsigned seed, float tolf,
                                                  const float* __restrict__ sv,
                                                  const float* __restrict__ sd,
                                                  const int* __restrict__ counts,
                                                  const int* __restrict__ hyp,
                                                  double* __restrict__ model) {
  const int b = blockIdx.x;
  const int n = counts[b];
  const float* v = sv + (size_t)b * cap;
  const float* d = sd + (size_t)b * cap;
  const int* hc = hyp + (size_t)b * n_hyp;
  __shared__ long long best_s[256];
  __shared__ double red[5][256];
  // argmax: most inliers, then lowest index  (key = count << 32 | ~index)
  long long key = -1;
  for (int h = threadIdx.x; h < n_hyp; h += blockDim.x) {
    const int c = hc[h];
    if (c >= 0) {
      const long long k = ((long long)c << 32) | (unsigned)(0x7fffffff - h);
      if (k > key) key = k;
    }
  }
  best_s[threadIdx.x] = key;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && best_s[threadIdx.x + s] > best_s[threadIdx.x]) best_s[threadIdx.x] = best_s[threadIdx.x + s];
    __syncthreads();
  }
  const long long bk = best_s[0];
  double* out = model + 3 * (size_t)b;
  if (bk < 0 || n < 2) {
    if (threadIdx.x == 0) { out[0] = nan(""); out[1] = nan(""); out[2] = 0.0; }
    return;
  }
  const int hb = 0x7fffffff - (int)(bk & 0xffffffff);
  int i, j;
  draw_pair(seed, hb, n, i, j);
  double a, bb;
  hyp_line(v, d, i, j, a, bb);
  const double tol = (double)tolf;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double vk = v[k], dk = d[k];
    if (inlier(vk, dk, a, bb, tol)) {
      s0 += 1.0; s1 += vk; s2 += dk; s3 += vk * vk; s4 += vk * dk;
    }
  }
  red[0][threadIdx.x] = s0; red[1][threadIdx.x] = s1; red[2][threadIdx.x] = s2;
  red[3][threadIdx.x] = s3; red[4][threadIdx.x] = s4;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
#pragma unroll
      for (int q = 0; q < 5; q++) red[q][threadIdx.x] += red[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double N = red[0][0], SV = red[1][0], SD = red[2][0], SVV = red[3][0], SVD = red[4][0];
    const double den = N * SVV - SV * SV;
    if (N < 2.0 || den == 0.0) {
      out[0] = nan(""); out[1] = nan("");
    } else {
      const double al = (N * SVD - SV * SD) / den;
      out[0] = al;
      out[1] = (SD - al * SV) / N;
    }
    out[2] = N;
  }
}

// Roll angle: least-squares plane d = g0 + g1 u + g2 v over the finite
// disparities of a near-field patch, gamma = arctan(-g1 / g2).  One CTA per frame:
// fp64 normal-equation sums (fixed reduction order), 3x3 solve by Cramer's rule.
// out [B][5] = {g0, g1, g2, gamma, n}.
RSR_DEVINL double det3(double a, double b, double c, double d, double e, double f, double g, double h,
                       double i) {
  return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

__global__ void __launch_bounds__(256) k_road_roll(int H, int W, int u0, int u1, int v0, int v1,
                                                   const float* __restrict__ disp, double* __restrict__ out) {
  const int b = blockIdx.x;
  const float* dm = disp + (size_t)b * H * W;
  __shared__ double red[9][256];
  double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};   // n, su, sv, suu, suv, svv, sd, sud, svd
  const int pw = u1 - u0, np_ = pw * (v1 - v0);
  for (int e = threadIdx.x; e < np_; e += blockDim.x) {
    const int u = u0 + e % pw, v = v0 + e / pw;
    const float dv = dm[(size_t)v * W + u];
    if (isfinite(dv)) {
      const double U = u, V = v, Dd = dv;
      s[0] += 1.0; s[1] += U; s[2] += V; s[3] += U * U; s[4] += U * V; s[5] += V * V;
      s[6] += Dd; s[7] += U * Dd; s[8] += V * Dd;
    }
  }
#pragma unroll
  for (int q = 0; q < 9; q++) red[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
#pragma unroll
      for (int q = 0; q < 9; q++) red[q][threadIdx.x] += red[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = out + 5 * (size_t)b;
    const double n = red[0][0], su = red[1][0], sv = red[2][0], suu = red[3][0], suv = red[4][0],
                 svv = red[5][0], sd = red[6][0], sud = red[7][0], svd = red[8][0];
    const double det = det3(n, su, sv, su, suu, suv, sv, suv, svv);
    if (n < 3.0 || det == 0.0 || !isfinite(det)) {
      o[0] = o[1] = o[2] = o[3] = nan("");
    } else {
      o[0] = det3(sd, su, sv, sud, suu, suv, svd, suv, svv) / det;
      o[1] = det3(n, sd, sv, su, sud, suv, sv, svd, svv) / det;
      o[2] = det3(n, su, sd, su, suu, sud, sv, suv, svd) / det;
      o[3] = atan(-o[1] / o[2]);
    }
    o[4] = n;
  }
}

cudaError_t launch_road_roll(int B, int H, int W, int u0, int u1, int v0, int v1, const float* disp,
                             double* out, cudaStream_t st) {
  k_road_roll<<<B, 256, 0, st>>>(H, W, u0, u1, v0, v1, disp, out);
  return cudaGetLastError();
}

size_t road_workspace_size(int B, int H, int W, int su, int sv, int n_hyp) {
  const size_t cap = (size_t)((W + su - 1) / su) * ((H + sv - 1) / sv);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  return 2 * al(sizeof(float) * B * cap) + al(sizeof(int) * B) + al(sizeof(int) * (size_t)B * n_hyp);
}

cudaError_t launch_road_model(int B, int H, int W, int su, int sv, int n_hyp, float tol, unsigned seed,
                              const float* disp, double* model, void* ws, cudaStream_t st) {
  const int cap = ((W + su - 1) / su) * ((H + sv - 1) / sv);
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* p = static_cast<char*>(ws);
  float* s_v = reinterpret_cast<float*>(p);
  p += al(sizeof(float) * B * (size_t)cap);
  float* s_d = reinterpret_cast<float*>(p);
  p += al(sizeof(float) * B * (size_t)cap);
  int* counts = reinterpret_cast<int*>(p);
  p += al(sizeof(int) * B);
  int* hyp = reinterpret_cast<int*>(p);
  k_road_samples<<<B, 1024, 0, st>>>(H, W, su, sv, cap, disp, s_v, s_d, counts);
  dim3 g2(B, (n_hyp + 7) / 8);
  k_road_hyp<<<g2, 256, 0, st>>>(cap, n_hyp, seed, tol, s_v, s_d, counts, hyp);
  k_road_fit<<<B, 256, 0, st>>>(cap, n_hyp, seed, tol, s_v, s_d, counts, hyp, model);
  return cudaGetLastError();
}

}  // namespace rsr
