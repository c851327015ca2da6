// Reconstruction-accuracy evaluation (NEXT row f4): the ground
// plane n0 x + n1 y + n2 z + n3 = 0 "interpolated" from the corners of a selected
// region, and the distances of reconstructed points to it (reading 19).
//
// k_plane_fit: one thread per frame.  Total least squares: the unit normal is the
// eigenvector of the corners' scatter matrix with the smallest eigenvalue (cyclic
// Jacobi rotations in fp64 until the off-diagonal vanishes), n3 = -n . centroid,
// oriented n3 > 0 (n3 == 0: last non-zero normal entry positive); NaN for fewer
// than 3 finite corners or lambda_2 <= 1e-24 lambda_1 (sigma_2 <= 1e-12 sigma_1).
// k_plane_distance: one thread per pixel, n . p + n3 in fp64, stored as float.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace rsr {

__global__ void k_plane_fit(int B, int K, const double* __restrict__ corners, double* __restrict__ plane) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* c = corners + (size_t)b * K * 3;
  double* out = plane + (size_t)b * 4;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  bool ok = K >= 3;
  double m[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < K; i++)
    for (int a = 0; a < 3; a++) {
      ok &= isfinite(c[3 * i + a]);
      m[a] += c[3 * i + a];
    }
  if (!ok) {
    out[0] = out[1] = out[2] = out[3] = nan;
    return;
  }
  for (int a = 0; a < 3; a++) m[a] /= K;
  double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int i = 0; i < K; i++) {
    const double x[3] = {c[3 * i] - m[0], c[3 * i + 1] - m[1], c[3 * i + 2] - m[2]};
    for (int a = 0; a < 3; a++)
      for (int e = 0; e < 3; e++) A[a][e] += x[a] * x[e];
  }
  double V[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  for (int sweep = 0; sweep < 64; sweep++) {
    const double off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
    const double dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
    if (off <= 1e-36 * dia || off == 0.0) break;
    for (int p = 0; p < 2; p++)
      for (int q = p + 1; q < 3; q++) {
        if (A[p][q] == 0.0) continue;
        // rotation zeroing A[p][q] (Golub & Van Loan, symmetric Schur)
        const double tau = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = t * cs;
        for (int k = 0; k < 3; k++) {   // A <- A J
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = cs * akp - sn * akq;
          A[k][q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 3; k++) {   // A <- J^T A
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = cs * apk - sn * aqk;
          A[q][k] = sn * apk + cs * aqk;
        }
        for (int k = 0; k < 3; k++) {   // V <- V J
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = cs * vkp - sn * vkq;
          V[k][q] = sn * vkp + cs * vkq;
        }
      }
  }
  // eigenvalues on the diagonal: smallest -> normal; largest / middle -> degeneracy
  int lo = 0, hi = 0;
  for (int a = 1; a < 3; a++) {
    if (A[a][a] < A[lo][lo]) lo = a;
    if (A[a][a] > A[hi][hi]) hi = a;
  }
  int mid = 3 - lo - hi;
  if (lo == hi) {   // all three equal
    hi = (lo + 1) % 3;
    mid = (lo + 2) % 3;
  }
  const double l1 = fmax(A[hi][hi], 0.0), l2 = fmax(A[mid][mid], 0.0);
  if (!(l1 > 0.0) || l2 <= 1e-24 * l1) {
    out[0] = out[1] = out[2] = out[3] = nan;
    return;
  }
  double n[3] = {V[0][lo], V[1][lo], V[2][lo]};
  const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
  for (int a = 0; a < 3; a++) n[a] /= nn;
  double n3 = -(n[0] * m[0] + n[1] * m[1] + n[2] * m[2]);
  bool flip = n3 < 0.0;
  if (n3 == 0.0) {
    const double last = n[2] != 0.0 ? n[2] : (n[1] != 0.0 ? n[1] : n[0]);
    flip = last < 0.0;
  }
  if (flip) {
    for (int a = 0; a < 3; a++) n[a] = -n[a];
    n3 = -n3;
  }
  out[0] = n[0]; out[1] = n[1]; out[2] = n[2]; out[3] = n3;
}

__global__ void k_plane_distance(long long HW, long long n_total, const double* __restrict__ plane,
                                 const float* __restrict__ xyz, float* __restrict__ dist) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_total;
       i += (long long)gridDim.x * blockDim.x) {
    const double* pl = plane + (i / HW) * 4;
    const float* p = xyz + 3 * i;
    dist[i] = (float)(p[0] * pl[0] + p[1] * pl[1] + p[2] * pl[2] + pl[3]);
  }
}

cudaError_t launch_plane_fit(int B, int K, const double* corners, double* plane, cudaStream_t st) {
  k_plane_fit<<<(B + 63) / 64, 64, 0, st>>>(B, K, corners, plane);
  return cudaGetLastError();
}

cudaError_t launch_plane_distance(int B, int H, int W, const double* plane, const float* xyz, float* dist,
                                  cudaStream_t st) {
  const long long n = (long long)B * H * W;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
  k_plane_distance<<<blocks, 256, 0, st>>>((long long)H * W, n, plane, xyz, dist);
  return cudaGetLastError();
}

}  // namespace rsr
