// K5 — triangulation (rectified pinhole, reading 15):
// Z = f b / d, X = (u - u0) Z / f, Y = (v - v0) Z / f for d > d_min, else NaN.
// Elementwise, HBM-bound: reads 4 B and writes 12 B per pixel.
#include "common.cuh"
#include "kernels.h"

namespace rsr {

__global__ void __launch_bounds__(256) k_reconstruct(long long npix, int H, int W, float fb,
                                                     float inv_f, float u0, float v0, float d_min,
                                                     const float* __restrict__ disp,
                                                     float* __restrict__ xyz) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < npix;
       i += (long long)gridDim.x * blockDim.x) {
    const float d = disp[i];
    const int u = (int)(i % W);
    const int v = (int)((i / W) % H);
    float X, Y, Z;
    if (d > d_min) {  // false for NaN
      Z = fb / d;
      X = ((float)u - u0) * Z * inv_f;
      Y = ((float)v - v0) * Z * inv_f;
    } else {
      X = Y = Z = qnan();
    }
    xyz[3 * i + 0] = X;
    xyz[3 * i + 1] = Y;
    xyz[3 * i + 2] = Z;
  }
}

cudaError_t launch_reconstruct(int B, int H, int W, double f, double baseline, double u0,
                               double v0, double d_min, const float* disp, float* xyz,
                               cudaStream_t st) {
  const long long npix = (long long)B * H * W;
  long long blocks = (npix + 255) / 256;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  k_reconstruct<<<(int)blocks, 256, 0, st>>>(npix, H, W, (float)(f * baseline), (float)(1.0 / f),
                                             (float)u0, (float)v0, (float)d_min, disp, xyz);
  return cudaGetLastError();
}

}  // namespace rsr
