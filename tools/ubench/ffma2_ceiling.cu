// FFMA2 issue ceiling for the K3 inner-loop shape: acc[a][q] = w[a] * c[q] + acc[a][q]
// (scalar-broadcast weight, packed cost pair, packed accumulator), 13 ages x 4 pairs,
// with the operands refreshed from shared memory every "tap" (6 LDS.128 per 52 FFMA2),
// for 1..4 warps per SMSP.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_ceiling ffma2_ceiling.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 fma2s(float w, float2 c, float2 a) {
  unsigned long long av, cv, wb, dv;
  asm("mov.b64 %0, {%1,%2};" : "=l"(av) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1,%2};" : "=l"(cv) : "f"(c.x), "f"(c.y));
  asm("mov.b64 %0, {%1,%1};" : "=l"(wb) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(dv) : "l"(wb), "l"(cv), "l"(av));
  float2 d;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(dv));
  return d;
}

template <bool LDS, int MODE>
__global__ void k(float* out, int iters) {
  __shared__ __align__(16) float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1e-3f * (i & 63);
  __syncthreads();
  float2 acc[13][4];
#pragma unroll
  for (int a = 0; a < 13; a++)
#pragma unroll
    for (int q = 0; q < 4; q++) acc[a][q] = make_float2(0.f, 0.f);
  const int lane = threadIdx.x & 31;
  const float* cb = sm + (lane & 7) * 4;
  const float* wb = sm + 1024 + (lane >> 3) * 20;
  float wv[16]; float2 cp[4];
#pragma unroll
  for (int i = 0; i < 16; i++) wv[i] = 1e-3f * i;
#pragma unroll
  for (int q = 0; q < 4; q++) cp[q] = make_float2(1e-3f * q, 2e-3f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int j = 0; j < 13; j++) {
      if (LDS && (MODE & 1)) {
        const float4 ca = *reinterpret_cast<const float4*>(cb + ((j * 64 + it * 4) & 511));
        const float4 cc = *reinterpret_cast<const float4*>(cb + ((j * 64 + it * 4) & 511) + 32);
        cp[0] = make_float2(ca.x, ca.y); cp[1] = make_float2(ca.z, ca.w);
        cp[2] = make_float2(cc.x, cc.y); cp[3] = make_float2(cc.z, cc.w);
      }
      if (LDS && (MODE & 2)) {
        const float4* w4 = reinterpret_cast<const float4*>(wb + ((j * 16 + it * 4) & 1023));
#pragma unroll
        for (int q = 0; q < 4; q++) { float4 t = w4[q]; wv[4*q]=t.x; wv[4*q+1]=t.y; wv[4*q+2]=t.z; wv[4*q+3]=t.w; }
      }
#pragma unroll
      for (int q = 0; q < 4; q++)
#pragma unroll
        for (int a = 0; a < 13; a++) acc[a][q] = fma2s(wv[a], cp[q], acc[a][q]);
    }
  }
  float s = 0;
#pragma unroll
  for (int a = 0; a < 13; a++)
#pragma unroll
    for (int q = 0; q < 4; q++) s += acc[a][q].x + acc[a][q].y;
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  float* out; cudaMalloc(&out, 1 << 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = 148;
  for (int lds = 0; lds < 4; lds++)
    for (int wps = 1; wps <= 2; wps++) {
      int threads = 128 * wps, iters = 2000;
      auto launch = [&] { if (lds == 0) k<false, 0><<<sms, threads>>>(out, iters);
                          else if (lds == 1) k<true, 1><<<sms, threads>>>(out, iters);
                          else if (lds == 2) k<true, 2><<<sms, threads>>>(out, iters);
                          else k<true, 3><<<sms, threads>>>(out, iters); };
      launch(); cudaDeviceSynchronize();
      float best = 1e30f;
      for (int r = 0; r < 5; r++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
      double flop = 2.0 * sms * threads * (double)iters * 13 * 13 * 8;
      printf("{\"lds\": %d, \"warps_per_smsp\": %d, \"ms\": %.3f, \"tflops\": %.2f, \"frac_of_74.45\": %.3f}\n", lds, wps, best, flop / best / 1e9, flop / best / 1e9 / 74.45);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
