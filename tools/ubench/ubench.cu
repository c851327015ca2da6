// Micro-benchmarks that fix the roofline denominators and the K3 (bilateral
// aggregation) design choices on sm_100a:
//   * FP32 FMA throughput: scalar FFMA vs packed FFMA2 (fma.rn.f32x2), with the
//     scalar-broadcast operand form the aggregation inner loop uses.
//   * shared-memory LDS.128 wavefront cost for the lane patterns K3 can use
//     (warp-uniform, quarter-uniform, 4-distinct, all-distinct).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float2 upk(unsigned long long v) {
  float2 r; asm("mov.b64 {%0,%1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v)); return r; }

template <int NACC>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = threadIdx.x * 1e-3f + i;
  float x = a + threadIdx.x * 1e-7f, y = b;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], x, y);
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fmaf(acc[i], y, x);
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// outer-product FFMA: acc[i][j] += w[i] * c[j]  (the K3 pattern), operands vary per iter
__global__ void k_ffma_outer(float* out, int iters) {
  float acc[8][8];
  float w[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { w[i] = 1e-3f * (threadIdx.x + i); c[i] = 1e-3f * i; }
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = fmaf(w[i], c[j], acc[i][j]);
#pragma unroll
    for (int i = 0; i < 8; i++) { w[i] = w[i] * 0.999f; c[i] = c[i] + 1e-7f; }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) s += acc[i][j];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// FFMA2 with scalar broadcast first operand: acc2[i][j] += w[i] * {c[2j], c[2j+1]}
__global__ void k_ffma2_outer(float* out, int iters) {
  unsigned long long acc[8][4];
  float w[8]; unsigned long long c[4];
#pragma unroll
  for (int i = 0; i < 8; i++) w[i] = 1e-3f * (threadIdx.x + i);
#pragma unroll
  for (int j = 0; j < 4; j++) c[j] = pk(1e-3f * j, 2e-3f * j);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0ull;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        unsigned long long wb = pk(w[i], w[i]);
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i][j]) : "l"(wb), "l"(c[j]));
      }
#pragma unroll
    for (int i = 0; i < 8; i++) w[i] = w[i] * 0.999f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) { float2 v = upk(acc[i][j]); s += v.x + v.y; }
  if (s == 12345.f) out[threadIdx.x] = s;
}

// LDS.128 throughput for a lane->address pattern. mode:
//  0 warp-uniform, 1 quarter-uniform (lane>>3), 2 lane&3 (4 distinct, spread over quarters),
//  3 all distinct contiguous (lane*16B), 4 lane>>2 (8 distinct, 4 lanes each)
__global__ void k_lds(float* out, int iters, int mode) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 1e-3f;
  __syncthreads();
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int slot;
  switch (mode) {
    case 0: slot = 0; break;
    case 1: slot = (lane >> 3) * 8 + (lane >> 3); break;   // 4 addrs in distinct bank groups
    case 2: slot = (lane & 3) * 9; break;
    case 3: slot = lane; break;
    default: slot = (lane >> 2) * 1; break;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  const float4* base = reinterpret_cast<const float4*>(sm) + wid * 64;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      float4 v = base[(slot + u * 40 + it * 8) & 255];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[threadIdx.x] = acc.x;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"regs_per_sm\": %d}\n",
         p.name, sms, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  float* out; CK(cudaMalloc(&out, 4096));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch, double flop_or_ops, const char* name, const char* unit) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"test\": \"%s\", \"ms\": %.4f, \"rate\": %.3f, \"unit\": \"%s\"}\n", name, best, flop_or_ops / (best * 1e-3) / 1e12, unit);
  };
  int blocks = sms * 4, threads = 256, iters = 4096;
  // FFMA chains: 2*NACC fma per iter
  timeit([&] { k_ffma<16><<<blocks, threads>>>(out, iters, 1.0001f, 0.999f); },
         2.0 * blocks * threads * iters * 32, "ffma_chain16", "TFLOP/s");
  timeit([&] { k_ffma_outer<<<blocks, threads>>>(out, iters); },
         2.0 * blocks * threads * iters * 64, "ffma_outer8x8", "TFLOP/s");
  timeit([&] { k_ffma2_outer<<<blocks, threads>>>(out, iters); },
         2.0 * blocks * threads * iters * 64, "ffma2_outer8x4x2", "TFLOP/s");
  // LDS: 16 LDS.128 per iter per thread; report warp-instructions per SM per clock-free (per ns)
  for (int mode = 0; mode < 5; mode++) {
    char nm[64]; snprintf(nm, 64, "lds128_mode%d", mode);
    timeit([&] { k_lds<<<blocks, threads>>>(out, iters, mode); },
           1.0 * blocks * (threads / 32) * iters * 16 / sms, nm, "Twarp-instr/s/SM");
  }
  CK(cudaGetLastError());
  return 0;
}
