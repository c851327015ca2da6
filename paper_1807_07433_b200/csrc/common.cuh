// Shared device helpers for the rsr kernels (sm_100a).
#pragma once
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

#define RSR_DEVINL __device__ __forceinline__

// Bounds checks of our own (compute-sanitizer is closed on this GPU pool): built with
// -DRSR_CHECKS (tools/checked_run.sh builds librsr_checked.so), every RSR_CHECK that
// fails prints its file, line and condition and traps the kernel; in the product build
// it compiles to nothing.
#ifdef RSR_CHECKS
#include <cstdio>
#define RSR_CHECK(cond)                                                                     \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("rsr check failed: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define RSR_CHECK(cond) \
  do {                  \
  } while (0)
#endif

namespace rsr {

// Packed fp32x2 FMA (SASS FFMA2) with a scalar operand broadcast to both lanes:
// acc.{x,y} = fma(w, v.{x,y}, acc.{x,y}).  sm_100a only.
RSR_DEVINL void ffma2_bcast(float2& acc, float w, float2 v) {
  unsigned long long a, vv, wb;
  asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1,%2};" : "=l"(vv) : "f"(v.x), "f"(v.y));
  asm("mov.b64 %0, {%1,%1};" : "=l"(wb) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(wb), "l"(vv));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(a));
}

RSR_DEVINL float ex2_approx(float x) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the MUFU pipe, flushing subnormal results to 0 (one MUFU.EX2, no
// range-reduction fix-up); exp2(-inf) = +0.
RSR_DEVINL float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 arithmetic (FFMA2 / FMUL2 family), element-wise.
RSR_DEVINL unsigned long long f2pack(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
RSR_DEVINL float2 f2unpack(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
RSR_DEVINL float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)), "l"(f2pack(c)));
  return f2unpack(d);
}
RSR_DEVINL float2 f2mul(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)));
  return f2unpack(d);
}

RSR_DEVINL float2 f2add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)));
  return f2unpack(d);
}
RSR_DEVINL float2 f2sub(float2 a, float2 b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)));
  return f2unpack(d);
}

// Clamp to [-1, 1], propagating NaN (max.NaN / min.NaN: one FMNMX each).
RSR_DEVINL float clamp_unit_nan(float c) {
  float t, r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(t) : "f"(c), "f"(-1.f));
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(t), "f"(1.f));
  return r;
}

RSR_DEVINL float qnan() { return __int_as_float(0x7fffffff); }

// 1/x on the MUFU pipe (rcp.approx.ftz, <= 1 ulp): the bilateral normalisation of
// every K3 variant (sliding, small-slab, fused) -- one instruction instead of the
// IEEE __frcp_rn sequence; 1/0 = +inf, so a zero weight sum still gives NaN.
RSR_DEVINL float rcp_fast(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Clamp to [-1, 1] keeping NaN (fminf/fmaxf would drop it).
RSR_DEVINL float clamp_unit_keep_nan(float c) {
  return c > 1.f ? 1.f : (c < -1.f ? -1.f : c);
}

// ---- mbarrier + 1-D bulk async copy (TMA engine, cp.async.bulk) ----------
RSR_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte asynchronous global -> shared copy (cp.async, LDGSTS); completion tracked
// by an mbarrier through cp_async_mbar_arrive_noinc
RSR_DEVINL void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

// 16-byte asynchronous global -> shared copy (cp.async.cg, L2 only), group-tracked
RSR_DEVINL void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
// 4-byte asynchronous global -> shared copy (cp.async.ca, LDGSTS), group-tracked.  No
// memory clobber: callers order the copy against shared-memory reads of its slot with
// a CTA barrier (and cp_async_wait_* before reading), both of which are compiler fences.
RSR_DEVINL void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc));
}
RSR_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
RSR_DEVINL void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// every committed group but the most recent one has landed (this thread's copies)
RSR_DEVINL void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// arrive on bar once every cp.async this thread issued so far has landed (counts as
// one of the barrier's expected arrivals)
RSR_DEVINL void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
RSR_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
RSR_DEVINL void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
RSR_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Wait for the mbarrier phase with the given parity.  A bounded spin: a
// protocol error traps (kernel fails loudly) instead of hanging the GPU.
RSR_DEVINL void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spins = 0;; spins++) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (spins > (1u << 24)) __trap();
  }
}
// global -> shared bulk copy completing on `bar` (bytes multiple of 16, 16-B aligned)
RSR_DEVINL void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Raise a kernel's dynamic shared-memory limit to at least `bytes` (host).  The
// limit is a property of the kernel, not of one launch, so it only ever grows
// (monotonic maximum per kernel and device, under a mutex): a concurrent call
// that needs less can never have its limit lowered under it (include/rsr.h:
// calls on different streams and host threads are safe).
inline cudaError_t smem_optin(const void* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& g = granted[{kern, dev}];
  if (g >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  g = bytes;
  return cudaSuccess;
}

}  // namespace rsr
