// Shared device helpers for libb200wd (sm_100a only).
//
// Complex numbers are double2 (c128) or float2 (c64).  For c64 the complex
// multiply-accumulate uses the Blackwell packed FP32 pipe (fma.rn.f32x2 ->
// SASS FFMA2): (re,im) of one complex number ride in one 64-bit register
// pair, the link entry is broadcast as a scalar, so one complex MAC is two
// FFMA2 instead of four FFMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <tuple>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libb200wd targets sm_100a only"
#endif

namespace b200wd {

template <typename R> struct cx_t;
template <> struct cx_t<double> { using type = double2; };
template <> struct cx_t<float>  { using type = float2; };
template <typename R> using cx = typename cx_t<R>::type;

__device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
__device__ __forceinline__ float2  mk(float a, float b)  { return make_float2(a, b); }

// ---- packed f32x2 helpers (PTX ISA 8.6+, sm_100+) --------------------------
__device__ __forceinline__ unsigned long long pk(float2 a) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long r) {
  float2 o;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
  return upk(r);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
  return upk(r);
}

// ---- complex arithmetic ----------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return add2(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return sub2(a, b); }

// acc + u*h
__device__ __forceinline__ double2 cmac(double2 acc, double2 u, double2 h) {
  acc.x = fma(u.x, h.x, acc.x);
  acc.x = fma(-u.y, h.y, acc.x);
  acc.y = fma(u.x, h.y, acc.y);
  acc.y = fma(u.y, h.x, acc.y);
  return acc;
}
// acc + conj(u)*h
__device__ __forceinline__ double2 cmacc(double2 acc, double2 u, double2 h) {
  acc.x = fma(u.x, h.x, acc.x);
  acc.x = fma(u.y, h.y, acc.x);
  acc.y = fma(u.x, h.y, acc.y);
  acc.y = fma(-u.y, h.x, acc.y);
  return acc;
}
// float: hs = i*h = (-h.y, h.x) is formed once per h and reused for 3 rows
__device__ __forceinline__ float2 cmac_s(float2 acc, float2 u, float2 h, float2 hs) {
  acc = fma2(mk(u.x, u.x), h, acc);
  return fma2(mk(u.y, u.y), hs, acc);
}
// conj(u)*h = u.x*h - u.y*(i h)
__device__ __forceinline__ float2 cmacc_s(float2 acc, float2 u, float2 h, float2 hs) {
  acc = fma2(mk(u.x, u.x), h, acc);
  return fma2(mk(-u.y, -u.y), hs, acc);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
template <typename C> __device__ __forceinline__ C cscale(C a, decltype(a.x) s) { return mk(a.x * s, a.y * s); }
template <typename C> __device__ __forceinline__ C cconj(C a) { return mk(a.x, -a.y); }
template <typename C> __device__ __forceinline__ C czero() { return mk(decltype(C{}.x)(0), decltype(C{}.x)(0)); }

// multiply by a unit phase code: 0:+1 1:+i 2:-1 3:-i  (free: swap/negate)
template <int CODE, typename C> __device__ __forceinline__ C phase(C a) {
  if constexpr (CODE == 0) return a;
  else if constexpr (CODE == 1) return mk(-a.y, a.x);
  else if constexpr (CODE == 2) return mk(-a.x, -a.y);
  else return mk(a.y, -a.x);
}

// ---- read-only, streaming loads --------------------------------------------
template <typename T> __device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(float2* p, float2 v) { __stcs(p, v); }

}  // namespace b200wd

// ---- TMA bulk copies and mbarriers (sm_90+ async proxy, used on sm_100a) ----
namespace b200wd {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifndef B200WD_WAIT_HINT_NS
#define B200WD_WAIT_HINT_NS 0  // experiment: try_wait suspend-time hint (0: none)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if B200WD_WAIT_HINT_NS > 0
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "B200WD_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra B200WD_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"((uint32_t)B200WD_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "B200WD_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra B200WD_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}
// one non-blocking test of a phase (true: the phase with this parity completed)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// L2 prefetch of a contiguous range by the bulk-copy engine (no smem, no registers)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 16-byte LDGSTS copy global -> shared (L1-bypassing) and its completion as an
// arrival on an mbarrier: the arrive fires once every earlier cp.async of the
// executing thread has landed and takes one of the barrier's expected arrivals
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// L2 eviction-priority policies for the bulk copies (createpolicy)
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
}  // namespace b200wd

// ---- per-device launch facts (host) -----------------------------------------
// A process may drive several GPUs (and several host threads may launch), so
// the dynamic shared-memory attribute, the occupancy of a (kernel, block,
// smem) shape and the SM count are cached per device ordinal under a mutex.
namespace b200wd {
struct LaunchFacts {
  int occ = 0;       // resident CTAs per SM (0: the shape does not fit)
  int sm_count = 0;  // SMs of the current device
};
inline bool launch_facts(const void* fn, int threads, size_t smem, LaunchFacts& out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, LaunchFacts> facts;
  static std::map<std::pair<const void*, int>, size_t> attr;  // dynamic smem attribute set per (kernel, device)
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(fn, dev, threads, smem);
  auto it = facts.find(key);
  if (it != facts.end()) {
    out = it->second;
    return out.occ > 0;
  }
  size_t& a = attr[std::make_pair(fn, dev)];
  if (smem > 48 * 1024 && a < smem) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    a = smem;
  }
  LaunchFacts f;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f.occ, fn, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    f.occ = 0;
  }
  cudaDeviceGetAttribute(&f.sm_count, cudaDevAttrMultiProcessorCount, dev);
  facts[key] = f;
  out = f;
  return f.occ > 0;
}
// SMs a persistent grid may cover: all of them less the calling thread's
// reserve (b200wd_set_sm_reserve), at least one
int persistent_sms(int sm_count);
}  // namespace b200wd
