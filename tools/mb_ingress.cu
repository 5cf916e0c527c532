// Microbenchmark: bytes per second an SM can pull from L2 / HBM into shared
// memory through (a) the TMA bulk-copy engine, (b) cp.async (LDGSTS, issued by
// the 32 lanes of a producer warp through the LSU / L1 path), (c) both at
// once (alternate tiles).  Question for the hop kernels: is the per-SM bulk
// copy engine the ring's limit, and does a second load path add throughput?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_ingress tools/mb_ingress.cu
//   tools/mb_ingress
//
// One CTA per SM: warp 0 consumes (waits full[s], frees empty[s] at once),
// warp 1 produces into an S-slot ring.  Full barriers expect 32 arrivals: a
// TMA tile is lane 0's arrive.expect_tx plus 31 plain arrivals, an LDGSTS tile
// the 32 lanes' cp.async.mbarrier.arrive.noinc.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));          \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t ph) {
  asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(
                   su32(bar)),
               "r"(ph)
               : "memory");
}

template <int MODE>  // 0 TMA, 1 LDGSTS, 2 alternate, 3 TMA tile + a 2304-byte second copy (the ring's link plane), 4 TMA tile as two half copies
__global__ void __launch_bounds__(64, 1) ring(const char* __restrict__ buf, size_t buf_bytes, int tile, int S,
                                              int iters) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)S * tile);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t ntiles = buf_bytes / tile;
  if (tid >= 32) {  // producer warp
    for (int k = 0; k < iters; ++k) {
      const int slot = k % S, use = k / S;
      if (use > 0) wait_parity(&empty[slot], (use - 1) & 1);
      const size_t t = ((size_t)blockIdx.x * 7919 + (size_t)k * 104729) % ntiles;
      const char* src = buf + t * tile;
      unsigned char* dst = sm + (size_t)slot * tile;
      const bool tma = MODE == 0 || MODE >= 3 || (MODE == 2 && (k & 1) == 0);
      if (tma && MODE >= 3) {
        if (lane == 0) {
          const int a = MODE == 3 ? tile - 2304 : tile / 2;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(tile)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(dst)),
              "l"(src), "r"(a), "r"(su32(&full[slot]))
              : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(dst + a)),
              "l"(buf + ((t * 31 + 17) % ntiles) * tile), "r"(tile - a), "r"(su32(&full[slot]))
              : "memory");
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[slot])) : "memory");
        }
      } else if (tma) {
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(tile)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  su32(dst)),
              "l"(src), "r"(tile), "r"(su32(&full[slot]))
              : "memory");
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[slot])) : "memory");
        }
      } else {
        for (int o = lane * 16; o < tile; o += 32 * 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + o)), "l"(src + o) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[slot])) : "memory");
      }
    }
  } else if (tid == 0) {  // consumer
    for (int k = 0; k < iters; ++k) {
      const int slot = k % S;
      wait_parity(&full[slot], (k / S) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
    }
  }
}

template <int MODE>
double run(const char* buf, size_t bytes, int tile, int S, int iters) {
  const size_t smem = (size_t)S * tile + 16 * S;
  CK(cudaFuncSetAttribute(ring<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ring<MODE><<<148, 64, smem>>>(buf, bytes, tile, S, 64);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ring<MODE><<<148, 64, smem>>>(buf, bytes, tile, S, iters);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return 148.0 * iters * tile / (ms * 1e-3) / 1e12;
}

int main() {
  const size_t big = 4ull << 30, small = 64ull << 20;
  char* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 1, big));
  struct {
    int tile, S;
  } cfgs[] = {{98304, 2}, {65536, 3}, {51456, 4}, {49152, 4}, {32768, 6}, {24576, 8}, {12288, 16}};
  for (auto c : cfgs) {
    const int iters = (int)(2ull * 1024 * 1024 * 1024 / 148 / c.tile);
    printf("tile %6d B x %2d slots: L2  TMA %6.2f | tile+2304B copy %6.2f | two halves %6.2f | LDGSTS %6.2f || "
           "HBM TMA %6.2f | tile+2304B %6.2f TB/s\n",
           c.tile, c.S, run<0>(buf, small, c.tile, c.S, iters), run<3>(buf, small, c.tile, c.S, iters),
           run<4>(buf, small, c.tile, c.S, iters), run<1>(buf, small, c.tile, c.S, iters),
           run<0>(buf, big, c.tile, c.S, iters), run<3>(buf, big, c.tile, c.S, iters));
  }
  return 0;
}
