// Microbenchmark: L2 -> SM bandwidth of cp.async.bulk (TMA 1-D) rings.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tma tools/mb_tma.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ring(const char* __restrict__ buf, size_t buf_bytes, int tile, int S, long long tiles_per_cta,
                     int consumers, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)S * tile);
  uint64_t* empty = full + S;
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(consumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  size_t ntiles = buf_bytes / tile;
  if (tid == consumers * 32) {
    for (long long k = 0; k < tiles_per_cta; ++k) {
      int slot = k % S; long long use = k / S;
      if (use > 0) {
        uint32_t ph = (use - 1) & 1;
        asm volatile("{.reg .pred p; W1_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W1_%=;}" ::"r"(su32(&empty[slot])), "r"(ph) : "memory");
      }
      size_t t = ((size_t)blockIdx.x * 7919 + (size_t)k * 104729) % ntiles;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[slot])), "r"(tile) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)slot * tile)), "l"(buf + t * tile), "r"(tile), "r"(su32(&full[slot])) : "memory");
    }
  } else if (tid < consumers * 32) {
    unsigned long long acc = 0;
    for (long long k = 0; k < tiles_per_cta; ++k) {
      int slot = k % S; uint32_t ph = (k / S) & 1;
      asm volatile("{.reg .pred p; W2_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2_%=;}" ::"r"(su32(&full[slot])), "r"(ph) : "memory");
      acc += sm[(size_t)slot * tile + (tid * 64) % tile];
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

int main(int argc, char** argv) {
  int sms = 148;
  size_t big = (size_t)4 << 30, small = (size_t)48 << 20;
  char* buf; cudaMalloc(&buf, big); cudaMemset(buf, 1, big);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int tiles[] = {8192, 24576, 49152};
  int Ss[] = {2, 4, 8};
  int ctas[] = {1, 2};
  for (int src = 0; src < 2; ++src) {
    size_t bb = src ? small : big;
    for (int tile : tiles) for (int S : Ss) for (int c : ctas) {
      size_t smem = (size_t)S * tile + 16 * S;
      if (smem * c > 227 * 1024) continue;
      cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      long long per = (long long)(2e9 / tile / (sms * c));
      int grid = sms * c;
      ring<<<grid, 160, smem>>>(buf, bb, tile, S, 8, 4, sink);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      ring<<<grid, 160, smem>>>(buf, bb, tile, S, per, 4, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t e = cudaGetLastError();
      double bytes = (double)per * grid * tile;
      printf("%s tile %6d S %d ctas/SM %d : %8.1f GB/s  (in flight/SM <= %zu KB) %s\n", src ? "L2 " : "HBM", tile, S, c,
             bytes / ms / 1e6, (size_t)S * tile * c / 1024, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
