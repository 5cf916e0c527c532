// Microbenchmark: does TMA multicast inside a thread-block cluster deliver
// more bytes to the SMs than the L2 -> SM cap of unicast copies?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_mcast tools/mb_mcast.cu
//   tools/mb_mcast <tile_bytes> <slots> <iters>
//
// Every CTA receives `iters` tiles of `tile_bytes` into an S-slot ring (a
// consumer warp waits and frees each slot; no arithmetic).  The source is a
// 64 MB L2-resident buffer.  Modes, for cluster size CS:
//   unicast-distinct : each CTA copies its own tiles (the baseline cap);
//   unicast-shared   : the CS CTAs of a cluster copy the SAME tiles at about
//                      the same time (does L2 de-duplicate them?);
//   multicast        : tile k of a cluster is copied once, by CTA k % CS, with
//                      .multicast::cluster into the same slot of all CS CTAs.
// Ring protocol (multicast): slot s is always issued by CTA s % CS; every
// CTA's consumer, after waiting full[s], re-arms its own full[s] with
// arrive.expect_tx for the next round and then arrives remotely on the
// issuer's empty[s] (count CS); the issuer waits empty[s] before re-issuing.
// Reported: bytes delivered into shared memory per second, summed over CTAs.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void wait_parity(uint64_t* bar, uint32_t ph) {
  asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(
                   su32(bar)),
               "r"(ph)
               : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
// arrive on the barrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void remote_arrive(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

template <int MODE, int CS>  // MODE 0 unicast-distinct, 1 unicast-shared, 2 multicast
__global__ void ring(const char* __restrict__ buf, size_t buf_bytes, int tile, int S, int iters) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + (size_t)S * tile);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  const uint32_t cluster = blockIdx.x / CS;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(MODE == 2 ? CS : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < S; ++i) expect_tx(&full[i], tile);  // arm round 0
  }
  if (CS > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  const size_t ntiles = buf_bytes / tile;
  if (tid == 32) {  // producer
    for (int k = 0; k < iters; ++k) {
      const int slot = k % S;
      const int use = k / S;
      if (MODE == 2 && (uint32_t)(slot % CS) != rank) continue;  // another CTA issues this slot
      if (use > 0) wait_parity(&empty[slot], (use - 1) & 1);
      const size_t who = MODE == 0 ? (size_t)blockIdx.x : (size_t)cluster;
      const size_t t = (who * 7919 + (size_t)k * 104729) % ntiles;
      if (MODE == 2) {
        const uint16_t mask = (uint16_t)((1u << CS) - 1);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
            "%4;" ::"r"(su32(sm + (size_t)slot * tile)),
            "l"(buf + t * tile), "r"(tile), "r"(su32(&full[slot])), "h"(mask)
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(sm + (size_t)slot * tile)),
            "l"(buf + t * tile), "r"(tile), "r"(su32(&full[slot]))
            : "memory");
      }
    }
  } else if (tid == 0) {  // consumer
    for (int k = 0; k < iters; ++k) {
      const int slot = k % S;
      wait_parity(&full[slot], (k / S) & 1);
      if (k + S < iters) expect_tx(&full[slot], tile);  // re-arm for the next round
      if (MODE == 2) remote_arrive(&empty[slot], slot % CS);
      else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[slot])) : "memory");
    }
  }
  if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, int CS>
static double run(const char* buf, size_t bytes, int tile, int S, int iters, int nsm) {
  const size_t smem = (size_t)S * tile + 16 * S;
  cudaFuncSetAttribute(ring<MODE, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((nsm / CS) * CS);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, ring<MODE, CS>, buf, bytes, tile, S, iters);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, ring<MODE, CS>, buf, bytes, tile, S, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(err));
    exit(1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return (double)cfg.gridDim.x * iters * tile / (ms * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  const int tile = argc > 1 ? atoi(argv[1]) : 49152;
  const int S = argc > 2 ? atoi(argv[2]) : 4;
  const int iters = argc > 3 ? atoi(argv[3]) : 2000;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 64ull << 20;
  char* buf = nullptr;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  printf("tile %d B, %d slots, %d tiles per CTA, %d SMs; TB/s delivered into shared memory\n", tile, S, iters, nsm);
  printf("unicast distinct   CS=1: %.2f\n", run<0, 1>(buf, bytes, tile, S, iters, nsm));
  printf("unicast distinct   CS=2: %.2f\n", run<0, 2>(buf, bytes, tile, S, iters, nsm));
  printf("unicast shared     CS=2: %.2f\n", run<1, 2>(buf, bytes, tile, S, iters, nsm));
  printf("unicast shared     CS=4: %.2f\n", run<1, 4>(buf, bytes, tile, S, iters, nsm));
  printf("multicast          CS=2: %.2f\n", run<2, 2>(buf, bytes, tile, S, iters, nsm));
  printf("multicast          CS=4: %.2f\n", run<2, 4>(buf, bytes, tile, S, iters, nsm));
  return 0;
}
