// Microbenchmark: consumer-only throughput of the Wilson hop arithmetic from
// shared memory (no TMA, no HBM traffic): the ceiling the ring / stream
// kernels' consumer warps can reach at a given warp count and code shape.
//
// A CTA holds two ring-style tiles of one item in shared memory (own blocks +
// one neighbour tile read by all six t/x/y hops, each with its link plane) and its consumers
// run the 8 hops of every site over and over.  Reported: site*rhs/s and the
// HBM fraction it would correspond to at the compulsory (24 b + 36) w bytes.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_05816_b200/csrc
//        -Xptxas -v -o tools/mb_consumer tools/mb_consumer.cu
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"

using namespace b200wd;

#define CK(x)                                                         \
  do {                                                                \
    cudaError_t e = (x);                                              \
    if (e != cudaSuccess) {                                           \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

// MODE 0: hop_full (all 12 components + 9 links live, then matvec2)
// MODE 1: ts_hop style (project while loading, one link row at a time)
// MODE 2: paired fwd/bwd of each direction: d = g_f - g_b chain, s = 2 g_f - d
template <int MU, bool FWD, typename R, int V, int KST>
__device__ __forceinline__ void hop_rows(cx<R> (&acc)[V][12], const cx<R>* sp, const cx<R>* up) {
  using C = cx<R>;
  C h[V][2][3];
#pragma unroll
  for (int S = 0; S < 2; ++S)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C a[V], b[V];
      VecIO<R, V>::lds(a, sp + (3 * S + c) * KST);
      VecIO<R, V>::lds(b, sp + (6 + 3 * a_perm(MU, S) + c) * KST);
      constexpr int code0 = FWD ? a_code(MU, 0) : ((a_code(MU, 0) + 2) & 3);
      constexpr int code1 = FWD ? a_code(MU, 1) : ((a_code(MU, 1) + 2) & 3);
#pragma unroll
      for (int v = 0; v < V; ++v) h[v][S][c] = cadd(a[v], S == 0 ? phase<code0>(b[v]) : phase<code1>(b[v]));
    }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    C m[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) m[j] = FWD ? up[(3 * i + j) * 8] : up[(3 * j + i) * 8];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      C g[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        C a = mk(R(0), R(0));
        if constexpr (sizeof(R) == 8) {
#pragma unroll
          for (int j = 0; j < 3; ++j) a = FWD ? cmac(a, m[j], h[v][q][j]) : cmacc(a, m[j], h[v][q][j]);
        } else {
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const C hs = mk(-h[v][q][j].y, h[v][q][j].x);
            a = FWD ? cmac_s(a, m[j], h[v][q][j], hs) : cmacc_s(a, m[j], h[v][q][j], hs);
          }
        }
        g[q] = a;
      }
      constexpr int c0 = FWD ? adj_code(MU, 0) : ((adj_code(MU, 0) + 2) & 3);
      constexpr int c1 = FWD ? adj_code(MU, 1) : ((adj_code(MU, 1) + 2) & 3);
      acc[v][i] = cadd(acc[v][i], g[0]);
      acc[v][3 + i] = cadd(acc[v][3 + i], g[1]);
      acc[v][6 + i] = cadd(acc[v][6 + i], phase<c0>(g[a_perm(MU, 0)]));
      acc[v][9 + i] = cadd(acc[v][9 + i], phase<c1>(g[a_perm(MU, 1)]));
    }
  }
}


// Software-pipelined hop: (1) load + project the neighbour half spinor and
// the 9 link entries into registers, (2) matvec + reconstruct from registers.
template <typename R, int V> struct HopRegs {
  cx<R> h[V][2][3];
  cx<R> u[9];
};
template <int MU, bool FWD, typename R, int V, int KST>
__device__ __forceinline__ void hop_load(HopRegs<R, V>& d, const cx<R>* sp, const cx<R>* up) {
  using C = cx<R>;
#pragma unroll
  for (int S = 0; S < 2; ++S)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C a[V], b[V];
      VecIO<R, V>::lds(a, sp + (3 * S + c) * KST);
      VecIO<R, V>::lds(b, sp + (6 + 3 * a_perm(MU, S) + c) * KST);
      constexpr int code0 = FWD ? a_code(MU, 0) : ((a_code(MU, 0) + 2) & 3);
      constexpr int code1 = FWD ? a_code(MU, 1) : ((a_code(MU, 1) + 2) & 3);
#pragma unroll
      for (int v = 0; v < V; ++v) d.h[v][S][c] = cadd(a[v], S == 0 ? phase<code0>(b[v]) : phase<code1>(b[v]));
    }
#pragma unroll
  for (int e = 0; e < 9; ++e) d.u[e] = up[e * 8];
}
template <int MU, bool FWD, typename R, int V>
__device__ __forceinline__ void hop_compute(cx<R> (&acc)[V][12], const HopRegs<R, V>& d) {
  using C = cx<R>;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    C g[2][3];
    matvec2<!FWD>(g, d.u, d.h[v]);
    accumulate_spin<MU, FWD, 0>(acc[v], g);
    accumulate_spin<MU, FWD, 1>(acc[v], g);
  }
}
__device__ __forceinline__ void fake_wait(uint64_t* bar) { mbar_wait(bar, 0); }

template <typename R, int V, int B, int NB, int MODE, int MINB>
__global__ void __launch_bounds__(B / V * 8 * NB, MINB) consumer(int iters, cx<R>* out) {
  using C = cx<R>;
  constexpr int SPIN = NB * 96 * B, SLOT = SPIN + NB * 72, KST = 8 * B;
  constexpr int NC = B / V * 8 * NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + 2 * SLOT);
  if (threadIdx.x == 0) {  // a completed phase-0 barrier: every wait succeeds at once
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(bar);
  for (int i = threadIdx.x; i < 2 * SLOT; i += NC)
    ring[i] = mk(R(0.001) * R((i * 7919) % 1000), R(0.002) * R((i * 104729) % 1000));
  __syncthreads();
  const int tid = threadIdx.x;
  const int r0 = (tid % (B / V)) * V;
  const int ysite = tid / (B / V);
  const int j = ysite >> 3, lo = ysite & 7;
  const int lofs = j * 72 + lo;
  const int so = j * 96 * B + lo * B + r0;
  C tot[V];  // one running checksum per rhs keeps every accumulator live
#pragma unroll
  for (int v = 0; v < V; ++v) tot[v] = mk(R(0), R(0));
  for (int it = 0; it < iters; ++it) {
    C acc[V][12];
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
    // z hops from the own tile (slot 6), neighbour site inside the item
    const int zp = (ysite + 1) % (8 * NB), zm = (ysite + 8 * NB - 1) % (8 * NB);
    const C* own = ring + SLOT;  // two tiles (own + one neighbour) keep smem from capping occupancy
    if constexpr (MODE == 0) {
      hop_full<3, true, R, V, true, true>(acc, own + (zp >> 3) * 96 * B + (zp & 7) * B + r0, KST, own + SPIN + lofs, 8);
      hop_full<3, false, R, V, true, true>(acc, own + (zm >> 3) * 96 * B + (zm & 7) * B + r0, KST,
                                           own + SPIN + (zm >> 3) * 72 + (zm & 7), 8);
#define HOPH(H) hop_full<((H) >> 1), !((H)&1), R, V, true, true>(acc, ring + so, KST, ring + SPIN + lofs, 8);
      HOPH(0) HOPH(1) HOPH(2) HOPH(3) HOPH(4) HOPH(5)
#undef HOPH
    } else if constexpr (MODE == 2) {  // hop_full with the ring's per-hop wait / syncwarp between hops
      hop_full<3, true, R, V, true, true>(acc, own + (zp >> 3) * 96 * B + (zp & 7) * B + r0, KST, own + SPIN + lofs, 8);
      hop_full<3, false, R, V, true, true>(acc, own + (zm >> 3) * 96 * B + (zm & 7) * B + r0, KST,
                                           own + SPIN + (zm >> 3) * 72 + (zm & 7), 8);
      __syncwarp();
#define HOPH(H) fake_wait(bar); hop_full<((H) >> 1), !((H)&1), R, V, true, true>(acc, ring + so, KST, ring + SPIN + lofs, 8); __syncwarp();
      HOPH(0) HOPH(1) HOPH(2) HOPH(3) HOPH(4) HOPH(5)
#undef HOPH
    } else if constexpr (MODE == 3) {  // pipelined: wait(k+1), load(k+1), compute(k)
      HopRegs<R, V> A, Bq;
      hop_load<3, true, R, V, KST>(A, own + (zp >> 3) * 96 * B + (zp & 7) * B + r0, own + SPIN + lofs);
      hop_load<3, false, R, V, KST>(Bq, own + (zm >> 3) * 96 * B + (zm & 7) * B + r0, own + SPIN + (zm >> 3) * 72 + (zm & 7));
      hop_compute<3, true, R, V>(acc, A);
      fake_wait(bar);
      hop_load<0, true, R, V, KST>(A, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<3, false, R, V>(acc, Bq);
      fake_wait(bar);
      hop_load<0, false, R, V, KST>(Bq, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<0, true, R, V>(acc, A);
      fake_wait(bar);
      hop_load<1, true, R, V, KST>(A, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<0, false, R, V>(acc, Bq);
      fake_wait(bar);
      hop_load<1, false, R, V, KST>(Bq, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<1, true, R, V>(acc, A);
      fake_wait(bar);
      hop_load<2, true, R, V, KST>(A, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<1, false, R, V>(acc, Bq);
      fake_wait(bar);
      hop_load<2, false, R, V, KST>(Bq, ring + so, ring + SPIN + lofs);
      __syncwarp();
      hop_compute<2, true, R, V>(acc, A);
      hop_compute<2, false, R, V>(acc, Bq);
    } else {
      hop_rows<3, true, R, V, KST>(acc, own + (zp >> 3) * 96 * B + (zp & 7) * B + r0, own + SPIN + lofs);
      hop_rows<3, false, R, V, KST>(acc, own + (zm >> 3) * 96 * B + (zm & 7) * B + r0,
                                    own + SPIN + (zm >> 3) * 72 + (zm & 7));
#define HOPH(H) hop_rows<((H) >> 1), !((H)&1), R, V, KST>(acc, ring + so, ring + SPIN + lofs);
      HOPH(0) HOPH(1) HOPH(2) HOPH(3) HOPH(4) HOPH(5)
#undef HOPH
    }
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int k = 0; k < 12; ++k) tot[v] = cadd(tot[v], acc[v][k]);
    __syncwarp();
  }
  C* o = out + ((int64_t)blockIdx.x * NC + tid) * V;
#pragma unroll
  for (int v = 0; v < V; ++v) o[v] = tot[v];
}

template <typename R, int V, int B, int NB, int MODE, int MINB>
void run(const char* name) {
  using C = cx<R>;
  constexpr int NC = B / V * 8 * NB;
  constexpr int SLOT = NB * 96 * B + NB * 72;
  const size_t smem = 2 * SLOT * sizeof(C) + 16;
  auto k = consumer<R, V, B, NB, MODE, MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NC, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  const int grid = 148 * occ;
  C* out;
  CK(cudaMalloc(&out, (size_t)grid * NC * V * sizeof(C)));
  const int iters = 400;
  k<<<grid, NC, smem>>>(10, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, NC, smem>>>(iters, out);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double sr = (double)grid * NC * V * iters / (ms * 1e-3);
  const double w = sizeof(C);
  const double frac = sr * (24.0 + 36.0 / B) * w / 6548.2e9;
  printf("%-34s regs %3d occ %d warps/SM %2d  %.3e site*rhs/s  = HBM frac %.3f\n", name, fa.numRegs, occ,
         occ * NC / 32, sr, frac);
  CK(cudaFree(out));
}

int main() {
  run<double, 1, 16, 2, 0, 1>("c128 b16 NB2 hop_full");
  run<double, 1, 16, 2, 2, 1>("c128 b16 NB2 hop_full+waits");
  run<double, 1, 16, 2, 3, 1>("c128 b16 NB2 pipelined+waits");
  run<double, 1, 16, 2, 2, 2>("c128 b16 NB2 hop_full+waits minb2");
  run<double, 1, 16, 2, 3, 2>("c128 b16 NB2 pipelined+waits minb2");
  run<double, 1, 16, 1, 3, 3>("c128 b16 NB1 pipelined+waits minb3");
  run<double, 1, 12, 2, 2, 1>("c128 b12 NB2 hop_full+waits");
  run<double, 1, 12, 2, 3, 1>("c128 b12 NB2 pipelined+waits");
  run<double, 1, 8, 2, 2, 2>("c128 b8 NB2 hop_full+waits minb2");
  run<double, 1, 8, 2, 3, 2>("c128 b8 NB2 pipelined+waits minb2");
  run<float, 2, 16, 2, 0, 1>("c64 b16 NB2 hop_full");
  run<float, 2, 16, 2, 2, 2>("c64 b16 NB2 hop_full+waits minb2");
  run<float, 2, 16, 2, 3, 2>("c64 b16 NB2 pipelined+waits minb2");
  run<float, 2, 16, 2, 2, 3>("c64 b16 NB2 hop_full+waits minb3");
  run<float, 2, 16, 2, 3, 3>("c64 b16 NB2 pipelined+waits minb3");
  return 0;
}
