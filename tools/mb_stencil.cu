// Microbenchmark: memory-system ceiling of the 9-point (self + 8 neighbours)
// gather pattern of the Wilson stencil in the site-blocked layout, without
// the SU(3) arithmetic.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/mb_stencil.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ long long sbase(long long s, int b) { return (((s >> 3) * 96) + (s & 7)) * (long long)b; }

template <int B, int MODE>
__global__ void __launch_bounds__(128, 3) gather(const double2* __restrict__ src, double2* __restrict__ out,
                                                 const double2* __restrict__ U, int T, int X, int Y, int Z) {
  long long d = (long long)blockIdx.x * blockDim.y + threadIdx.y;
  int r = threadIdx.x;
  int z = d % Z; long long q = d / Z; int y = q % Y; q /= Y; int x = q % X; int t = q / X;
  long long sY = Z, sX = (long long)Y * Z, sT = (long long)X * Y * Z;
  long long nb[8] = {
      (t + 1 == T) ? d - (T - 1) * sT : d + sT, (t == 0) ? d + (T - 1) * sT : d - sT,
      (x + 1 == X) ? d - (X - 1) * sX : d + sX, (x == 0) ? d + (X - 1) * sX : d - sX,
      (y + 1 == Y) ? d - (Y - 1) * sY : d + sY, (y == 0) ? d + (Y - 1) * sY : d - sY,
      (z + 1 == Z) ? d - (Z - 1) : d + 1, (z == 0) ? d + (Z - 1) : d - 1};
  double2 acc[12];
  __shared__ double2 lk[(MODE == 3) ? 576 * (128 / B / 8) : 1];
  if (MODE == 3) {
    // cooperative staging of the links of this CTA's site blocks (own 288 + 4 backward mu-planes)
    const int nsb = 128 / B / 8;
    const long long gb0 = ((long long)blockIdx.x * blockDim.y) >> 3;
    const int tid = threadIdx.y * B + threadIdx.x;
    for (int i = tid; i < 576 * nsb; i += 128) {
      const int jb = i / 576, w = i % 576;
      const long long g = gb0 + jb;
      long long s0 = g * 8;
      int z0 = s0 % Z; long long q0 = s0 / Z; int y0 = q0 % Y; q0 /= Y; int x0 = q0 % X; int t0 = q0 / X;
      double2 v;
      if (w < 288) v = __ldg(U + g * 288 + w);
      else {
        const int mu = (w - 288) / 72, e = (w - 288) % 72;
        long long nbs = mu == 0 ? ((t0 == 0) ? s0 + (T - 1) * sT : s0 - sT)
                      : mu == 1 ? ((x0 == 0) ? s0 + (X - 1) * sX : s0 - sX)
                      : mu == 2 ? ((y0 == 0) ? s0 + (Y - 1) * sY : s0 - sY)
                      : ((z0 == 0) ? s0 + (Z - 8) : s0 - 8);
        v = __ldg(U + (nbs >> 3) * 288 + mu * 72 + e);
      }
      lk[i] = v;
    }
    __syncthreads();
  }
  const double2* sp = src + sbase(d, B) + r;
#pragma unroll
  for (int k = 0; k < 12; ++k) acc[k] = __ldg(sp + k * 8 * B);
  if (MODE >= 1) {
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2* np = src + sbase(nb[h], B) + r;
#pragma unroll
      for (int k = 0; k < 12; ++k) { double2 v = __ldg(np + k * 8 * B); acc[k].x += v.x; acc[k].y += v.y; }
      if (MODE == 3) {
        const int jb = threadIdx.y >> 3, lo = threadIdx.y & 7, mu = h >> 1;
        const double2* up = (h & 1) ? lk + jb * 576 + 288 + mu * 72 + lo : lk + jb * 576 + mu * 72 + lo;
#pragma unroll
        for (int e = 0; e < 9; ++e) { double2 v = up[e * 8]; acc[e].x += v.x; acc[e].y -= v.y; }
      } else if (MODE >= 2) {
        long long ls = (h & 1) ? nb[h] : d;
        const double2* up = U + (ls >> 3) * 288 + (ls & 7) + (h >> 1) * 72;
#pragma unroll
        for (int e = 0; e < 9; ++e) { double2 v = __ldg(up + e * 8); acc[e].x += v.x; acc[e].y -= v.y; }
      }
    }
  }
  double2* op = out + sbase(d, B) + r;
#pragma unroll
  for (int k = 0; k < 12; ++k) __stcs(op + k * 8 * B, acc[k]);
}

template <int B, int MODE>
float run(int T, int X, int Y, int Z, int nbuf, std::vector<double2*>& in, std::vector<double2*>& out, double2* U) {
  long long n = (long long)T * X * Y * Z;
  dim3 blk(B, 128 / B);
  dim3 grid((unsigned)(n / blk.y));
  for (int i = 0; i < 3; ++i) gather<B, MODE><<<grid, blk>>>(in[i % nbuf], out[i % nbuf], U, T, X, Y, Z);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int it = 20;
  cudaEventRecord(e0);
  for (int i = 0; i < it; ++i) gather<B, MODE><<<grid, blk>>>(in[i % nbuf], out[i % nbuf], U, T, X, Y, Z);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / it;
}

int main() {
  const int T = 32, X = 16, Y = 16, Z = 16; const int B = 16;
  long long n = (long long)T * X * Y * Z;
  size_t fb = n * 12 * B * sizeof(double2);
  int nbuf = 3;
  std::vector<double2*> in(nbuf), out(nbuf);
  for (int i = 0; i < nbuf; ++i) { CK(cudaMalloc(&in[i], fb)); CK(cudaMalloc(&out[i], fb)); cudaMemset(in[i], 0, fb); }
  double2* U; CK(cudaMalloc(&U, n * 36 * sizeof(double2))); cudaMemset(U, 0, n * 36 * sizeof(double2));
  const char* names[4] = {"copy (self in, out)", "gather 9 spinors", "gather 9 spinors + links LDG",
                          "gather 9 + links smem-staged"};
  float t0 = run<B, 0>(T, X, Y, Z, nbuf, in, out, U);
  float t1 = run<B, 1>(T, X, Y, Z, nbuf, in, out, U);
  float t2 = run<B, 2>(T, X, Y, Z, nbuf, in, out, U);
  float t3 = run<B, 3>(T, X, Y, Z, nbuf, in, out, U);
  float ts[4] = {t0, t1, t2, t3};
  double alg[4] = {2.0 * fb, 2.0 * fb, 2.0 * fb + n * 36 * 16.0, 2.0 * fb + n * 36 * 16.0};
  for (int m = 0; m < 4; ++m)
    printf("%-28s %8.4f ms  alg %7.1f GB/s  (site*rhs/s %.3e)\n", names[m], ts[m], alg[m] / ts[m] / 1e6, n * B / (ts[m] * 1e-3));
  return 0;
}
