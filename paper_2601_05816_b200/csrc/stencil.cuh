// Device building blocks of the Wilson hopping term shared by the generic
// (LDG) and the TMA-pipelined (cp.async.bulk -> smem) kernels.
#pragma once
#include "common.cuh"
#include "layout.cuh"

namespace b200wd {

// A_mu blocks of the chiral basis as (permutation, unit phase code)
// (projectors.py:40-48, 88-92).  Phase codes: 0:+1 1:+i 2:-1 3:-i.
__host__ __device__ constexpr int a_perm(int mu, int s) { return (mu == 1 || mu == 2) ? 1 - s : s; }
__host__ __device__ constexpr int a_code(int mu, int s) {
  return mu == 0 ? 0 : mu == 1 ? 1 : mu == 2 ? (s == 0 ? 0 : 2) : (s == 0 ? 1 : 3);
}
// A_mu^H has the same permutation; its phases are the conjugates.
__host__ __device__ constexpr int adj_code(int mu, int s) {
  return mu == 0 ? 0 : mu == 1 ? 3 : mu == 2 ? (s == 0 ? 2 : 0) : (s == 0 ? 3 : 1);
}

struct HopParams {
  int32_t T, X, Y, Z;
  int32_t par0;        // parity of local slice 0 (t_origin & 1)
  int32_t b;           // rhs count
  int32_t dst_parity;  // -1: full lattice
  int64_t n;           // local sites
  int64_t n_src, n_dst;
  int64_t d_begin, d_end;  // destination index range in the dst field
  int64_t per_t;           // X*Y*Z
  int64_t nf;              // face sites of the src field
  const void* U;
  const void* src;
  const void* xself;
  void* out;
  double alpha, beta;  // beta carries the 1/2 of the projectors
  const double* scale;
  const void* lam_halo;
  const void* chi_halo;
  // site-local term (clover, dirac.py:137-157): packed Hermitian 6x6 blocks,
  // 2 x 21 complex per dst site (layout.cuh clover_base).  mode 1:
  // out = s (alpha x - M x + beta H src); mode 2: out = s M (alpha x + beta H src)
  const void* clov;
  int32_t clov_mode;
  // ring-kernel traversal order (0 = natural site order): items sweep the T
  // slices of one tile_x x tile_y patch of z lines before the next patch, so
  // the t-1 / t / t+1 slices of the patch stay in L2 (lattices whose T slice
  // is larger than L2).  tile_nt = slices in [d_begin, d_end).
  int32_t tile_x, tile_y, tile_nt;
  // L2 policy of the t+1 neighbour tile copies: 0 default, 1 evict-first (a T
  // slice exceeds L2: no reuse before eviction), 2 evict-last (patched order:
  // the blocks return as own blocks one patch slice later)
  int32_t hint_t1;
  int32_t hint_tm1;  // 1: the t-1 neighbour tile (its last use) is copied evict-first
  // device stop flag of a GMRES cycle enqueued without host round trips
  // (b200wd_gmres_cycle): when *stop != 0 at launch the kernel does nothing
  const int* stop;
  // wave-synchronised traversal (patched order, lattices whose T slice exceeds
  // L2): items [k*wave_items, (k+1)*wave_items) form wave k (one patch slice);
  // a producer issues no item of wave k before every item of wave k-wave_slack
  // was issued (per-wave counters in wave_cnt, zeroed before the launch), so
  // the CTAs march the patch's slices together and a block loaded as a t+1
  // neighbour is still in L2 when it is read as an own block and as a t-1
  // neighbour.  Only a locality hint: the wait is bounded and never needed
  // for correctness.  wave_cnt == nullptr: off.
  int* wave_cnt;
  int64_t wave_items;
  int32_t wave_slack;
  // both T-split boundary slices in one launch: destination field indices
  // d >= d_begin + jump_at are shifted by jump_by (skipping the interior
  // slices); the range [d_begin, d_end) counts the two slices only.  0: off
  int64_t jump_at, jump_by;
};

// bounded wait until wave w-slack is complete; false once a wait timed out
// (then the caller stops synchronising: e.g. a CTA that is not co-resident)
__device__ __forceinline__ bool wave_wait(const HopParams& p, int64_t it, int64_t n_items) {
  const int64_t w = it / p.wave_items - p.wave_slack;
  if (w < 0) return true;
  const int64_t lo = w * p.wave_items;
  const int need = (int)((lo + p.wave_items <= n_items ? p.wave_items : n_items - lo));
  for (int i = 0; i < 4096; ++i) {  // <= ~0.5 ms
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p.wave_cnt + w) : "memory");
    if (v >= need) return true;
    __nanosleep(128);
  }
  return false;
}
__device__ __forceinline__ void wave_arrive(const HopParams& p, int64_t it) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(p.wave_cnt + it / p.wave_items) : "memory");
}

__device__ __forceinline__ bool hop_stopped(const HopParams& p) {
  return p.stop != nullptr && *static_cast<const volatile int*>(p.stop) != 0;
}

// y = M t for the two packed Hermitian 6x6 blocks of one site (fields.py:212-247:
// lower triangle, row-major, element (i,j), i >= j, at i(i+1)/2 + j)
template <bool GLOBAL = true, typename C>
__device__ __forceinline__ void clover_mul(C (&y)[12], const C (&t)[12], const C* __restrict__ cl) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    C a[21];
#pragma unroll
    for (int e = 0; e < 21; ++e) a[e] = GLOBAL ? __ldg(cl + (q * 21 + e) * 8) : cl[(q * 21 + e) * 8];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      C acc = mk(decltype(t[0].x)(0), decltype(t[0].x)(0));
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const C m = i >= j ? a[i * (i + 1) / 2 + j] : cconj(a[j * (j + 1) / 2 + i]);
        const C v = t[6 * q + j];
        acc = mk(acc.x + m.x * v.x - m.y * v.y, acc.y + m.x * v.y + m.y * v.x);
      }
      y[6 * q + i] = acc;
    }
  }
}

// ---- V-wide loads/stores of consecutive rhs ---------------------------------
template <typename R, int V> struct VecIO;
template <> struct VecIO<double, 1> {
  static __device__ __forceinline__ void ld(double2 (&o)[1], const double2* p) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void lds(double2 (&o)[1], const double2* p) { o[0] = *p; }
  static __device__ __forceinline__ void st(double2* p, const double2 (&v)[1]) { __stcs(p, v[0]); }
};
template <> struct VecIO<double, 2> {
  static __device__ __forceinline__ void ld(double2 (&o)[2], const double2* p) {
    o[0] = __ldg(p);
    o[1] = __ldg(p + 1);
  }
  static __device__ __forceinline__ void lds(double2 (&o)[2], const double2* p) {
    o[0] = p[0];
    o[1] = p[1];
  }
  static __device__ __forceinline__ void st(double2* p, const double2 (&v)[2]) {
    __stcs(p, v[0]);
    __stcs(p + 1, v[1]);
  }
};
template <> struct VecIO<float, 1> {
  static __device__ __forceinline__ void ld(float2 (&o)[1], const float2* p) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void lds(float2 (&o)[1], const float2* p) { o[0] = *p; }
  static __device__ __forceinline__ void st(float2* p, const float2 (&v)[1]) { __stcs(p, v[0]); }
};
template <> struct VecIO<float, 2> {
  static __device__ __forceinline__ void ld(float2 (&o)[2], const float2* p) {
    float4 q = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = make_float2(q.x, q.y);
    o[1] = make_float2(q.z, q.w);
  }
  static __device__ __forceinline__ void lds(float2 (&o)[2], const float2* p) {
    float4 q = *reinterpret_cast<const float4*>(p);
    o[0] = make_float2(q.x, q.y);
    o[1] = make_float2(q.z, q.w);
  }
  static __device__ __forceinline__ void st(float2* p, const float2 (&v)[2]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0].x, v[0].y, v[1].x, v[1].y));
  }
};

// g = M h for the two colour vectors, M = U (DAG=false) or U^H (DAG=true).
template <bool DAG>
__device__ __forceinline__ void matvec2(double2 (&g)[2][3], const double2 (&u)[9],
                                        const double2 (&h)[2][3]) {
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double2 a = mk(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < 3; ++j) a = DAG ? cmacc(a, u[3 * j + i], h[s][j]) : cmac(a, u[3 * i + j], h[s][j]);
      g[s][i] = a;
    }
}
template <bool DAG>
__device__ __forceinline__ void matvec2(float2 (&g)[2][3], const float2 (&u)[9], const float2 (&h)[2][3]) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    float2 hs[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) hs[j] = mk(-h[s][j].y, h[s][j].x);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      float2 a = mk(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 3; ++j)
        a = DAG ? cmacc_s(a, u[3 * j + i], h[s][j], hs[j]) : cmac_s(a, u[3 * i + j], h[s][j], hs[j]);
      g[s][i] = a;
    }
  }
}

// h_s = u_s - sign * A_mu l_s without the 1/2 (projectors.py:126-136);
// FWD is the sign -1 (lambda) projection, !FWD the sign +1 (chi) one.
template <int MU, bool FWD, int S, typename C>
__device__ __forceinline__ void project_spin(C (&h)[3], const C (&psi)[12]) {
  constexpr int code = FWD ? a_code(MU, S) : ((a_code(MU, S) + 2) & 3);
  constexpr int lp = 6 + 3 * a_perm(MU, S);
#pragma unroll
  for (int c = 0; c < 3; ++c) h[c] = cadd(psi[3 * S + c], phase<code>(psi[lp + c]));
}

// acc += reconstruct(g) for sign -1 (FWD: lower += A^H g) or +1 (lower -= A^H g)
// (projectors.py:144-147, dirac.py:258-263)
template <int MU, bool FWD, int S, typename C>
__device__ __forceinline__ void accumulate_spin(C (&acc)[12], const C (&g)[2][3]) {
  constexpr int code = FWD ? adj_code(MU, S) : ((adj_code(MU, S) + 2) & 3);
  constexpr int gp = a_perm(MU, S);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    acc[3 * S + c] = cadd(acc[3 * S + c], g[S][c]);
    acc[6 + 3 * S + c] = cadd(acc[6 + 3 * S + c], phase<code>(g[gp][c]));
  }
}

// One hop from a full neighbour spinor (12 components).  SS / SL: the
// spinor / link pointer is in shared memory (plain loads -> LDS) rather than
// global memory (read-only LDG).
template <int MU, bool FWD, typename R, int V, bool SS = false, bool SL = false, bool GL = false>
__device__ __forceinline__ void hop_full(cx<R> (&acc)[V][12], const cx<R>* __restrict__ sp, int64_t kstride,
                                         const cx<R>* __restrict__ up, int64_t estride) {
  using C = cx<R>;
  C psi[V][12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    C tmp[V];
    if constexpr (SS) VecIO<R, V>::lds(tmp, sp + k * kstride);
    else VecIO<R, V>::ld(tmp, sp + k * kstride);
#pragma unroll
    for (int v = 0; v < V; ++v) psi[v][k] = tmp[v];
  }
  C u[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    if constexpr (GL) u[e] = up[e * estride];  // generic pointer: shared or global
    else u[e] = SL ? up[e * estride] : __ldg(up + e * estride);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    C h[2][3], g[2][3];
    project_spin<MU, FWD, 0>(h[0], psi[v]);
    project_spin<MU, FWD, 1>(h[1], psi[v]);
    matvec2<!FWD>(g, u, h);
    accumulate_spin<MU, FWD, 0>(acc[v], g);
    accumulate_spin<MU, FWD, 1>(acc[v], g);
  }
}

// Split hop for early slot release: (1) hop_load reads the neighbour spinor
// (projected 12 -> 6 as the components arrive) and the 9 link entries from
// shared memory into registers -- after it the ring slot can be handed back
// to the producer --, (2) hop_compute multiplies and reconstructs.
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

// A hand-over of a shared-memory buffer must not become visible before this warp's
// loads from it have returned: mbarrier.arrive is not ordered behind outstanding
// LDS (not even after a MEMBAR -- measured: with the early release below and a
// fast producer the refill's small link copy overtook the last link loads of a
// warp in 13% of the launches on 16x32x16x16, c128 nrhs 32).  Summing a word of
// every loaded value and branching on the sum makes the arrival data-dependent
// on the loads (the branch is never taken for finite data).
template <typename C> __device__ __forceinline__ uint32_t touch_word(const C& v) {
  if constexpr (sizeof(v.x) == 8) return (uint32_t)__double2hiint(v.y);
  else return __float_as_uint(v.y);
}
constexpr uint32_t kTouchMagic = 0x7ff8dea5u;
template <typename R, int V> __device__ __forceinline__ uint32_t hop_touch(const HopRegs<R, V>& d) {
  uint32_t s = 0;
#pragma unroll
  for (int e = 0; e < 9; ++e) s += touch_word(d.u[e]);
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int c = 0; c < 3; ++c) s += touch_word(d.h[v][q][c]);
  return s;
}
__device__ __forceinline__ void arrive_after(uint64_t* bar, uint32_t chk) {
  if (chk == kTouchMagic) __nanosleep(20);  // never for finite data; keeps the dependency
  mbar_arrive(bar);
}


// g = M h for ONE colour vector (the per-spin half of matvec2, same operation order)
template <bool DAG>
__device__ __forceinline__ void matvec1(double2 (&g)[3], const double2 (&u)[9], const double2 (&h)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double2 a = mk(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 3; ++j) a = DAG ? cmacc(a, u[3 * j + i], h[j]) : cmac(a, u[3 * i + j], h[j]);
    g[i] = a;
  }
}
template <bool DAG>
__device__ __forceinline__ void matvec1(float2 (&g)[3], const float2 (&u)[9], const float2 (&h)[3]) {
  float2 hs[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) hs[j] = mk(-h[j].y, h[j].x);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float2 a = mk(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 3; ++j) a = DAG ? cmacc_s(a, u[3 * j + i], h[j], hs[j]) : cmac_s(a, u[3 * i + j], h[j], hs[j]);
    g[i] = a;
  }
}
// hop_compute with the buffer release in the middle: the first spin half of the
// product has consumed every link entry and h[.][0]; together with a word of
// h[.][1] the arrival then depends on every load of hop_load.
template <int MU, bool FWD, typename R, int V>
__device__ __forceinline__ void hop_compute_release(cx<R> (&acc)[V][12], const HopRegs<R, V>& d, uint64_t* bar,
                                                    bool lead) {
  using C = cx<R>;
  C g[V][2][3];
  uint32_t chk = 0;
  if constexpr (sizeof(R) == 8) {
    // complex128: release after the first spin half (FP64 work left to overlap the refill)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      matvec1<!FWD>(g[v][0], d.u, d.h[v][0]);
#pragma unroll
      for (int c = 0; c < 3; ++c) chk += touch_word(g[v][0][c]) + touch_word(d.h[v][1][c]);
    }
    __syncwarp();
    if (lead) arrive_after(bar, chk);
#pragma unroll
    for (int v = 0; v < V; ++v) matvec1<!FWD>(g[v][1], d.u, d.h[v][1]);
  } else {
    // complex64: the product is short (packed FP32); splitting it cost the ring 11%,
    // so release after the whole product, before the reconstruction
#pragma unroll
    for (int v = 0; v < V; ++v) {
      matvec2<!FWD>(g[v], d.u, d.h[v]);
#pragma unroll
      for (int c = 0; c < 3; ++c) chk += touch_word(g[v][0][c]) + touch_word(g[v][1][c]);
    }
    __syncwarp();
    if (lead) arrive_after(bar, chk);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    accumulate_spin<MU, FWD, 0>(acc[v], g[v]);
    accumulate_spin<MU, FWD, 1>(acc[v], g[v]);
  }
}

// Forward T hop whose projected half spinor comes from the lam halo face.
// SS / SL: face / link in shared memory (the ring kernel's halo tiles).
template <typename R, int V, bool SS = false, bool SL = false>
__device__ __forceinline__ void hop_lam_halo(cx<R> (&acc)[V][12], const cx<R>* __restrict__ hp, int64_t hstride,
                                             const cx<R>* __restrict__ up, int64_t estride) {
  using C = cx<R>;
  C hh[V][6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    C tmp[V];
    if constexpr (SS) VecIO<R, V>::lds(tmp, hp + k * hstride);
    else VecIO<R, V>::ld(tmp, hp + k * hstride);
#pragma unroll
    for (int v = 0; v < V; ++v) hh[v][k] = tmp[v];
  }
  C u[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) u[e] = SL ? up[e * estride] : __ldg(up + e * estride);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    C h[2][3], g[2][3];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int c = 0; c < 3; ++c) h[s][c] = hh[v][3 * s + c];
    matvec2<false>(g, u, h);
    accumulate_spin<0, true, 0>(acc[v], g);
    accumulate_spin<0, true, 1>(acc[v], g);
  }
}

// Backward T hop whose U^H-multiplied half spinor comes from the chi face.
template <typename R, int V, bool SS = false>
__device__ __forceinline__ void hop_chi_halo(cx<R> (&acc)[V][12], const cx<R>* __restrict__ hp, int64_t hstride) {
  using C = cx<R>;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    C tmp[V];
    if constexpr (SS) VecIO<R, V>::lds(tmp, hp + k * hstride);
    else VecIO<R, V>::ld(tmp, hp + k * hstride);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      // sign +1 reconstruction with A_0 = I: upper += g, lower -= g
      acc[v][k] = cadd(acc[v][k], tmp[v]);
      acc[v][6 + k] = csub(acc[v][6 + k], tmp[v]);
    }
  }
}

}  // namespace b200wd
