// T-marching column kernel with the t window in registers (full-lattice
// fields), sm_100a.
//
// Why (profiles/r2_ring_exp.txt, tools/ring_exp.sh): the ring kernel moves 7
// tiles per item through the SM's 64 B/clk ingress port and through shared
// memory twice (TMA write + consumer read); with the output stores that data
// path alone takes 0.67 of the roofline time for c128 nrhs 16 and the FP64
// work (~0.55 of it) overlaps it only partly.  A ring without its two t tiles
// (results wrong, timing only) runs 21% faster.
//
// What changes: a CTA owns a column (a z-line segment at fixed x, y) and
// marches along t over a chunk of slices, one consumer thread per (site, V
// rhs) as in the ring.  The thread keeps the t window of its own site in
// REGISTERS:
//   * psi(s+1) is loaded straight from global memory into registers (one
//     128-bit load per component, coalesced across the warp) at the start of
//     step s and lands while the other six hops are computed; it feeds the
//     forward t hop of site s at the end of the step and stays in registers as
//     the own spinor of step s+1 (self term, z hops via a shared-memory copy);
//   * the backward t hop of site s+1, U_0(s)^H P+ psi(s), is finished at step
//     s (U_0(s) is in shared memory for the forward hop anyway) and carried as
//     6 complex per rhs.
// So a step moves 4 neighbour tiles (x+, x-, y+, y-) through the TMA ring plus
// one tile-equivalent through the load/store unit: 5 instead of 7, each own
// spinor is fetched once per apply whatever the size of a T slice, and the
// registers add a tile of bytes in flight to what shared memory holds.  The
// consumers need ~200 registers; a 9-warp CTA is capped at 168 (three warps on
// one SM sub-partition), so the CTA carries a whole producer warpgroup and
// moves its registers to the consumers with setmaxnreg.
//
// Work units are (t-chunk, column) pairs, columns fastest, so the CTAs running
// at one time march neighbouring columns through the same slices and their x/y
// neighbour tiles hit L2.
#pragma once

#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"
#include "tstream.cuh"  // TsGrid, ts_decode, ts_blk, wrapi, ts_choose_nch

namespace b200wd {

template <typename R, int V, int B, int NB> struct MarchShape {
  static constexpr int BT = B / V;                 // threads per site
  static constexpr int SEG = 8 * NB;               // sites per column segment
  static constexpr int NC = BT * SEG;              // consumer threads
  static constexpr int NCW = NC / 32;
  static constexpr bool REALLOC = NC % 128 == 0;   // whole consumer warpgroups: setmaxnreg
  static constexpr int NP = REALLOC ? 128 : 32;    // producer threads (one issues)
  static constexpr int NT = NC + NP;
  static constexpr int MINB = NC <= 128 ? 2 : 1;
  // registers after reallocation (per SM sub-partition: 16384 >= 32 * sum over its warps)
  static constexpr int REG_C = MINB == 2 ? 208 : 232;
  static constexpr int REG_P = 40;
  static constexpr int SPIN = NB * 96 * B;         // spinor complex per tile
  static constexpr int LNK = NB * 72;              // link complex per tile, one direction
  static constexpr int SLOT = SPIN + LNK;          // neighbour tile + its link plane
  static constexpr int LST = 2;                    // stages of the own link planes (U_0, U_3)
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
  static constexpr size_t smem(int S) {
    return ((size_t)SPIN + (size_t)S * SLOT + (size_t)LST * 2 * LNK) * sizeof(cx<R>) + 8 * (2 * S + 2 * LST + 2);
  }
  static constexpr bool valid = (B % V == 0) && (NC % 32 == 0) && NC >= 64 && NC <= 256 &&
                                smem(2) <= 227 * 1024;
};

// loads pinned in program order: psi(s+1) must be issued where the code says,
// most of a step before its use.  ptxas sinks ordinary and non-coherent loads
// down to their first use (across named barriers and mbarrier waits alike) to
// save registers; it keeps volatile loads in place.
template <typename R, int V> struct PinLd;
template <> struct PinLd<double, 1> {
  static __device__ __forceinline__ void ld(double2 (&o)[1], const double2* p) {
    asm volatile("ld.volatile.global.v2.f64 {%0,%1}, [%2];" : "=d"(o[0].x), "=d"(o[0].y) : "l"(p));
  }
};
template <> struct PinLd<double, 2> {
  static __device__ __forceinline__ void ld(double2 (&o)[2], const double2* p) {
    asm volatile("ld.volatile.global.v2.f64 {%0,%1}, [%2];" : "=d"(o[0].x), "=d"(o[0].y) : "l"(p));
    asm volatile("ld.volatile.global.v2.f64 {%0,%1}, [%2];" : "=d"(o[1].x), "=d"(o[1].y) : "l"(p + 1));
  }
};
template <> struct PinLd<float, 1> {
  static __device__ __forceinline__ void ld(float2 (&o)[1], const float2* p) {
    asm volatile("ld.volatile.global.v2.f32 {%0,%1}, [%2];" : "=f"(o[0].x), "=f"(o[0].y) : "l"(p));
  }
};
template <> struct PinLd<float, 2> {
  static __device__ __forceinline__ void ld(float2 (&o)[2], const float2* p) {
    asm volatile("ld.volatile.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(o[0].x), "=f"(o[0].y), "=f"(o[1].x), "=f"(o[1].y)
                 : "l"(p));
  }
};

template <typename R, int V> struct StS;  // V-wide shared-memory store
template <> struct StS<double, 1> {
  static __device__ __forceinline__ void st(double2* p, const double2 (&v)[1]) { *p = v[0]; }
};
template <> struct StS<double, 2> {
  static __device__ __forceinline__ void st(double2* p, const double2 (&v)[2]) {
    p[0] = v[0];
    p[1] = v[1];
  }
};
template <> struct StS<float, 1> {
  static __device__ __forceinline__ void st(float2* p, const float2 (&v)[1]) { *p = v[0]; }
};
template <> struct StS<float, 2> {
  static __device__ __forceinline__ void st(float2* p, const float2 (&v)[2]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
  }
};

template <int N> __device__ __forceinline__ void reg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N> __device__ __forceinline__ void reg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
#ifndef B200WD_MARCH_SKEW_NS
#define B200WD_MARCH_SKEW_NS 0
#endif

// ZG: segments are not whole z lines; the z hops at the segment edges read
// global memory through generic pointers.
template <typename R, int V, int B, int NB, bool ZG>
__global__ void __launch_bounds__(MarchShape<R, V, B, NB>::NT, MarchShape<R, V, B, NB>::MINB)
    hop_march_kernel(const HopParams p, const TsGrid g, int S) {
  using C = cx<R>;
  using Sh = MarchShape<R, V, B, NB>;
  constexpr int KST = 8 * B;
  constexpr int SEG = Sh::SEG;
  if (hop_stopped(p)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* own = reinterpret_cast<C*>(smem_raw);           // psi(s) of the segment (z hops)
  C* ring = own + Sh::SPIN;                          // S neighbour slots
  C* lks = ring + S * Sh::SLOT;                      // LST x (U_0 plane, U_3 plane) of the own blocks
  uint64_t* full = reinterpret_cast<uint64_t*>(lks + Sh::LST * 2 * Sh::LNK);
  uint64_t* empty = full + S;
  uint64_t* lfull = empty + S;
  uint64_t* lempty = lfull + Sh::LST;
  uint64_t* own_full = lempty + Sh::LST;  // every warp stored its part of psi(s)
  uint64_t* own_free = own_full + 1;      // every warp is done with the z hops of the step

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Sh::NCW);
    }
    for (int i = 0; i < Sh::LST; ++i) {
      mbar_init(&lfull[i], 1);
      mbar_init(&lempty[i], Sh::NCW);
    }
    mbar_init(own_full, Sh::NCW);
    mbar_init(own_free, Sh::NCW);
    fence_barrier_init();
  }
  __syncthreads();

  const int64_t nblk = p.n >> 3;
  const int64_t slice_blks = p.per_t >> 3;
  constexpr int SB = 96 * B;

  if (tid >= Sh::NC) {
    // ---------------- producer warpgroup: one lane issues every copy ----------------
    if constexpr (Sh::REALLOC) reg_dec<Sh::REG_P>();
    if (tid != Sh::NC) return;
    const C* src = static_cast<const C*>(p.src);
    const C* U = static_cast<const C*>(p.U);
    int pslot = 0, pfirst = 1, ls = 0, lfirst = 1;
    uint32_t pphase = 0, lphase = 0;
    auto tile = [&](int64_t bn, int64_t bl, int mu) {
      if (!pfirst) mbar_wait(&empty[pslot], pphase ^ 1u);
      C* slot = ring + pslot * Sh::SLOT;
      mbar_expect_tx(&full[pslot], (uint32_t)(Sh::SLOT * sizeof(C)));
      bulk_g2s(slot, src + bn * SB, (uint32_t)(Sh::SPIN * sizeof(C)), &full[pslot]);
      bulk_g2s(slot + Sh::SPIN, U + (mu * nblk + bl) * 72, (uint32_t)(Sh::LNK * sizeof(C)), &full[pslot]);
      if (++pslot == S) {
        pslot = 0;
        pphase ^= 1u;
        pfirst = 0;
      }
    };
    for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
      const TsUnit w = ts_decode(u, g);
      for (int s = w.t0; s < w.t1; ++s) {
        const int64_t b0 = ts_blk(s, w.x, w.y, w.zi, p, NB);
        {  // U_0 and U_3 of the own blocks
          if (!lfirst) mbar_wait(&lempty[ls], lphase ^ 1u);
          C* d = lks + ls * 2 * Sh::LNK;
          mbar_expect_tx(&lfull[ls], (uint32_t)(2 * Sh::LNK * sizeof(C)));
          bulk_g2s(d, U + (0 * nblk + b0) * 72, (uint32_t)(Sh::LNK * sizeof(C)), &lfull[ls]);
          bulk_g2s(d + Sh::LNK, U + (3 * nblk + b0) * 72, (uint32_t)(Sh::LNK * sizeof(C)), &lfull[ls]);
          if (++ls == Sh::LST) {
            ls = 0;
            lphase ^= 1u;
            lfirst = 0;
          }
        }
        const int64_t bxp = ts_blk(s, wrapi(w.x + 1, p.X), w.y, w.zi, p, NB);
        const int64_t bxm = ts_blk(s, wrapi(w.x - 1, p.X), w.y, w.zi, p, NB);
        const int64_t byp = ts_blk(s, w.x, wrapi(w.y + 1, p.Y), w.zi, p, NB);
        const int64_t bym = ts_blk(s, w.x, wrapi(w.y - 1, p.Y), w.zi, p, NB);
        tile(bxp, b0, 1);
        tile(bxm, bxm, 1);
        tile(byp, b0, 2);
        tile(bym, bym, 2);
        if (s == w.t1 - 1 && u + gridDim.x < g.n_units) {
          // warm L2 with the two own tiles the next unit's prologue loads
          const TsUnit wn = ts_decode(u + gridDim.x, g);
          bulk_prefetch_l2(src + ts_blk(wrapi(wn.t0 - 1, p.T), wn.x, wn.y, wn.zi, p, NB) * SB,
                           (uint32_t)(Sh::SPIN * sizeof(C)));
          bulk_prefetch_l2(src + ts_blk(wn.t0, wn.x, wn.y, wn.zi, p, NB) * SB, (uint32_t)(Sh::SPIN * sizeof(C)));
          bulk_prefetch_l2(U + ts_blk(wrapi(wn.t0 - 1, p.T), wn.x, wn.y, wn.zi, p, NB) * 72,
                           (uint32_t)(Sh::LNK * sizeof(C)));
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  if constexpr (Sh::REALLOC) reg_inc<Sh::REG_C>();
  const int r0 = (tid % Sh::BT) * V;
  const int ys = tid / Sh::BT;         // site in the segment
  const int j = ys >> 3, lo = ys & 7;  // block, site in block
  const int so = (j * 96 + lo) * B + r0;   // own spinor (k = 0) in a tile
  const int lofs = j * 72 + lo;            // own link (e = 0) in a plane
  const bool lead = (tid & 31) == 0;
  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  R scb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) scb[v] = (p.scale ? R(__ldg(p.scale + r0 + v)) : R(1)) * R(p.beta);
  const R ab = (p.xself != nullptr) ? R(p.alpha / p.beta) : R(0);
  const bool self_is_src = p.xself == p.src;

  int cslot = 0, ls = 0;
  uint32_t cphase = 0, lphase = 0, ophase = 0;
  if (lead) mbar_arrive(own_free);  // phase 0: the own tile starts out free
  // The consumer warps are never synchronised as a group (the own tile is
  // handed over through mbarriers waited on long after their completion), so
  // a one-time skew of every other warp persists: while one warp of an SM
  // sub-partition loads from shared memory the other one computes.
  if (B200WD_MARCH_SKEW_NS > 0 && ((tid >> 5) & 1)) __nanosleep(B200WD_MARCH_SKEW_NS);

  for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
    const TsUnit w = ts_decode(u, g);
    const int z = w.zi * SEG + ys;
    const int64_t col_blk = ((int64_t)w.x * p.Y + w.y) * (int64_t)(p.Z >> 3) + (int64_t)w.zi * NB + j;
    // element (k = 0) of this thread's site in slice t
    auto elem = [&](int t) { return ((int64_t)t * slice_blks + col_blk) * SB + lo * B + r0; };
    C nxt[V][12];       // psi(s) at the top of step s, psi(s+1) from its middle on
    C carry[V][2][3];   // U_0(s-1)^H P+ psi(s-1), without the 1/2
    {  // prologue: psi(t0-1) seeds the carry, psi(t0) is the first own spinor
      const int tm = wrapi(w.t0 - 1, p.T);
      C a[V][12];
      const C* pa = src + elem(tm);
      const C* pn = src + elem(w.t0);
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        C t0[V], t1[V];
        PinLd<R, V>::ld(t0, pa + k * KST);
        PinLd<R, V>::ld(t1, pn + k * KST);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          a[v][k] = t0[v];
          nxt[v][k] = t1[v];
        }
      }
      const C* up = U + (0 * nblk + (int64_t)tm * slice_blks + col_blk) * 72 + lo;
      C um[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) um[e] = __ldg(up + e * 8);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        C h[2][3];
        project_spin<0, false, 0>(h[0], a[v]);
        project_spin<0, false, 1>(h[1], a[v]);
        matvec2<true>(carry[v], um, h);
      }
    }
    for (int s = w.t0; s < w.t1; ++s) {
      C acc[V][12];
      mbar_wait(own_free, ophase);  // every warp is done with the z hops of the previous step (long ago)
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        C tmp[V];
#pragma unroll
        for (int v = 0; v < V; ++v) tmp[v] = nxt[v][k];
        StS<R, V>::st(own + so + k * KST, tmp);
      }
      __syncwarp();
      if (lead) mbar_arrive(own_full);
      // self term
      if (self_is_src) {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(ab * nxt[v][k].x, ab * nxt[v][k].y);
      } else if (p.xself) {
        const C* xp = static_cast<const C*>(p.xself) + elem(s);
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C xv[V];
          VecIO<R, V>::ld(xv, xp + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][k] = mk(ab * xv[v].x, ab * xv[v].y);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
      }
      // backward t hop of site s from the carry
#pragma unroll
      for (int v = 0; v < V; ++v) {
        accumulate_spin<0, false, 0>(acc[v], carry[v]);
        accumulate_spin<0, false, 1>(acc[v], carry[v]);
      }
      // own link planes of this step
      mbar_wait(&lfull[ls], lphase);
      const C* lk = lks + ls * 2 * Sh::LNK;
      {  // next carry: U_0(s)^H P+ psi(s)
        C um[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) um[e] = lk[lofs + e * 8];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          C h[2][3];
          project_spin<0, false, 0>(h[0], nxt[v]);
          project_spin<0, false, 1>(h[1], nxt[v]);
          matvec2<true>(carry[v], um, h);
        }
      }
      {  // psi(s+1) into the registers psi(s) just left
        const C* pn = src + elem(wrapi(s + 1, p.T));
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C t1[V];
          PinLd<R, V>::ld(t1, pn + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) nxt[v][k] = t1[v];
        }
      }
#define B200WD_MARCH_TILE(MU, FWD)                                              \
  {                                                                             \
    mbar_wait(&full[cslot], cphase);                                            \
    const C* sb = ring + cslot * Sh::SLOT;                                      \
    HopRegs<R, V> hr;                                                           \
    hop_load<MU, FWD, R, V, KST>(hr, sb + so, sb + Sh::SPIN + lofs);            \
    __syncwarp();                                                               \
    if (lead) mbar_arrive(&empty[cslot]);                                       \
    if (++cslot == S) {                                                         \
      cslot = 0;                                                                \
      cphase ^= 1u;                                                             \
    }                                                                           \
    hop_compute<MU, FWD, R, V>(acc, hr);                                        \
  }
      B200WD_MARCH_TILE(1, true)
      B200WD_MARCH_TILE(1, false)
      B200WD_MARCH_TILE(2, true)
      mbar_wait(own_full, ophase);  // the own tile is complete (every warp stored its part at the top of the step)
      {  // z hops from the own tile, U_3 in the second plane
        const C* ua = lk + Sh::LNK;
        const int zp = ys + 1, zm = ys - 1;
        if constexpr (!ZG) {
          const int zpp = zp == SEG ? 0 : zp, zmm = zm < 0 ? SEG - 1 : zm;
          hop_full<3, true, R, V, true, true>(acc, own + ((zpp >> 3) * 96 + (zpp & 7)) * B + r0, KST, ua + lofs, 8);
          hop_full<3, false, R, V, true, true>(acc, own + ((zmm >> 3) * 96 + (zmm & 7)) * B + r0, KST,
                                               ua + (zmm >> 3) * 72 + (zmm & 7), 8);
        } else {
          const int64_t line0 = (int64_t)s * p.per_t + ((int64_t)w.x * p.Y + w.y) * p.Z;  // first site of the z line
          {
            const C* sp = zp < SEG ? own + ((zp >> 3) * 96 + (zp & 7)) * B + r0
                                   : src + spinor_base(line0 + wrapi(z + 1, p.Z), 12, B) + r0;
            hop_full<3, true, R, V, true, true>(acc, sp, KST, ua + lofs, 8);
          }
          {
            const C *sp, *up;
            if (zm >= 0) {
              sp = own + ((zm >> 3) * 96 + (zm & 7)) * B + r0;
              up = ua + (zm >> 3) * 72 + (zm & 7);
            } else {
              const int64_t xs = line0 + wrapi(z - 1, p.Z);
              sp = src + spinor_base(xs, 12, B) + r0;
              up = U + link_base(xs, 3, nblk);
            }
            hop_full<3, false, R, V, true, true>(acc, sp, KST, up, 8);
          }
        }
      }
      __syncwarp();
      if (lead) mbar_arrive(own_free);
      ophase ^= 1u;
      {  // forward t hop of site s: U_0(s) P- psi(s+1), psi(s+1) from registers
        C um[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) um[e] = lk[lofs + e * 8];
        __syncwarp();
        if (lead) mbar_arrive(&lempty[ls]);
        if (++ls == Sh::LST) {
          ls = 0;
          lphase ^= 1u;
        }
#pragma unroll
        for (int v = 0; v < V; ++v) {
          C h[2][3], gg[2][3];
          project_spin<0, true, 0>(h[0], nxt[v]);
          project_spin<0, true, 1>(h[1], nxt[v]);
          matvec2<false>(gg, um, h);
          accumulate_spin<0, true, 0>(acc[v], gg);
          accumulate_spin<0, true, 1>(acc[v], gg);
        }
      }
      B200WD_MARCH_TILE(2, false)
#undef B200WD_MARCH_TILE
      C* out = static_cast<C*>(p.out) + elem(s);
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        C res[V];
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = mk(scb[v] * acc[v][k].x, scb[v] * acc[v][k].y);
        VecIO<R, V>::st(out + k * KST, res);
      }
    }
  }
}

// ---- host side ----------------------------------------------------------------

struct MarchCfg {
  int nb = 0, s = 0, nch = 0;
};
static MarchCfg march_env() {
  static MarchCfg c{-1, -1, -1};
  if (c.nb < 0) {
    c = MarchCfg{};
    const char* e = getenv("B200WD_MARCH_CFG");
    if (e) sscanf(e, "%d,%d,%d", &c.nb, &c.s, &c.nch);
  }
  return c;
}
// B200WD_MARCH: 0 never, 1 wherever the shape allows (tuning, tests); unset: the table
static int march_mode() {
  static int m = -2;
  if (m == -2) {
    const char* e = getenv("B200WD_MARCH");
    m = e ? atoi(e) : -1;
  }
  return m;
}

template <typename R, int V, int B, int NB, bool ZG>
static bool launch_march_kernel(const HopParams& p, const TsGrid& g0, int S, int nch, cudaStream_t st) {
  using Sh = MarchShape<R, V, B, NB>;
  const size_t smem = Sh::smem(S);
  LaunchFacts f;
  if (!launch_facts((const void*)hop_march_kernel<R, V, B, NB, ZG>, Sh::NT, smem, f)) return false;
  TsGrid g = g0;
  const int64_t grid_max = (int64_t)f.occ * persistent_sms(f.sm_count);
  g.nch = nch > 0 ? (nch > g.nT ? g.nT : nch) : ts_choose_nch(g.ncol, g.nT, grid_max, 5);
  g.n_units = g.ncol * g.nch;
  const int64_t grid = grid_max < g.n_units ? grid_max : g.n_units;
  hop_march_kernel<R, V, B, NB, ZG><<<(unsigned)grid, Sh::NT, smem, st>>>(p, g, S);
  return true;
}

template <typename R, int V, int B, int NB>
static bool launch_march_nb(const HopParams& p, int S, int nch, cudaStream_t st) {
  using Sh = MarchShape<R, V, B, NB>;
  if constexpr (!Sh::valid) {
    return false;
  } else {
    if (p.Z % Sh::SEG) return false;
    TsGrid g{};
    g.lz = p.Z / Sh::SEG;
    g.ny = p.Y;
    g.ncol = (int64_t)p.X * g.ny * g.lz;
    g.ta = (int32_t)(p.d_begin / p.per_t);
    g.nT = (int32_t)((p.d_end - p.d_begin) / p.per_t);
    const size_t budget = (Sh::MINB == 2 ? 113 : 227) * 1024;
    if (S <= 0) S = 8;
    if (S > 8) S = 8;
    while (S > 2 && Sh::smem(S) > budget) --S;
    if (Sh::smem(S) > 227 * 1024) return false;
    if (g.lz == 1) return launch_march_kernel<R, V, B, NB, false>(p, g, S, nch, st);
    return launch_march_kernel<R, V, B, NB, true>(p, g, S, nch, st);
  }
}

// Where the march is the default: (NB, S) per (dtype, b); nb = 0: not used.
template <typename R, int V, int B>
static MarchCfg march_table(int Z) {
  (void)Z;
  return MarchCfg{};
}

// Full-lattice fields, no halos, no clover, slice-aligned destination range.
template <typename R, int V, int B>
static bool try_launch_march(const HopParams& p, cudaStream_t st) {
  const int mode = march_mode();
  if (mode == 0) return false;
  if (p.dst_parity >= 0 || p.lam_halo != nullptr || p.beta == 0.0 || p.clov_mode != 0 || p.jump_by) return false;
  if (p.Z % 8 != 0) return false;
  if (p.d_begin % p.per_t || p.d_end % p.per_t || p.d_end <= p.d_begin) return false;
  MarchCfg c = march_table<R, V, B>(p.Z);
  const MarchCfg e = march_env();
  if (mode != 1 && e.nb <= 0 && c.nb <= 0) return false;
  if (e.nb > 0) c.nb = e.nb;
  if (e.s > 0) c.s = e.s;
  if (e.nch > 0) c.nch = e.nch;
  if (c.nb <= 0) {  // the largest segment dividing the z line that fits 256 consumer threads
    for (int nb : {4, 2, 1})
      if (c.nb <= 0 && p.Z % (8 * nb) == 0 && (B / V) * 8 * nb <= 256) c.nb = nb;
  }
#define B200WD_MARCH_TRY(NB_) \
  if (c.nb == NB_ && launch_march_nb<R, V, B, NB_>(p, c.s, c.nch, st)) return true;
  B200WD_MARCH_TRY(1)
  B200WD_MARCH_TRY(2)
  B200WD_MARCH_TRY(4)
#undef B200WD_MARCH_TRY
  return false;
}

}  // namespace b200wd
