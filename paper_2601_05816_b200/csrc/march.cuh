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
//     128-bit load per component, coalesced across the warp; three batches of
//     four during the first tile hops of step s, pinned with ld.volatile) and
//     lands while the other hops are computed; it feeds the
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
// An item is LY y-adjacent segments (LY = 1, 2 or 4), sized so that a CTA has
// 192 or 256 consumer threads; one CTA per SM.  Three hazards found with the race
// detector (tools/stress_march.py) shape the synchronisation:
//   * mbarrier.arrive is NOT ordered behind the warp's outstanding shared-memory
//     loads, not even after a MEMBAR: a buffer handed back right after issuing the
//     loads was refilled (the small link copy of the next tile lands within a few
//     hundred ns) before the last loads had read it.  Every hand-over is made
//     data-dependent on the loaded values (arrive_after / hop_compute_release).
//   * setmaxnreg: the idle warps of the producer warpgroup must not exit before
//     every consumer warp finished setmaxnreg.inc (regs_ok), or consumer registers
//     are corrupted; and the copy-issuing thread needs >= 56 registers or it starves
//     the ring.
//   * two resident CTAs per SM together with setmaxnreg corrupted results: 1 CTA/SM.
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

#ifndef B200WD_MARCH_REG_C
// registers per consumer / producer thread after setmaxnreg (2 C + P <= 504 = 3 x 168).
// The producer needs room: measured on 16^3x32 c128 nrhs 16 (same box, safe exit
// order): P = 24 0.344, P = 40 0.506-0.509 whatever C (200 ... 232), P = 56 0.574-0.580,
// P = 72 0.563, P = 88 0.589 (C = 208), P = 104 0.586 (C = 200) -- with 40 registers the
// copy-issuing thread is slow enough to starve the ring.
#define B200WD_MARCH_REG_C 224
#define B200WD_MARCH_REG_P 56
#endif
#ifndef B200WD_MARCH_EXP
#define B200WD_MARCH_EXP 0  // experiments: 1 link copy before the spinor copy, 4 producer waits 1 us before each refill
#endif
#ifndef B200WD_MARCH_LD0
#define B200WD_MARCH_LD0 4  // psi(s+1) loads before the x+ tile / before the x- tile (the rest before y+)
#define B200WD_MARCH_LD1 4
#endif
#ifndef B200WD_MARCH_RACY
#define B200WD_MARCH_RACY 0  // experiments: 1 idle producer warps exit at once (corrupts registers), > 1 also delays setmaxnreg.inc by that many ns
#endif

template <typename R, int V, int B, int NB, int LY> struct MarchShape {
  static constexpr int BT = B / V;                 // threads per site
  static constexpr int SEG = 8 * NB;               // sites per line segment
  static constexpr int NC = BT * SEG * LY;         // consumer threads
  static constexpr int NCW = NC / 32;
  static constexpr bool REALLOC = NC == 256;       // 8 consumer warps + producer: setmaxnreg (9 warps cap at 168)
  static constexpr int NP = REALLOC ? 128 : 32;    // producer threads (one issues)
  static constexpr int NT = NC + NP;
  // registers after reallocation (per SM sub-partition: 16384 >= 32 * sum over its warps)
  static constexpr int REG_C = B200WD_MARCH_REG_C;
  static constexpr int REG_P = B200WD_MARCH_REG_P;
  static constexpr int LSP = NB * 96 * B;          // spinor complex per line segment
  static constexpr int LLK = NB * 72;              // link complex per line segment, one direction
  static constexpr int SPIN = LY * LSP;            // spinor complex per tile
  static constexpr int LNK = LY * LLK;             // link complex per tile, one direction
  static constexpr int SLOT = SPIN + LNK;          // neighbour tile + its link plane
  static constexpr int LST = 2;                    // stages of the own link planes (U_0, U_3)
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
  static constexpr size_t smem(int S) {
    return ((size_t)SPIN + (size_t)S * SLOT + (size_t)LST * 2 * LNK) * sizeof(cx<R>) + 8 * (2 * S + 2 * LST + 3);
  }
  static constexpr bool valid = (B % V == 0) && (NC % 32 == 0) && NC >= 128 && NC <= 256 &&
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


// Work decomposition.  Columns [0, n1) are marched over the whole slice range
// by one unit each (n1 is a multiple of the grid: whole rounds in which every
// CTA carries one column through the same slices); the remaining ncol - n1
// columns are cut into nch2 t chunks each so that they balance over the grid.
// Units are ordered (chunk, column): the CTAs running at one time march
// neighbouring columns through the same slices.
struct MarchGrid {
  int32_t px, py;   // column patch (x, y items) of the traversal; 0: natural order
  int32_t lz, ny;   // segments per z line, lines in y
  int64_t ncol;     // X * ny * lz
  int32_t ta, nT;   // destination slices [ta, ta + nT)
  int64_t n1;       // columns marched whole
  int32_t nch2;     // t chunks of the other columns
  int64_t n_units;  // n1 + (ncol - n1) * nch2
};
__device__ __forceinline__ TsUnit march_decode(int64_t u, const MarchGrid& g) {
  TsUnit w;
  uint32_t c;
  if (u < g.n1) {
    c = (uint32_t)u;
    w.t0 = g.ta;
    w.t1 = g.ta + g.nT;
  } else {
    const int64_t v = u - g.n1, r = g.ncol - g.n1;
    const int64_t chunk = v / r;
    c = (uint32_t)(g.n1 + (v - chunk * r));
    w.t0 = g.ta + (int)((chunk * g.nT) / g.nch2);
    w.t1 = g.ta + (int)(((chunk + 1) * g.nT) / g.nch2);
  }
  w.zi = (int)(c % (uint32_t)g.lz);
  c /= (uint32_t)g.lz;
  if (g.px == 0) {
    w.y = (int)(c % (uint32_t)g.ny);
    w.x = (int)(c / (uint32_t)g.ny);
  } else {
    // patched order: all columns of one px x py patch before the next patch, so the
    // CTAs of a round cover a compact x-y region and find their x and y neighbours in L2
    const uint32_t pa = (uint32_t)(g.px * g.py);
    const uint32_t within = c % pa, patch = c / pa;
    const uint32_t npy = (uint32_t)(g.ny / g.py);
    w.x = (int)((patch / npy) * g.px + within / g.py);
    w.y = (int)((patch % npy) * g.py + within % g.py);
  }
  return w;
}

// ZG: segments are not whole z lines; the z hops at the segment edges read
// global memory through generic pointers.
template <typename R, int V, int B, int NB, int LY, bool ZG>
__global__ void __launch_bounds__(MarchShape<R, V, B, NB, LY>::NT, 1)
    hop_march_kernel(const HopParams p, const MarchGrid g, int S) {
  using C = cx<R>;
  using Sh = MarchShape<R, V, B, NB, LY>;
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
  uint64_t* regs_ok = own_free + 1;       // every consumer warp completed setmaxnreg.inc

  const int tid = threadIdx.x;
  if (threadIdx.x == 0) {
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
    mbar_init(regs_ok, Sh::NCW);
    fence_barrier_init();
  }
  __syncthreads();

  const int64_t nblk = p.n >> 3;
  const int64_t slice_blks = p.per_t >> 3;
  constexpr int SB = 96 * B;

  if (tid >= Sh::NC) {
    // ---------------- producer warpgroup: one lane issues every copy ----------------
    if constexpr (Sh::REALLOC) reg_dec<Sh::REG_P>();
    // The idle warps of the producer warpgroup leave only after every consumer warp
    // holds its reallocated registers (regs_ok): when they exited right after
    // setmaxnreg.dec, racing the consumers' setmaxnreg.inc, consumer registers were
    // corrupted at random (a few wrong half spinors per launch on B200; tools/
    // stress_march.py), and keeping them resident for the whole kernel cost 18%.
    if (tid >= Sh::NC + 32) {
      if constexpr (Sh::REALLOC && !B200WD_MARCH_RACY) mbar_wait(regs_ok, 0);
      return;
    }
    if (tid != Sh::NC) return;  // idle lanes of the issuing warp: lanes leaving frees nothing
    {
    const C* src = static_cast<const C*>(p.src);
    const C* U = static_cast<const C*>(p.U);
    int pslot = 0, pfirst = 1, ls = 0, lfirst = 1;
    uint32_t pphase = 0, lphase = 0;
    const bool whole = g.lz == 1;
    // LY lines y0 .. y0+LY-1 (mod Y) of segment zi at (t, x): NB blocks of `per` complex
    // each per line, from `base`; one copy when the lines are contiguous in memory
    auto lines = [&](C* dst, const C* base, int per, int t, int x, int y0, int zi, uint64_t* bar) {
      if (LY == 1 || (whole && y0 >= 0 && y0 + LY <= p.Y)) {
        bulk_g2s(dst, base + ts_blk(t, x, wrapi(y0, p.Y), zi, p, NB) * per, (uint32_t)(LY * NB * per * sizeof(C)), bar);
      } else {
#pragma unroll
        for (int l = 0; l < LY; ++l)
          bulk_g2s(dst + l * NB * per, base + ts_blk(t, x, wrapi(y0 + l, p.Y), zi, p, NB) * per,
                   (uint32_t)(NB * per * sizeof(C)), bar);
      }
    };
    // neighbour tile: spinor lines (xs, ys..) and one link direction of lines (xl, yl..)
    auto tile = [&](int s, int xs, int ys, int xl, int yl, int zi, int mu) {
      if (!pfirst) mbar_wait(&empty[pslot], pphase ^ 1u);
      if (B200WD_MARCH_EXP & 4) __nanosleep(1000);
      C* slot = ring + pslot * Sh::SLOT;
      mbar_expect_tx(&full[pslot], (uint32_t)(Sh::SLOT * sizeof(C)));
      if (B200WD_MARCH_EXP & 1) {
        lines(slot + Sh::SPIN, U + mu * nblk * 72, 72, s, xl, yl, zi, &full[pslot]);
        lines(slot, src, SB, s, xs, ys, zi, &full[pslot]);
      } else {
        lines(slot, src, SB, s, xs, ys, zi, &full[pslot]);
        lines(slot + Sh::SPIN, U + mu * nblk * 72, 72, s, xl, yl, zi, &full[pslot]);
      }
      if (++pslot == S) {
        pslot = 0;
        pphase ^= 1u;
        pfirst = 0;
      }
    };
    for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
      const TsUnit w = march_decode(u, g);
      const int y0 = w.y * LY;  // first line of the item
      for (int s = w.t0; s < w.t1; ++s) {
        {  // U_0 and U_3 of the own blocks
          if (!lfirst) mbar_wait(&lempty[ls], lphase ^ 1u);
          C* d = lks + ls * 2 * Sh::LNK;
          mbar_expect_tx(&lfull[ls], (uint32_t)(2 * Sh::LNK * sizeof(C)));
          lines(d, U + 0 * nblk * 72, 72, s, w.x, y0, w.zi, &lfull[ls]);
          lines(d + Sh::LNK, U + 3 * nblk * 72, 72, s, w.x, y0, w.zi, &lfull[ls]);
          if (++ls == Sh::LST) {
            ls = 0;
            lphase ^= 1u;
            lfirst = 0;
          }
        }
        const int xp = wrapi(w.x + 1, p.X), xm = wrapi(w.x - 1, p.X);
        tile(s, xp, y0, w.x, y0, w.zi, 1);          // x+: U_1 of the own lines
        tile(s, xm, y0, xm, y0, w.zi, 1);           // x-: U_1 of the neighbour lines
        tile(s, w.x, y0 + 1, w.x, y0, w.zi, 2);     // y+: lines y0+1 .., U_2 of the own lines
        tile(s, w.x, y0 - 1, w.x, y0 - 1, w.zi, 2); // y-: lines y0-1 .., their U_2
        if (s == w.t1 - 1 && u + gridDim.x < g.n_units) {
          // warm L2 with what the next unit's prologue loads: two own tiles and U_0(t0-1)
          const TsUnit wn = march_decode(u + gridDim.x, g);
          const int tm = wrapi(wn.t0 - 1, p.T);
#pragma unroll
          for (int l = 0; l < LY; ++l) {
            bulk_prefetch_l2(src + ts_blk(tm, wn.x, wn.y * LY + l, wn.zi, p, NB) * SB, (uint32_t)(Sh::LSP * sizeof(C)));
            bulk_prefetch_l2(src + ts_blk(wn.t0, wn.x, wn.y * LY + l, wn.zi, p, NB) * SB,
                             (uint32_t)(Sh::LSP * sizeof(C)));
            bulk_prefetch_l2(U + ts_blk(tm, wn.x, wn.y * LY + l, wn.zi, p, NB) * 72, (uint32_t)(Sh::LLK * sizeof(C)));
          }
        }
      }
    }
    }
    return;
  }

  // ---------------- consumers ----------------
  if constexpr (Sh::REALLOC) {
    if (B200WD_MARCH_RACY > 1) __nanosleep(B200WD_MARCH_RACY);  // experiment: let the idle warps exit first
    reg_inc<Sh::REG_C>();
    if ((tid & 31) == 0) mbar_arrive(regs_ok);
  }
  const int r0 = (tid % Sh::BT) * V;
  const int ys = tid / Sh::BT;                 // site in the item
  const int ln = ys / SEG, zs = ys % SEG;      // line of the item, z offset in its segment
  const int j = ln * NB + (zs >> 3), lo = zs & 7;  // block of the tile, site in block
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

  for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
    const TsUnit w = march_decode(u, g);
    const int z = w.zi * SEG + zs;
    const int yl = w.y * LY + ln;  // this thread's line
    const int64_t col_blk = ((int64_t)w.x * p.Y + yl) * (int64_t)(p.Z >> 3) + (int64_t)w.zi * NB + (zs >> 3);
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
      // own link planes of this step
      mbar_wait(&lfull[ls], lphase);
      const C* lk = lks + ls * 2 * Sh::LNK;
      {
        // z hops, sender side: this site's half spinors for its two z neighbours --
        // P-_3 psi(s) for the forward hop of z-1 (multiplied there by U_3(z-1)) and
        // U_3(z)^H P+_3 psi(s), the finished backward hop of z+1 -- go to the own
        // tile as components 0-5 and 6-11: 12 stores as for psi itself, but the
        // receivers read 6 + 6 instead of 12 + 12 components and one link less
        C um[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) um[e] = lk[Sh::LNK + lofs + e * 8];
        C hf[V][2][3], hb[V][2][3];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          C h[2][3];
          project_spin<3, true, 0>(hf[v][0], nxt[v]);
          project_spin<3, true, 1>(hf[v][1], nxt[v]);
          project_spin<3, false, 0>(h[0], nxt[v]);
          project_spin<3, false, 1>(h[1], nxt[v]);
          matvec2<true>(hb[v], um, h);
        }
        mbar_wait(own_free, ophase);  // every warp is done with the z hops of the previous step (long ago)
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          C t0[V], t1[V];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            t0[v] = hf[v][k / 3][k % 3];
            t1[v] = hb[v][k / 3][k % 3];
          }
          StS<R, V>::st(own + so + k * KST, t0);
          StS<R, V>::st(own + so + (6 + k) * KST, t1);
        }
      }
      // The own tile is the one buffer consumers hand to each other within ~100 ns
      // (the TMA-filled buffers come back after a memory round trip): the fence makes
      // every lane's stores (below: loads) complete before the warp's arrival is seen.
      __threadfence_block();
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
      // psi(s+1) into the registers psi(s) just left, in three batches (before the x+,
      // x- and y+ tiles): twelve 128-bit loads at once throttle the shared-memory loads of
      // the first tile hop behind them (MIO queue); B200WD_MARCH_LD0/1 = batch sizes
      const C* pn = src + elem(wrapi(s + 1, p.T));
      auto load_next = [&](int k0, int k1) {
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          if (k >= k0 && k < k1) {
            C t1[V];
            PinLd<R, V>::ld(t1, pn + k * KST);
#pragma unroll
            for (int v = 0; v < V; ++v) nxt[v][k] = t1[v];
          }
        }
      };
      load_next(0, B200WD_MARCH_LD0);
#define B200WD_MARCH_TILE(MU, FWD)                                              \
  {                                                                             \
    mbar_wait(&full[cslot], cphase);                                            \
    const C* sb = ring + cslot * Sh::SLOT;                                      \
    HopRegs<R, V> hr;                                                           \
    hop_load<MU, FWD, R, V, KST>(hr, sb + so, sb + Sh::SPIN + lofs);            \
    hop_compute_release<MU, FWD, R, V>(acc, hr, &empty[cslot], lead);           \
    if (++cslot == S) {                                                         \
      cslot = 0;                                                                \
      cphase ^= 1u;                                                             \
    }                                                                           \
  }
      B200WD_MARCH_TILE(1, true)
      load_next(B200WD_MARCH_LD0, B200WD_MARCH_LD0 + B200WD_MARCH_LD1);
      B200WD_MARCH_TILE(1, false)
      load_next(B200WD_MARCH_LD0 + B200WD_MARCH_LD1, 12);
      B200WD_MARCH_TILE(2, true)
      mbar_wait(own_full, ophase);  // the own tile is complete (every warp stored its part at the top of the step)
      {  // z hops, receiver side (U_3 in the second link plane)
        const C* ua = lk + Sh::LNK;
        const int zp = zs + 1, zm = zs - 1;
        auto fwd_in = [&](int zz) {  // U_3(z) applied to the neighbour's P- half spinor
          const C* hp = own + ((ln * NB + (zz >> 3)) * 96 + (zz & 7)) * B + r0;
          C um[9];
#pragma unroll
          for (int e = 0; e < 9; ++e) um[e] = ua[lofs + e * 8];
          C hh[V][2][3];
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            C tmp[V];
            VecIO<R, V>::lds(tmp, hp + k * KST);
#pragma unroll
            for (int v = 0; v < V; ++v) hh[v][k / 3][k % 3] = tmp[v];
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            C gg[2][3];
            matvec2<false>(gg, um, hh[v]);
            accumulate_spin<3, true, 0>(acc[v], gg);
            accumulate_spin<3, true, 1>(acc[v], gg);
          }
        };
        auto bwd_in = [&](int zz) {  // the neighbour's finished backward hop
          const C* hp = own + ((ln * NB + (zz >> 3)) * 96 + (zz & 7)) * B + r0 + 6 * KST;
          C gg[V][2][3];
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            C tmp[V];
            VecIO<R, V>::lds(tmp, hp + k * KST);
#pragma unroll
            for (int v = 0; v < V; ++v) gg[v][k / 3][k % 3] = tmp[v];
          }
#pragma unroll
          for (int v = 0; v < V; ++v) {
            accumulate_spin<3, false, 0>(acc[v], gg[v]);
            accumulate_spin<3, false, 1>(acc[v], gg[v]);
          }
        };
        if constexpr (!ZG) {
          fwd_in(zp == SEG ? 0 : zp);
          bwd_in(zm < 0 ? SEG - 1 : zm);
        } else {
          // segment edges: the neighbour belongs to another column, whole hop from global memory
          const int64_t line0 = (int64_t)s * p.per_t + ((int64_t)w.x * p.Y + yl) * p.Z;  // first site of the z line
          if (zp < SEG) {
            fwd_in(zp);
          } else {
            hop_full<3, true, R, V, false, true>(acc, src + spinor_base(line0 + wrapi(z + 1, p.Z), 12, B) + r0, KST,
                                                 ua + lofs, 8);
          }
          if (zm >= 0) {
            bwd_in(zm);
          } else {
            const int64_t xs = line0 + wrapi(z - 1, p.Z);
            hop_full<3, false, R, V, false, false>(acc, src + spinor_base(xs, 12, B) + r0, KST,
                                                   U + link_base(xs, 3, nblk), 8);
          }
        }
      }
      {
        // the z-hop loads of the own tile feed acc: the arrival waits for them through it
        uint32_t chk = 0;
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) chk += touch_word(acc[v][k]);
        __syncwarp();
        if (lead) arrive_after(own_free, chk);
      }
      ophase ^= 1u;
      {  // forward t hop of site s: U_0(s) P- psi(s+1), psi(s+1) from registers
        HopRegs<R, V> hr;
#pragma unroll
        for (int e = 0; e < 9; ++e) hr.u[e] = lk[lofs + e * 8];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          project_spin<0, true, 0>(hr.h[v][0], nxt[v]);
          project_spin<0, true, 1>(hr.h[v][1], nxt[v]);
        }
        hop_compute_release<0, true, R, V>(acc, hr, &lempty[ls], lead);  // hands the link planes back
        if (++ls == Sh::LST) {
          ls = 0;
          lphase ^= 1u;
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
  int nb = 0, ly = 0, s = 0, nch = 0;
};
// B200WD_MARCH_CFG="NB,LY,S,NCH" forces a shape (0: default for that field)
static MarchCfg march_env() {
  static MarchCfg c{-1, -1, -1, -1};
  if (c.nb < 0) {
    c = MarchCfg{};
    const char* e = getenv("B200WD_MARCH_CFG");
    if (e) sscanf(e, "%d,%d,%d,%d", &c.nb, &c.ly, &c.s, &c.nch);
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

template <typename R, int V, int B, int NB, int LY, bool ZG>
static bool launch_march_kernel(const HopParams& p, const MarchGrid& g0, int S, int nch, cudaStream_t st) {
  using Sh = MarchShape<R, V, B, NB, LY>;
  const size_t smem = Sh::smem(S);
  LaunchFacts f;
  if (!launch_facts((const void*)hop_march_kernel<R, V, B, NB, LY, ZG>, Sh::NT, smem, f)) return false;
  MarchGrid g = g0;
  // one CTA per SM whatever the occupancy calculator allows (see the header)
  int64_t grid_max = persistent_sms(f.sm_count);
  static const int grid_cap = ring_knob("B200WD_MARCH_GRID", 0);  // tuning / debugging: cap the persistent grid
  if (grid_cap > 0 && grid_cap < grid_max) grid_max = grid_cap;
  if (nch > 0) {  // forced: every column in nch chunks
    g.n1 = 0;
    g.nch2 = nch > g.nT ? g.nT : nch;
  } else {
    g.n1 = (g.ncol / grid_max) * grid_max;
    g.nch2 = g.ncol > g.n1 ? ts_choose_nch(g.ncol - g.n1, g.nT, grid_max, 5) : 1;
  }
  g.n_units = g.n1 + (g.ncol - g.n1) * g.nch2;
  // Column patches when a round of the grid covers less than two x rows (then the x
  // neighbours of most columns belong to other rounds and miss L2: 48^3x96): the patch
  // px | X, py | ny with px * py * lz <= grid and the smallest perimeter / area.
  // B200WD_MARCH_PATCH="px,py" forces a patch, "0,0" turns patching off.
  g.px = g.py = 0;
  {
    static int fx = -1, fy = -1;
    if (fx < 0) {
      fx = fy = -2;
      const char* e = getenv("B200WD_MARCH_PATCH");
      if (e) sscanf(e, "%d,%d", &fx, &fy);
    }
    if (fx > 0 && fy > 0) {
      if (p.X % fx == 0 && g.ny % fy == 0) {
        g.px = fx;
        g.py = fy;
      }
    } else if (fx != 0 && (int64_t)g.ny * g.lz * 2 > grid_max) {
      double best = 1e30;
      for (int px = 1; px <= p.X; ++px) {
        if (p.X % px) continue;
        for (int py = 1; py <= g.ny; ++py) {
          if (g.ny % py || (int64_t)px * py * g.lz > grid_max) continue;
          const double perim = 1.0 / px + 1.0 / py;
          if (perim < best - 1e-12) {
            best = perim;
            g.px = px;
            g.py = py;
          }
        }
      }
      if (g.px == p.X && g.py == g.ny) g.px = g.py = 0;
    }
  }
  const int64_t grid = grid_max < g.n_units ? grid_max : g.n_units;
  hop_march_kernel<R, V, B, NB, LY, ZG><<<(unsigned)grid, Sh::NT, smem, st>>>(p, g, S);
  return true;
}

template <typename R, int V, int B, int NB, int LY>
static bool launch_march_shape(const HopParams& p, int S, int nch, cudaStream_t st) {
  using Sh = MarchShape<R, V, B, NB, LY>;
  if constexpr (!Sh::valid) {
    return false;
  } else {
    if (p.Z % Sh::SEG || p.Y % LY) return false;
    MarchGrid g{};
    g.lz = p.Z / Sh::SEG;
    g.ny = p.Y / LY;
    g.ncol = (int64_t)p.X * g.ny * g.lz;
    g.ta = (int32_t)(p.d_begin / p.per_t);
    g.nT = (int32_t)((p.d_end - p.d_begin) / p.per_t);
    // more than half the shared memory: a second CTA can never become resident
    const size_t floor_bytes = 116 * 1024;
    if (S <= 0) S = 8;
    if (S > 8) S = 8;
    while (S > 2 && Sh::smem(S) > 227 * 1024) --S;
    if (Sh::smem(S) > 227 * 1024) return false;
    size_t smem = Sh::smem(S);
    (void)smem;
    if (Sh::smem(S) < floor_bytes) return false;  // small tiles: the ring kernels serve those shapes
    if (g.lz == 1) return launch_march_kernel<R, V, B, NB, LY, false>(p, g, S, nch, st);
    return launch_march_kernel<R, V, B, NB, LY, true>(p, g, S, nch, st);
  }
}

// Default shape: whole z lines when a line fits 256 consumer threads, else the
// largest segment that does; then as many y lines as keep the item at or below
// 256 threads.
template <typename R, int V, int B>
static MarchCfg march_default_shape(const HopParams& p) {
  MarchCfg c{};
  constexpr int BT = B / V;
  for (int nb : {4, 2, 1})
    if (c.nb == 0 && p.Z % (8 * nb) == 0 && BT * 8 * nb <= 256) c.nb = nb;
  if (c.nb == 0) return c;
  for (int ly : {4, 2, 1})
    if (c.ly == 0 && p.Y % ly == 0 && BT * 8 * c.nb * ly <= 256) c.ly = ly;
  return c;
}

// Where the march is the default: shapes that measured faster than the ring
// kernels on B200 (profiles/r2_march_tuning.txt; fraction of the HBM roofline, march
// vs ring, same box and session) and come through the race detector clean
// (tools/stress_march.py).  16^3x32: c128 nrhs 6 0.575 vs 0.507, 8 0.502 vs 0.492,
// 12 0.590 vs 0.468, 16 0.601 vs 0.490, 24 0.447 vs 0.438 (32: 0.466 vs 0.489, 4: 0.466
// vs 0.530: ring); c64 nrhs 12 0.414 vs 0.403, 24 0.506 vs 0.448, 32 0.576 vs 0.479
// (6, 8, 16: ring / two-line ring / stream are faster).  Partial z lines, nrhs 12:
// c64 48^3x96 0.365 vs 0.291, 24^3x48 0.330 vs 0.306 (c128 there 0.341 vs 0.346 and
// 0.394 vs 0.435: ring).  Unmeasured shapes stay on the ring.  B200WD_MARCH=1 forces
// the march wherever a shape exists, B200WD_MARCH=0 turns it off.
template <typename R, int V, int B>
static bool march_table(const HopParams& p) {
  if constexpr (sizeof(R) == 8) {
    return p.Z == 16 && (B == 6 || B == 8 || B == 12 || B == 16 || B == 24);
  } else {
    if (p.Z == 16) return B == 12 || B == 24 || B == 32;
    return B == 12 && (p.Z == 24 || p.Z == 48);
  }
}

// Full-lattice fields, no halos, no clover, slice-aligned destination range.
template <typename R, int V, int B>
static bool try_launch_march(const HopParams& p, cudaStream_t st) {
  const int mode = march_mode();
  if (mode == 0) return false;
  if (p.dst_parity >= 0 || p.lam_halo != nullptr || p.beta == 0.0 || p.clov_mode != 0 || p.jump_by) return false;
  if (p.Z % 8 != 0) return false;
  if (p.d_begin % p.per_t || p.d_end % p.per_t || p.d_end <= p.d_begin) return false;
  const MarchCfg e = march_env();
  if (mode != 1 && e.nb <= 0 && !march_table<R, V, B>(p)) return false;
  // short slice ranges (the T chunks of the host-pipelined apply, thin T-split interiors):
  // a unit re-reads two own tiles whatever its length, so the ring serves ranges under 8 slices
  if (mode != 1 && e.nb <= 0 && (p.d_end - p.d_begin) / p.per_t < 8) return false;
  MarchCfg c = march_default_shape<R, V, B>(p);
  if (e.nb > 0) {
    c.nb = e.nb;
    c.ly = e.ly > 0 ? e.ly : 1;
  }
  if (e.s > 0) c.s = e.s;
  if (e.nch > 0) c.nch = e.nch;
#define B200WD_MARCH_TRY(NB_, LY_) \
  if (c.nb == NB_ && c.ly == LY_ && launch_march_shape<R, V, B, NB_, LY_>(p, c.s, c.nch, st)) return true;
  B200WD_MARCH_TRY(1, 1)
  B200WD_MARCH_TRY(2, 1)
  B200WD_MARCH_TRY(4, 1)
  B200WD_MARCH_TRY(1, 2)
  B200WD_MARCH_TRY(2, 2)
  B200WD_MARCH_TRY(4, 2)
  B200WD_MARCH_TRY(1, 4)
  B200WD_MARCH_TRY(2, 4)
#undef B200WD_MARCH_TRY
  return false;
}

}  // namespace b200wd
