// T-streaming Wilson hopping kernel (full-lattice fields), sm_100a.
//
// Why: the TMA ring kernel (dirac_kernels.cuh) moves 7 tiles per work item
// from L2 into shared memory (own blocks + the t/x/y neighbour blocks).  ncu on
// 16^3x32 (profiles/r1_ncu_ring_*_b16_cfg2_s2.json) shows those TMA reads
// running at 11.2-11.7 TB/s for both c128 and c64 -- the L2 -> SM throughput
// cap of the part -- with the consumer warps stalled on tile arrival.  The
// apply is bound by L2 -> SM bytes, not by HBM.
//
// What changes: a CTA owns a *column* (one z-line segment of LY adjacent
// lines in y, at fixed x) and marches along t over a chunk of slices.  The
// t hops never touch a neighbour tile:
//   * the forward t hop of site s-1 needs psi(s), which is this step's own
//     tile -- the contribution is added to the accumulator kept in registers
//     from the previous step, and out(s-1) is written then;
//   * the backward t hop of site s needs U_0(s-1)^H P+ psi(s-1): the projected
//     half spinor P+ psi(s-1) is carried in registers from the previous step.
// So a step streams 5 tiles (own, x+, x-, y+, y-) instead of 7, and with
// LY = 2 the y neighbour tiles shrink to one line each (the inner y hops read
// the own tile): 4 tiles per line.  Link tiles: U_0(s-1) and U_3 come with the
// own tile; U_1 (own / x-1) with the x tiles; U_2 (own / y-1) with the y tiles
// (and with the own tile when LY > 1).
//
// Work units are (column, t-chunk) pairs; a unit costs one extra own tile at
// each end (the prologue slice t0-1 seeds the carry, the epilogue slice t1
// closes the forward hop of t1-1).  The chunk count is chosen on the host to
// balance units over the persistent grid.
//
// Accumulation order per site (self, z+, z-, [inner y], x+, x-, y+, y-, t-,
// t+) differs from the ring kernel; results agree to rounding (tests compare
// against the oracle at 1e-12 / 1e-5).
#pragma once

#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"

namespace b200wd {

template <typename R, int V, int B, int NB, int LY> struct TsShape {
  static constexpr int BT = B / V;              // threads per site
  static constexpr int SEG = 8 * NB;            // sites per line segment
  static constexpr int NC = BT * SEG * LY;      // consumer threads
  static constexpr int NCW = NC / 32;           // consumer warps
  static constexpr int NT = NC + 32;            // + producer warp
  // CTAs per SM the register allocation must allow.  With 5 (or 3) warps per
  // CTA some SM sub-partitions hold one warp more than others, so two CTAs fit
  // only if ptxas keeps 3 warps within the 16K registers of a sub-partition
  // (<= 168 per thread); otherwise a 160-thread CTA runs alone on its SM.
  static constexpr int MINB = NT <= 96 ? 4 : (NT <= 160 ? 2 : 1);
  static constexpr int SEGC = NB * 96 * B;      // spinor complex per segment
  static constexpr int LSEG = NB * 72;          // link complex per segment, one direction
  static constexpr int SPIN = LY * SEGC;        // own / x tiles: LY segments
  static constexpr int LNK = LY * LSEG;
  static constexpr int NREG = LY > 1 ? 3 : 2;   // link regions of the own tile (U_3, U_0(s-1)[, U_2])
  static constexpr int SLOT = SPIN + NREG * LNK;
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
  static constexpr bool valid = (NC % 32 == 0) && NC >= 64 && NC <= 512 && (B % V == 0) &&
                                (size_t)SLOT_BYTES * 3 + 64 <= 227 * 1024;
  static size_t smem(int S) { return (size_t)SLOT_BYTES * S + 16 * S; }
};

// Column / chunk decomposition of the destination slices [ta, ta + nT).
struct TsGrid {
  int32_t lz;      // segments per z line
  int32_t ny;      // line groups in y (Y / LY)
  int64_t ncol;    // X * ny * lz
  int32_t ta, nT;  // destination slices
  int32_t nch;     // t chunks per column
  int64_t n_units; // ncol * nch
  int32_t px, py;  // column patch (x, y-groups) of the traversal; 0: natural order
  int32_t pf;      // L2 prefetch distance of the own tiles in steps (0: off)
};

struct TsUnit {
  int x, y, zi;  // y: line group (first line y * LY)
  int t0, t1;
};

__device__ __forceinline__ TsUnit ts_decode(int64_t u, const TsGrid& g) {
  TsUnit w;
  const int64_t chunk = u / g.ncol;
  uint32_t c = (uint32_t)(u - chunk * g.ncol);
  w.t0 = g.ta + (int)((chunk * g.nT) / g.nch);
  w.t1 = g.ta + (int)(((chunk + 1) * g.nT) / g.nch);
  w.zi = (int)(c % (uint32_t)g.lz);
  c /= (uint32_t)g.lz;
  int yg;
  if (g.px == 0) {
    yg = (int)(c % (uint32_t)g.ny);
    w.x = (int)(c / (uint32_t)g.ny);
  } else {
    const uint32_t pa = (uint32_t)(g.px * g.py);
    const uint32_t within = c % pa, patch = c / pa;
    const uint32_t npy = (uint32_t)(g.ny / g.py);
    w.x = (int)((patch / npy) * g.px + within / g.py);
    yg = (int)((patch % npy) * g.py + within % g.py);
  }
  w.y = yg;  // line group; the first line is yg * LY
  return w;
}

__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// site block index of the first block of segment zi of line (t, x, y)
__device__ __forceinline__ int64_t ts_blk(int t, int x, int y, int zi, const HopParams& p, int nb) {
  return (((int64_t)t * p.X + x) * p.Y + y) * (int64_t)(p.Z >> 3) + (int64_t)zi * nb;
}

// Copy nl consecutive lines (y .. y+nl-1, no wrap) of segment zi into dst:
// spinor segments (SEGC complex each) or one link direction (LSEG each).
template <typename C>
__device__ __forceinline__ void ts_copy(C* dst, const C* base, int64_t blk0, int nl, int64_t line_blks,
                                        int per_seg, int blk_elems, bool whole, uint64_t* bar) {
  if (whole || nl == 1) {
    bulk_g2s(dst, base + blk0 * blk_elems, (uint32_t)(nl * per_seg * sizeof(C)), bar);
  } else {
    for (int l = 0; l < nl; ++l)
      bulk_g2s(dst + l * per_seg, base + (blk0 + l * line_blks) * blk_elems, (uint32_t)(per_seg * sizeof(C)), bar);
  }
}

// acc += reconstruct(M h) with M = U (FWD) or U^H (!FWD) read from `up`
// (entry e at up[8 e]), one output colour at a time: row i of M yields g[0][i]
// and g[1][i], which are folded into the accumulator at once, so neither g
// nor the whole link matrix is live.
template <int MU, bool FWD, typename R, int V>
__device__ __forceinline__ void ts_mv_acc(cx<R> (&acc)[V][12], const cx<R>* up, const cx<R> (&h)[V][2][3]) {
  using C = cx<R>;
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
        if constexpr (sizeof(R) == 8) {
          C a = mk(R(0), R(0));
#pragma unroll
          for (int j = 0; j < 3; ++j) a = FWD ? cmac(a, m[j], h[v][q][j]) : cmacc(a, m[j], h[v][q][j]);
          g[q] = a;
        } else {
          C a = mk(R(0), R(0));
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const C hs = mk(-h[v][q][j].y, h[v][q][j].x);
            a = FWD ? cmac_s(a, m[j], h[v][q][j], hs) : cmacc_s(a, m[j], h[v][q][j], hs);
          }
          g[q] = a;
        }
      }
      // reconstruction (accumulate_spin): upper spin S += g[S]; lower spin S += phase(g[a_perm(S)])
      constexpr int c0 = FWD ? adj_code(MU, 0) : ((adj_code(MU, 0) + 2) & 3);
      constexpr int c1 = FWD ? adj_code(MU, 1) : ((adj_code(MU, 1) + 2) & 3);
      acc[v][i] = cadd(acc[v][i], g[0]);
      acc[v][3 + i] = cadd(acc[v][3 + i], g[1]);
      acc[v][6 + i] = cadd(acc[v][6 + i], phase<c0>(g[a_perm(MU, 0)]));
      acc[v][9 + i] = cadd(acc[v][9 + i], phase<c1>(g[a_perm(MU, 1)]));
    }
  }
}

// One hop with the spinor in shared memory (or behind a generic pointer),
// projecting 12 -> 6 as the components arrive so the neighbour spinor is never
// live in registers as a whole: the t stream keeps the accumulator and the
// carried half spinor live across every hop.
template <int MU, bool FWD, int S, typename C>
__device__ __forceinline__ C ts_phase(C b) {
  constexpr int code = FWD ? a_code(MU, S) : ((a_code(MU, S) + 2) & 3);
  return phase<code>(b);
}
template <int MU, bool FWD, typename R, int V, int KST>
__device__ __forceinline__ void ts_hop(cx<R> (&acc)[V][12], const cx<R>* sp, const cx<R>* up) {
  using C = cx<R>;
  C h[V][2][3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    C a[V], b[V];
    VecIO<R, V>::lds(a, sp + c * KST);
    VecIO<R, V>::lds(b, sp + (6 + 3 * a_perm(MU, 0) + c) * KST);
#pragma unroll
    for (int v = 0; v < V; ++v) h[v][0][c] = cadd(a[v], ts_phase<MU, FWD, 0>(b[v]));
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    C a[V], b[V];
    VecIO<R, V>::lds(a, sp + (3 + c) * KST);
    VecIO<R, V>::lds(b, sp + (6 + 3 * a_perm(MU, 1) + c) * KST);
#pragma unroll
    for (int v = 0; v < V; ++v) h[v][1][c] = cadd(a[v], ts_phase<MU, FWD, 1>(b[v]));
  }
  ts_mv_acc<MU, FWD, R, V>(acc, up, h);
}

// L2 prefetch cursor over a CTA's concatenated (unit, slice) step sequence: the
// own tile data of the step g.pf ahead is requested into L2 with
// cp.async.bulk.prefetch, so the first-touch DRAM latency of a new column's
// prologue / first steps overlaps the previous column's last steps.
template <typename C, int NB, int LY, int B>
struct TsPrefetch {
  const HopParams& p;
  const TsGrid& g;
  const C* src;
  const C* U;
  int64_t u;
  TsUnit w;
  int s = 0;
  __device__ TsPrefetch(const HopParams& p_, const TsGrid& g_, const C* s_, const C* u_)
      : p(p_), g(g_), src(s_), U(u_), u(blockIdx.x) {
    if (u < g.n_units) {
      w = ts_decode(u, g);
      s = w.t0 - 1;
    }
  }
  __device__ void issue() const {
    if (u >= g.n_units) return;
    const int64_t nblk = p.n >> 3, line_blks = p.Z >> 3;
    const int y = w.y * LY;
    const int64_t bq = ts_blk(wrapi(s, p.T), w.x, y, w.zi, p, NB);
    const int64_t bq1 = ts_blk(wrapi(s - 1, p.T), w.x, y, w.zi, p, NB);
    const bool main = s >= w.t0 && s < w.t1;
    for (int ll = 0; ll < LY; ++ll) {
      const int64_t o = ll * line_blks;
      bulk_prefetch_l2(src + (bq + o) * 96 * B, (uint32_t)(NB * 96 * B * sizeof(C)));
      if (s >= w.t0) bulk_prefetch_l2(U + (bq1 + o) * 72, (uint32_t)(NB * 72 * sizeof(C)));
      if (main) {
#pragma unroll
        for (int mu = 1; mu < 4; ++mu) bulk_prefetch_l2(U + (mu * nblk + bq + o) * 72, (uint32_t)(NB * 72 * sizeof(C)));
      }
    }
  }
  __device__ void advance() {
    if (u >= g.n_units) return;
    if (++s > w.t1) {
      u += gridDim.x;
      if (u < g.n_units) {
        w = ts_decode(u, g);
        s = w.t0 - 1;
      }
    }
  }
  __device__ void prime() {  // point the cursor g.pf steps ahead of the first step
    for (int k = 0; k < g.pf; ++k) advance();
  }
  __device__ void step() {  // once per producer step
    issue();
    advance();
  }
};

// ZG: segments are not whole z lines; the z hops at the segment edges read
// global memory through generic pointers.
template <typename R, int V, int B, int NB, int LY, bool ZG>
__global__ void __launch_bounds__(TsShape<R, V, B, NB, LY>::NT, TsShape<R, V, B, NB, LY>::MINB) hop_tstream_kernel(const HopParams p, const TsGrid g,
                                                                                    int S) {
  using C = cx<R>;
  using Sh = TsShape<R, V, B, NB, LY>;
  constexpr int KST = 8 * B;
  constexpr int SEG = Sh::SEG;
  if (hop_stopped(p)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * Sh::SLOT);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Sh::NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int64_t nblk = p.n >> 3;
  const int64_t line_blks = p.Z >> 3;  // blocks per z line = distance between y-adjacent segments
  const bool whole = g.lz == 1;

  if (tid >= Sh::NC) {
    // ---------------- producer: one elected lane issues every copy ----------------
    if (tid == Sh::NC) {
      const C* src = static_cast<const C*>(p.src);
      const C* U = static_cast<const C*>(p.U);
      int pslot = 0, pfirst = 1;
      uint32_t pphase = 0;
      auto acquire = [&]() {
        if (!pfirst) mbar_wait(&empty[pslot], pphase ^ 1u);
      };
      auto advance = [&]() {
        if (++pslot == S) {
          pslot = 0;
          pphase ^= 1u;
          pfirst = 0;
        }
      };
      constexpr int SB = 96 * B;  // spinor complex per block
      TsPrefetch<C, NB, LY, B> pfc(p, g, src, U);
      if (g.pf > 0) pfc.prime();
      for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
        const TsUnit w = ts_decode(u, g);
        const int y = w.y * LY;
        for (int s = w.t0 - 1; s <= w.t1; ++s) {
          const int ts = wrapi(s, p.T);
          const int kind = s < w.t0 ? 0 : (s == w.t1 ? 2 : 1);  // prologue / main / epilogue
          if (g.pf > 0) pfc.step();  // warm L2 with the own data g.pf steps ahead (across units)
          {  // own tile
            acquire();
            C* slot = ring + pslot * Sh::SLOT;
            uint64_t* bar = &full[pslot];
            const int nlink = kind == 0 ? 0 : (kind == 2 ? 1 : Sh::NREG);
            mbar_expect_tx(bar, (uint32_t)((Sh::SPIN + nlink * Sh::LNK) * sizeof(C)));
            const int64_t b0 = ts_blk(ts, w.x, y, w.zi, p, NB);
            ts_copy(slot, src, b0, LY, line_blks, Sh::SEGC, SB, whole, bar);
            if (kind >= 1) {
              const int64_t bp = ts_blk(wrapi(s - 1, p.T), w.x, y, w.zi, p, NB);
              ts_copy(slot + Sh::SPIN + Sh::LNK, U + 0 * nblk * 72, bp, LY, line_blks, Sh::LSEG, 72, whole, bar);
            }
            if (kind == 1) {
              ts_copy(slot + Sh::SPIN, U + 3 * nblk * 72, b0, LY, line_blks, Sh::LSEG, 72, whole, bar);
              if constexpr (LY > 1)
                ts_copy(slot + Sh::SPIN + 2 * Sh::LNK, U + 2 * nblk * 72, b0, LY, line_blks, Sh::LSEG, 72, whole,
                        bar);
            }
            advance();
          }
          if (kind != 1) continue;
          const int64_t b0 = ts_blk(ts, w.x, y, w.zi, p, NB);
          {  // x+ : neighbour lines, U_1 own
            acquire();
            C* slot = ring + pslot * Sh::SLOT;
            uint64_t* bar = &full[pslot];
            mbar_expect_tx(bar, (uint32_t)((Sh::SPIN + Sh::LNK) * sizeof(C)));
            const int64_t bn = ts_blk(ts, wrapi(w.x + 1, p.X), y, w.zi, p, NB);
            ts_copy(slot, src, bn, LY, line_blks, Sh::SEGC, SB, whole, bar);
            ts_copy(slot + Sh::SPIN, U + 1 * nblk * 72, b0, LY, line_blks, Sh::LSEG, 72, whole, bar);
            advance();
          }
          {  // x- : neighbour lines and their U_1
            acquire();
            C* slot = ring + pslot * Sh::SLOT;
            uint64_t* bar = &full[pslot];
            mbar_expect_tx(bar, (uint32_t)((Sh::SPIN + Sh::LNK) * sizeof(C)));
            const int64_t bn = ts_blk(ts, wrapi(w.x - 1, p.X), y, w.zi, p, NB);
            ts_copy(slot, src, bn, LY, line_blks, Sh::SEGC, SB, whole, bar);
            ts_copy(slot + Sh::SPIN, U + 1 * nblk * 72, bn, LY, line_blks, Sh::LSEG, 72, whole, bar);
            advance();
          }
          {  // y+ : line y+LY, U_2 of line y+LY-1
            acquire();
            C* slot = ring + pslot * Sh::SLOT;
            uint64_t* bar = &full[pslot];
            mbar_expect_tx(bar, (uint32_t)((Sh::SEGC + Sh::LSEG) * sizeof(C)));
            const int64_t bn = ts_blk(ts, w.x, wrapi(y + LY, p.Y), w.zi, p, NB);
            bulk_g2s(slot, src + bn * SB, (uint32_t)(Sh::SEGC * sizeof(C)), bar);
            const int64_t bl = ts_blk(ts, w.x, y + LY - 1, w.zi, p, NB);
            bulk_g2s(slot + Sh::SEGC, U + (2 * nblk + bl) * 72, (uint32_t)(Sh::LSEG * sizeof(C)), bar);
            advance();
          }
          {  // y- : line y-1 and its U_2
            acquire();
            C* slot = ring + pslot * Sh::SLOT;
            uint64_t* bar = &full[pslot];
            mbar_expect_tx(bar, (uint32_t)((Sh::SEGC + Sh::LSEG) * sizeof(C)));
            const int64_t bn = ts_blk(ts, w.x, wrapi(y - 1, p.Y), w.zi, p, NB);
            bulk_g2s(slot, src + bn * SB, (uint32_t)(Sh::SEGC * sizeof(C)), bar);
            bulk_g2s(slot + Sh::SEGC, U + (2 * nblk + bn) * 72, (uint32_t)(Sh::LSEG * sizeof(C)), bar);
            advance();
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int r0 = (tid % Sh::BT) * V;
  const int ys = tid / Sh::BT;  // site in the item
  const int l = ys / SEG;       // line in the item
  const int zs = ys % SEG;      // z offset in the segment
  const int so = ((l * NB + (zs >> 3)) * 96 + (zs & 7)) * B + r0;  // own spinor (k = 0) in a LY-segment tile
  const int lso = (l * NB + (zs >> 3)) * 72 + (zs & 7);            // own link (e = 0) in a LY-segment region
  const int so1 = ((zs >> 3) * 96 + (zs & 7)) * B + r0;            // own spinor in a 1-segment tile
  const int lso1 = (zs >> 3) * 72 + (zs & 7);                      // own link in a 1-segment region
  const bool lead = (tid & 31) == 0;
  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  R scb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) scb[v] = (p.scale ? R(__ldg(p.scale + r0 + v)) : R(1)) * R(p.beta);
  const R ab = (p.xself != nullptr) ? R(p.alpha / p.beta) : R(0);
  const bool self_is_src = p.xself == p.src;
  const int64_t sY = p.Z, sX = (int64_t)p.Y * p.Z;

  int cslot = 0;
  uint32_t cphase = 0;
  auto wait_tile = [&]() -> const C* {
    mbar_wait(&full[cslot], cphase);
    return ring + cslot * Sh::SLOT;
  };
  auto release = [&]() {
    __syncwarp();
    if (lead) mbar_arrive(&empty[cslot]);
    if (++cslot == S) {
      cslot = 0;
      cphase ^= 1u;
    }
  };

  for (int64_t u = blockIdx.x; u < g.n_units; u += gridDim.x) {
    const TsUnit w = ts_decode(u, g);
    const int yl = w.y * LY + l;          // this thread's line
    const int z = w.zi * SEG + zs;        // this thread's z
    const int64_t s_xyz = (int64_t)w.x * sX + (int64_t)yl * sY + z;  // site offset inside a slice
    C acc[V][12];
    C carry[V][2][3];  // P+ psi(s-1) (without the 1/2)
    {  // prologue: seed the carry from slice t0-1
      const C* own = wait_tile();
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        C tmp[V];
        VecIO<R, V>::lds(tmp, own + so + k * KST);
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v][k] = tmp[v];  // acc as scratch
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        project_spin<0, false, 0>(carry[v][0], acc[v]);
        project_spin<0, false, 1>(carry[v][1], acc[v]);
      }
      release();
    }
    for (int s = w.t0; s <= w.t1; ++s) {
      const C* own = wait_tile();
      {
        // Ordered to keep few values live: (1) forward t hop of site s-1 from
        // P- psi(s) and its output, (2) acc(s) from the carried P+ psi(s-1),
        // (3) psi(s) re-read for the self term and the next carry.
        const C* u0 = own + Sh::SPIN + Sh::LNK + lso;  // U_0(s-1) at this (x, y, z)
        if (s > w.t0) {
          C hm[V][2][3];
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            C up[V], lo[V];
            VecIO<R, V>::lds(up, own + so + k * KST);
            VecIO<R, V>::lds(lo, own + so + (k + 6) * KST);
#pragma unroll
            for (int v = 0; v < V; ++v) hm[v][k / 3][k % 3] = cadd(up[v], lo[v]);  // P-_0 (A_0 = 1)
          }
          ts_mv_acc<0, true, R, V>(acc, u0, hm);
          C* out = static_cast<C*>(p.out) + spinor_base((int64_t)(s - 1) * p.per_t + s_xyz, 12, B) + r0;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            C res[V];
#pragma unroll
            for (int v = 0; v < V; ++v) res[v] = mk(scb[v] * acc[v][k].x, scb[v] * acc[v][k].y);
            VecIO<R, V>::st(out + k * KST, res);
          }
        }
        if (s == w.t1) {
          release();
          break;
        }
        {  // backward t hop of site s: acc = reconstruct(U_0(s-1)^H carry)
#pragma unroll
          for (int v = 0; v < V; ++v)
#pragma unroll
            for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
          ts_mv_acc<0, false, R, V>(acc, u0, carry);
        }
        {  // self term and the next carry P+ psi(s) = u - l
          const int64_t d = (int64_t)s * p.per_t + s_xyz;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            C up[V], lo[V];
            VecIO<R, V>::lds(up, own + so + k * KST);
            VecIO<R, V>::lds(lo, own + so + (k + 6) * KST);
#pragma unroll
            for (int v = 0; v < V; ++v) carry[v][k / 3][k % 3] = csub(up[v], lo[v]);
            if (self_is_src || p.xself) {
              if (!self_is_src) {
                VecIO<R, V>::ld(up, static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0 + k * KST);
                VecIO<R, V>::ld(lo, static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0 + (k + 6) * KST);
              }
#pragma unroll
              for (int v = 0; v < V; ++v) {
                acc[v][k] = mk(acc[v][k].x + ab * up[v].x, acc[v][k].y + ab * up[v].y);
                acc[v][k + 6] = mk(acc[v][k + 6].x + ab * lo[v].x, acc[v][k + 6].y + ab * lo[v].y);
              }
            }
          }
        }
      }
      // z hops from the own tile (U_3 own in region A)
      {
        const C* ua = own + Sh::SPIN;
        const int64_t slice = (int64_t)wrapi(s, p.T) * p.per_t;
        const int zp = zs + 1, zm = zs - 1;
        if constexpr (!ZG) {
          const int zpp = zp == SEG ? 0 : zp, zmm = zm < 0 ? SEG - 1 : zm;
          ts_hop<3, true, R, V, KST>(acc, own + ((l * NB + (zpp >> 3)) * 96 + (zpp & 7)) * B + r0, ua + lso);
          ts_hop<3, false, R, V, KST>(acc, own + ((l * NB + (zmm >> 3)) * 96 + (zmm & 7)) * B + r0,
                                      ua + (l * NB + (zmm >> 3)) * 72 + (zmm & 7));
        } else {
          {
            const C* sp;
            if (zp < SEG) sp = own + ((l * NB + (zp >> 3)) * 96 + (zp & 7)) * B + r0;
            else sp = src + spinor_base(slice + s_xyz - z + wrapi(z + 1, p.Z), 12, B) + r0;
            ts_hop<3, true, R, V, KST>(acc, sp, ua + lso);
          }
          {
            const C *sp, *up;
            if (zm >= 0) {
              sp = own + ((l * NB + (zm >> 3)) * 96 + (zm & 7)) * B + r0;
              up = ua + (l * NB + (zm >> 3)) * 72 + (zm & 7);
            } else {
              const int64_t xs = slice + s_xyz - z + wrapi(z - 1, p.Z);
              sp = src + spinor_base(xs, 12, B) + r0;
              up = U + link_base(xs, 3, nblk);
            }
            ts_hop<3, false, R, V, KST>(acc, sp, up);
          }
        }
      }
      if constexpr (LY > 1) {  // inner y hops from the own tile (U_2 own in region C)
        const C* uc = own + Sh::SPIN + 2 * Sh::LNK;
        if (l + 1 < LY) ts_hop<2, true, R, V, KST>(acc, own + so + NB * 96 * B, uc + lso);
        if (l > 0) ts_hop<2, false, R, V, KST>(acc, own + so - NB * 96 * B, uc + lso - NB * 72);
      }
      release();
      {  // x+
        const C* t = wait_tile();
        ts_hop<1, true, R, V, KST>(acc, t + so, t + Sh::SPIN + lso);
        release();
      }
      {  // x-
        const C* t = wait_tile();
        ts_hop<1, false, R, V, KST>(acc, t + so, t + Sh::SPIN + lso);
        release();
      }
      {  // y+ (outer line only)
        const C* t = wait_tile();
        if (l == LY - 1) ts_hop<2, true, R, V, KST>(acc, t + so1, t + Sh::SEGC + lso1);
        release();
      }
      {  // y- (first line only)
        const C* t = wait_tile();
        if (l == 0) ts_hop<2, false, R, V, KST>(acc, t + so1, t + Sh::SEGC + lso1);
        release();
      }
    }
  }
}

// ---- host side ----------------------------------------------------------------

struct TsCfg {
  int nb = 0, ly = 0, s = 0, nch = 0, pf = -1, px = 0, py = 0;
};
static TsCfg ts_env() {
  static TsCfg c{-1, -1, -1, -1, -1, 0, 0};
  if (c.nb < 0) {
    c = TsCfg{};
    const char* e = getenv("B200WD_TS_CFG");
    if (e) sscanf(e, "%d,%d,%d,%d,%d,%d,%d", &c.nb, &c.ly, &c.s, &c.nch, &c.pf, &c.px, &c.py);
  }
  return c;
}
static bool ts_enabled() {
  static int en = -1;
  if (en < 0) {
    const char* e = getenv("B200WD_TSTREAM");
    en = (e && e[0] == '0') ? 0 : 1;
  }
  return en == 1;
}

// chunks per column: balance ceil(units / grid) * (tiles per unit)
static int ts_choose_nch(int64_t ncol, int nT, int64_t grid, int tiles_per_step) {
  int best = 1;
  double best_cost = 1e300;
  for (int nch = 1; nch <= nT; ++nch) {
    const int64_t units = ncol * nch;
    const int64_t waves = (units + grid - 1) / grid;
    const int steps = (nT + nch - 1) / nch;
    const double cost = (double)waves * (tiles_per_step * steps + 2);
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = nch;
    }
  }
  return best;
}

template <typename R, int V, int B, int NB, int LY, bool ZG>
static bool launch_ts_kernel(const HopParams& p, const TsGrid& g0, int S, int nch, int pf, cudaStream_t st) {
  using Sh = TsShape<R, V, B, NB, LY>;
  const size_t smem = Sh::smem(S);
  LaunchFacts f;
  if (!launch_facts((const void*)hop_tstream_kernel<R, V, B, NB, LY, ZG>, Sh::NT, smem, f)) return false;
  TsGrid g = g0;
  const int64_t grid_max = (int64_t)f.occ * persistent_sms(f.sm_count);
  g.nch = nch > 0 ? (nch > g.nT ? g.nT : nch) : ts_choose_nch(g.ncol, g.nT, grid_max, LY > 1 ? 4 : 5);
  g.n_units = g.ncol * g.nch;
  g.pf = pf < 0 ? 0 : pf;
  int64_t grid = grid_max < g.n_units ? grid_max : g.n_units;
  hop_tstream_kernel<R, V, B, NB, LY, ZG><<<(unsigned)grid, Sh::NT, smem, st>>>(p, g, S);
  return true;
}

template <typename R, int V, int B, int NB, int LY>
static bool launch_ts_nb(const HopParams& p, int S, int nch, int pf, int px, int py, cudaStream_t st) {
  using Sh = TsShape<R, V, B, NB, LY>;
  if constexpr (!Sh::valid) {
    return false;
  } else {
    if (p.Z % Sh::SEG || p.Y % LY) return false;
    TsGrid g{};
    g.lz = p.Z / Sh::SEG;
    g.ny = p.Y / LY;
    g.ncol = (int64_t)p.X * g.ny * g.lz;
    g.ta = (int32_t)(p.d_begin / p.per_t);
    g.nT = (int32_t)((p.d_end - p.d_begin) / p.per_t);
    if (px > 0 && py > 0 && p.X % px == 0 && g.ny % py == 0) {
      g.px = px;
      g.py = py;
    }
    if (S <= 0) S = (int)((200 * 1024) / Sh::SLOT_BYTES);
    if (S < 3) S = 3;
    if (S > 8) S = 8;
    while (Sh::smem(S) > 227 * 1024 && S > 3) --S;
    if (Sh::smem(S) > 227 * 1024) return false;
    if (g.lz == 1) return launch_ts_kernel<R, V, B, NB, LY, false>(p, g, S, nch, pf, st);
    return launch_ts_kernel<R, V, B, NB, LY, true>(p, g, S, nch, pf, st);
  }
}

// Where the stream is used by default: (NB, LY, S) per (dtype, b), measured on
// B200 against the ring kernel (tools/tune_ts.sh, tools/time_apply.py; DESIGN
// section 3): c64 b=16 0.124 vs 0.130 ms on 16^3x32 (c64 b=8: 0.072 vs 0.078,
// superseded by the two-line ring at 0.070).
// Everywhere else the ring kernel measured equal or faster (c128: the stream's
// consumers are bound by FP64 / shared-memory latency at 8 warps per SM while
// the ring is bound by L2 -> SM bytes at a similar time), so nb = 0 disables.
// B200WD_TS_CFG="NB,LY,S,NCH,PF,PX,PY" forces a shape (tuning, tests).
template <typename R, int V, int B>
static TsCfg ts_table() {
  if constexpr (sizeof(R) == 4) {
    if (B == 16) return TsCfg{2, 1, 4, 0};  // (c64 nrhs 8: the two-line ring, ring2.cuh, measured faster)
  }
  return TsCfg{};
}

// Full-lattice fields, no halos, no clover, slice-aligned destination range.
template <typename R, int V, int B>
static bool try_launch_tstream(const HopParams& p, cudaStream_t st) {
  if (!ts_enabled()) return false;
  if (p.dst_parity >= 0 || p.lam_halo != nullptr || p.beta == 0.0 || p.clov_mode != 0) return false;
  if (p.Z % 8 != 0) return false;
  if (p.d_begin % p.per_t || p.d_end % p.per_t || p.d_end <= p.d_begin) return false;
  TsCfg c = ts_table<R, V, B>();
  const TsCfg e = ts_env();
  if (e.nb <= 0 && (c.nb <= 0 || p.Z != 8 * c.nb)) return false;  // default: whole z lines only
  if (e.nb > 0) c.nb = e.nb;
  if (e.ly > 0) c.ly = e.ly;
  if (e.s > 0) c.s = e.s;
  if (e.nch > 0) c.nch = e.nch;
  if (e.pf >= 0) c.pf = e.pf;
  if (e.px > 0) c.px = e.px;
  if (e.py > 0) c.py = e.py;
#define B200WD_TS_TRY(NB_, LY_) \
  if (c.nb == NB_ && c.ly == LY_ && launch_ts_nb<R, V, B, NB_, LY_>(p, c.s, c.nch, c.pf, c.px, c.py, st)) return true;
  B200WD_TS_TRY(1, 1)
  B200WD_TS_TRY(2, 1)
  B200WD_TS_TRY(1, 2)
  B200WD_TS_TRY(2, 2)
  B200WD_TS_TRY(3, 1)
#undef B200WD_TS_TRY
  return false;
}

}  // namespace b200wd
