// Fused rhs-blocked Wilson hopping kernel for sm_100a.
//
// One thread owns V right-hand sides (V = 1 for c128, V = 2 for c64 with an
// even rhs count, so each spinor load is one 128-bit LDG) of one destination
// site.  It walks the 8 hops of the stencil (dirac.py:172-263), for each hop
//   - loads the 12 neighbour components of its rhs (component planes: the b
//     threads of a site, and the sites of a warp, read contiguous memory),
//   - projects 12 -> 6 with the monomial A_mu blocks (projectors.py:40-147;
//     sign/swap only, no multiplies),
//   - multiplies the two colour vectors by U_mu(x) or U_mu(x-mu)^H.  All b
//     threads of a site read the same link addresses, so each link entry is
//     fetched once per site and broadcast to every rhs of the block,
//   - reconstructs the lower spin half and accumulates in registers,
// and finally writes  out = scale_r (alpha * xself + beta * H src)  once.
// Neither lambda nor chi (the reference's 8 materialised half-spinor fields,
// dirac.py:273-296) ever touches memory.
#pragma once
#include <cstdio>
#include <cstdlib>

#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"

namespace b200wd {

#ifndef B200WD_L2_PREFETCH
#define B200WD_L2_PREFETCH 0  // items ahead for L2 prefetch of compulsory misses (0: off)
#endif
#ifndef B200WD_RING_NOMATH
#define B200WD_RING_NOMATH 0  // experiment: consumers skip the t/x/y arithmetic
#endif
// Experiment builds (timing only, results are wrong): bit 0 consumers only wait
// for and release every tile (no LDS, no arithmetic), bit 1 no link copies,
// bit 2 no t+1 / t-1 tiles, bit 3 consumers prefetch the t+1 blocks of a later
// item into L2 (valid results), bit 4 no output stores.
#ifndef B200WD_RING_EXP
#define B200WD_RING_EXP 0
#endif
// Link planes of a tile through the producer warp's 32 lanes (cp.async /
// LDGSTS, completion as mbarrier arrivals) instead of a second bulk copy per
// tile: the bulk-copy engine handles ~4.9 M copies/s per SM whatever their
// size (tools/mb_ingress.cu), and half of the ring's copies were 1-2 KB link
// planes.
#ifndef B200WD_LINK_LDGSTS
#define B200WD_LINK_LDGSTS 1
#endif
#ifndef B200WD_RING_PFD
#define B200WD_RING_PFD 1  // bit 3: items of this CTA ahead
#endif
// Consumers hand a t/x/y tile back to the producer as soon as its data is in
// registers (hop_load), then compute (hop_compute): the slot refills while the
// FP64 work runs.  Measured (tools/sweep_dirac.py, 16^3x32; tools/time_apply.py
// 48^3x96): c128 nrhs 16 0.564 -> 0.575, nrhs 32 0.485 -> 0.495, c64 nrhs 12
// 0.467 -> 0.485, 48^3x96 c128 nrhs 12 21.9 -> 20.8 ms; c128 nrhs <= 8 lost
// 3% (two hops of registers at 8 consumer warps), so it stays off there.
// B200WD_RING_EARLY_RELEASE=0/1 forces it (variant builds).
#ifdef B200WD_RING_EARLY_RELEASE
template <typename R, int B> __host__ __device__ constexpr bool ring_early_release() { return B200WD_RING_EARLY_RELEASE != 0; }
#else
template <typename R, int B> __host__ __device__ constexpr bool ring_early_release() { return !(sizeof(R) == 8 && B <= 8); }
#endif

// Threads per block of the hopping kernel and the occupancy target handed
// to ptxas (c128: <= 168 registers -> 3 blocks = 12 warps per SM; c64: 4 blocks).
#ifndef B200WD_HOP_THREADS
#define B200WD_HOP_THREADS 128
#endif
constexpr int kHopThreads = B200WD_HOP_THREADS;
#ifndef B200WD_MINB_C128
#define B200WD_MINB_C128 3
#endif
#ifndef B200WD_MINB_C64
#define B200WD_MINB_C64 4
#endif
// c128 nrhs 1 measured faster with a 2-block target (0.0353 vs 0.0368 ms on
// 16^3x32; nrhs 2 equal, nrhs 3 and c64 slower: profiles/r1_tstream_tuning.txt)
template <typename R, int B> struct HopMinBlocks;
template <int B> struct HopMinBlocks<double, B> { static constexpr int value = B == 1 ? 2 : B200WD_MINB_C128; };
template <int B> struct HopMinBlocks<float, B> { static constexpr int value = B200WD_MINB_C64; };

// B > 0: rhs count known at compile time (all component / link strides are
// immediates); B == 0: runtime rhs count.
template <typename R, int V, int B>
__global__ void __launch_bounds__(kHopThreads, HopMinBlocks<R, B>::value) hop_kernel(const HopParams p) {
  using C = cx<R>;
  if (hop_stopped(p)) return;
  int64_t d = p.d_begin + (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (d >= p.d_end) return;
  if (p.jump_by && d >= p.d_begin + p.jump_at) d += p.jump_by;  // two boundary slices in one launch
  const int b = B > 0 ? B : p.b;
  const int r0 = threadIdx.x * V;
  const int Z = p.Z, Y = p.Y, X = p.X, T = p.T;
  const bool par = p.dst_parity >= 0;

  // natural site and its coordinates (geometry.py:51-72)
  int64_t site = par ? 2 * d : d;
  int z = (int)(site % Z);
  int64_t q = site / Z;
  const int y = (int)(q % Y);
  q /= Y;
  const int x = (int)(q % X);
  const int t = (int)(q / X);
  if (par) {
    const int zz = z + ((t + x + y + z + p.par0 + p.dst_parity) & 1);
    site += zz - z;
    z = zz;
  }
  const int64_t sY = Z, sX = (int64_t)Y * Z, sT = p.per_t;

  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  const int kst = 8 * b;  // component stride (elements)

  C acc[V][12];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));

  auto sptr = [&](int64_t s) {
    const int64_t i = par ? (s >> 1) : s;
    return src + spinor_base(i, 12, b) + r0;
  };
  const bool halo = p.lam_halo != nullptr;

  // forward hops: P-_mu U_mu(x) psi(x+mu)  (dirac.py:222-245)
  {
    const int64_t nblk = p.n >> 3;
    const C* ux0 = U + link_base(site, 0, nblk);
    const int64_t mstr = nblk * 72;  // distance between directions
    const int64_t f3 = (z + 1 == Z) ? site - (Z - 1) : site + 1;
    const int64_t f2 = (y + 1 == Y) ? site - (int64_t)(Y - 1) * sY : site + sY;
    const int64_t f1 = (x + 1 == X) ? site - (int64_t)(X - 1) * sX : site + sX;
    const int64_t f0 = (t + 1 == T) ? site - (int64_t)(T - 1) * sT : site + sT;
    if (halo && t + 1 == T) {
      const int64_t fi = par ? (f0 >> 1) : f0;
      const C* hp = static_cast<const C*>(p.lam_halo) + fi * b + r0;
      hop_lam_halo<R, V>(acc, hp, p.nf * b, ux0, 8);
    } else {
      hop_full<0, true, R, V>(acc, sptr(f0), kst, ux0, 8);
    }
    hop_full<1, true, R, V>(acc, sptr(f1), kst, ux0 + 1 * mstr, 8);
    hop_full<2, true, R, V>(acc, sptr(f2), kst, ux0 + 2 * mstr, 8);
    hop_full<3, true, R, V>(acc, sptr(f3), kst, ux0 + 3 * mstr, 8);
  }
  // backward hops: P+_mu U_mu(x-mu)^H psi(x-mu)  (dirac.py:185-219, 248-255)
  {
    const int64_t b3 = (z == 0) ? site + (Z - 1) : site - 1;
    const int64_t b2 = (y == 0) ? site + (int64_t)(Y - 1) * sY : site - sY;
    const int64_t b1 = (x == 0) ? site + (int64_t)(X - 1) * sX : site - sX;
    const int64_t b0 = (t == 0) ? site + (int64_t)(T - 1) * sT : site - sT;
    if (halo && t == 0) {
      const int64_t fi = par ? (site >> 1) : site;
      const C* hp = static_cast<const C*>(p.chi_halo) + fi * b + r0;
      hop_chi_halo<R, V>(acc, hp, p.nf * b);
    } else {
      hop_full<0, false, R, V>(acc, sptr(b0), kst, U + link_base(b0, 0, p.n >> 3), 8);
    }
    hop_full<1, false, R, V>(acc, sptr(b1), kst, U + link_base(b1, 1, p.n >> 3), 8);
    hop_full<2, false, R, V>(acc, sptr(b2), kst, U + link_base(b2, 2, p.n >> 3), 8);
    hop_full<3, false, R, V>(acc, sptr(b3), kst, U + link_base(b3, 3, p.n >> 3), 8);
  }

  // epilogue: out = scale_r (alpha xself + beta acc)
  const int64_t o = spinor_base(d, 12, b) + r0;
  C* out = static_cast<C*>(p.out) + o;
  const C* xs = p.xself ? static_cast<const C*>(p.xself) + o : nullptr;
  R sc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sc[v] = p.scale ? R(__ldg(p.scale + r0 + v)) : R(1);
  const R beta = R(p.beta), alpha = R(p.alpha);
  if (p.clov_mode != 0) {  // site-local 12x12 block term (clover or its inverse)
    const C* cl = static_cast<const C*>(p.clov) + clover_base(d);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      C x[12], t[12], y[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        if (xs) {
          C xv[V];
          VecIO<R, V>::ld(xv, xs + k * kst);
          x[k] = xv[v];
        } else {
          x[k] = mk(R(0), R(0));
        }
      }
      if (p.clov_mode == 1) {
        clover_mul(y, x, cl);
#pragma unroll
        for (int k = 0; k < 12; ++k)
          acc[v][k] = mk(sc[v] * (alpha * x[k].x - y[k].x + beta * acc[v][k].x),
                         sc[v] * (alpha * x[k].y - y[k].y + beta * acc[v][k].y));
      } else {
#pragma unroll
        for (int k = 0; k < 12; ++k)
          t[k] = mk(alpha * x[k].x + beta * acc[v][k].x, alpha * x[k].y + beta * acc[v][k].y);
        clover_mul(y, t, cl);
#pragma unroll
        for (int k = 0; k < 12; ++k) acc[v][k] = mk(sc[v] * y[k].x, sc[v] * y[k].y);
      }
    }
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      C res[V];
#pragma unroll
      for (int v = 0; v < V; ++v) res[v] = acc[v][k];
      VecIO<R, V>::st(out + k * kst, res);
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    C res[V];
    if (xs) {
      C xv[V];
      VecIO<R, V>::ld(xv, xs + k * kst);
#pragma unroll
      for (int v = 0; v < V; ++v)
        res[v] = mk(sc[v] * (alpha * xv[v].x + beta * acc[v][k].x), sc[v] * (alpha * xv[v].y + beta * acc[v][k].y));
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) res[v] = mk(sc[v] * beta * acc[v][k].x, sc[v] * beta * acc[v][k].y);
    }
    VecIO<R, V>::st(out + k * kst, res);
  }
}

// ---- persistent TMA ring kernel (full lattice) ---------------------------------
//
// Warp-specialised and persistent: one producer warp per CTA streams the
// inputs of consecutive work items (NB site blocks of 8 z-consecutive sites x
// all b rhs) into shared memory with cp.async.bulk (TMA 1-D bulk copies),
// completion counted by mbarrier transactions; the consumer warps compute from
// shared memory and hand each slot back through an "empty" mbarrier.
//
// A work item needs 7 tiles: its own blocks (z hops + the xself of the
// epilogue) and the neighbour blocks in -+t, -+x, -+y.  Because a site block is
// 8 z-consecutive sites and Z % 8 == 0, the t/x/y neighbours of NB consecutive
// blocks are again NB consecutive blocks: one contiguous run of NB*96*b
// complex.  With the direction-major link layout the links a tile needs (U_mu
// of the own blocks for a forward hop, of the neighbour blocks for a backward
// hop, U_3 of the own blocks for the z tile) are one more contiguous run.  So
// every tile is exactly two bulk copies -- the TMA unit has a per-copy cost
// (~200-300 cycles per CTA, tools/mb_tma.cu), so copies are kept few and big.
// When an item covers whole z lines (NB*8 == Z) the z hops never leave the
// item; otherwise the z-edge sites are read with ordinary loads.
template <typename R, int V, int B, int NB_, bool PAR = false> struct RingShape {
  static constexpr int F = PAR ? 2 : 1;                  // natural sites per field site
  static constexpr int BT = B / V;                       // threads per site
  static constexpr int NB = NB_;                         // field site blocks per item
  static constexpr int NC = BT * 8 * NB;                 // consumer threads
  static constexpr int NCW = NC / 32;                    // consumer warps
  static constexpr int NT = NC + 32;                     // + producer warp
  static constexpr int SPIN = NB * 96 * B;               // complex per spinor tile
  static constexpr int LPB = 72 * F;                     // link complex per field block (one direction)
  static constexpr int SLOT = SPIN + NB * LPB;           // + one link direction per block
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
  static constexpr bool valid = (NC % 32 == 0) && NC >= 64 && NC <= 256 && (size_t)SLOT_BYTES * 2 <= 220 * 1024;
  static size_t smem(int S) { return (size_t)SLOT_BYTES * S + 16 * S; }
};

// Coordinates of the first site of a site block (32-bit arithmetic: a rank's
// local lattice has < 2^31 sites).
struct BlkCoord {
  int t, x, y, z0;
};
__device__ __forceinline__ BlkCoord block_coord(int64_t s0_nat, const HopParams& p) {
  uint32_t s0 = (uint32_t)s0_nat;
  BlkCoord c;
  c.z0 = (int)(s0 % (uint32_t)p.Z);
  s0 /= (uint32_t)p.Z;
  c.y = (int)(s0 % (uint32_t)p.Y);
  s0 /= (uint32_t)p.Y;
  c.x = (int)(s0 % (uint32_t)p.X);
  c.t = (int)(s0 / (uint32_t)p.X);
  return c;
}
template <int F = 1>
__device__ __forceinline__ void block_step(BlkCoord& c, const HopParams& p) {
  c.z0 += 8 * F;
  if (c.z0 == p.Z) {
    c.z0 = 0;
    if (++c.y == p.Y) {
      c.y = 0;
      if (++c.x == p.X) {
        c.x = 0;
        ++c.t;
      }
    }
  }
}
// natural base site of the neighbour block (natural base s0 of the own block)
template <int MU, bool FWD>
__device__ __forceinline__ int64_t block_neighbor(int64_t s0, const BlkCoord& c, const HopParams& p) {
  const int64_t sY = p.Z, sX = (int64_t)p.Y * p.Z, sT = p.per_t;
  int64_t ns;
  if constexpr (MU == 0) ns = FWD ? (c.t + 1 == p.T ? s0 - (int64_t)(p.T - 1) * sT : s0 + sT)
                                  : (c.t == 0 ? s0 + (int64_t)(p.T - 1) * sT : s0 - sT);
  else if constexpr (MU == 1) ns = FWD ? (c.x + 1 == p.X ? s0 - (int64_t)(p.X - 1) * sX : s0 + sX)
                                       : (c.x == 0 ? s0 + (int64_t)(p.X - 1) * sX : s0 - sX);
  else ns = FWD ? (c.y + 1 == p.Y ? s0 - (int64_t)(p.Y - 1) * sY : s0 + sY)
                : (c.y == 0 ? s0 + (int64_t)(p.Y - 1) * sY : s0 - sY);
  return ns;
}
__device__ __forceinline__ int64_t z_neighbor(int64_t d, int z, int Z, int step) {
  if (step > 0) return (z + 1 == Z) ? d - (Z - 1) : d + 1;
  return (z == 0) ? d + (Z - 1) : d - 1;
}

// Item index in traversal order -> item index in natural order (relative to
// d_begin).  Items are NB field blocks; lz items per z line.
__device__ __forceinline__ int64_t item_nat(int64_t it, const HopParams& p, uint32_t lz) {
  if (p.tile_x == 0) return it;
  uint32_t i = (uint32_t)it;
  const uint32_t zi = i % lz;
  i /= lz;
  const uint32_t tl = (uint32_t)(p.tile_x * p.tile_y);
  const uint32_t q = i % tl;
  i /= tl;
  const uint32_t t = i % (uint32_t)p.tile_nt;
  const uint32_t tile = i / (uint32_t)p.tile_nt;
  const uint32_t ny = (uint32_t)(p.Y / p.tile_y);
  const uint32_t x = (tile / ny) * p.tile_x + q / p.tile_y;
  const uint32_t y = (tile % ny) * p.tile_y + q % p.tile_y;
  return (((int64_t)t * p.X + x) * p.Y + y) * lz + zi;
}

// tile H in 0..5: hop (mu = H/2, forward if H even); H == 6: own blocks (z tile).
// PAR: checkerboard fields (a field block of 8 cb sites = 16 natural sites of
// one z line, Z % 16 == 0); links are always natural-site blocks.
template <typename R, int V, int B, int NB, bool PAR, int H, bool HALO = false>
__device__ __forceinline__ void ring_issue(const HopParams& p, int64_t gb0, const BlkCoord& c0, cx<R>* slot,
                                           uint64_t* full, uint64_t pol_first, uint64_t pol_t1) {
  using C = cx<R>;
  using Sh = RingShape<R, V, B, NB, PAR>;
  constexpr int F = Sh::F;
  const C* src = static_cast<const C*>(p.src);
  const C* U = static_cast<const C*>(p.U);
  const int64_t nblk = p.n >> 3;  // natural link blocks
  constexpr bool kLinks = !(B200WD_RING_EXP & 2) && !B200WD_LINK_LDGSTS;
  constexpr int kSlotTx = kLinks ? Sh::SLOT : Sh::SPIN;
  if constexpr (H == 6) {
    mbar_expect_tx(full, (uint32_t)(kSlotTx * sizeof(C)));
    bulk_g2s(slot, src + gb0 * 96 * B, Sh::SPIN * sizeof(C), full);
    if (kLinks) bulk_g2s(slot + Sh::SPIN, U + (3 * nblk + F * gb0) * 72, NB * Sh::LPB * sizeof(C), full);
  } else {
    constexpr int MU = H >> 1;
    constexpr bool FWD = !(H & 1);
    if constexpr (HALO && H <= 1) {
      // T-split boundary slice (halo.py:370-387): the t+1 neighbour of the last
      // local slice is the lam face of rank+1, the t-1 neighbour of slice 0 the
      // chi face of rank-1 -- 6 half-spinor components per face site, stored
      // (6, nf, b); the item's NB*8 field sites are one run per component.
      const void* face = H == 0 ? (c0.t + 1 == p.T ? p.lam_halo : nullptr) : (c0.t == 0 ? p.chi_halo : nullptr);
      if (face != nullptr) {
        const C* fp = static_cast<const C*>(face);
        const int64_t i0 = gb0 * 8 - (int64_t)c0.t * (p.per_t / F);  // face index of the item's first field site
        constexpr int RUN = NB * 8 * B;
        mbar_expect_tx(full, (uint32_t)((6 * RUN + (kLinks ? NB * Sh::LPB : 0)) * sizeof(C)));
#pragma unroll
        for (int k = 0; k < 6; ++k) bulk_g2s(slot + k * RUN, fp + (k * p.nf + i0) * B, RUN * sizeof(C), full);
        // U_0 of the own blocks (the lam hop multiplies at the destination; unused by chi)
        if (kLinks) bulk_g2s(slot + Sh::SPIN, U + (0 * nblk + F * gb0) * 72, NB * Sh::LPB * sizeof(C), full);
        return;
      }
    }
    // neighbour field blocks of the NB own blocks: contiguous unless a wrap falls inside the item
    mbar_expect_tx(full, (uint32_t)(kSlotTx * sizeof(C)));
    const int64_t nb0 = block_neighbor<MU, FWD>(gb0 * 8 * F, c0, p) / (8 * F);
    bool contiguous = true;
    if constexpr (NB > 1) {
      BlkCoord c = c0;
#pragma unroll
      for (int jj = 1; jj < NB; ++jj) {
        block_step<F>(c, p);
        contiguous &= block_neighbor<MU, FWD>((gb0 + jj) * 8 * F, c, p) / (8 * F) == nb0 + jj;
      }
    }
    if (contiguous) {
      if (H == 1 && p.hint_tm1)  // t-1 neighbour: the last use of these blocks in either order
        bulk_g2s_hint(slot, src + nb0 * 96 * B, Sh::SPIN * sizeof(C), full, pol_first);
      else if (H == 0 && p.hint_t1)  // t+1 neighbour: first touch
        bulk_g2s_hint(slot, src + nb0 * 96 * B, Sh::SPIN * sizeof(C), full, pol_t1);
      else
        bulk_g2s(slot, src + nb0 * 96 * B, Sh::SPIN * sizeof(C), full);
      if (kLinks)
        bulk_g2s(slot + Sh::SPIN, U + (MU * nblk + F * (FWD ? gb0 : nb0)) * 72, NB * Sh::LPB * sizeof(C), full);
    } else {
      BlkCoord c = c0;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        if (jj) block_step<F>(c, p);
        const int64_t nb = block_neighbor<MU, FWD>((gb0 + jj) * 8 * F, c, p) / (8 * F);
        bulk_g2s(slot + jj * 96 * B, src + nb * 96 * B, 96 * B * sizeof(C), full);
        if (kLinks)
          bulk_g2s(slot + Sh::SPIN + jj * Sh::LPB, U + (MU * nblk + F * (FWD ? gb0 + jj : nb)) * 72,
                   Sh::LPB * sizeof(C), full);
      }
    }
  }
}

// The link plane of tile H by the 32 lanes of the producer warp: 16-byte
// cp.async copies, then one mbarrier arrival per lane (the full barrier expects
// 1 + 32 arrivals per phase).  Same source runs as the bulk copies of ring_issue.
template <typename R, int V, int B, int NB, bool PAR, int H, bool HALO = false>
__device__ __forceinline__ void ring_issue_links(const HopParams& p, int64_t gb0, const BlkCoord& c0, cx<R>* slot,
                                                 uint64_t* full, int lane) {
  using C = cx<R>;
  using Sh = RingShape<R, V, B, NB, PAR>;
  constexpr int F = Sh::F;
  constexpr int CH = 16 / (int)sizeof(C);  // complex per 16-byte chunk
  const C* U = static_cast<const C*>(p.U);
  const int64_t nblk = p.n >> 3;
  C* dst = slot + Sh::SPIN;
  auto run = [&](C* d, const C* s, int n_cx) {
    for (int i = lane * CH; i < n_cx; i += 32 * CH) cp_async16(d + i, s + i);
  };
  if constexpr (H == 6) {
    run(dst, U + (3 * nblk + F * gb0) * 72, NB * Sh::LPB);
  } else {
    constexpr int MU = H >> 1;
    constexpr bool FWD = !(H & 1);
    bool face = false;
    if constexpr (HALO && H <= 1) face = H == 0 ? (c0.t + 1 == p.T) : (c0.t == 0);
    if (face) {
      run(dst, U + (0 * nblk + F * gb0) * 72, NB * Sh::LPB);
    } else if constexpr (FWD) {
      run(dst, U + (MU * nblk + F * gb0) * 72, NB * Sh::LPB);  // own blocks: one run
    } else {
      BlkCoord c = c0;
#pragma unroll
      for (int jj = 0; jj < NB; ++jj) {
        if (jj) block_step<F>(c, p);
        const int64_t nb = block_neighbor<MU, FWD>((gb0 + jj) * 8 * F, c, p) / (8 * F);
        run(dst + jj * Sh::LPB, U + (MU * nblk + F * nb) * 72, Sh::LPB);
      }
    }
  }
  cp_async_mbar_arrive(full);
}

// TILED: patched traversal order (checkerboard fields).  ZG: items are not
// whole z lines, the z hops at the item edges read global memory.
#ifdef B200WD_RING_MINB  // experiment builds only: CTAs per SM the register allocation must allow
#define B200WD_RING_BOUNDS(...) __launch_bounds__(__VA_ARGS__, B200WD_RING_MINB)
#else
#define B200WD_RING_BOUNDS(...) __launch_bounds__(__VA_ARGS__)
#endif
// CLOV: site-local 12x12 block term (p.clov_mode 1: - C x; 2: M (alpha x +
// beta H)) in the epilogue, the generic kernel's algebra.  The producer stages
// each item's packed blocks in a double-buffered shared-memory area behind the
// ring (kClovBufs buffers with their own full/empty barriers).
constexpr int kClovBufs = 2;
template <typename R, int NB> __host__ __device__ constexpr int clov_tile() { return NB * 336; }

template <typename R, int V, int B, int NB, bool PAR, bool TILED, bool ZG, bool CLOV = false, bool HALO = false>
__global__ void B200WD_RING_BOUNDS(RingShape<R, V, B, NB, PAR>::NT) hop_ring_kernel(const HopParams p,
                                                                                   int64_t n_items, int S) {
  using C = cx<R>;
  using Sh = RingShape<R, V, B, NB, PAR>;
  constexpr int F = Sh::F;
  constexpr int KST = 8 * B;
  if (hop_stopped(p)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  C* cbuf = ring + S * Sh::SLOT;  // CLOV: kClovBufs block tiles
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf + (CLOV ? kClovBufs * clov_tile<R, NB>() : 0));
  uint64_t* empty = full + S;
  uint64_t* cfull = empty + S;
  uint64_t* cempty = cfull + kClovBufs;

  const int tid = threadIdx.x;  // 1-D block: consumers [0, NC), producer warp [NC, NC+32)
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], B200WD_LINK_LDGSTS ? 33 : 1);
      mbar_init(&empty[i], Sh::NCW);
    }
    if constexpr (CLOV) {
      for (int i = 0; i < kClovBufs; ++i) {
        mbar_init(&cfull[i], 1);
        mbar_init(&cempty[i], Sh::NCW);
      }
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (tid >= Sh::NC) {
    const int lane = tid - Sh::NC;
    // lane 0 issues every bulk copy; with B200WD_LINK_LDGSTS all 32 lanes copy the link planes
    if (lane == 0 || B200WD_LINK_LDGSTS) {
      int pslot = 0, pfirst = 1;
      const uint64_t pol_first = l2_evict_first_policy();
      // t+1 blocks come back as own blocks one patch slice later (tiled) or
      // after a whole T slice (natural order: no reuse to protect)
      const uint64_t pol_t1 = p.hint_t1 == 2 ? l2_evict_last_policy() : pol_first;
      uint32_t pphase = 0;  // phase of the next fill of pslot; its release is phase^1 of empty
      int cb_slot = 0, cb_first = 1;
      uint32_t cb_phase = 0;
      const uint32_t lz = (uint32_t)(p.Z / (8 * F * NB));
      bool sync = TILED && p.wave_cnt != nullptr;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        if (TILED && p.wave_cnt != nullptr) {
          if (lane == 0 && sync) sync = wave_wait(p, it, n_items);
          if (B200WD_LINK_LDGSTS) __syncwarp();
        }
        int64_t gb0 = (p.d_begin >> 3) + (TILED ? item_nat(it, p, lz) : it) * NB;
        if (HALO && p.jump_by && gb0 * 8 >= p.d_begin + p.jump_at) gb0 += p.jump_by >> 3;
        const BlkCoord c0 = block_coord(gb0 * 8 * F, p);
#if B200WD_L2_PREFETCH
        if (lane == 0) {  // warm L2 with the compulsory misses of a later item of this CTA:
           // its t+1 neighbour blocks (first touch in sweep order) and links
          const int64_t nx = it + (int64_t)B200WD_L2_PREFETCH * gridDim.x;
          if (nx < n_items) {
            const int64_t gn = (p.d_begin >> 3) + (TILED ? item_nat(nx, p, lz) : nx) * NB;
            const BlkCoord cn = block_coord(gn * 8 * F, p);
            const int64_t nb = block_neighbor<0, true>(gn * 8 * F, cn, p) / (8 * F);
            const C* srcp = static_cast<const C*>(p.src);
            const C* Up = static_cast<const C*>(p.U);
            bulk_prefetch_l2(srcp + nb * 96 * B, Sh::SPIN * sizeof(C));
            const int64_t nbl = p.n >> 3;
#pragma unroll
            for (int mu = 0; mu < 4; ++mu) bulk_prefetch_l2(Up + (mu * nbl + F * gn) * 72, NB * Sh::LPB * sizeof(C));
          }
        }
#endif
#define B200WD_PRODUCE(H)                                                                   \
  {                                                                                         \
    if (pfirst == 0) {                                                                      \
      if (lane == 0) mbar_wait(&empty[pslot], pphase ^ 1u);                                 \
      if (B200WD_LINK_LDGSTS) __syncwarp();                                                 \
    }                                                                                       \
    if (lane == 0)                                                                          \
      ring_issue<R, V, B, NB, PAR, H, HALO>(p, gb0, c0, ring + pslot * Sh::SLOT, &full[pslot], pol_first, pol_t1); \
    if (B200WD_LINK_LDGSTS && !(B200WD_RING_EXP & 2))                                       \
      ring_issue_links<R, V, B, NB, PAR, H, HALO>(p, gb0, c0, ring + pslot * Sh::SLOT, &full[pslot], lane); \
    else if (B200WD_LINK_LDGSTS)                                                            \
      cp_async_mbar_arrive(&full[pslot]);                                                   \
    if (++pslot == S) {                                                                     \
      pslot = 0;                                                                            \
      pphase ^= 1u;                                                                         \
      pfirst = 0;                                                                           \
    }                                                                                       \
  }
        B200WD_PRODUCE(6)
        if (CLOV && lane == 0) {  // this item's blocks (read in the epilogue)
          if (cb_first == 0) mbar_wait(&cempty[cb_slot], cb_phase ^ 1u);
          constexpr uint32_t cbytes = (uint32_t)(clov_tile<R, NB>() * sizeof(C));
          mbar_expect_tx(&cfull[cb_slot], cbytes);
          bulk_g2s(cbuf + cb_slot * clov_tile<R, NB>(), static_cast<const C*>(p.clov) + gb0 * 336, cbytes,
                   &cfull[cb_slot]);
          if (++cb_slot == kClovBufs) {
            cb_slot = 0;
            cb_phase ^= 1u;
            cb_first = 0;
          }
        }
        if (!(B200WD_RING_EXP & 4)) {
          B200WD_PRODUCE(0)
          B200WD_PRODUCE(1)
        }
        B200WD_PRODUCE(2)
        B200WD_PRODUCE(3)
        B200WD_PRODUCE(4)
        B200WD_PRODUCE(5)
#undef B200WD_PRODUCE
        if (TILED && p.wave_cnt != nullptr && lane == 0) wave_arrive(p, it);
      }
    }
    return;
  }

  // ---- consumers ----
  const int r0 = (tid % Sh::BT) * V;
  const int ysite = tid / Sh::BT;
  const int j = ysite >> 3, lo = ysite & 7;
  const bool lead = (tid & 31) == 0;
  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  const int64_t nblk = p.n >> 3;
  const int Z = p.Z;
  R scb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) scb[v] = (p.scale ? R(__ldg(p.scale + r0 + v)) : R(1)) * R(p.beta);
  // acc accumulates (alpha/beta) xself + 2H src; out = (scale beta) acc
  const R ab = (p.xself != nullptr) ? R(p.alpha / p.beta) : R(0);
  const bool self_is_src = p.xself == p.src;

  int cslot = 0;
  uint32_t cphase = 0;
  int kslot = 0;
  uint32_t kphase = 0;
  const uint32_t lz = (uint32_t)(p.Z / (8 * F * NB));
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    // natural order keeps gb0 affine in `it`: a separate instantiation,
    // the compiler schedules that loop markedly better (tools/bench_strong.py)
    int64_t gb0 = (p.d_begin >> 3) + (TILED ? item_nat(it, p, lz) : it) * NB;
    if (HALO && p.jump_by && gb0 * 8 >= p.d_begin + p.jump_at) gb0 += p.jump_by >> 3;
    const int64_t d = (gb0 + j) * 8 + lo;  // field index of this thread's site
    // natural site: full lattice d; checkerboard 2d + (parity fix of the block's line)
    int64_t xn = d;
    if constexpr (PAR) {
      const BlkCoord cb = block_coord((gb0 + j) * 16, p);
      xn = 2 * d + ((cb.t + cb.x + cb.y + p.par0 + p.dst_parity) & 1);
    }
    const int64_t nat0 = gb0 * 8 * F;        // natural base site of the item
    const int li = (int)(xn - nat0);         // natural index inside the item's link blocks
    const int lofs = (li >> 3) * 72 + (li & 7);
    int item_t = -1;  // HALO: local slice of the item (items never straddle slices)
    if constexpr (HALO) item_t = block_coord(nat0, p).t;
    C acc[V][12];
    {  // own blocks: xself, z hops
      const int slot = cslot;
      mbar_wait(&full[slot], cphase);
      const C* zt = ring + slot * Sh::SLOT;
      if constexpr ((B200WD_RING_EXP & 8) != 0) {
        // first touch of the sweep: the t+1 blocks of a later item of this CTA,
        // requested into L2 by the consumer threads (one 128-byte line each)
        const int64_t nx = it + (int64_t)B200WD_RING_PFD * gridDim.x;
        if (nx < n_items) {
          const int64_t gn = (p.d_begin >> 3) + (TILED ? item_nat(nx, p, lz) : nx) * NB;
          const BlkCoord cn = block_coord(gn * 8 * F, p);
          const int64_t nb = block_neighbor<0, true>(gn * 8 * F, cn, p) / (8 * F);
          const char* base = reinterpret_cast<const char*>(src + nb * 96 * B);
          constexpr int kLines = (int)(Sh::SPIN * sizeof(C) / 128);
          for (int ln = tid; ln < kLines; ln += Sh::NC)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)ln * 128));
        }
      }
      if constexpr ((B200WD_RING_EXP & 1) != 0) {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
      } else {
      if (self_is_src || p.xself) {
        const C* xp = self_is_src ? zt + j * 96 * B + lo * B + r0
                                  : static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C xv[V];
          if (self_is_src) VecIO<R, V>::lds(xv, xp + k * KST);
          else VecIO<R, V>::ld(xv, xp + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][k] = mk(ab * xv[v].x, ab * xv[v].y);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
      }
      const int z = (int)((uint32_t)xn % (uint32_t)Z);
      if constexpr (ZG) {
        // z hops through generic pointers (shared memory inside the item, global
        // memory at its z edges): one branch-free load batch per hop
        {
          const int64_t xp = z_neighbor(xn, z, Z, 1);
          const int64_t fi = PAR ? (xp >> 1) : xp;
          const int64_t jb = (fi >> 3) - gb0;
          const C* sp = (jb >= 0 && jb < NB) ? zt + jb * 96 * B + (fi & 7) * B + r0
                                             : src + spinor_base(fi, 12, B) + r0;
          hop_full<3, true, R, V, true, true>(acc, sp, KST, zt + Sh::SPIN + lofs, 8);
        }
        {
          const int64_t xp = z_neighbor(xn, z, Z, -1);
          const int64_t fi = PAR ? (xp >> 1) : xp;
          const int64_t jb = (fi >> 3) - gb0;
          const int lj = (int)(xp - nat0);
          const C* sp = (jb >= 0 && jb < NB) ? zt + jb * 96 * B + (fi & 7) * B + r0
                                             : src + spinor_base(fi, 12, B) + r0;
          const C* up = (lj >= 0 && lj < 8 * F * NB) ? zt + Sh::SPIN + (lj >> 3) * 72 + (lj & 7)
                                                     : U + link_base(xp, 3, nblk);
          hop_full<3, false, R, V, true, true>(acc, sp, KST, up, 8);
        }
      } else {
        {
          const int64_t xp = z_neighbor(xn, z, Z, 1);
          const int64_t fi = PAR ? (xp >> 1) : xp;
          const int64_t jb = (fi >> 3) - gb0;
          const C* ul = zt + Sh::SPIN + lofs;  // U_3(x), own blocks
          if (jb >= 0 && jb < NB)
            hop_full<3, true, R, V, true, true>(acc, zt + jb * 96 * B + (fi & 7) * B + r0, KST, ul, 8);
          else
            hop_full<3, true, R, V, false, true>(acc, src + spinor_base(fi, 12, B) + r0, KST, ul, 8);
        }
        {
          const int64_t xp = z_neighbor(xn, z, Z, -1);
          const int64_t fi = PAR ? (xp >> 1) : xp;
          const int64_t jb = (fi >> 3) - gb0;
          const int lj = (int)(xp - nat0);
          const bool lin = lj >= 0 && lj < 8 * F * NB;
          if (jb >= 0 && jb < NB && lin)
            hop_full<3, false, R, V, true, true>(acc, zt + jb * 96 * B + (fi & 7) * B + r0, KST,
                                                 zt + Sh::SPIN + (lj >> 3) * 72 + (lj & 7), 8);
          else
            hop_full<3, false, R, V, false, false>(acc, src + spinor_base(fi, 12, B) + r0, KST,
                                                   U + link_base(xp, 3, nblk), 8);
        }
      }
      }  // !(B200WD_RING_EXP & 1)
      __syncwarp();
      if (lead) mbar_arrive(&empty[slot]);
      if (++cslot == S) {
        cslot = 0;
        cphase ^= 1u;
      }
    }

#define B200WD_CONSUME(H)                                                                            \
  {                                                                                                  \
    const int slot = cslot;                                                                          \
    mbar_wait(&full[slot], cphase);                                                                  \
    const C* sb = ring + slot * Sh::SLOT;                                                            \
    if ((B200WD_RING_EXP & 1) != 0) {                                                                \
    } else if (HALO && (H) == 0 && item_t == p.T - 1)                                                     \
      hop_lam_halo<R, V, true, true>(acc, sb + (j * 8 + lo) * B + r0, NB * 8 * B, sb + Sh::SPIN + lofs, 8); \
    else if (HALO && (H) == 1 && item_t == 0)                                                        \
      hop_chi_halo<R, V, true>(acc, sb + (j * 8 + lo) * B + r0, NB * 8 * B);                         \
    else if (ring_early_release<R, B>()) {                                                           \
      HopRegs<R, V> hr;                                                                              \
      hop_load<((H) >> 1), !((H)&1), R, V, KST>(hr, sb + j * 96 * B + lo * B + r0, sb + Sh::SPIN + lofs); \
      /* release in the middle of the product, data-dependent on every load (stencil.cuh) */        \
      hop_compute_release<((H) >> 1), !((H)&1), R, V>(acc, hr, &empty[slot], lead);                  \
      released = true;                                                                               \
    } else if (!B200WD_RING_NOMATH)                                                                  \
      hop_full<((H) >> 1), !((H)&1), R, V, true, true>(acc, sb + j * 96 * B + lo * B + r0, KST,      \
                                                        sb + Sh::SPIN + lofs, 8);                    \
    if (!released) {                                                                                 \
      __syncwarp();                                                                                  \
      if (lead) mbar_arrive(&empty[slot]);                                                           \
    }                                                                                                \
    released = false;                                                                                \
    if (++cslot == S) {                                                                              \
      cslot = 0;                                                                                     \
      cphase ^= 1u;                                                                                  \
    }                                                                                                \
  }
    bool released = false;
    if (!(B200WD_RING_EXP & 4)) {
      B200WD_CONSUME(0)
      B200WD_CONSUME(1)
    }
    B200WD_CONSUME(2)
    B200WD_CONSUME(3)
    B200WD_CONSUME(4)
    B200WD_CONSUME(5)
#undef B200WD_CONSUME

    C* out = static_cast<C*>(p.out) + spinor_base(d, 12, B) + r0;
    if constexpr (CLOV) {
      // beta acc = alpha x + beta H; mode 1: s (beta acc - C x), mode 2: s M (beta acc).
      // One 6x6 block at a time, its elements read from shared memory as used
      // (volatile: not hoisted into registers).
      const C* xs = p.xself ? static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0 : nullptr;
      mbar_wait(&cfull[kslot], kphase);
      const volatile C* cl = cbuf + kslot * clov_tile<R, NB>() + j * 336 + lo;
      const R beta = R(p.beta);
      const bool m1 = p.clov_mode == 1;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const R sc = p.scale ? R(__ldg(p.scale + r0 + v)) : R(1);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          C in[6];  // mode 1: x; mode 2: beta acc
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            if (m1) {
              C t[V];
              if (xs) VecIO<R, V>::ld(t, xs + (6 * q + k) * KST);
              in[k] = xs ? t[v] : mk(R(0), R(0));
            } else {
              in[k] = mk(beta * acc[v][6 * q + k].x, beta * acc[v][6 * q + k].y);
            }
          }
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            C y = mk(R(0), R(0));
#pragma unroll
            for (int jj = 0; jj < 6; ++jj) {
              const volatile C& e = cl[(q * 21 + (i >= jj ? i * (i + 1) / 2 + jj : jj * (jj + 1) / 2 + i)) * 8];
              const R ex = e.x, ey = i >= jj ? e.y : -e.y;
              y = mk(y.x + ex * in[jj].x - ey * in[jj].y, y.y + ex * in[jj].y + ey * in[jj].x);
            }
            const C a = acc[v][6 * q + i];
            acc[v][6 * q + i] = m1 ? mk(sc * (beta * a.x - y.x), sc * (beta * a.y - y.y)) : mk(sc * y.x, sc * y.y);
          }
        }
      }
      __syncwarp();
      if (lead) mbar_arrive(&cempty[kslot]);
      if (++kslot == kClovBufs) {
        kslot = 0;
        kphase ^= 1u;
      }
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        C res[V];
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = acc[v][k];
        VecIO<R, V>::st(out + k * KST, res);
      }
    } else if (!(B200WD_RING_EXP & 16)) {
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

// Ring configuration: site blocks per item (compile time) and ring depth
// (runtime).  Default: whole z lines per item when that gives <= 256
// consumer threads, a ring of ~100 KB per CTA (two CTAs per SM) or ~200 KB
// (one CTA) for large slots; B200WD_RING_CFG="NB,S" overrides (tuning).
struct RingCfg {
  int nb = 0, s = 0;
};
static RingCfg ring_env() {
  static RingCfg c{-1, -1};
  if (c.nb < 0) {
    c = RingCfg{};
    const char* e = getenv("B200WD_RING_CFG");
    if (e) sscanf(e, "%d,%d", &c.nb, &c.s);
  }
  return c;
}

// integer tuning knob from the environment (B200WD_L2HINT=0 turns the L2
// eviction hints of the ring copies off; measured neutral on 48^3 x 96)
static int ring_knob(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// A T slice of the source field larger than this is not reused from L2 by
// the t+1 hop of the next slice (tools/bench_strong.py on 48^3 x 96).
// (B200WD_SLICE_KB overrides: tests force the large-lattice paths on small lattices)
static int64_t slice_noreuse() {
  static const int64_t kb = ring_knob("B200WD_SLICE_KB", 48 * 1024);
  return kb << 10;
}

// L2 budget for one T slice of a traversal patch (B200WD_TILE_KB, default
// 24 MB; 0 = natural order everywhere).  The patch's t-1, t and t+1 slices
// (~3x this) must stay resident next to the streaming output and links.
static int64_t tile_budget() {
  static int64_t kb = -1;
  if (kb < 0) {
    const char* e = getenv("B200WD_TILE_KB");
    kb = e ? atoll(e) : 24 * 1024;
  }
  return kb << 10;
}

// Patch the traversal order when one T slice of the source field does not
// fit the budget: the largest tile_x | X, tile_y | Y patch (most nearly square)
// whose slice fits.  Needs whole z lines per item set and slice-aligned ranges.
static void choose_tiles(HopParams& p, int F, int NB, size_t bytes_per_field_site) {
  p.tile_x = p.tile_y = p.tile_nt = 0;
  const int64_t budget = tile_budget();
  if (budget <= 0 || p.Z % (8 * F * NB)) return;
  const int64_t per_t_field = p.per_t / F;
  if (p.d_begin % per_t_field || p.d_end % per_t_field) return;
  const int64_t line_bytes = (int64_t)(p.Z / F) * (int64_t)bytes_per_field_site;
  if ((int64_t)p.X * p.Y * line_bytes <= budget) return;
  int best_x = 0, best_y = 0;
  double best = 1e30;
  for (int tx = 1; tx <= p.X; ++tx) {
    if (p.X % tx) continue;
    for (int ty = 1; ty <= p.Y; ++ty) {
      if (p.Y % ty || (int64_t)tx * ty * line_bytes > budget) continue;
      const double perim = 1.0 / tx + 1.0 / ty;  // re-read fraction of the x/y neighbours
      if (perim < best - 1e-12) {
        best = perim;
        best_x = tx;
        best_y = ty;
      }
    }
  }
  if (best_x == 0 || (best_x == p.X && best_y == p.Y)) return;
  p.tile_x = best_x;
  p.tile_y = best_y;
  p.tile_nt = (int32_t)((p.d_end - p.d_begin) / per_t_field);
}

template <int NB>
static int64_t n_items_of(int64_t nblk) { return nblk / NB; }

// Per-device wave counters of the synchronised traversal (grown on demand,
// zeroed on the launch stream before each launch that uses them).
static int* wave_counters(int64_t n, cudaStream_t st) {
  static std::mutex mu;
  static std::map<int, std::pair<int*, int64_t>> bufs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto& b = bufs[dev];
  if (b.second < n) {
    if (b.first) cudaFree(b.first);  // synchronous: only while growing
    b.first = nullptr;
    b.second = 0;
    int64_t cap = 1 << 16;
    while (cap < n) cap <<= 1;
    if (cudaMalloc(&b.first, cap * sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    b.second = cap;
  }
  if (cudaMemsetAsync(b.first, 0, n * sizeof(int), st) != cudaSuccess) return nullptr;
  return b.first;
}

// Wave synchronisation of a patched (TILED) traversal: one wave per patch
// slice (B200WD_WAVE=1 turns it on, B200WD_WAVE_SLACK sets the slack).  Off by
// default: on the checkerboard Schur hops of 32^3 x 64 it cost 0.549 -> 0.484
// of HBM (their patch slices are small, so the waits dominate).
static void setup_waves(HopParams& p, int64_t n_items, int lz, cudaStream_t st) {
  static const int en = ring_knob("B200WD_WAVE", 0);
  static const int slack = ring_knob("B200WD_WAVE_SLACK", 2);
  p.wave_cnt = nullptr;
  if (!en || p.tile_x == 0) return;
  p.wave_items = (int64_t)p.tile_x * p.tile_y * lz;
  p.wave_slack = slack < 1 ? 1 : slack;
  const int64_t n_waves = (n_items + p.wave_items - 1) / p.wave_items;
  p.wave_cnt = wave_counters(n_waves, st);
}

// Full-lattice patched order for lattices whose T slice exceeds the L2 reuse
// limit: the largest patch (tile_x | X, tile_y | Y) whose three slices fit the
// budget (B200WD_WAVE_KB per slice), most nearly square in lines.  Off by
// default: on 48^3 x 96 (c128 nrhs 12) the synchronised patched order cuts the
// DRAM reads from 81.5 to 43.8 GB per apply (ncu, profiles/r2_wave_ncu.txt) but
// runs 23.2 ms against 22.0 ms for the natural order -- the patched item order
// costs 17% on its own even on an L2-resident lattice and the per-wave waits
// add more (tools/wave_cost.sh), while the natural order is DRAM-bound at 89%
// of the copy peak with 1.94x the compulsory traffic.
static void choose_full_tiles(HopParams& p, int NB, size_t bytes_per_site) {
  static const int64_t kb = ring_knob("B200WD_WAVE_KB", 0);
  p.tile_x = p.tile_y = p.tile_nt = 0;
  if (kb <= 0 || p.Z % (8 * NB)) return;
  if (p.d_begin % p.per_t || p.d_end % p.per_t) return;
  const int64_t line_bytes = (int64_t)p.Z * (int64_t)bytes_per_site;
  const int64_t budget = kb << 10;
  int best_x = 0, best_y = 0;
  double best = 1e30;
  for (int tx = 1; tx <= p.X; ++tx) {
    if (p.X % tx) continue;
    for (int ty = 1; ty <= p.Y; ++ty) {
      if (p.Y % ty || (int64_t)tx * ty * line_bytes > budget) continue;
      const double perim = 1.0 / tx + 1.0 / ty;
      if (perim < best - 1e-12) {
        best = perim;
        best_x = tx;
        best_y = ty;
      }
    }
  }
  if (best_x == 0 || (best_x == p.X && best_y == p.Y)) return;
  p.tile_x = best_x;
  p.tile_y = best_y;
  p.tile_nt = (int32_t)((p.d_end - p.d_begin) / p.per_t);
}

template <typename R, int V, int B, int NB, bool PAR, bool TILED, bool ZG, bool CLOV = false, bool HALO = false>
static bool launch_ring_kernel(const HopParams& p, int64_t n_items, int S, size_t smem, cudaStream_t st) {
  using Sh = RingShape<R, V, B, NB, PAR>;
  LaunchFacts f;
  if (!launch_facts((const void*)hop_ring_kernel<R, V, B, NB, PAR, TILED, ZG, CLOV, HALO>, Sh::NT, smem, f))
    return false;
  int64_t grid = (int64_t)f.occ * persistent_sms(f.sm_count);
  if (grid > n_items) grid = n_items;
  hop_ring_kernel<R, V, B, NB, PAR, TILED, ZG, CLOV, HALO><<<(unsigned)grid, Sh::NT, smem, st>>>(p, n_items, S);
  return true;
}

template <typename R, int V, int B, int NB, bool PAR>
static bool launch_ring_nb(const HopParams& p_in, int64_t nblk, int S, cudaStream_t st) {
  using Sh = RingShape<R, V, B, NB, PAR>;
  if constexpr (!Sh::valid) {
    return false;
  } else {
    if (nblk % NB) return false;
    if (p_in.jump_by && ((p_in.jump_at >> 3) % NB)) return false;  // items must not straddle the jump
    HopParams p = p_in;
    const size_t site_bytes = (size_t)12 * B * sizeof(cx<R>);
    // patched order for checkerboard fields only: measured +2-8% on the Schur
    // hops of 32^3 x 64 (tools/variants_cmp.sh); for the full-lattice apply on
    // 48^3 x 96 every patch shape tried (1..8 x 48, 48 x 2..8, 6 x 12) was
    // 10-25% slower than the natural order
    const bool clov = p.clov_mode != 0;
    const bool halo = p.lam_halo != nullptr;  // T-split boundary slices: natural order, halo tiles
    const int64_t slice_bytes = (int64_t)(p.per_t / Sh::F) * (int64_t)site_bytes;
    if (PAR && !clov && !halo) choose_tiles(p, Sh::F, NB, site_bytes);
    // full lattice, T slice beyond L2 reuse: wave-synchronised patched order
    if (!PAR && !clov && !halo && slice_bytes > slice_noreuse() && (8 * NB) <= p.Z)
      choose_full_tiles(p, NB, site_bytes);
    static const int hints = ring_knob("B200WD_L2HINT", 1);  // read once per process
    p.hint_t1 = hints ? (p.tile_x ? 2 : (slice_bytes > slice_noreuse() ? 1 : 0)) : 0;
    p.hint_tm1 = hints;
    const bool whole_lines = (8 * Sh::F * NB) % p.Z == 0;
    if (S <= 0) S = (Sh::SLOT_BYTES >= 40 * 1024) ? (200 * 1024) / Sh::SLOT_BYTES : (100 * 1024) / Sh::SLOT_BYTES;
    if (S < 2) S = 2;
    if (S > 8) S = 8;
    size_t smem = Sh::smem(S);
    while (smem > 227 * 1024 && S > 2) smem = Sh::smem(--S);
    const int64_t ni = n_items_of<NB>(nblk);
    if (clov) {  // staged blocks take ring slots' place in the same shared-memory budget; natural order
      if constexpr (sizeof(R) == 8) {  // complex64: the generic kernel is faster (tuning log)
        const size_t cextra = kClovBufs * (clov_tile<R, NB>() * sizeof(cx<R>) + 16);
        const size_t budget = smem;
        while (Sh::smem(S) + cextra > budget && S > 2) --S;
        smem = Sh::smem(S) + cextra;
        if (smem > 227 * 1024) return false;
        if (halo) {
          if (whole_lines) return launch_ring_kernel<R, V, B, NB, PAR, false, false, true, true>(p, ni, S, smem, st);
          return launch_ring_kernel<R, V, B, NB, PAR, false, true, true, true>(p, ni, S, smem, st);
        }
        if (whole_lines) return launch_ring_kernel<R, V, B, NB, PAR, false, false, true>(p, ni, S, smem, st);
        return launch_ring_kernel<R, V, B, NB, PAR, false, true, true>(p, ni, S, smem, st);
      }
      return false;
    }
    if (halo) {
      if (whole_lines) return launch_ring_kernel<R, V, B, NB, PAR, false, false, false, true>(p, ni, S, smem, st);
      return launch_ring_kernel<R, V, B, NB, PAR, false, true, false, true>(p, ni, S, smem, st);
    }
    if (p.tile_x) {
      setup_waves(p, ni, p.Z / (8 * Sh::F * NB), st);
      if (whole_lines) return launch_ring_kernel<R, V, B, NB, PAR, true, false>(p, ni, S, smem, st);
      return launch_ring_kernel<R, V, B, NB, PAR, true, true>(p, ni, S, smem, st);
    }
    if (whole_lines) return launch_ring_kernel<R, V, B, NB, PAR, false, false>(p, ni, S, smem, st);
    return launch_ring_kernel<R, V, B, NB, PAR, false, true>(p, ni, S, smem, st);
  }
}

// Measured best (NB, S) per (dtype, b) (tools/tune_ring.py on B200); {0,0}
// = defaults (whole z lines per item, ~100/200 KB ring).
template <typename R, int V, int B>
static RingCfg ring_table(int Z) {
  if constexpr (sizeof(R) == 8) {
    switch (B) {
      case 4: return RingCfg{2, 3};
      case 6: return RingCfg{2, 3};
      case 8: return RingCfg{2, 4};
      case 12: return RingCfg{2, 5};  // 16^3x32: 0.556 vs 0.523 at S=4
      case 16: return RingCfg{2, 4};
      case 24: return RingCfg{1, 6};
      case 32: return RingCfg{2, 6};
      default: return RingCfg{};
    }
  } else {
    switch (B) {
      case 4: return RingCfg{4, 3};
      case 6: return RingCfg{4, 2};
      case 8: return RingCfg{2, 4};
      case 12: return Z >= 48 ? RingCfg{4, 3} : RingCfg{2, 2};  // 48^3x96: 0.381 vs 0.351
      case 16: return RingCfg{2, 2};
      case 24: return RingCfg{1, 3};
      case 32: return RingCfg{2, 4};
      default: return RingCfg{};
    }
  }
}

// Launch the ring kernel when its shape preconditions hold (full lattice, no
// halos, Z % 8 == 0); false -> the caller uses the generic kernel.
static bool par_ring_enabled() {
  static int en = -1;
  if (en < 0) {
    const char* e = getenv("B200WD_PAR_RING");
    en = (e && e[0] == '0') ? 0 : 1;
  }
  return en == 1;
}

template <typename R, int V, int B, bool PAR>
static bool try_launch_ring_par(const HopParams& p, int64_t nblk, RingCfg c, cudaStream_t st) {
  constexpr int F = PAR ? 2 : 1;
  const int line = p.Z / (8 * F);  // field blocks per z line
  if (c.nb <= 0) c.nb = line;
  switch (c.nb) {
    case 4:
      if (launch_ring_nb<R, V, B, 4, PAR>(p, nblk, c.s, st)) return true;
      break;
    case 2:
      if (launch_ring_nb<R, V, B, 2, PAR>(p, nblk, c.s, st)) return true;
      break;
    case 1:
      if (launch_ring_nb<R, V, B, 1, PAR>(p, nblk, c.s, st)) return true;
      break;
    default:
      break;
  }
  // partial lines: the z edges use ordinary loads
  if (launch_ring_nb<R, V, B, 2, PAR>(p, nblk, 0, st)) return true;
  return launch_ring_nb<R, V, B, 1, PAR>(p, nblk, 0, st);
}

// Launch the ring kernel when its shape preconditions hold (no halos; full
// lattice: Z % 8 == 0; checkerboard fields: Z % 16 == 0); false -> the caller
// uses the generic kernel.  Clover hops take the ring in complex128 except
// the checkerboard -C x hop with a separate xself (measured slower there);
// B200WD_RING_CLOVER=0 keeps every clover hop generic.
template <typename R, int V, int B>
static bool try_launch_ring(const HopParams& p, cudaStream_t st) {
  static const int ring_clover = ring_knob("B200WD_RING_CLOVER", 1);
  if (p.beta == 0.0) return false;
  // boundary slices consuming halo faces: slice-aligned ranges only
  if (p.lam_halo != nullptr && (p.d_begin % (p.dst_parity >= 0 ? p.per_t / 2 : p.per_t) ||
                                p.d_end % (p.dst_parity >= 0 ? p.per_t / 2 : p.per_t)))
    return false;
  if (p.clov_mode != 0 && (!ring_clover || sizeof(R) != 8 || (p.dst_parity >= 0 && p.clov_mode == 1)))
    return false;
  const bool par = p.dst_parity >= 0;
  if (p.Z % (par ? 16 : 8) != 0) return false;
  if ((p.d_begin & 7) || (p.d_end & 7)) return false;
  const int64_t nblk = (p.d_end - p.d_begin) >> 3;
  const RingCfg env = ring_env();
  RingCfg c = ring_table<R, V, B>(p.Z);
  if (env.nb > 0) c.nb = env.nb;
  if (env.s > 0) c.s = env.s;
  if (par) {
    if (!par_ring_enabled()) return false;
    // measured (tools/sweep_dirac.py --parity 0 on 32^3x64): (NB, S) per nrhs
    RingCfg cp{};
    if constexpr (sizeof(R) == 8) {
      if (B == 4 || B == 8) cp = RingCfg{2, 3};
      // nrhs 12 / 16 keep the default depth: deeper rings are faster for a lone
      // hop without xself (0.573 vs 0.541, 0.546 vs 0.517) but slower for the
      // Schur apply, whose second hop reads xself (4.20 vs 4.03 ms, 5.60 vs 5.32 ms)
    } else {
      if (B == 8) cp = RingCfg{2, 3};
    }
    if (env.nb > 0) cp.nb = env.nb;
    if (env.s > 0) cp.s = env.s;
    return try_launch_ring_par<R, V, B, true>(p, nblk, cp, st);
  }
  return try_launch_ring_par<R, V, B, false>(p, nblk, c, st);
}

// ---- site-local block apply: out = M x (D_oo^-1 eta_o of reduce_rhs) ---------
template <typename R>
__global__ void __launch_bounds__(256) clover_apply_kernel(int64_t n, int b, const cx<R>* __restrict__ M,
                                                           const cx<R>* __restrict__ x, cx<R>* __restrict__ out) {
  using C = cx<R>;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (site, r)
  if (i >= n * b) return;
  const int64_t site = i / b;
  const int r = (int)(i % b);
  const int64_t o = spinor_base(site, 12, b) + r;
  C t[12], y[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) t[k] = __ldg(x + o + k * 8 * b);
  clover_mul(y, t, M + clover_base(site));
#pragma unroll
  for (int k = 0; k < 12; ++k) out[o + k * 8 * b] = y[k];
}

// ---- halo face pack (halo.py:352-368) ---------------------------------------
template <typename R, int V>
__global__ void __launch_bounds__(256) halo_pack_kernel(const HopParams p, void* lam_face, void* chi_face) {
  using C = cx<R>;
  const int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;  // face index
  if (i >= p.nf) return;
  const int r0 = threadIdx.x * V;
  const int b = p.b;
  const bool par = p.dst_parity >= 0;  // parity of the source field
  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  const int kst = 8 * b;
  const int64_t fstride = p.nf * b;
  for (int face = 0; face < 2; ++face) {
    const int tf = face == 0 ? 0 : p.T - 1;
    const int64_t sidx = par ? i + (int64_t)tf * (p.per_t / 2) : i + (int64_t)tf * p.per_t;
    int64_t site = sidx;
    if (par) {
      site = 2 * sidx;
      const int z = (int)(site % p.Z);
      int64_t q = site / p.Z;
      const int y = (int)(q % p.Y);
      q /= p.Y;
      const int x = (int)(q % p.X);
      const int t = (int)(q / p.X);
      site += (t + x + y + z + p.par0 + p.dst_parity) & 1;
    }
    const C* sp = src + spinor_base(sidx, 12, b) + r0;
    C psi[V][12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      C tmp[V];
      VecIO<R, V>::ld(tmp, sp + k * kst);
#pragma unroll
      for (int v = 0; v < V; ++v) psi[v][k] = tmp[v];
    }
    if (face == 0) {
      C* out = static_cast<C*>(lam_face) + i * b + r0;
#pragma unroll
      for (int hk = 0; hk < 6; ++hk) {
        C res[V];
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = cadd(psi[v][hk], psi[v][6 + hk]);  // u + A_0 l
        VecIO<R, V>::st(out + hk * fstride, res);
      }
    } else {
      const C* ux = U + link_base(site, 0, p.n >> 3);
      C u[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) u[e] = __ldg(ux + e * 8);
      C g[V][2][3];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        C h[2][3];
        project_spin<0, false, 0>(h[0], psi[v]);
        project_spin<0, false, 1>(h[1], psi[v]);
        matvec2<true>(g[v], u, h);
      }
      C* out = static_cast<C*>(chi_face) + i * b + r0;
#pragma unroll
      for (int hk = 0; hk < 6; ++hk) {
        C res[V];
#pragma unroll
        for (int v = 0; v < V; ++v) res[v] = g[v][hk / 3][hk % 3];
        VecIO<R, V>::st(out + hk * fstride, res);
      }
    }
  }
}

}  // namespace b200wd
#include "tstream.cuh"
#include "ring2.cuh"
#include "march.cuh"
namespace b200wd {

static bool bulk_enabled() {
  static int en = -1;
  if (en < 0) {
    const char* e = getenv("B200WD_NO_TMA");
    en = (e && e[0] == '1') ? 0 : 1;
  }
  return en == 1;
}

template <typename R, int V, int B>
static void launch_hop_b(const HopParams& p, cudaStream_t st) {
  if constexpr (B >= 4) {
    if (bulk_enabled() && try_launch_march<R, V, B>(p, st)) return;
    if (bulk_enabled() && try_launch_tstream<R, V, B>(p, st)) return;
    if (bulk_enabled() && try_launch_ring2<R, V, B>(p, st)) return;
    if (bulk_enabled() && try_launch_ring<R, V, B>(p, st)) return;
  }
  const int bt = (B > 0 ? B : p.b) / V;
  const int S = bt >= kHopThreads ? 1 : kHopThreads / bt;
  dim3 block(bt, S);
  const int64_t nd = p.d_end - p.d_begin;
  dim3 grid((unsigned)((nd + S - 1) / S));
  hop_kernel<R, V, B><<<grid, block, 0, st>>>(p);
}

// compile-time rhs counts that get their own instantiation per (R, V)
template <typename R, int V> __host__ __device__ constexpr bool wanted_b(int bb) {
  return bb % V == 0 && (V == 2 || sizeof(R) == 8 || bb % 2 == 1);
}

// One entry point per (R, V, B), defined (B200WD_HOP_ENTRY_DEF) and explicitly
// instantiated in the dirac_c*_b*.cu units so the builds run in parallel.
template <typename R, int V, int B> void hop_entry(const HopParams& p, cudaStream_t st);
#ifdef B200WD_HOP_ENTRY_DEF
template <typename R, int V, int B> void hop_entry(const HopParams& p, cudaStream_t st) {
  launch_hop_b<R, V, B>(p, st);
}
#endif

template <typename R, int V>
static void launch_hop(const HopParams& p, cudaStream_t st) {
  switch (p.b) {
#define B200WD_CASE(BB)                       \
  case BB:                                    \
    if constexpr (wanted_b<R, V>(BB)) {       \
      hop_entry<R, V, BB>(p, st);             \
      return;                                 \
    }                                         \
    break;
    B200WD_CASE(1)
    B200WD_CASE(2)
    B200WD_CASE(3)
    B200WD_CASE(4)
    B200WD_CASE(6)
    B200WD_CASE(8)
    B200WD_CASE(12)
    B200WD_CASE(16)
    B200WD_CASE(24)
    B200WD_CASE(32)
#undef B200WD_CASE
    default:
      break;
  }
  hop_entry<R, V, 0>(p, st);
}

template <typename R, int V>
static void launch_pack(const HopParams& p, void* lam, void* chi, cudaStream_t st) {
  const int bt = p.b / V;
  const int S = bt >= 256 ? 1 : 256 / bt;
  dim3 block(bt, S);
  dim3 grid((unsigned)((p.nf + S - 1) / S));
  halo_pack_kernel<R, V><<<grid, block, 0, st>>>(p, lam, chi);
}

// per-dtype launch entry points (dirac_c128.cu / dirac_c64.cu)
void launch_hop_c128(const HopParams& p, cudaStream_t st);
void launch_hop_c64(const HopParams& p, cudaStream_t st);
void launch_pack_c128(const HopParams& p, void* lam, void* chi, cudaStream_t st);
void launch_pack_c64(const HopParams& p, void* lam, void* chi, cudaStream_t st);
void launch_clover_apply_c128(int64_t n, int b, const void* M, const void* x, void* out, cudaStream_t st);
void launch_clover_apply_c64(int64_t n, int b, const void* M, const void* x, void* out, cudaStream_t st);

}  // namespace b200wd
