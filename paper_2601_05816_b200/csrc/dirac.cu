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
#include <cstdlib>

#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"

namespace b200wd {

// Threads per block of the hopping kernel and the occupancy target handed
// to ptxas (c128: <= 168 registers -> 3 blocks = 12 warps per SM; c64: 4 blocks).
constexpr int kHopThreads = 128;
#ifndef B200WD_MINB_C128
#define B200WD_MINB_C128 3
#endif
#ifndef B200WD_MINB_C64
#define B200WD_MINB_C64 4
#endif
template <typename R> struct HopMinBlocks;
template <> struct HopMinBlocks<double> { static constexpr int value = B200WD_MINB_C128; };
template <> struct HopMinBlocks<float> { static constexpr int value = B200WD_MINB_C64; };

// B > 0: rhs count known at compile time (all component / link strides are
// immediates); B == 0: runtime rhs count.
template <typename R, int V, int B>
__global__ void __launch_bounds__(kHopThreads, HopMinBlocks<R>::value) hop_kernel(const HopParams p) {
  using C = cx<R>;
  const int64_t d = p.d_begin + (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (d >= p.d_end) return;
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
    const C* ux = U + link_base(site);
    const int64_t f3 = (z + 1 == Z) ? site - (Z - 1) : site + 1;
    const int64_t f2 = (y + 1 == Y) ? site - (int64_t)(Y - 1) * sY : site + sY;
    const int64_t f1 = (x + 1 == X) ? site - (int64_t)(X - 1) * sX : site + sX;
    const int64_t f0 = (t + 1 == T) ? site - (int64_t)(T - 1) * sT : site + sT;
    if (halo && t + 1 == T) {
      const int64_t fi = par ? (f0 >> 1) : f0;
      const C* hp = static_cast<const C*>(p.lam_halo) + fi * b + r0;
      hop_lam_halo<R, V>(acc, hp, p.nf * b, ux + 0 * 72, 8);
    } else {
      hop_full<0, true, R, V>(acc, sptr(f0), kst, ux + 0 * 72, 8);
    }
    hop_full<1, true, R, V>(acc, sptr(f1), kst, ux + 1 * 72, 8);
    hop_full<2, true, R, V>(acc, sptr(f2), kst, ux + 2 * 72, 8);
    hop_full<3, true, R, V>(acc, sptr(f3), kst, ux + 3 * 72, 8);
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
      hop_full<0, false, R, V>(acc, sptr(b0), kst, U + link_base(b0) + 0 * 72, 8);
    }
    hop_full<1, false, R, V>(acc, sptr(b1), kst, U + link_base(b1) + 1 * 72, 8);
    hop_full<2, false, R, V>(acc, sptr(b2), kst, U + link_base(b2) + 2 * 72, 8);
    hop_full<3, false, R, V>(acc, sptr(b3), kst, U + link_base(b3) + 3 * 72, 8);
  }

  // epilogue: out = scale_r (alpha xself + beta acc)
  const int64_t o = spinor_base(d, 12, b) + r0;
  C* out = static_cast<C*>(p.out) + o;
  const C* xs = p.xself ? static_cast<const C*>(p.xself) + o : nullptr;
  R sc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sc[v] = p.scale ? R(__ldg(p.scale + r0 + v)) : R(1);
  const R beta = R(p.beta), alpha = R(p.alpha);
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
// Warp-specialised, persistent: one producer warp per CTA streams the inputs
// of consecutive work items (NB site blocks of 8 z-consecutive sites x all b
// rhs) into shared memory with cp.async.bulk (TMA 1-D bulk copies),
// completion counted by mbarrier transactions; the consumer warps compute
// from shared memory and hand each slot back through an "empty" mbarrier.
// For the t, x and y hops the 8 neighbours of a site block are exactly one
// other site block (Z % 8 == 0), i.e. one contiguous 96*b-complex run, so a
// hop tile is NB bulk copies of spinor blocks + NB copies of one 72-complex
// link plane (U_mu of the own block for forward hops, of the neighbour block
// for backward hops).  Each item streams 6 hop tiles through an S-slot ring,
// then its own block ("z tile": z hops + the xself of the epilogue) through
// a dedicated buffer.  Loads in flight live in shared memory, not registers,
// so the bytes in flight per SM (Little's law) are set by the ring depth.
template <typename R, int V, int B> struct RingShape {
  static constexpr int BT = B / V;                                   // threads per site
  static constexpr int NB = (BT * 8 >= 96) ? 1 : (128 / (BT * 8));   // site blocks per item
  static constexpr int NC = BT * 8 * NB;                             // consumer threads
  static constexpr int NCW = NC / 32;                                // consumer warps
  static constexpr int NT = NC + 32;                                 // + producer warp
  static constexpr int SPIN = NB * 96 * B;                           // complex per spinor tile
  static constexpr int SLOT = SPIN + NB * 72;                        // + one link plane per block
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
#ifndef B200WD_RING_BYTES
#define B200WD_RING_BYTES (104 * 1024)
#endif
  static constexpr int S0 = B200WD_RING_BYTES / SLOT_BYTES;
  static constexpr int S = S0 < 2 ? 2 : (S0 > 7 ? 7 : S0);          // ring depth (<= 7 tiles per item)
  static constexpr int EDGE = 2 * NB * 12 * B;  // z-edge sites of the own blocks (one buffer: see producer)
  static constexpr size_t SMEM = (size_t)SLOT_BYTES * S + EDGE * sizeof(cx<R>) + 8 * 2 * S;
};

// Coordinates of the first site of a site block (32-bit arithmetic: a rank's
// local lattice has < 2^31 sites).
struct BlkCoord {
  int t, x, y, z0;
};
__device__ __forceinline__ BlkCoord block_coord(int64_t g, const HopParams& p) {
  uint32_t s0 = (uint32_t)(g * 8);
  BlkCoord c;
  c.z0 = (int)(s0 % (uint32_t)p.Z);
  s0 /= (uint32_t)p.Z;
  c.y = (int)(s0 % (uint32_t)p.Y);
  s0 /= (uint32_t)p.Y;
  c.x = (int)(s0 % (uint32_t)p.X);
  c.t = (int)(s0 / (uint32_t)p.X);
  return c;
}
// step to the next site block (z0 += 8 with carries)
__device__ __forceinline__ void block_step(BlkCoord& c, const HopParams& p) {
  c.z0 += 8;
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

template <int MU, bool FWD>
__device__ __forceinline__ int64_t block_neighbor(int64_t g, const BlkCoord& c, const HopParams& p) {
  const int64_t s0 = g * 8;
  const int64_t sY = p.Z, sX = (int64_t)p.Y * p.Z, sT = p.per_t;
  int64_t ns;
  if constexpr (MU == 0) ns = FWD ? (c.t + 1 == p.T ? s0 - (int64_t)(p.T - 1) * sT : s0 + sT)
                                  : (c.t == 0 ? s0 + (int64_t)(p.T - 1) * sT : s0 - sT);
  else if constexpr (MU == 1) ns = FWD ? (c.x + 1 == p.X ? s0 - (int64_t)(p.X - 1) * sX : s0 + sX)
                                       : (c.x == 0 ? s0 + (int64_t)(p.X - 1) * sX : s0 - sX);
  else ns = FWD ? (c.y + 1 == p.Y ? s0 - (int64_t)(p.Y - 1) * sY : s0 + sY)
                : (c.y == 0 ? s0 + (int64_t)(p.Y - 1) * sY : s0 - sY);
  return ns >> 3;
}

// z neighbour (step +1 / -1 along z) of site d of a line with extent Z
__device__ __forceinline__ int64_t z_neighbor(int64_t d, int z, int Z, int step) {
  if (step > 0) return (z + 1 == Z) ? d - (Z - 1) : d + 1;
  return (z == 0) ? d + (Z - 1) : d - 1;
}

// tile H in 0..5: hop (mu = H/2, forward if H even); H == 6: own block (z tile)
// plus the z-edge sites outside the item (into `edge`)
template <typename R, int V, int B, int H>
__device__ __forceinline__ void ring_issue(const HopParams& p, int64_t gb0, BlkCoord c, cx<R>* slot,
                                           uint64_t* full, cx<R>* edge) {
  using C = cx<R>;
  using Sh = RingShape<R, V, B>;
  const C* src = static_cast<const C*>(p.src);
  const C* U = static_cast<const C*>(p.U);
  uint32_t bytes = (uint32_t)(Sh::SLOT * sizeof(C));
  if constexpr (H == 6) {
    // z-edge sites: site lo=0's z-1 and lo=7's z+1 neighbour of every block,
    // when they fall outside the item's blocks (12 runs of B complex each)
    BlkCoord ce = c;
    uint32_t extra = 0;
#pragma unroll 1
    for (int jj = 0; jj < Sh::NB; ++jj) {
      const int64_t g = gb0 + jj;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int64_t dd = g * 8 + (side ? 7 : 0);
        const int64_t nd = z_neighbor(dd, ce.z0 + (side ? 7 : 0), p.Z, side ? 1 : -1);
        const int64_t jb = (nd >> 3) - gb0;
        if (jb < 0 || jb >= Sh::NB) extra += 12 * B * sizeof(C);
      }
      if (jj + 1 < Sh::NB) block_step(ce, p);
    }
    bytes += extra;
  }
  mbar_expect_tx(full, bytes);
  if constexpr (H == 6) {
    BlkCoord ce = c;
#pragma unroll 1
    for (int jj = 0; jj < Sh::NB; ++jj) {
      const int64_t g = gb0 + jj;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        const int64_t dd = g * 8 + (side ? 7 : 0);
        const int64_t nd = z_neighbor(dd, ce.z0 + (side ? 7 : 0), p.Z, side ? 1 : -1);
        const int64_t jb = (nd >> 3) - gb0;
        if (jb < 0 || jb >= Sh::NB) {
          const C* es = src + spinor_base(nd, 12, B);
          C* ed = edge + (jj * 2 + side) * 12 * B;
#pragma unroll 1
          for (int k = 0; k < 12; ++k) bulk_g2s(ed + k * B, es + k * 8 * B, B * sizeof(C), full);
        }
      }
      if (jj + 1 < Sh::NB) block_step(ce, p);
    }
  }
#pragma unroll
  for (int jj = 0; jj < Sh::NB; ++jj) {
    const int64_t g = gb0 + jj;
    int64_t nb = g, lb = g;
    int mu = 3;
    if constexpr (H < 6) {
      constexpr int MU = H >> 1;
      constexpr bool FWD = !(H & 1);
      mu = MU;
      nb = block_neighbor<MU, FWD>(g, c, p);
      lb = FWD ? g : nb;
    }
    bulk_g2s(slot + jj * 96 * B, src + nb * 96 * B, 96 * B * sizeof(C), full);
    bulk_g2s(slot + Sh::SPIN + jj * 72, U + lb * 288 + mu * 72, 72 * sizeof(C), full);
    if (jj + 1 < Sh::NB) block_step(c, p);
  }
}

template <typename R, int V, int B>
__global__ void __launch_bounds__(RingShape<R, V, B>::NT) hop_ring_kernel(const HopParams p, int64_t n_items) {
  using C = cx<R>;
  using Sh = RingShape<R, V, B>;
  constexpr int S = Sh::S;
  constexpr int KST = 8 * B;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  C* ring = reinterpret_cast<C*>(smem_raw);
  C* edge = ring + S * Sh::SLOT;  // single buffer: item i's z tile is issued only after
                                  // item i-1's z tile was consumed (S <= 7 tiles per item)
  uint64_t* full = reinterpret_cast<uint64_t*>(edge + Sh::EDGE);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x;  // 1-D block: consumers [0, NC), producer warp [NC, NC+32)
  const bool producer = tid >= Sh::NC;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Sh::NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (producer) {
    if (tid == Sh::NC) {  // one elected lane issues every copy
      int seq = 0;
      const C* srcp = static_cast<const C*>(p.src);
      const C* Up = static_cast<const C*>(p.U);
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int64_t gb0 = (p.d_begin >> 3) + it * Sh::NB;
        const BlkCoord c0 = block_coord(gb0, p);
        // warm L2 with the compulsory misses of the next item of this CTA: its
        // t+1 neighbour blocks and its own link blocks (first touch in sweep order)
        const int64_t nx = it + gridDim.x;
        if (nx < n_items) {
          const int64_t gn = (p.d_begin >> 3) + nx * Sh::NB;
          BlkCoord cn = block_coord(gn, p);
#pragma unroll 1
          for (int jj = 0; jj < Sh::NB; ++jj) {
            const int64_t nb = block_neighbor<0, true>(gn + jj, cn, p);
            bulk_prefetch_l2(srcp + nb * 96 * B, 96 * B * sizeof(C));
            if (jj + 1 < Sh::NB) block_step(cn, p);
          }
          bulk_prefetch_l2(Up + gn * 288, Sh::NB * 288 * sizeof(C));
        }
#define B200WD_PRODUCE(H)                                                                 \
  {                                                                                       \
    const int slot = seq % S, use = seq / S;                                              \
    if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);                                  \
    ring_issue<R, V, B, H>(p, gb0, c0, ring + slot * Sh::SLOT, &full[slot], edge);        \
    ++seq;                                                                                \
  }
        B200WD_PRODUCE(6)
        B200WD_PRODUCE(0)
        B200WD_PRODUCE(1)
        B200WD_PRODUCE(2)
        B200WD_PRODUCE(3)
        B200WD_PRODUCE(4)
        B200WD_PRODUCE(5)
#undef B200WD_PRODUCE
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
  const int Z = p.Z;
  R sc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sc[v] = p.scale ? R(__ldg(p.scale + r0 + v)) : R(1);
  const R beta = R(p.beta), alpha = R(p.alpha);
  const bool self_is_src = p.xself == p.src;

  // acc accumulates (alpha/beta) xself + 2H src, so out = (sc beta) acc: the own
  // block (z tile) is consumed first and its slot recycled immediately
  const R ab = (p.xself != nullptr && p.beta != 0.0) ? R(p.alpha / p.beta) : R(0);
  R scb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) scb[v] = sc[v] * beta;
  int seq = 0;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gb0 = (p.d_begin >> 3) + it * Sh::NB;
    const int64_t d = (gb0 + j) * 8 + lo;
    C acc[V][12];
    {
      const int slot = seq % S;
      mbar_wait(&full[slot], (seq / S) & 1);
      const C* zt = ring + slot * Sh::SLOT;
      // init from xself
      if (self_is_src) {
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C xv[V];
          VecIO<R, V>::lds(xv, zt + j * 96 * B + lo * B + r0 + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][k] = mk(ab * xv[v].x, ab * xv[v].y);
        }
      } else if (p.xself) {
        const C* xs = static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C xv[V];
          VecIO<R, V>::ld(xv, xs + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][k] = mk(ab * xv[v].x, ab * xv[v].y);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
      }
      // z hops from the own blocks; z-edge sites from the edge buffer
      const int z = (int)((uint32_t)d % (uint32_t)Z);
      {
        const int64_t nd = z_neighbor(d, z, Z, 1);
        const int64_t jb = (nd >> 3) - gb0;
        const bool in = jb >= 0 && jb < Sh::NB;
        const C* sp = in ? zt + jb * 96 * B + (nd & 7) * B + r0 : edge + (j * 2 + 1) * 12 * B + r0;
        const int kst = in ? KST : B;
        hop_full<3, true, R, V, true, true>(acc, sp, kst, zt + Sh::SPIN + j * 72 + lo, 8);
      }
      {
        const int64_t nd = z_neighbor(d, z, Z, -1);
        const int64_t jb = (nd >> 3) - gb0;
        const bool in = jb >= 0 && jb < Sh::NB;
        const C* sp = in ? zt + jb * 96 * B + (nd & 7) * B + r0 : edge + (j * 2 + 0) * 12 * B + r0;
        const int kst = in ? KST : B;
        // U_3(x - z): own link plane, or global for an edge site (generic load)
        const C* ul = in ? zt + Sh::SPIN + jb * 72 + (nd & 7) : U + link_base(nd) + 3 * 72;
        hop_full<3, false, R, V, true, false, true>(acc, sp, kst, ul, 8);
      }
      __syncwarp();
      if (lead) mbar_arrive(&empty[slot]);
      ++seq;
    }

#define B200WD_CONSUME(H)                                                                            \
  {                                                                                                  \
    const int slot = seq % S;                                                                        \
    mbar_wait(&full[slot], (seq / S) & 1);                                                           \
    const C* sb = ring + slot * Sh::SLOT;                                                            \
    hop_full<((H) >> 1), !((H)&1), R, V, true, true>(acc, sb + j * 96 * B + lo * B + r0, KST,        \
                                                      sb + Sh::SPIN + j * 72 + lo, 8);               \
    __syncwarp();                                                                                    \
    if (lead) mbar_arrive(&empty[slot]);                                                             \
    ++seq;                                                                                           \
  }
    B200WD_CONSUME(0)
    B200WD_CONSUME(1)
    B200WD_CONSUME(2)
    B200WD_CONSUME(3)
    B200WD_CONSUME(4)
    B200WD_CONSUME(5)
#undef B200WD_CONSUME

    // epilogue: out = sc beta acc = sc (alpha xself + beta 2H src / 2)
    C* out = static_cast<C*>(p.out) + spinor_base(d, 12, B) + r0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      C res[V];
#pragma unroll
      for (int v = 0; v < V; ++v) res[v] = mk(scb[v] * acc[v][k].x, scb[v] * acc[v][k].y);
      VecIO<R, V>::st(out + k * KST, res);
    }
  }
}

static int g_sm_count = 0;

// Launch the ring kernel when its shape preconditions hold; false -> the
// caller uses the generic kernel.
template <typename R, int V, int B>
static bool try_launch_ring(const HopParams& p, cudaStream_t st) {
  using Sh = RingShape<R, V, B>;
  if (Sh::NC % 32 != 0 || p.beta == 0.0) return false;
  if (p.dst_parity >= 0 || p.lam_halo != nullptr || p.Z % 8 != 0) return false;
  if ((p.d_begin & 7) || (p.d_end & 7)) return false;
  const int64_t nblk = (p.d_end - p.d_begin) >> 3;
  if (nblk % Sh::NB) return false;
  static int ctas_per_sm = -1;
  if (ctas_per_sm < 0) {
    if (cudaFuncSetAttribute(hop_ring_kernel<R, V, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Sh::SMEM) != cudaSuccess) {
      ctas_per_sm = 0;
      return false;
    }
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, hop_ring_kernel<R, V, B>, Sh::NT, Sh::SMEM) != cudaSuccess)
      nb = 0;
    ctas_per_sm = nb;
    if (g_sm_count == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
  }
  if (ctas_per_sm <= 0) return false;
  const int64_t n_items = nblk / Sh::NB;
  int64_t grid = (int64_t)ctas_per_sm * g_sm_count;
  if (grid > n_items) grid = n_items;
  hop_ring_kernel<R, V, B><<<(unsigned)grid, Sh::NT, Sh::SMEM, st>>>(p, n_items);
  return true;
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
      const C* ux = U + link_base(site);
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

template <typename R, int V>
static void launch_hop(const HopParams& p, cudaStream_t st) {
  switch (p.b) {
#define B200WD_CASE(BB)                       \
  case BB:                                    \
    if constexpr (wanted_b<R, V>(BB)) {       \
      launch_hop_b<R, V, BB>(p, st);          \
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
  launch_hop_b<R, V, 0>(p, st);
}

template <typename R, int V>
static void launch_pack(const HopParams& p, void* lam, void* chi, cudaStream_t st) {
  const int bt = p.b / V;
  const int S = bt >= 256 ? 1 : 256 / bt;
  dim3 block(bt, S);
  dim3 grid((unsigned)((p.nf + S - 1) / S));
  halo_pack_kernel<R, V><<<grid, block, 0, st>>>(p, lam, chi);
}

static int fill_params(HopParams& p, const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t parity) {
  B200WD_REQUIRE(lat != nullptr, "lattice descriptor is NULL");
  for (int d = 0; d < 4; ++d)
    B200WD_REQUIRE(lat->dims[d] >= 2 && lat->dims[d] % 2 == 0,
                   "extent %d in direction %d is not an even number >= 2", lat->dims[d], d);
  B200WD_REQUIRE(dtype == B200WD_C128 || dtype == B200WD_C64, "unknown dtype %d", dtype);
  B200WD_REQUIRE(b >= 1 && b <= 128, "rhs count b=%d out of range [1,128]", b);
  B200WD_REQUIRE(parity >= -1 && parity <= 1, "parity must be -1, 0 or 1 (got %d)", parity);
  B200WD_REQUIRE((lat->t_origin & 1) == 0, "t_origin must be even (got %d)", lat->t_origin);
  p = HopParams{};
  p.T = lat->dims[0];
  p.X = lat->dims[1];
  p.Y = lat->dims[2];
  p.Z = lat->dims[3];
  p.par0 = lat->t_origin & 1;
  p.b = b;
  p.dst_parity = parity;
  p.per_t = (int64_t)p.X * p.Y * p.Z;
  p.n = p.per_t * p.T;
  p.n_src = parity < 0 ? p.n : p.n / 2;
  p.n_dst = p.n_src;
  p.nf = parity < 0 ? p.per_t : p.per_t / 2;
  return B200WD_OK;
}

}  // namespace b200wd

using namespace b200wd;

extern "C" int b200wd_hop(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
                          const void* links, const void* src, const void* xself, void* out, double alpha,
                          double beta, const double* scale, int32_t t_begin, int32_t t_end,
                          const void* lam_halo, const void* chi_halo, void* stream) {
  HopParams p;
  if (int rc = fill_params(p, lat, dtype, b, dst_parity)) return rc;
  B200WD_REQUIRE(links && src && out, "NULL field pointer");
  B200WD_REQUIRE(0 <= t_begin && t_begin <= t_end && t_end <= p.T, "slice range [%d,%d) outside [0,%d)", t_begin,
                 t_end, p.T);
  B200WD_REQUIRE((lam_halo == nullptr) == (chi_halo == nullptr), "lam_halo and chi_halo must both be set or NULL");
  if (t_begin == t_end) return B200WD_OK;
  p.U = links;
  p.src = src;
  p.xself = xself;
  p.out = out;
  p.alpha = alpha;
  p.beta = 0.5 * beta;  // the kernel accumulates 2 H (projectors without the 1/2)
  p.scale = scale;
  p.lam_halo = lam_halo;
  p.chi_halo = chi_halo;
  const int64_t per = dst_parity < 0 ? p.per_t : p.per_t / 2;
  p.d_begin = per * t_begin;
  p.d_end = per * t_end;
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) {
    launch_hop<double, 1>(p, st);
  } else if (b % 2 == 0) {
    launch_hop<float, 2>(p, st);
  } else {
    launch_hop<float, 1>(p, st);
  }
  return check_launch("b200wd_hop");
}

extern "C" int b200wd_dirac_apply(const b200wd_lattice* lat, int32_t dtype, int32_t b, double m0,
                                  const void* links, const void* psi, void* eta, void* stream) {
  B200WD_REQUIRE(lat != nullptr, "lattice descriptor is NULL");
  return b200wd_hop(lat, dtype, b, -1, links, psi, psi, eta, 4.0 + m0, -1.0, nullptr, 0, lat->dims[0], nullptr,
                    nullptr, stream);
}

extern "C" int b200wd_halo_pack(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t src_parity,
                                const void* links, const void* src, void* lam_face, void* chi_face,
                                void* stream) {
  HopParams p;
  if (int rc = fill_params(p, lat, dtype, b, src_parity)) return rc;
  B200WD_REQUIRE(links && src && lam_face && chi_face, "NULL pointer");
  p.U = links;
  p.src = src;
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) launch_pack<double, 1>(p, lam_face, chi_face, st);
  else if (b % 2 == 0) launch_pack<float, 2>(p, lam_face, chi_face, st);
  else launch_pack<float, 1>(p, lam_face, chi_face, st);
  return check_launch("b200wd_halo_pack");
}
