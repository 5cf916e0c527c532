// Two-line TMA ring kernel (full-lattice fields, whole z lines), sm_100a.
//
// Same producer / consumer ring as hop_ring_kernel (dirac_kernels.cuh), but a
// work item is TWO y-adjacent z lines (y even) instead of one.  The y hop
// between the two lines reads the item's own tile, so an item streams 12 line
// tiles for 2 lines (own x2, t+-, x+- x2 each, one outer line in y+ and in y-)
// instead of 14: 14% fewer L2->SM bytes per site.  ncu shows the c64 ring
// bound by tile delivery (consumers stalled on the full barriers), which is
// what this targets; the item keeps the natural site order, so CTAs stay in
// lockstep and the t/x neighbour tiles keep hitting L2.
//
// Tiles (H): 6 own lines (spinor, U_3 of both lines, U_2 of both lines),
// 0/1 t+-, 2/3 x+- (two lines each, U_mu of the own or the neighbour lines),
// 4 y+ (line y+2, U_2 of line y+1), 5 y- (line y-1 and its U_2).
#pragma once

#include "capi.cuh"
#include "common.cuh"
#include "layout.cuh"
#include "stencil.cuh"

namespace b200wd {

template <typename R, int V, int B, int NB> struct Ring2Shape {
  static constexpr int LY = 2;
  static constexpr int BT = B / V;
  static constexpr int NC = BT * 8 * NB * LY;
  static constexpr int NCW = NC / 32;
  static constexpr int NT = NC + 32;
  static constexpr int LSP = NB * 96 * B;  // spinor complex per line segment
  static constexpr int LLK = NB * 72;      // link complex per line, one direction
  static constexpr int SPIN = LY * LSP;
  static constexpr int SLOT = SPIN + 2 * LY * LLK;  // own tile: U_3 and U_2 of both lines
  static constexpr int SLOT_BYTES = SLOT * (int)sizeof(cx<R>);
  static constexpr bool valid = (B % V == 0) && (NC % 32 == 0) && NC >= 64 && NC <= 256 &&
                                (size_t)SLOT_BYTES * 2 <= 220 * 1024;
  static size_t smem(int S) { return (size_t)SLOT_BYTES * S + 16 * S; }
};

template <typename R, int V, int B, int NB, int H>
__device__ __forceinline__ void ring2_issue(const HopParams& p, int64_t gb0, const BlkCoord& c0, cx<R>* slot,
                                            uint64_t* full) {
  using C = cx<R>;
  using Sh = Ring2Shape<R, V, B, NB>;
  const C* src = static_cast<const C*>(p.src);
  const C* U = static_cast<const C*>(p.U);
  const int64_t nblk = p.n >> 3;
  if constexpr (H == 6) {
    mbar_expect_tx(full, (uint32_t)(Sh::SLOT * sizeof(C)));
    bulk_g2s(slot, src + gb0 * 96 * B, Sh::SPIN * sizeof(C), full);
    bulk_g2s(slot + Sh::SPIN, U + (3 * nblk + gb0) * 72, 2 * Sh::LLK * sizeof(C), full);
    bulk_g2s(slot + Sh::SPIN + 2 * Sh::LLK, U + (2 * nblk + gb0) * 72, 2 * Sh::LLK * sizeof(C), full);
  } else if constexpr (H < 4) {
    constexpr int MU = H >> 1;
    constexpr bool FWD = !(H & 1);
    // t / x shifts keep the two lines adjacent: one copy each
    const int64_t nb0 = block_neighbor<MU, FWD>(gb0 * 8, c0, p) >> 3;
    mbar_expect_tx(full, (uint32_t)((Sh::SPIN + 2 * Sh::LLK) * sizeof(C)));
    bulk_g2s(slot, src + nb0 * 96 * B, Sh::SPIN * sizeof(C), full);
    bulk_g2s(slot + Sh::SPIN, U + (MU * nblk + (FWD ? gb0 : nb0)) * 72, 2 * Sh::LLK * sizeof(C), full);
  } else {
    constexpr bool FWD = H == 4;
    int64_t nb;
    if constexpr (FWD) {  // line y+2: the +y neighbour of the item's second line
      BlkCoord c1 = c0;
      c1.y += 1;
      nb = block_neighbor<2, true>((gb0 + NB) * 8, c1, p) >> 3;
    } else {
      nb = block_neighbor<2, false>(gb0 * 8, c0, p) >> 3;
    }
    mbar_expect_tx(full, (uint32_t)((Sh::LSP + Sh::LLK) * sizeof(C)));
    bulk_g2s(slot, src + nb * 96 * B, Sh::LSP * sizeof(C), full);
    bulk_g2s(slot + Sh::SPIN, U + (2 * nblk + (FWD ? gb0 + NB : nb)) * 72, Sh::LLK * sizeof(C), full);
  }
}

template <typename R, int V, int B, int NB>
__global__ void __launch_bounds__(Ring2Shape<R, V, B, NB>::NT) hop_ring2_kernel(const HopParams p, int64_t n_items,
                                                                                int S) {
  using C = cx<R>;
  using Sh = Ring2Shape<R, V, B, NB>;
  constexpr int KST = 8 * B;
  constexpr int SEG = 8 * NB;  // sites per line
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

  if (tid >= Sh::NC) {
    if (tid == Sh::NC) {
      int pslot = 0, pfirst = 1;
      uint32_t pphase = 0;
      for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int64_t gb0 = (p.d_begin >> 3) + it * (2 * NB);
        const BlkCoord c0 = block_coord(gb0 * 8, p);
#define B200WD_PRODUCE2(H)                                                              \
  {                                                                                     \
    if (pfirst == 0) mbar_wait(&empty[pslot], pphase ^ 1u);                             \
    ring2_issue<R, V, B, NB, H>(p, gb0, c0, ring + pslot * Sh::SLOT, &full[pslot]);     \
    if (++pslot == S) {                                                                 \
      pslot = 0;                                                                        \
      pphase ^= 1u;                                                                     \
      pfirst = 0;                                                                       \
    }                                                                                   \
  }
        B200WD_PRODUCE2(6)
        B200WD_PRODUCE2(0)
        B200WD_PRODUCE2(1)
        B200WD_PRODUCE2(2)
        B200WD_PRODUCE2(3)
        B200WD_PRODUCE2(4)
        B200WD_PRODUCE2(5)
#undef B200WD_PRODUCE2
      }
    }
    return;
  }

  // ---- consumers ----
  const int r0 = (tid % Sh::BT) * V;
  const int ys = tid / Sh::BT;
  const int l = ys / SEG;              // line of the item (0: y, 1: y+1)
  const int zs = ys % SEG;             // z in the line
  const int j = zs >> 3, lo = zs & 7;  // block in the line, site in the block
  const int jj = l * NB + j;           // block in the two-line tile
  const int so2 = (jj * 96 + lo) * B + r0;  // own spinor (k = 0) in a two-line tile
  const int so1 = (j * 96 + lo) * B + r0;   // in a one-line tile
  const int lo2 = jj * 72 + lo;             // own link (e = 0) in a two-line region
  const int lo1 = j * 72 + lo;              // in a one-line region
  const bool lead = (tid & 31) == 0;
  R scb[V];
#pragma unroll
  for (int v = 0; v < V; ++v) scb[v] = (p.scale ? R(__ldg(p.scale + r0 + v)) : R(1)) * R(p.beta);
  const R ab = (p.xself != nullptr) ? R(p.alpha / p.beta) : R(0);
  const bool self_is_src = p.xself == p.src;
  const int zp = zs + 1 == SEG ? 0 : zs + 1, zm = zs == 0 ? SEG - 1 : zs - 1;
  const int so_zp = ((l * NB + (zp >> 3)) * 96 + (zp & 7)) * B + r0;
  const int so_zm = ((l * NB + (zm >> 3)) * 96 + (zm & 7)) * B + r0;
  const int lo_zm = (l * NB + (zm >> 3)) * 72 + (zm & 7);

  int cslot = 0;
  uint32_t cphase = 0;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int64_t gb0 = (p.d_begin >> 3) + it * (2 * NB);
    const int64_t d = (gb0 + jj) * 8 + lo;
    C acc[V][12];
    {  // own lines: self, z hops, the y hop between the two lines
      mbar_wait(&full[cslot], cphase);
      const C* zt = ring + cslot * Sh::SLOT;
      if (self_is_src || p.xself) {
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          C xv[V];
          if (self_is_src) VecIO<R, V>::lds(xv, zt + so2 + k * KST);
          else VecIO<R, V>::ld(xv, static_cast<const C*>(p.xself) + spinor_base(d, 12, B) + r0 + k * KST);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][k] = mk(ab * xv[v].x, ab * xv[v].y);
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));
      }
      const C* u3 = zt + Sh::SPIN;
      const C* u2 = zt + Sh::SPIN + 2 * Sh::LLK;
      hop_full<3, true, R, V, true, true>(acc, zt + so_zp, KST, u3 + lo2, 8);
      hop_full<3, false, R, V, true, true>(acc, zt + so_zm, KST, u3 + lo_zm, 8);
      if (l == 0) hop_full<2, true, R, V, true, true>(acc, zt + so2 + Sh::LSP, KST, u2 + lo2, 8);
      else hop_full<2, false, R, V, true, true>(acc, zt + so2 - Sh::LSP, KST, u2 + lo2 - Sh::LLK, 8);
      __syncwarp();
      if (lead) mbar_arrive(&empty[cslot]);
      if (++cslot == S) {
        cslot = 0;
        cphase ^= 1u;
      }
    }
#define B200WD_CONSUME2(H, COND, SO, LO)                                                       \
  {                                                                                            \
    mbar_wait(&full[cslot], cphase);                                                           \
    const C* sb = ring + cslot * Sh::SLOT;                                                     \
    if (COND) hop_full<((H) >> 1), !((H)&1), R, V, true, true>(acc, sb + (SO), KST, sb + Sh::SPIN + (LO), 8); \
    __syncwarp();                                                                              \
    if (lead) mbar_arrive(&empty[cslot]);                                                      \
    if (++cslot == S) {                                                                        \
      cslot = 0;                                                                               \
      cphase ^= 1u;                                                                            \
    }                                                                                          \
  }
    B200WD_CONSUME2(0, true, so2, lo2)
    B200WD_CONSUME2(1, true, so2, lo2)
    B200WD_CONSUME2(2, true, so2, lo2)
    B200WD_CONSUME2(3, true, so2, lo2)
    B200WD_CONSUME2(4, l == 1, so1, lo1)
    B200WD_CONSUME2(5, l == 0, so1, lo1)
#undef B200WD_CONSUME2
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

// (S) per (dtype, nrhs) where the two-line ring is the default; 0 = off.
// B200WD_RING2_S overrides (0 disables, 1 enables with the default depth,
// > 1 forces that ring depth).
// Measured on 16^3x32 (profiles/r1_tstream_tuning.txt, ring2 section): c64
// nrhs 4 0.0434 vs 0.0460 ms (ring), nrhs 8 0.0701 vs 0.0727 ms (stream);
// c128 nrhs 4/8 and c64 nrhs 12/16/24 were slower or equal.
template <typename R, int V, int B>
static int ring2_table() {
  if constexpr (sizeof(R) == 4) {
    if (B == 4) return 3;
    if (B == 6) return 3;  // 0.0620 vs 0.0682 ms (ring)
    if (B == 8) return 2;
  }
  return 0;
}

template <typename R, int V, int B, int NB>
static bool launch_ring2_nb(const HopParams& p, int S, cudaStream_t st) {
  using Sh = Ring2Shape<R, V, B, NB>;
  if constexpr (!Sh::valid) {
    return false;
  } else {
    if (p.Z != 8 * NB) return false;
    const int64_t nblk = (p.d_end - p.d_begin) >> 3;
    if (nblk % (2 * NB)) return false;
    if (S <= 0) S = (Sh::SLOT_BYTES >= 40 * 1024) ? (200 * 1024) / Sh::SLOT_BYTES : (100 * 1024) / Sh::SLOT_BYTES;
    if (S < 2) S = 2;
    if (S > 8) S = 8;
    size_t smem = Sh::smem(S);
    while (smem > 227 * 1024 && S > 2) smem = Sh::smem(--S);
    LaunchFacts f;
    if (!launch_facts((const void*)hop_ring2_kernel<R, V, B, NB>, Sh::NT, smem, f)) return false;
    const int64_t n_items = nblk / (2 * NB);
    int64_t grid = (int64_t)f.occ * persistent_sms(f.sm_count);
    if (grid > n_items) grid = n_items;
    hop_ring2_kernel<R, V, B, NB><<<(unsigned)grid, Sh::NT, smem, st>>>(p, n_items, S);
    return true;
  }
}

// Full-lattice fields, whole z lines of 8, 16 or 32 sites, no halos, no clover,
// slice-aligned range.
template <typename R, int V, int B>
static bool try_launch_ring2(const HopParams& p, cudaStream_t st) {
  static const int env = ring_knob("B200WD_RING2_S", -1);
  const int S = env >= 0 ? env : ring2_table<R, V, B>();
  if (S == 0) return false;
  if (p.dst_parity >= 0 || p.lam_halo != nullptr || p.beta == 0.0 || p.clov_mode != 0) return false;
  if (p.d_begin % p.per_t || p.d_end % p.per_t) return false;
  const int s = S > 1 ? S : 0;  // 1: default ring depth
  switch (p.Z) {
    case 8: return launch_ring2_nb<R, V, B, 1>(p, s, st);
    case 16: return launch_ring2_nb<R, V, B, 2>(p, s, st);
    case 32: return launch_ring2_nb<R, V, B, 4>(p, s, st);
    default: return false;
  }
}

}  // namespace b200wd
