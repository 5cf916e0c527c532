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
#include "capi.cuh"
#include "common.cuh"

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
};

// ---- V-wide loads/stores of consecutive rhs ---------------------------------
template <typename R, int V> struct VecIO;
template <> struct VecIO<double, 1> {
  static __device__ __forceinline__ void ld(double2 (&o)[1], const double2* p) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void st(double2* p, const double2 (&v)[1]) { __stcs(p, v[0]); }
};
template <> struct VecIO<float, 1> {
  static __device__ __forceinline__ void ld(float2 (&o)[1], const float2* p) { o[0] = __ldg(p); }
  static __device__ __forceinline__ void st(float2* p, const float2 (&v)[1]) { __stcs(p, v[0]); }
};
template <> struct VecIO<float, 2> {
  static __device__ __forceinline__ void ld(float2 (&o)[2], const float2* p) {
    float4 q = __ldg(reinterpret_cast<const float4*>(p));
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

// One hop from a full neighbour spinor (12 components loaded from src).
template <int MU, bool FWD, typename R, int V>
__device__ __forceinline__ void hop_full(cx<R> (&acc)[V][12], const cx<R>* __restrict__ sp, int64_t kstride,
                                         const cx<R>* __restrict__ up, int64_t estride) {
  using C = cx<R>;
  C psi[V][12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    C tmp[V];
    VecIO<R, V>::ld(tmp, sp + k * kstride);
#pragma unroll
    for (int v = 0; v < V; ++v) psi[v][k] = tmp[v];
  }
  C u[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) u[e] = __ldg(up + e * estride);
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

// Forward T hop whose projected half spinor comes from the lam halo face.
template <typename R, int V>
__device__ __forceinline__ void hop_lam_halo(cx<R> (&acc)[V][12], const cx<R>* __restrict__ hp, int64_t hstride,
                                             const cx<R>* __restrict__ up, int64_t estride) {
  using C = cx<R>;
  C hh[V][6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    C tmp[V];
    VecIO<R, V>::ld(tmp, hp + k * hstride);
#pragma unroll
    for (int v = 0; v < V; ++v) hh[v][k] = tmp[v];
  }
  C u[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) u[e] = __ldg(up + e * estride);
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
template <typename R, int V>
__device__ __forceinline__ void hop_chi_halo(cx<R> (&acc)[V][12], const cx<R>* __restrict__ hp, int64_t hstride) {
  using C = cx<R>;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    C tmp[V];
    VecIO<R, V>::ld(tmp, hp + k * hstride);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      // sign +1 reconstruction with A_0 = I: upper += g, lower -= g
      acc[v][k] = cadd(acc[v][k], tmp[v]);
      acc[v][6 + k] = csub(acc[v][6 + k], tmp[v]);
    }
  }
}

template <typename R, int V, bool PAR, bool HALO>
__global__ void __launch_bounds__(256) hop_kernel(const HopParams p) {
  using C = cx<R>;
  const int64_t d = p.d_begin + (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (d >= p.d_end) return;
  const int r0 = threadIdx.x * V;
  const int b = p.b;
  const int Z = p.Z, Y = p.Y, X = p.X, T = p.T;

  // natural site and its coordinates (geometry.py:51-72)
  int64_t site = PAR ? 2 * d : d;
  int z = (int)(site % Z);
  int64_t q = site / Z;
  const int y = (int)(q % Y);
  q /= Y;
  const int x = (int)(q % X);
  const int t = (int)(q / X);
  if (PAR) {
    const int zz = z + ((t + x + y + z + p.par0 + p.dst_parity) & 1);
    site += zz - z;
    z = zz;
  }
  const int64_t sY = Z, sX = (int64_t)Y * Z, sT = p.per_t;

  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  const int64_t kstride = p.n_src * b;
  const int64_t n = p.n;

  C acc[V][12];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int k = 0; k < 12; ++k) acc[v][k] = mk(R(0), R(0));

  auto sidx = [&](int64_t s) -> int64_t { return PAR ? (s >> 1) : s; };
  auto sptr = [&](int64_t s) { return src + sidx(s) * b + r0; };

  // forward hops: P-_mu U_mu(x) psi(x+mu)  (dirac.py:222-245)
  {
    const int64_t f3 = (z + 1 == Z) ? site - (Z - 1) : site + 1;
    const int64_t f2 = (y + 1 == Y) ? site - (int64_t)(Y - 1) * sY : site + sY;
    const int64_t f1 = (x + 1 == X) ? site - (int64_t)(X - 1) * sX : site + sX;
    const int64_t f0 = (t + 1 == T) ? site - (int64_t)(T - 1) * sT : site + sT;
    if (HALO && t + 1 == T) {
      const C* hp = static_cast<const C*>(p.lam_halo) + sidx(f0) * b + r0;
      hop_lam_halo<R, V>(acc, hp, p.nf * b, U + 0 * 9 * n + site, n);
    } else {
      hop_full<0, true, R, V>(acc, sptr(f0), kstride, U + 0 * 9 * n + site, n);
    }
    hop_full<1, true, R, V>(acc, sptr(f1), kstride, U + 1 * 9 * n + site, n);
    hop_full<2, true, R, V>(acc, sptr(f2), kstride, U + 2 * 9 * n + site, n);
    hop_full<3, true, R, V>(acc, sptr(f3), kstride, U + 3 * 9 * n + site, n);
  }
  // backward hops: P+_mu U_mu(x-mu)^H psi(x-mu)  (dirac.py:185-219, 248-255)
  {
    const int64_t b3 = (z == 0) ? site + (Z - 1) : site - 1;
    const int64_t b2 = (y == 0) ? site + (int64_t)(Y - 1) * sY : site - sY;
    const int64_t b1 = (x == 0) ? site + (int64_t)(X - 1) * sX : site - sX;
    const int64_t b0 = (t == 0) ? site + (int64_t)(T - 1) * sT : site - sT;
    if (HALO && t == 0) {
      const C* hp = static_cast<const C*>(p.chi_halo) + sidx(site) * b + r0;
      hop_chi_halo<R, V>(acc, hp, p.nf * b);
    } else {
      hop_full<0, false, R, V>(acc, sptr(b0), kstride, U + 0 * 9 * n + b0, n);
    }
    hop_full<1, false, R, V>(acc, sptr(b1), kstride, U + 1 * 9 * n + b1, n);
    hop_full<2, false, R, V>(acc, sptr(b2), kstride, U + 2 * 9 * n + b2, n);
    hop_full<3, false, R, V>(acc, sptr(b3), kstride, U + 3 * 9 * n + b3, n);
  }

  // epilogue: out = scale_r (alpha xself + beta acc)
  const int64_t okstride = p.n_dst * b;
  C* out = static_cast<C*>(p.out) + d * b + r0;
  const C* xs = static_cast<const C*>(p.xself);
  R sc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) sc[v] = p.scale ? R(__ldg(p.scale + r0 + v)) : R(1);
  const R beta = R(p.beta), alpha = R(p.alpha);
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    C res[V];
    if (xs) {
      C xv[V];
      VecIO<R, V>::ld(xv, xs + d * b + r0 + k * okstride);
#pragma unroll
      for (int v = 0; v < V; ++v)
        res[v] = mk(sc[v] * (alpha * xv[v].x + beta * acc[v][k].x), sc[v] * (alpha * xv[v].y + beta * acc[v][k].y));
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) res[v] = mk(sc[v] * beta * acc[v][k].x, sc[v] * beta * acc[v][k].y);
    }
    VecIO<R, V>::st(out + k * okstride, res);
  }
}

// ---- halo face pack (halo.py:352-368) ---------------------------------------
template <typename R, int V, bool PAR>
__global__ void __launch_bounds__(256) halo_pack_kernel(const HopParams p, void* lam_face, void* chi_face) {
  using C = cx<R>;
  const int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;  // face index
  if (i >= p.nf) return;
  const int r0 = threadIdx.x * V;
  const int b = p.b;
  const C* __restrict__ src = static_cast<const C*>(p.src);
  const C* __restrict__ U = static_cast<const C*>(p.U);
  const int64_t kstride = p.n_src * b;
  const int64_t fstride = p.nf * b;
  // src parity for PAR is p.dst_parity (reused field)
  for (int face = 0; face < 2; ++face) {
    const int tf = face == 0 ? 0 : p.T - 1;
    int64_t sidx = PAR ? i + (int64_t)tf * (p.per_t / 2) : i + (int64_t)tf * p.per_t;
    int64_t site = sidx;
    if (PAR) {
      site = 2 * sidx;
      int z = (int)(site % p.Z);
      int64_t q = site / p.Z;
      const int y = (int)(q % p.Y);
      q /= p.Y;
      const int x = (int)(q % p.X);
      const int t = (int)(q / p.X);
      site += (t + x + y + z + p.par0 + p.dst_parity) & 1;
    }
    C psi[V][12];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      C tmp[V];
      VecIO<R, V>::ld(tmp, src + sidx * b + r0 + k * kstride);
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
      C u[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) u[e] = __ldg(U + (int64_t)e * p.n + site);
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

template <typename R, int V>
static void launch_hop(const HopParams& p, bool par, bool halo, cudaStream_t st) {
  const int bt = p.b / V;
  const int S = bt >= 256 ? 1 : 256 / bt;
  dim3 block(bt, S);
  const int64_t nd = p.d_end - p.d_begin;
  dim3 grid((unsigned)((nd + S - 1) / S));
  if (par) {
    if (halo) hop_kernel<R, V, true, true><<<grid, block, 0, st>>>(p);
    else hop_kernel<R, V, true, false><<<grid, block, 0, st>>>(p);
  } else {
    if (halo) hop_kernel<R, V, false, true><<<grid, block, 0, st>>>(p);
    else hop_kernel<R, V, false, false><<<grid, block, 0, st>>>(p);
  }
}

template <typename R, int V>
static void launch_pack(const HopParams& p, bool par, void* lam, void* chi, cudaStream_t st) {
  const int bt = p.b / V;
  const int S = bt >= 256 ? 1 : 256 / bt;
  dim3 block(bt, S);
  dim3 grid((unsigned)((p.nf + S - 1) / S));
  if (par) halo_pack_kernel<R, V, true><<<grid, block, 0, st>>>(p, lam, chi);
  else halo_pack_kernel<R, V, false><<<grid, block, 0, st>>>(p, lam, chi);
}

static int fill_params(HopParams& p, const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t parity) {
  B200WD_REQUIRE(lat != nullptr, "lattice descriptor is NULL");
  for (int d = 0; d < 4; ++d)
    B200WD_REQUIRE(lat->dims[d] >= 2 && lat->dims[d] % 2 == 0,
                   "extent %d in direction %d is not an even number >= 2", lat->dims[d], d);
  B200WD_REQUIRE(dtype == B200WD_C128 || dtype == B200WD_C64, "unknown dtype %d", dtype);
  B200WD_REQUIRE(b >= 1 && b <= 256, "rhs count b=%d out of range [1,256]", b);
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
  const bool halo = lam_halo != nullptr;
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) {
    launch_hop<double, 1>(p, dst_parity >= 0, halo, st);
  } else if (b % 2 == 0) {
    launch_hop<float, 2>(p, dst_parity >= 0, halo, st);
  } else {
    launch_hop<float, 1>(p, dst_parity >= 0, halo, st);
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
  if (dtype == B200WD_C128) launch_pack<double, 1>(p, src_parity >= 0, lam_face, chi_face, st);
  else if (b % 2 == 0) launch_pack<float, 2>(p, src_parity >= 0, lam_face, chi_face, st);
  else launch_pack<float, 1>(p, src_parity >= 0, lam_face, chi_face, st);
  return check_launch("b200wd_halo_pack");
}
