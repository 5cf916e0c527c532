// Per-rhs BLAS-1 and the batched-GMRES Arnoldi kernels (complex128 planes).
//
// Reductions are lane-per-rhs: a block is (b, S) threads, thread (r, y)
// owns rhs r and walks sites y, y+S*G, ... in a fixed order, so every rhs
// sees an identical summation tree (replicated right-hand sides give
// bit-identical histories, tests/test_gmres.py:141-151).  Block partials go
// to scratch; the last block to finish (atomic ticket) folds them in a fixed
// order -- the result is deterministic run to run.  The GMRES kernels fuse
// each MGS axpy with the next inner product (or the final norm), keep the
// basis unnormalised (V_p = sigma_p Z_p) so no separate normalise pass is
// needed, and run the Givens/least-squares bookkeeping on the device with
// one thread per rhs (gmres.py:101-177).
#include <math.h>

#include <cooperative_groups.h>

#include "capi.cuh"
#include "common.cuh"

namespace b200wd {
namespace cg = cooperative_groups;

constexpr int kMaxGrid = 148 * 4;
constexpr int kBlock = 256;

// (site, component) groups of a field, storage padded to whole 8-site blocks
__host__ __device__ __forceinline__ int64_t groups(int64_t n, int s) { return ((n + 7) / 8) * 8 * s; }

static inline int rows_per_block(int b) { return b >= kBlock ? 1 : kBlock / b; }

// Reduction grid: at least kRowsPerThread (site, component) groups per thread
// (small fields: fewer blocks, cheaper folds and grid barriers), at most
// kMaxGrid blocks.  B200WD_RED_ROWS overrides (tuning).
static inline int rows_per_thread() {
  static int k = -1;
  if (k < 0) {
    const char* e = getenv("B200WD_RED_ROWS");
    k = e ? atoi(e) : 4;
    if (k < 1) k = 1;
  }
  return k;
}
static inline int grid_for_sites(int64_t n, int S) {
  n = ((n + 7) / 8) * 8 * 12;  // group count of a full spinor field (upper bound for s <= 12)
  const int64_t per_block = (int64_t)S * rows_per_thread();
  int64_t g = (n + per_block - 1) / per_block;
  if (g > kMaxGrid) g = kMaxGrid;
  return (int)(g < 1 ? 1 : g);
}

struct Scratch {
  double2* partials;   // [kMaxGrid][b]
  unsigned* ticket;    // 64 bytes
  double2* partials2;  // [kMaxGrid][b], second buffer of the single-launch Arnoldi sweep
};
static inline Scratch scratch_of(void* p, int b) {
  Scratch s;
  s.partials = static_cast<double2*>(p);
  s.ticket = reinterpret_cast<unsigned*>(static_cast<char*>(p) + (size_t)kMaxGrid * b * sizeof(double2));
  s.partials2 = reinterpret_cast<double2*>(reinterpret_cast<char*>(s.ticket) + 64);
  return s;
}

// Block-reduce `v` over threadIdx.y (fixed tree), write the block partial,
// and let the last block fold all partials into out[r].
__device__ void reduce_finish(double2 v, Scratch sc, double2* out) {
  extern __shared__ double2 red[];  // [S][b]
  const int b = blockDim.x, S = blockDim.y, r = threadIdx.x, y = threadIdx.y;
  __shared__ unsigned s_last;
  red[y * b + r] = v;
  __syncthreads();
  int p2 = 1;
  while (p2 < S) p2 <<= 1;
  for (int stride = p2 >> 1; stride > 0; stride >>= 1) {
    if (y < stride && y + stride < S) {
      double2 a = red[y * b + r], c = red[(y + stride) * b + r];
      red[y * b + r] = make_double2(a.x + c.x, a.y + c.y);
    }
    __syncthreads();
  }
  if (y == 0) sc.partials[(size_t)blockIdx.x * b + r] = red[r];
  __threadfence();
  __syncthreads();
  if (r == 0 && y == 0) s_last = (atomicAdd(sc.ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double2 acc = make_double2(0.0, 0.0);
  for (int g = y; g < (int)gridDim.x; g += S) {
    double2 q = __ldcg(sc.partials + (size_t)g * b + r);
    acc.x += q.x;
    acc.y += q.y;
  }
  red[y * b + r] = acc;
  __syncthreads();
  for (int stride = p2 >> 1; stride > 0; stride >>= 1) {
    if (y < stride && y + stride < S) {
      double2 a = red[y * b + r], c = red[(y + stride) * b + r];
      red[y * b + r] = make_double2(a.x + c.x, a.y + c.y);
    }
    __syncthreads();
  }
  if (y == 0) {
    out[r] = red[r];
    if (r == 0) *sc.ticket = 0u;
  }
}

__device__ __forceinline__ void acc_dot(double2& a, double2 x, double2 y) {
  // conj(x) * y
  a.x = fma(x.x, y.x, a.x);
  a.x = fma(x.y, y.y, a.x);
  a.y = fma(x.x, y.y, a.y);
  a.y = fma(-x.y, y.x, a.y);
}

// ---- reference BLAS ----------------------------------------------------------
__global__ void dot_kernel(int64_t n, int s, const double2* __restrict__ x, const double2* __restrict__ yv,
                           double2* out, Scratch sc) {
  const int b = blockDim.x, r = threadIdx.x;
  double2 a = make_double2(0.0, 0.0);
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const int64_t i = g * b + r;
      acc_dot(a, __ldg(x + i), __ldg(yv + i));
    }
  reduce_finish(a, sc, out);
}

__global__ void norm2_kernel(int64_t n, int s, const double2* __restrict__ x, double2* out, Scratch sc) {
  const int b = blockDim.x, r = threadIdx.x;
  double2 a = make_double2(0.0, 0.0);
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const double2 v = __ldg(x + g * b + r);
      a.x = fma(v.x, v.x, a.x);
      a.x = fma(v.y, v.y, a.x);
    }
  reduce_finish(a, sc, out);
}

__global__ void axpy_kernel(int64_t total, int b, const double2* __restrict__ alpha, const double2* __restrict__ x,
                            double2* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = __ldg(alpha + i % b);
    y[i] = cmac(y[i], a, __ldg(x + i));
  }
}

__global__ void scale_kernel(int64_t total, int b, const double2* __restrict__ alpha, double2* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = cmul(__ldg(alpha + i % b), x[i]);
}

// ---- GMRES ------------------------------------------------------------------
struct GState {
  int b, m;
  double brk_rel;
  double2 *h_raw, *h, *gamma, *sn, *dot, *y;
  double *cs, *sigma, *eta_norm, *relnorm;
  int* brk;
  Scratch sc;
  double2* cgs;  // [m+1][grid][b] block partials of the CGS projection pass
};

static GState gstate(const b200wd_gmres_state* st) {
  GState g;
  g.b = st->b;
  g.m = st->m;
  g.brk_rel = st->breakdown_rel;
  g.h_raw = static_cast<double2*>(st->h_raw);
  g.h = static_cast<double2*>(st->h);
  g.gamma = static_cast<double2*>(st->gamma);
  g.sn = static_cast<double2*>(st->sn);
  g.dot = static_cast<double2*>(st->dot);
  g.y = static_cast<double2*>(st->y);
  g.cs = static_cast<double*>(st->cs);
  g.sigma = static_cast<double*>(st->sigma);
  g.eta_norm = static_cast<double*>(st->eta_norm);
  g.relnorm = static_cast<double*>(st->relnorm);
  g.brk = static_cast<int*>(st->breakdown);
  g.sc = scratch_of(st->scratch, st->b);
  g.cgs = static_cast<double2*>(st->cgs_partials);
  return g;
}

constexpr double kTiny = 1e-300;  // gmres.py:39

__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }

// r := eta - r ; dot := ||r||^2
__global__ void residual_kernel(int64_t n, int s, const double2* __restrict__ eta, double2* __restrict__ r,
                                GState g) {
  const int b = blockDim.x, rr = threadIdx.x;
  double2 a = make_double2(0.0, 0.0);
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const int64_t i = g * b + rr;
      const double2 e = __ldg(eta + i), v = r[i];
      const double2 d = make_double2(e.x - v.x, e.y - v.y);
      r[i] = d;
      a.x = fma(d.x, d.x, a.x);
      a.x = fma(d.y, d.y, a.x);
    }
  reduce_finish(a, g.sc, g.dot);
}

// eta_norm = sqrt(dot), breakdown flags cleared (gmres.py:204-205)
__global__ void init_kernel(GState g) {
  const int r = threadIdx.x;
  if (r >= g.b) return;
  g.eta_norm[r] = sqrt(g.dot[r].x);
  g.brk[r] = 0;
}

// cycle start (gmres.py:180-198)
__global__ void start_kernel(GState g) {
  const int r = threadIdx.x;
  if (r >= g.b) return;
  const int m = g.m;
  const double beta = sqrt(g.dot[r].x);
  for (int i = 0; i < (m + 1) * m; ++i) {
    g.h[(size_t)r * (m + 1) * m + i] = make_double2(0.0, 0.0);
    g.h_raw[(size_t)r * (m + 1) * m + i] = make_double2(0.0, 0.0);
  }
  for (int i = 0; i <= m; ++i) g.gamma[(size_t)r * (m + 1) + i] = make_double2(0.0, 0.0);
  for (int i = 0; i < m; ++i) {
    g.cs[(size_t)r * m + i] = 0.0;
    g.sn[(size_t)r * m + i] = make_double2(0.0, 0.0);
  }
  for (int i = 0; i <= m; ++i) g.sigma[(size_t)i * g.b + r] = 0.0;
  g.gamma[(size_t)r * (m + 1)] = make_double2(beta, 0.0);
  g.sigma[r] = beta > 0 ? 1.0 / beta : 0.0;
  const double en = g.eta_norm[r];
  g.relnorm[r] = en > 0 ? beta / fmax(en, kTiny) : 0.0;
}

// dot := <Z, w>
__global__ void gdot_kernel(int64_t n, int s, const double2* __restrict__ z, const double2* __restrict__ w, GState g) {
  const int b = blockDim.x, r = threadIdx.x;
  double2 a = make_double2(0.0, 0.0);
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const int64_t i = g * b + r;
      acc_dot(a, __ldg(z + i), __ldg(w + i));
    }
  reduce_finish(a, g.sc, g.dot);
}

// fused MGS pass p of column j (gmres.py:118-121)
template <bool NEXT>
__global__ void mgs_kernel(int j, int p, int64_t n, int s, double2* __restrict__ w, const double2* __restrict__ zp,
                           const double2* __restrict__ zn, GState g) {
  const int b = blockDim.x, r = threadIdx.x;
  const int m = g.m;
  const double sig = g.sigma[(size_t)p * g.b + r];
  const double2 d = g.dot[r];
  const double2 hp = make_double2(sig * d.x, sig * d.y);  // h_p = <V_p, w>
  const double2 c = make_double2(-sig * hp.x, -sig * hp.y);  // w -= h_p V_p = h_p sigma_p Z_p
  if (blockIdx.x == 0 && threadIdx.y == 0) g.h_raw[((size_t)r * (m + 1) + p) * m + j] = hp;
  double2 a = make_double2(0.0, 0.0);
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const int64_t i = g * b + r;
      const double2 wn = cmac(w[i], c, __ldg(zp + i));
      w[i] = wn;
      if (NEXT) {
        acc_dot(a, __ldg(zn + i), wn);
      } else {
        a.x = fma(wn.x, wn.x, a.x);
        a.x = fma(wn.y, wn.y, a.x);
      }
    }
  reduce_finish(a, g.sc, g.dot);
}

// Givens pair (gmres.py:101-112): c real, s = phase(a) conj(b) / rho
__device__ void givens(double2 a, double2 bb, double& c, double2& s) {
  const double aa = cabs_(a), ab = cabs_(bb);
  const double rho = sqrt(aa * aa + ab * ab);
  if (rho > 0) {
    c = aa > 0 ? aa / rho : 0.0;
    const double2 ph = aa > 0 ? make_double2(a.x / aa, a.y / aa) : make_double2(1.0, 0.0);
    const double2 t = cmul(ph, make_double2(bb.x, -bb.y));
    s = make_double2(t.x / rho, t.y / rho);
  } else {
    c = 1.0;
    s = make_double2(0.0, 0.0);
  }
}

// close column j (gmres.py:135-157), rhs r, from dot[r].x = ||w||^2
__device__ void close_column_body(int j, const GState& g, int r);
__global__ void close_column_kernel(int j, GState g) {
  const int r = threadIdx.x;
  if (r >= g.b) return;
  close_column_body(j, g, r);
}
__device__ void close_column_body(int j, const GState& g, int r) {
  const int m = g.m;
  const double hn = sqrt(g.dot[r].x);
  const double en = g.eta_norm[r];
  int brk = g.brk[r] | (hn <= g.brk_rel * en ? 1 : 0);
  g.brk[r] = brk;
  double2* hraw = g.h_raw + (size_t)r * (m + 1) * m;
  double2* hh = g.h + (size_t)r * (m + 1) * m;
  hraw[(j + 1) * m + j] = make_double2(brk ? 0.0 : hn, 0.0);
  g.sigma[(size_t)(j + 1) * g.b + r] = (brk || hn <= 0) ? 0.0 : 1.0 / hn;
  // fold the new column through the stored rotations
  double2 col[2];
  col[0] = hraw[0 * m + j];
  double* cs = g.cs + (size_t)r * m;
  double2* sn = g.sn + (size_t)r * m;
  for (int p = 0; p < j; ++p) {
    const double2 a0 = col[0], a1 = hraw[(p + 1) * m + j];
    const double2 sp = sn[p];
    const double2 t0 = cmul(sp, a1);
    const double2 top = make_double2(cs[p] * a0.x + t0.x, cs[p] * a0.y + t0.y);
    const double2 t1 = cmul(make_double2(-sp.x, sp.y), a0);  // -conj(s) a0
    col[0] = make_double2(t1.x + cs[p] * a1.x, t1.y + cs[p] * a1.y);
    hh[p * m + j] = top;
  }
  col[1] = hraw[(j + 1) * m + j];
  double c;
  double2 s;
  givens(col[0], col[1], c, s);
  cs[j] = c;
  sn[j] = s;
  const double2 t = cmul(s, col[1]);
  hh[j * m + j] = make_double2(c * col[0].x + t.x, c * col[0].y + t.y);
  hh[(j + 1) * m + j] = make_double2(0.0, 0.0);
  double2* gam = g.gamma + (size_t)r * (m + 1);
  const double2 gj = gam[j];
  gam[j + 1] = cmul(make_double2(-s.x, s.y), gj);
  gam[j] = make_double2(c * gj.x, c * gj.y);
  g.relnorm[r] = en > 0 ? cabs_(gam[j + 1]) / fmax(en, kTiny) : 0.0;
}

// back substitution (gmres.py:161-177): one warp per rhs.  Row by row the lanes
// form the products h[row][c] y[c] in parallel; lane 0 subtracts them in
// ascending c, the same arithmetic and order as a sequential loop.
__global__ void backsub_kernel(int jd, GState g) {
  __shared__ double2 ys[64], prod[64];
  const int r = blockIdx.x, lane = threadIdx.x;
  if (r >= g.b) return;
  const int m = g.m;
  const double2* hh = g.h + (size_t)r * (m + 1) * m;
  const double2* gam = g.gamma + (size_t)r * (m + 1);
  double2* y = g.y + (size_t)r * m;
  for (int row = jd - 1; row >= 0; --row) {
    for (int c2 = row + 1 + lane; c2 < jd; c2 += 32) prod[c2] = cmul(hh[row * m + c2], ys[c2]);
    __syncwarp();
    if (lane == 0) {
      double2 acc = gam[row];
      for (int c2 = row + 1; c2 < jd; ++c2) {
        acc.x -= prod[c2].x;
        acc.y -= prod[c2].y;
      }
      const double2 dg = hh[row * m + row];
      double2 yr = make_double2(0.0, 0.0);
      if (cabs_(dg) > 0) {
        const double den = dg.x * dg.x + dg.y * dg.y;
        yr = make_double2((acc.x * dg.x + acc.y * dg.y) / den, (acc.y * dg.x - acc.x * dg.y) / den);
      }
      ys[row] = yr;
      y[row] = yr;
    }
    __syncwarp();
  }
}

constexpr int kMaxBasis = 64;
struct ZList {
  const double2* z[kMaxBasis];
};

// psi += sum_p y_p sigma_p Z_p  (one pass over psi and the basis)
__global__ void update_kernel(int jd, int64_t n, int s, ZList zl, double2* __restrict__ psi, GState g) {
  extern __shared__ double2 coef_s[];  // [jd][b]
  const int b = blockDim.x, r = threadIdx.x;
  const int m = g.m;
  for (int p = threadIdx.y; p < jd; p += blockDim.y) {
    const double2 yp = g.y[(size_t)r * m + p];
    const double sg = g.sigma[(size_t)p * g.b + r];
    coef_s[p * b + r] = make_double2(yp.x * sg, yp.y * sg);
  }
  __syncthreads();
  const double2* coef = coef_s + r;
  const int64_t ng = groups(n, s);
  for (int64_t g = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; g < ng; g += (int64_t)gridDim.x * blockDim.y) {
      const int64_t i = g * b + r;
      double2 a = psi[i];
#pragma unroll 1
      for (int p = 0; p < jd; ++p) a = cmac(a, coef[p * b], __ldg(zl.z[p] + i));
      psi[i] = a;
    }
}

// ---- single-launch Arnoldi sweep (cooperative grid) --------------------------
// The whole Gram-Schmidt sweep of column j -- <Z_0,w>, the j+1 fused MGS passes,
// ||w||^2 and the column close -- in one launch with a grid barrier per
// reduction instead of one kernel per pass.  Same grid, block shape, per-thread
// site walk, block trees and partial fold order as gdot/mgs/reduce_finish, so
// the results are bit-identical to the multi-launch sequence; every block folds
// the partials itself (no ticket), partial buffers alternate between passes.
__device__ __forceinline__ void block_partial(double2 v, double2* red, double2* out) {
  const int b = blockDim.x, S = blockDim.y, r = threadIdx.x, y = threadIdx.y;
  __syncthreads();  // red may still be read by the previous fold
  red[y * b + r] = v;
  __syncthreads();
  int p2 = 1;
  while (p2 < S) p2 <<= 1;
  for (int stride = p2 >> 1; stride > 0; stride >>= 1) {
    if (y < stride && y + stride < S) {
      double2 a = red[y * b + r], c = red[(y + stride) * b + r];
      red[y * b + r] = make_double2(a.x + c.x, a.y + c.y);
    }
    __syncthreads();
  }
  if (y == 0) out[(size_t)blockIdx.x * b + r] = red[r];
}
__device__ __forceinline__ double2 fold_partials(const double2* part, double2* red) {
  const int b = blockDim.x, S = blockDim.y, r = threadIdx.x, y = threadIdx.y;
  double2 acc = make_double2(0.0, 0.0);
  for (int q = y; q < (int)gridDim.x; q += S) {
    double2 v = __ldcg(part + (size_t)q * b + r);
    acc.x += v.x;
    acc.y += v.y;
  }
  __syncthreads();
  red[y * b + r] = acc;
  __syncthreads();
  int p2 = 1;
  while (p2 < S) p2 <<= 1;
  for (int stride = p2 >> 1; stride > 0; stride >>= 1) {
    if (y < stride && y + stride < S) {
      double2 a = red[y * b + r], c = red[(y + stride) * b + r];
      red[y * b + r] = make_double2(a.x + c.x, a.y + c.y);
    }
    __syncthreads();
  }
  return red[r];
}

__global__ void arnoldi_sweep_kernel(int j, int64_t n, int s, ZList zl, double2* w, GState g, const int* stop) {
  if (stop != nullptr && *static_cast<const volatile int*>(stop) != 0) return;  // cycle already converged
  extern __shared__ double2 red[];
  cg::grid_group grid = cg::this_grid();
  const int b = blockDim.x, r = threadIdx.x, y = threadIdx.y;
  const int m = g.m;
  const int64_t ng = groups(n, s);
  const int64_t g0 = (int64_t)blockIdx.x * blockDim.y + y, gst = (int64_t)gridDim.x * blockDim.y;
  double2 a = make_double2(0.0, 0.0);
  const double2* __restrict__ z0 = zl.z[0];
  for (int64_t q = g0; q < ng; q += gst) {
    const int64_t i = q * b + r;
    acc_dot(a, __ldg(z0 + i), w[i]);
  }
  block_partial(a, red, g.sc.partials);
  grid.sync();
  double2 d = fold_partials(g.sc.partials, red);
  for (int p = 0; p <= j; ++p) {
    const double sig = g.sigma[(size_t)p * g.b + r];
    const double2 hp = make_double2(sig * d.x, sig * d.y);
    const double2 c = make_double2(-sig * hp.x, -sig * hp.y);
    if (blockIdx.x == 0 && y == 0) g.h_raw[((size_t)r * (m + 1) + p) * m + j] = hp;
    const double2* __restrict__ zp = zl.z[p];
    a = make_double2(0.0, 0.0);
    if (p < j) {
      const double2* __restrict__ zn = zl.z[p + 1];
      for (int64_t q = g0; q < ng; q += gst) {
        const int64_t i = q * b + r;
        const double2 wn = cmac(w[i], c, __ldg(zp + i));
        w[i] = wn;
        acc_dot(a, __ldg(zn + i), wn);
      }
    } else {
      for (int64_t q = g0; q < ng; q += gst) {
        const int64_t i = q * b + r;
        const double2 wn = cmac(w[i], c, __ldg(zp + i));
        w[i] = wn;
        a.x = fma(wn.x, wn.x, a.x);
        a.x = fma(wn.y, wn.y, a.x);
      }
    }
    double2* buf = (p & 1) ? g.sc.partials : g.sc.partials2;
    block_partial(a, red, buf);
    grid.sync();
    d = fold_partials(buf, red);
  }
  if (blockIdx.x == 0 && y == 0) {
    g.dot[r] = d;
    close_column_body(j, g, r);
  }
}


// ---- classical Gram-Schmidt sweep (B200 extension, b200wd_gmres_state.orth) --
// Pass A: all j+1 projections <Z_p, w> in one pass over the basis (the
// accumulators of kCgsChunk basis vectors live in registers, so w is re-read
// once per chunk); block partials per p, block p folds projection p (distributed
// fold), h_raw[p][j] = sigma_p <Z_p,w> and the update coefficient
// -sigma_p h_p go to y (free scratch until the cycle's back substitution).
// Pass B: w -= sum_p c_p Z_p with ||w||^2 formed from the stored result, then
// the column close.  Traffic (j+1)(2 + 1/kCgsChunk) F + 3F vs 4(j+1)+2 F for MGS.
constexpr int kCgsChunk = 8;

__global__ void arnoldi_cgs_kernel(int j, int64_t n, int s, ZList zl, double2* w, GState g, const int* stop) {
  if (stop != nullptr && *static_cast<const volatile int*>(stop) != 0) return;  // cycle already converged
  extern __shared__ double2 red[];  // [S][b] reduction tree, then [j+1][b] coefficients
  cg::grid_group grid = cg::this_grid();
  const int b = blockDim.x, r = threadIdx.x, y = threadIdx.y, S = blockDim.y;
  const int m = g.m;
  const int64_t ng = groups(n, s);
  const int64_t g0 = (int64_t)blockIdx.x * S + y, gst = (int64_t)gridDim.x * S;
  const size_t pstride = (size_t)gridDim.x * b;
  for (int p0 = 0; p0 <= j; p0 += kCgsChunk) {
    const int np = min(kCgsChunk, j + 1 - p0);
    double2 a[kCgsChunk];
#pragma unroll
    for (int k = 0; k < kCgsChunk; ++k) a[k] = make_double2(0.0, 0.0);
    for (int64_t q = g0; q < ng; q += gst) {
      const int64_t i = q * b + r;
      const double2 wv = w[i];
#pragma unroll
      for (int k = 0; k < kCgsChunk; ++k)
        if (k < np) acc_dot(a[k], __ldg(zl.z[p0 + k] + i), wv);
    }
#pragma unroll
    for (int k = 0; k < kCgsChunk; ++k)
      if (k < np) block_partial(a[k], red, g.cgs + (size_t)(p0 + k) * pstride);
  }
  grid.sync();
  for (int p = blockIdx.x; p <= j; p += gridDim.x) {
    const double2 d = fold_partials(g.cgs + (size_t)p * pstride, red);
    if (y == 0) {
      const double sig = g.sigma[(size_t)p * g.b + r];
      const double2 hp = make_double2(sig * d.x, sig * d.y);
      g.h_raw[((size_t)r * (m + 1) + p) * m + j] = hp;
      g.y[(size_t)r * m + p] = make_double2(-sig * hp.x, -sig * hp.y);
    }
  }
  grid.sync();
  double2* coef = red + (size_t)S * b;
  for (int p = y; p <= j; p += S) coef[p * b + r] = __ldcg(g.y + (size_t)r * m + p);
  __syncthreads();
  double2 a = make_double2(0.0, 0.0);
  for (int64_t q = g0; q < ng; q += gst) {
    const int64_t i = q * b + r;
    double2 v = w[i];
#pragma unroll 4
    for (int p = 0; p <= j; ++p) v = cmac(v, coef[p * b + r], __ldg(zl.z[p] + i));
    w[i] = v;
    a.x = fma(v.x, v.x, a.x);
    a.x = fma(v.y, v.y, a.x);
  }
  block_partial(a, red, g.sc.partials);
  grid.sync();
  const double2 d = fold_partials(g.sc.partials, red);
  if (blockIdx.x == 0 && y == 0) {
    g.dot[r] = d;
    close_column_body(j, g, r);
  }
}

static dim3 red_block(int b) { return dim3(b, rows_per_block(b)); }
static size_t red_smem(int b) { return (size_t)b * rows_per_block(b) * sizeof(double2); }

}  // namespace b200wd

using namespace b200wd;

extern "C" int64_t b200wd_cgs_scratch_bytes(int32_t b, int32_t m) {
  return (int64_t)(m + 1) * kMaxGrid * b * (int64_t)sizeof(double2);
}

extern "C" int64_t b200wd_reduce_scratch_bytes(int32_t b) {
  return 2 * (int64_t)kMaxGrid * b * (int64_t)sizeof(double2) + 64;
}

#define CHECK_FIELD(n, s, b)                                                                        \
  B200WD_REQUIRE((n) >= 1 && (s) >= 1 && (b) >= 1 && (b) <= kBlock, "bad field shape n=%lld s=%d b=%d", \
                 (long long)(n), (s), (b))

extern "C" int b200wd_block_dot(int64_t n_sites, int32_t s, int32_t b, const void* x, const void* y, void* out,
                                void* scratch, void* stream) {
  CHECK_FIELD(n_sites, s, b);
  B200WD_REQUIRE(x && y && out && scratch, "NULL pointer");
  dim3 blk = red_block(b);
  dot_kernel<<<grid_for_sites(n_sites, blk.y), blk, red_smem(b), as_stream(stream)>>>(
      n_sites, s, static_cast<const double2*>(x), static_cast<const double2*>(y), static_cast<double2*>(out),
      scratch_of(scratch, b));
  return check_launch("b200wd_block_dot");
}

extern "C" int b200wd_block_norm2(int64_t n_sites, int32_t s, int32_t b, const void* x, void* out, void* scratch,
                                  void* stream) {
  CHECK_FIELD(n_sites, s, b);
  B200WD_REQUIRE(x && out && scratch, "NULL pointer");
  dim3 blk = red_block(b);
  norm2_kernel<<<grid_for_sites(n_sites, blk.y), blk, red_smem(b), as_stream(stream)>>>(
      n_sites, s, static_cast<const double2*>(x), static_cast<double2*>(out), scratch_of(scratch, b));
  return check_launch("b200wd_block_norm2");
}

extern "C" int b200wd_block_axpy(int64_t n_sites, int32_t s, int32_t b, const void* alpha, const void* x, void* y,
                                 void* stream) {
  CHECK_FIELD(n_sites, s, b);
  B200WD_REQUIRE(alpha && x && y, "NULL pointer");
  const int64_t total = groups(n_sites, s) * b;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  axpy_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(total, b, static_cast<const double2*>(alpha),
                                                          static_cast<const double2*>(x), static_cast<double2*>(y));
  return check_launch("b200wd_block_axpy");
}

extern "C" int b200wd_block_scale(int64_t n_sites, int32_t s, int32_t b, const void* alpha, void* x, void* stream) {
  CHECK_FIELD(n_sites, s, b);
  B200WD_REQUIRE(alpha && x, "NULL pointer");
  const int64_t total = groups(n_sites, s) * b;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  scale_kernel<<<(unsigned)g, 256, 0, as_stream(stream)>>>(total, b, static_cast<const double2*>(alpha),
                                                           static_cast<double2*>(x));
  return check_launch("b200wd_block_scale");
}

#define CHECK_STATE(st)                                                                        \
  B200WD_REQUIRE((st) != nullptr && (st)->b >= 1 && (st)->b <= kBlock && (st)->m >= 1 &&      \
                     (st)->m <= kMaxBasis - 1 &&                                               \
                     ((st)->orth == B200WD_ORTH_MGS ||                                         \
                      ((st)->orth == B200WD_ORTH_CGS && (st)->cgs_partials != nullptr)),       \
                 "bad GMRES state (b must be in [1,%d], restart length in [1,%d], orth 0 or 1 " \
                 "with cgs_partials for CGS)", kBlock, kMaxBasis - 1)

extern "C" int b200wd_gmres_residual(const b200wd_gmres_state* st, int64_t n_sites, int32_t s, const void* eta,
                                     void* r, void* stream) {
  CHECK_STATE(st);
  CHECK_FIELD(n_sites, s, st->b);
  B200WD_REQUIRE(eta && r, "NULL pointer");
  dim3 blk = red_block(st->b);
  residual_kernel<<<grid_for_sites(n_sites, blk.y), blk, red_smem(st->b), as_stream(stream)>>>(
      n_sites, s, static_cast<const double2*>(eta), static_cast<double2*>(r), gstate(st));
  return check_launch("b200wd_gmres_residual");
}

extern "C" int b200wd_gmres_init(const b200wd_gmres_state* st, void* stream) {
  CHECK_STATE(st);
  init_kernel<<<1, st->b, 0, as_stream(stream)>>>(gstate(st));
  return check_launch("b200wd_gmres_init");
}

extern "C" int b200wd_gmres_start(const b200wd_gmres_state* st, void* stream) {
  CHECK_STATE(st);
  start_kernel<<<1, st->b, 0, as_stream(stream)>>>(gstate(st));
  return check_launch("b200wd_gmres_start");
}

extern "C" int b200wd_gmres_dot(const b200wd_gmres_state* st, int64_t n_sites, int32_t s, const void* z,
                                const void* w, void* stream) {
  CHECK_STATE(st);
  CHECK_FIELD(n_sites, s, st->b);
  B200WD_REQUIRE(z && w, "NULL pointer");
  dim3 blk = red_block(st->b);
  gdot_kernel<<<grid_for_sites(n_sites, blk.y), blk, red_smem(st->b), as_stream(stream)>>>(
      n_sites, s, static_cast<const double2*>(z), static_cast<const double2*>(w), gstate(st));
  return check_launch("b200wd_gmres_dot");
}

extern "C" int b200wd_gmres_mgs(const b200wd_gmres_state* st, int32_t j, int32_t p, int64_t n_sites, int32_t s,
                                void* w, const void* z_p, const void* z_next, void* stream) {
  CHECK_STATE(st);
  CHECK_FIELD(n_sites, s, st->b);
  B200WD_REQUIRE(0 <= p && p <= j && j < st->m, "MGS index p=%d j=%d outside restart length %d", p, j, st->m);
  B200WD_REQUIRE(w && z_p, "NULL pointer");
  dim3 blk = red_block(st->b);
  const int grid = grid_for_sites(n_sites, blk.y);
  if (z_next)
    mgs_kernel<true><<<grid, blk, red_smem(st->b), as_stream(stream)>>>(
        j, p, n_sites, s, static_cast<double2*>(w), static_cast<const double2*>(z_p),
        static_cast<const double2*>(z_next), gstate(st));
  else
    mgs_kernel<false><<<grid, blk, red_smem(st->b), as_stream(stream)>>>(
        j, p, n_sites, s, static_cast<double2*>(w), static_cast<const double2*>(z_p), nullptr, gstate(st));
  return check_launch("b200wd_gmres_mgs");
}

extern "C" int b200wd_gmres_close_column(const b200wd_gmres_state* st, int32_t j, void* stream) {
  CHECK_STATE(st);
  B200WD_REQUIRE(0 <= j && j < st->m, "column %d outside restart length %d", j, st->m);
  close_column_kernel<<<1, st->b, 0, as_stream(stream)>>>(j, gstate(st));
  return check_launch("b200wd_gmres_close_column");
}

extern "C" int b200wd_gmres_update(const b200wd_gmres_state* st, int32_t j_done, int64_t n_sites, int32_t s,
                                   const void* const* z, void* psi, void* stream) {
  CHECK_STATE(st);
  CHECK_FIELD(n_sites, s, st->b);
  B200WD_REQUIRE(0 <= j_done && j_done <= st->m, "j_done=%d outside [0,%d]", j_done, st->m);
  B200WD_REQUIRE(psi && (j_done == 0 || z), "NULL pointer");
  if (j_done == 0) return B200WD_OK;
  ZList zl{};
  for (int p = 0; p < j_done; ++p) {
    B200WD_REQUIRE(z[p] != nullptr, "basis pointer %d is NULL", p);
    zl.z[p] = static_cast<const double2*>(z[p]);
  }
  backsub_kernel<<<st->b, 32, 0, as_stream(stream)>>>(j_done, gstate(st));
  dim3 blk = red_block(st->b);
  update_kernel<<<grid_for_sites(n_sites, blk.y), blk, (size_t)j_done * st->b * sizeof(double2), as_stream(stream)>>>(
      j_done, n_sites, s, zl, static_cast<double2*>(psi), gstate(st));
  return check_launch("b200wd_gmres_update");
}

// Cooperative launch of arnoldi_sweep_kernel when the reduction grid is
// co-resident (B200WD_NO_COOP=1 forces the per-pass launches).
static bool sweep_single_launch(const b200wd_gmres_state* st, int j, int64_t n_sites, int s, const void* const* z,
                                void* w, void* stream) {
  static int en = -1;
  if (en < 0) {
    const char* e = getenv("B200WD_NO_COOP");
    en = (e && e[0] == '1') ? 0 : 1;
  }
  if (!en) return false;
  const dim3 blk = red_block(st->b);
  const int grid = grid_for_sites(n_sites, blk.y);
  const bool cgs = st->orth == B200WD_ORTH_CGS;
  const size_t smem = cgs ? red_smem(st->b) + (size_t)st->m * st->b * sizeof(double2) : red_smem(st->b);
  const void* kern = cgs ? (const void*)arnoldi_cgs_kernel : (const void*)arnoldi_sweep_kernel;
  LaunchFacts f;
  if (cgs && smem > 48 * 1024) return false;
  if (!launch_facts(kern, blk.x * blk.y, smem, f)) return false;
  int dev = 0, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return false;
  const int occupancy = f.occ, sm_count = f.sm_count;
  if (occupancy <= 0 || (int64_t)occupancy * sm_count < grid) return false;
  ZList zl{};
  for (int p = 0; p <= j + 1; ++p) zl.z[p] = static_cast<const double2*>(z[p]);
  GState g = gstate(st);
  int jj = j, ss = s;
  int64_t nn = n_sites;
  double2* wp = static_cast<double2*>(w);
  const int* stop = g_hop_stop;
  void* args[] = {&jj, &nn, &ss, &zl, &wp, &g, &stop};
  if (cudaLaunchCooperativeKernel(kern, dim3(grid), blk, args, smem, as_stream(stream)) == cudaSuccess)
    return true;
  (void)cudaGetLastError();  // not sticky: fall back to the per-pass launches
  return false;
}

extern "C" int b200wd_gmres_arnoldi(const b200wd_gmres_state* st, const b200wd_operator* op, int32_t j,
                                    int64_t n_sites, const void* const* z, double* relnorm_host, void* stream) {
  CHECK_STATE(st);
  B200WD_REQUIRE(op != nullptr && z != nullptr, "NULL pointer");
  B200WD_REQUIRE(0 <= j && j < st->m, "column %d outside restart length %d", j, st->m);
  B200WD_REQUIRE(op->dtype == B200WD_C128, "the device GMRES runs in complex128");
  const int32_t s = 12;
  CHECK_FIELD(n_sites, s, st->b);
  for (int p = 0; p <= j + 1; ++p) B200WD_REQUIRE(z[p] != nullptr, "basis pointer %d is NULL", p);
  void* w = const_cast<void*>(z[j + 1]);
  // w = A V_j = sigma_j A Z_j  (row j of sigma)
  const double* sig = static_cast<const double*>(st->sigma) + (int64_t)j * st->b;
  if (int rc = b200wd_operator_apply(op, st->b, z[j], w, sig, stream)) return rc;
  if (!sweep_single_launch(st, j, n_sites, s, z, w, stream)) {
    if (st->orth == B200WD_ORTH_CGS) {
      set_error("b200wd_gmres_arnoldi: classical Gram-Schmidt needs the cooperative sweep (m*b <= 2816, co-resident grid)");
      return B200WD_ERR_UNSUPPORTED;
    }
    if (int rc = b200wd_gmres_dot(st, n_sites, s, z[0], w, stream)) return rc;
    for (int p = 0; p <= j; ++p)
      if (int rc = b200wd_gmres_mgs(st, j, p, n_sites, s, w, z[p], p < j ? z[p + 1] : nullptr, stream)) return rc;
    if (int rc = b200wd_gmres_close_column(st, j, stream)) return rc;
  } else if (int rc = check_launch("b200wd_gmres_arnoldi (sweep)")) {
    return rc;
  }
  if (relnorm_host) {
    cudaStream_t cs = as_stream(stream);
    cudaError_t e = cudaMemcpyAsync(relnorm_host, st->relnorm, sizeof(double) * st->b, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) {
      set_error("b200wd_gmres_arnoldi: %s", cudaGetErrorString(e));
      return B200WD_ERR_CUDA;
    }
  }
  return B200WD_OK;
}

// After Arnoldi step j of a device-driven cycle: store relnorm into row j of
// the cycle history and raise the stop flag when every rhs is below tol (the
// reference's `relnorm.max() < tol`, gmres.py:222-224; a NaN never converges).
// ctl[0]: stop flag, ctl[1]: steps completed in this cycle.
__global__ void gmres_record_kernel(int j, int b, const double* __restrict__ relnorm, double tol, int fixed,
                                    double* hist, int* ctl) {
  if (*static_cast<volatile int*>(ctl) != 0) return;
  __shared__ int all_below;
  if (threadIdx.x == 0) all_below = 1;
  __syncthreads();
  for (int r = threadIdx.x; r < b; r += blockDim.x) {
    const double v = relnorm[r];
    hist[(int64_t)j * b + r] = v;
    if (!(v < tol)) all_below = 0;  // benign race: every writer stores 0
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl[1] = j + 1;
    if (!fixed && all_below) ctl[0] = 1;
  }
}

namespace {
struct StopScope {  // routes the hop launchers' stop flag for the calls in scope
  explicit StopScope(const int* f) { g_hop_stop = f; }
  ~StopScope() { g_hop_stop = nullptr; }
};
}  // namespace

extern "C" int b200wd_gmres_cycle(const b200wd_gmres_state* st, const b200wd_operator* op, int32_t m_run,
                                  int64_t n_sites, const void* const* z, double tol, int32_t fixed, void* ctl_dev,
                                  void* hist_dev, int32_t* ctl_host, double* hist_host, void* stream) {
  CHECK_STATE(st);
  B200WD_REQUIRE(op != nullptr && z != nullptr && ctl_dev && hist_dev && ctl_host && hist_host, "NULL pointer");
  B200WD_REQUIRE(1 <= m_run && m_run <= st->m, "cycle length %d outside [1, %d]", m_run, st->m);
  B200WD_REQUIRE(op->dtype == B200WD_C128, "the device GMRES runs in complex128");
  const int32_t s = 12;
  CHECK_FIELD(n_sites, s, st->b);
  for (int p = 0; p <= m_run; ++p) B200WD_REQUIRE(z[p] != nullptr, "basis pointer %d is NULL", p);
  cudaStream_t cs = as_stream(stream);
  int* ctl = static_cast<int*>(ctl_dev);
  double* hist = static_cast<double*>(hist_dev);
  if (cudaMemsetAsync(ctl, 0, 2 * sizeof(int), cs) != cudaSuccess) return check_launch("b200wd_gmres_cycle");
  {
    StopScope scope(ctl);
    for (int j = 0; j < m_run; ++j) {
      void* w = const_cast<void*>(z[j + 1]);
      const double* sig = static_cast<const double*>(st->sigma) + (int64_t)j * st->b;
      if (int rc = b200wd_operator_apply(op, st->b, z[j], w, sig, stream)) return rc;
      if (!sweep_single_launch(st, j, n_sites, s, z, w, stream)) {
        // the per-pass kernels carry no stop flag: this path needs the
        // cooperative sweep (the caller falls back to per-step calls)
        if (j == 0) {
          set_error("b200wd_gmres_cycle: cooperative sweep unavailable");
          return B200WD_ERR_UNSUPPORTED;
        }
        set_error("b200wd_gmres_cycle: cooperative sweep failed at step %d", j);
        return B200WD_ERR_CUDA;
      }
      gmres_record_kernel<<<1, 128, 0, cs>>>(j, st->b, static_cast<const double*>(st->relnorm), tol, fixed, hist,
                                             ctl);
      if (int rc = check_launch("b200wd_gmres_cycle")) return rc;
    }
  }
  cudaError_t e = cudaMemcpyAsync(ctl_host, ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hist_host, hist, sizeof(double) * m_run * st->b, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) {
    set_error("b200wd_gmres_cycle: %s", cudaGetErrorString(e));
    return B200WD_ERR_CUDA;
  }
  return B200WD_OK;
}
