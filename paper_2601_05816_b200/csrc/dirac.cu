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
#include "dirac_kernels.cuh"

namespace b200wd {

// Stop flag of the GMRES cycle being enqueued on this thread (b200wd_gmres_cycle
// sets it around its operator applications); nullptr everywhere else.
thread_local const int* g_hop_stop = nullptr;
thread_local int g_sm_reserve = 0;

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
  p.stop = g_hop_stop;
  return B200WD_OK;
}

}  // namespace b200wd

using namespace b200wd;

extern "C" int b200wd_set_sm_reserve(int32_t sm_reserve) {
  const int prev = g_sm_reserve;
  g_sm_reserve = sm_reserve < 0 ? 0 : sm_reserve;
  return prev;
}

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
  if (dtype == B200WD_C128) launch_hop_c128(p, st);
  else launch_hop_c64(p, st);
  return check_launch("b200wd_hop");
}

extern "C" int b200wd_hop_clover(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
                                 const void* links, const void* src, const void* xself, void* out, double alpha,
                                 double beta, const double* scale, int32_t t_begin, int32_t t_end,
                                 const void* lam_halo, const void* chi_halo, const void* clover, int32_t clover_mode,
                                 void* stream) {
  HopParams p;
  if (int rc = fill_params(p, lat, dtype, b, dst_parity)) return rc;
  B200WD_REQUIRE(links && src && out, "NULL field pointer");
  B200WD_REQUIRE(clover_mode >= 0 && clover_mode <= 2, "clover_mode must be 0, 1 or 2 (got %d)", clover_mode);
  B200WD_REQUIRE(clover_mode == 0 || clover != nullptr, "clover_mode %d needs a clover array", clover_mode);
  B200WD_REQUIRE(0 <= t_begin && t_begin <= t_end && t_end <= p.T, "slice range [%d,%d) outside [0,%d)", t_begin,
                 t_end, p.T);
  B200WD_REQUIRE((lam_halo == nullptr) == (chi_halo == nullptr), "lam_halo and chi_halo must both be set or NULL");
  if (t_begin == t_end) return B200WD_OK;
  p.U = links;
  p.src = src;
  p.xself = xself;
  p.out = out;
  p.alpha = alpha;
  p.beta = 0.5 * beta;
  p.scale = scale;
  p.lam_halo = lam_halo;
  p.chi_halo = chi_halo;
  p.clov = clover;
  p.clov_mode = clover_mode;
  const int64_t per = dst_parity < 0 ? p.per_t : p.per_t / 2;
  p.d_begin = per * t_begin;
  p.d_end = per * t_end;
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) launch_hop_c128(p, st);
  else launch_hop_c64(p, st);
  return check_launch("b200wd_hop_clover");
}

extern "C" int b200wd_hop_boundary(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
                                   const void* links, const void* src, const void* xself, void* out, double alpha,
                                   double beta, const double* scale, const void* lam_halo, const void* chi_halo,
                                   const void* clover, int32_t clover_mode, void* stream) {
  HopParams p;
  if (int rc = fill_params(p, lat, dtype, b, dst_parity)) return rc;
  B200WD_REQUIRE(links && src && out, "NULL field pointer");
  B200WD_REQUIRE(lam_halo && chi_halo, "the boundary slices need both halo faces");
  B200WD_REQUIRE(clover_mode >= 0 && clover_mode <= 2, "clover_mode must be 0, 1 or 2 (got %d)", clover_mode);
  B200WD_REQUIRE(clover_mode == 0 || clover != nullptr, "clover_mode %d needs a clover array", clover_mode);
  p.U = links;
  p.src = src;
  p.xself = xself;
  p.out = out;
  p.alpha = alpha;
  p.beta = 0.5 * beta;
  p.scale = scale;
  p.lam_halo = lam_halo;
  p.chi_halo = chi_halo;
  p.clov = clover;
  p.clov_mode = clover_mode;
  const int64_t per = dst_parity < 0 ? p.per_t : p.per_t / 2;
  p.d_begin = 0;
  p.d_end = 2 * per;  // slice 0 and slice T-1 (contiguous when T == 2)
  if (p.T > 2) {
    p.jump_at = per;
    p.jump_by = (int64_t)(p.T - 2) * per;
  }
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) launch_hop_c128(p, st);
  else launch_hop_c64(p, st);
  return check_launch("b200wd_hop_boundary");
}

extern "C" int b200wd_clover_apply(int64_t n_sites, int32_t dtype, int32_t b, const void* blocks, const void* x,
                                   void* out, void* stream) {
  B200WD_REQUIRE(n_sites >= 8 && n_sites % 8 == 0, "site count %lld must be a positive multiple of 8",
                 (long long)n_sites);
  B200WD_REQUIRE(b >= 1 && blocks && x && out, "bad clover_apply arguments");
  cudaStream_t st = as_stream(stream);
  if (dtype == B200WD_C128) launch_clover_apply_c128(n_sites, b, blocks, x, out, st);
  else if (dtype == B200WD_C64) launch_clover_apply_c64(n_sites, b, blocks, x, out, st);
  else B200WD_REQUIRE(false, "unknown dtype %d", dtype);
  return check_launch("b200wd_clover_apply");
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
  if (dtype == B200WD_C128) launch_pack_c128(p, lam_face, chi_face, st);
  else launch_pack_c64(p, lam_face, chi_face, st);
  return check_launch("b200wd_halo_pack");
}

extern "C" int b200wd_operator_apply(const b200wd_operator* op, int32_t b, const void* in, void* out,
                                     const double* scale, void* stream) {
  B200WD_REQUIRE(op != nullptr, "operator descriptor is NULL");
  B200WD_REQUIRE(op->n_stages >= 1 && op->n_stages <= B200WD_MAX_STAGES, "operator has %d stages (1..%d)",
                 op->n_stages, B200WD_MAX_STAGES);
  B200WD_REQUIRE(in && out, "NULL field pointer");
  for (int i = 0; i < op->n_stages; ++i) {
    const b200wd_hop_stage& g = op->stage[i];
    const void* opnd[4] = {nullptr, in, out, op->tmp};
    B200WD_REQUIRE(g.src >= 1 && g.src <= 3 && g.out >= 1 && g.out <= 3 && g.xself >= 0 && g.xself <= 3,
                   "stage %d: operand codes src=%d xself=%d out=%d", i, g.src, g.xself, g.out);
    B200WD_REQUIRE(g.out != B200WD_OPND_IN, "stage %d writes the operator input", i);
    B200WD_REQUIRE((g.src != B200WD_OPND_TMP && g.out != B200WD_OPND_TMP && g.xself != B200WD_OPND_TMP) ||
                       op->tmp != nullptr,
                   "stage %d uses the scratch field but tmp is NULL", i);
    if (int rc = b200wd_hop_clover(&op->lat, op->dtype, b, g.dst_parity, op->links, opnd[g.src], opnd[g.xself],
                                   const_cast<void*>(opnd[g.out]), g.alpha, g.beta, g.use_scale ? scale : nullptr,
                                   0, op->lat.dims[0], nullptr, nullptr, g.clover, g.clover_mode, stream))
      return rc;
  }
  return B200WD_OK;
}
