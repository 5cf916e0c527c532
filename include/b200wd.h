/*
 * libb200wd -- B200 (sm_100a) rhs-blocked Wilson-Dirac operator and batched
 * GMRES kernels behind a plain C ABI.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * lqcdlab 0.1.0 (/root/reference/pkg/src/lqcdlab).  The reference is pure
 * Python/numpy and has no FFI of its own; every entry point below replaces
 * the reference function cited beside it, and the Python package
 * paper_2601_05816_b200 binds them with ctypes (INTEGRATION.md shows the
 * binding a maintainer would add to lqcdlab itself).
 *
 * Conventions
 *  - All data pointers are DEVICE pointers owned by the caller (the library
 *    never allocates on the hot path).  `stream` is a cudaStream_t passed as
 *    void*; NULL means the legacy default stream.  Calls are stream-ordered
 *    and asynchronous: no hidden device synchronisation.
 *  - Return 0 on success or a B200WD_ERR_* code; b200wd_last_error() then
 *    returns a message (thread-local).  No C++ exception crosses the ABI.
 *  - dtype: B200WD_C128 (complex128, double2) or B200WD_C64 (complex64,
 *    float2).  Scalars are always passed as double.
 *  - Device spinor layout ("site-blocked component planes", n % 8 == 0):
 *    element (site, k, r) of a field with s components and b right-hand
 *    sides lives at (((site>>3)*s + k)*8 + (site&7))*b + r, i.e. blocks of 8
 *    sites in which component k of the 8 sites is one contiguous run of 8*b
 *    complex numbers.  rhs is innermost, so a warp's loads of one component
 *    over consecutive (site, rhs) pairs are contiguous.  Parity
 *    (checkerboard) fields use n/2 sites indexed by cb = site >> 1, which
 *    equals the reference's ascending-natural-order parity numbering
 *    (oddeven.py:62-65) because the fastest extent is even.
 *  - Device link layout, direction-major: element (site, mu, e=3*row+col)
 *    at ((mu*(n/8) + (site>>3))*9 + e)*8 + (site&7).
 *  - Clover blocks: 2 x 21 packed complex per site, element (site, q) at
 *    ((site>>3)*42 + q)*8 + (site&7).
 *  - Lattice: extents (T,X,Y,Z) = dims[0..3], site = ((t*X+x)*Y+y)*Z+z,
 *    T slowest (geometry.py:1-11).  Time is direction 0.
 */
#ifndef B200WD_H
#define B200WD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B200WD_ABI_VERSION 3

#define B200WD_OK 0
#define B200WD_ERR_ARG 1         /* bad shape / layout / parameter -> ValueError      */
#define B200WD_ERR_CUDA 2        /* CUDA runtime or launch failure -> RuntimeError    */
#define B200WD_ERR_SINGULAR 3    /* singular eliminated block -> SingularBlockError   */
#define B200WD_ERR_UNSUPPORTED 4 /* combination not implemented -> NotImplementedError */

#define B200WD_C128 0
#define B200WD_C64 1

/* Local lattice of one rank.  With a T-only split over R ranks, dims[0] is
 * the local T extent; t_origin is the global T coordinate of local slice 0
 * (even, so local and global parity agree). */
typedef struct b200wd_lattice {
  int32_t dims[4];
  int32_t t_origin;
  int32_t reserved;
} b200wd_lattice;

/* ---- library ------------------------------------------------------------ */
int b200wd_abi_version(void);
const char* b200wd_last_error(void);
/* Device properties the host needs for launch sizing (SM count, L2 bytes). */
int b200wd_device_info(int device, int32_t* sm_count, int64_t* l2_bytes, int32_t* cc_major,
                       int32_t* cc_minor);
/* SMs left free by the persistent (one-CTA-per-SM ring / stream) hop kernels
 * launched from the calling thread: with sm_reserve = k their grid covers
 * sm_count - k SMs, so kernels enqueued concurrently on other streams (NCCL's
 * P2P halo exchange, halo.py:339-387's overlap) find resident room.  0 (the
 * default) uses every SM.  Returns the previous value. */
int b200wd_set_sm_reserve(int32_t sm_reserve);

/* ---- layouts (fields.py:48-137, 156-161) -------------------------------- */
/* Reference storage (complex128, Layout 1 rhs-major or 2 component-major,
 * fields.py:53-64), already copied to the device, -> device component
 * planes of `dtype`.  Replaces BlockSpinorField.ksi()/convert(). */
int b200wd_spinor_import(const void* src_c128, int32_t layout, int64_t n_sites, int32_t s,
                         int32_t b, void* dst, int32_t dtype, void* stream);
/* Inverse of b200wd_spinor_import (device planes -> reference storage). */
int b200wd_spinor_export(const void* src, int32_t dtype, int64_t n_sites, int32_t s, int32_t b,
                         void* dst_c128, int32_t layout, void* stream);
/* GaugeField.data (n,4,3,3) complex128 row-major (fields.py:156-161) ->
 * device link planes of `dtype`. */
int b200wd_gauge_import(const void* src_c128, int64_t n_sites, void* dst, int32_t dtype,
                        void* stream);
/* CloverField.data (n,2,21) complex128 packed blocks (fields.py:212-247) ->
 * device site-blocked blocks: element (site, q) at ((site>>3)*42 + q)*8 +
 * (site&7).  Also used for the packed inverse blocks of the Schur operator. */
int b200wd_clover_import(const void* src_c128, int64_t n_sites, void* dst, int32_t dtype,
                         void* stream);
/* Full-lattice planes <-> (even, odd) parity planes; replaces split_fields /
 * merge_fields (oddeven.py:72-95). */
int b200wd_parity_split(const b200wd_lattice* lat, int32_t dtype, int32_t s, int32_t b,
                        const void* full, void* even, void* odd, void* stream);
int b200wd_parity_merge(const b200wd_lattice* lat, int32_t dtype, int32_t s, int32_t b,
                        const void* even, const void* odd, void* full, void* stream);

/* ---- Wilson-Dirac operator (dirac.py:137-334) --------------------------- */
/* Generic fused hopping kernel:
 *   out = scale[r] * ( alpha * xself + beta * H src )
 * with H src(x) = sum_mu [ P-_mu U_mu(x) src(x+mu) + P+_mu U_mu(x-mu)^H src(x-mu) ]
 * (P-+ = (I +- gamma_mu)/2 as in dirac.py:172-263 / oracle.py:60-61).
 *   dst_parity = -1 : full lattice, src/xself/out have n sites.
 *   dst_parity = 0|1: out/xself are parity-p fields, src is the parity 1-p
 *                     field (D_eo / D_oe blocks, oddeven.py:146-156).
 *   xself may be NULL (then alpha is ignored); scale may be NULL (= 1), else
 *   it is a device array of b doubles.
 *   Only local slices t_begin <= t < t_end are written.
 *   lam_halo / chi_halo: NULL -> T is periodic inside this lattice (single
 *   rank).  Otherwise the forward T neighbour of slice dims[0]-1 comes from
 *   lam_halo and the backward T neighbour of slice 0 from chi_halo, in the
 *   face layout of b200wd_halo_pack (halo.py:370-387). */
int b200wd_hop(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
               const void* links, const void* src, const void* xself, void* out, double alpha,
               double beta, const double* scale, int32_t t_begin, int32_t t_end,
               const void* lam_halo, const void* chi_halo, void* stream);

/* b200wd_hop plus a site-local term (the clover, dirac.py:137-157, or the
 * inverse of the eliminated diagonal blocks, oddeven.py:123-144): `clover`
 * holds two packed Hermitian 6x6 blocks (21 complex each, lower triangle
 * row-major as CloverField.data, fields.py:212-247) per dst site, imported
 * with b200wd_clover_import.
 *   clover_mode 0: as b200wd_hop
 *   clover_mode 1: out = scale (alpha xself - M xself + beta H src)
 *   clover_mode 2: out = scale  M (alpha xself + beta H src)              */
int b200wd_hop_clover(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
                      const void* links, const void* src, const void* xself, void* out, double alpha,
                      double beta, const double* scale, int32_t t_begin, int32_t t_end,
                      const void* lam_halo, const void* chi_halo, const void* clover,
                      int32_t clover_mode, void* stream);
/* Both T-split boundary slices (local slices 0 and T-1) consuming the halo
 * faces in ONE launch (halo.py:370-387): the same arithmetic as two
 * b200wd_hop(_clover) calls with t ranges [0,1) and [T-1,T); clover may be
 * NULL (clover_mode 0). */
int b200wd_hop_boundary(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t dst_parity,
                        const void* links, const void* src, const void* xself, void* out, double alpha,
                        double beta, const double* scale, const void* lam_halo, const void* chi_halo,
                        const void* clover, int32_t clover_mode, void* stream);
/* out = M x, site-local (D_oo^-1 eta_o of reduce_rhs, oddeven.py:179-188). */
int b200wd_clover_apply(int64_t n_sites, int32_t dtype, int32_t b, const void* blocks,
                        const void* x, void* out, void* stream);

/* eta = D psi = (4+m0) psi - H psi on the full (single-rank) lattice with
 * C = 0; replaces apply_dirac (dirac.py:299-334). */
int b200wd_dirac_apply(const b200wd_lattice* lat, int32_t dtype, int32_t b, double m0,
                       const void* links, const void* psi, void* eta, void* stream);

/* Face messages of the T split (halo.py:352-368): lam_face = sign -1 half
 * spinor of local slice 0 (sent to rank-1), chi_face = U_0^H times the sign
 * +1 half spinor of slice dims[0]-1 (sent to rank+1).  Face layout: element
 * (h = 3*spin+colour in 0..5, i, r) at ((h*nf + i)*b + r), nf = face sites
 * (X*Y*Z, or half of it for a parity field); both faces carry a factor 2
 * relative to the reference's half spinors.  src_parity = -1 for a
 * full-lattice field, else the parity of the field `src`. */
int b200wd_halo_pack(const b200wd_lattice* lat, int32_t dtype, int32_t b, int32_t src_parity,
                     const void* links, const void* src, void* lam_face, void* chi_face,
                     void* stream);

/* ---- per-rhs BLAS (blas.py:50-110), complex128 planes -------------------- */
/* Bytes of reduction scratch needed by the reducing calls below. */
int64_t b200wd_reduce_scratch_bytes(int32_t b);
/* out[r] = sum conj(x) y over the field (b complex128, device). */
int b200wd_block_dot(int64_t n_sites, int32_t s, int32_t b, const void* x, const void* y,
                     void* out, void* scratch, void* stream);
/* out[r] = ||x_r||^2 (b doubles stored as the .x of b complex128). */
int b200wd_block_norm2(int64_t n_sites, int32_t s, int32_t b, const void* x, void* out,
                       void* scratch, void* stream);
/* y += alpha[r] x (alpha: b complex128 on the device). */
int b200wd_block_axpy(int64_t n_sites, int32_t s, int32_t b, const void* alpha, const void* x,
                      void* y, void* stream);
/* x *= alpha[r]. */
int b200wd_block_scale(int64_t n_sites, int32_t s, int32_t b, const void* alpha, void* x,
                       void* stream);

/* ---- batched GMRES Arnoldi kernels (gmres.py:101-251) -------------------- */
/* Device-resident solver state; every pointer is caller-owned device memory.
 * The basis is stored unnormalised: V_p = sigma[r][p] * Z_p. */
typedef struct b200wd_gmres_state {
  int32_t b, m;          /* rhs count, restart length                          */
  double breakdown_rel;  /* gmres.py:56                                         */
  void* h_raw;           /* complex128 [b][m+1][m]   pre-rotation Hessenberg    */
  void* h;               /* complex128 [b][m+1][m]   rotated                    */
  void* gamma;           /* complex128 [b][m+1]                                 */
  void* cs;              /* double     [b][m]                                   */
  void* sn;              /* complex128 [b][m]                                   */
  void* sigma;           /* double     [m+1][b]  (row p = scale of Z_p per rhs) */
  void* eta_norm;        /* double     [b]                                      */
  void* relnorm;         /* double     [b]                                      */
  void* breakdown;       /* int32      [b]                                      */
  void* dot;             /* complex128 [b]  result of the last reducing pass    */
  void* y;               /* complex128 [b][m] least-squares solution            */
  void* scratch;         /* b200wd_reduce_scratch_bytes(b) bytes                */
  /* B200 extension (not in the reference): Gram-Schmidt variant of the
   * library-issued Arnoldi step.  B200WD_ORTH_MGS (0, zero-initialised
   * default) is the reference's modified Gram-Schmidt (gmres.py:118-121);
   * B200WD_ORTH_CGS (1) is classical Gram-Schmidt: all j+1 projections in one
   * pass over the basis, then one update pass that also forms ||w||^2 -- about
   * half the HBM traffic of MGS, orthogonality loss O(eps kappa^2) instead of
   * O(eps kappa).  CGS needs the cooperative sweep (single rank) and
   * cgs_partials (b200wd_cgs_scratch_bytes(b, m) bytes). */
  int32_t orth;
  void* cgs_partials;
} b200wd_gmres_state;

#define B200WD_ORTH_MGS 0
#define B200WD_ORTH_CGS 1

/* Bytes of b200wd_gmres_state.cgs_partials for b rhs and restart length m. */
int64_t b200wd_cgs_scratch_bytes(int32_t b, int32_t m);

/* eta_norm := sqrt(dot) (dot = ||eta||^2 from b200wd_block_norm2 into
 * st->dot, all-reduced), breakdown flags cleared (gmres.py:204-205). */
int b200wd_gmres_init(const b200wd_gmres_state* st, void* stream);
/* r := eta - r (r holds A psi on entry), and dot := ||r||^2 (partial sum of
 * this rank; all-reduce `dot` across ranks before the next call). */
int b200wd_gmres_residual(const b200wd_gmres_state* st, int64_t n_sites, int32_t s,
                          const void* eta, void* r, void* stream);
/* Cycle start from dot = ||r||^2 (gmres.py:180-198): gamma = beta e1,
 * sigma_0 = 1/beta (0 if beta = 0), rotations cleared, relnorm. */
int b200wd_gmres_start(const b200wd_gmres_state* st, void* stream);
/* dot := <Z_p, w> (opens the MGS sweep of column j). */
int b200wd_gmres_dot(const b200wd_gmres_state* st, int64_t n_sites, int32_t s, const void* z,
                     const void* w, void* stream);
/* One fused MGS pass (gmres.py:118-121): with dot = <Z_p, w>,
 * h_raw[p][j] = sigma_p dot, w -= sigma_p^2 dot Z_p, then
 * dot := <Z_next, w> (z_next != NULL) or ||w||^2 (z_next == NULL). */
int b200wd_gmres_mgs(const b200wd_gmres_state* st, int32_t j, int32_t p, int64_t n_sites,
                     int32_t s, void* w, const void* z_p, const void* z_next, void* stream);
/* Close column j from dot = ||w||^2 (gmres.py:135-157): breakdown test,
 * h_raw[j+1][j], sigma_{j+1}, stored rotations, new Givens pair, gamma,
 * relnorm. */
int b200wd_gmres_close_column(const b200wd_gmres_state* st, int32_t j, void* stream);
/* y = back substitution (gmres.py:161-177), then
 * psi += sum_{p<j_done} y_p sigma_p Z_p in one pass (gmres.py:226-229). */
int b200wd_gmres_update(const b200wd_gmres_state* st, int32_t j_done, int64_t n_sites,
                        int32_t s, const void* const* z, void* psi, void* stream);

/* ---- operator programs and the native Arnoldi step ---------------------- */
/* A linear operator as a short program of hop stages, so the library can
 * apply it without a round trip through the host language (the reference's
 * operator callables, gmres.py:335-339 dirac_op and oddeven.py:165-174).  Each stage is one
 * b200wd_hop_clover launch over all local slices; its src / xself / out are
 * picked from the call's input (B200WD_OPND_IN), output (B200WD_OPND_OUT) or
 * the program's scratch field `tmp` (B200WD_OPND_TMP).  The call's `scale`
 * array goes to the stages with use_scale = 1.
 *   full D_W (dirac.py:266-305):      1 stage, dst_parity -1,
 *                                     src = xself = IN, out = OUT
 *   Schur S = D_kk - D_ke D_ee^-1 D_ek (oddeven.py:165-174):
 *                                     stage 0 dst = elim parity, IN -> TMP
 *                                     stage 1 dst = keep parity, TMP -> OUT,
 *                                             xself = IN                    */
#define B200WD_OPND_NONE 0
#define B200WD_OPND_IN 1
#define B200WD_OPND_OUT 2
#define B200WD_OPND_TMP 3
#define B200WD_MAX_STAGES 4

typedef struct b200wd_hop_stage {
  int32_t dst_parity;   /* -1 full lattice, 0|1 checkerboard                   */
  int32_t src, xself, out; /* B200WD_OPND_*                                    */
  double alpha, beta;   /* as b200wd_hop_clover                                 */
  const void* clover;   /* packed blocks or NULL                                */
  int32_t clover_mode;  /* 0, 1, 2 as b200wd_hop_clover                         */
  int32_t use_scale;    /* 1: multiply by the call's scale[b]                   */
} b200wd_hop_stage;

typedef struct b200wd_operator {
  b200wd_lattice lat;
  int32_t dtype;
  int32_t n_stages;     /* 1 .. B200WD_MAX_STAGES                               */
  const void* links;
  void* tmp;            /* scratch field for B200WD_OPND_TMP (or NULL)          */
  b200wd_hop_stage stage[B200WD_MAX_STAGES];
} b200wd_operator;

/* out = op(in) (scale: device array of b doubles or NULL). */
int b200wd_operator_apply(const b200wd_operator* op, int32_t b, const void* in, void* out,
                          const double* scale, void* stream);

/* One whole Arnoldi step of column j on a single rank (gmres.py:115-157):
 * Z_{j+1} = sigma_j op(Z_j), the fused MGS sweep against Z_0..Z_j, the column
 * close (breakdown test, Givens rotation, relnorm), then the relnorm of every
 * rhs is copied into relnorm_host (b doubles, pinned host memory) and the
 * stream is synchronised, so the caller can run the reference's stop test.
 * Equivalent to b200wd_operator_apply + b200wd_gmres_dot + (j+1) x
 * b200wd_gmres_mgs + b200wd_gmres_close_column, issued from native code.
 * relnorm_host may be NULL (no copy, no synchronisation). */
int b200wd_gmres_arnoldi(const b200wd_gmres_state* st, const b200wd_operator* op, int32_t j,
                         int64_t n_sites, const void* const* z, double* relnorm_host,
                         void* stream);

/* A whole restart cycle of Arnoldi steps (gmres.py:218-224) enqueued with no
 * host round trip: steps j = 0 .. m_run-1 as in b200wd_gmres_arnoldi, each
 * followed by a record kernel that stores the b relnorms in row j of
 * hist_dev (double [m_run][b]) and sets ctl_dev[0] (int) once every rhs is
 * below tol (never when fixed != 0); kernels of later steps see the flag and
 * do nothing.  ctl_dev[1] = steps completed.  One synchronisation at the end
 * copies ctl_dev (2 ints) and the used rows of hist_dev to ctl_host /
 * hist_host.  Same kernels in the same order as the per-step call, so the
 * results are bit-identical.  B200WD_ERR_UNSUPPORTED if the cooperative
 * sweep cannot be launched (use b200wd_gmres_arnoldi). */
int b200wd_gmres_cycle(const b200wd_gmres_state* st, const b200wd_operator* op, int32_t m_run,
                       int64_t n_sites, const void* const* z, double tol, int32_t fixed, void* ctl_dev,
                       void* hist_dev, int32_t* ctl_host, double* hist_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200WD_H */
