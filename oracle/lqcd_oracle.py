"""CPU oracle for the rhs-blocked Wilson-Dirac path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product package
(``paper_2601_05816_b200``) never imports anything from ``oracle/``.

It is a numpy restatement of the reference algorithm (``lqcdlab`` 0.1.0,
``/root/reference/pkg/src/lqcdlab``); every function cites the reference
file:line it follows.  All arrays use the *logical* view of a block field:
``(n_sites, s, b)`` complex, i.e. ``[site, component, rhs]`` where component
``k = 3*spin + colour``.  Links are ``(n_sites, 4, 3, 3)`` row-major.

Parity pinning: ``tests/test_oracle.py`` checks this module against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py``) -- operator outputs, Schur outputs, GMRES
iteration counts and residual histories, generator checksums -- and against
the reference's own known-answer identities (free field, Schur constant
factor, dense-matrix equality).

Harness additions the reference lacks:
``near_unit_gauge`` (U = exp(i eps H)), ``flip_time_boundary`` (antiperiodic T
as a link sign flip on the last T slice, verified equal to explicit boundary
signs) and complex64 rounding helpers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NDIM = 4
NSPIN = 4
NCOL = 3
NSC = 12          # spinor components per site
NHALF = 6         # half-spinor components

# ---------------------------------------------------------------------------
# geometry  (reference geometry.py:26-123)
# ---------------------------------------------------------------------------


def check_dims(dims) -> tuple:
    """Extents must be 4 even numbers >= 2 (geometry.py:40-45)."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != NDIM:
        raise ValueError(f"expected {NDIM} extents, got {len(dims)}")
    for d, n in enumerate(dims):
        if n < 2 or n % 2:
            raise ValueError(f"extent {n} in direction {d} is not an even number >= 2")
    return dims


def site_coords(dims) -> np.ndarray:
    """(n,4) coordinates in mixed-radix order, x3 fastest (geometry.py:1-11, 89-93)."""
    grids = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1)


def site_index_of(dims, coords: np.ndarray) -> np.ndarray:
    """Vectorised mixed-radix index (geometry.py:51-59, 100-105)."""
    idx = np.zeros(len(coords), dtype=np.int64)
    for d in range(NDIM):
        idx = idx * dims[d] + coords[:, d]
    return idx


def neighbor_table(dims, mu: int, step: int) -> np.ndarray:
    """Periodic neighbour permutation (geometry.py:107-115)."""
    c = site_coords(dims)
    c[:, mu] = (c[:, mu] + step) % dims[mu]
    return site_index_of(dims, c)


def parities(dims) -> np.ndarray:
    """(x0+x1+x2+x3) mod 2 (geometry.py:70-72, 95-98)."""
    return site_coords(dims).sum(axis=1) % 2


def parity_sites(dims, parity: int) -> np.ndarray:
    """Ascending natural indices of one parity (geometry.py:117-123)."""
    return np.nonzero(parities(dims) == parity)[0]


# ---------------------------------------------------------------------------
# generators (reference fields.py:43-45, 140-153, 185-205, 253-263)
# ---------------------------------------------------------------------------


def make_rng(seed: int) -> np.random.Generator:
    """Seeded PCG64 stream (fields.py:43-45)."""
    return np.random.Generator(np.random.PCG64(seed))


def gen_spinor(n_sites: int, b: int, seed: int, s: int = NSC) -> np.ndarray:
    """Gaussian block field, logical (n,s,b) view (fields.py:140-153).

    Real and imaginary parts are both N(0,1) (variance 1 each, not 1/2).
    """
    rng = make_rng(seed)
    shape = (n_sites, s, b)
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    return re + 1j * im


def gen_gauge_random(dims, seed: int) -> np.ndarray:
    """Random SU(3) links by QR of a complex Gaussian (fields.py:185-205).

    Steps: Gaussian matrix -> QR -> rotate columns so diag(R) is positive
    real -> push the determinant phase into the first column.
    """
    n = math.prod(dims)
    rng = make_rng(seed)
    shape = (n, NDIM, 3, 3)
    g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    q, r = np.linalg.qr(g)
    rd = np.einsum("...ii->...i", r)
    q = q * (rd.conj() / np.abs(rd))[..., None, :]
    det = np.linalg.det(q)
    q[..., :, 0] *= det.conj()[..., None]
    return np.ascontiguousarray(q)


def gen_gauge_unit(dims) -> np.ndarray:
    """Identity links (fields.py:163-167)."""
    n = math.prod(dims)
    u = np.zeros((n, NDIM, 3, 3), dtype=np.complex128)
    u[..., np.arange(3), np.arange(3)] = 1.0
    return u


def near_unit_gauge(dims, eps: float, seed: int) -> np.ndarray:
    """Harness generator (BASELINE configs 3-5): U = exp(i eps H).

    H is the traceless Hermitian part of a complex Gaussian 3x3 matrix; the
    exponential is formed from the eigendecomposition so det U = 1 exactly in
    exact arithmetic.  The random stream is drawn one T slice at a time from
    ``PCG64(SeedSequence([seed, t]))`` so that any T slab of the lattice can
    be generated independently (the multi-GPU T split generates only its own
    slab); the result does not depend on how the lattice is split.
    """
    dims = check_dims(dims)
    per_t = math.prod(dims[1:])
    out = np.empty((dims[0] * per_t, NDIM, 3, 3), dtype=np.complex128)
    for t in range(dims[0]):
        out[t * per_t:(t + 1) * per_t] = near_unit_slab(dims, eps, seed, t)
    return out


def near_unit_slab(dims, eps: float, seed: int, t: int) -> np.ndarray:
    """Links of one T slice of :func:`near_unit_gauge`."""
    per_t = math.prod(dims[1:])
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, t])))
    shape = (per_t, NDIM, 3, 3)
    g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    h = 0.5 * (g + np.conj(np.swapaxes(g, -1, -2)))
    tr = np.einsum("...ii->...", h).real / 3.0
    h[..., np.arange(3), np.arange(3)] -= tr[..., None]
    w, v = np.linalg.eigh(h)
    ph = np.exp(1j * eps * w)
    return np.einsum("...ij,...j,...kj->...ik", v, ph, np.conj(v))


def flip_time_boundary(links: np.ndarray, dims) -> np.ndarray:
    """Antiperiodic T: negate U_0 on the last T slice.

    Direction 0 (the slowest index) is time.  Returns a new array.
    """
    out = links.copy()
    per_t = math.prod(dims[1:])
    out[(dims[0] - 1) * per_t:, 0] *= -1.0
    return out


def gen_clover_random(dims, scale: float, seed: int) -> np.ndarray:
    """Hermitian 6x6 blocks, (n,2,6,6) unpacked (fields.py:253-263)."""
    n = math.prod(dims)
    rng = make_rng(seed)
    shape = (n, 2, 6, 6)
    g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    blocks = scale * 0.5 * (g + np.conj(np.swapaxes(g, -1, -2)))
    # the reference packs the lower triangle with a real diagonal
    # (fields.py:228-238) and unpacks it again (fields.py:240-247)
    return unpack_clover(pack_clover(blocks))


def pack_clover(blocks: np.ndarray) -> np.ndarray:
    """(n,2,6,6) -> (n,2,21) packed lower triangle, real diagonal (fields.py:228-238)."""
    rows, cols = np.tril_indices(6)
    packed = blocks[..., rows, cols].copy()
    diag = rows == cols
    packed[..., diag] = packed[..., diag].real
    return packed


def unpack_clover(packed: np.ndarray) -> np.ndarray:
    """(n,2,21) -> (n,2,6,6) Hermitian (fields.py:240-247)."""
    rows, cols = np.tril_indices(6)
    out = np.zeros(packed.shape[:-1] + (6, 6), dtype=np.complex128)
    out[..., rows, cols] = packed
    strict = rows != cols
    out[..., cols[strict], rows[strict]] = np.conj(packed[..., strict])
    return out


def round_c64(a: np.ndarray) -> np.ndarray:
    """complex128 -> complex64 -> complex128 (the c64 parity inputs)."""
    return a.astype(np.complex64).astype(np.complex128)


# ---------------------------------------------------------------------------
# storage layouts (reference fields.py:48-64, 105-137)
# ---------------------------------------------------------------------------


def to_storage(logical: np.ndarray, layout: int) -> np.ndarray:
    """Logical (n,s,b) -> flat storage; 1 = rhs-major, 2 = component-major."""
    if layout == 1:
        return np.ascontiguousarray(logical.transpose(0, 2, 1)).reshape(-1)
    return np.ascontiguousarray(logical).reshape(-1)


def from_storage(flat: np.ndarray, n: int, s: int, b: int, layout: int) -> np.ndarray:
    if layout == 1:
        return flat.reshape(n, b, s).transpose(0, 2, 1).copy()
    return flat.reshape(n, s, b).copy()


def element_offset(layout: int, s: int, b: int, x: int, k: int, i: int) -> int:
    """fields.py:53-64."""
    base = x * s * b
    return base + (i * s + k if layout == 1 else k * b + i)


# ---------------------------------------------------------------------------
# spin projection (reference projectors.py:40-147)
# ---------------------------------------------------------------------------

# A_mu blocks of the chiral gamma basis (projectors.py:40-48)
A_BLOCKS = np.array(
    [
        [[1, 0], [0, 1]],
        [[0, 1j], [1j, 0]],
        [[0, 1], [-1, 0]],
        [[1j, 0], [0, -1j]],
    ],
    dtype=np.complex128,
)


def gamma_matrices() -> np.ndarray:
    """gamma_mu = [[0, A], [A^H, 0]] (projectors.py:51-55)."""
    g = np.zeros((NDIM, 4, 4), dtype=np.complex128)
    for mu in range(NDIM):
        g[mu, :2, 2:] = A_BLOCKS[mu]
        g[mu, 2:, :2] = A_BLOCKS[mu].conj().T
    return g


def half_project(spin: np.ndarray, mu: int, sign: int) -> np.ndarray:
    """h = (u - sign * A_mu l)/2 on a (..., 4, 3, b) spin view (projectors.py:126-136)."""
    upper = spin[..., :2, :, :]
    lower = spin[..., 2:, :, :]
    a_l = np.einsum("st,...tcb->...scb", A_BLOCKS[mu], lower)
    return 0.5 * (upper - sign * a_l)


def half_expand(half: np.ndarray, mu: int, sign: int) -> np.ndarray:
    """(h, -sign * A_mu^H h) (projectors.py:139-147)."""
    adj = A_BLOCKS[mu].conj().T
    lower = -sign * np.einsum("st,...tcb->...scb", adj, half)
    return np.concatenate([half, lower], axis=-3)


# ---------------------------------------------------------------------------
# Wilson-Dirac apply (reference dirac.py:137-157, 172-296, 299-334)
# ---------------------------------------------------------------------------

FLOPS_PER_SITE_RHS = 2574          # dirac.py:43-48
VALUES_PER_SITE_RHS = 168
VALUES_PER_SITE_FIXED = 114


def self_coupling(m0: float, clover: np.ndarray | None, psi: np.ndarray) -> np.ndarray:
    """eta = (4+m0) psi - C psi with C as two 6x6 blocks (dirac.py:137-157)."""
    eta = (4.0 + m0) * psi
    if clover is not None:
        n, _, b = psi.shape
        halves = psi.reshape(n, 2, 6, b)
        eta = eta - np.einsum("xpkl,xplb->xpkb", clover, halves).reshape(n, NSC, b)
    return eta


def hop_sum(dims, links: np.ndarray, psi: np.ndarray) -> np.ndarray:
    """H psi = sum_mu [P-_mu U_mu(x) psi(x+mu) + P+_mu U_mu(x-mu)^H psi(x-mu)].

    Staged exactly as subtract_hops (dirac.py:273-296): every lambda (forward,
    projector sign -1, dirac.py:172-182) and chi (backward, sign +1, U^H at
    the source site then moved to the destination, dirac.py:185-219) is
    materialised, then reconstructed and accumulated for mu ascending
    (dirac.py:222-263).  D = self_coupling - H.
    """
    n, s, b = psi.shape
    spin = psi.reshape(n, NSPIN, NCOL, b)
    acc = np.zeros((n, NSC, b), dtype=np.complex128)
    lam = [half_project(spin, mu, -1) for mu in range(NDIM)]
    chi = []
    for mu in range(NDIM):
        vals = np.einsum("xdc,xsdb->xscb", np.conj(links[:, mu]), half_project(spin, mu, +1))
        chi.append(vals[neighbor_table(dims, mu, -1)])
    for mu in range(NDIM):
        moved = np.einsum("xcd,xsdb->xscb", links[:, mu], lam[mu][neighbor_table(dims, mu, +1)])
        acc += half_expand(moved, mu, -1).reshape(n, NSC, b)
    for mu in range(NDIM):
        acc += half_expand(chi[mu], mu, +1).reshape(n, NSC, b)
    return acc


def apply_dirac(dims, m0: float, links: np.ndarray, clover: np.ndarray | None, psi: np.ndarray) -> np.ndarray:
    """D psi on logical (n,12,b) fields (dirac.py:299-334)."""
    if psi.shape[1] != NSC:
        raise ValueError(f"expected full spinor field (s={NSC}), got s={psi.shape[1]}")
    if psi.shape[0] != math.prod(dims):
        raise ValueError("field / lattice size mismatch")
    return self_coupling(m0, clover, psi) - hop_sum(dims, links, psi)


def account_traffic(b: int) -> dict:
    """Paper ledger (dirac.py:111-118)."""
    if b < 1:
        raise ValueError(f"b must be >= 1, got {b}")
    return {
        "flops_per_site": FLOPS_PER_SITE_RHS * b,
        "bytes_per_site": (VALUES_PER_SITE_RHS * b + VALUES_PER_SITE_FIXED) * 16,
    }


# ---------------------------------------------------------------------------
# dense oracle (reference oracle.py:36-107)
# ---------------------------------------------------------------------------


def assemble_dirac_dense(dims, m0: float, links: np.ndarray, clover: np.ndarray | None) -> np.ndarray:
    """Explicit (12N,12N) matrix from full 4x4 projectors (oracle.py:36-62)."""
    n = math.prod(dims)
    if NSC * n > 20736:
        raise ValueError("dense operator exceeds the 6^4 guard (oracle.py:28)")
    g = gamma_matrices()
    eye4 = np.eye(4)
    a = np.zeros((NSC * n, NSC * n), dtype=np.complex128)
    for x in range(n):
        r = NSC * x
        a[r:r + 12, r:r + 12] = (4.0 + m0) * np.eye(NSC)
        if clover is not None:
            a[r:r + 6, r:r + 6] -= clover[x, 0]
            a[r + 6:r + 12, r + 6:r + 12] -= clover[x, 1]
    for mu in range(NDIM):
        fwd = neighbor_table(dims, mu, +1)
        bwd = neighbor_table(dims, mu, -1)
        p_minus = (eye4 + g[mu]) / 2
        p_plus = (eye4 - g[mu]) / 2
        for x in range(n):
            r = NSC * x
            a[r:r + 12, NSC * fwd[x]:NSC * fwd[x] + 12] -= np.kron(p_minus, links[x, mu])
            a[r:r + 12, NSC * bwd[x]:NSC * bwd[x] + 12] -= np.kron(p_plus, links[bwd[x], mu].conj().T)
    return a


def columns(logical: np.ndarray) -> np.ndarray:
    """(n*s, b) matrix view (fields.py:132-134)."""
    n, s, b = logical.shape
    return logical.reshape(n * s, b)


# ---------------------------------------------------------------------------
# odd-even Schur complement (reference oddeven.py:51-222)
# ---------------------------------------------------------------------------


class SingularBlockError(np.linalg.LinAlgError):
    """oddeven.py:38-48."""

    def __init__(self, site: int, block: int, cond: float):
        self.site, self.block, self.cond = site, block, cond
        super().__init__(f"site-local block {block} at site {site} is numerically singular "
                         f"(condition estimate {cond:.3e})")


class SchurOracle:
    """S = D_kk - D_ke D_ee^-1 D_ek, parity k kept (oddeven.py:98-201).

    The eliminated diagonal blocks (4+m0) I - C are inverted per site and
    checked against ``cond_limit`` (oddeven.py:123-132); the off-diagonal
    blocks embed a parity field into the full lattice and hop every site
    (oddeven.py:146-156), exactly as the reference does.
    """

    def __init__(self, dims, m0, links, clover=None, keep_parity=0, cond_limit=1e12):
        if keep_parity not in (0, 1):
            raise ValueError(f"parity must be 0 (even) or 1 (odd), got {keep_parity}")
        self.dims = check_dims(dims)
        self.m0, self.links, self.clover = m0, links, clover
        self.keep_parity = keep_parity
        self.keep_sites = parity_sites(self.dims, keep_parity)
        self.elim_sites = parity_sites(self.dims, 1 - keep_parity)
        n_el = len(self.elim_sites)
        blocks = np.broadcast_to((4.0 + m0) * np.eye(6), (n_el, 2, 6, 6)).astype(np.complex128)
        if clover is not None:
            blocks = blocks - clover[self.elim_sites]
        cond = np.linalg.cond(blocks)
        bad = ~np.isfinite(cond) | (cond > cond_limit)
        if bad.any():
            row, half = np.argwhere(bad)[0]
            raise SingularBlockError(int(self.elim_sites[row]), int(half), float(cond[row, half]))
        self._inv = np.linalg.inv(blocks)

    @property
    def n_sites(self) -> int:
        return len(self.keep_sites)

    def solve_eliminated(self, rhs: np.ndarray) -> np.ndarray:
        """D_elim^-1 on (n_elim,12,b) (oddeven.py:138-144)."""
        n, _, b = rhs.shape
        h = rhs.reshape(n, 2, 6, b)
        return np.einsum("xpkl,xplb->xpkb", self._inv, h).reshape(n, NSC, b)

    def _hop_to(self, vals, src, dst):
        """Off-diagonal block: embed, hop all sites, read dst (oddeven.py:146-156)."""
        n = math.prod(self.dims)
        full = np.zeros((n, NSC, vals.shape[2]), dtype=np.complex128)
        full[src] = vals
        return -hop_sum(self.dims, self.links, full)[dst]

    def _diag_keep(self, v):
        """oddeven.py:158-163."""
        cl = None if self.clover is None else self.clover[self.keep_sites]
        return self_coupling(self.m0, cl, v)

    def apply(self, v: np.ndarray) -> np.ndarray:
        """oddeven.py:165-174."""
        if v.shape[0] != self.n_sites:
            raise ValueError(f"field has {v.shape[0]} sites, Schur system has {self.n_sites}")
        t = self._hop_to(v, self.keep_sites, self.elim_sites)
        z = self.solve_eliminated(t)
        u = self._hop_to(z, self.elim_sites, self.keep_sites)
        return self._diag_keep(v) - u

    __call__ = apply

    def reduce_rhs(self, eta: np.ndarray):
        """oddeven.py:179-188."""
        z = self.solve_eliminated(eta[self.elim_sites])
        u = self._hop_to(z, self.elim_sites, self.keep_sites)
        return eta[self.keep_sites] - u, eta[self.elim_sites].copy()

    def reconstruct(self, x_kept, eta_elim):
        """oddeven.py:190-196."""
        t = self._hop_to(x_kept, self.keep_sites, self.elim_sites)
        return self.solve_eliminated(eta_elim - t)

    def merge(self, x_kept, x_elim):
        """oddeven.py:198-201 / 87-95."""
        n = math.prod(self.dims)
        out = np.zeros((n, NSC, x_kept.shape[2]), dtype=np.complex128)
        out[self.keep_sites] = x_kept
        out[self.elim_sites] = x_elim
        return out


# ---------------------------------------------------------------------------
# per-rhs BLAS (reference blas.py:50-110)
# ---------------------------------------------------------------------------


def block_dot(w: np.ndarray, e: np.ndarray) -> np.ndarray:
    """(b,) conj(w_i) . e_i (blas.py:83-110; both strategies are the same sum)."""
    return np.einsum("xkb,xkb->b", np.conj(w), e)


def block_norms(x: np.ndarray) -> np.ndarray:
    """(b,) 2-norms (blas.py:65-68)."""
    return np.sqrt(np.einsum("xkb,xkb->b", np.conj(x), x).real)


# ---------------------------------------------------------------------------
# batched restarted GMRES (reference gmres.py:42-385)
# ---------------------------------------------------------------------------

_TINY = 1e-300


@dataclass
class GmresConfig:
    """gmres.py:42-56."""

    restart_len: int = 10
    restarts: int = 10
    tol: float = 1e-8
    fixed_iterations: bool = False
    reorthogonalize: bool = False
    breakdown_rel: float = 1e-14


@dataclass
class GmresOutcome:
    """gmres.py:90-98."""

    psi: np.ndarray
    history: list = field(default_factory=list)
    iterations: int = 0
    converged: np.ndarray | None = None
    final_relnorms: np.ndarray | None = None
    stagnated: bool = False
    breakdown: np.ndarray | None = None


def givens(a: np.ndarray, b: np.ndarray):
    """Complex Givens pair, c real, s = phase(a) conj(b)/rho (gmres.py:101-112)."""
    rho = np.sqrt(np.abs(a) ** 2 + np.abs(b) ** 2)
    nz = rho > 0
    az = np.abs(a) > 0
    safe_rho = np.where(nz, rho, 1.0)
    c = np.where(nz & az, np.abs(a) / safe_rho, np.where(nz, 0.0, 1.0))
    phase = np.where(az, a / np.where(az, np.abs(a), 1.0), 1.0)
    s = np.where(nz, phase * np.conj(b) / safe_rho, 0.0)
    return c, s


def gmres(op, eta: np.ndarray, psi0: np.ndarray | None, cfg: GmresConfig) -> GmresOutcome:
    """Lock-step batched GMRES(m) with MGS Arnoldi (gmres.py:115-251).

    Stops when max_i relnorm_i < tol (gmres.py:223-225); each restart begins
    from the true residual (gmres.py:180-198); breakdown when
    ||w|| <= breakdown_rel ||eta|| zeroes the new basis column
    (gmres.py:135-140); the final residual is explicit (gmres.py:236-251).
    """
    m = cfg.restart_len
    n, s, b = eta.shape
    psi = np.zeros_like(eta) if psi0 is None else psi0.copy()
    eta_norms = block_norms(eta)
    brk = np.zeros(b, dtype=bool)
    history, iterations = [], 0
    finish = stagnated = False
    inv_eta = np.maximum(eta_norms, _TINY)

    for _cycle in range(cfg.restarts):
        # true-residual restart (gmres.py:180-198)
        r = eta - op(psi)
        beta = block_norms(r)
        v = [r * np.where(beta > 0, 1.0 / np.where(beta > 0, beta, 1.0), 0.0)]
        h = np.zeros((b, m + 1, m), dtype=np.complex128)
        h_raw = np.zeros_like(h)
        gam = np.zeros((b, m + 1), dtype=np.complex128)
        gam[:, 0] = beta
        cs = np.zeros((b, m))
        sn = np.zeros((b, m), dtype=np.complex128)
        rel = np.where(eta_norms > 0, beta / inv_eta, 0.0)
        start_rel = rel.copy()
        if not cfg.fixed_iterations and rel.max() < cfg.tol:
            finish = True
        j_done = 0
        if not finish:
            for j in range(m):
                # Arnoldi step with MGS (gmres.py:115-158)
                w = op(v[j])
                for p in range(j + 1):
                    hp = block_dot(v[p], w)
                    h_raw[:, p, j] = hp
                    w = w - hp * v[p]
                if cfg.reorthogonalize:
                    wn = block_norms(w)
                    corr = [block_dot(v[p], w) for p in range(j + 1)]
                    defect = max(np.max(np.abs(c) / np.maximum(wn, _TINY)) for c in corr)
                    if defect > 1e-8:
                        for p, cp in enumerate(corr):
                            h_raw[:, p, j] += cp
                            w = w - cp * v[p]
                hn = block_norms(w)
                brk |= hn <= cfg.breakdown_rel * eta_norms
                h_raw[:, j + 1, j] = np.where(brk, 0.0, hn)
                inv = np.where(brk | (hn <= 0), 0.0, 1.0 / np.where(hn > 0, hn, 1.0))
                v.append(w * inv)
                col = h_raw[:, :j + 2, j].copy()
                for p in range(j):
                    a0, a1 = col[:, p].copy(), col[:, p + 1].copy()
                    col[:, p] = cs[:, p] * a0 + sn[:, p] * a1
                    col[:, p + 1] = -np.conj(sn[:, p]) * a0 + cs[:, p] * a1
                c, sg = givens(col[:, j], col[:, j + 1])
                cs[:, j], sn[:, j] = c, sg
                col[:, j] = c * col[:, j] + sg * col[:, j + 1]
                col[:, j + 1] = 0.0
                h[:, :j + 2, j] = col
                gam[:, j + 1] = -np.conj(sg) * gam[:, j]
                gam[:, j] = c * gam[:, j]
                rel = np.where(eta_norms > 0, np.abs(gam[:, j + 1]) / inv_eta, 0.0)
                iterations += 1
                history.append(rel.copy())
                j_done = j + 1
                if not cfg.fixed_iterations and rel.max() < cfg.tol:
                    finish = True
                    break
        if j_done:
            y = back_substitute(h, gam, j_done)
            for p in range(j_done):
                psi = psi + y[:, p] * v[p]
        if j_done == m and np.all(rel >= start_rel) and beta.max() > 0:
            stagnated = True
        if finish:
            break

    rfin = eta - op(psi)
    final = np.where(eta_norms > 0, block_norms(rfin) / inv_eta, 0.0)
    return GmresOutcome(psi, history, iterations, final <= max(cfg.tol, 1e-300), final,
                        stagnated, brk.copy())


def back_substitute(h: np.ndarray, gam: np.ndarray, m: int) -> np.ndarray:
    """Triangular solve skipping vanished diagonals (gmres.py:161-177)."""
    b = gam.shape[0]
    y = np.zeros((b, m), dtype=np.complex128)
    for row in range(m - 1, -1, -1):
        acc = gam[:, row].copy()
        if row + 1 < m:
            acc -= np.einsum("bc,bc->b", h[:, row, row + 1:m], y[:, row + 1:])
        d = h[:, row, row]
        ok = np.abs(d) > 0
        y[:, row] = np.where(ok, acc / np.where(ok, d, 1.0), 0.0)
    return y


def solve_dirac(dims, m0, links, clover, eta, cfg: GmresConfig, odd_even=False, psi0=None):
    """Full or even-site Schur solve (gmres.py:353-385).

    Returns (psi, outcome, full_relnorms).  For odd_even the stop test runs
    on the reduced system and full_relnorms is the explicit full-system
    residual (gmres.py:379-384).
    """
    if not odd_even:
        out = gmres(lambda v: apply_dirac(dims, m0, links, clover, v), eta, psi0, cfg)
        return out.psi, out, out.final_relnorms
    schur = SchurOracle(dims, m0, links, clover)
    reduced, eta_elim = schur.reduce_rhs(eta)
    x0 = None if psi0 is None else psi0[schur.keep_sites]
    out = gmres(schur.apply, reduced, x0, cfg)
    x_elim = schur.reconstruct(out.psi, eta_elim)
    psi = schur.merge(out.psi, x_elim)
    r = eta - apply_dirac(dims, m0, links, clover, psi)
    en = block_norms(eta)
    full = np.where(en > 0, block_norms(r) / np.maximum(en, _TINY), 0.0)
    return psi, out, full


# ---------------------------------------------------------------------------
# T-split halo semantics (reference halo.py:339-387, geometry.py:187-219)
# ---------------------------------------------------------------------------


def tsplit_faces(links_loc: np.ndarray, psi_loc: np.ndarray, per_t: int):
    """Face messages of one rank's T slab (halo.py:352-368).

    Returns ``(lam_down, chi_up)``: ``lam_down`` is the sign -1 half spinor
    of the local t=0 slice, sent to rank-1; ``chi_up`` is U_0^H times the
    sign +1 half spinor of the local t=T_loc-1 slice (link applied at the
    source), sent to rank+1.  Both are (per_t, 2, 3, b) complex, ascending
    site order -- the reference message shape (tests/test_halo.py:91-108).
    """
    b = psi_loc.shape[2]
    first = psi_loc[:per_t].reshape(per_t, NSPIN, NCOL, b)
    last = psi_loc[-per_t:].reshape(per_t, NSPIN, NCOL, b)
    lam_down = half_project(first, 0, -1)
    chi_up = np.einsum("xdc,xsdb->xscb", np.conj(links_loc[-per_t:, 0]), half_project(last, 0, +1))
    return lam_down, chi_up


def tsplit_local_apply(ldims, m0, links_loc, psi_loc, lam_from_up, chi_from_down) -> np.ndarray:
    """One rank's D psi given the two received faces (halo.py:370-387).

    Directions 1..3 and the interior T pairs are local; the forward T hop of
    the last slice uses ``lam_from_up`` (rank+1's t=0 face) with the local
    link, the backward T hop of the first slice uses ``chi_from_down``.
    """
    ldims = tuple(ldims)
    tl = ldims[0]
    per_t = math.prod(ldims[1:])
    n, _, b = psi_loc.shape
    spin = psi_loc.reshape(n, NSPIN, NCOL, b)
    acc = np.zeros_like(psi_loc)
    for mu in range(1, NDIM):
        fwd = neighbor_table(ldims, mu, +1)
        bwd = neighbor_table(ldims, mu, -1)
        moved = np.einsum("xcd,xsdb->xscb", links_loc[:, mu], half_project(spin, mu, -1)[fwd])
        acc += half_expand(moved, mu, -1).reshape(n, NSC, b)
        chi = np.einsum("xdc,xsdb->xscb", np.conj(links_loc[:, mu]), half_project(spin, mu, +1))[bwd]
        acc += half_expand(chi, mu, +1).reshape(n, NSC, b)
    lam0 = half_project(spin, 0, -1)
    chi0 = np.einsum("xdc,xsdb->xscb", np.conj(links_loc[:, 0]), half_project(spin, 0, +1))
    # forward T hop: site x at slice t reads slice t+1 (halo for t = tl-1)
    lam_next = np.concatenate([lam0[per_t:], lam_from_up])
    moved = np.einsum("xcd,xsdb->xscb", links_loc[:, 0], lam_next)
    acc += half_expand(moved, 0, -1).reshape(n, NSC, b)
    # backward T hop: site x at slice t receives chi from slice t-1 (halo for t = 0)
    chi_prev = np.concatenate([chi_from_down, chi0[:-per_t]])
    acc += half_expand(chi_prev, 0, +1).reshape(n, NSC, b)
    return (4.0 + m0) * psi_loc - acc


def tsplit_apply(dims, m0, links, psi, nranks: int) -> np.ndarray:
    """Dirac apply over a T-only rank split (grid (nranks,1,1,1)).

    Exchanges the faces of :func:`tsplit_faces` between ranks in a ring and
    runs :func:`tsplit_local_apply` per rank; equals :func:`apply_dirac` to
    roundoff for every nranks dividing T with T/nranks >= 2
    (geometry.py:187-219, halo.py:20-22).
    """
    t_all = dims[0]
    if t_all % nranks:
        raise ValueError("rank count must divide T")
    tl = t_all // nranks
    if nranks > 1 and tl < 2:
        raise ValueError("local T extent must be >= 2")
    per_t = math.prod(dims[1:])
    ldims = (tl,) + tuple(dims[1:])
    slabs = [slice(r * tl * per_t, (r + 1) * tl * per_t) for r in range(nranks)]
    faces = [tsplit_faces(links[s], psi[s], per_t) for s in slabs]
    out = np.empty_like(psi)
    for r, s in enumerate(slabs):
        lam_from_up = faces[(r + 1) % nranks][0]
        chi_from_down = faces[(r - 1) % nranks][1]
        out[s] = tsplit_local_apply(ldims, m0, links[s], psi[s], lam_from_up, chi_from_down)
    return out
