"""Batched restarted GMRES on the device: drop-in for ``lqcdlab.gmres`` (gmres.py:1-385).

Same mathematics and stopping semantics as the reference: b right-hand sides
advance in lock step, modified Gram-Schmidt Arnoldi, per-rhs complex Givens
rotations (c real), breakdown at ||w|| <= breakdown_rel ||eta||, stop when
max_i relnorm_i < tol, true-residual restarts, explicit final residual.

What changes is where it runs.  The basis, the solution and every field
pass live in HBM; the Hessenberg/Givens/least-squares bookkeeping runs in
one-thread-per-rhs kernels, so each Arnoldi step costs 1 operator apply +
(j+2) fused MGS passes (axpy of pass p fused with the inner product of
pass p+1, the last one with the norm) + 1 tiny kernel, and the host reads
back only the b relative residuals per iteration (the history).  The basis
is kept unnormalised, V_p = sigma_p Z_p, and sigma_j is folded into the
operator apply's output scale, which removes the normalisation pass.
"""

from __future__ import annotations

import ctypes
import logging
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .blas import block_dot_device, block_norm2_device, new_reduce_scratch
from .device import DeviceField, require_device, stream_ptr, upload
from .dirac import DiracOperator, DiracParams
from .fields import BlockSpinorField
from .oddeven import SchurOperator

# B200WD_PY_ARNOLDI=1 issues the Arnoldi step kernel by kernel from Python
# (the multi-rank path always does, to all-reduce between passes).
NATIVE_ARNOLDI = os.environ.get("B200WD_PY_ARNOLDI", "0") != "1"
# whole restart cycles enqueued by the library with a device-side stop flag
# (b200wd_gmres_cycle); B200WD_STEP_ARNOLDI=1 keeps one ABI call per step
NATIVE_CYCLE = os.environ.get("B200WD_STEP_ARNOLDI", "0") != "1"
log = logging.getLogger(__name__)
_TINY = 1e-300


@dataclass
class GmresConfig:
    """gmres.py:42-56.  ``dot_strategy`` is accepted for compatibility.

    ``orthogonalization`` is a B200 extension (not in the reference):
    ``"mgs"`` (default) is the reference's modified Gram-Schmidt
    (gmres.py:118-121); ``"cgs"`` is classical Gram-Schmidt in the
    library-issued Arnoldi step -- one projection pass over the whole basis
    and one update pass, about half the HBM traffic per iteration.  Its
    orthogonality loss grows as eps*kappa^2 instead of eps*kappa, so the
    iteration count can drift from the reference's on ill-conditioned
    systems; single rank only, and not combined with ``reorthogonalize``."""

    restart_len: int = 10
    restarts: int = 10
    tol: float = 1e-8
    fixed_iterations: bool = False
    dot_strategy: str = "deferred"
    reorthogonalize: bool = False
    breakdown_rel: float = 1e-14
    orthogonalization: str = "mgs"

    def __post_init__(self) -> None:
        if self.orthogonalization not in ("mgs", "cgs"):
            raise ValueError(f"orthogonalization must be 'mgs' or 'cgs', got {self.orthogonalization!r}")
        if self.restart_len < 1 or self.restarts < 1:
            raise ValueError("restart_len and restarts must be >= 1")
        if not self.tol > 0:
            raise ValueError("tol must be positive")
        if self.restart_len > 63:
            raise ValueError("restart_len must be <= 63 on the device solver")


@dataclass
class GmresResult:
    """gmres.py:90-98 (``psi`` has the type of ``eta``: host or device)."""

    psi: object
    history: list = field(default_factory=list)
    iterations: int = 0
    converged: np.ndarray | None = None
    final_relnorms: np.ndarray | None = None
    stagnated: bool = False
    breakdown: np.ndarray | None = None
    timings: dict = field(default_factory=dict)


class _State:
    """Device-resident solver state (b200wd_gmres_state)."""

    def __init__(self, b: int, m: int, brk_rel: float, dev, cgs: bool = False):
        c128 = dict(dtype=torch.complex128, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        self.h_raw = torch.zeros((b, m + 1, m), **c128)
        self.h = torch.zeros((b, m + 1, m), **c128)
        self.gamma = torch.zeros((b, m + 1), **c128)
        self.cs = torch.zeros((b, m), **f64)
        self.sn = torch.zeros((b, m), **c128)
        self.sigma = torch.zeros((m + 1, b), **f64)
        self.eta_norm = torch.zeros(b, **f64)
        self.relnorm = torch.zeros(b, **f64)
        self.brk = torch.zeros(b, dtype=torch.int32, device=dev)
        self.dot = torch.zeros(b, **c128)
        self.y = torch.zeros((b, m), **c128)
        self.scratch = new_reduce_scratch(b, dev)  # owned by this solve: no cross-stream sharing
        st = _lib.GmresState()
        st.b, st.m, st.breakdown_rel = b, m, brk_rel
        for name, t in (("h_raw", self.h_raw), ("h", self.h), ("gamma", self.gamma), ("cs", self.cs),
                        ("sn", self.sn), ("sigma", self.sigma), ("eta_norm", self.eta_norm),
                        ("relnorm", self.relnorm), ("breakdown", self.brk), ("dot", self.dot), ("y", self.y),
                        ("scratch", self.scratch)):
            setattr(st, name, t.data_ptr())
        if cgs:
            nbytes = int(_lib.load().b200wd_cgs_scratch_bytes(b, m))
            self.cgs_partials = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            st.orth, st.cgs_partials = 1, self.cgs_partials.data_ptr()
        self.st = st
        self.ref = ctypes.byref(st)


class _HostOp:
    """Adapter for a reference-style host callable op(BlockSpinorField) -> BlockSpinorField."""

    def __init__(self, fn, layout):
        self.fn, self.layout, self.allreduce = fn, layout, None

    def apply_device(self, v: DeviceField, out=None, scale=None):
        res = upload(self.fn(v.to_host(self.layout)), v.dtype)
        if scale is not None:
            res.data.mul_(scale.to(res.data.dtype)[None, None, None, :])
        if out is None:
            return res
        out.data.copy_(res.data)
        return out


class MatrixOp:
    """Dense matrix as a field operator (gmres.py:324-332), applied on the
    device with a cuBLAS matmul.  Test plumbing for the reference's
    fake-operator GMRES tests, not part of the stencil path."""

    def __init__(self, a):
        self.a = torch.as_tensor(np.asarray(a, dtype=np.complex128), device=require_device())
        self.allreduce = None

    def apply_device(self, v: DeviceField, out=None, scale=None):
        cols = v.logical_tensor().reshape(v.n_sites * v.s, v.b)
        res = (self.a @ cols).reshape(v.n_sites, v.s, v.b)
        if scale is not None:
            res = res * scale.to(res.dtype)[None, None, :]
        out = v.empty_like() if out is None else out
        out.data.copy_(DeviceField.from_logical(res).data)
        return out

    def __call__(self, v):
        if isinstance(v, DeviceField):
            return self.apply_device(v)
        return self.apply_device(upload(v)).to_host(v.layout)


def matrix_op(a) -> MatrixOp:
    return MatrixOp(a)


def dirac_op(params: DiracParams, gauge, clover, comm=None, dtype: str = "c128"):
    """gmres.py:335-339: the Dirac operator as a GMRES operator."""
    if comm is not None:
        return comm.operator(params, gauge, clover)
    return DiracOperator(params, gauge, clover, dtype)


def _as_device_op(op, layout):
    if hasattr(op, "apply_device"):
        return op
    if isinstance(getattr(op, "__self__", None), SchurOperator):
        return op.__self__
    return _HostOp(op, layout)


def gmres_solve(op, eta, psi0, cfg: GmresConfig) -> GmresResult:
    """Restarted batched GMRES for op(psi) = eta (gmres.py:201-251)."""
    host = not isinstance(eta, DeviceField)
    layout = eta.layout
    dev = require_device()
    dop = _as_device_op(op, layout)
    reduce = getattr(dop, "allreduce", None)
    d_eta = upload(eta, "c128", parity=getattr(eta, "parity", None)) if host else eta
    if d_eta.dtype != "c128":
        raise NotImplementedError("the device GMRES runs in complex128")
    n, s, b = d_eta.n_sites, d_eta.s, d_eta.b
    m = cfg.restart_len
    stream = stream_ptr()
    cgs = cfg.orthogonalization == "cgs"
    st = _State(b, m, cfg.breakdown_rel, dev, cgs=cgs)
    L = _lib.load()

    def chk(rc, name):
        if rc:
            raise RuntimeError(f"{name}: {L.b200wd_last_error().decode()}")

    def allreduce():
        if reduce is not None:
            reduce(st.dot)

    if psi0 is None:
        psi = d_eta.zeros_like()
    else:
        psi = upload(psi0, "c128", parity=d_eta.parity) if not isinstance(psi0, DeviceField) else psi0.copy()
    z = [d_eta.empty_like() for _ in range(m + 1)]
    zptrs = (ctypes.c_void_p * (m + 1))(*[zz.ptr for zz in z])
    # Single rank, stencil operator: the whole Arnoldi step is issued by the
    # library (b200wd_gmres_arnoldi), one ABI call per iteration.
    nop = None
    if reduce is None and not cfg.reorthogonalize and NATIVE_ARNOLDI and hasattr(dop, "native_operator"):
        nop = dop.native_operator(z[0])
    if cgs and nop is None:
        raise ValueError("orthogonalization='cgs' runs in the library-issued Arnoldi step only: a single-rank "
                         "stencil operator without reorthogonalize")
    rel_host = torch.empty(b, dtype=torch.float64, pin_memory=True) if nop is not None else None
    cycle = None
    if nop is not None and NATIVE_CYCLE:  # device-side stop test: one host round trip per cycle
        cycle = {"ctl": torch.zeros(2, dtype=torch.int32, device=dev),
                 "hist": torch.empty((m, b), dtype=torch.float64, device=dev),
                 "ctl_host": torch.zeros(2, dtype=torch.int32, pin_memory=True),
                 "hist_host": torch.empty((m, b), dtype=torch.float64, pin_memory=True)}

    block_norm2_device(d_eta, st.dot)
    allreduce()
    chk(L.b200wd_gmres_init(st.ref, stream), "gmres_init")
    eta_norms = np.sqrt(st.dot.real.cpu().numpy())

    history: list[np.ndarray] = []
    iterations = 0
    finish = stagnated = False
    for _cycle in range(cfg.restarts):
        # true-residual restart (gmres.py:180-198)
        dop.apply_device(psi, z[0])
        chk(L.b200wd_gmres_residual(st.ref, n, s, d_eta.ptr, z[0].ptr, stream), "gmres_residual")
        allreduce()
        chk(L.b200wd_gmres_start(st.ref, stream), "gmres_start")
        rel = st.relnorm.cpu().numpy().copy()
        start_rel = rel.copy()
        start_norm_max = float(st.gamma[:, 0].real.max().item())
        if not cfg.fixed_iterations and rel.max() < cfg.tol:
            finish = True
        j_done = 0
        if not finish and cycle is not None:
            rc = L.b200wd_gmres_cycle(st.ref, ctypes.byref(nop), m, n, zptrs, float(cfg.tol),
                                      int(bool(cfg.fixed_iterations)), cycle["ctl"].data_ptr(),
                                      cycle["hist"].data_ptr(), cycle["ctl_host"].data_ptr(),
                                      cycle["hist_host"].data_ptr(), stream)
            if rc == _lib.ERR_UNSUPPORTED and iterations == 0:
                cycle = None  # no cooperative sweep here: per-step calls below
            else:
                chk(rc, "gmres_cycle")
                stop, j_done = (int(v) for v in cycle["ctl_host"].numpy())
                hist = cycle["hist_host"].numpy()
                for jj in range(j_done):
                    history.append(hist[jj].copy())
                iterations += j_done
                rel = hist[j_done - 1].copy()
                finish = bool(stop)
        if not finish and cycle is None:
            for j in range(m):
                if nop is not None:
                    chk(L.b200wd_gmres_arnoldi(st.ref, ctypes.byref(nop), j, n, zptrs, rel_host.data_ptr(),
                                               stream), "gmres_arnoldi")
                    rel = rel_host.numpy().copy()
                else:
                    w = z[j + 1]
                    dop.apply_device(z[j], w, st.sigma[j])  # w = A V_j = sigma_j A Z_j
                    chk(L.b200wd_gmres_dot(st.ref, n, s, z[0].ptr, w.ptr, stream), "gmres_dot")
                    allreduce()
                    for p in range(j + 1):
                        nxt = z[p + 1].ptr if p < j else None
                        chk(L.b200wd_gmres_mgs(st.ref, j, p, n, s, w.ptr, z[p].ptr, nxt, stream), "gmres_mgs")
                        allreduce()
                    if cfg.reorthogonalize:
                        _reorthogonalize(st, z, j, w, reduce)
                    chk(L.b200wd_gmres_close_column(st.ref, j, stream), "gmres_close_column")
                    rel = st.relnorm.cpu().numpy().copy()
                iterations += 1
                history.append(rel)
                j_done = j + 1
                if not cfg.fixed_iterations and rel.max() < cfg.tol:
                    finish = True
                    break
        if j_done:
            chk(L.b200wd_gmres_update(st.ref, j_done, n, s, zptrs, psi.ptr, stream), "gmres_update")
        if j_done == m and np.all(rel >= start_rel) and start_norm_max > 0:
            stagnated = True
            log.warning("gmres cycle made no progress (max relnorm %.3e)", rel.max())
        if finish:
            break

    # explicit final residual (gmres.py:236-251)
    dop.apply_device(psi, z[0])
    chk(L.b200wd_gmres_residual(st.ref, n, s, d_eta.ptr, z[0].ptr, stream), "gmres_residual")
    allreduce()
    fin = np.sqrt(st.dot.real.cpu().numpy())
    final = np.where(eta_norms > 0, fin / np.maximum(eta_norms, _TINY), 0.0)
    brk = st.brk.cpu().numpy().astype(bool)
    out_psi = psi.to_host(layout) if host else psi
    return GmresResult(out_psi, history, iterations, final <= max(cfg.tol, 1e-300), final, stagnated, brk)


def _reorthogonalize(st: _State, z, j: int, w: DeviceField, reduce) -> None:
    """Optional second Gram-Schmidt pass (gmres.py:122-133)."""
    nrm = block_norm2_device(w)
    if reduce is not None:
        reduce(nrm)
    wnorm = torch.sqrt(nrm.real)
    corr = []
    for p in range(j + 1):
        d = block_dot_device(z[p], w)
        if reduce is not None:
            reduce(d)
        corr.append(d * st.sigma[p])
    defect = max(float((c.abs() / torch.clamp(wnorm, min=_TINY)).max()) for c in corr)
    if defect > 1e-8:
        for p, cp in enumerate(corr):
            st.h_raw[:, p, j] += cp
            coef = (-cp * st.sigma[p]).contiguous()
            _lib.call("b200wd_block_axpy", w.n_sites, w.s, w.b, coef.data_ptr(), z[p].ptr, w.ptr, stream_ptr())
    block_norm2_device(w, st.dot)
    if reduce is not None:
        reduce(st.dot)


@dataclass
class SolveReport:
    """gmres.py:342-350."""

    psi: object
    result: GmresResult
    odd_even: bool
    full_relnorms: np.ndarray
    iterations: int


def solve_dirac(params: DiracParams, gauge, clover, eta, cfg: GmresConfig, odd_even: bool = False, psi0=None,
                comm=None) -> SolveReport:
    """Solve D psi = eta directly or through the even-site Schur system (gmres.py:353-385)."""
    host = not isinstance(eta, DeviceField)
    if comm is not None:
        return comm.solve_dirac(params, gauge, clover, eta, cfg, odd_even=odd_even, psi0=psi0)
    d_eta = upload(eta, "c128") if host else eta
    # the links (and clover) cross PCIe once per solve: both operators share the device copy
    from .device import gauge_cache
    gauge = gauge_cache.get(gauge, "c128")
    dirac = DiracOperator(params, gauge, clover, "c128")
    if not odd_even:
        res = gmres_solve(dirac, d_eta, psi0, cfg)
        psi = res.psi
        full = res.final_relnorms
    else:
        schur = SchurOperator(params, gauge, clover, dtype="c128", gauge_dev=gauge)
        reduced, eta_elim = schur.reduce_rhs(d_eta)
        x0 = None
        if psi0 is not None:
            d_psi0 = upload(psi0, "c128") if not isinstance(psi0, DeviceField) else psi0
            keep, _ = schur._split_full(d_psi0)
            x0 = keep
        res = gmres_solve(schur, reduced, x0, cfg)
        x_elim = schur.reconstruct_device(res.psi, eta_elim)
        psi = schur.merge(res.psi, x_elim)
        r = dirac.apply_device(psi)
        st_dot = block_norm2_device(_sub(d_eta, r))
        en = np.sqrt(block_norm2_device(d_eta).real.cpu().numpy())
        full = np.where(en > 0, np.sqrt(st_dot.real.cpu().numpy()) / np.maximum(en, _TINY), 0.0)
    if host:
        psi = psi.to_host(eta.layout)
        res.psi = res.psi.to_host(eta.layout) if isinstance(res.psi, DeviceField) else res.psi
    return SolveReport(psi, res, odd_even, full, res.iterations)


def _sub(a: DeviceField, b: DeviceField) -> DeviceField:
    """a - b on the device via the axpy kernel (b is consumed)."""
    minus_one = torch.full((a.b,), -1.0 + 0j, dtype=torch.complex128, device=a.data.device)
    _lib.call("b200wd_block_scale", b.n_sites, b.s, b.b, minus_one.data_ptr(), b.ptr, stream_ptr())
    one = torch.ones(a.b, dtype=torch.complex128, device=a.data.device)
    _lib.call("b200wd_block_axpy", a.n_sites, a.s, a.b, one.data_ptr(), a.ptr, b.ptr, stream_ptr())
    return b


def batched_vs_independent_audit(op, eta, psi0, cfg: GmresConfig) -> float:
    """gmres.py:254-281."""
    batched = gmres_solve(op, eta, psi0, cfg)
    worst = 0.0
    host_eta = eta.to_host() if isinstance(eta, DeviceField) else eta
    cols = host_eta.ksi()
    for i in range(host_eta.b):
        e_i = BlockSpinorField.zeros(host_eta.n_sites, 1, host_eta.layout, host_eta.s, host_eta.geom)
        e_i.set_ksi(cols[:, :, i:i + 1])
        p_i = None
        if psi0 is not None:
            hp = psi0.to_host() if isinstance(psi0, DeviceField) else psi0
            p_i = BlockSpinorField.zeros(hp.n_sites, 1, hp.layout, hp.s, hp.geom)
            p_i.set_ksi(hp.ksi()[:, :, i:i + 1])
        single = gmres_solve(op, e_i, p_i, cfg)
        for it in range(min(len(batched.history), len(single.history))):
            ref = single.history[it][0]
            worst = max(worst, abs(batched.history[it][i] - ref) / max(ref, 1e-30))
    return worst


def gamma_residual_audit(op, eta, psi0, cfg: GmresConfig) -> float:
    """gmres.py:284-318: |gamma_{j+1}| vs the explicit residual at every step.

    Runs the fixed-iteration protocol with the device kernels, expanding the
    current least-squares minimiser after every Arnoldi step.
    """
    cfg = GmresConfig(restart_len=cfg.restart_len, restarts=cfg.restarts, tol=cfg.tol, fixed_iterations=True,
                      reorthogonalize=cfg.reorthogonalize)
    host = not isinstance(eta, DeviceField)
    dev = require_device()
    dop = _as_device_op(op, eta.layout)
    d_eta = upload(eta) if host else eta
    n, s, b = d_eta.n_sites, d_eta.s, d_eta.b
    m = cfg.restart_len
    cgs = cfg.orthogonalization == "cgs"
    st = _State(b, m, cfg.breakdown_rel, dev, cgs=cgs)
    L = _lib.load()
    stream = stream_ptr()
    psi = d_eta.zeros_like() if psi0 is None else (upload(psi0) if host else psi0.copy())
    z = [d_eta.empty_like() for _ in range(m + 1)]
    zptrs = (ctypes.c_void_p * (m + 1))(*[zz.ptr for zz in z])
    block_norm2_device(d_eta, st.dot)
    L.b200wd_gmres_init(st.ref, stream)
    worst = 0.0
    for _ in range(cfg.restarts):
        dop.apply_device(psi, z[0])
        L.b200wd_gmres_residual(st.ref, n, s, d_eta.ptr, z[0].ptr, stream)
        L.b200wd_gmres_start(st.ref, stream)
        for j in range(m):
            w = z[j + 1]
            dop.apply_device(z[j], w, st.sigma[j])
            L.b200wd_gmres_dot(st.ref, n, s, z[0].ptr, w.ptr, stream)
            for p in range(j + 1):
                L.b200wd_gmres_mgs(st.ref, j, p, n, s, w.ptr, z[p].ptr, z[p + 1].ptr if p < j else None, stream)
            L.b200wd_gmres_close_column(st.ref, j, stream)
            gam = st.gamma[:, j + 1].abs().cpu().numpy()
            probe = psi.copy()
            L.b200wd_gmres_update(st.ref, j + 1, n, s, zptrs, probe.ptr, stream)
            r = dop.apply_device(probe)
            _sub(d_eta, r)
            explicit = np.sqrt(block_norm2_device(r).real.cpu().numpy())
            worst = max(worst, float((np.abs(gam - explicit) / np.maximum(explicit, 1e-30)).max()))
        L.b200wd_gmres_update(st.ref, m, n, s, zptrs, psi.ptr, stream)
    return worst
