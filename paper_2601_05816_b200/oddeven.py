"""Odd-even (Schur) preconditioning: drop-in for ``lqcdlab.oddeven`` (oddeven.py:1-222).

With C = 0 the site-local blocks are (4+m0) I, so with H the hopping sum
(D = (4+m0) - H, D_eo = -H_eo):

    S v        = (4+m0) v - H_eo H_oe v / (4+m0)
    reduce_rhs : eta~_e = eta_e + H_eo eta_o / (4+m0)
    reconstruct: x_o    = (eta_o + H_oe x_e) / (4+m0)

With a clover term the eliminated blocks (4+m0) I - C are inverted once on
the host with the reference's condition check and applied in the kernel
epilogue (clover_mode 2); the kept blocks are applied as -C v (mode 1).
Each line is one or two launches of the parity-restricted fused hopping
kernel (``b200wd_hop`` with dst_parity = 0/1); the reference instead embeds
the half field in the full lattice and hops every site twice per apply
(oddeven.py:146-156) with a per-site LU loop (oddeven.py:138-144).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DeviceField, dtype_code, gauge_cache, ptr, require_device, stream_ptr, upload, upload_packed_blocks
from .dirac import DiracParams, _lattice, clover_is_zero, hop_device
from .fields import SPINOR_LEN, BlockSpinorField, Layout
from .geometry import LatticeGeometry

PARITY_NAME = {0: "even", 1: "odd"}


class SingularBlockError(np.linalg.LinAlgError):
    """A site-local block of the eliminated parity is numerically singular (oddeven.py:38-48)."""

    def __init__(self, site: int, block: int, cond: float):
        self.site = site
        self.block = block
        self.cond = cond
        super().__init__(f"site-local block {block} at site {site} is numerically singular "
                         f"(condition estimate {cond:.3e})")


@dataclass(frozen=True)
class OeSplit:
    """Parity index sets (oddeven.py:51-69); on the device cb = site >> 1."""

    geom: LatticeGeometry
    even: np.ndarray
    odd: np.ndarray
    perm: np.ndarray

    @classmethod
    def from_geom(cls, geom: LatticeGeometry) -> "OeSplit":
        even, odd = geom.even_sites, geom.odd_sites
        perm = np.empty(geom.n_sites, dtype=np.int64)
        perm[even] = np.arange(len(even))
        perm[odd] = len(even) + np.arange(len(odd))
        return cls(geom, even, odd, perm)

    def sites(self, parity: int) -> np.ndarray:
        return self.even if parity == 0 else self.odd


def split_fields(v, split: OeSplit | None = None):
    """Host partition into (even, odd) halves (oddeven.py:72-84)."""
    if split is None:
        if v.geom is None:
            raise ValueError("field carries no geometry; pass an explicit OeSplit")
        split = OeSplit.from_geom(v.geom)
    vv = v.ksi()
    halves = []
    for sites in (split.even, split.odd):
        half = BlockSpinorField.zeros(len(sites), v.b, v.layout, v.s)
        half.set_ksi(vv[sites])
        halves.append(half)
    return halves[0], halves[1]


def merge_fields(v_even, v_odd, split: OeSplit):
    """Inverse of :func:`split_fields` (oddeven.py:87-95)."""
    out = BlockSpinorField.zeros(split.geom.n_sites, v_even.b, v_even.layout, v_even.s, split.geom)
    ov = out.ksi()
    ov[split.even] = v_even.ksi()
    ov[split.odd] = v_odd.ksi()
    return out


def device_split(lat, v: DeviceField) -> tuple[DeviceField, DeviceField]:
    """Full device field -> (even, odd) device fields."""
    half = v.n_sites // 2
    e = DeviceField.empty(half, v.b, v.s, v.dtype, v.geom, 0, v.layout)
    o = DeviceField.empty(half, v.b, v.s, v.dtype, v.geom, 1, v.layout)
    _lib.call("b200wd_parity_split", lat, dtype_code(v.dtype), v.s, v.b, v.ptr, e.ptr, o.ptr, stream_ptr())
    return e, o


def device_merge(lat, e: DeviceField, o: DeviceField, geom) -> DeviceField:
    out = DeviceField.empty(2 * e.n_sites, e.b, e.s, e.dtype, geom, None, e.layout)
    _lib.call("b200wd_parity_merge", lat, dtype_code(e.dtype), e.s, e.b, e.ptr, o.ptr, out.ptr, stream_ptr())
    return out


class SchurOperator:
    """S = D_kk - D_ke D_ee^-1 D_ek, parity k kept (oddeven.py:98-201)."""

    def __init__(self, params: DiracParams, gauge, clover=None, keep_parity: int = 0, cond_limit: float = 1e12,
                 dtype: str = "c128", lattice=None, gauge_dev=None, comm=None):
        if keep_parity not in (0, 1):
            raise ValueError(f"parity must be 0 (even) or 1 (odd), got {keep_parity}")
        self.params = params
        self.keep_parity = keep_parity
        self.elim_parity = 1 - keep_parity
        self.geom = gauge.geom
        self.dtype = dtype
        self.split = None
        # diagonal blocks of the eliminated parity are (4+m0) I (C = 0):
        # condition number 1, or infinite when 4+m0 = 0 (oddeven.py:123-132)
        self.diag = 4.0 + params.m0
        self.clover_inv = self.clover_keep = None
        # local parity == global parity: slab extents and T origins are even (dirac.cu fill_params)
        elim = self.geom.odd_sites if keep_parity == 0 else self.geom.even_sites
        if clover_is_zero(clover):
            if self.diag == 0.0 or not np.isfinite(self.diag):
                raise SingularBlockError(int(elim[0]), 0, float("inf"))
        require_device()
        if not clover_is_zero(clover):
            # eliminated diagonal blocks (4+m0) I - C: condition check as the
            # reference (np.linalg.cond, oddeven.py:123-132), inverse packed like
            # the clover (Hermitian) and uploaded once; applied in-kernel
            keep = self.geom.even_sites if keep_parity == 0 else self.geom.odd_sites
            blocks = self.diag * np.eye(6) - clover.blocks()[elim]
            cond = np.linalg.cond(blocks)
            bad = ~np.isfinite(cond) | (cond > cond_limit)
            if bad.any():
                row, half = np.argwhere(bad)[0]
                raise SingularBlockError(int(elim[row]), int(half), float(cond[row, half]))
            inv = np.linalg.inv(blocks)
            rows, cols = np.tril_indices(6)
            self.clover_inv = upload_packed_blocks(inv[..., rows, cols], dtype)
            self.clover_keep = upload_packed_blocks(np.asarray(clover.data)[keep], dtype)
        self.gauge = gauge_dev if gauge_dev is not None else gauge_cache.get(gauge, dtype)
        self.lat = lattice if lattice is not None else _lattice(self.geom)
        self.comm = comm
        self.allreduce = None if comm is None else comm.allreduce
        self._tmp = None

    @property
    def n_sites(self) -> int:
        return self.geom.n_sites // 2

    # -- device kernels ----------------------------------------------------------
    def _hop(self, dst_parity, src, out, xself, alpha, beta, scale=None, clover=None, mode=0):
        if self.comm is not None:
            self.comm.hop(dst_parity, src, out, xself, alpha, beta, scale, clover=clover, mode=mode)
        else:
            hop_device(self.lat, self.dtype, src.b, dst_parity, self.gauge, src, out, xself, alpha, beta, scale,
                       clover=clover, clover_mode=mode)

    def _tmp_like(self, v: DeviceField) -> DeviceField:
        t = self._tmp
        if t is None or t.data.shape != v.data.shape or t.dtype != v.dtype:
            t = DeviceField.empty(v.n_sites, v.b, v.s, v.dtype, self.geom, self.elim_parity, v.layout)
            self._tmp = t
        return t

    def native_operator(self, v: DeviceField):
        """S as a two-stage b200wd_operator program (same launches as
        apply_device); None when the operator runs over a T split."""
        if self.comm is not None:
            return None
        tmp = self._tmp_like(v)
        a = self.diag
        I, O, T = _lib.OPND_IN, _lib.OPND_OUT, _lib.OPND_TMP
        if self.clover_inv is None:
            stages = [dict(dst_parity=self.elim_parity, src=I, out=T, beta=1.0 / a),
                      dict(dst_parity=self.keep_parity, src=T, xself=I, out=O, alpha=a, beta=-1.0, use_scale=True)]
        else:
            stages = [dict(dst_parity=self.elim_parity, src=I, out=T, beta=1.0, clover=self.clover_inv.ptr,
                           clover_mode=2),
                      dict(dst_parity=self.keep_parity, src=T, xself=I, out=O, alpha=a, beta=-1.0, use_scale=True,
                           clover=self.clover_keep.ptr, clover_mode=1)]
        return _lib.Operator.make(self.lat, dtype_code(self.dtype), self.gauge.ptr, stages, tmp.ptr)

    def apply_device(self, v: DeviceField, out: DeviceField | None = None, scale=None) -> DeviceField:
        """out = scale_r * S v: two parity-restricted hop launches (oddeven.py:165-174)."""
        if v.n_sites != self.n_sites:
            raise ValueError(f"field has {v.n_sites} sites, Schur system has {self.n_sites}")
        if v.s != SPINOR_LEN:
            raise ValueError(f"expected full spinor components (s={SPINOR_LEN}), got s={v.s}")
        tmp = self._tmp_like(v)
        out = DeviceField.empty(v.n_sites, v.b, v.s, v.dtype, self.geom, self.keep_parity, v.layout) \
            if out is None else out
        a = self.diag
        if self.clover_inv is None:
            # tmp_o = D_oo^-1 (-D_oe) v = H_oe v / a
            self._hop(self.elim_parity, v, tmp, None, 0.0, 1.0 / a)
            # out_e = a v - H_eo tmp
            self._hop(self.keep_parity, tmp, out, v, a, -1.0, scale)
        else:
            # tmp_o = D_oo^-1 H_oe v ; out_e = (a - C_e) v - H_eo tmp
            self._hop(self.elim_parity, v, tmp, None, 0.0, 1.0, None, self.clover_inv, 2)
            self._hop(self.keep_parity, tmp, out, v, a, -1.0, scale, self.clover_keep, 1)
        return out

    def reduce_rhs_device(self, eta_keep: DeviceField, eta_elim: DeviceField) -> DeviceField:
        """eta~ = eta_k - D_ke D_ee^-1 eta_e = eta_k + H_ke eta_e / a (oddeven.py:179-188)."""
        out = eta_keep.empty_like()
        out.parity = self.keep_parity
        if self.clover_inv is None:
            self._hop(self.keep_parity, eta_elim, out, eta_keep, 1.0, 1.0 / self.diag)
        else:
            z = eta_elim.empty_like()
            _lib.call("b200wd_clover_apply", eta_elim.n_sites, dtype_code(self.dtype), eta_elim.b,
                      self.clover_inv.ptr, eta_elim.ptr, z.ptr, stream_ptr())
            self._hop(self.keep_parity, z, out, eta_keep, 1.0, 1.0)
        return out

    def reconstruct_device(self, x_keep: DeviceField, eta_elim: DeviceField) -> DeviceField:
        """x_e = D_ee^-1 (eta_e - D_ek x_k) = (eta_e + H_ek x_k) / a (oddeven.py:190-196)."""
        out = eta_elim.empty_like()
        out.parity = self.elim_parity
        a = self.diag
        if self.clover_inv is None:
            self._hop(self.elim_parity, x_keep, out, eta_elim, 1.0 / a, 1.0 / a)
        else:
            self._hop(self.elim_parity, x_keep, out, eta_elim, 1.0, 1.0, None, self.clover_inv, 2)
        return out

    # -- reference-facing API -------------------------------------------------------
    def apply(self, v):
        if isinstance(v, DeviceField):
            return self.apply_device(v)
        if v.n_sites != self.n_sites:
            raise ValueError(f"field has {v.n_sites} sites, Schur system has {self.n_sites}")
        dv = upload(v, self.dtype, parity=self.keep_parity)
        return self.apply_device(dv).to_host(v.layout)

    def __call__(self, v):
        return self.apply(v)

    def _split_full(self, eta):
        if isinstance(eta, DeviceField):
            de = eta
        else:
            de = upload(eta, self.dtype)
        even, odd = device_split(self.lat, de)
        return (even, odd) if self.keep_parity == 0 else (odd, even)

    def reduce_rhs(self, eta):
        keep, elim = self._split_full(eta)
        red = self.reduce_rhs_device(keep, elim)
        if isinstance(eta, DeviceField):
            return red, elim
        return red.to_host(eta.layout), elim.to_host(eta.layout)

    def reconstruct(self, x_kept, eta_elim):
        host = not isinstance(x_kept, DeviceField)
        xk = upload(x_kept, self.dtype, parity=self.keep_parity) if host else x_kept
        ee = upload(eta_elim, self.dtype, parity=self.elim_parity) if not isinstance(eta_elim, DeviceField) \
            else eta_elim
        out = self.reconstruct_device(xk, ee)
        return out.to_host(x_kept.layout) if host else out

    def merge(self, x_kept, x_elim):
        if isinstance(x_kept, DeviceField):
            e, o = (x_kept, x_elim) if self.keep_parity == 0 else (x_elim, x_kept)
            return device_merge(self.lat, e, o, self.geom)
        if self.split is None:
            self.split = OeSplit.from_geom(self.geom)
        if self.keep_parity == 0:
            return merge_fields(x_kept, x_elim, self.split)
        return merge_fields(x_elim, x_kept, self.split)


def apply_schur(params, gauge, clover, v_even):
    """oddeven.py:204-211."""
    return SchurOperator(params, gauge, clover).apply(v_even)


def reconstruct_full(params, gauge, clover, x_even, rhs_odd):
    """oddeven.py:214-222."""
    return SchurOperator(params, gauge, clover).reconstruct(x_even, rhs_odd)
