"""Wilson-Dirac operator: drop-in for ``lqcdlab.dirac`` (dirac.py:1-334).

``apply_dirac(params, gauge, clover, psi, comm=None, flops=None, perf=None)``
keeps the reference signature.  ``psi`` may be a host ``BlockSpinorField``
(reference layouts; uploaded, applied, downloaded) or a
:class:`~paper_2601_05816_b200.device.DeviceField` (stays on the device).
The apply itself is one launch of the fused sm_100a hopping kernel
(``b200wd_hop`` in csrc/dirac.cu): D psi = (4+m0) psi - C psi - H psi.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import (DeviceField, DeviceGauge, dtype_code, gauge_cache, ptr, require_device, stream_ptr,
                     upload)
from .fields import SPINOR_LEN

# traffic ledger of the paper (dirac.py:43-48), kept for the perf records
FLOPS_PER_SITE_RHS = 2574
VALUES_PER_SITE_RHS = 168
VALUES_PER_SITE_FIXED = 114
BYTES_PER_VALUE = 16


@dataclass(frozen=True)
class DiracParams:
    """dirac.py:51-60."""

    m0: float = -0.5
    a: float = 1.0

    def __post_init__(self) -> None:
        if self.a != 1.0:
            raise ValueError("lattice spacing is fixed to 1")


@dataclass
class FlopCounter:
    """dirac.py:63-73.  The GPU kernel is fused, so the tally records the
    reference's structured operation count for the same operator (the
    mathematical work), not the fused kernel's instruction mix."""

    cmul: int = 0
    cadd: int = 0
    rmul: int = 0

    @property
    def total_flops(self) -> int:
        return 6 * self.cmul + 2 * self.cadd + 2 * self.rmul

    def add_apply(self, n_sites: int, b: int) -> None:
        per = n_sites * b
        # self coupling (dirac.py:150-157)
        self.cmul += 72 * per
        self.cadd += 72 * per
        self.rmul += 12 * per
        # 8 compressions, 4 chi matvecs, 4 lambda matvecs, 8 reconstructions
        self.cmul += (8 * 6 + 4 * 18 + 4 * 18 + 8 * 6) * per
        self.cadd += (8 * 6 + 4 * 12 + 4 * 12 + 8 * 12) * per
        self.rmul += 8 * 6 * per


@dataclass
class DiracPerfRecord:
    """dirac.py:76-100."""

    seconds: float
    sites: int
    b: int
    layout: int
    flops: int
    bytes: int

    @property
    def gflops(self) -> float:
        return self.flops / self.seconds / 1e9 if self.seconds > 0 else float("inf")

    def as_dict(self) -> dict:
        return {"seconds": self.seconds, "sites": self.sites, "b": self.b, "layout": self.layout,
                "flops": self.flops, "bytes": self.bytes, "gflops": self.gflops}


def account_traffic(b: int) -> dict:
    """dirac.py:111-118."""
    if b < 1:
        raise ValueError(f"b must be >= 1, got {b}")
    return {"flops_per_site": FLOPS_PER_SITE_RHS * b,
            "bytes_per_site": (VALUES_PER_SITE_RHS * b + VALUES_PER_SITE_FIXED) * BYTES_PER_VALUE}


def compulsory_bytes_per_site(b: int, dtype: str = "c128") -> int:
    """Algorithmic HBM bytes of one full apply per site: read psi, write eta,
    read the 4 links of the site once: (24 b + 36) w."""
    w = 16 if dtype == "c128" else 8
    return (24 * b + 36) * w


def _lattice(geom, t_origin: int = 0):
    return _lib.Lattice.make(geom.dims, t_origin)


def clover_is_zero(clover) -> bool:
    return clover is None or (clover.is_zero() if hasattr(clover, "is_zero") else not np.any(clover.data))


class DiracOperator:
    """D = (4+m0) - H on the full (single-GPU) lattice, device resident.

    ``apply_device(v, out, scale)`` computes out = scale_r * D v in one
    launch; ``scale`` (device, b doubles) lets GMRES fold the basis
    normalisation into the apply.
    """

    def __init__(self, params: DiracParams, gauge, clover=None, dtype: str = "c128"):
        require_device()
        self.params = params
        self.dtype = dtype
        self.geom = gauge.geom
        self.gauge = gauge_cache.get(gauge, dtype)
        # site-local clover term C (dirac.py:137-157): fused into the hop epilogue
        self.clover = None if clover_is_zero(clover) else gauge_cache.get_clover(clover, dtype)
        self.lat = _lattice(self.geom)
        self.n_sites = self.geom.n_sites
        self.allreduce = None

    def apply_device(self, v: DeviceField, out: DeviceField | None = None, scale=None,
                     stream=None) -> DeviceField:
        if v.n_sites != self.n_sites or v.s != SPINOR_LEN:
            raise ValueError(f"field has {v.n_sites} sites / s={v.s}, lattice has {self.n_sites} sites")
        if v.dtype != self.dtype:
            raise ValueError(f"field dtype {v.dtype} != operator dtype {self.dtype}")
        out = v.empty_like() if out is None else out
        hop_device(self.lat, self.dtype, v.b, -1, self.gauge, v, out, v, 4.0 + self.params.m0, -1.0, scale,
                   clover=self.clover, clover_mode=1, stream=stream)
        return out

    def native_operator(self, v: DeviceField) -> "_lib.Operator":
        """This operator as a b200wd_operator program (one hop stage), for
        library-side drivers such as b200wd_gmres_arnoldi."""
        stage = dict(dst_parity=-1, src=_lib.OPND_IN, xself=_lib.OPND_IN, out=_lib.OPND_OUT,
                     alpha=4.0 + self.params.m0, beta=-1.0, use_scale=True,
                     clover=None if self.clover is None else self.clover.ptr, clover_mode=1)
        return _lib.Operator.make(self.lat, dtype_code(self.dtype), self.gauge.ptr, [stage])

    def apply_range(self, v: DeviceField, out: DeviceField, t_begin: int, t_end: int, stream=None) -> None:
        """Write only the T slices [t_begin, t_end) of out = D v."""
        hop_device(self.lat, self.dtype, v.b, -1, self.gauge, v, out, v, 4.0 + self.params.m0, -1.0, None,
                   t_begin, t_end, clover=self.clover, clover_mode=1, stream=stream)

    def apply_host_pipelined(self, psi, out=None, chunks: int = 16):
        """Host field in -> host field out with the PCIe transfers overlapped.

        The lattice is cut into T-slab chunks, copied H2D and converted to
        the device layout on an upload stream, the last chunk first (it holds
        slice 0's t-1 neighbour).  As chunk c lands, the slices
        [c*tc - 1, (c+1)*tc - 1) have both T neighbours resident; they are
        computed, converted back and copied D2H on a download stream at once,
        so uploads, compute and downloads overlap (PCIe is full duplex) and only
        tc + 1 slices remain after the last upload.  Results are identical to
        the unpipelined apply.
        """
        import torch

        T = self.geom.dims[0]
        nck = max(d for d in range(1, min(chunks, T) + 1) if T % d == 0)
        if nck < 2:
            return self.apply_device(upload(psi, self.dtype)).to_host(psi.layout, out)
        tc = T // nck
        per_t = self.geom.sites_per_slice
        n, b, s = psi.n_sites, psi.b, psi.s
        layout = int(psi.layout)
        if out is None:
            from .fields import BlockSpinorField
            out = BlockSpinorField.zeros(n, b, layout, s, self.geom)
        host_in = torch.from_numpy(np.ascontiguousarray(np.asarray(psi.data)).reshape(-1))
        host_out = torch.from_numpy(out.data.reshape(-1))
        dev = require_device()
        raw_in = torch.empty(n * s * b, dtype=torch.complex128, device=dev)
        raw_out = torch.empty_like(raw_in)
        d_psi = DeviceField.empty(n, b, s, self.dtype, self.geom)
        d_eta = DeviceField.empty(n, b, s, self.dtype, self.geom)
        cur = torch.cuda.current_stream()
        s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
        s_up.wait_stream(cur)
        chunk = tc * per_t * s * b  # complex elements per chunk (both layouts are site-major)
        esz = d_psi.data.element_size()
        up_order = [nck - 1] + list(range(nck - 1))  # the last chunk first: slice 0's t-1 neighbour
        up_ev = {}
        with torch.cuda.stream(s_up):
            for c in up_order:
                sl = slice(c * chunk, (c + 1) * chunk)
                raw_in[sl].copy_(host_in[sl], non_blocking=True)
                _lib.call("b200wd_spinor_import", raw_in[sl].data_ptr(), layout, tc * per_t, s, b,
                          d_psi.ptr + c * chunk * esz, dtype_code(self.dtype), stream_ptr(s_up))
                ev = torch.cuda.Event()
                ev.record(s_up)
                up_ev[c] = ev
        # As chunk c lands, the slices [c*tc - 1, (c+1)*tc - 1) have both T
        # neighbours resident: compute them and send them back at once.
        ranges = [(0, tc - 1, 0)] + [(c * tc - 1, (c + 1) * tc - 1, c) for c in range(1, nck - 1)]
        ranges.append(((nck - 1) * tc - 1, T, up_order[-1]))
        per_slice = per_t * s * b
        for t0, t1, c in ranges:
            if t1 <= t0:
                continue
            cur.wait_event(up_ev[c])
            self.apply_range(d_psi, d_eta, t0, t1, cur)
            sl = slice(t0 * per_slice, t1 * per_slice)
            _lib.call("b200wd_spinor_export", d_eta.ptr + t0 * per_slice * esz, dtype_code(self.dtype),
                      (t1 - t0) * per_t, s, b, raw_out[sl].data_ptr(), layout, stream_ptr(cur))
            s_dn.wait_stream(cur)
            with torch.cuda.stream(s_dn):
                host_out[sl].copy_(raw_out[sl], non_blocking=True)
        s_dn.synchronize()
        cur.wait_stream(s_dn)
        return out

    def __call__(self, v):
        return _apply_any(self, v)


def _apply_any(op, v):
    """Host fields in -> host fields out; device fields stay on the device."""
    if isinstance(v, DeviceField):
        return op.apply_device(v)
    dv = upload(v, op.dtype)
    return op.apply_device(dv).to_host(v.layout)


def apply_dirac(params: DiracParams, gauge, clover, psi, comm=None, flops: FlopCounter | None = None,
                perf: list | None = None, dtype: str | None = None, out=None):
    """eta = D psi over all rhs columns (dirac.py:299-334).

    ``comm`` routes the apply through a communicator (the multi-GPU T
    split, :class:`paper_2601_05816_b200.tsplit.TSplitComm`), as the
    reference routes it through its halo executor (dirac.py:313-314).
    """
    if comm is not None:
        return comm.apply_dirac(params, gauge, clover, psi, flops=flops, perf=perf)
    if psi.s != SPINOR_LEN:
        raise ValueError(f"expected full spinor field (s={SPINOR_LEN}), got s={psi.s}")
    if psi.n_sites != gauge.geom.n_sites:
        raise ValueError(f"field has {psi.n_sites} sites, gauge lattice has {gauge.geom.n_sites}")
    if dtype is None:
        dtype = psi.dtype if isinstance(psi, DeviceField) else "c128"
    t0 = time.perf_counter()
    op = DiracOperator(params, gauge, clover, dtype)
    if isinstance(psi, DeviceField):
        res = op.apply_device(psi, out)
    else:
        res = op.apply_host_pipelined(psi, out)
    if flops is not None:
        flops.add_apply(psi.n_sites, psi.b)
    if perf is not None:
        import torch
        torch.cuda.synchronize()
        ledger = account_traffic(psi.b)
        perf.append(DiracPerfRecord(time.perf_counter() - t0, psi.n_sites, psi.b, int(psi.layout),
                                    ledger["flops_per_site"] * psi.n_sites, ledger["bytes_per_site"] * psi.n_sites))
    return res


def hop_device(lat, dtype: str, b: int, dst_parity: int, gauge: DeviceGauge, src: DeviceField, out: DeviceField,
               xself: DeviceField | None, alpha: float, beta: float, scale=None, t_begin: int = 0,
               t_end: int | None = None, lam_halo=None, chi_halo=None, stream=None, clover=None,
               clover_mode: int = 0) -> None:
    """Thin wrapper over ``b200wd_hop`` / ``b200wd_hop_clover`` (include/b200wd.h)."""
    t_end = lat.dims[0] if t_end is None else t_end
    args = (lat, dtype_code(dtype), b, dst_parity, gauge.ptr, src.ptr, None if xself is None else xself.ptr,
            out.ptr, float(alpha), float(beta), ptr(scale), int(t_begin), int(t_end), ptr(lam_halo), ptr(chi_halo))
    if clover is None or clover_mode == 0:
        _lib.call("b200wd_hop", *args, stream_ptr(stream))
    else:
        _lib.call("b200wd_hop_clover", *args, clover.ptr, int(clover_mode), stream_ptr(stream))
