"""``MultiRankExecutor`` / ``apply_dirac_multirank`` (halo.py:216-401) on one GPU.

The reference's executor takes whole-lattice fields, cuts them into the rank
blocks of a ``RankGrid``, runs every rank's staged apply with halo messages
between them (sequentially in phase lockstep, or one thread per rank), and
merges the local results; passed as ``comm=`` to ``apply_dirac`` it routes the
apply through that path.  Here the ranks are the slabs of a T-only grid
(R, 1, 1, 1) -- the decomposition the multi-GPU path uses -- and
each rank's apply runs the same device kernels as the multi-GPU T split
(``tsplit.TSplitComm``): every rank packs its two T faces (``b200wd_halo_pack``:
the lambda face of its first slice for rank-1, the U_0^H-applied chi face of its
last slice for rank+1), then computes its interior slices and its two boundary
slices from the neighbours' faces (``b200wd_hop`` / ``b200wd_hop_clover`` with
halos).  Only the transport differs: the faces stay in one GPU's memory instead
of crossing NVLink.  Results equal the single-rank apply up to summation order
(tests: <= 1e-14 relative).  ``mode`` ("sequential" / "threads") is accepted
for the reference's signature; the device work is stream-ordered either way.
Grids that split X, Y or Z raise ``NotImplementedError``.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DeviceField, require_device, upload, upload_gauge, upload_packed_blocks
from .dirac import DiracPerfRecord, account_traffic, hop_device
from .fields import SPINOR_LEN, GaugeField
from .geometry import RankGrid, t_split

DEFAULT_TIMEOUT = 30.0  # halo.py: seconds a receive waits (host mailboxes; unused on the device)


@dataclass
class EpochStats:
    """Per-rank timing of one apply (halo.py:101-110); on the device the
    'wait' is the halo hand-off and is folded into compute."""

    epoch: int
    rank: int
    wait_seconds: float
    compute_seconds: float

    def as_dict(self) -> dict:
        return {"epoch": self.epoch, "rank": self.rank, "wait_seconds": self.wait_seconds,
                "compute_seconds": self.compute_seconds}


class MultiRankExecutor:
    """Whole-lattice fields in, whole-lattice result out, computed rank by rank
    over a T-only rank grid with device halo exchange (halo.py:216-387)."""

    def __init__(self, grid: RankGrid, mode: str = "sequential", timeout: float = DEFAULT_TIMEOUT):
        if mode not in ("sequential", "threads"):
            raise ValueError(f"unknown execution mode {mode!r}")
        if any(g != 1 for g in grid.grid[1:]):
            raise NotImplementedError(f"rank grid {grid.grid}: the B200 path splits T only (grid (R, 1, 1, 1))")
        self.grid, self.mode, self.timeout = grid, mode, timeout
        self.epoch = 0
        self.last_stats: list[EpochStats] = []
        self._plan_key = None
        self._plan_refs = (lambda: None,)
        self._plan = None

    def _plan_for(self, gauge, clover, dtype):
        from .tsplit import CudaHaloKernels
        # reuse the uploaded slabs only for read-only host arrays (device._GaugeCache
        # semantics: a writeable array may have changed in place since the last call)
        frozen = not gauge.data.flags.writeable and (clover is None or not clover.data.flags.writeable)
        key = (gauge.geom.dims, id(gauge.data), None if clover is None else id(clover.data), dtype)
        if frozen and self._plan_key == key and self._plan_refs[0]() is gauge.data:
            return self._plan
        geom, ranks = gauge.geom, self.grid.grid[0]
        slabs = []
        for r in range(ranks):
            lg, t0 = t_split(geom, ranks, r)
            lo, hi = t0 * geom.sites_per_slice, (t0 + lg.dims[0]) * geom.sites_per_slice
            dg = upload_gauge(GaugeField(lg, np.ascontiguousarray(gauge.data[lo:hi])), dtype)
            dc = None
            if clover is not None and np.any(clover.data):
                dc = upload_packed_blocks(clover.data[lo:hi], dtype)
            slabs.append((lg, t0, lo, hi, _lib.Lattice.make(lg.dims, t0), dg, dc))
        self._plan, self._plan_key = (slabs, CudaHaloKernels()), key
        self._plan_refs = (weakref.ref(gauge.data),)
        return self._plan

    def apply_device(self, params, gauge, clover, psi: DeviceField, out: DeviceField | None = None,
                     scale=None) -> DeviceField:
        """Device fields in and out (whole lattice); ``scale`` (device, b
        doubles) multiplies each rhs of the result, as in DiracOperator."""
        if psi.n_sites != gauge.geom.n_sites or psi.s != SPINOR_LEN:
            raise ValueError(f"field has {psi.n_sites} sites / s={psi.s}, lattice has {gauge.geom.n_sites} sites")
        slabs, k = self._plan_for(gauge, clover, psi.dtype)
        out = psi.empty_like() if out is None else out
        b, dt = psi.b, psi.dtype
        alpha = 4.0 + params.m0
        views = [(DeviceField(psi.data[lo // 8:hi // 8], hi - lo, lg),
                  DeviceField(out.data[lo // 8:hi // 8], hi - lo, lg)) for lg, _, lo, hi, _, _, _ in slabs]
        faces = []
        for (lg, _, _, _, lat, dg, _), (x, _) in zip(slabs, views):  # every rank posts its two faces
            lam, chi = (k.face_buffer(lg.sites_per_slice, b, dt, psi.data.device) for _ in range(2))
            k.pack(lat, dt, b, -1, dg, x, lam, chi)
            faces.append((lam, chi))
        t_start = time.perf_counter()
        ranks = len(slabs)
        for r, ((lg, _, _, _, lat, dg, dc), (x, y)) in enumerate(zip(slabs, views)):
            lam_in = faces[(r + 1) % ranks][0]  # lambda of rank r+1's first slice
            chi_in = faces[(r - 1) % ranks][1]  # chi of rank r-1's last slice
            T = lg.dims[0]
            if T > 2:
                hop_device(lat, dt, b, -1, dg, x, y, x, alpha, -1.0, scale, 1, T - 1, clover=dc, clover_mode=1)
            for t in (0, T - 1):
                hop_device(lat, dt, b, -1, dg, x, y, x, alpha, -1.0, scale, t, t + 1, lam_in, chi_in, clover=dc,
                           clover_mode=1)
        wall = time.perf_counter() - t_start  # host issue time (the device work is asynchronous)
        self.last_stats = [EpochStats(self.epoch, r, 0.0, wall / ranks) for r in range(ranks)]
        self.epoch += 1
        return out

    def apply_dirac(self, params, gauge, clover, psi, flops=None, perf=None):
        """comm= seam of apply_dirac (dirac.py:313-314): host fields in -> host out."""
        if psi.n_sites != gauge.geom.n_sites:
            raise ValueError(f"field has {psi.n_sites} sites, lattice has {gauge.geom.n_sites}")
        require_device()
        t0 = time.perf_counter()
        if isinstance(psi, DeviceField):
            res = self.apply_device(params, gauge, clover, psi)
        else:
            res = self.apply_device(params, gauge, clover, upload(psi, "c128")).to_host(psi.layout)
        if flops is not None:
            flops.add_apply(psi.n_sites, psi.b)
        if perf is not None:
            led = account_traffic(psi.b)
            perf.append(DiracPerfRecord(time.perf_counter() - t0, psi.n_sites, psi.b, int(psi.layout),
                                        led["flops_per_site"] * psi.n_sites, led["bytes_per_site"] * psi.n_sites))
        return res

    def operator(self, params, gauge, clover=None, dtype: str = "c128"):
        """The Dirac operator applied through this executor (gmres.py:335-339)."""
        return _ExecutorOp(self, params, gauge, clover)

    def solve_dirac(self, params, gauge, clover, eta, cfg, odd_even: bool = False, psi0=None):
        """gmres.py:353-385 with comm=this executor: the unpreconditioned solve
        applies D through the rank slabs; the odd-even Schur system is
        single-rank, as in the reference."""
        from .gmres import SolveReport, gmres_solve
        from .gmres import solve_dirac as single_rank_solve
        if odd_even:
            return single_rank_solve(params, gauge, clover, eta, cfg, odd_even=True, psi0=psi0)
        res = gmres_solve(self.operator(params, gauge, clover), eta, psi0, cfg)
        return SolveReport(res.psi, res, False, res.final_relnorms, res.iterations)


class _ExecutorOp:
    """GMRES operator view of a MultiRankExecutor (device fields)."""

    allreduce = None

    def __init__(self, ex: MultiRankExecutor, params, gauge, clover):
        self.ex, self.params, self.gauge, self.clover = ex, params, gauge, clover
        self.n_sites = gauge.geom.n_sites

    def apply_device(self, v: DeviceField, out: DeviceField | None = None, scale=None) -> DeviceField:
        return self.ex.apply_device(self.params, self.gauge, self.clover, v, out, scale)


def apply_dirac_multirank(params, gauge, clover, psi, grid: RankGrid, mode: str = "sequential",
                          timeout: float = DEFAULT_TIMEOUT):
    """One-shot multi-rank apply; returns (result, executor) (halo.py:390-401)."""
    ex = MultiRankExecutor(grid, mode=mode, timeout=timeout)
    return ex.apply_dirac(params, gauge, clover, psi), ex
