"""Multi-GPU T split: the `comm=` seam of the reference (dirac.py:313-314, halo.py).

One process per GPU (``torchrun --nproc-per-node N``), ``torch.distributed`` with
the NCCL backend for the plumbing.  The lattice is split along T (direction 0,
the slowest index), so each rank's slab is a contiguous range of sites and its
links and fields are ordinary local device fields of extents (T/N, X, Y, Z).

Per operator apply (halo.py:339-387 semantics, on the device):

1. ``b200wd_halo_pack``: the lambda face (sign -1 half spinor of local slice 0)
   and the chi face (U_0^H times the sign +1 half spinor of slice T_loc-1, link
   applied at the source so no links travel), 6*b complex per face site;
2. NCCL P2P: lambda -> rank-1, chi -> rank+1 (``batch_isend_irecv``), enqueued
   right after the pack;
3. the interior slices 1..T_loc-2 run concurrently with the transfers (they
   never read a halo);
4. after the receives complete, the two boundary slices consume the halos
   (``b200wd_hop`` with ``lam_halo``/``chi_halo``).

A clover term (this rank's slab of packed blocks, uploaded once in ``bind``)
rides in the epilogue of every interior and boundary hop (``b200wd_hop_clover``),
so the full apply and the distributed Schur operator take it too.

GMRES reductions are one ``all_reduce`` of the b partial sums per reducing pass.
With one rank the split degenerates to the single-GPU periodic apply.

Transports.  The face exchange and the reductions go through a transport:
``DistTransport`` (``torch.distributed``: NCCL between GPUs, gloo on CPU) or
``ThreadTransport``, the reference's in-process "threads" mode (halo.py:296-316,
one Python thread per rank, ``CommunicatorSet`` / ``_Mailbox``): ranks are
threads of one process sharing one device, every exchange is a host barrier
plus device copies, so no kernel ever waits on another rank's kernel.  It runs
the whole distributed solve (split hops, distributed Schur operator, the
all-reduce flow of ``gmres_solve``) on a single GPU for testing.

Failure detection and accounting (halo.py:43-53, 91-114): a receive that does
not complete within ``timeout_s`` raises :class:`HaloTimeoutError` naming the
rank, direction and face; ``stats`` keeps the reference's ``EpochStats``
analogue per rank -- applies, bytes sent, host time spent waiting for halos,
and the device time of the interior and boundary hops (CUDA events).
The antiperiodic time boundary rides in the links of the rank that owns global
slice T-1 (``fields.flip_time_boundary(..., t_global, t_origin)``).
"""

from __future__ import annotations

import os
import threading
import time
from datetime import timedelta

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .device import DeviceField, dtype_code, gauge_cache, ptr, require_device, stream_ptr, upload
from .fields import SPINOR_LEN
from .geometry import LatticeGeometry, t_split


def _real_view(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


class CudaHaloKernels:
    """Device kernels used by the T split (libb200wd)."""

    def pack(self, lat, dtype, b, src_parity, gauge, src, lam, chi):
        _lib.call("b200wd_halo_pack", lat, dtype_code(dtype), b, src_parity, gauge.ptr, src.ptr, ptr(lam), ptr(chi),
                  stream_ptr())

    def hop(self, lat, dtype, b, dst_parity, gauge, src, out, xself, alpha, beta, scale, t0, t1, lam=None, chi=None,
            clover=None, mode=0):
        if clover is not None:  # site-local block term in the epilogue (mode 1: -C x, 2: M (...))
            _lib.call("b200wd_hop_clover", lat, dtype_code(dtype), b, dst_parity, gauge.ptr, src.ptr,
                      None if xself is None else xself.ptr, out.ptr, float(alpha), float(beta), ptr(scale), int(t0),
                      int(t1), ptr(lam), ptr(chi), clover.ptr, int(mode), stream_ptr())
            return
        _lib.call("b200wd_hop", lat, dtype_code(dtype), b, dst_parity, gauge.ptr, src.ptr,
                  None if xself is None else xself.ptr, out.ptr, float(alpha), float(beta), ptr(scale), int(t0),
                  int(t1), ptr(lam), ptr(chi), stream_ptr())

    def hop_boundary(self, lat, dtype, b, dst_parity, gauge, src, out, xself, alpha, beta, scale, lam, chi,
                     clover=None, mode=0):
        """Both boundary slices (0 and T-1) with their halos in one launch."""
        _lib.call("b200wd_hop_boundary", lat, dtype_code(dtype), b, dst_parity, gauge.ptr, src.ptr,
                  None if xself is None else xself.ptr, out.ptr, float(alpha), float(beta), ptr(scale), ptr(lam),
                  ptr(chi), None if clover is None else clover.ptr, int(mode), stream_ptr())

    def face_buffer(self, nf, b, dtype, device):
        t = torch.complex128 if dtype == "c128" else torch.complex64
        return torch.empty((6, nf, b), dtype=t, device=device)

    def reserve_sms(self, k: int) -> int:
        """Leave k SMs free for the persistent hop kernels launched next from
        this thread (b200wd_set_sm_reserve); returns the previous value."""
        return int(_lib.load().b200wd_set_sm_reserve(int(k)))


class HaloTimeoutError(RuntimeError):
    """A halo receive did not complete in time (halo.py:43-53)."""

    def __init__(self, rank: int, mu: int, direction: str, timeout_s: float):
        self.rank, self.mu, self.direction, self.timeout_s = rank, mu, direction, timeout_s
        super().__init__(f"rank {rank}: halo receive mu={mu} from the {direction} neighbour timed out "
                         f"after {timeout_s:.1f} s")


class DistTransport:
    """Face exchange and reductions over ``torch.distributed`` (NCCL / gloo)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def allreduce(self, t: torch.Tensor) -> None:
        dist.all_reduce(_real_view(t), op=dist.ReduceOp.SUM, group=self.group)

    def exchange(self, lam, chi, lam_in, chi_in, up: int, down: int):
        # complex faces travel as their real views (NCCL has no complex dtype)
        ops = [
            dist.P2POp(dist.isend, _real_view(lam), down, self.group, tag=1),
            dist.P2POp(dist.irecv, _real_view(lam_in), up, self.group, tag=1),
            dist.P2POp(dist.isend, _real_view(chi), up, self.group, tag=2),
            dist.P2POp(dist.irecv, _real_view(chi_in), down, self.group, tag=2),
        ]
        reqs = dist.batch_isend_irecv(ops)
        # (lam_in from up, chi_in from down) per request, for error naming
        return [(r, ("up", "down")[i // 2] if len(reqs) == 4 else "up") for i, r in enumerate(reqs)]

    def wait(self, handles, timeout_s: float, rank: int) -> None:
        for r, direction in handles:
            try:
                ok = r.wait(timeout=timedelta(seconds=timeout_s)) if timeout_s else r.wait()
            except RuntimeError as e:  # gloo / NCCL report a timed-out or failed work item
                if "imeout" in str(e) or "imed out" in str(e):
                    raise HaloTimeoutError(rank, 0, direction, timeout_s) from e
                raise
            if ok is False:
                raise HaloTimeoutError(rank, 0, direction, timeout_s)


class ThreadGroup:
    """Shared state of an in-process rank group (halo.py CommunicatorSet)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots: list = [None] * world

    def transport(self, rank: int) -> "ThreadTransport":
        return ThreadTransport(self, rank)


class ThreadTransport:
    """One rank of a :class:`ThreadGroup` (a thread of this process).

    Every operation synchronises the rank's current CUDA stream, meets the
    other ranks at a host barrier and combines their tensors with device
    copies in rank order, so every rank sees bit-identical sums."""

    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.world = group, rank, group.world

    def _sync(self, t):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def _meet(self, timeout_s: float, what: str):
        try:
            self.g.barrier.wait(timeout=timeout_s or None)
        except threading.BrokenBarrierError:
            raise HaloTimeoutError(self.rank, 0, what, timeout_s) from None

    def allreduce(self, t: torch.Tensor, timeout_s: float = 120.0) -> None:
        self._sync(t)
        self.g.slots[self.rank] = t
        self._meet(timeout_s, "allreduce")
        acc = self.g.slots[0].clone()
        for r in range(1, self.world):
            acc += self.g.slots[r].to(acc.device)
        self._sync(acc)
        self._meet(timeout_s, "allreduce")
        t.copy_(acc)
        self._sync(t)

    def exchange(self, lam, chi, lam_in, chi_in, up: int, down: int, timeout_s: float = 120.0):
        self._sync(lam)
        self.g.slots[self.rank] = (lam, chi)
        self._meet(timeout_s, "exchange")
        lam_in.copy_(self.g.slots[up][0])   # lambda face of slice 0 of rank+1
        chi_in.copy_(self.g.slots[down][1])  # chi face of slice T-1 of rank-1
        self._sync(lam_in)
        self._meet(timeout_s, "exchange")
        return []

    def wait(self, handles, timeout_s: float, rank: int) -> None:
        return None


class TSplitComm:
    """T-only domain decomposition over the ranks of a process group.

    ``global_geom`` is the whole lattice; every rank owns slab
    ``[rank*T/N, (rank+1)*T/N)`` (``local_geom``, ``t_origin``).  Fields given to
    :meth:`apply_dirac` / :meth:`operator` are the rank-local slabs.
    """

    def __init__(self, global_geom: LatticeGeometry, group=None, kernels=None, device=None, transport=None,
                 timeout_s: float = 300.0):
        self.group = group
        self.transport = transport if transport is not None else DistTransport(group)
        self.world = self.transport.world
        self.rank = self.transport.rank
        self.timeout_s = timeout_s
        # SMs the interior hop leaves free while the halos are in flight, so
        # NCCL's P2P kernels are resident next to the persistent ring kernel
        # (B200WD_HALO_SMS, default 8)
        self.sm_reserve = int(os.environ.get("B200WD_HALO_SMS", "8"))
        self.global_geom = global_geom
        self.local_geom, self.t_origin = t_split(global_geom, self.world, self.rank)
        if self.world > 1 and self.local_geom.dims[0] < 2:
            raise ValueError("local T extent must be >= 2 (geometry.py:200-201)")
        self.lat = _lib.Lattice.make(self.local_geom.dims, self.t_origin)
        self.kernels = kernels or CudaHaloKernels()
        self.device = device
        self.up = (self.rank + 1) % self.world
        self.down = (self.rank - 1) % self.world
        self._faces = {}
        # EpochStats analogue (halo.py:101-114): host seconds blocked on halos,
        # device milliseconds of the interior and boundary hops
        self.stats = {"applies": 0, "bytes_sent": 0, "wait_s": 0.0, "interior_ms": 0.0, "boundary_ms": 0.0,
                      "launches": 0}
        self.timing = False  # set True to record the device hop times (adds event syncs)

    # -- plumbing -------------------------------------------------------------
    def allreduce(self, t: torch.Tensor) -> torch.Tensor:
        """Sum per-rank partial reductions (GMRES dots / norms) in place."""
        if self.world > 1:
            self.transport.allreduce(t)
        return t

    def _face_buffers(self, parity, b, dtype, device):
        key = (parity, b, dtype)
        if key not in self._faces:
            nf = self.local_geom.sites_per_slice if parity is None else self.local_geom.sites_per_slice // 2
            mk = lambda: self.kernels.face_buffer(nf, b, dtype, device)  # noqa: E731
            self._faces[key] = {"lam": mk(), "chi": mk(), "lam_in": mk(), "chi_in": mk()}
        return self._faces[key]

    def exchange(self, lam: torch.Tensor, chi: torch.Tensor, lam_in: torch.Tensor, chi_in: torch.Tensor):
        """lambda face -> rank-1, chi face -> rank+1; returns the work handles."""
        if self.world == 1:
            lam_in.copy_(lam)
            chi_in.copy_(chi)
            return []
        self.stats["bytes_sent"] += 2 * lam.numel() * lam.element_size()
        return self.transport.exchange(lam, chi, lam_in, chi_in, self.up, self.down)

    # -- the split hop ----------------------------------------------------------
    def hop(self, dst_parity, src, out, xself, alpha, beta, scale=None, gauge=None, clover=None, mode=0):
        """out = scale (alpha xself + beta H src) on the local slab with halos.

        ``dst_parity`` None/-1 for full fields, else the parity of ``out``
        (``src`` has the other parity).  ``clover`` (device packed blocks of the
        destination sites) with ``mode`` 1 subtracts C xself, mode 2 applies the
        blocks to the whole result (the Schur D_ee^-1 hop)."""
        gauge = gauge if gauge is not None else self.gauge
        par = -1 if dst_parity is None else dst_parity
        b, dtype = src.b, src.dtype
        T = self.local_geom.dims[0]
        k = self.kernels
        extra = {} if clover is None else {"clover": clover, "mode": mode}
        if self.world == 1:
            k.hop(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, 0, T, **extra)
            self.stats["launches"] += 1
            return out
        f = self._face_buffers(None if par < 0 else 1 - par, b, dtype, src.data.device)
        k.pack(self.lat, dtype, b, -1 if par < 0 else 1 - par, gauge, src, f["lam"], f["chi"])
        reqs = self.exchange(f["lam"], f["chi"], f["lam_in"], f["chi_in"])
        ev = self._events() if self.timing else None
        if ev:
            ev[0].record()
        if T > 2:
            prev = k.reserve_sms(self.sm_reserve) if hasattr(k, "reserve_sms") else None
            try:
                k.hop(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, 1, T - 1, **extra)
            finally:
                if prev is not None:
                    k.reserve_sms(prev)
        if ev:
            ev[1].record()
        t_w = time.perf_counter()
        self.transport.wait(reqs, self.timeout_s, self.rank)
        self.stats["wait_s"] += time.perf_counter() - t_w
        if ev:
            ev[2].record()
        # both boundary slices in one launch (b200wd_hop_boundary); kernels
        # without it (test stand-ins) take one launch per slice
        if hasattr(k, "hop_boundary"):
            k.hop_boundary(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, f["lam_in"],
                           f["chi_in"], **extra)
        elif T == 2:
            k.hop(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, 0, 2, f["lam_in"],
                  f["chi_in"], **extra)
        else:
            k.hop(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, 0, 1, f["lam_in"],
                  f["chi_in"], **extra)
            k.hop(self.lat, dtype, b, par, gauge, src, out, xself, alpha, beta, scale, T - 1, T, f["lam_in"],
                  f["chi_in"], **extra)
        if ev:
            ev[3].record()
            ev[3].synchronize()
            self.stats["interior_ms"] += ev[0].elapsed_time(ev[1])
            self.stats["boundary_ms"] += ev[2].elapsed_time(ev[3])
        self.stats["applies"] += 1
        # pack + interior (T > 2) + boundary slices (one launch with hop_boundary)
        self.stats["launches"] += 1 + (1 if T > 2 else 0) + (1 if (T == 2 or hasattr(k, "hop_boundary")) else 2)
        return out

    def _events(self):
        if not torch.cuda.is_available():
            return None
        if not hasattr(self, "_ev"):
            self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        return self._ev

    # -- reference comm protocol ----------------------------------------------------
    def bind(self, params, gauge, clover=None, dtype="c128"):
        """Attach the local links and clover (this rank's slab) and mass; returns self."""
        from .dirac import clover_is_zero
        if gauge.geom.dims != self.local_geom.dims:
            raise ValueError(f"gauge slab {gauge.geom.dims} != local geometry {self.local_geom.dims}")
        self.params = params
        self.dtype = dtype
        self.gauge = gauge_cache.get(gauge, dtype)
        if clover_is_zero(clover):
            self.clover = None
        else:
            if clover.geom.dims != self.local_geom.dims:
                raise ValueError(f"clover slab {clover.geom.dims} != local geometry {self.local_geom.dims}")
            self.clover = gauge_cache.get_clover(clover, dtype)  # exact invalidation (device._GaugeCache)
        return self

    def apply_device(self, v: DeviceField, out: DeviceField | None = None, scale=None) -> DeviceField:
        out = v.empty_like() if out is None else out
        return self.hop(None, v, out, v, 4.0 + self.params.m0, -1.0, scale, clover=self.clover,
                        mode=0 if self.clover is None else 1)

    def __call__(self, v):
        if isinstance(v, DeviceField):
            return self.apply_device(v)
        return self.apply_device(upload(v, self.dtype)).to_host(v.layout)

    def apply_dirac(self, params, gauge, clover, psi, flops=None, perf=None, out=None):
        """dirac.py:313-314 seam: psi and gauge are this rank's T slab.
        ``out`` (a host BlockSpinorField of psi's shape) receives a host result
        in place, as ``dirac.apply_dirac(..., out=)`` does."""
        if psi.s != SPINOR_LEN or psi.n_sites != self.local_geom.n_sites:
            raise ValueError(f"field has {psi.n_sites} sites / s={psi.s}; local slab has "
                             f"{self.local_geom.n_sites} sites")
        t0 = time.perf_counter()
        dtype = psi.dtype if isinstance(psi, DeviceField) else "c128"
        self.bind(params, gauge, clover, dtype)
        if out is not None and not isinstance(psi, DeviceField):
            res = self.apply_device(upload(psi, self.dtype)).to_host(out.layout, out=out)
        else:
            res = self(psi)
        if flops is not None:
            flops.add_apply(psi.n_sites, psi.b)
        if perf is not None:
            from .dirac import DiracPerfRecord, account_traffic
            require_device()
            torch.cuda.synchronize()
            led = account_traffic(psi.b)
            perf.append(DiracPerfRecord(time.perf_counter() - t0, psi.n_sites, psi.b, int(psi.layout),
                                        led["flops_per_site"] * psi.n_sites, led["bytes_per_site"] * psi.n_sites))
        return res

    def operator(self, params, gauge, clover=None, dtype="c128"):
        return self.bind(params, gauge, clover, dtype)

    def schur(self, params, gauge, clover=None, dtype="c128", keep_parity=0):
        """Distributed Schur operator (parity-restricted split hops)."""
        from .oddeven import SchurOperator
        self.bind(params, gauge, clover, dtype)
        return SchurOperator(params, gauge, clover, keep_parity=keep_parity, dtype=dtype, lattice=self.lat,
                             gauge_dev=self.gauge, comm=self)

    def solve_dirac(self, params, gauge, clover, eta, cfg, odd_even=False, psi0=None):
        """gmres.py:353-385 on the split lattice (eta: this rank's slab)."""
        from .blas import block_norm2_device
        from .gmres import SolveReport, _sub, gmres_solve
        from .oddeven import device_split
        host = not isinstance(eta, DeviceField)
        d_eta = upload(eta, "c128") if host else eta
        gauge = gauge_cache.get(gauge, "c128")  # one upload of this rank's links per solve
        op = self.operator(params, gauge, clover, "c128")
        if not odd_even:
            res = gmres_solve(op, d_eta, psi0, cfg)
            psi, full = res.psi, res.final_relnorms
        else:
            schur = self.schur(params, gauge, clover, "c128")
            keep, elim = device_split(self.lat, d_eta)
            reduced = schur.reduce_rhs_device(keep, elim)
            x0 = None
            if psi0 is not None:
                x0, _ = device_split(self.lat, upload(psi0) if not isinstance(psi0, DeviceField) else psi0)
            res = gmres_solve(schur, reduced, x0, cfg)
            x_elim = schur.reconstruct_device(res.psi, elim)
            psi = schur.merge(res.psi, x_elim)
            r = op.apply_device(psi)
            rn = self.allreduce(block_norm2_device(_sub(d_eta, r)))
            en = self.allreduce(block_norm2_device(d_eta))
            en = np.sqrt(en.real.cpu().numpy())
            full = np.where(en > 0, np.sqrt(rn.real.cpu().numpy()) / np.maximum(en, 1e-300), 0.0)
        if host:
            psi = psi.to_host(eta.layout)
        return SolveReport(psi, res, odd_even, full, res.iterations)
