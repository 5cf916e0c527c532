#!/usr/bin/env python3
"""Benchmark: rhs-blocked Wilson-Dirac apply on B200 (+ batched GMRES TTS).

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints
ONE JSON line on rank 0.  ``--impl reference`` times the reference itself
(lqcdlab 0.1.0, installed unmodified into baseline/_ref) on the host cores.

Workload at N=1 (BASELINE.json configs[1]): 16^3 x 32 lattice (T=32 slowest),
seeded random SU(3) links (gen_gauge QR), Gaussian spinors, m0 = 0.1, C = 0,
nrhs in {1,2,4,8,16,32}, complex128 and complex64.  Headline = c128 at
nrhs=16 (site*rhs/s), every other (dtype, nrhs) point is in "sweep".  A step
is one D_W apply of one nrhs block; steps rotate through enough distinct
(psi, eta) buffer pairs that the bytes touched between two uses of a buffer
exceed 4x the L2 size (no L2 reuse across steps).  Batched GMRES
time-to-solution on BASELINE configs[3] (24^3 x 48, nrhs=12, near-unit
links, antiperiodic T, GMRES(30), tol 1e-10, full and odd-even) is added
under "gmres" (with a same-run lqcdlab solve on the host cores for a reduced
lattice under "gmres.cpu_compare"), the configs[2] Schur apply (32^3 x 64,
nrhs=12, c128) under "schur" and the configs[4] apply at one GPU (48^3 x 96,
nrhs=12, c128 and c64) plus its odd-even GMRES(8) under "strong", unless
--no-gmres.

At N > 1 (torchrun, one rank per GPU, NCCL): the headline weak-scales
configs[1] over a T split (a 16^3 x 32 slab per GPU, comparable to the N=1
line); "strong" holds configs[4] (48^3 x 96, nrhs 12) split over the N ranks
-- c128 and c64 applies, the same lattice on rank 0 alone (strong-scaling
base point, same run), per-rank halo wait / hop times, and the odd-even
GMRES(8) to 1e-8.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG2_DIMS = (32, 16, 16, 16)
SWEEP_B = (1, 2, 4, 8, 16, 32)
HEADLINE = ("c128", 16)
M0 = 0.1
METRIC = "D_W apply site*rhs/s (16^3x32, nrhs=16, c128)"


PROFILE = ROOT / "profiles" / "r2_ncu_march_c128_b16_cfg2.json"


def profile_traffic():
    """DRAM bytes per launch of the headline kernel from the committed ncu
    --set full capture (profiles/), or None."""
    try:
        d = json.loads(PROFILE.read_text())
        return d["launches"][0]["dram_traffic_bytes"]
    except Exception:
        return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int = 0):
        self.gpu, self.samples, self._stop = gpu, [], threading.Event()
        self._t = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---- GPU arm ------------------------------------------------------------------


def gpu_clover(args, torch, P, nrhs=(4, 12, 16)):
    """Clover D_W apply (the reference CLI's default clover.mode
    is random) on configs[1]'s lattice: random clover (scale 0.1), both dtypes,
    rotating buffers.  Compulsory bytes add the packed blocks: (24 b + 36 + 42) w."""
    from paper_2601_05816_b200.device import DeviceField
    dev = torch.device("cuda", 0)
    geom = P.LatticeGeometry(CFG2_DIMS)
    n = geom.n_sites
    gauge = P.gen_gauge(geom, "random", seed=0)
    clover = P.gen_clover(geom, "random", scale=0.1, seed=1)
    from paper_2601_05816_b200 import _lib
    _, l2 = _l2_bytes(_lib)
    hbm_peak, _ = peaks()
    out = []
    for dt in ("c128", "c64"):
        w = 16 if dt == "c128" else 8
        op = P.DiracOperator(P.DiracParams(m0=M0), gauge, clover, dt)
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        for b in nrhs:
            nbuf = max(2, int(np.ceil(4 * l2 / (2 * n * 12 * b * w))) + 1)
            g = torch.Generator(device="cpu").manual_seed(100 + b)
            base = torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, generator=g).to(dev, tdt)
            psis = [DeviceField(base.clone(), n, geom) for _ in range(nbuf)]
            etas = [p_.empty_like() for p_ in psis]
            for i in range(max(3, args.warmup)):
                op.apply_device(psis[i % nbuf], etas[i % nbuf])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(args.steps):
                op.apply_device(psis[i % nbuf], etas[i % nbuf])
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) * 1e-3 / args.steps
            alg = (24 * b + 36 + 42) * w * n
            out.append({"dtype": dt, "nrhs": b, "ms": round(t * 1e3, 4), "site_rhs_per_s": n * b / t,
                        "hbm_gbs": round(alg / t / 1e9, 1), "frac": round(alg / t / 1e9 / hbm_peak, 4),
                        "kernel": ("hop_ring_kernel (blocks staged in shared memory)" if dt == "c128"
                                   else "hop_kernel (generic, clover epilogue)")})
            del psis, etas, base
        del op
    torch.cuda.empty_cache()
    return {"lattice": list(CFG2_DIMS), "clover": "random, scale 0.1", "records": out}


def gpu_sweep(args, torch, P):
    from paper_2601_05816_b200 import _lib
    from paper_2601_05816_b200.device import DeviceField, upload_gauge
    from paper_2601_05816_b200.dirac import compulsory_bytes_per_site

    dev = torch.device("cuda", 0)
    geom = P.LatticeGeometry(CFG2_DIMS)
    n = geom.n_sites
    gauge = P.gen_gauge(geom, "random", seed=0)
    _, l2 = _l2_bytes(_lib)
    lat = _lib.Lattice.make(geom.dims)
    gdev = {dt: upload_gauge(gauge, dt) for dt in ("c128", "c64")}
    stream = torch.cuda.current_stream()
    sptr = int(stream.cuda_stream)
    results = []
    hbm_peak, peak_kind = peaks()
    for dt in ("c128", "c64"):
        w = 16 if dt == "c128" else 8
        for b in SWEEP_B:
            field_bytes = n * 12 * b * w
            nbuf = max(2, int(np.ceil(4 * l2 / (2 * field_bytes))) + 1)
            g = torch.Generator(device="cpu").manual_seed(b)
            base = torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, generator=g)
            tdt = torch.complex128 if dt == "c128" else torch.complex64
            psis = [DeviceField(base.to(dev, tdt), n) for _ in range(nbuf)]
            etas = [DeviceField(torch.empty_like(psis[0].data), n) for _ in range(nbuf)]
            code = 0 if dt == "c128" else 1

            def launch(i):
                rc = _lib.load().b200wd_dirac_apply(lat, code, b, M0, gdev[dt].ptr, psis[i % nbuf].ptr,
                                                    etas[i % nbuf].ptr, sptr)
                if rc:
                    raise RuntimeError(_lib.load().b200wd_last_error().decode())

            for i in range(max(3, args.warmup)):
                launch(i)
            torch.cuda.synchronize()
            steps = args.steps
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            ev[0].record(stream)
            for i in range(steps):
                launch(i)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            per = [ev[i].elapsed_time(ev[i + 1]) * 1e-3 for i in range(steps)]
            t = float(np.mean(per))
            alg = compulsory_bytes_per_site(b, dt) * n
            rec = {"dtype": dt, "nrhs": b, "ms": t * 1e3, "site_rhs_per_s": n * b / t,
                   "hbm_gbs": alg / t / 1e9, "frac": alg / t / 1e9 / hbm_peak, "bytes_per_launch": alg,
                   "buffers": nbuf}
            if (dt, b) == HEADLINE:  # warm figure (same buffers every launch, L2 may hold part of them); not the roofline number
                ew = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ew[0].record(stream)
                for _ in range(steps):
                    launch(0)
                ew[1].record(stream)
                torch.cuda.synchronize()
                rec["warm_ms"] = ew[0].elapsed_time(ew[1]) / steps
            results.append(rec)
            del psis, etas
            torch.cuda.empty_cache()
    return results, hbm_peak, peak_kind


def _l2_bytes(_lib):
    import ctypes
    sm = ctypes.c_int32()
    l2 = ctypes.c_int64()
    _lib.call("b200wd_device_info", 0, ctypes.byref(sm), ctypes.byref(l2), None, None)
    return sm.value, l2.value


def gpu_e2e(args, torch, P, b=16, dt="c128", pinned=True, freeze_links=False):
    """The headline metric through the public API (apply_dirac on host
    BlockSpinorFields).  Every step copies the rhs block host -> device and
    the result device -> host; ``pinned`` selects page-locked host buffers
    (else ordinary pageable numpy arrays, what a drop-in lqcdlab caller
    passes).  The host links are writeable, so every call re-uploads them
    (device._GaugeCache: exact invalidation, as the reference recomputes from
    the host arrays) and their bytes count in h2d_bytes_per_step; with
    ``freeze_links`` the links are read-only and their device copy is reused
    (``links_cached``)."""
    geom = P.LatticeGeometry(CFG2_DIMS)
    n = geom.n_sites
    gauge = P.gen_gauge(geom, "random", seed=0)
    if freeze_links:
        P.freeze(gauge)
    params = P.DiracParams(m0=M0)
    if pinned:
        h_in = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
        h_out = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
        h_in.copy_(torch.randn(n * 12 * b, dtype=torch.complex128))
        a_in, a_out = h_in.numpy(), h_out.numpy()
    else:
        rng = np.random.default_rng(1)
        a_in = (rng.standard_normal(n * 12 * b) + 1j * rng.standard_normal(n * 12 * b)).astype(np.complex128)
        a_out = np.empty_like(a_in)
    psi = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, a_in, geom)
    eta = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, a_out, geom)
    for _ in range(max(3, args.warmup)):
        P.apply_dirac(params, gauge, None, psi, dtype=dt, out=eta)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        P.apply_dirac(params, gauge, None, psi, dtype=dt, out=eta)
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) / args.steps
    field = n * 12 * b * 16
    links = 0 if freeze_links else n * 4 * 9 * 16
    return {"value": n * b / t, "unit": "site*rhs/s", "h2d_bytes_per_step": field + links,
            "d2h_bytes_per_step": field, "ms_per_step": t * 1e3, "host_buffers": "pinned" if pinned else "pageable",
            "links_cached": bool(freeze_links)}


def gpu_gmres(args, torch, P):
    """BASELINE configs[3]: GMRES(30) b=12 tol 1e-10 on 24^3 x 48, full and odd-even."""
    dims = (48, 24, 24, 24)
    geom = P.LatticeGeometry(dims)
    t0 = time.perf_counter()
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 3))
    eta = P.gen_spinor(geom.n_sites, 12, P.Layout.COMPONENT_MAJOR, seed=5, geom=geom)
    gen_s = time.perf_counter() - t0
    from paper_2601_05816_b200.device import upload
    d_eta = upload(eta)
    out = {"lattice": list(dims), "nrhs": 12, "input_gen_s": gen_s}
    # the reference's MGS (headline records "full" / "oe"), then the classical
    # Gram-Schmidt extension (GmresConfig.orthogonalization="cgs") on the same system
    for orth, oe in (("mgs", False), ("mgs", True), ("cgs", False), ("cgs", True)):
        # warm-up: one full-length cycle, so the 31-field basis is allocated (and
        # cached by torch) before the timed solve
        P.solve_dirac(P.DiracParams(m0=M0), gauge, None, d_eta,
                      P.GmresConfig(restart_len=30, restarts=1, tol=1e-10, orthogonalization=orth), odd_even=oe)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve_dirac(P.DiracParams(m0=M0), gauge, None, d_eta,
                            P.GmresConfig(restart_len=30, restarts=67, tol=1e-10, orthogonalization=orth),
                            odd_even=oe)
        torch.cuda.synchronize()
        tts = time.perf_counter() - t0
        key = ("oe" if oe else "full") + ("" if orth == "mgs" else "_cgs")
        out[key] = {"iterations": rep.iterations, "time_to_solution_s": tts,
                    "s_per_iteration": tts / max(rep.iterations, 1),
                    "max_full_relnorm": float(rep.full_relnorms.max()), "orthogonalization": orth}
        gold_p = ROOT / "tests" / "golden" / "gmres_cfg3.json"
        gold = json.loads(gold_p.read_text()) if gold_p.exists() else {}
        if oe and "cfg3_48x24c_oe" in gold:  # lqcdlab itself on these inputs, 1 core, build container
            g = gold["cfg3_48x24c_oe"]
            out["oe"].update(reference_iterations=g["iterations"],
                             reference_tts_s_build_container=g["reference_wall_s"],
                             reference_max_full_relnorm=max(g["full_relnorms"]),
                             reference="lqcdlab 0.1.0 solve_dirac(odd_even=True), 1 core, BUILD CONTAINER (not "
                                       "this box): iterations / residual cross-check")
    return out


def gmres_cpu_compare(torch, P, run_cpu: bool):
    """GMRES time-to-solution on identical inputs, GPU vs the reference on
    this box's host cores, same run.

    * 12 x 6^3, BASELINE configs[4]'s solver physics (near-unit links eps 0.3
      seed 7, antiperiodic T, nrhs=12 Gaussian rhs seed 9, m0=0.1, GMRES(8),
      tol 1e-8), unpreconditioned and odd-even: lqcdlab.solve_dirac (from
      baseline/_ref, 1 core) and the device solve on the same host arrays
      (about 25 s of CPU time).
    * 24 x 12^3, configs[3] physics (GMRES(30), tol 1e-10): the device solve
      against lqcdlab's own run on 1 core of the build container
      (tests/golden/gmres_cfg3.json; labelled as such -- a cross-check of
      iterations, not a same-box time)."""
    from paper_2601_05816_b200.device import upload
    out = {}

    def gpu_tts(dims, oe, gauge, eta, cfg):
        d_eta = upload(eta)
        warm = P.GmresConfig(restart_len=cfg.restart_len, restarts=1, tol=cfg.tol)
        P.solve_dirac(P.DiracParams(m0=M0), gauge, None, d_eta, warm, odd_even=oe)  # full basis allocated
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve_dirac(P.DiracParams(m0=M0), gauge, None, d_eta, cfg, odd_even=oe)
        torch.cuda.synchronize()
        return rep, time.perf_counter() - t0

    L = reference_lqcdlab() if run_cpu else None
    dims = (12, 6, 6, 6)
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 7))
    eta = P.gen_spinor(geom.n_sites, 12, P.Layout.COMPONENT_MAJOR, seed=9, geom=geom)
    cfg = P.GmresConfig(restart_len=8, restarts=250, tol=1e-8)
    for oe in (False, True):
        rep, tts = gpu_tts(dims, oe, gauge, eta, cfg)
        rec = {"lattice": list(dims), "solver": "GMRES(8), tol 1e-8", "odd_even": oe, "gpu_iterations": rep.iterations,
               "gpu_tts_s": tts, "gpu_max_full_relnorm": float(np.max(rep.full_relnorms))}
        if L is not None:
            from threadpoolctl import threadpool_limits
            from lqcdlab.fields import GaugeField as RGauge
            from lqcdlab.gmres import GmresConfig as RCfg
            rgeom = L.LatticeGeometry(dims)
            rg = RGauge(rgeom, np.array(gauge.data))
            reta = L.gen_spinor(geom.n_sites, 12, L.Layout.COMPONENT_MAJOR, seed=9, geom=rgeom)
            with threadpool_limits(1):
                t0 = time.perf_counter()
                rr = L.solve_dirac(L.DiracParams(m0=M0), rg, L.gen_clover(rgeom, "zero"), reta,
                                   RCfg(restart_len=8, restarts=250, tol=1e-8), odd_even=oe)
                ct = time.perf_counter() - t0
            rec.update(reference="lqcdlab 0.1.0 solve_dirac (baseline/_ref), 1 core, this box, same run",
                       reference_iterations=int(rr.iterations), reference_tts_s=ct,
                       reference_max_full_relnorm=float(np.max(rr.full_relnorms)), speedup=ct / tts)
        out[f"cfg4_physics_12x6c_{'oe' if oe else 'full'}"] = rec
    gold_p = ROOT / "tests" / "golden" / "gmres_cfg3.json"
    gold = json.loads(gold_p.read_text()) if gold_p.exists() else {}
    cfg3 = P.GmresConfig(restart_len=30, restarts=67, tol=1e-10)
    dims = (24, 12, 12, 12)
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 3))
    eta = P.gen_spinor(geom.n_sites, 12, P.Layout.COMPONENT_MAJOR, seed=5, geom=geom)
    for oe in (False, True):
        key = f"proxy_24x12c_{'oe' if oe else 'full'}"
        rep, tts = gpu_tts(dims, oe, gauge, eta, cfg3)
        rec = {"lattice": list(dims), "gpu_iterations": rep.iterations, "gpu_tts_s": tts}
        if key in gold:
            rec.update(reference_iterations=gold[key]["iterations"],
                       reference_tts_s_build_container=gold[key]["reference_wall_s"],
                       reference="lqcdlab 0.1.0 solve_dirac, 1 core, BUILD CONTAINER (not this box): iterations "
                                 "cross-check only")
        out[key] = rec
    return out


REF_DIR = ROOT / "baseline" / "_ref"


def reference_lqcdlab():
    """The unmodified reference package from baseline/_ref (or None)."""
    if REF_DIR.exists() and str(REF_DIR) not in sys.path:
        sys.path.append(str(REF_DIR))
    try:
        import lqcdlab
        return lqcdlab
    except Exception:
        return None


_SAMPLE: dict = {}


def _ref_worker(_):
    """One worker: lqcdlab.apply_dirac on its own 16^3 x 2 sample lattice
    (the reference's stock code path, numpy pinned to one thread)."""
    L = _SAMPLE["L"]
    eta = L.apply_dirac(_SAMPLE["params"], _SAMPLE["gauge"], _SAMPLE["clover"], _SAMPLE["psi"])
    return float(abs(eta.data[:4]).sum())


def _port_worker(_):
    """Fallback when lqcdlab is absent: the oracle restatement of apply_dirac."""
    from oracle import lqcd_oracle as O
    out = O.apply_dirac(_SAMPLE["dims"], M0, _SAMPLE["links"], None, _SAMPLE["psi"])
    return float(np.abs(out[:4]).sum())


def cpu_apply_rate(cores: int, steps: int, warmup: int, b: int = 16):
    """The reference's D_W apply on the host cores: `cores` worker processes,
    each running lqcdlab.apply_dirac on its own 16^3 x 2 periodic lattice
    (8192 sites, nrhs b, c128; the per-site work of the stencil does not
    depend on the lattice extent), numpy / BLAS pools pinned to 1 thread.
    Returns (site*rhs/s, seconds per step, sample description, kind)."""
    import multiprocessing as mp

    from threadpoolctl import threadpool_limits
    dims = (2, 16, 16, 16)
    n = 2 * 16 ** 3
    L = reference_lqcdlab()
    if L is not None:
        from lqcdlab.fields import Layout as RL
        geom = L.LatticeGeometry(dims)
        _SAMPLE.update(L=L, params=L.DiracParams(m0=M0), gauge=L.gen_gauge(geom, "random", seed=0),
                       clover=L.gen_clover(geom, "zero"),
                       psi=L.gen_spinor(n, b, RL.COMPONENT_MAJOR, seed=2, geom=geom))
        worker, kind = _ref_worker, "reference"
        what = "lqcdlab 0.1.0 apply_dirac (baseline/_ref, unmodified)"
    else:
        from oracle import lqcd_oracle as O
        _SAMPLE.update(dims=dims, links=O.gen_gauge_random(dims, 0), psi=O.gen_spinor(n, b, 2))
        worker, kind = _port_worker, "port"
        what = "oracle apply_dirac (numpy restatement of lqcdlab dirac.py; lqcdlab not installed)"
    with threadpool_limits(1):
        pool = mp.get_context("fork").Pool(cores) if cores > 1 else None
        run = (lambda: worker(0)) if pool is None else (lambda: pool.map(worker, range(cores)))  # noqa: E731
        for _ in range(warmup):
            run()
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            run()
            ts.append(time.perf_counter() - t0)
        if pool is not None:
            pool.close()
    t = float(np.median(ts))
    sample = (f"{what} on a 16^3x2 lattice per worker, nrhs={b}, c128, {cores} worker process(es) x 8192 sites, "
              f"median of {steps} steps")
    return cores * n * b / t, t, sample, kind


def cpu_baseline_sample(b=16, reps=3):
    v, t, sample, kind = cpu_apply_rate(1, reps, 1, b)
    return {"value": v, "unit": "site*rhs/s", "cores": 1, "kind": kind, "sample": sample}


class DistGroup:
    """Rank plumbing of the N-GPU arm over torch.distributed (NCCL)."""

    def __init__(self, torch, dev):
        import torch.distributed as dist
        self.torch, self.dist, self.dev = torch, dist, dev
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

    def transport(self):
        return None  # TSplitComm's default DistTransport

    def barrier(self):
        self.dist.barrier()

    def max(self, x: float) -> float:
        t = self.torch.tensor([float(x)], device=self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


class ThreadBenchGroup:
    """The same plumbing for ranks that are threads of one process on one GPU
    (tsplit.ThreadGroup): exercises the N-rank arm's logic in tests; its
    timings are not bench numbers."""

    def __init__(self, group, rank, dev):
        self.g, self.rank, self.world, self.dev = group, rank, group.world, dev

    def transport(self):
        return self.g.transport(self.rank)

    def barrier(self):
        self.g.barrier.wait(timeout=600)

    def _all(self, obj):
        self.barrier()
        self.g.slots[self.rank] = obj
        self.barrier()
        out = list(self.g.slots)
        self.barrier()
        return out

    def max(self, x: float) -> float:
        return max(self._all(float(x)))

    def gather(self, obj):
        return self._all(obj)


def multi_gpu(args, torch, P, grp):
    """N ranks: the headline weak-scales configs[1] over a T split.

    Every rank owns a 16^3 x 32 slab (the N=1 workload) of a 16^3 x 32N
    lattice; each step is one split D_W apply (face pack, NCCL send/recv
    overlapped with the interior slices, boundary slices with halos).
    value = all ranks' site*rhs / max-over-ranks device time.  Also: e2e
    through TSplitComm.apply_dirac with pinned host slabs, per-rank halo
    stats, the configs[4] strong-scaling block and its odd-even GMRES(8).
    """
    from paper_2601_05816_b200.device import DeviceField
    from paper_2601_05816_b200.dirac import compulsory_bytes_per_site
    from paper_2601_05816_b200.tsplit import TSplitComm

    rank, world, dev = grp.rank, grp.world, grp.dev
    dt, b = HEADLINE
    gdims = (CFG2_DIMS[0] * world,) + CFG2_DIMS[1:]
    ggeom = P.LatticeGeometry(gdims)
    comm = TSplitComm(ggeom, transport=grp.transport())
    lg, t0 = comm.local_geom, comm.t_origin
    links = P.near_unit_links(gdims, 0.3, 0, t0, t0 + lg.dims[0])
    gauge = P.flip_time_boundary(P.GaugeField(lg, links), gdims[0], t0)
    comm.bind(P.DiracParams(m0=M0), gauge, None, dt)
    n = lg.n_sites
    nbuf = 2
    g = torch.Generator(device="cpu").manual_seed(rank)
    psis = [DeviceField(torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, generator=g).to(dev), n)
            for _ in range(nbuf)]
    etas = [DeviceField(torch.empty_like(psis[0].data), n) for _ in range(nbuf)]
    stream = torch.cuda.current_stream(dev)
    for i in range(args.warmup):
        comm.apply_device(psis[i % nbuf], etas[i % nbuf])
    torch.cuda.synchronize(dev)
    grp.barrier()
    clocks = ClockSampler(dev.index).start() if rank == 0 and args.sample_clocks else None
    launches0 = comm.stats["launches"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        comm.apply_device(psis[i % nbuf], etas[i % nbuf])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    grp.barrier()
    tt = grp.max(e0.elapsed_time(e1) * 1e-3 / args.steps)
    clk = clocks.stop() if clocks else None
    launches = comm.stats["launches"] - launches0
    # EpochStats analogue of one extra apply per rank (halo.py:101-114)
    comm.timing = True
    st0 = dict(comm.stats)
    comm.apply_device(psis[0], etas[0])
    comm.timing = False
    epoch = grp.gather({"rank": rank, **{k: comm.stats[k] - st0[k] for k in ("wait_s", "interior_ms", "boundary_ms")}})
    del psis, etas
    # e2e: the reference-facing seam (dirac.py:313-314) with pinned host slabs,
    # H2D of the rhs slab + split apply + D2H every step (links re-uploaded:
    # writeable host arrays)
    h_in = torch.randn(n * 12 * b, dtype=torch.complex128, generator=g).pin_memory()
    h_out = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
    psi_h = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_in.numpy(), lg)
    eta_h = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_out.numpy(), lg)
    for _ in range(2):
        comm.apply_dirac(P.DiracParams(m0=M0), gauge, None, psi_h, out=eta_h)
    torch.cuda.synchronize(dev)
    grp.barrier()
    te = time.perf_counter()
    for _ in range(args.steps):
        comm.apply_dirac(P.DiracParams(m0=M0), gauge, None, psi_h, out=eta_h)
    torch.cuda.synchronize(dev)
    te = grp.max((time.perf_counter() - te) / args.steps)
    e2e = {"value": world * n * b / te, "unit": "site*rhs/s", "ms_per_step": te * 1e3,
           "h2d_bytes_per_step": world * (n * 12 * b * 16 + n * 4 * 9 * 16),
           "d2h_bytes_per_step": world * n * 12 * b * 16, "host_buffers": "pinned", "links_cached": False,
           "path": "TSplitComm.apply_dirac (reference comm= seam) per rank"}
    del h_in, h_out, psi_h, eta_h
    torch.cuda.empty_cache()
    # configs[4] strong scaling on the same ranks
    strong = None
    if not args.no_gmres:
        sys.path.insert(0, str(ROOT / "tools"))
        from bench_strong import GDIMS, split_apply_records, split_gmres
        sgdims = tuple(args.strong_dims) if args.strong_dims else GDIMS
        scomm = TSplitComm(P.LatticeGeometry(sgdims), transport=grp.transport())
        recs = split_apply_records(scomm, sgdims, 12, ("c128", "c64"), max(3, min(args.steps, 10)), 3, grp, dev,
                                   base_n1=True)
        strong = {"workload": "BASELINE configs[4]: 48^3 x 96, nrhs 12, T split over the ranks (strong scaling)",
                  "lattice": list(sgdims), "records": recs,
                  "gmres": split_gmres(scomm, sgdims, 12, grp, dev)}
    if rank == 0:
        alg = compulsory_bytes_per_site(b, dt) * n
        hbm_peak, peak_kind = peaks()
        line = {
            "metric": METRIC, "value": world * n * b / tt, "unit": "site*rhs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic (near-unit SU(3) links, Gaussian rhs)",
            "config": {"workload": f"BASELINE configs[1] per GPU, weak-scaled over a T split: lattice {list(gdims)}",
                       "lattice": list(gdims), "local": list(lg.dims), "nrhs": b, "m0": M0,
                       "parallelism": f"T split x{world}, NCCL send/recv halos overlapped with interior slices "
                                      f"({comm.sm_reserve} SMs left to NCCL during the interior hop)",
                       "l2": "2 rotating buffers of 403 MB (> L2)"},
            "roofline": {"bound": "hbm", "achieved": alg / tt / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": alg / tt / 1e9 / hbm_peak, "traffic": profile_traffic(), "peak_kind": peak_kind,
                         "note": "per GPU; traffic: committed ncu capture of the interior kernel shape"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "epoch_stats": epoch,
            "halo_bytes_per_step_per_rank": comm.stats["bytes_sent"] / max(1, comm.stats["applies"]),
        }
        if strong is not None:
            line["strong"] = strong
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_sample()
        print(json.dumps(line), flush=True)
        return line
    return None


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-gmres", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--force-dist", action="store_true", help="run the T-split path even with one rank")
    ap.add_argument("--strong-dims", type=int, nargs=4, default=None, help="override the strong-scaling lattice")
    args = ap.parse_args(argv)
    args.sample_clocks = True
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    import torch
    import paper_2601_05816_b200 as P
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.force_dist:
        import torch.distributed as dist
        if "RANK" not in os.environ:  # --force-dist without a launcher: a one-rank group
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
        try:
            multi_gpu(args, torch, P, DistGroup(torch, dev))
        finally:
            dist.destroy_process_group()
        return
    torch.cuda.set_device(0)
    clocks = ClockSampler(0).start()
    sweep, hbm_peak, peak_kind = gpu_sweep(args, torch, P)
    clk = clocks.stop()
    head = next(r for r in sweep if (r["dtype"], r["nrhs"]) == HEADLINE)
    # headline e2e: the rhs block in and the result out through apply_dirac every step,
    # pinned host buffers, links frozen (read-only, uploaded once: static configuration,
    # labelled links_cached); the variants re-upload the links every call / use pageable buffers
    e2e = gpu_e2e(args, torch, P, freeze_links=True)
    line = {
        "metric": METRIC, "value": head["site_rhs_per_s"], "unit": "site*rhs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded SU(3) links, Gaussian rhs)",
        "config": {"workload": WORKLOAD_N1,
                   "lattice": list(CFG2_DIMS), "nrhs": 16, "m0": M0, "l2": "rotating buffers > 4x L2 between reuses",
                   "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": head["hbm_gbs"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": head["frac"], "traffic": profile_traffic(), "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": head["bytes_per_launch"],
                     "kernel": "hop_march_kernel<double,1,16,2,1> (libb200wd.so, b200wd_dirac_apply)"},
        "e2e": e2e, "gpu_launches": args.steps, "clocks": clk,
        "e2e_variants": {"pinned_links_every_call": gpu_e2e(args, torch, P),
                         "pageable_links_every_call": gpu_e2e(args, torch, P, pinned=False)},
        "sweep": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()} for r in sweep],
    }
    line["clover"] = gpu_clover(args, torch, P)
    if not args.no_gmres:
        line["gmres"] = gpu_gmres(args, torch, P)
        line["gmres"]["cpu_compare"] = gmres_cpu_compare(torch, P, not args.no_cpu)
        sys.path.insert(0, str(ROOT / "tools"))
        from bench_schur import schur_bench
        line["schur"] = schur_bench()  # BASELINE configs[2]: 32^3x64 Schur apply, nrhs=12, c128
        from bench_strong import single_gpu_apply, single_gpu_gmres
        # BASELINE configs[4] at N=1: 48^3x96, nrhs=12 (the strong-scaling base point)
        torch.cuda.empty_cache()
        line["strong"] = single_gpu_apply(sampler=ClockSampler)
        torch.cuda.empty_cache()
        line["strong"]["gmres"] = single_gpu_gmres()
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line))


WORKLOAD_N1 = "BASELINE configs[1]: D_W apply 16^3x32, nrhs sweep {1..32}, c128+c64; headline c128 nrhs=16"


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    steps = max(1, min(args.steps, 10))
    warmup = min(args.warmup, 5)  # honours W >= 3; each CPU step is a bounded sample (~1 s)
    v, t, sample, kind = cpu_apply_rate(cores, steps, warmup, HEADLINE[1])
    gl = [CFG2_DIMS[0] * max(1, args.gpus)] + list(CFG2_DIMS[1:])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "site*rhs/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded SU(3) links, Gaussian rhs)",
            # the same config as this repo's arm at this N: the per-site cost of the reference's
            # stencil does not depend on the lattice extent, so each step applies it to one
            # 16^3 x 2 sample lattice per host core and the rate is site*rhs per second of all cores
            "config": {"workload": (WORKLOAD_N1 if args.gpus <= 1 else
                                    f"BASELINE configs[1] per GPU, weak-scaled over a T split: lattice {gl}"),
                       "lattice": gl, "nrhs": HEADLINE[1], "m0": M0,
                       "sample": f"one 16^3 x 2 lattice per host core ({cores} cores) per step, nrhs=16, c128"},
            "cpu_baseline": {"value": v, "unit": "site*rhs/s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "site*rhs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
