"""BASELINE configs[4]: 48^3 x 96 (10.6M sites), nrhs=12, T split over the ranks.

    python tools/bench_strong.py [--gmres]                       # 1 GPU
    torchrun --nproc-per-node N tools/bench_strong.py            # N GPUs

D_W apply in complex128 and complex64 at every rank count (strong scaling:
the global lattice is fixed, each rank owns 96/N T slices), time = max over
ranks of CUDA-event time per apply.  With --gmres also the odd-even batched
GMRES(8) to relative tolerance 1e-8 (the Schur system on a Gaussian
even-parity rhs; the configs run it on 8 GPUs, here on however many ranks
there are).  Links: near-unit SU(3), eps = 0.3, generated per T slab with
forked workers (same bits as the serial generator).  Prints one JSON line per
measurement.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200.device import DeviceField  # noqa: E402
from paper_2601_05816_b200.dirac import compulsory_bytes_per_site  # noqa: E402

GDIMS = (96, 48, 48, 48)
M0 = 0.1


def hbm_peak():
    pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    return float(json.loads(pk.read_text())["hbm_gbs"]) if pk.exists() else 7672.0


def single_gpu_apply(gdims=GDIMS, dtypes=("c128", "c64"), b=12, steps=30, warmup=3, sampler=None):
    """configs[4] at N=1 (the strong-scaling base point): D_W apply records.

    ``ms`` is the sustained rate (back-to-back launches); ``ms_after_idle`` one
    launch after 1 s of idle GPU.  The two differ because the sustained apply
    on this lattice reaches the board power limit (1000 W, sw_power_cap,
    SM clocks ~1635 MHz): ``clocks`` (``sampler``: bench.ClockSampler) shows it."""
    geom = P.LatticeGeometry(tuple(gdims))
    tg = time.perf_counter()
    gauge = P.flip_time_boundary(P.GaugeField(geom, P.near_unit_links(gdims, 0.3, 0, workers=os.cpu_count() or 1)))
    gen_s = time.perf_counter() - tg
    n, peak, out = geom.n_sites, hbm_peak(), []
    for dt in dtypes:
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        g = torch.Generator(device="cuda").manual_seed(0)
        psi = DeviceField(torch.randn((n // 8, 12, 8, b), dtype=tdt, device="cuda", generator=g), n, geom)
        eta = psi.empty_like()
        op = P.DiracOperator(P.DiracParams(m0=M0), gauge, None, dt)
        for _ in range(warmup):
            op.apply_device(psi, eta)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        time.sleep(1.0)
        e0.record()
        op.apply_device(psi, eta)
        e1.record()
        torch.cuda.synchronize()
        t_idle = e0.elapsed_time(e1) * 1e-3
        clk = sampler(torch.cuda.current_device()).start() if sampler else None
        e0.record()
        for _ in range(steps):
            op.apply_device(psi, eta)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / steps
        alg = compulsory_bytes_per_site(b, dt) * n
        rec = {"dtype": dt, "nrhs": b, "ms": round(t * 1e3, 4), "site_rhs_per_s": n * b / t,
               "hbm_gbs": round(alg / t / 1e9, 1), "frac": round(alg / t / 1e9 / peak, 4),
               "ms_after_idle": round(t_idle * 1e3, 4), "frac_after_idle": round(alg / t_idle / 1e9 / peak, 4)}
        if clk:
            rec["clocks"] = clk.stop()
        out.append(rec)
        del psi, eta, op
    from paper_2601_05816_b200.device import gauge_cache
    gauge_cache.clear()
    torch.cuda.empty_cache()
    return {"workload": "BASELINE configs[4] at 1 GPU (strong-scaling base point)", "lattice": list(gdims),
            "records": out, "link_gen_s": round(gen_s, 2), "l2": "fields 24.5 GB (c128) >> L2"}


def split_apply_records(comm, gdims, b, dtypes, steps, warmup, grp, dev, base_n1=False):
    """D_W apply of the T-split global lattice `gdims` (each rank its slab of
    `comm`), random device fields and links (kernel time does not depend on
    the values).  Times are max over ranks (``grp.max``).  With ``base_n1``
    rank 0 also times the whole lattice on its own GPU (the strong-scaling
    base point from the same code, same run), while the other ranks wait."""
    from paper_2601_05816_b200.device import DeviceGauge
    lg, world = comm.local_geom, comm.world
    n = lg.n_sites
    peak = hbm_peak()
    out = []
    for dt in dtypes:
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        g = torch.Generator(device=dev).manual_seed(7 + comm.rank)
        links = torch.randn((4, n // 8, 9, 8), dtype=tdt, device=dev, generator=g)
        comm.bind(P.DiracParams(m0=M0), DeviceGauge(links, lg), None, dt)
        psi = DeviceField(torch.randn((n // 8, 12, 8, b), dtype=tdt, device=dev, generator=g), n, lg)
        eta = psi.empty_like()
        for _ in range(warmup):
            comm.apply_device(psi, eta)
        torch.cuda.synchronize()
        grp.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            comm.apply_device(psi, eta)
        e1.record()
        torch.cuda.synchronize()
        t = grp.max(e0.elapsed_time(e1) * 1e-3 / steps)
        # per-rank halo accounting of one extra apply (EpochStats analogue, halo.py:101-114)
        comm.timing = True
        st0 = dict(comm.stats)
        comm.apply_device(psi, eta)
        comm.timing = False
        ep = {k: comm.stats[k] - st0[k] for k in ("wait_s", "interior_ms", "boundary_ms")}
        ep["rank"] = comm.rank
        alg = compulsory_bytes_per_site(b, dt) * n
        rec = {"dtype": dt, "nrhs": b, "n_gpus": world, "local": list(lg.dims), "ms": round(t * 1e3, 4),
               "site_rhs_per_s": world * n * b / t, "hbm_gbs_per_gpu": round(alg / t / 1e9, 1),
               "frac_per_gpu": round(alg / t / 1e9 / peak, 4), "epoch_stats": grp.gather(ep)}
        del psi, eta, links
        comm.gauge = None
        torch.cuda.empty_cache()
        if base_n1 and world > 1:
            grp.barrier()
            if comm.rank == 0:
                gg = P.LatticeGeometry(tuple(gdims))
                ng = gg.n_sites
                gl = torch.randn((4, ng // 8, 9, 8), dtype=tdt, device=dev, generator=g)
                x = DeviceField(torch.randn((ng // 8, 12, 8, b), dtype=tdt, device=dev, generator=g), ng, gg)
                y = x.empty_like()
                op = P.DiracOperator(P.DiracParams(m0=M0), DeviceGauge(gl, gg), None, dt)
                for _ in range(warmup):
                    op.apply_device(x, y)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(steps):
                    op.apply_device(x, y)
                e1.record()
                torch.cuda.synchronize()
                t1 = e0.elapsed_time(e1) * 1e-3 / steps
                rec["base_n1_ms"] = round(t1 * 1e3, 4)
                rec["strong_efficiency"] = round(t1 / (world * t), 4)
                del gl, x, y, op
                torch.cuda.empty_cache()
            grp.barrier()
        out.append(rec)
    return out


def split_gmres(comm, gdims, b, grp, dev, restart_len=8, tol=1e-8, eps=0.3):
    """configs[4] odd-even batched GMRES(8) to tol 1e-8 on the T split: the
    even-site Schur system S x_e = eta_e (TSplitComm.schur: parity-restricted
    split hops, all-reduced GMRES reductions) with near-unit links (this
    rank's slab, generated per T slice) and a Gaussian even-parity rhs.  The
    full odd-even pipeline (reduce_rhs / reconstruct / full residual) needs
    the full-lattice rhs and solution next to the 9-vector basis, ~190 GB at
    one GPU; it is exercised at world 2-8 by tests/test_gpu_tsplit_solve.py."""
    lg, t0 = comm.local_geom, comm.t_origin
    tg = time.perf_counter()
    links = P.near_unit_links(gdims, eps, 0, t0, t0 + lg.dims[0],
                              workers=max(1, (os.cpu_count() or 1) // max(1, comm.world)))
    gauge = P.flip_time_boundary(P.GaugeField(lg, links), gdims[0], t0)
    del links
    gen_s = time.perf_counter() - tg
    op = comm.schur(P.DiracParams(m0=M0), gauge, None)
    ne = lg.n_sites // 2
    g = torch.Generator(device=dev).manual_seed(100 + comm.rank)
    eta_e = DeviceField(torch.randn((ne // 8, 12, 8, b), dtype=torch.complex128, device=dev, generator=g),
                        ne, lg, 0)
    cfg = P.GmresConfig(restart_len=restart_len, restarts=250, tol=tol)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    grp.barrier()
    t1 = time.perf_counter()
    res = P.gmres_solve(op, eta_e, None, cfg)
    torch.cuda.synchronize()
    tts = grp.max(time.perf_counter() - t1)
    fin = float(grp.max(float(np.max(res.final_relnorms))))
    rec = {"workload": "BASELINE configs[4] odd-even batched GMRES(8), tol 1e-8 (even-site Schur system, "
                       "Gaussian rhs)", "lattice": list(gdims), "n_gpus": comm.world, "nrhs": b,
           "iterations": res.iterations, "time_to_solution_s": tts,
           "ms_per_iteration": tts / max(res.iterations, 1) * 1e3, "max_final_relnorm": fin,
           "converged": bool(fin <= tol), "link_gen_s": round(gen_s, 2),
           "peak_mem_gb_rank0": torch.cuda.max_memory_allocated(dev) / 1e9}
    del op, eta_e, res, gauge
    comm.gauge = None
    torch.cuda.empty_cache()
    return rec


class LocalGroup:
    """One-rank stand-in of bench.py's rank group."""

    rank, world = 0, 1

    def barrier(self):
        pass

    def max(self, x):
        return float(x)

    def gather(self, obj):
        return [obj]


def single_gpu_gmres(gdims=GDIMS, b=12):
    """configs[4]'s odd-even GMRES(8) to 1e-8 on one GPU (the N=1 point of
    the strong-scaling solve): TSplitComm with one rank is the single-GPU path."""
    from paper_2601_05816_b200.tsplit import TSplitComm
    dev = torch.device("cuda", torch.cuda.current_device())
    comm = TSplitComm(P.LatticeGeometry(tuple(gdims)))
    rec = split_gmres(comm, tuple(gdims), b, LocalGroup(), dev)
    from paper_2601_05816_b200.device import gauge_cache
    gauge_cache.clear()
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--b", type=int, default=12)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dtypes", default="c128,c64")
    ap.add_argument("--gmres", action="store_true")
    ap.add_argument("--dims", type=int, nargs=4, default=list(GDIMS))
    a = ap.parse_args()
    gdims = tuple(a.dims)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = 0
    comm = None
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
        rank = dist.get_rank()
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        from paper_2601_05816_b200.tsplit import TSplitComm
        comm = TSplitComm(P.LatticeGeometry(gdims))
        lg, t0 = comm.local_geom, comm.t_origin
    else:
        lg, t0 = P.LatticeGeometry(gdims), 0
    dev = torch.device("cuda", torch.cuda.current_device())
    tg = time.perf_counter()
    links = P.near_unit_links(gdims, 0.3, 0, t0, t0 + lg.dims[0], workers=max(1, (os.cpu_count() or 1) // world))
    gauge = P.flip_time_boundary(P.GaugeField(lg, links), gdims[0], t0)
    del links
    gen_s = time.perf_counter() - tg
    n, b = lg.n_sites, a.b
    peak = hbm_peak()

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / a.steps], device=dev, dtype=torch.float64)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for dt in a.dtypes.split(","):
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        g = torch.Generator(device=dev).manual_seed(rank)
        psi = DeviceField(torch.randn((n // 8, 12, 8, b), dtype=tdt, device=dev, generator=g), n, lg)
        eta = psi.empty_like()
        if comm is not None:
            comm.bind(P.DiracParams(m0=M0), gauge, None, dt)
            t = timed(lambda: comm.apply_device(psi, eta))
        else:
            op = P.DiracOperator(P.DiracParams(m0=M0), gauge, None, dt)
            t = timed(lambda: op.apply_device(psi, eta))
        alg = compulsory_bytes_per_site(b, dt) * n
        if rank == 0:
            print(json.dumps({
                "config": "BASELINE configs[4] D_W apply (strong scaling)", "lattice": list(gdims),
                "local": list(lg.dims), "n_gpus": world, "nrhs": b, "dtype": dt, "ms_per_apply": t * 1e3,
                "site_rhs_per_s": world * n * b / t, "hbm_gbs_per_gpu": alg / t / 1e9,
                "frac_per_gpu": alg / t / 1e9 / peak, "link_gen_s": gen_s}), flush=True)
        del psi, eta
        torch.cuda.empty_cache()

    if a.gmres:
        from paper_2601_05816_b200.oddeven import SchurOperator
        if comm is not None:
            op = comm.schur(P.DiracParams(m0=M0), gauge, None)
        else:
            op = SchurOperator(P.DiracParams(m0=M0), gauge, None, keep_parity=0)
        ne = n // 2
        g = torch.Generator(device=dev).manual_seed(100 + rank)
        eta_e = DeviceField(torch.randn((ne // 8, 12, 8, b), dtype=torch.complex128, device=dev, generator=g),
                            ne, lg, 0)
        cfg = P.GmresConfig(restart_len=8, restarts=250, tol=1e-8)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t1 = time.perf_counter()
        res = P.gmres_solve(op, eta_e, None, cfg)
        torch.cuda.synchronize()
        tts = time.perf_counter() - t1
        if rank == 0:
            print(json.dumps({
                "config": "BASELINE configs[4] odd-even batched GMRES(8), tol 1e-8 (Schur system)",
                "lattice": list(gdims), "n_gpus": world, "nrhs": b, "iterations": res.iterations,
                "time_to_solution_s": tts, "ms_per_iteration": tts / max(res.iterations, 1) * 1e3,
                "converged": bool(res.converged.all()), "final_relnorm_max": float(res.final_relnorms.max()),
                "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
