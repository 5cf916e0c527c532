"""Command line: the reference's measurement surface on the B200 path.

``python -m paper_2601_05816_b200 <command> ...`` with the reference CLI's
record formats (cli.py:96-184):

* ``bench-dirac``: per (nrhs, layout) the median D_W apply time and the
  reference's record fields (b, layout, seconds, gflops from the 2574
  flop/site/rhs ledger, ai, bytes, checksums), plus the B200 columns:
  device-resident time (CUDA events), site*rhs/s, algorithmic HBM GB/s and the
  fraction of the measured HBM peak.
* ``solve``: batched GMRES (full or odd-even), writes ``psi.snap`` and
  ``history.csv`` (iter, rhs, relnorm) and prints the final explicit relnorms.
* ``gen-fields``: writes gauge / clover / psi snapshots (fields.py:266-337).

Every command first prints the JSON header {version, config_hash, seed, rng}
(cli.py:60-67).  Exit codes: 0 ok, 1 invalid arguments, 2 numerical
failure, 3 internal error (cli.py:405-424).
"""

from __future__ import annotations

import argparse
import csv
import hashlib
import json
import os
import statistics
import sys
import time

import numpy as np

from . import __version__
from .fields import (RNG_ALGORITHM, flip_time_boundary, gen_clover, gen_gauge, gen_spinor,
                     near_unit_gauge, write_clover, write_gauge, write_spinor)
from .geometry import LatticeGeometry


class NumericalFailure(RuntimeError):
    pass


class UsageError(ValueError):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def _checksum(data) -> str:
    return hashlib.sha256(np.ascontiguousarray(data).tobytes()).hexdigest()[:16]


def _header(args) -> None:
    text = json.dumps({k: v for k, v in sorted(vars(args).items()) if k != "func"}, default=str)
    print(json.dumps({"version": __version__, "config_hash": hashlib.sha256(text.encode()).hexdigest()[:12],
                      "seed": args.seed, "rng": RNG_ALGORITHM}))


def _ints(text: str) -> list[int]:
    return [int(p) for p in text.replace(",", " ").split()]


def _fields(args, b: int, layout: int):
    geom = LatticeGeometry(tuple(_ints(args.dims)))
    if args.gauge == "near-unit":
        gauge = near_unit_gauge(geom, args.eps, args.seed)
    else:
        gauge = gen_gauge(geom, args.gauge, seed=args.seed)
    if args.antiperiodic:
        gauge = flip_time_boundary(gauge)
    clover = gen_clover(geom, args.clover, args.clover_scale, seed=args.seed + 1)
    psi = gen_spinor(geom.n_sites, b, layout, seed=args.seed + 2, geom=geom)
    return geom, gauge, clover, psi


def cmd_bench_dirac(args) -> int:
    import torch

    from .device import upload
    from .dirac import FLOPS_PER_SITE_RHS, DiracOperator, DiracParams, account_traffic, compulsory_bytes_per_site

    _header(args)
    peak = 6546.6
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = float(json.load(open(pk))["hbm_gbs"])
    records = []
    for b in _ints(args.b_list):
        for layout in _ints(args.layouts):
            geom, gauge, clover, psi = _fields(args, b, layout)
            op = DiracOperator(DiracParams(m0=args.m0), gauge, clover, args.dtype)
            times = []
            op.apply_host_pipelined(psi)  # warm-up
            for _ in range(args.reps):
                t0 = time.perf_counter()
                op.apply_host_pipelined(psi)
                times.append(time.perf_counter() - t0)
            seconds = statistics.median(times)
            d = upload(psi, args.dtype)
            out = d.empty_like()
            op.apply_device(d, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                op.apply_device(d, out)
            e1.record()
            torch.cuda.synchronize()
            dev_s = e0.elapsed_time(e1) * 1e-3 / args.reps
            flops = FLOPS_PER_SITE_RHS * geom.n_sites * b
            led = account_traffic(b)
            alg = compulsory_bytes_per_site(b, args.dtype) * geom.n_sites
            records.append({
                "b": b, "layout": layout, "seconds": seconds, "gflops": flops / seconds / 1e9,
                "ai": FLOPS_PER_SITE_RHS * b / led["bytes_per_site"], "flops": flops,
                "bytes": led["bytes_per_site"] * geom.n_sites,
                "checksums": {"gauge": _checksum(gauge.data), "clover": _checksum(clover.data),
                              "psi": _checksum(psi.data)},
                "device_seconds": dev_s, "site_rhs_per_s": geom.n_sites * b / dev_s,
                "hbm_gbs": alg / dev_s / 1e9, "roofline_frac": alg / dev_s / 1e9 / peak, "dtype": args.dtype,
            })
    text = json.dumps({"records": records}, indent=2)
    print(text)
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text + "\n")
    return 0


def cmd_solve(args) -> int:
    from .dirac import DiracParams
    from .gmres import GmresConfig, solve_dirac

    _header(args)
    _, gauge, clover, eta = _fields(args, args.b, args.layout)
    cfg = GmresConfig(restart_len=args.restart_len, restarts=args.restarts, tol=args.tol,
                      fixed_iterations=args.fixed_iterations)
    rep = solve_dirac(DiracParams(m0=args.m0), gauge, clover, eta, cfg, odd_even=args.odd_even)
    psi_path = f"{args.out}psi.snap" if args.out else "psi.snap"
    hist_path = f"{args.out}history.csv" if args.out else "history.csv"
    for path in (psi_path, hist_path):
        if os.path.dirname(path):
            os.makedirs(os.path.dirname(path), exist_ok=True)
    write_spinor(psi_path, rep.psi)
    with open(hist_path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "rhs", "relnorm"])
        for it, rel in enumerate(rep.result.history):
            for r in range(len(rel)):
                w.writerow([it, r, repr(float(rel[r]))])
    for r, rel in enumerate(rep.full_relnorms):
        print(f"rhs {r}: final explicit relnorm {rel:.6e}")
    ok = bool(np.all(rep.full_relnorms <= args.tol))
    print(json.dumps({"iterations": rep.iterations, "odd_even": rep.odd_even,
                      "converged": ok if not args.fixed_iterations else None, "psi": psi_path, "history": hist_path}))
    if not args.fixed_iterations and not ok:
        raise NumericalFailure(f"solver did not reach tol {args.tol:g}; worst relnorm {rep.full_relnorms.max():.3e}")
    return 0


def cmd_gen_fields(args) -> int:
    _header(args)
    _, gauge, clover, psi = _fields(args, args.b, args.layout)
    pre = args.out or ""
    paths = {"gauge": f"{pre}gauge.snap", "clover": f"{pre}clover.snap", "psi": f"{pre}psi.snap"}
    for p in paths.values():
        if os.path.dirname(p):
            os.makedirs(os.path.dirname(p), exist_ok=True)
    write_gauge(paths["gauge"], gauge)
    write_clover(paths["clover"], clover)
    write_spinor(paths["psi"], psi)
    print(json.dumps({"files": paths, "checksums": {"gauge": _checksum(gauge.data), "clover": _checksum(clover.data),
                                                    "psi": _checksum(psi.data)}}, indent=2))
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="paper_2601_05816_b200")
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)

    def common(sp):
        sp.add_argument("--dims", default="8 8 8 8", help="T X Y Z (T slowest)")
        sp.add_argument("--m0", type=float, default=0.1)
        sp.add_argument("--seed", type=int, default=0, help="gauge=seed, clover=seed+1, psi=seed+2 (cli.py:81-86)")
        sp.add_argument("--gauge", choices=["unit", "random", "near-unit"], default="random")
        sp.add_argument("--eps", type=float, default=0.3)
        sp.add_argument("--antiperiodic", action="store_true", help="antiperiodic T (U_0 flipped on the last slice)")
        sp.add_argument("--clover", choices=["zero", "random"], default="zero")
        sp.add_argument("--clover-scale", type=float, default=0.1)
        sp.add_argument("--out", default=None)

    sp = sub.add_parser("bench-dirac")
    common(sp)
    sp.add_argument("--b-list", default="1 2 4 8 16")
    sp.add_argument("--layouts", default="2")
    sp.add_argument("--reps", type=int, default=5)
    sp.add_argument("--dtype", choices=["c128", "c64"], default="c128")
    sp.set_defaults(func=cmd_bench_dirac)

    sp = sub.add_parser("solve")
    common(sp)
    sp.add_argument("--b", type=int, default=4)
    sp.add_argument("--layout", type=int, default=2)
    sp.add_argument("--restart-len", type=int, default=30)
    sp.add_argument("--restarts", type=int, default=67)
    sp.add_argument("--tol", type=float, default=1e-10)
    sp.add_argument("--fixed-iterations", action="store_true")
    sp.add_argument("--odd-even", action="store_true")
    sp.set_defaults(func=cmd_solve)

    sp = sub.add_parser("gen-fields")
    common(sp)
    sp.add_argument("--b", type=int, default=4)
    sp.add_argument("--layout", type=int, default=2)
    sp.set_defaults(func=cmd_gen_fields)
    return p


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        return args.func(args)
    except (UsageError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except NumericalFailure as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return 2
    except Exception as exc:  # noqa: BLE001 - map to the reference's internal-error code
        print(f"internal error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
