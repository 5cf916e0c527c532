"""Command line: the reference CLI (``lqcdlab``, cli.py:1-424) on the B200 path.

``python -m paper_2601_05816_b200 <command> [--config FILE] [--set KEY=VALUE ...]``
takes the reference's run-config files and overrides (``config.py``; the
canonical text and hash are the reference's for reference keys) and writes
the reference's records:

* ``bench-dirac [--b-list ...] [--layout-list ...] [--reps N]``: per
  (nrhs, layout) the median apply time through the host-field API and the
  reference's record fields (b, layout, seconds, gflops from the 2574
  flop/site/rhs ledger, ai, flops, bytes, checksums), plus the B200 columns:
  device-resident time (CUDA events), site*rhs/s, algorithmic HBM GB/s and
  the fraction of the measured HBM peak, dtype;
* ``solve``: batched GMRES (full or odd-even; ``ranks.grid`` > 1 runs the
  apply through ``MultiRankExecutor``), writes ``psi.snap`` and
  ``history.csv`` (iter, rhs, relnorm), prints the final explicit relnorms;
* ``gen-fields``: gauge / clover / psi snapshots (fields.py:266-337).

* ``oracle-check [--corrupt-gauge]``: invariant suites evaluated with the
  device kernels (unitarity, free field, gamma5-hermiticity, Schur identity).

``stream``, ``roofline`` and ``cost-model`` (the CPU model tools) are not part
of the B200 path and exit with status 1.  Every
command first prints the JSON header {version, config_hash, seed, rng}
(cli.py:60-67).  Exit codes: 0 ok, 1 invalid configuration or arguments,
2 numerical failure, 3 internal error (cli.py:405-424).
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
from .config import ConfigError, RunConfig, canonical, layout_of, load_config, set_key, validate
from .fields import (RNG_ALGORITHM, flip_time_boundary, gen_clover, gen_gauge, gen_spinor, near_unit_gauge,
                     write_clover, write_gauge, write_spinor)
from .geometry import LatticeGeometry, RankGrid, decompose


class NumericalFailure(RuntimeError):
    pass


class UsageError(ConfigError):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise UsageError(message)


def _checksum(data) -> str:
    return hashlib.sha256(np.ascontiguousarray(data).tobytes()).hexdigest()[:16]


def _header(cfg: RunConfig) -> None:
    print(json.dumps({"version": __version__,
                      "config_hash": hashlib.sha256(canonical(cfg).encode()).hexdigest()[:12],
                      "seed": cfg.seed, "rng": RNG_ALGORITHM}))


def _runconfig(args) -> RunConfig:
    """--config file, then every --set KEY=VALUE, then validation (cli.py:70-78)."""
    cfg = load_config(args.config) if args.config else RunConfig()
    for item in args.set or []:
        key, sep, value = item.partition("=")
        if not sep:
            raise ConfigError(f"--set needs key=value, got {item!r}")
        set_key(cfg, key.strip(), value.strip())
    validate(cfg)
    return cfg


def _ints(text: str) -> list[int]:
    return [int(p) for p in text.replace(",", " ").split()]


def _out_file(path: str) -> str:
    if os.path.dirname(path):
        os.makedirs(os.path.dirname(path), exist_ok=True)
    return path


def _gauge_clover(cfg: RunConfig):
    geom = LatticeGeometry(tuple(cfg.dims))
    if cfg.gauge_mode == "near-unit":
        gauge = near_unit_gauge(geom, cfg.gauge_eps, cfg.seed)
    else:
        gauge = gen_gauge(geom, cfg.gauge_mode, seed=cfg.seed)
    if cfg.antiperiodic_time:
        gauge = flip_time_boundary(gauge)
    clover = gen_clover(geom, cfg.clover_mode, cfg.clover_scale, seed=cfg.seed + 1)
    return geom, gauge, clover


def _problem(cfg: RunConfig, b: int | None = None, layout: int | None = None):
    """Seeds: gauge = seed, clover = seed+1, spinor = seed+2 (cli.py:81-86)."""
    geom, gauge, clover = _gauge_clover(cfg)
    psi = gen_spinor(geom.n_sites, cfg.b if b is None else b, layout_of(cfg) if layout is None else layout,
                     seed=cfg.seed + 2, geom=geom)
    return geom, gauge, clover, psi


def cmd_bench_dirac(args) -> int:
    import torch

    from .device import upload
    from .dirac import FLOPS_PER_SITE_RHS, DiracOperator, DiracParams, account_traffic, compulsory_bytes_per_site
    from .perf import arithmetic_intensity

    cfg = _runconfig(args)
    _header(cfg)
    peak = 6546.6
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    b_list = _ints(args.b_list) if args.b_list else [cfg.b]
    layouts = _ints(args.layout_list) if args.layout_list else [cfg.layout]
    geom, gauge, clover = _gauge_clover(cfg)
    op = DiracOperator(DiracParams(m0=cfg.m0), gauge, clover, cfg.dtype)
    records = []
    for b in b_list:
        for layout in layouts:
            psi = gen_spinor(geom.n_sites, b, layout, seed=cfg.seed + 2, geom=geom)
            op.apply_host_pipelined(psi)  # warm-up
            times = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                op.apply_host_pipelined(psi)
                times.append(time.perf_counter() - t0)
            seconds = statistics.median(times)
            d = upload(psi, cfg.dtype)
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
            alg = compulsory_bytes_per_site(b, cfg.dtype) * geom.n_sites
            records.append({
                "b": b, "layout": layout, "seconds": seconds, "gflops": flops / seconds / 1e9,
                "ai": float(arithmetic_intensity(b)), "flops": flops,
                "bytes": account_traffic(b)["bytes_per_site"] * geom.n_sites,
                "checksums": {"gauge": _checksum(gauge.data), "clover": _checksum(clover.data),
                              "psi": _checksum(psi.data)},
                "device_seconds": dev_s, "site_rhs_per_s": geom.n_sites * b / dev_s,
                "hbm_gbs": alg / dev_s / 1e9, "roofline_frac": alg / dev_s / 1e9 / peak, "dtype": cfg.dtype,
            })
    text = json.dumps({"records": records}, indent=2)
    print(text)
    if cfg.out_path:
        with open(_out_file(cfg.out_path), "w", encoding="utf-8") as fh:
            fh.write(text + "\n")
    return 0


def cmd_solve(args) -> int:
    from .dirac import DiracParams
    from .gmres import GmresConfig, solve_dirac
    from .multirank import MultiRankExecutor

    cfg = _runconfig(args)
    _header(cfg)
    geom, gauge, clover, eta = _problem(cfg)
    gcfg = GmresConfig(restart_len=cfg.restart_len, restarts=cfg.restarts, tol=cfg.tol,
                       fixed_iterations=cfg.fixed_iterations, orthogonalization=cfg.orthogonalization)
    comm = None
    if any(g > 1 for g in cfg.grid):
        grid = RankGrid(tuple(cfg.grid))
        decompose(geom, grid)  # validate before building the executor
        comm = MultiRankExecutor(grid)
    rep = solve_dirac(DiracParams(m0=cfg.m0), gauge, clover, eta, gcfg, odd_even=cfg.odd_even, comm=comm)
    psi_path = f"{cfg.out_path}psi.snap"
    hist_path = f"{cfg.out_path}history.csv"
    write_spinor(_out_file(psi_path), rep.psi)
    with open(_out_file(hist_path), "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "rhs", "relnorm"])
        for it, rel in enumerate(rep.result.history):
            for r in range(len(rel)):
                w.writerow([it, r, repr(float(rel[r]))])
    for r, rel in enumerate(rep.full_relnorms):
        print(f"rhs {r}: final explicit relnorm {rel:.6e}")
    ok = bool(np.all(rep.full_relnorms <= cfg.tol))
    print(json.dumps({"iterations": rep.iterations, "odd_even": rep.odd_even,
                      "converged": ok if not cfg.fixed_iterations else None, "psi": psi_path,
                      "history": hist_path}))
    if not cfg.fixed_iterations and not ok:
        raise NumericalFailure(f"solver did not reach tol {cfg.tol:g}; worst relnorm {rep.full_relnorms.max():.3e}")
    return 0


def cmd_gen_fields(args) -> int:
    cfg = _runconfig(args)
    _header(cfg)
    _, gauge, clover, psi = _problem(cfg)
    pre = cfg.out_path
    paths = {"gauge": f"{pre}gauge.snap", "clover": f"{pre}clover.snap", "psi": f"{pre}psi.snap"}
    write_gauge(_out_file(paths["gauge"]), gauge)
    write_clover(_out_file(paths["clover"]), clover)
    write_spinor(_out_file(paths["psi"]), psi)
    print(json.dumps({"files": paths, "checksums": {"gauge": _checksum(gauge.data), "clover": _checksum(clover.data),
                                                    "psi": _checksum(psi.data)}}, indent=2))
    return 0


def cmd_oracle_check(args) -> int:
    """Invariant suites of the B200 operators, evaluated with device kernels
    (cli.py:190-268 runs dense-matrix suites on the CPU; here every suite is a
    property that needs no CPU reference): link unitarity, the free-field
    identity D psi = m0 psi (unit links, constant psi), gamma5-hermiticity
    <phi, g5 D psi> = <g5 D phi, psi> at nrhs 1 and 8, and the Schur
    complement identity (D x)_e = S v_e, (D x)_o = 0 for x = (v_e, -D_oo^-1
    D_oe v_e).  Any failing suite -> exit status 2."""
    import torch

    from .device import DeviceField, upload
    from .dirac import DiracOperator, DiracParams
    from .fields import BlockSpinorField, GaugeField
    from .oddeven import SchurOperator, device_merge, device_split

    cfg = _runconfig(args)
    _header(cfg)
    geom, gauge, clover = _gauge_clover(cfg)
    if args.corrupt_gauge:
        gauge = GaugeField(geom, gauge.data.copy())
        gauge.data[0, 0, 0, 0] += 0.5
    params = DiracParams(m0=cfg.m0)
    tol = 1e-12 if cfg.dtype == "c128" else 1e-5
    g5 = torch.tensor([1.0] * 6 + [-1.0] * 6, dtype=torch.float64)
    failures = []

    def suite(name: str, fn) -> None:
        try:
            print(f"{name}: PASS ({fn()})")
        except Exception as exc:  # report, keep running the other suites
            print(f"{name}: FAIL ({exc})")
            failures.append(name)

    def unitarity():
        links = gauge.data
        if cfg.antiperiodic_time:  # undo the boundary sign before the SU(3) test
            links = flip_time_boundary(GaugeField(geom, links)).data
        GaugeField(geom, links).validate()
        return "links unitary, det 1" + (" (up to the antiperiodic T sign)" if cfg.antiperiodic_time else "")

    def free_field():
        unit = gen_gauge(geom, "unit")
        psi = BlockSpinorField.zeros(geom.n_sites, 2, layout_of(cfg), geom=geom)
        psi.set_ksi(np.ones((geom.n_sites, 12, 2), dtype=np.complex128))
        eta = DiracOperator(params, unit, None, cfg.dtype)(psi)
        err = float(np.abs(eta.ksi() - params.m0 * psi.ksi()).max())
        if err > (1e-14 if cfg.dtype == "c128" else 1e-6):
            raise NumericalFailure(f"max err {err:.3e}")
        return f"max err {err:.3e}"

    def gamma5(b: int):
        def run():
            op = DiracOperator(params, gauge, clover, cfg.dtype)
            phi = upload(gen_spinor(geom.n_sites, b, 2, seed=cfg.seed + 3, geom=geom), cfg.dtype)
            psi = upload(gen_spinor(geom.n_sites, b, 2, seed=cfg.seed + 4, geom=geom), cfg.dtype)
            g = g5.to(phi.data.device).view(1, 12, 1, 1)
            dphi, dpsi = op.apply_device(phi).data, op.apply_device(psi).data
            lhs = (phi.data.conj() * g * dpsi).sum(dim=(0, 1, 2))
            rhs = ((g * dphi).conj() * psi.data).sum(dim=(0, 1, 2))
            err = float(((lhs - rhs).abs().max() / lhs.abs().max()).item())
            if err > tol:
                raise NumericalFailure(f"rel err {err:.3e}")
            return f"rel err {err:.3e}"
        return run

    def schur_identity():
        schur = SchurOperator(params, gauge, clover, keep_parity=0, dtype=cfg.dtype)
        dirac = DiracOperator(params, gauge, clover, cfg.dtype)
        half = geom.n_sites // 2
        v = upload(gen_spinor(half, 2, 2, seed=cfg.seed + 5), cfg.dtype, parity=0)
        v.geom = geom
        zero = DeviceField(torch.zeros_like(v.data), half, geom, 1)
        x = device_merge(schur.lat, v, schur.reconstruct_device(v, zero), geom)
        ye, yo = device_split(schur.lat, dirac.apply_device(x))
        sv = schur.apply_device(v)
        e1 = float((torch.linalg.vector_norm(ye.data - sv.data) / torch.linalg.vector_norm(sv.data)).item())
        e2 = float((torch.linalg.vector_norm(yo.data) / torch.linalg.vector_norm(ye.data)).item())
        if e1 > tol or e2 > tol:
            raise NumericalFailure(f"rel err {e1:.3e} (even), {e2:.3e} (odd)")
        return f"rel err {e1:.3e} (even), {e2:.3e} (odd)"

    suite("gauge-unitarity", unitarity)
    suite("free-field-identity", free_field)
    suite("gamma5-hermiticity-b1", gamma5(1))
    suite("gamma5-hermiticity-b8", gamma5(8))
    suite("schur-identity", schur_identity)
    if failures:
        raise NumericalFailure("failing suites: " + ", ".join(failures))
    return 0


def cmd_not_provided(args) -> int:
    raise UsageError(f"'{args.command}' is a CPU-model tool of the reference CLI and is not part of the B200 "
                     "path (DESIGN.md section 7)")


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="paper_2601_05816_b200", description=__doc__)
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)

    def runconfig_args(sp):
        sp.add_argument("--config", help="path to a key = value config file")
        sp.add_argument("--set", action="append", metavar="KEY=VALUE", help="override one config key (repeatable)")

    sp = sub.add_parser("bench-dirac", help="time the operator over b/layout sweeps")
    runconfig_args(sp)
    sp.add_argument("--b-list", help="comma/space-separated b values to sweep")
    sp.add_argument("--layout-list", help="comma/space-separated layouts to sweep")
    sp.add_argument("--reps", type=int, default=3, help="timed repetitions (median)")
    sp.set_defaults(func=cmd_bench_dirac)

    sp = sub.add_parser("solve", help="run the batched solver on a seeded problem")
    runconfig_args(sp)
    sp.set_defaults(func=cmd_solve)

    sp = sub.add_parser("gen-fields", help="write seeded gauge/clover/spinor snapshots")
    runconfig_args(sp)
    sp.set_defaults(func=cmd_gen_fields)

    sp = sub.add_parser("oracle-check", help="invariant suites of the device operators")
    runconfig_args(sp)
    sp.add_argument("--corrupt-gauge", action="store_true", help="perturb one link to demonstrate failure detection")
    sp.set_defaults(func=cmd_oracle_check)

    for name in ("stream", "roofline", "cost-model"):
        sp = sub.add_parser(name, help="reference CPU-model tool (not part of the B200 path)")
        sp.add_argument("rest", nargs=argparse.REMAINDER)
        sp.set_defaults(func=cmd_not_provided)
    return p


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        return args.func(args)
    except (ConfigError, ValueError, NotImplementedError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except (NumericalFailure, np.linalg.LinAlgError) as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return 2
    except RuntimeError as exc:
        from ._lib import B200Unavailable
        if isinstance(exc, B200Unavailable):
            print(f"internal error: {exc}", file=sys.stderr)
            return 3
        print(f"numerical failure: {exc}", file=sys.stderr)
        return 2
    except Exception as exc:  # noqa: BLE001 - map to the reference's internal-error code
        print(f"internal error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
