"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by ``lqcdlab`` 0.1.0 itself (the reference under
/root/reference/pkg/src/lqcdlab).  Inputs come from the reference's own
generators (``gen_gauge``/``gen_clover``/``gen_spinor``, fields.py:140-263);
the harness-only inputs the reference lacks (near-unit links and the
antiperiodic-T link flip) come from
``oracle.lqcd_oracle`` and are then fed to the reference unchanged.  The
fixtures are small (<= a few hundred KB each); on the GPU box, where
/root/reference does not exist, they are the only link to the reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import lqcdlab as L  # noqa: E402
from lqcdlab.fields import BlockSpinorField, GaugeField, Layout  # noqa: E402
from lqcdlab.gmres import GmresConfig, dirac_op, gmres_solve, solve_dirac  # noqa: E402

from oracle import lqcd_oracle as O  # noqa: E402

CHECK_SEED = 999


def weights(n: int, s: int = 12) -> np.ndarray:
    """Fixed pseudo-random checksum weights w[x,k] (same formula in tests)."""
    rng = np.random.Generator(np.random.PCG64(CHECK_SEED))
    return rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))


def checksum(logical: np.ndarray) -> np.ndarray:
    """(b,) complex: sum_{x,k} w[x,k] * field[x,k,r]."""
    n, s, _ = logical.shape
    return np.einsum("xk,xkb->b", weights(n, s), logical)


def gen_checksums():
    out = {}
    geom = L.LatticeGeometry((4, 4, 4, 4))
    g = L.gen_gauge(geom, "random", seed=21).data
    out["gauge_4444_s21"] = [float(np.sum(g.real)), float(np.sum(g.imag)), g[17, 2, 1, 0].real, g[17, 2, 1, 0].imag]
    c = L.gen_clover(geom, "random", scale=0.1, seed=22).data
    out["clover_4444_s22_packed"] = [float(np.sum(c.real)), float(np.sum(c.imag)), c[5, 1, 7].real, c[5, 1, 7].imag]
    p = L.gen_spinor(256, 3, Layout.COMPONENT_MAJOR, seed=33).ksi()
    out["spinor_256x3_s33"] = [float(np.sum(p.real)), float(np.sum(p.imag)), p[200, 11, 2].real, p[200, 11, 2].imag]
    return out


def dirac_4444_clover():
    geom = L.LatticeGeometry((4, 4, 4, 4))
    gauge = L.gen_gauge(geom, "random", seed=21)
    clover = L.gen_clover(geom, "random", scale=0.1, seed=22)
    params = L.DiracParams(m0=-0.5)
    psi = L.gen_spinor(geom.n_sites, 3, Layout.COMPONENT_MAJOR, seed=33, geom=geom)
    eta = L.apply_dirac(params, gauge, clover, psi)
    np.savez_compressed(HERE / "dirac_4444_clover.npz", dims=np.array(geom.dims), m0=-0.5,
                        gauge_seed=21, clover_seed=22, psi_seed=33, b=3,
                        links=gauge.data, clover_packed=clover.data, psi=psi.ksi(), eta=eta.ksi())


def dirac_cfg1():
    """BASELINE config 1: 8^4, random SU(3) seed 0, antiperiodic T, C=0, m0=0.1, b=4."""
    geom = L.LatticeGeometry((8, 8, 8, 8))
    links = O.flip_time_boundary(L.gen_gauge(geom, "random", seed=0).data, geom.dims)
    gauge = GaugeField(geom, links)
    clover = L.gen_clover(geom, "zero")
    params = L.DiracParams(m0=0.1)
    psi = L.gen_spinor(geom.n_sites, 4, Layout.COMPONENT_MAJOR, seed=2, geom=geom)
    eta = L.apply_dirac(params, gauge, clover, psi).ksi()
    per_t = 512
    np.savez_compressed(HERE / "dirac_cfg1.npz", dims=np.array(geom.dims), m0=0.1, gauge_seed=0,
                        psi_seed=2, b=4, eta_last_slice=eta[7 * per_t:], checksum=checksum(eta),
                        norms=np.linalg.norm(eta.reshape(-1, 4), axis=0))


def schur_fixtures():
    geom = L.LatticeGeometry((4, 4, 4, 4))
    gauge = L.gen_gauge(geom, "random", seed=61)
    clover = L.gen_clover(geom, "random", scale=0.1, seed=62)
    params = L.DiracParams(m0=-0.5)
    schur = L.SchurOperator(params, gauge, clover)
    v = L.gen_spinor(schur.n_sites, 2, Layout.COMPONENT_MAJOR, seed=72)
    out = schur.apply(v).ksi()
    eta = L.gen_spinor(geom.n_sites, 2, Layout.COMPONENT_MAJOR, seed=73, geom=geom)
    reduced, eta_elim = schur.reduce_rhs(eta)
    x_odd = schur.reconstruct(reduced, eta_elim)  # back substitution with x_e := reduced rhs
    np.savez_compressed(HERE / "schur_4444_clover.npz", m0=-0.5, gauge_seed=61, clover_seed=62,
                        v_seed=72, eta_seed=73, v=v.ksi(), out=out, reduced=reduced.ksi(),
                        x_odd=x_odd.ksi())

    # C = 0, near-unit links, antiperiodic T: the GPU production case
    geom8 = L.LatticeGeometry((8, 4, 4, 4))
    links = O.flip_time_boundary(O.near_unit_gauge(geom8.dims, 0.3, 7), geom8.dims)
    gauge8 = GaugeField(geom8, links)
    zero = L.gen_clover(geom8, "zero")
    p01 = L.DiracParams(m0=0.1)
    s8 = L.SchurOperator(p01, gauge8, zero)
    v8 = L.gen_spinor(s8.n_sites, 3, Layout.COMPONENT_MAJOR, seed=74)
    out8 = s8.apply(v8).ksi()
    eta8 = L.gen_spinor(geom8.n_sites, 3, Layout.COMPONENT_MAJOR, seed=75, geom=geom8)
    red8, el8 = s8.reduce_rhs(eta8)
    xo8 = s8.reconstruct(red8, el8)
    psi8 = L.gen_spinor(geom8.n_sites, 3, Layout.COMPONENT_MAJOR, seed=76, geom=geom8)
    d8 = L.apply_dirac(p01, gauge8, zero, psi8).ksi()
    np.savez_compressed(HERE / "schur_8444_nearunit.npz", m0=0.1, eps=0.3, link_seed=7,
                        v_seed=74, eta_seed=75, psi_seed=76, out=out8, reduced=red8.ksi(),
                        x_odd=xo8.ksi(), dirac_out=d8)


def _hist(res):
    return [list(map(float, h)) for h in res.history]


def gmres_fixtures():
    out = {}
    # (a) 4^4 clover, m0=1.0, b=4 (tests/test_gmres.py:72-81)
    geom = L.LatticeGeometry((4, 4, 4, 4))
    gauge = L.gen_gauge(geom, "random", seed=81)
    clover = L.gen_clover(geom, "random", scale=0.1, seed=82)
    params = L.DiracParams(m0=1.0)
    eta = L.gen_spinor(geom.n_sites, 4, Layout.RHS_MAJOR, seed=5, geom=geom)
    res = gmres_solve(dirac_op(params, gauge, clover), eta, None, GmresConfig(tol=1e-10, restarts=40))
    out["clover_4444_m1"] = dict(dims=[4, 4, 4, 4], gauge_seed=81, clover_seed=82, m0=1.0, eta_seed=5,
                                 b=4, restart_len=10, restarts=40, tol=1e-10, iterations=res.iterations,
                                 history=_hist(res), final_relnorms=list(map(float, res.final_relnorms)),
                                 psi_checksum=[[c.real, c.imag] for c in checksum(res.psi.ksi())])
    # (b) fixed-iteration protocol (tests/test_gmres.py:96-103)
    eta7 = L.gen_spinor(geom.n_sites, 2, Layout.RHS_MAJOR, seed=7, geom=geom)
    cfg = GmresConfig(restart_len=10, restarts=10, fixed_iterations=True)
    res7 = gmres_solve(dirac_op(params, gauge, clover), eta7, None, cfg)
    out["clover_4444_fixed100"] = dict(dims=[4, 4, 4, 4], gauge_seed=81, clover_seed=82, m0=1.0, eta_seed=7,
                                       b=2, restart_len=10, restarts=10, fixed=True,
                                       iterations=res7.iterations, history=_hist(res7),
                                       final_relnorms=list(map(float, res7.final_relnorms)))
    # (c) near-unit eps=0.3, antiperiodic T, C=0, m0=0.1, b=12, GMRES(30), tol 1e-10
    #     (BASELINE config 4 physics on a reduced 8x4^3 lattice), full and odd-even
    geom8 = L.LatticeGeometry((8, 4, 4, 4))
    links = O.flip_time_boundary(O.near_unit_gauge(geom8.dims, 0.3, 11), geom8.dims)
    gauge8 = GaugeField(geom8, links)
    zero = L.gen_clover(geom8, "zero")
    p01 = L.DiracParams(m0=0.1)
    eta8 = L.gen_spinor(geom8.n_sites, 12, Layout.COMPONENT_MAJOR, seed=13, geom=geom8)
    cfg30 = GmresConfig(restart_len=30, restarts=67, tol=1e-10)
    for oe in (False, True):
        rep = solve_dirac(p01, gauge8, zero, eta8, cfg30, odd_even=oe)
        out[f"nearunit_8444_{'oe' if oe else 'full'}"] = dict(
            dims=[8, 4, 4, 4], eps=0.3, link_seed=11, antiperiodic=True, m0=0.1, eta_seed=13, b=12,
            restart_len=30, restarts=67, tol=1e-10, odd_even=oe, iterations=rep.iterations,
            history=_hist(rep.result), final_relnorms=list(map(float, rep.result.final_relnorms)),
            full_relnorms=list(map(float, rep.full_relnorms)),
            psi_checksum=[[c.real, c.imag] for c in checksum(rep.psi.ksi())])
    (HERE / "gmres.json").write_text(json.dumps(out, indent=1))


def main():
    (HERE / "generators.json").write_text(json.dumps(gen_checksums(), indent=1))
    dirac_4444_clover()
    dirac_cfg1()
    schur_fixtures()
    gmres_fixtures()
    for p in sorted(HERE.iterdir()):
        print(f"{p.name:32s} {p.stat().st_size:>9d} B")


if __name__ == "__main__":
    main()
