"""Golden GMRES(8) results for BASELINE configs[4]'s solver physics, produced by
the REFERENCE on reduced lattices.

Run in the build container only (needs /root/reference); long-running:

    PYTHONPATH=/root/reference/pkg/src nice python tests/golden/make_golden_cfg5.py [small|proxy|mid|all]

configs[4] solver: odd-even preconditioned batched restarted GMRES(8) to
relative tolerance 1e-8, nrhs=12 Gaussian rhs, m0=0.1, near-unit links
(eps=0.3), antiperiodic T, C=0, the 2000-iteration cap of SURVEY §8(d)
(restarts = 250).  The 48^3 x 96 lattice itself is far beyond the reference
(hours per apply), so its physics is pinned on reduced lattices (T first):

* ``small``: 12 x 6^3, odd-even and unpreconditioned (seconds to minutes).
* ``proxy``: 24 x 12^3, odd-even (minutes).
* ``mid``: 16 x 8^3, odd-even (splits evenly over 2, 4 and 8 ranks).

Inputs: links = flip_time_boundary(near_unit_gauge(dims, 0.3, seed 7)),
rhs = gen_spinor(n, 12, seed 9), both the oracle's harness generators
(pinned to the reference's own generators by tests/test_oracle.py).
Writes tests/golden/gmres_cfg5.json (iterations, per-iteration relnorm
history, final and full-system residuals, wall time of the reference).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import lqcdlab as L  # noqa: E402
from lqcdlab.fields import GaugeField, Layout  # noqa: E402
from lqcdlab.gmres import GmresConfig, solve_dirac  # noqa: E402

from oracle import lqcd_oracle as O  # noqa: E402

OUT = HERE / "gmres_cfg5.json"
LINK_SEED, ETA_SEED = 7, 9
RESTART_LEN, RESTARTS, TOL = 8, 250, 1e-8


def run(dims, oe: bool) -> dict:
    geom = L.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, LINK_SEED), dims)
    gauge = GaugeField(geom, links)
    eta = L.gen_spinor(geom.n_sites, 12, Layout.COMPONENT_MAJOR, seed=ETA_SEED, geom=geom)
    cfg = GmresConfig(restart_len=RESTART_LEN, restarts=RESTARTS, tol=TOL)
    t0 = time.perf_counter()
    rep = solve_dirac(L.DiracParams(m0=0.1), gauge, L.gen_clover(geom, "zero"), eta, cfg, odd_even=oe)
    wall = time.perf_counter() - t0
    return dict(dims=list(dims), eps=0.3, link_seed=LINK_SEED, antiperiodic=True, m0=0.1, eta_seed=ETA_SEED, b=12,
                restart_len=RESTART_LEN, restarts=RESTARTS, tol=TOL, odd_even=oe, iterations=int(rep.iterations),
                converged=[bool(c) for c in rep.result.converged],
                history=[list(map(float, h)) for h in rep.result.history],
                final_relnorms=list(map(float, rep.result.final_relnorms)),
                full_relnorms=list(map(float, rep.full_relnorms)), reference_wall_s=wall, reference_threads=1)


def save(key: str, rec: dict) -> None:
    cur = json.loads(OUT.read_text()) if OUT.exists() else {}
    cur[key] = rec
    OUT.write_text(json.dumps(cur, indent=1))
    print(f"{key}: {rec['iterations']} iterations in {rec['reference_wall_s']:.1f} s", flush=True)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what in ("small", "all"):
        for oe in (True, False):
            save(f"small_12x6c_{'oe' if oe else 'full'}", run((12, 6, 6, 6), oe))
    if what in ("proxy", "all"):
        save("proxy_24x12c_oe", run((24, 12, 12, 12), True))
    if what in ("mid", "all"):
        save("mid_16x8c_oe", run((16, 8, 8, 8), True))


if __name__ == "__main__":
    main()
