"""Golden GMRES results for BASELINE configs[3] produced by the REFERENCE.

Run in the build container only (needs /root/reference); long-running:

    PYTHONPATH=/root/reference/pkg/src nice python tests/golden/make_golden_cfg3.py [proxy|oe|mid|all]

configs[3]: batched restarted GMRES(30), nrhs=12 Gaussian rhs, m0=0.1,
near-unit links (eps=0.3), antiperiodic T, C=0, relative tolerance 1e-10,
2000-iteration cap (restarts = ceil(2000/30) = 67), unpreconditioned and
odd-even preconditioned.  Inputs are the ones bench.py uses (links seed 3,
rhs seed 5), built with the oracle's harness generators (verified equal to
the package's) and fed to ``lqcdlab.solve_dirac`` unchanged.

* ``proxy``: the same physics on 24 x 12^3 (T first), full and odd-even
  (minutes).
* ``oe``: the full-size 48 x 24^3 odd-even solve (about 1.3 h on one core,
  ~40 GB; the full-size unpreconditioned solve needs ~58 GB of host memory
  for its 31-vector basis and is not run here).
* ``mid``: the unpreconditioned solve on 32 x 16^3 (~20 min, ~10 GB).

Writes tests/golden/gmres_cfg3.json (iterations, per-iteration relnorm
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

OUT = HERE / "gmres_cfg3.json"


def run(dims, oe: bool, link_seed: int = 3, eta_seed: int = 5) -> dict:
    geom = L.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, link_seed), dims)
    gauge = GaugeField(geom, links)
    eta = L.gen_spinor(geom.n_sites, 12, Layout.COMPONENT_MAJOR, seed=eta_seed, geom=geom)
    cfg = GmresConfig(restart_len=30, restarts=67, tol=1e-10)
    t0 = time.perf_counter()
    rep = solve_dirac(L.DiracParams(m0=0.1), gauge, L.gen_clover(geom, "zero"), eta, cfg, odd_even=oe)
    wall = time.perf_counter() - t0
    return dict(dims=list(dims), eps=0.3, link_seed=link_seed, antiperiodic=True, m0=0.1, eta_seed=eta_seed, b=12,
                restart_len=30, restarts=67, tol=1e-10, odd_even=oe, iterations=int(rep.iterations),
                history=[list(map(float, h)) for h in rep.result.history],
                final_relnorms=list(map(float, rep.result.final_relnorms)),
                full_relnorms=list(map(float, rep.full_relnorms)), reference_wall_s=wall, reference_threads=1)


def save(key: str, rec: dict) -> None:
    cur = json.loads(OUT.read_text()) if OUT.exists() else {}
    cur[key] = rec
    OUT.write_text(json.dumps(cur, indent=1))
    print(f"{key}: {rec['iterations']} iterations in {rec['reference_wall_s']:.1f} s", flush=True)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "proxy"
    if what in ("proxy", "all"):
        for oe in (False, True):
            save(f"proxy_24x12c_{'oe' if oe else 'full'}", run((24, 12, 12, 12), oe))
    if what in ("oe", "all"):
        save("cfg3_48x24c_oe", run((48, 24, 24, 24), True))
    if what in ("mid", "all"):
        save("mid_32x16c_full", run((32, 16, 16, 16), False))


if __name__ == "__main__":
    main()
