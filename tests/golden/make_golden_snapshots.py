"""Snapshot files (LQML spinor / LQMG gauge / LQMC clover, fields.py:264-337)
written by the REFERENCE itself, for the byte-compatibility tests of
paper_2601_05816_b200.fields (tests/test_host_mirror.py).

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_snapshots.py

Fields on a (4, 2, 2, 4) lattice: gen_gauge(random, seed 11), gen_clover(random,
scale 0.1, seed 12), gen_spinor(b=3, seed 13) in Layout 1 (rhs-major) and 2
(component-major).
"""
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import lqcdlab as L  # noqa: E402
from lqcdlab.fields import write_clover, write_gauge, write_spinor  # noqa: E402


def main():
    geom = L.LatticeGeometry((4, 2, 2, 4))
    write_gauge(HERE / "snap_gauge.lqmg", L.gen_gauge(geom, "random", seed=11))
    write_clover(HERE / "snap_clover.lqmc", L.gen_clover(geom, "random", scale=0.1, seed=12))
    for layout in (L.Layout.RHS_MAJOR, L.Layout.COMPONENT_MAJOR):
        f = L.gen_spinor(geom.n_sites, 3, layout, seed=13, geom=geom)
        write_spinor(HERE / f"snap_spinor_l{int(layout)}.lqml", f)
    print("wrote", sorted(p.name for p in HERE.glob("snap_*")))


if __name__ == "__main__":
    main()
