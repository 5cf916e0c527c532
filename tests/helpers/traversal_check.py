"""Run in a subprocess with B200WD_TILE_KB set (the budget is read once per
process): D_W and Schur applies under the patched traversal order vs the
oracle.  Prints one JSON object of max relative errors."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from oracle import lqcd_oracle as O  # noqa: E402


def host_field(logical, geom=None):
    n, s, b = logical.shape
    f = P.BlockSpinorField.zeros(n, b, 2, s, geom)
    f.set_ksi(logical)
    return f


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


out = {}
dims = (6, 8, 12, 16)
geom = P.LatticeGeometry(dims)
links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 4), dims)
gauge = P.GaugeField(geom, links)
for b in (4, 12):
    psi = O.gen_spinor(geom.n_sites, b, 20 + b)
    ref = O.apply_dirac(dims, 0.1, links, None, psi)
    for dt in ("c128", "c64"):
        got = P.DiracOperator(P.DiracParams(m0=0.1), gauge, None, dt)(host_field(psi, geom)).ksi()
        out[f"full_b{b}_{dt}"] = rel(got, ref)
    so = O.SchurOracle(dims, 0.1, links, None, keep_parity=0)
    v = O.gen_spinor(geom.n_sites // 2, b, 40 + b)
    sp = P.SchurOperator(P.DiracParams(m0=0.1), gauge, None, keep_parity=0)
    out[f"schur_b{b}"] = rel(sp.apply(host_field(v)).ksi(), so.apply(v))
print(json.dumps(out))
