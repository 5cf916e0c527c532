import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2601_05816_b200 as P
from paper_2601_05816_b200 import _lib
from paper_2601_05816_b200.device import DeviceField, upload, upload_gauge
from oracle import lqcd_oracle as O
dims = tuple(int(x) for x in sys.argv[1].split("x")); b = int(sys.argv[2]); dt = sys.argv[3]
geom = P.LatticeGeometry(dims)
links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 7), dims)
gauge = P.GaugeField(geom, links)
psi = O.gen_spinor(geom.n_sites, b, 30 + b)
inp = (psi, links) if dt == "c128" else (O.round_c64(psi), O.round_c64(links))
ref = O.apply_dirac(dims, 0.1, inp[1], None, inp[0])
f = P.BlockSpinorField.zeros(geom.n_sites, b, 2, 12, geom); f.set_ksi(psi)
for rep in range(3):
    got = P.DiracOperator(P.DiracParams(m0=0.1), gauge, None, dt)(f).ksi()
    err = np.abs(got - ref).max(axis=(1, 2)) / np.abs(ref).max()
    bad = np.nonzero(err > 1e-4)[0]
    T, X, Y, Z = dims
    print("rep", rep, "max", err.max(), "nbad", len(bad))
    if len(bad):
        t = bad // (X * Y * Z); x = (bad // (Y * Z)) % X; y = (bad // Z) % Y; z = bad % Z
        print(" t:", np.unique(t, return_counts=True)); print(" z:", np.unique(z, return_counts=True))
        print(" x:", np.unique(x)[:20], " y:", np.unique(y)[:20])
        # which rhs / components
        e2 = np.abs(got - ref)[bad] / np.abs(ref).max()
        print(" comps:", (e2.max(axis=(0, 2)) > 1e-4).astype(int), " rhs:", (e2.max(axis=(0, 1)) > 1e-4).astype(int))
