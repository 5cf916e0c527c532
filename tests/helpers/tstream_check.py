"""Run in a subprocess with B200WD_TS_CFG or B200WD_RING2_S set (read once per process): the
T-streaming hop kernel in a forced shape vs the oracle, on lattices that
exercise whole-line and partial-line (z-edge) segments, one and several t
chunks, patched column order and a slice sub-range (the T-split interior
call).  Prints one JSON object of max relative errors."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200 import _lib  # noqa: E402
from paper_2601_05816_b200.device import DeviceField, upload, upload_gauge  # noqa: E402
from oracle import lqcd_oracle as O  # noqa: E402


def host_field(logical, geom=None):
    n, s, b = logical.shape
    f = P.BlockSpinorField.zeros(n, b, 2, s, geom)
    f.set_ksi(logical)
    return f


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


out = {}
for dims in [tuple(int(x) for x in d.split("x")) for d in sys.argv[1].split(",")]:
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 7), dims)
    gauge = P.GaugeField(geom, links)
    for b in [int(x) for x in sys.argv[2].split(",")]:
        psi = O.gen_spinor(geom.n_sites, b, 30 + b)
        ref = O.apply_dirac(dims, 0.1, links, None, psi)
        key = "x".join(map(str, dims)) + f"_b{b}"
        for dt in ("c128", "c64"):
            inp = (psi, links) if dt == "c128" else (O.round_c64(psi), O.round_c64(links))
            r = ref if dt == "c128" else O.apply_dirac(dims, 0.1, inp[1], None, inp[0])
            got = P.DiracOperator(P.DiracParams(m0=0.1), gauge, None, dt)(host_field(psi, geom)).ksi()
            out[f"{key}_{dt}"] = rel(got, r)
            # interior slices [1, T-1) only (T-split interior launch): out = 4.1 x - (1/2)... via the raw ABI
            T = dims[0]
            if T >= 3:
                x = upload(host_field(psi, geom), dt)
                y = DeviceField.zeros(geom.n_sites, b, dtype=dt, geom=geom)
                g = upload_gauge(gauge, dt)
                lat = _lib.Lattice.make(dims)
                _lib.call("b200wd_hop", lat, 0 if dt == "c128" else 1, b, -1, g.ptr, x.ptr, x.ptr, y.ptr,
                          4.1, -1.0, None, 1, T - 1, None, None, None)
                torch.cuda.synchronize()
                per = geom.n_sites // T
                got_r = y.logical()[per:(T - 1) * per]
                out[f"{key}_{dt}_range"] = rel(got_r, r[per:(T - 1) * per])
print(json.dumps(out))
