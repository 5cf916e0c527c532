"""Run the D_W apply a few times for ncu (one config per invocation).

python tools/prof_dirac.py --dtype c128 --b 16 [--dims 32 16 16 16] [--reps 3] [--parity -1]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200 import _lib  # noqa: E402
from paper_2601_05816_b200.device import DeviceField, upload_gauge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="c128")
ap.add_argument("--b", type=int, default=16)
ap.add_argument("--dims", type=int, nargs=4, default=[32, 16, 16, 16])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--parity", type=int, default=-1)
a = ap.parse_args()
geom = P.LatticeGeometry(tuple(a.dims))
gauge = upload_gauge(P.gen_gauge(geom, "random", seed=0), a.dtype)
n = geom.n_sites if a.parity < 0 else geom.n_sites // 2
tdt = torch.complex128 if a.dtype == "c128" else torch.complex64
psi = DeviceField(torch.randn((n // 8, 12, 8, a.b), dtype=torch.complex128, device="cuda").to(tdt), n)
eta = DeviceField(torch.empty_like(psi.data), n)
lat = _lib.Lattice.make(geom.dims)
code = 0 if a.dtype == "c128" else 1
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps):
    ev0.record()
    _lib.call("b200wd_hop", lat, code, a.b, a.parity, gauge.ptr, psi.ptr, psi.ptr if a.parity < 0 else None,
              eta.ptr, 4.1, -1.0, None, 0, geom.dims[0], None, None, 0)
    ev1.record()
    torch.cuda.synchronize()
    print(f"rep {i}: {ev0.elapsed_time(ev1):.4f} ms")
