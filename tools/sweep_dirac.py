"""Quick D_W sweep for kernel tuning (one process per library variant).

B200WD_LIB=... python tools/sweep_dirac.py [--dims 32 16 16 16] [--bs 1 4 8 12 16 32]
Prints one line per (dtype, b): ms, site*rhs/s, algorithmic GB/s, fraction of HBM peak.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200 import _lib  # noqa: E402
from paper_2601_05816_b200.device import DeviceField, upload_gauge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[32, 16, 16, 16])
ap.add_argument("--bs", type=int, nargs="+", default=[1, 4, 8, 12, 16, 32])
ap.add_argument("--dtypes", nargs="+", default=["c128", "c64"])
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--parity", type=int, default=-1)
a = ap.parse_args()
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0
geom = P.LatticeGeometry(tuple(a.dims))
gauge = P.gen_gauge(geom, "random", seed=0)
lat = _lib.Lattice.make(geom.dims)
L = _lib.load()
l2 = 126 * 2**20
for dt in a.dtypes:
    g = upload_gauge(gauge, dt)
    w = 16 if dt == "c128" else 8
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    for b in a.bs:
        n = geom.n_sites if a.parity < 0 else geom.n_sites // 2
        fb = n * 12 * b * w
        nbuf = max(2, int(np.ceil(4 * l2 / (2 * fb))) + 1)
        base = torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, device="cuda").to(tdt)
        ps = [DeviceField(base.clone(), n) for _ in range(nbuf)]
        es = [DeviceField(torch.empty_like(base), n) for _ in range(nbuf)]
        code = 0 if dt == "c128" else 1

        def go(i):
            x = ps[i % nbuf]
            rc = L.b200wd_hop(lat, code, b, a.parity, g.ptr, x.ptr, x.ptr if a.parity < 0 else None,
                              es[i % nbuf].ptr, 4.1, -1.0, None, 0, geom.dims[0], None, None, None)
            assert rc == 0, L.b200wd_last_error()
        for i in range(5):
            go(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(a.iters):
            go(i)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / a.iters * 1e-3
        if a.parity < 0:
            alg = (24 * b + 36) * w * n
        else:
            alg = (24 * b + 72) * w * n  # half-field in/out + all links
        print(f"{dt} b={b:3d} {t*1e3:8.4f} ms  {n*b/t:10.3e} site*rhs/s  {alg/t/1e9:8.1f} GB/s  frac {alg/t/1e9/peak:.3f}",
              flush=True)
        del ps, es, base
        torch.cuda.empty_cache()
