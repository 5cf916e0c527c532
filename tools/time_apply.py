"""Time the D_W hop kernel on arbitrary lattices with device-generated fields.

python tools/time_apply.py --dims 96 48 48 48 --b 12 --dtypes c128 c64 [--iters 10]

Link and spinor VALUES are random numbers drawn on the device (not SU(3)):
kernel time does not depend on them, and large lattices skip the host-side
link generation.  Buffers rotate so > 4x L2 bytes are touched between reuses.
Prints ms, site*rhs/s and the fraction of the measured HBM copy peak for the
compulsory bytes (24 b + 36) w per site.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_05816_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[32, 16, 16, 16])
ap.add_argument("--b", type=int, nargs="+", default=[12])
ap.add_argument("--dtypes", nargs="+", default=["c128", "c64"])
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--parity", type=int, default=-1, help="destination parity of a checkerboard hop (-1: full)")
ap.add_argument("--cold", action="store_true", help="time each launch alone after an L2 flush (512 MB memset)")
ap.add_argument("--clover", type=int, default=0, help="clover mode of the hop (1: -C x, 2: M(...)); random blocks")
ap.add_argument("--idle", type=float, default=0.0, help="with --cold: seconds the GPU idles before each launch")
a = ap.parse_args()
pk = ROOT / "MEASURED_PEAKS.json"
peak = float(json.loads(pk.read_text())["hbm_gbs"]) if pk.exists() else 6650.0
T, X, Y, Z = a.dims
n = T * X * Y * Z
lat = _lib.Lattice.make(tuple(a.dims))
l2 = 126 * 2**20
for dt in a.dtypes:
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    w = 16 if dt == "c128" else 8
    code = 0 if dt == "c128" else 1
    U = torch.randn((4 * (n // 8) * 72,), dtype=tdt, device="cuda")
    # packed 2 x 21 Hermitian blocks per destination site, 8-site blocked (layout.cuh clover_base)
    CL = torch.randn((((n if a.parity < 0 else n // 2) // 8) * 336,), dtype=tdt, device="cuda") if a.clover else None
    for b in a.b:
        nf = n if a.parity < 0 else n // 2
        fb = nf * 12 * b * w
        nbuf = max(1, int(np.ceil(4 * l2 / (2 * fb))))
        ps = [torch.randn((nf // 8, 12, 8, b), dtype=tdt, device="cuda") for _ in range(nbuf)]
        es = [torch.empty_like(ps[0]) for _ in range(nbuf)]

        def go(i):
            x = ps[i % nbuf]
            if a.clover:
                _lib.call("b200wd_hop_clover", lat, code, b, a.parity, U.data_ptr(), x.data_ptr(), x.data_ptr(),
                          es[i % nbuf].data_ptr(), 4.1, -1.0, None, 0, T, None, None, CL.data_ptr(), a.clover,
                          None)
                return
            _lib.call("b200wd_hop", lat, code, b, a.parity, U.data_ptr(), x.data_ptr(),
                      x.data_ptr() if a.parity < 0 else None,
                      es[i % nbuf].data_ptr(), 4.1, -1.0, None, 0, T, None, None, None)

        for i in range(3):
            go(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if a.cold:
            flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
            ts = []
            for i in range(a.iters):
                flush.fill_(i & 255)
                if a.idle > 0:
                    torch.cuda.synchronize()
                    time.sleep(a.idle)
                e0.record()
                go(i)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            t = float(np.median(ts))
            if a.idle > 0:
                print("  per launch ms:", " ".join(f"{x*1e3:.2f}" for x in ts))
            del flush
        else:
            e0.record()
            for i in range(a.iters):
                go(i)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / a.iters * 1e-3
        alg = (24 * b + 36) * w * n if a.parity < 0 else (24 * b + 72) * w * nf  # parity: half fields, all links
        if a.clover:
            alg += 42 * w * nf + (12 * b * w * nf if a.parity >= 0 else 0)  # clover blocks (+ xself of a parity hop)
        print(f"{dt} dims={a.dims} par={a.parity} clov={a.clover} b={b:3d} {t*1e3:8.4f} ms  {nf*b/t:10.3e} site*rhs/s  {alg/t/1e9:8.1f} GB/s  "
              f"frac {alg/t/1e9/peak:.3f}", flush=True)
        del ps, es
        torch.cuda.empty_cache()
    del U
