"""Schur apply timing (BASELINE configs[2]: 32^3 x 64, nrhs=12, c128, near-unit links).
python tools/bench_schur.py [--dims 64 32 32 32] [--b 12] [--dtype c128]"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200.device import DeviceField  # noqa: E402


def schur_bench(dims=(64, 32, 32, 32), b=12, dtype="c128", iters=10, m0=0.1):
    geom = P.LatticeGeometry(tuple(dims))
    t0 = time.perf_counter()
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 3))
    gen = time.perf_counter() - t0
    s = P.SchurOperator(P.DiracParams(m0=m0), gauge, None, dtype=dtype)
    n = geom.n_sites // 2
    tdt = torch.complex128 if dtype == "c128" else torch.complex64
    vs = [DeviceField(torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, device="cuda").to(tdt), n, geom, 0)
          for _ in range(2)]
    outs = [v.empty_like() for v in vs]
    for i in range(3):
        s.apply_device(vs[i % 2], outs[i % 2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        s.apply_device(vs[i % 2], outs[i % 2])
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / iters * 1e-3
    w = 16 if dtype == "c128" else 8
    alg = (60 * b + 144) * w * n
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    return {"lattice": list(dims), "nrhs": b, "dtype": dtype, "ms": t * 1e3, "even_site_rhs_per_s": n * b / t,
            "hbm_gbs": alg / t / 1e9, "frac": alg / t / 1e9 / peak, "alg_bytes": alg, "input_gen_s": gen}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=4, default=[64, 32, 32, 32])
    ap.add_argument("--b", type=int, default=12)
    ap.add_argument("--dtype", default="c128")
    a = ap.parse_args()
    print(json.dumps(schur_bench(a.dims, a.b, a.dtype)))
