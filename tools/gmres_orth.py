"""BASELINE configs[3] GMRES(30) with the reference's MGS and the classical
Gram-Schmidt extension, side by side: iterations, time-to-solution, and the
Gram-Schmidt traffic model per iteration.

    python tools/gmres_orth.py [--orth mgs,cgs] [--oe 0,1] [--dims 48,24,24,24]

Under ncu, pass --once to run a single solve per (orth, oe) without the warm-up.
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orth", default="mgs,cgs")
    ap.add_argument("--oe", default="0,1")
    ap.add_argument("--dims", default="48,24,24,24")
    ap.add_argument("--once", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2601_05816_b200 as P
    from paper_2601_05816_b200.device import upload
    dims = tuple(int(x) for x in a.dims.split(","))
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 3))
    eta = upload(P.gen_spinor(geom.n_sites, 12, P.Layout.COMPONENT_MAJOR, seed=5, geom=geom))
    for orth in a.orth.split(","):
        for oe in (bool(int(x)) for x in a.oe.split(",")):
            if not a.once:
                P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta,
                              P.GmresConfig(restart_len=30, restarts=1, tol=1e-10, orthogonalization=orth),
                              odd_even=oe)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta,
                                P.GmresConfig(restart_len=30, restarts=67, tol=1e-10, orthogonalization=orth),
                                odd_even=oe)
            torch.cuda.synchronize()
            tts = time.perf_counter() - t0
            print(json.dumps({"dims": dims, "orth": orth, "odd_even": oe, "iterations": rep.iterations,
                              "tts_s": round(tts, 4), "ms_per_it": round(1e3 * tts / rep.iterations, 3),
                              "max_full_relnorm": float(rep.full_relnorms.max())}), flush=True)


if __name__ == "__main__":
    main()
