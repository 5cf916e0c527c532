"""A short batched-GMRES run for kernel timing (BASELINE configs[3] lattice).
python tools/prof_gmres.py [--dims 48 24 24 24] [--oe]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
from paper_2601_05816_b200.device import DeviceField  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[48, 24, 24, 24])
ap.add_argument("--oe", action="store_true")
ap.add_argument("--b", type=int, default=12)
a = ap.parse_args()
geom = P.LatticeGeometry(tuple(a.dims))
links = np.zeros((geom.n_sites, 4, 3, 3), dtype=np.complex128)
links[..., np.arange(3), np.arange(3)] = 1.0  # unit links: timing only
gauge = P.GaugeField(geom, links)
n = geom.n_sites
eta = DeviceField(torch.randn((n // 8, 12, 8, a.b), dtype=torch.complex128, device="cuda"), n, geom)
cfg = P.GmresConfig(restart_len=10, restarts=1, fixed_iterations=True)
P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg, odd_even=a.oe)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rep = P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg, odd_even=a.oe)
e1.record()
torch.cuda.synchronize()
print(f"10 iterations: {e0.elapsed_time(e1):.2f} ms  ({'oe' if a.oe else 'full'})")
