"""Small-lattice batched GMRES wall time per iteration (host-overhead check)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402
import paper_2601_05816_b200.gmres as G  # noqa: E402
from paper_2601_05816_b200.device import upload  # noqa: E402

for dims, b in (((8, 8, 8, 8), 4), ((8, 4, 4, 4), 12), ((16, 8, 8, 8), 12)):
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 1))
    eta = upload(P.gen_spinor(geom.n_sites, b, 2, seed=2, geom=geom))
    cfg = P.GmresConfig(restart_len=30, restarts=67, tol=1e-10)
    for oe, mode in [(o, m) for o in (False, True) for m in ("cycle", "step", "python")]:
        G.NATIVE_ARNOLDI = mode != "python"
        G.NATIVE_CYCLE = mode == "cycle"
        P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg, odd_even=oe)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, eta, cfg, odd_even=oe)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        print(f"{dims} b={b} {'oe  ' if oe else 'full'} {mode:6s}: {rep.iterations} it, {t*1e3:.1f} ms, "
              f"{t/rep.iterations*1e6:.0f} us/it")
