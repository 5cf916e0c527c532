"""PCIe bandwidth probe (pinned host <-> device): H2D, D2H, both directions at
once, and the host-pipelined D_W apply at several chunk counts.

python tools/pcie_probe.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2601_05816_b200 as P  # noqa: E402

nbytes = 403 * 2**20
h_a = torch.empty(nbytes // 16, dtype=torch.complex128).pin_memory()
h_b = torch.empty_like(h_a).pin_memory()
d_a = torch.empty(nbytes // 16, dtype=torch.complex128, device="cuda")
d_b = torch.empty_like(d_a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    d_a.copy_(h_a, non_blocking=True)


def d2h():
    h_b.copy_(d_b, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_a, non_blocking=True)
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timed(fn)
    print(f"{name}: {t*1e3:.2f} ms  {nbytes/t/1e9:.1f} GB/s per direction", flush=True)

geom = P.LatticeGeometry((32, 16, 16, 16))
n, b = geom.n_sites, 16
gauge = P.gen_gauge(geom, "random", seed=0)
op = P.DiracOperator(P.DiracParams(m0=0.1), gauge, None, "c128")
h_in = torch.randn(n * 12 * b, dtype=torch.complex128).pin_memory()
h_out = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
psi = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_in.numpy(), geom)
eta = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_out.numpy(), geom)
for ch in (4, 8, 16, 32):
    t = timed(lambda: op.apply_host_pipelined(psi, eta, chunks=ch))
    print(f"pipelined apply chunks={ch}: {t*1e3:.2f} ms", flush=True)
