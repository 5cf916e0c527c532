"""Host-pipelined apply (apply_dirac with host fields) timed per T-chunk count; checks the
outputs are bit-identical.  python tools/e2e_chunks.py (GPU)."""
import time, torch, numpy as np, sys
sys.path.insert(0, ".")
import paper_2601_05816_b200 as P
from paper_2601_05816_b200.dirac import DiracOperator
geom = P.LatticeGeometry((32, 16, 16, 16)); n = geom.n_sites; b = 16
gauge = P.gen_gauge(geom, "random", seed=0)
h_in = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
h_out = torch.empty(n * 12 * b, dtype=torch.complex128).pin_memory()
h_in.copy_(torch.randn(n * 12 * b, dtype=torch.complex128))
psi = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_in.numpy(), geom)
eta = P.BlockSpinorField(n, 12, b, P.Layout.COMPONENT_MAJOR, h_out.numpy(), geom)
op = DiracOperator(P.DiracParams(m0=0.1), gauge, None, "c128")
ref = None
for rep in range(2):
    for ck in (4, 8, 16, 32):
        for _ in range(3):
            op.apply_host_pipelined(psi, eta, chunks=ck)
        torch.cuda.synchronize()
        if ref is None: ref = h_out.clone()
        else: assert torch.equal(ref, h_out)
        t0 = time.perf_counter()
        for _ in range(20):
            op.apply_host_pipelined(psi, eta, chunks=ck)
        torch.cuda.synchronize()
        print(ck, (time.perf_counter() - t0) / 20 * 1e3, "ms", flush=True)
# apply_dirac per-call overhead (constructs the operator each call)
for _ in range(3): P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, psi, dtype="c128", out=eta)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(20): P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, psi, dtype="c128", out=eta)
torch.cuda.synchronize(); print("apply_dirac", (time.perf_counter() - t0) / 20 * 1e3, "ms")
