"""Race detector for the hop kernels: the same apply repeated on the same
device inputs must give bit-identical outputs (every kernel here is
deterministic); a lost or early hand-over of a shared-memory buffer shows up
as a difference between repetitions.

B200WD_MARCH=1 python tools/stress_march.py --dims 32 16 16 16 --b 16 --dtypes c128 --reps 20
Prints one line per (dims, dtype, b): repetitions that differ from the first, and the
max-norm relative difference to a reference apply through the generic kernel
(b200wd_hop with the bulk-copy kernels disabled cannot be toggled per call, so the
reference is the same kernel's first repetition unless --ref FILE.pt names a tensor
saved by a B200WD_NO_TMA=1 run with --save).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2601_05816_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, action="append")
ap.add_argument("--b", type=int, nargs="+", default=[16])
ap.add_argument("--dtypes", nargs="+", default=["c128"])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--save", default=None)
ap.add_argument("--ref", default=None)
ap.add_argument("--where", action="store_true", help="print which sites / components differ")
a = ap.parse_args()
bad_total = 0
for dims in a.dims or [[32, 16, 16, 16]]:
    T, X, Y, Z = dims
    n = T * X * Y * Z
    lat = _lib.Lattice.make(tuple(dims))
    for dt in a.dtypes:
        tdt = torch.complex128 if dt == "c128" else torch.complex64
        code = 0 if dt == "c128" else 1
        g = torch.Generator(device="cuda").manual_seed(1234)
        U = torch.randn((4 * (n // 8) * 72,), dtype=tdt, device="cuda", generator=g)
        for b in a.b:
            x = torch.randn((n // 8, 12, 8, b), dtype=tdt, device="cuda", generator=g)
            outs = []
            first = None
            nbad = 0
            for r_ in range(a.reps):
                y = torch.zeros_like(x)
                _lib.call("b200wd_hop", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(), 4.1,
                          -1.0, None, 0, T, None, None, None)
                torch.cuda.synchronize()
                if first is None:
                    first = y
                elif not torch.equal(torch.view_as_real(first), torch.view_as_real(y)):
                    nbad += 1
                    if a.where:
                        d = (first != y)  # (block, k, lo, r)
                        blk, k, lo, r = torch.nonzero(d, as_tuple=True)
                        site = (blk * 8 + lo).unique().cpu().numpy()
                        zz, yy, xx, tt = site % Z, (site // Z) % Y, (site // (Z * Y)) % X, site // (Z * Y * X)
                        print(f"  rep {r_}: {len(site)} sites; t {sorted(set(tt.tolist()))} x {sorted(set(xx.tolist()))} "
                              f"y {sorted(set(yy.tolist()))} z {sorted(set(zz.tolist()))} comps {sorted(set(k.cpu().tolist()))} "
                              f"rhs {sorted(set(r.cpu().tolist()))}", flush=True)
            msg = f"dims={dims} {dt} b={b}: {nbad}/{a.reps - 1} repetitions differ"
            tag = "x".join(map(str, dims)) + f"_{dt}_b{b}"
            if a.save:
                torch.save(first.cpu(), f"{a.save}_{tag}.pt")
            if a.ref:
                ref = torch.load(f"{a.ref}_{tag}.pt").cuda()
                msg += f"; vs reference {float((first - ref).abs().max() / ref.abs().max()):.2e}"
            print(msg, flush=True)
            bad_total += nbad
            del x, first
sys.exit(1 if bad_total else 0)
