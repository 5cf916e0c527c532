"""Split apply vs unsplit apply at one rank's local shape (the T-split
overhead on one GPU): (a) one D_W launch over all local slices; (b) the
split sequence of TSplitComm.hop -- halo pack, interior slices [1, T-1),
the two boundary slices consuming the halo faces (here the rank's own faces,
i.e. a periodic one-rank ring).

python tools/time_split.py --dims 12 48 48 48 --b 12 --dtypes c128 c64
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2601_05816_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=4, default=[12, 48, 48, 48])
ap.add_argument("--b", type=int, default=12)
ap.add_argument("--dtypes", nargs="+", default=["c128", "c64"])
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
T, X, Y, Z = a.dims
n = T * X * Y * Z
per_t = X * Y * Z
lat = _lib.Lattice.make(tuple(a.dims))
L = _lib.load()
for dt in a.dtypes:
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    code = 0 if dt == "c128" else 1
    b = a.b
    U = torch.randn((4 * (n // 8) * 72,), dtype=tdt, device="cuda")
    x = torch.randn((n // 8, 12, 8, b), dtype=tdt, device="cuda")
    y = torch.empty_like(x)
    lam, chi = (torch.empty((6, per_t, b), dtype=tdt, device="cuda") for _ in range(2))

    def full():
        _lib.call("b200wd_hop", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(), 4.1, -1.0,
                  None, 0, T, None, None, None)

    def split(merged=False):
        _lib.call("b200wd_halo_pack", lat, code, b, -1, U.data_ptr(), x.data_ptr(), lam.data_ptr(), chi.data_ptr(),
                  None)
        _lib.call("b200wd_hop", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(), 4.1, -1.0,
                  None, 1, T - 1, None, None, None)
        _lib.call("b200wd_hop_boundary", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(),
                  4.1, -1.0, None, lam.data_ptr(), chi.data_ptr(), None, 0, None)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.iters

    tf, ts = timed(full), timed(split)
    # pieces of the split
    ti = timed(lambda: _lib.call("b200wd_hop", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(),
                                 y.data_ptr(), 4.1, -1.0, None, 1, T - 1, None, None, None))
    tb = timed(lambda: _lib.call("b200wd_hop_boundary", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(), 4.1, -1.0, None, lam.data_ptr(), chi.data_ptr(), None, 0, None))
    tb2 = timed(lambda: [_lib.call("b200wd_hop", lat, code, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(),
                                  y.data_ptr(), 4.1, -1.0, None, t0, t1, lam.data_ptr(), chi.data_ptr(), None)
                        for t0, t1 in ((0, 1), (T - 1, T))])
    tp = timed(lambda: _lib.call("b200wd_halo_pack", lat, code, b, -1, U.data_ptr(), x.data_ptr(), lam.data_ptr(),
                                 chi.data_ptr(), None))
    print(json.dumps({"dims": a.dims, "dtype": dt, "b": b, "full_ms": round(tf, 4), "split_ms": round(ts, 4),
                      "overhead": round(ts / tf - 1, 4), "interior_ms": round(ti, 4), "boundary_ms": round(tb, 4), "boundary_two_launches_ms": round(tb2, 4),
                      "pack_ms": round(tp, 4),
                      "boundary_per_slice_vs_full_per_slice": round((tb / 2) / (tf / T), 3)}), flush=True)
    del U, x, y, lam, chi
    torch.cuda.empty_cache()
