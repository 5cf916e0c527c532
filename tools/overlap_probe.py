"""Does a kernel enqueued on another stream run next to the persistent
interior hop?  The T split's halo exchange (NCCL P2P kernels on NCCL's
stream) must overlap the interior slices (halo.py:339-387 semantics); the
ring kernel's persistent grid can fill every SM, so TSplitComm leaves
`sm_reserve` SMs free for the duration of the interior launch
(b200wd_set_sm_reserve).  One GPU stand-in for the P2P kernel: a 127 MB
elementwise kernel on a second stream, launched right after the interior hop.

python tools/overlap_probe.py [--dims 12 48 48 48] [--b 12]

Prints, per reserve: interior hop time alone, side kernel time alone, and the
side kernel's completion measured from the interior launch (overlapped: about
its own time; serialised: the interior time plus its own).
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2601_05816_b200 import _lib  # noqa: E402


def probe(dims=(12, 48, 48, 48), b=12, reserves=(0, 8), reps=5):
    T, X, Y, Z = dims
    n = T * X * Y * Z
    lat = _lib.Lattice.make(tuple(dims))
    L = _lib.load()
    U = torch.randn((4 * (n // 8) * 72,), dtype=torch.complex128, device="cuda")
    x = torch.randn((n // 8, 12, 8, b), dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    side = torch.randn(127 * 2**20 // 8, dtype=torch.float64, device="cuda")
    s_main = torch.cuda.current_stream()
    s_side = torch.cuda.Stream()

    def interior():
        _lib.call("b200wd_hop", lat, 0, b, -1, U.data_ptr(), x.data_ptr(), x.data_ptr(), y.data_ptr(), 4.1, -1.0,
                  None, 1, T - 1, None, None, None)

    def side_kernel():
        side.mul_(1.0000001)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    out = []
    for k in reserves:
        prev = L.b200wd_set_sm_reserve(k)
        for _ in range(2):
            interior()
            side_kernel()
        torch.cuda.synchronize()
        alone_i, alone_s, done = [], [], []
        for _ in range(reps):
            ev[0].record(s_main)
            interior()
            ev[1].record(s_main)
            torch.cuda.synchronize()
            alone_i.append(ev[0].elapsed_time(ev[1]))
            ev[0].record(s_side)
            with torch.cuda.stream(s_side):
                side_kernel()
            ev[1].record(s_side)
            torch.cuda.synchronize()
            alone_s.append(ev[0].elapsed_time(ev[1]))
            # concurrent: interior on the main stream, the side kernel right behind it
            ev[2].record(s_main)
            s_side.wait_event(ev[2])
            interior()
            with torch.cuda.stream(s_side):
                side_kernel()
                ev[3].record(s_side)
            torch.cuda.synchronize()
            done.append(ev[2].elapsed_time(ev[3]))
        L.b200wd_set_sm_reserve(prev)
        med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
        out.append({"sm_reserve": k, "interior_ms": round(med(alone_i), 4), "side_alone_ms": round(med(alone_s), 4),
                    "side_done_after_interior_launch_ms": round(med(done), 4),
                    "overlapped": med(done) < 0.75 * med(alone_i)})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=4, default=[12, 48, 48, 48])
    ap.add_argument("--b", type=int, default=12)
    a = ap.parse_args()
    for r in probe(tuple(a.dims), a.b):
        print(json.dumps(r))
