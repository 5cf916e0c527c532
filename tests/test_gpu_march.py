"""The T-marching column kernel (csrc/march.cuh) in the shapes the dispatcher
can pick, forced through B200WD_MARCH=1 / B200WD_MARCH_CFG (read once per
process, hence one subprocess per case), against the oracle: c128 <= 1e-12, c64
<= 1e-5 on c64-rounded inputs (max-norm relative error); and a race detector --
repeated applies on the same device inputs must be bit-identical (the kernel's
hand-overs of shared-memory buffers and its register reallocation once were
not: tools/stress_march.py, march.cuh header)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

# (B200WD_MARCH_CFG "NB,LY,S,NCH" or "" for the default shape [+ "|px,py" column patch], lattices, rhs counts)
CASES = [
    ("", "4x4x4x16,6x2x4x32", "6,8,12,16,32"),      # default shapes: whole lines, 1/2/4 y lines per item
    ("", "8x16x12x16", "12,16,32"),                  # more columns than CTAs: whole columns + chunked rest
    ("", "6x10x8x24", "12,16,24"),                   # partial lines (z edges from global memory)
    ("1,1,3,2", "4x2x2x24,4x4x2x16", "16,32"),       # 8-site segments, 2 t chunks, ring depth 3
    ("1,2,3,2", "4x2x2x24,6x4x6x16", "8,16"),        # two y lines of partial segments (one copy per line)
    ("2,2,0,3", "8x4x6x16,6x2x2x32", "8,12"),        # two y lines, 3 chunks (wrap-around y tiles)
    ("1,4,0,0", "4x2x4x24,4x16x12x16", "8"),         # four y lines
    ("2,1,2,1", "4x4x4x16", "12,16"),                # ring depth 2, one chunk
    ("|2,2", "4x4x4x16,6x4x8x24", "12,16"),          # patched column order (B200WD_MARCH_PATCH)
]


@pytest.mark.parametrize("cfg,dims,bs", CASES)
def test_march_shape_matches_oracle(cfg, dims, bs):
    env = dict(os.environ, B200WD_MARCH="1")
    cfg, _, patch = cfg.partition("|")
    if cfg:
        env["B200WD_MARCH_CFG"] = cfg
    if patch:
        env["B200WD_MARCH_PATCH"] = patch
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "tstream_check.py"), dims, bs], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert errs
    for k, v in errs.items():
        assert v < (1e-5 if "_c64" in k else 1e-12), (cfg, k, v)


def test_march_is_deterministic_at_scale():
    """Race detector on lattices with several units per CTA, whole and partial z lines,
    the 192- and the 256-thread shapes: 25 repetitions bit-identical (exit code 1
    otherwise).  Before the buffer hand-overs were made data-dependent on the loads, 1-13%
    of such launches returned a few sites with stale link rows."""
    env = dict(os.environ, B200WD_MARCH="1")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "stress_march.py"), "--dims", "32", "16", "16", "16",
                        "--dims", "16", "32", "16", "16", "--dims", "16", "10", "8", "24", "--b", "6", "12", "16",
                        "24", "32", "--dtypes", "c128", "c64", "--reps", "25"], env=env, capture_output=True,
                       text=True, timeout=1800)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
    assert "repetitions differ" in r.stdout


def test_default_dispatch_uses_the_march_for_the_headline_shape():
    """BASELINE configs[1], nrhs 16 complex128: the default dispatch (no environment
    switches) must agree with the ring kernel (B200WD_MARCH=0) to rounding."""
    code = ("import sys, torch; sys.path.insert(0, %r)\n"
            "from paper_2601_05816_b200 import _lib\n"
            "T,X,Y,Z=8,16,16,16; n=T*X*Y*Z; b=16\n"
            "g=torch.Generator(device='cuda').manual_seed(5)\n"
            "U=torch.randn((4*(n//8)*72,),dtype=torch.complex128,device='cuda',generator=g)\n"
            "x=torch.randn((n//8,12,8,b),dtype=torch.complex128,device='cuda',generator=g)\n"
            "y=torch.zeros_like(x); lat=_lib.Lattice.make((T,X,Y,Z))\n"
            "_lib.call('b200wd_hop',lat,0,b,-1,U.data_ptr(),x.data_ptr(),x.data_ptr(),y.data_ptr(),4.1,-1.0,None,0,T,None,None,None)\n"
            "torch.cuda.synchronize(); torch.save(y.cpu(), sys.argv[1])\n") % str(ROOT)
    import tempfile

    import torch
    with tempfile.TemporaryDirectory() as d:
        outs = []
        for name, extra in (("default", {}), ("ring", {"B200WD_MARCH": "0"})):
            f = os.path.join(d, name + ".pt")
            env = {k: v for k, v in os.environ.items() if not k.startswith("B200WD_MARCH")}
            env.update(extra)
            r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(torch.load(f))
        a, b = outs
        assert not torch.equal(a, b), "identical bits: the default dispatch did not take the march kernel"
        assert float((a - b).abs().max() / b.abs().max()) < 1e-13
