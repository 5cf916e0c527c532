"""The T-streaming hop kernel (csrc/tstream.cuh) in every shape the
dispatcher can pick, forced through B200WD_TS_CFG (read once per process,
hence one subprocess per shape), against the oracle: c128 <= 1e-12, c64 <=
1e-5 on c64-rounded inputs (max-norm relative error)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

# (NB, LY, S, NCH, PF, PX, PY), lattices (T x X x Y x Z), rhs counts
CASES = [
    ("2,1,2,0,0", "4x4x4x16,6x2x2x32", "8,16"),      # whole lines; 2 segments per line
    ("2,1,4,3,1", "6x4x4x16", "8,16"),               # 3 t chunks, L2 prefetch
    ("1,1,3,0,0", "4x2x2x24,4x4x2x16", "8,16,32"),  # partial lines (z edges from global memory)
    ("2,2,3,0,0", "4x4x4x16,4x2x6x16", "4,8,16"),    # two y lines per item
    ("1,2,2,2,0", "4x2x4x24", "8,16"),               # two y lines, partial lines, 2 chunks
    ("3,1,2,1,0", "4x2x2x24", "8,12"),               # 24-site segments
    ("2,1,3,1,0,2,2", "4x4x4x16", "8,16"),           # patched column order
]


@pytest.mark.parametrize("cfg,dims,bs", CASES)
def test_tstream_shape_matches_oracle(cfg, dims, bs):
    env = dict(os.environ, B200WD_TS_CFG=cfg)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "tstream_check.py"), dims, bs], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert errs
    for k, v in errs.items():
        assert v < (1e-5 if "_c64" in k else 1e-12), (cfg, k, v)
