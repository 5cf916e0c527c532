"""The two-line ring kernel (csrc/ring2.cuh) forced through B200WD_RING2_S
(read once per process, hence subprocesses; the stream kernel is switched off
so the dispatcher reaches it) against the oracle: whole z lines of 8/16/32
sites, nrhs 4/8/16, c128 and c64, full range and the [1, T-1) slice range."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("depth", ["1", "3"])
def test_ring2_matches_oracle(depth):
    env = dict(os.environ, B200WD_TSTREAM="0", B200WD_RING2_S=depth)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "tstream_check.py"),
                        "4x4x4x16,4x2x6x8,6x4x2x32,4x2x2x16", "4,8,16"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    assert errs
    for k, v in errs.items():
        assert v < (1e-5 if "_c64" in k else 1e-12), (depth, k, v)
