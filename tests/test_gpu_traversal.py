"""The ring kernel's patched traversal order (T slices of one x-y patch of z
lines at a time, used when a T slice exceeds the L2 budget) gives the same
results as the oracle.  A tiny B200WD_TILE_KB forces the patching on a small
lattice; the budget is read once per process, hence the subprocess."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("kb", ["64", "200", "0"])
def test_patched_traversal_matches_oracle(kb):
    env = dict(os.environ, B200WD_TILE_KB=kb)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "traversal_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    for k, v in errs.items():
        assert v < (1e-5 if k.endswith("c64") else 1e-12), (k, v)


@pytest.mark.parametrize("kb", ["64", "200"])
def test_wave_synchronised_full_lattice_traversal_matches_oracle(kb):
    """The full-lattice patched order with wave synchronisation (used when a
    T slice exceeds the L2 reuse limit, e.g. 48^3 x 96) forced on a small
    lattice: B200WD_SLICE_KB lowers the limit, B200WD_WAVE_KB sizes the patch."""
    env = dict(os.environ, B200WD_SLICE_KB="1", B200WD_WAVE_KB=kb, B200WD_TILE_KB=kb, B200WD_WAVE="1")
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "traversal_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    errs = json.loads(r.stdout.strip().splitlines()[-1])
    for k, v in errs.items():
        assert v < (1e-5 if k.endswith("c64") else 1e-12), (k, v)
