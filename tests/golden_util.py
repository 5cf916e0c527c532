"""Helpers to read the golden fixtures (see tests/golden/make_golden.py)."""

import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CHECK_SEED = 999


def load_npz(name):
    return dict(np.load(GOLDEN / name))


def load_gmres():
    return json.loads((GOLDEN / "gmres.json").read_text())


def weights(n, s=12):
    rng = np.random.Generator(np.random.PCG64(CHECK_SEED))
    return rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))


def checksum(logical):
    n, s, _ = logical.shape
    return np.einsum("xk,xkb->b", weights(n, s), logical)
