"""CPU checks of the C-ABI boundary: the in-tree library loads and exports
every symbol include/b200wd.h declares (no compute without a GPU)."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "b200wd.h").read_text()
    return sorted(set(re.findall(r"\b(b200wd_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_05816_b200 import _build, _lib
    _build.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2601_05816_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (b200wd_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the ctypes binding types every one of them
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_abi_version_and_error_paths(lib):
    from paper_2601_05816_b200 import _lib
    assert lib.b200wd_abi_version() == _lib.ABI_VERSION
    # argument validation runs before any CUDA call, so it works without a GPU
    lat = _lib.Lattice.make((4, 4, 3, 4))
    rc = lib.b200wd_hop(lat, 0, 4, -1, 1, 1, None, 1, 1.0, -1.0, None, 0, 4, None, None, None)
    assert rc == _lib.ERR_ARG
    assert b"extent 3" in lib.b200wd_last_error()
    with pytest.raises(ValueError):
        _lib.call("b200wd_spinor_import", 1, 3, 16, 12, 1, 1, 0, None)
    assert lib.b200wd_reduce_scratch_bytes(12) > 0


def test_sm100a_cubin_only(lib):
    from paper_2601_05816_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out
