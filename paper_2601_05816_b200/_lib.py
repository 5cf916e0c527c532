"""ctypes binding of libb200wd.so (include/b200wd.h).

The library is built in-tree by ``paper_2601_05816_b200._build`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the shared
library or a CUDA device is missing, every compute entry point raises
:class:`B200Unavailable`.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("B200WD_LIB") or Path(__file__).resolve().parent / "libb200wd.so")

OK, ERR_ARG, ERR_CUDA, ERR_SINGULAR, ERR_UNSUPPORTED = 0, 1, 2, 3, 4
C128, C64 = 0, 1
ABI_VERSION = 3


class B200Unavailable(RuntimeError):
    """The CUDA library or a B200 device is not available (no CPU fallback)."""


class Lattice(C.Structure):
    _fields_ = [("dims", C.c_int32 * 4), ("t_origin", C.c_int32), ("reserved", C.c_int32)]

    @classmethod
    def make(cls, dims, t_origin: int = 0) -> "Lattice":
        lat = cls()
        for i, d in enumerate(dims):
            lat.dims[i] = int(d)
        lat.t_origin = int(t_origin)
        return lat


class GmresState(C.Structure):
    _fields_ = [
        ("b", C.c_int32), ("m", C.c_int32), ("breakdown_rel", C.c_double),
        ("h_raw", C.c_void_p), ("h", C.c_void_p), ("gamma", C.c_void_p), ("cs", C.c_void_p),
        ("sn", C.c_void_p), ("sigma", C.c_void_p), ("eta_norm", C.c_void_p), ("relnorm", C.c_void_p),
        ("breakdown", C.c_void_p), ("dot", C.c_void_p), ("y", C.c_void_p), ("scratch", C.c_void_p),
        ("orth", C.c_int32), ("cgs_partials", C.c_void_p),
    ]


OPND_NONE, OPND_IN, OPND_OUT, OPND_TMP = 0, 1, 2, 3
MAX_STAGES = 4


class HopStage(C.Structure):
    _fields_ = [
        ("dst_parity", C.c_int32), ("src", C.c_int32), ("xself", C.c_int32), ("out", C.c_int32),
        ("alpha", C.c_double), ("beta", C.c_double), ("clover", C.c_void_p), ("clover_mode", C.c_int32),
        ("use_scale", C.c_int32),
    ]


class Operator(C.Structure):
    """b200wd_operator: a linear operator as a program of hop stages."""

    _fields_ = [
        ("lat", Lattice), ("dtype", C.c_int32), ("n_stages", C.c_int32), ("links", C.c_void_p),
        ("tmp", C.c_void_p), ("stage", HopStage * MAX_STAGES),
    ]

    @classmethod
    def make(cls, lat: Lattice, dtype: int, links: int, stages, tmp: int | None = None) -> "Operator":
        if not 1 <= len(stages) <= MAX_STAGES:
            raise ValueError(f"operator needs 1..{MAX_STAGES} stages, got {len(stages)}")
        op = cls()
        op.lat = lat
        op.dtype = int(dtype)
        op.n_stages = len(stages)
        op.links = links
        op.tmp = tmp
        for i, g in enumerate(stages):
            st = op.stage[i]
            st.dst_parity = int(g["dst_parity"])
            st.src, st.xself, st.out = int(g["src"]), int(g.get("xself", OPND_NONE)), int(g["out"])
            st.alpha, st.beta = float(g.get("alpha", 0.0)), float(g["beta"])
            st.clover = g.get("clover")
            st.clover_mode = int(g.get("clover_mode", 0)) if g.get("clover") else 0
            st.use_scale = int(bool(g.get("use_scale", False)))
        return op


_vp, _i32, _i64, _dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
_LAT = C.POINTER(Lattice)
_ST = C.POINTER(GmresState)
_OP = C.POINTER(Operator)

# name -> argtypes (restype int unless noted)
SIGNATURES = {
    "b200wd_abi_version": [],
    "b200wd_last_error": [],
    "b200wd_device_info": [C.c_int, C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32)],
    "b200wd_set_sm_reserve": [_i32],
    "b200wd_spinor_import": [_vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp],
    "b200wd_spinor_export": [_vp, _i32, _i64, _i32, _i32, _vp, _i32, _vp],
    "b200wd_gauge_import": [_vp, _i64, _vp, _i32, _vp],
    "b200wd_parity_split": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "b200wd_parity_merge": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
    "b200wd_hop": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _dbl, _dbl, _vp, _i32, _i32, _vp, _vp, _vp],
    "b200wd_dirac_apply": [_LAT, _i32, _i32, _dbl, _vp, _vp, _vp, _vp],
    "b200wd_hop_clover": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _dbl, _dbl, _vp, _i32, _i32, _vp, _vp, _vp,
                          _i32, _vp],
    "b200wd_hop_boundary": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _dbl, _dbl, _vp, _vp, _vp, _vp, _i32, _vp],
    "b200wd_clover_apply": [_i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "b200wd_clover_import": [_vp, _i64, _vp, _i32, _vp],
    "b200wd_halo_pack": [_LAT, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
    "b200wd_reduce_scratch_bytes": [_i32],
    "b200wd_cgs_scratch_bytes": [_i32, _i32],
    "b200wd_block_dot": [_i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
    "b200wd_block_norm2": [_i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "b200wd_block_axpy": [_i64, _i32, _i32, _vp, _vp, _vp, _vp],
    "b200wd_block_scale": [_i64, _i32, _i32, _vp, _vp, _vp],
    "b200wd_gmres_init": [_ST, _vp],
    "b200wd_gmres_residual": [_ST, _i64, _i32, _vp, _vp, _vp],
    "b200wd_gmres_start": [_ST, _vp],
    "b200wd_gmres_dot": [_ST, _i64, _i32, _vp, _vp, _vp],
    "b200wd_gmres_mgs": [_ST, _i32, _i32, _i64, _i32, _vp, _vp, _vp, _vp],
    "b200wd_gmres_close_column": [_ST, _i32, _vp],
    "b200wd_gmres_update": [_ST, _i32, _i64, _i32, C.POINTER(_vp), _vp, _vp],
    "b200wd_operator_apply": [_OP, _i32, _vp, _vp, _vp, _vp],
    "b200wd_gmres_arnoldi": [_ST, _OP, _i32, _i64, C.POINTER(_vp), _vp, _vp],
    "b200wd_gmres_cycle": [_ST, _OP, _i32, _i64, C.POINTER(_vp), _dbl, _i32, _vp, _vp, _vp, _vp, _vp],
}
RESTYPES = {"b200wd_last_error": C.c_char_p, "b200wd_reduce_scratch_bytes": _i64,
            "b200wd_cgs_scratch_bytes": _i64}

_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raises B200Unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise B200Unavailable(
            f"{p} is missing: build it with `python -m paper_2601_05816_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = RESTYPES.get(name, C.c_int)
    if lib.b200wd_abi_version() != ABI_VERSION:
        raise B200Unavailable(f"libb200wd ABI {lib.b200wd_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


class SingularBlockFromLib(RuntimeError):
    pass


def call(name: str, *args) -> int:
    """Call an entry point and map its status code to a Python exception."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != OK:
        msg = lib.b200wd_last_error().decode(errors="replace")
        if rc == ERR_ARG:
            raise ValueError(f"{name}: {msg}")
        if rc == ERR_UNSUPPORTED:
            raise NotImplementedError(f"{name}: {msg}")
        if rc == ERR_SINGULAR:
            raise SingularBlockFromLib(f"{name}: {msg}")
        raise RuntimeError(f"{name}: {msg}")
    return rc
