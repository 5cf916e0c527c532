"""Per-rhs BLAS-1 on block fields: drop-in for ``lqcdlab.blas`` (blas.py:1-110).

All work runs in the lane-per-rhs CUDA kernels of csrc/blas.cu.  Host
fields are uploaded, processed and (for in-place ops) written back, so the
reference API keeps its semantics; device fields never leave HBM.  The
reference's ``dot_strategy`` selects between two CPU SIMD summation orders
(blas.py:3-16); on the GPU every rhs owns its lanes, which subsumes both,
so the argument is validated and otherwise ignored.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import DeviceField, require_device, stream_ptr, upload

ACC_LANES = 8
DOT_STRATEGIES = ("naive", "deferred")

_scratch: dict = {}


def new_reduce_scratch(b: int, device=None) -> torch.Tensor:
    """A private zero-initialised reduction scratch (partials + last-block ticket)."""
    dev = device or require_device()
    nbytes = int(_lib.load().b200wd_reduce_scratch_bytes(b))
    return torch.zeros(nbytes, dtype=torch.uint8, device=dev)


def reduce_scratch(b: int, device=None) -> torch.Tensor:
    """Reduction scratch for rhs count b, one per (device, stream, b).

    The reduction kernels fold their block partials with a last-block atomic
    ticket in this buffer, so two reductions may share it only when they are
    ordered on one stream; keying by the current stream keeps concurrent
    reductions on different streams apart."""
    dev = device or require_device()
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream, b)
    t = _scratch.get(key)
    if t is None:
        t = new_reduce_scratch(b, dev)
        _scratch[key] = t
    return t


def _check_pair(x, y) -> None:
    if (x.n_sites, x.s, x.b) != (y.n_sites, y.s, y.b):
        raise ValueError(f"field shapes differ: ({x.n_sites},{x.s},{x.b}) vs ({y.n_sites},{y.s},{y.b})")
    if not isinstance(x, DeviceField) and not isinstance(y, DeviceField) and x.layout != y.layout:
        raise ValueError(f"field layouts differ: {x.layout} vs {y.layout}")


def _as_coeffs(alpha, b: int) -> np.ndarray:
    a = np.asarray(alpha, dtype=np.complex128)
    if a.ndim == 0:
        a = np.full(b, a)
    if a.shape != (b,):
        raise ValueError(f"expected {b} coefficients, got shape {a.shape}")
    return a


def _dev(f) -> DeviceField:
    d = f if isinstance(f, DeviceField) else upload(f, "c128")
    if d.dtype != "c128":
        raise NotImplementedError("the per-rhs BLAS runs in complex128 (the GMRES precision)")
    return d


def _writeback(host, dev: DeviceField) -> None:
    if not isinstance(host, DeviceField):
        dev.to_host(host.layout, out=host)


def block_axpy(alpha, x, y) -> None:
    """y[:, i] += alpha[i] x[:, i] in place (blas.py:50-55)."""
    _check_pair(x, y)
    a = torch.from_numpy(_as_coeffs(alpha, x.b)).to(require_device())
    dx, dy = _dev(x), _dev(y)
    _lib.call("b200wd_block_axpy", dx.n_sites, dx.s, dx.b, a.data_ptr(), dx.ptr, dy.ptr, stream_ptr())
    _writeback(y, dy)


def block_scale(alpha, x) -> None:
    """x[:, i] *= alpha[i] in place (blas.py:58-62)."""
    a = torch.from_numpy(_as_coeffs(alpha, x.b)).to(require_device())
    dx = _dev(x)
    _lib.call("b200wd_block_scale", dx.n_sites, dx.s, dx.b, a.data_ptr(), dx.ptr, stream_ptr())
    _writeback(x, dx)


def block_norm2_device(x: DeviceField, out: torch.Tensor | None = None) -> torch.Tensor:
    """(b,) complex128 device tensor whose real part is ||x_i||^2."""
    out = torch.empty(x.b, dtype=torch.complex128, device=x.data.device) if out is None else out
    _lib.call("b200wd_block_norm2", x.n_sites, x.s, x.b, x.ptr, out.data_ptr(),
              reduce_scratch(x.b, x.data.device).data_ptr(), stream_ptr())
    return out


def block_dot_device(w: DeviceField, e: DeviceField, out: torch.Tensor | None = None) -> torch.Tensor:
    out = torch.empty(w.b, dtype=torch.complex128, device=w.data.device) if out is None else out
    _lib.call("b200wd_block_dot", w.n_sites, w.s, w.b, w.ptr, e.ptr, out.data_ptr(),
              reduce_scratch(w.b, w.data.device).data_ptr(), stream_ptr())
    return out


def block_norms(x) -> np.ndarray:
    """(b,) Euclidean norms (blas.py:65-68)."""
    return np.sqrt(block_norm2_device(_dev(x)).real.cpu().numpy())


def _lane_width(b: int) -> int:
    """Deferred-dot lane width of the reference (blas.py:75-76), kept for API parity."""
    return max(1, -(-ACC_LANES // b)) * b


def block_dot(w, e, strategy: str = "deferred") -> np.ndarray:
    """(b,) inner products conj(w_i) . e_i (blas.py:103-110)."""
    _check_pair(w, e)
    if strategy not in DOT_STRATEGIES:
        raise ValueError(f"unknown dot strategy {strategy!r}; expected one of {DOT_STRATEGIES}")
    return block_dot_device(_dev(w), _dev(e)).cpu().numpy()
