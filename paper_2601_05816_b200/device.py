"""Device-resident fields and the host <-> device boundary.

PyTorch is used only as plumbing: CUDA memory (caching allocator), streams
and pinned host buffers.  Every byte of compute goes through libb200wd.

Device layouts (include/b200wd.h, csrc/layout.cuh):
  * spinor block field -> torch tensor (n/8, s, 8, b), complex128 or
    complex64: site-blocked component planes, rhs innermost;
  * links -> (4, n/8, 9, 8): direction-major, per 8-site block one run of
    8 per 3x3 entry.
The upload path copies the reference storage (Layout 1 or 2, complex128) as
raw bytes and converts with a device kernel; the download path is the exact
inverse.
"""

from __future__ import annotations

import warnings
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fields import SPINOR_LEN, BlockSpinorField, Layout
from .geometry import LatticeGeometry

try:
    import torch
except Exception as exc:  # pragma: no cover - torch is in the image
    raise ImportError("paper_2601_05816_b200 needs torch for device memory and streams") from exc

DTYPES = {"c128": (_lib.C128, torch.complex128, 16), "c64": (_lib.C64, torch.complex64, 8)}


def dtype_code(dtype: str) -> int:
    try:
        return DTYPES[dtype][0]
    except KeyError:
        raise ValueError(f"dtype must be 'c128' or 'c64', got {dtype!r}") from None


def torch_dtype(dtype: str):
    return DTYPES[dtype][1]


def require_device() -> "torch.device":
    """The CUDA device to use; raises B200Unavailable (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise _lib.B200Unavailable("no CUDA device: the B200 path has no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


SITE_BLOCK = 8


def _blocks(n: int) -> int:
    return -(-n // SITE_BLOCK)


@dataclass
class DeviceField:
    """A block spinor field resident in HBM.

    Storage is the site-blocked component-plane layout of csrc/layout.cuh:
    ``data`` has shape (ceil(n/8), s, 8, b), i.e. element (site, k, r) at
    data[site // 8, k, site % 8, r]; rhs is innermost.  Fields whose site
    count is not a multiple of 8 (only synthetic, non-lattice fields) carry
    zero padding sites.  ``parity`` is None for a full-lattice field, 0/1 for
    a checkerboard field whose site cb is the natural site 2*cb + (0|1).
    """

    data: "torch.Tensor"
    n: int
    geom: LatticeGeometry | None = None
    parity: int | None = None
    layout: Layout = Layout.COMPONENT_MAJOR  # layout used when downloaded

    @property
    def s(self) -> int:
        return int(self.data.shape[1])

    @property
    def n_sites(self) -> int:
        return self.n

    @property
    def b(self) -> int:
        return int(self.data.shape[3])

    @property
    def dtype(self) -> str:
        return "c128" if self.data.dtype == torch.complex128 else "c64"

    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    @classmethod
    def zeros(cls, n_sites, b, s=SPINOR_LEN, dtype="c128", geom=None, parity=None, layout=Layout.COMPONENT_MAJOR):
        dev = require_device()
        t = torch.zeros((_blocks(n_sites), s, SITE_BLOCK, b), dtype=torch_dtype(dtype), device=dev)
        return cls(t, int(n_sites), geom, parity, Layout(layout))

    @classmethod
    def empty(cls, n_sites, b, s=SPINOR_LEN, dtype="c128", geom=None, parity=None, layout=Layout.COMPONENT_MAJOR):
        if n_sites % SITE_BLOCK:
            return cls.zeros(n_sites, b, s, dtype, geom, parity, layout)  # padding must read as zero
        dev = require_device()
        t = torch.empty((_blocks(n_sites), s, SITE_BLOCK, b), dtype=torch_dtype(dtype), device=dev)
        return cls(t, int(n_sites), geom, parity, Layout(layout))

    @classmethod
    def from_logical(cls, logical: "torch.Tensor", geom=None, parity=None) -> "DeviceField":
        """(n, s, b) device tensor in logical order -> DeviceField (tests, benches)."""
        n, s, b = logical.shape
        nb = _blocks(n)
        if nb * SITE_BLOCK != n:
            pad = torch.zeros((nb * SITE_BLOCK - n, s, b), dtype=logical.dtype, device=logical.device)
            logical = torch.cat([logical, pad])
        data = logical.reshape(nb, SITE_BLOCK, s, b).permute(0, 2, 1, 3).contiguous()
        return cls(data, int(n), geom, parity)

    def empty_like(self) -> "DeviceField":
        alloc = torch.zeros_like if self.n % SITE_BLOCK else torch.empty_like
        return DeviceField(alloc(self.data), self.n, self.geom, self.parity, self.layout)

    def zeros_like(self) -> "DeviceField":
        return DeviceField(torch.zeros_like(self.data), self.n, self.geom, self.parity, self.layout)

    def copy(self) -> "DeviceField":
        return DeviceField(self.data.clone(), self.n, self.geom, self.parity, self.layout)

    @property
    def ptr(self) -> int:
        return int(self.data.data_ptr())

    def to_host(self, layout=None, out: BlockSpinorField | None = None) -> BlockSpinorField:
        """Download into the reference storage order (complex128)."""
        return download(self, layout, out)

    def logical_tensor(self) -> "torch.Tensor":
        """(n, s, b) device view in logical [site, component, rhs] order (copy)."""
        nb = self.data.shape[0]
        return self.data.permute(0, 2, 1, 3).reshape(nb * SITE_BLOCK, self.s, self.b)[: self.n]

    def logical(self) -> np.ndarray:
        """(n, s, b) complex128 numpy copy (tests / diagnostics)."""
        return self.logical_tensor().to(torch.complex128).cpu().numpy()


def _host_array(field) -> np.ndarray:
    data = np.asarray(field.data)
    if data.dtype != np.complex128:
        raise ValueError(f"host fields are complex128 (fields.py:95), got {data.dtype}")
    expect = field.n_sites * field.s * field.b
    if data.size != expect:
        raise ValueError(f"field data has {data.size} values, expected {expect}")
    return np.ascontiguousarray(data.reshape(-1))


def upload(field, dtype: str = "c128", stream=None, parity=None) -> DeviceField:
    """Host BlockSpinorField (any reference layout) -> DeviceField."""
    if isinstance(field, DeviceField):
        if field.dtype == dtype:
            return field
        return DeviceField(field.data.to(torch_dtype(dtype)), field.n, field.geom, field.parity, field.layout)
    dev = require_device()
    arr = _host_array(field)
    raw = _host_tensor(arr).to(dev, non_blocking=True)
    out = DeviceField.empty(field.n_sites, field.b, field.s, dtype, getattr(field, "geom", None), parity,
                            Layout(int(field.layout)))
    _lib.call("b200wd_spinor_import", ptr(raw), int(field.layout), field.n_sites, field.s, field.b,
              out.ptr, dtype_code(dtype), stream_ptr(stream))
    return out


def download(df: DeviceField, layout=None, out: BlockSpinorField | None = None, stream=None) -> BlockSpinorField:
    """DeviceField -> host BlockSpinorField in ``layout`` (default: df.layout)."""
    layout = Layout(int(layout if layout is not None else (out.layout if out is not None else df.layout)))
    raw = torch.empty(df.n_sites * df.s * df.b, dtype=torch.complex128, device=df.data.device)
    _lib.call("b200wd_spinor_export", df.ptr, dtype_code(df.dtype), df.n_sites, df.s, df.b, ptr(raw),
              int(layout), stream_ptr(stream))
    if out is None:
        out = BlockSpinorField.zeros(df.n_sites, df.b, layout, df.s, df.geom)
    elif (out.n_sites, out.s, out.b) != (df.n_sites, df.s, df.b):
        raise ValueError("output field shape mismatch")
    host = torch.from_numpy(out.data.reshape(-1))
    host.copy_(raw, non_blocking=False)
    return out


# ---- links ------------------------------------------------------------------


@dataclass
class DeviceGauge:
    """Links resident in HBM as (4, n/8, 9, 8) direction-major site-blocked planes."""

    data: "torch.Tensor"
    geom: LatticeGeometry

    @property
    def ptr(self) -> int:
        return int(self.data.data_ptr())

    @property
    def dtype(self) -> str:
        return "c128" if self.data.dtype == torch.complex128 else "c64"


def _host_tensor(a: np.ndarray) -> torch.Tensor:
    """CPU tensor view of a host array that is only read (frozen arrays are
    read-only; torch warns about non-writable views but never writes here)."""
    if a.flags.writeable:
        return torch.from_numpy(a)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(a)


def upload_gauge(gauge, dtype: str = "c128", stream=None) -> DeviceGauge:
    dev = require_device()
    data = np.ascontiguousarray(np.asarray(gauge.data, dtype=np.complex128))
    n = gauge.geom.n_sites
    if data.shape != (n, 4, 3, 3):
        raise ValueError(f"gauge data has shape {data.shape}, expected {(n, 4, 3, 3)}")
    raw = _host_tensor(data.reshape(-1)).to(dev, non_blocking=True)
    out = torch.empty((4, n // SITE_BLOCK, 9, SITE_BLOCK), dtype=torch_dtype(dtype), device=dev)
    _lib.call("b200wd_gauge_import", ptr(raw), n, ptr(out), dtype_code(dtype), stream_ptr(stream))
    return DeviceGauge(out, gauge.geom)


@dataclass
class DeviceClover:
    """Packed Hermitian 6x6 block pairs (clover or inverse blocks) in HBM:
    (n/8, 42, 8) site-blocked (csrc/layout.cuh clover_base)."""

    data: "torch.Tensor"
    n: int

    @property
    def ptr(self) -> int:
        return int(self.data.data_ptr())


def upload_packed_blocks(packed: np.ndarray, dtype: str = "c128", stream=None) -> DeviceClover:
    """(n, 2, 21) complex128 packed blocks (CloverField.data layout) -> device."""
    dev = require_device()
    arr = np.ascontiguousarray(np.asarray(packed, dtype=np.complex128))
    n = arr.shape[0]
    if arr.shape != (n, 2, 21) or n % SITE_BLOCK:
        raise ValueError(f"packed blocks have shape {arr.shape}; need (n, 2, 21) with n % 8 == 0")
    raw = _host_tensor(arr.reshape(-1)).to(dev, non_blocking=True)
    out = torch.empty((n // SITE_BLOCK, 42, SITE_BLOCK), dtype=torch_dtype(dtype), device=dev)
    _lib.call("b200wd_clover_import", ptr(raw), n, ptr(out), dtype_code(dtype), stream_ptr(stream))
    return DeviceClover(out, n)


class _GaugeCache:
    """Device copies of host gauge / clover arrays, with exact invalidation.

    The reference recomputes from the host arrays on every call, so an
    in-place edit of ``gauge.data`` must be seen by the next apply.  A host
    array is therefore cached only while it is read-only
    (``arr.flags.writeable == False``, e.g. after :func:`freeze`): such an array
    cannot change in place, and its identity (weakref) keys the entry.  A
    writeable array is uploaded again on every call.  Callers that apply the
    same links many times either freeze them or pass an explicit
    :class:`DeviceGauge` / :class:`DeviceClover` handle (``upload_gauge``,
    ``upload_packed_blocks``), which is never re-uploaded.
    """

    def __init__(self):
        self._entries: dict = {}
        self.uploads = 0  # host -> device link/clover uploads issued (accounting, tests)

    def get(self, gauge, dtype: str) -> DeviceGauge:
        if isinstance(gauge, DeviceGauge):
            return gauge
        return self._get(gauge.data, dtype, "gauge", lambda: upload_gauge(gauge, dtype))

    def get_clover(self, clover, dtype: str) -> DeviceClover:
        if isinstance(clover, DeviceClover):
            return clover
        return self._get(clover.data, dtype, "clover", lambda: upload_packed_blocks(clover.data, dtype))

    def _get(self, arr, dtype, kind, make):
        if not isinstance(arr, np.ndarray) or arr.flags.writeable:
            self.uploads += 1
            return make()
        key = (id(arr), dtype, kind)
        hit = self._entries.get(key)
        if hit is not None:
            ref, dg = hit
            if ref() is arr:
                return dg
        self.uploads += 1
        dg = make()
        self._entries[key] = (weakref.ref(arr), dg)
        # drop entries whose arrays died
        for k in [k for k, (r, _) in self._entries.items() if r() is None]:
            del self._entries[k]
        return dg

    def clear(self) -> None:
        self._entries.clear()


def freeze(field):
    """Mark a host GaugeField / CloverField read-only so its device copy is
    cached across calls (see :class:`_GaugeCache`); returns the field."""
    field.data.flags.writeable = False
    return field


gauge_cache = _GaugeCache()
