"""B200-native rhs-blocked Wilson-Dirac operator and batched GMRES.

A drop-in for the hot path of ``lqcdlab`` 0.1.0 (arXiv 2601.05816's
multi-rhs Wilson-Dirac + batched GMRES, with and without odd-even
preconditioning): the public names below mirror ``lqcdlab/__init__.py``
(__init__.py:12-66) for the operator, Schur, BLAS and solver entry points.
All compute runs in hand-written sm_100a CUDA kernels (libb200wd.so, C ABI
in include/b200wd.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .fields import (  # noqa: F401
    BlockSpinorField, CloverField, GaugeField, Layout, element_offset, flip_time_boundary, gen_clover,
    gen_gauge, gen_spinor, make_rng, near_unit_gauge, near_unit_links, read_clover, read_gauge, read_spinor,
    write_clover, write_gauge, write_spinor,
)
from .geometry import LatticeGeometry, RankGrid, decompose, t_split  # noqa: F401

_LAZY = {
    "DiracParams": "dirac", "FlopCounter": "dirac", "DiracPerfRecord": "dirac", "account_traffic": "dirac",
    "apply_dirac": "dirac", "DiracOperator": "dirac",
    "SchurOperator": "oddeven", "SingularBlockError": "oddeven", "apply_schur": "oddeven",
    "reconstruct_full": "oddeven", "OeSplit": "oddeven", "split_fields": "oddeven", "merge_fields": "oddeven",
    "GmresConfig": "gmres", "GmresResult": "gmres", "gmres_solve": "gmres", "solve_dirac": "gmres",
    "dirac_op": "gmres", "matrix_op": "gmres", "SolveReport": "gmres",
    "batched_vs_independent_audit": "gmres", "gamma_residual_audit": "gmres",
    "block_axpy": "blas", "block_scale": "blas", "block_norms": "blas", "block_dot": "blas",
    "DeviceField": "device", "DeviceGauge": "device", "upload": "device", "download": "device",
    "upload_gauge": "device", "upload_packed_blocks": "device", "freeze": "device",
    "ThreadGroup": "tsplit", "HaloTimeoutError": "tsplit",
    "TSplitComm": "tsplit",
    "MultiRankExecutor": "multirank", "apply_dirac_multirank": "multirank", "EpochStats": "multirank",
    "RunConfig": "config", "ConfigError": "config", "parse_config": "config", "load_config": "config",
    "canonical": "config", "config_hash": "config",
    "arithmetic_intensity": "perf", "theoretical_perf": "perf", "read_write_ratio": "perf",
    "effective_bandwidth": "perf", "arch_efficiency": "perf", "CounterSample": "perf",
}


def __getattr__(name):
    # torch-dependent modules load on first use so that host-only users
    # (field generators, geometry) do not pay the torch import.
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = sorted(set(_LAZY) | {
    "BlockSpinorField", "CloverField", "GaugeField", "Layout", "element_offset", "flip_time_boundary",
    "gen_clover", "gen_gauge", "gen_spinor", "make_rng", "near_unit_gauge", "near_unit_links", "LatticeGeometry",
    "RankGrid", "decompose", "t_split", "read_spinor", "write_spinor", "read_gauge", "write_gauge",
    "read_clover", "write_clover",
})
