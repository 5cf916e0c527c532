"""Parity at the BASELINE configurations' full sizes (the benchmarked shapes).

* configs[1]: D_W on 16^3 x 32 with seeded random SU(3) links and Gaussian
  nrhs-16 spinors, m0 = 0.1 -- small enough for the oracle to check directly
  (c128 <= 1e-12, c64 <= 1e-5 on c64-rounded inputs).
* configs[2]: the odd-even Schur operator on 32^3 x 64, nrhs 12, near-unit
  links, antiperiodic T -- checked at full size through an identity that needs
  no CPU reference: for x = (v_e, -D_oo^-1 D_oe v_e), (D x)_e = S v_e and
  (D x)_o = 0, with D, S, the elimination and the parity split/merge all
  computed by different device kernels.
"""
import numpy as np
import pytest
import torch

from oracle import lqcd_oracle as O

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2601_05816_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_configs1_full_size_matches_oracle():
    dims = (32, 16, 16, 16)
    geom = P.LatticeGeometry(dims)
    links = O.gen_gauge_random(dims, 0)
    psi = O.gen_spinor(geom.n_sites, 16, 2)
    f = P.BlockSpinorField.zeros(geom.n_sites, 16, P.Layout.COMPONENT_MAJOR, geom=geom)
    f.set_ksi(psi)
    gauge = P.GaugeField(geom, links)
    got = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, f).ksi()
    assert rel(got, O.apply_dirac(dims, 0.1, links, None, psi)) < 1e-12
    got64 = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, f, dtype="c64").ksi()
    assert rel(got64, O.apply_dirac(dims, 0.1, O.round_c64(links), None, O.round_c64(psi))) < 1e-5


def test_configs2_full_size_schur_identity():
    from paper_2601_05816_b200.device import DeviceField
    from paper_2601_05816_b200.oddeven import device_merge, device_split
    dims = (64, 32, 32, 32)
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 3))
    params = P.DiracParams(m0=0.1)
    schur = P.SchurOperator(params, gauge, None, keep_parity=0)
    dirac = P.DiracOperator(params, gauge, None)
    half = geom.n_sites // 2
    g = torch.Generator(device="cuda").manual_seed(5)
    v = DeviceField(torch.randn((half // 8, 12, 8, 12), dtype=torch.complex128, device="cuda", generator=g), half,
                    geom, 0)
    zero = DeviceField(torch.zeros_like(v.data), half, geom, 1)
    x_odd = schur.reconstruct_device(v, zero)  # -D_oo^-1 D_oe v
    x = device_merge(schur.lat, v, x_odd, geom)
    y_even, y_odd = device_split(schur.lat, dirac.apply_device(x))
    s_v = schur.apply_device(v)
    torch.cuda.synchronize()
    ye, yo, sv = y_even.data, y_odd.data, s_v.data
    assert (torch.linalg.vector_norm(ye - sv) / torch.linalg.vector_norm(sv)).item() < 1e-12
    assert (torch.linalg.vector_norm(yo) / torch.linalg.vector_norm(ye)).item() < 1e-13


def test_configs4_full_size_eight_way_t_split():
    """configs[4] (48^3 x 96, nrhs 12, near-unit links, antiperiodic T): the
    8-rank T split through the device face pack and halo-consuming kernels
    (MultiRankExecutor, the multi-GPU path's kernels) reproduces the
    single-GPU apply to rounding."""
    import os

    from paper_2601_05816_b200.device import DeviceField
    dims = (96, 48, 48, 48)
    geom = P.LatticeGeometry(dims)
    links = P.near_unit_links(dims, 0.3, 0, workers=os.cpu_count() or 1)
    gauge = P.flip_time_boundary(P.GaugeField(geom, links))
    params = P.DiracParams(m0=0.1)
    n = geom.n_sites
    g = torch.Generator(device="cuda").manual_seed(7)
    psi = DeviceField(torch.randn((n // 8, 12, 8, 12), dtype=torch.complex128, device="cuda", generator=g), n, geom)
    ref = P.DiracOperator(params, gauge, None).apply_device(psi)
    ex = P.MultiRankExecutor(P.RankGrid((8, 1, 1, 1)))
    got = ex.apply_device(params, gauge, None, psi)
    torch.cuda.synchronize()
    err = (torch.linalg.vector_norm(got.data - ref.data) / torch.linalg.vector_norm(ref.data)).item()
    assert err < 1e-14, err
