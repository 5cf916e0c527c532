"""Drop-in correctness hazards: the reference
recomputes from the host arrays on every call, so the device path must never
apply stale links or clover, and process-global scratch must not be shared by
concurrent work on different streams."""

import numpy as np
import pytest

from oracle import lqcd_oracle as O

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2601_05816_b200")


def _field(arr, geom):
    f = P.BlockSpinorField.zeros(arr.shape[0], arr.shape[2], P.Layout.COMPONENT_MAJOR, geom=geom)
    f.set_ksi(arr)
    return f


def test_in_place_link_edit_is_seen_by_the_next_apply():
    dims = (8, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.gen_gauge_random(dims, 3), dims)
    gauge = P.GaugeField(geom, links.copy())
    psi = O.gen_spinor(geom.n_sites, 4, 5)
    f = _field(psi, geom)
    params = P.DiracParams(m0=0.1)
    a = P.apply_dirac(params, gauge, None, f).ksi()
    # one entry far from any strided sample point, edited in place
    gauge.data[777, 2, 1, 2] += 0.25 - 0.5j
    b = P.apply_dirac(params, gauge, None, f).ksi()
    want = O.apply_dirac(dims, 0.1, gauge.data, None, psi)
    assert np.linalg.norm(b - want) / np.linalg.norm(want) < 1e-12
    assert np.abs(b - a).max() > 1e-3


def test_frozen_links_upload_once_and_writeable_links_every_call():
    from paper_2601_05816_b200.device import gauge_cache
    dims = (8, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    gauge = P.GaugeField(geom, O.gen_gauge_random(dims, 4))
    f = _field(O.gen_spinor(geom.n_sites, 2, 6), geom)
    params = P.DiracParams(m0=0.1)
    u0 = gauge_cache.uploads
    P.apply_dirac(params, gauge, None, f)
    P.apply_dirac(params, gauge, None, f)
    assert gauge_cache.uploads - u0 == 2  # writeable: re-uploaded every call
    P.freeze(gauge)
    u1 = gauge_cache.uploads
    r1 = P.apply_dirac(params, gauge, None, f).ksi()
    r2 = P.apply_dirac(params, gauge, None, f).ksi()
    assert gauge_cache.uploads - u1 == 1  # read-only: cached
    assert np.array_equal(r1, r2)
    with pytest.raises(ValueError):
        gauge.data[0, 0, 0, 0] = 1.0  # a frozen array cannot change behind the cache


def test_in_place_clover_edit_is_seen_by_tsplit_bind():
    from paper_2601_05816_b200.tsplit import TSplitComm
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.near_unit_gauge(dims, 0.3, 2)
    gauge = P.GaugeField(geom, links)
    packed = O.pack_clover(O.gen_clover_random(dims, 0.1, 3))
    clover = P.CloverField(geom, packed.copy())
    psi = O.gen_spinor(geom.n_sites, 4, 7)
    comm = TSplitComm(geom)
    params = P.DiracParams(m0=0.1)
    P.apply_dirac(params, gauge, clover, _field(psi, geom), comm=comm)
    clover.data[100, 1, 5] += 0.3
    got = P.apply_dirac(params, gauge, clover, _field(psi, geom), comm=comm).ksi()
    want = O.apply_dirac(dims, 0.1, links, O.unpack_clover(clover.data), psi)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_concurrent_reductions_on_two_streams():
    """Reduction scratch is per stream: norms issued on two streams at once
    must both be exact."""
    import torch

    from paper_2601_05816_b200.blas import block_norm2_device
    from paper_2601_05816_b200.device import upload
    geom = P.LatticeGeometry((16, 8, 8, 8))
    xs = [O.gen_spinor(geom.n_sites, 12, s) for s in (1, 2)]
    d = [upload(_field(x, geom)) for x in xs]
    want = [np.einsum("xkb,xkb->b", np.conj(x), x).real for x in xs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [None, None]
    torch.cuda.synchronize()
    for _ in range(20):
        for i in (0, 1):
            with torch.cuda.stream(streams[i]):
                outs[i] = block_norm2_device(d[i])
        torch.cuda.synchronize()
        for i in (0, 1):
            got = outs[i].real.cpu().numpy()
            assert np.allclose(got, want[i], rtol=1e-12), i
