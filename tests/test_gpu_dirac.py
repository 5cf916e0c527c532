"""GPU parity: the sm_100a Wilson-Dirac / Schur kernels vs the oracle and
the reference-generated golden fixtures.

Tolerances (BASELINE.json north_star): relative Frobenius error <= 1e-12
for complex128 and <= 1e-5 for complex64 (against the reference run on the
c64-rounded inputs).
"""

import numpy as np
import pytest

from oracle import lqcd_oracle as O
from tests.golden_util import checksum, load_npz

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2601_05816_b200")


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def host_field(logical, layout, geom=None):
    n, s, b = logical.shape
    f = P.BlockSpinorField.zeros(n, b, layout, s, geom)
    f.set_ksi(logical)
    return f


@pytest.fixture(scope="module")
def cfg1():
    dims = (8, 8, 8, 8)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.gen_gauge_random(dims, 0), dims)
    psi = O.gen_spinor(geom.n_sites, 4, 2)
    return geom, links, psi


def test_cfg1_matches_reference_golden(cfg1):
    geom, links, psi = cfg1
    f = load_npz("dirac_cfg1.npz")
    gauge = P.GaugeField(geom, links)
    eta = P.apply_dirac(P.DiracParams(m0=0.1), gauge, P.gen_clover(geom, "zero"),
                        host_field(psi, P.Layout.COMPONENT_MAJOR, geom)).ksi()
    assert rel(eta[7 * 512:], f["eta_last_slice"]) < 1e-12
    assert np.abs(checksum(eta) - f["checksum"]).max() < 1e-12 * np.abs(f["checksum"]).max()
    assert np.abs(np.linalg.norm(eta.reshape(-1, 4), axis=0) - f["norms"]).max() < 1e-12 * f["norms"].max()


@pytest.mark.parametrize("b", [1, 2, 3, 4, 8, 12, 16, 32])
@pytest.mark.parametrize("layout", [1, 2])
def test_dirac_c128_matches_oracle(b, layout):
    dims = (4, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.gen_gauge_random(dims, 100 + b)
    psi = O.gen_spinor(geom.n_sites, b, 200 + b)
    ref = O.apply_dirac(dims, -0.5, links, None, psi)
    got = P.apply_dirac(P.DiracParams(m0=-0.5), P.GaugeField(geom, links), None,
                        host_field(psi, P.Layout(layout), geom))
    assert got.layout == layout and got.b == b
    assert rel(got.ksi(), ref) < 1e-12


@pytest.mark.parametrize("b", [1, 2, 3, 4, 12, 16])
def test_dirac_c64_matches_oracle_on_rounded_inputs(b):
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 5), dims)
    psi = O.gen_spinor(geom.n_sites, b, 300 + b)
    ref = O.apply_dirac(dims, 0.1, O.round_c64(links), None, O.round_c64(psi))
    got = P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None,
                        host_field(psi, P.Layout.COMPONENT_MAJOR, geom), dtype="c64")
    assert rel(got.ksi(), ref) < 1e-5


def test_free_field_identity():
    geom = P.LatticeGeometry((4, 4, 4, 4))
    psi = np.full((256, 12, 2), 1.0 + 0.5j)
    eta = P.apply_dirac(P.DiracParams(m0=-0.5), P.gen_gauge(geom, "unit"), P.gen_clover(geom, "zero"),
                        host_field(psi, P.Layout.RHS_MAJOR, geom))
    assert np.abs(eta.ksi() + 0.5 * psi).max() < 1e-14


def test_device_field_roundtrip_and_linearity():
    from paper_2601_05816_b200.device import upload
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    a = O.gen_spinor(256, 3, 1)
    c = O.gen_spinor(256, 3, 2)
    for layout in (1, 2):
        d = upload(host_field(a, P.Layout(layout), geom))
        assert np.array_equal(d.to_host(layout).ksi(), a)
    links = O.gen_gauge_random(dims, 3)
    g = P.GaugeField(geom, links)
    prm = P.DiracParams(m0=0.3)
    lhs = P.apply_dirac(prm, g, None, host_field(a + 2 * c, 2, geom)).ksi()
    rhs = P.apply_dirac(prm, g, None, host_field(a, 2, geom)).ksi() + \
        2 * P.apply_dirac(prm, g, None, host_field(c, 2, geom)).ksi()
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()


def test_perf_record_and_flops():
    geom = P.LatticeGeometry((4, 4, 4, 4))
    psi = host_field(O.gen_spinor(256, 2, 3), 1, geom)
    perf, flops = [], P.FlopCounter()
    P.apply_dirac(P.DiracParams(), P.gen_gauge(geom, "random", 1), None, psi, flops=flops, perf=perf)
    (r,) = perf
    assert r.sites == 256 and r.b == 2 and r.flops == 2574 * 256 * 2 and r.seconds > 0
    assert 0.85 <= flops.total_flops / (256 * 2) / 2574 <= 1.15


def test_schur_nearunit_matches_reference_golden():
    f = load_npz("schur_8444_nearunit.npz")
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 7), dims)
    gauge = P.GaugeField(geom, links)
    s = P.SchurOperator(P.DiracParams(m0=0.1), gauge, None)
    v = host_field(O.gen_spinor(256, 3, 74), P.Layout.COMPONENT_MAJOR)
    assert rel(s.apply(v).ksi(), f["out"]) < 1e-12
    eta = host_field(O.gen_spinor(512, 3, 75), P.Layout.COMPONENT_MAJOR, geom)
    red, el = s.reduce_rhs(eta)
    assert rel(red.ksi(), f["reduced"]) < 1e-12
    assert rel(s.reconstruct(red, el).ksi(), f["x_odd"]) < 1e-12
    d = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, host_field(O.gen_spinor(512, 3, 76), 2, geom))
    assert rel(d.ksi(), f["dirac_out"]) < 1e-12


@pytest.mark.parametrize("keep", [0, 1])
@pytest.mark.parametrize("dtype,tol", [("c128", 1e-12), ("c64", 1e-5)])
def test_schur_matches_oracle(keep, dtype, tol):
    dims = (4, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.near_unit_gauge(dims, 0.3, 9)
    v = O.gen_spinor(256, 4, 11)
    so = O.SchurOracle(dims, 0.1, O.round_c64(links) if dtype == "c64" else links, None, keep_parity=keep)
    ref = so.apply(O.round_c64(v) if dtype == "c64" else v)
    sp = P.SchurOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, keep_parity=keep, dtype=dtype)
    from paper_2601_05816_b200.device import upload
    got = sp.apply_device(upload(host_field(v, 2), dtype, parity=keep)).logical()
    assert rel(got, ref) < tol


def test_schur_constant_field_and_singular():
    geom = P.LatticeGeometry((4, 4, 4, 4))
    s = P.SchurOperator(P.DiracParams(m0=0.5), P.gen_gauge(geom, "unit"), P.gen_clover(geom, "zero"))
    v = host_field(np.full((128, 12, 2), 1.0 + 0j), 1)
    assert np.abs(s.apply(v).ksi() - (4.5 - 16 / 4.5)).max() < 1e-12
    with pytest.raises(P.SingularBlockError) as err:
        P.SchurOperator(P.DiracParams(m0=-4.0), P.gen_gauge(P.LatticeGeometry((2, 2, 2, 2)), "unit"), None)
    assert "site" in str(err.value)


HALO_SHAPES = [((8, 4, 4, 6), 3, "c128"),    # generic kernel
               ((8, 4, 4, 16), 4, "c128"),   # ring kernel with halo tiles
               ((8, 4, 4, 16), 12, "c128"),
               ((8, 4, 4, 16), 16, "c64"),
               ((8, 4, 4, 32), 8, "c64")]


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("parity", [None, 0, 1])
@pytest.mark.parametrize("shape", HALO_SHAPES, ids=lambda s: f"{s[0][3]}z_b{s[1]}_{s[2]}")
@pytest.mark.parametrize("split_launch", [0, 1, 2], ids=["whole_slab", "interior_boundary", "boundary_merged"])
def test_tsplit_halo_kernels_reproduce_single_gpu(nranks, parity, shape, split_launch):
    """Emulate the T split on one GPU: per-slab pack -> face swap -> hop with
    halos, either one launch over the slab or TSplitComm's sequence (interior
    slices, then the two boundary slices); nrhs >= 4 runs the ring kernel with
    the halo faces as bulk-copied tiles (the boundary fast path)."""
    import torch
    from paper_2601_05816_b200 import _lib
    from paper_2601_05816_b200.device import DeviceField, upload, upload_gauge
    from paper_2601_05816_b200.dirac import hop_device
    from paper_2601_05816_b200.oddeven import device_split

    dims, b, dt = shape
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 21), dims)
    psi = O.gen_spinor(geom.n_sites, b, 22)
    full_lat = _lib.Lattice.make(dims)
    g_full = upload_gauge(P.GaugeField(geom, links), dt)
    d_psi = upload(host_field(psi, 2, geom), dt)
    code = 0 if dt == "c128" else 1
    tdt = torch.complex128 if dt == "c128" else torch.complex64
    if parity is None:
        ref = DeviceField.empty(geom.n_sites, b, dtype=dt)
        hop_device(full_lat, dt, b, -1, g_full, d_psi, ref, d_psi, 4.1, -1.0)
        src_full = d_psi
    else:
        e, o = device_split(full_lat, d_psi)
        src_full = o if parity == 0 else e  # source parity 1-p
        ref = DeviceField.empty(geom.n_sites // 2, b, dtype=dt)
        hop_device(full_lat, dt, b, parity, g_full, src_full, ref, None, 0.0, 1.0)
    tl = dims[0] // nranks
    per_t = geom.sites_per_slice
    per = per_t if parity is None else per_t // 2
    slabs = []
    for r in range(nranks):
        lg = P.LatticeGeometry((tl,) + dims[1:])
        lat = _lib.Lattice.make(lg.dims, r * tl)
        gl = upload_gauge(P.GaugeField(lg, links[r * tl * per_t:(r + 1) * tl * per_t]), dt)
        nloc = tl * per
        src = DeviceField(src_full.data[r * nloc // 8:(r + 1) * nloc // 8].contiguous(), nloc)
        lam = torch.empty((6, per, b), dtype=tdt, device="cuda")
        chi = torch.empty_like(lam)
        sp = -1 if parity is None else 1 - parity
        _lib.call("b200wd_halo_pack", lat, code, b, sp, gl.ptr, src.ptr, lam.data_ptr(), chi.data_ptr(), 0)
        slabs.append((lg, lat, gl, src, lam, chi))
    outs = []
    for r, (lg, lat, gl, src, _, _) in enumerate(slabs):
        lam_from_up = slabs[(r + 1) % nranks][4]
        chi_from_down = slabs[(r - 1) % nranks][5]
        out = DeviceField(torch.empty_like(src.data), src.n)
        xs, al, be = (src, 4.1, -1.0) if parity is None else (None, 0.0, 1.0)
        pp = -1 if parity is None else parity
        if not split_launch:
            hop_device(lat, dt, b, pp, gl, src, out, xs, al, be, lam_halo=lam_from_up, chi_halo=chi_from_down)
        else:
            if tl > 2:
                hop_device(lat, dt, b, pp, gl, src, out, xs, al, be, t_begin=1, t_end=tl - 1)
            if split_launch == 1:
                for t0, t1 in ((0, 1), (tl - 1, tl)):
                    hop_device(lat, dt, b, pp, gl, src, out, xs, al, be, t_begin=t0, t_end=t1,
                               lam_halo=lam_from_up, chi_halo=chi_from_down)
            else:  # both boundary slices in one launch (b200wd_hop_boundary)
                _lib.call("b200wd_hop_boundary", lat, code, b, pp, gl.ptr, src.ptr,
                          None if xs is None else xs.ptr, out.ptr, al, be, None, lam_from_up.data_ptr(),
                          chi_from_down.data_ptr(), None, 0, 0)
        outs.append(out.data)
    got = torch.cat(outs, dim=0)
    err = (got - ref.data).abs().max().item() / ref.data.abs().max().item()
    assert err < (1e-14 if dt == "c128" else 1e-6), err


# ---- clover term (reference fixtures use random clover) ----


def test_dirac_clover_matches_reference_golden():
    f = load_npz("dirac_4444_clover.npz")
    dims = tuple(int(x) for x in f["dims"])
    geom = P.LatticeGeometry(dims)
    gauge = P.GaugeField(geom, f["links"])
    clover = P.CloverField(geom, f["clover_packed"])
    psi = host_field(f["psi"], 2, geom)
    eta = P.apply_dirac(P.DiracParams(m0=float(f["m0"])), gauge, clover, psi).ksi()
    assert rel(eta, f["eta"]) < 1e-12
    # Layout 1 input, c64
    eta1 = P.apply_dirac(P.DiracParams(m0=float(f["m0"])), gauge, clover, host_field(f["psi"], 1, geom)).ksi()
    assert rel(eta1, f["eta"]) < 1e-12
    ref64 = O.apply_dirac(dims, float(f["m0"]), O.round_c64(f["links"]),
                          O.round_c64(O.unpack_clover(f["clover_packed"])), O.round_c64(f["psi"]))
    eta64 = P.apply_dirac(P.DiracParams(m0=float(f["m0"])), gauge, clover, psi, dtype="c64").ksi()
    assert rel(eta64, ref64) < 1e-5


def test_schur_clover_matches_reference_golden():
    f = load_npz("schur_4444_clover.npz")
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    gauge = P.GaugeField(geom, O.gen_gauge_random(dims, 61))
    clover = P.gen_clover(geom, "random", scale=0.1, seed=62)
    s = P.SchurOperator(P.DiracParams(m0=-0.5), gauge, clover)
    v = host_field(f["v"], 2)
    assert rel(s.apply(v).ksi(), f["out"]) < 1e-12
    eta = host_field(O.gen_spinor(256, 2, 73), 2, geom)
    red, el = s.reduce_rhs(eta)
    assert rel(red.ksi(), f["reduced"]) < 1e-12
    assert rel(s.reconstruct(red, el).ksi(), f["x_odd"]) < 1e-12


def test_schur_clover_keep_odd_matches_oracle():
    dims = (4, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.gen_gauge_random(dims, 5)
    cl = O.gen_clover_random(dims, 0.1, 6)
    so = O.SchurOracle(dims, 0.2, links, cl, keep_parity=1)
    v = O.gen_spinor(256, 3, 7)
    sp = P.SchurOperator(P.DiracParams(m0=0.2), P.GaugeField(geom, links),
                         P.CloverField(geom, O.pack_clover(cl)), keep_parity=1)
    assert rel(sp.apply(host_field(v, 2)).ksi(), so.apply(v)) < 1e-12


def test_gmres_clover_matches_reference_golden():
    from tests.golden_util import load_gmres
    g = load_gmres()["clover_4444_m1"]
    dims = tuple(g["dims"])
    geom = P.LatticeGeometry(dims)
    gauge = P.GaugeField(geom, O.gen_gauge_random(dims, g["gauge_seed"]))
    clover = P.gen_clover(geom, "random", scale=0.1, seed=g["clover_seed"])
    eta = P.gen_spinor(256, g["b"], P.Layout.RHS_MAJOR, seed=g["eta_seed"], geom=geom)
    res = P.gmres_solve(P.dirac_op(P.DiracParams(m0=g["m0"]), gauge, clover), eta, None,
                        P.GmresConfig(tol=g["tol"], restarts=g["restarts"]))
    assert abs(res.iterations - g["iterations"]) <= 1 and res.converged.all()
    ref_h = np.array(g["history"])
    k = min(len(ref_h), len(res.history))
    live = ref_h[:k] > 1e-10
    assert np.all(np.abs(np.array(res.history[:k]) - ref_h[:k])[live] <= 1e-8 * ref_h[:k][live])
    # odd-even solve with clover agrees with the direct one
    cfg = P.GmresConfig(tol=1e-10, restarts=40)
    d = P.solve_dirac(P.DiracParams(m0=g["m0"]), gauge, clover, eta, cfg, odd_even=False)
    s = P.solve_dirac(P.DiracParams(m0=g["m0"]), gauge, clover, eta, cfg, odd_even=True)
    assert np.all(s.full_relnorms <= 1e-9) and s.iterations < d.iterations
    assert np.abs(d.psi.ksi() - s.psi.ksi()).max() / np.abs(d.psi.ksi()).max() < 1e-7


@pytest.mark.parametrize("dims", [(4, 4, 4, 16), (4, 2, 2, 32), (6, 2, 4, 8), (2, 2, 2, 48)])
@pytest.mark.parametrize("b,dtype,tol", [(4, "c128", 1e-12), (12, "c128", 1e-12), (16, "c128", 1e-12),
                                         (8, "c64", 1e-5), (16, "c64", 1e-5)])
def test_dirac_clover_wide_rhs_matches_oracle(dims, b, dtype, tol):
    """Clover at nrhs >= 4 on ring-shaped lattices (the clover epilogue stays in
    the generic kernel: profiles/r1_tstream_tuning.txt, clover section)."""
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 21), dims)
    cl = O.gen_clover_random(dims, 0.1, 22)
    psi = O.gen_spinor(geom.n_sites, b, 23)
    c64 = dtype == "c64"
    ref = O.apply_dirac(dims, 0.1, O.round_c64(links) if c64 else links, O.round_c64(cl) if c64 else cl,
                        O.round_c64(psi) if c64 else psi)
    got = P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), P.CloverField(geom, O.pack_clover(cl)),
                        host_field(psi, 2, geom), dtype=dtype).ksi()
    assert rel(got, ref) < tol


@pytest.mark.parametrize("dims", [(4, 4, 4, 16), (4, 2, 2, 32)])
@pytest.mark.parametrize("b,dtype,tol", [(4, "c128", 1e-12), (12, "c128", 1e-12), (8, "c64", 1e-5)])
def test_schur_clover_wide_rhs_matches_oracle(dims, b, dtype, tol):
    """Both clover modes at nrhs >= 4: M = D_oo^-1 on the eliminated hop,
    -C_ee x on the kept one."""
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 24), dims)
    cl = O.gen_clover_random(dims, 0.1, 25)
    v = O.gen_spinor(geom.n_sites // 2, b, 26)
    c64 = dtype == "c64"
    from paper_2601_05816_b200.device import upload
    for keep in (0, 1):
        so = O.SchurOracle(dims, 0.1, O.round_c64(links) if c64 else links, O.round_c64(cl) if c64 else cl,
                           keep_parity=keep)
        ref = so.apply(O.round_c64(v) if c64 else v)
        sp = P.SchurOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links),
                             P.CloverField(geom, O.pack_clover(cl)), keep_parity=keep, dtype=dtype)
        got = sp.apply_device(upload(host_field(v, 2), dtype, parity=keep)).logical()
        assert rel(got, ref) < tol


@pytest.mark.parametrize("dims", [(4, 4, 4, 16), (4, 2, 2, 32), (6, 2, 4, 16), (4, 2, 2, 48)])
@pytest.mark.parametrize("b,dtype,tol", [(4, "c128", 1e-12), (12, "c128", 1e-12), (16, "c128", 1e-12),
                                         (8, "c64", 1e-5), (16, "c64", 1e-5)])
def test_schur_ring_path_matches_oracle(dims, b, dtype, tol):
    """Z % 16 == 0 lattices take the checkerboard TMA ring kernel."""
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 17), dims)
    v = O.gen_spinor(geom.n_sites // 2, b, 18)
    for keep in (0, 1):
        so = O.SchurOracle(dims, 0.1, O.round_c64(links) if dtype == "c64" else links, None, keep_parity=keep)
        ref = so.apply(O.round_c64(v) if dtype == "c64" else v)
        sp = P.SchurOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, keep_parity=keep, dtype=dtype)
        from paper_2601_05816_b200.device import upload
        got = sp.apply_device(upload(host_field(v, 2), dtype, parity=keep)).logical()
        assert rel(got, ref) < tol
    # reduce_rhs / reconstruct on the same lattice
    eta = O.gen_spinor(geom.n_sites, b, 19)
    so = O.SchurOracle(dims, 0.1, links, None)
    red_ref, el_ref = so.reduce_rhs(eta)
    sp = P.SchurOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None)
    red, el = sp.reduce_rhs(host_field(eta, 2, geom))
    assert rel(red.ksi(), red_ref) < 1e-12
    assert rel(sp.reconstruct(red, el).ksi(), so.reconstruct(red_ref, el_ref)) < 1e-12


@pytest.mark.parametrize("dims", [(4, 4, 4, 16), (4, 2, 6, 24), (4, 2, 2, 32), (4, 2, 2, 48)])
@pytest.mark.parametrize("b", [4, 6, 12, 16, 24, 32])
def test_ring_full_lattice_shapes(dims, b):
    """Z = 16, 24, 32, 48 exercise whole-line, partial-line (z-edge) and
    line-straddling ring items (c64 nrhs 12 on Z >= 48 uses 32-site items)."""
    geom = P.LatticeGeometry(dims)
    links = O.near_unit_gauge(dims, 0.3, 23)
    psi = O.gen_spinor(geom.n_sites, b, 24)
    ref = O.apply_dirac(dims, 0.1, links, None, psi)
    got = P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, host_field(psi, 2, geom))
    assert rel(got.ksi(), ref) < 1e-12
    got64 = P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, host_field(psi, 2, geom),
                          dtype="c64")
    assert rel(got64.ksi(), O.apply_dirac(dims, 0.1, O.round_c64(links), None, O.round_c64(psi))) < 1e-5


@pytest.mark.parametrize("layout", [1, 2])
def test_host_pipelined_apply_matches_device_apply(layout):
    """apply_dirac on host fields overlaps H2D/compute/D2H over T chunks."""
    import torch
    dims = (16, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 31), dims)
    psi = O.gen_spinor(geom.n_sites, 4, 32)
    ref = O.apply_dirac(dims, 0.1, links, None, psi)
    n = geom.n_sites
    pin_in = torch.empty(n * 48, dtype=torch.complex128).pin_memory()
    pin_out = torch.empty(n * 48, dtype=torch.complex128).pin_memory()
    f = P.BlockSpinorField(n, 12, 4, P.Layout(layout), pin_in.numpy(), geom)
    f.set_ksi(psi)
    o = P.BlockSpinorField(n, 12, 4, P.Layout(layout), pin_out.numpy(), geom)
    for chunks in (1, 2, 4, 8, 16):
        op = P.DiracOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None)
        op.apply_host_pipelined(f, o, chunks=chunks)
        assert rel(o.ksi(), ref) < 1e-12
    ref64 = O.apply_dirac(dims, 0.1, O.round_c64(links), None, O.round_c64(psi))
    for chunks in (3, 16):  # 16 % 3 != 0: falls back to 2 chunks
        op = P.DiracOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, "c64")
        op.apply_host_pipelined(f, o, chunks=chunks)
        assert rel(o.ksi(), ref64) < 1e-5


@pytest.mark.parametrize("dims", [(2, 2, 2, 2), (2, 4, 2, 6), (6, 2, 2, 4)])
@pytest.mark.parametrize("b", [5, 7, 10, 40])
def test_runtime_nrhs_and_small_lattices(dims, b):
    """nrhs outside the compiled set (the runtime-b kernel), the minimum 2^4
    lattice and z extents 2/4/6 (generic kernel), full operator and Schur, c128
    and c64."""
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 31 + b), dims)
    psi = O.gen_spinor(geom.n_sites, b, 32 + b)
    gauge = P.GaugeField(geom, links)
    ref = O.apply_dirac(dims, 0.1, links, None, psi)
    got = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, host_field(psi, 2, geom))
    assert rel(got.ksi(), ref) < 1e-12
    got64 = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, host_field(psi, 1, geom), dtype="c64")
    assert rel(got64.ksi(), O.apply_dirac(dims, 0.1, O.round_c64(links), None, O.round_c64(psi))) < 1e-5
    v = O.gen_spinor(geom.n_sites // 2, b, 33 + b)
    so = O.SchurOracle(dims, 0.1, links, None, keep_parity=0)
    sp = P.SchurOperator(P.DiracParams(m0=0.1), gauge, None, keep_parity=0)
    assert rel(sp.apply(host_field(v, 2)).ksi(), so.apply(v)) < 1e-12


def test_max_nrhs():
    """b = 128, the largest rhs block the ABI accepts; 129 is rejected."""
    dims = (2, 2, 2, 4)
    geom = P.LatticeGeometry(dims)
    links = O.gen_gauge_random(dims, 5)
    psi = O.gen_spinor(geom.n_sites, 128, 6)
    got = P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, host_field(psi, 2, geom))
    assert rel(got.ksi(), O.apply_dirac(dims, 0.1, links, None, psi)) < 1e-12
    with pytest.raises(ValueError):
        P.apply_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None,
                      host_field(O.gen_spinor(geom.n_sites, 129, 6), 2, geom))


@pytest.mark.parametrize("b,dtype", [(16, "c128"), (12, "c128"), (4, "c128"), (16, "c64"), (8, "c64"), (4, "c64")])
def test_slice_range_applies_default_dispatch(b, dtype):
    """apply_range (the T-split interior / pipelined-apply call) through the
    default kernel choice (ring, two-line ring, T stream) on a whole-line
    lattice: every slice range reproduces the oracle on those slices."""
    import torch
    from paper_2601_05816_b200.device import upload
    dims = (8, 4, 4, 16)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 41), dims)
    psi = O.gen_spinor(geom.n_sites, b, 42)
    if dtype == "c64":
        links_r, psi_r, tol = O.round_c64(links), O.round_c64(psi), 1e-5
    else:
        links_r, psi_r, tol = links, psi, 1e-12
    ref = O.apply_dirac(dims, 0.1, links_r, None, psi_r)
    op = P.DiracOperator(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, dtype)
    x = upload(host_field(psi, 2, geom), dtype)
    per = geom.sites_per_slice
    for t0, t1 in [(1, 7), (0, 3), (3, 8), (5, 6)]:
        y = x.zeros_like()
        op.apply_range(x, y, t0, t1)
        torch.cuda.synchronize()
        got = y.logical()
        assert rel(got[t0 * per:t1 * per], ref[t0 * per:t1 * per]) < tol, (t0, t1)
        assert not np.any(got[:t0 * per]) and not np.any(got[t1 * per:])
