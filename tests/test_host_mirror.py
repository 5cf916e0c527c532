"""CPU tests of the host-side mirror of the reference API (geometry, fields,
layouts, snapshots, parity split, GMRES config): the reference's own unit
tests (tests/test_geometry.py, test_fields.py, test_oddeven.py:29-49,
test_gmres.py:31-35, test_blas.py:25-31) restated against this package."""

import numpy as np
import pytest

import paper_2601_05816_b200 as P
from oracle import lqcd_oracle as O


def test_geometry_frozen_values():
    g = P.LatticeGeometry((4, 4, 4, 4))
    assert g.site_index((0, 0, 0, 0)) == 0 and g.site_index((0, 0, 0, 1)) == 1
    assert g.site_index((0, 0, 1, 0)) == 4 and g.site_index((1, 2, 3, 0)) == 108
    assert g.site_index((3, 3, 3, 3)) == 255
    assert all(g.site_index(g.site_coord(i)) == i for i in range(256))
    assert len(g.even_sites) == len(g.odd_sites) == 128
    for bad in ((4, 4, 4), (4, 3, 4, 4), (4, 0, 4, 4)):
        with pytest.raises(ValueError):
            P.LatticeGeometry(bad)
    for mu in range(4):
        for step in (1, -1):
            assert np.array_equal(g.neighbor_table(mu, step), O.neighbor_table(g.dims, mu, step))


def test_checkerboard_index_equals_reference_parity_order():
    # device parity fields use cb = site >> 1
    for dims in ((4, 4, 4, 4), (8, 4, 6, 2), (2, 2, 2, 8)):
        g = P.LatticeGeometry(dims)
        assert np.array_equal(g.even_sites >> 1, np.arange(g.n_sites // 2))
        assert np.array_equal(g.odd_sites >> 1, np.arange(g.n_sites // 2))


def test_decompose_and_rank_grid():
    g = P.LatticeGeometry((8, 4, 4, 4))
    doms = P.decompose(g, P.RankGrid((2, 1, 1, 1)))
    assert len(doms) == 2 and doms[0].local_geom.dims == (4, 4, 4, 4)
    assert np.array_equal(np.sort(np.concatenate([d.global_sites for d in doms])), np.arange(g.n_sites))
    assert len(doms[0].boundary[(0, 1)]) == 64 and len(doms[0].boundary[(1, 1)]) == 0
    with pytest.raises(ValueError):
        P.decompose(g, P.RankGrid((3, 1, 1, 1)))


def test_element_offset_and_layouts():
    assert P.element_offset(P.Layout.RHS_MAJOR, 6, 2, 5, 4, 1) == 70
    assert P.element_offset(P.Layout.COMPONENT_MAJOR, 6, 2, 5, 4, 1) == 69
    with pytest.raises(ValueError):
        P.element_offset(P.Layout.RHS_MAJOR, 6, 2, 0, 6, 0)
    f1 = P.gen_spinor(16, 3, P.Layout.RHS_MAJOR, seed=9)
    f2 = P.gen_spinor(16, 3, P.Layout.COMPONENT_MAJOR, seed=9)
    assert np.array_equal(f1.ksi(), f2.ksi()) and not np.array_equal(f1.data, f2.data)
    assert np.array_equal(f1.convert(2).convert(1).data, f1.data)


def test_generators_match_oracle_and_reference_streams():
    g = P.LatticeGeometry((4, 4, 4, 4))
    assert np.array_equal(P.gen_gauge(g, "random", seed=21).data, O.gen_gauge_random(g.dims, 21))
    assert np.array_equal(P.gen_clover(g, "random", 0.1, seed=22).blocks(), O.gen_clover_random(g.dims, 0.1, 22))
    assert np.array_equal(P.gen_spinor(256, 3, 2, seed=33).ksi(), O.gen_spinor(256, 3, 33))
    assert np.array_equal(P.near_unit_links(g.dims, 0.3, 5), O.near_unit_gauge(g.dims, 0.3, 5))
    P.gen_gauge(g, "random", seed=1).validate()
    P.near_unit_gauge(g, 0.3, 5).validate()
    with pytest.raises(ValueError):
        P.flip_time_boundary(P.near_unit_gauge(g, 0.3, 5)).validate()  # det = -1 on the flipped slice
    with pytest.raises(ValueError):
        P.gen_gauge(g, "hot")


def test_snapshot_roundtrip(tmp_path):
    g = P.LatticeGeometry((2, 2, 2, 4))
    f = P.gen_spinor(g.n_sites, 3, 2, seed=4, geom=g)
    P.write_spinor(tmp_path / "psi.snap", f)
    r = P.read_spinor(tmp_path / "psi.snap")
    assert np.array_equal(r.data, f.data) and r.layout == f.layout and r.geom.dims == g.dims
    u = P.gen_gauge(g, "random", seed=3)
    P.write_gauge(tmp_path / "u.snap", u)
    assert np.array_equal(P.read_gauge(tmp_path / "u.snap").data, u.data)
    c = P.gen_clover(g, "random", seed=5)
    P.write_clover(tmp_path / "c.snap", c)
    assert np.array_equal(P.read_clover(tmp_path / "c.snap").data, c.data)
    (tmp_path / "bad.snap").write_bytes(b"XXXX" + b"\0" * 40)
    with pytest.raises(ValueError):
        P.read_spinor(tmp_path / "bad.snap")


def test_split_merge_fields_host():
    from paper_2601_05816_b200.oddeven import OeSplit, merge_fields, split_fields
    g = P.LatticeGeometry((4, 4, 4, 4))
    v = P.gen_spinor(g.n_sites, 3, 1, seed=70, geom=g)
    split = OeSplit.from_geom(g)
    ve, vo = split_fields(v, split)
    assert ve.n_sites == vo.n_sites == 128
    assert np.array_equal(merge_fields(ve, vo, split).data, v.data)
    assert np.array_equal(ve.ksi(), v.ksi()[split.even])


def test_gmres_config_and_ledger():
    from paper_2601_05816_b200.blas import _lane_width
    from paper_2601_05816_b200.dirac import FlopCounter, account_traffic
    with pytest.raises(ValueError):
        P.GmresConfig(restart_len=0)
    with pytest.raises(ValueError):
        P.GmresConfig(tol=0.0)
    with pytest.raises(ValueError, match="orthogonalization"):
        P.GmresConfig(orthogonalization="householder")
    assert P.GmresConfig().orthogonalization == "mgs"  # the reference's MGS by default
    assert account_traffic(1) == {"flops_per_site": 2574, "bytes_per_site": 4512}
    assert account_traffic(16) == {"flops_per_site": 41184, "bytes_per_site": 44832}
    assert FlopCounter(cmul=2, cadd=3, rmul=4).total_flops == 26
    assert [_lane_width(b) for b in (1, 2, 3, 8, 16)] == [8, 8, 9, 8, 16]
    with pytest.raises(ValueError):
        P.DiracParams(m0=0.0, a=0.5)


def test_compute_paths_fail_loudly_without_gpu():
    """No CPU fallback: without a CUDA device every compute entry point raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2601_05816_b200._lib import B200Unavailable
    g = P.LatticeGeometry((2, 2, 2, 8))
    psi = P.gen_spinor(g.n_sites, 2, 2, seed=1, geom=g)
    with pytest.raises(B200Unavailable):
        P.apply_dirac(P.DiracParams(), P.gen_gauge(g, "unit"), None, psi)
    with pytest.raises(B200Unavailable):
        P.block_norms(psi)


def test_near_unit_links_forked_workers_same_bits():
    from paper_2601_05816_b200.fields import near_unit_links
    dims = (6, 4, 4, 2)
    ref = near_unit_links(dims, 0.3, 5)
    assert np.array_equal(near_unit_links(dims, 0.3, 5, workers=4), ref)
    assert np.array_equal(near_unit_links(dims, 0.3, 5, 1, 5, workers=3), ref[32:160])


def test_multirank_executor_arguments():
    """halo.py:225-233 argument rules; the B200 executor splits T only."""
    P.MultiRankExecutor(P.RankGrid((2, 1, 1, 1)), mode="threads")
    with pytest.raises(ValueError):
        P.MultiRankExecutor(P.RankGrid((2, 1, 1, 1)), mode="processes")
    with pytest.raises(NotImplementedError):
        P.MultiRankExecutor(P.RankGrid((1, 2, 1, 1)))


def test_perf_model_formulas():
    """perf.py:64-99: AI(1) = 0.570, AI(16) = 0.919, ratios, bandwidth."""
    from fractions import Fraction
    assert abs(float(P.arithmetic_intensity(1)) - 0.570) < 1e-3
    assert abs(float(P.arithmetic_intensity(16)) - 0.919) < 1e-3
    assert P.read_write_ratio(2) == Fraction(204 * 2 + 330, 408)
    assert P.theoretical_perf(1e9, 4) == 1e9 * float(P.arithmetic_intensity(4))
    s = P.CounterSample(l2_refill=100, l2_writeback=50, cycles=1000, frequency=2e9, ranks=2)
    assert P.effective_bandwidth(s) == 150 * 256 * 2e9 / 1000 * 2
    with pytest.raises(ValueError):
        P.arithmetic_intensity(0)
    with pytest.raises(ValueError):
        P.CounterSample(-1, 0, 1, 1.0)


def test_reference_written_snapshots_read_and_rewrite_byte_identical(tmp_path, golden_dir):
    """Files written by lqcdlab itself (tests/golden/make_golden_snapshots.py)
    read back into the generators' values, and this package writes the very
    same bytes (fields.py:264-337)."""
    import paper_2601_05816_b200 as P
    geom = P.LatticeGeometry((4, 2, 2, 4))
    g = P.read_gauge(golden_dir / "snap_gauge.lqmg")
    assert np.array_equal(g.data, P.gen_gauge(geom, "random", seed=11).data)
    c = P.read_clover(golden_dir / "snap_clover.lqmc")
    assert np.array_equal(c.data, P.gen_clover(geom, "random", scale=0.1, seed=12).data)
    P.write_gauge(tmp_path / "g", g)
    P.write_clover(tmp_path / "c", c)
    assert (tmp_path / "g").read_bytes() == (golden_dir / "snap_gauge.lqmg").read_bytes()
    assert (tmp_path / "c").read_bytes() == (golden_dir / "snap_clover.lqmc").read_bytes()
    for layout in (1, 2):
        name = f"snap_spinor_l{layout}.lqml"
        f = P.read_spinor(golden_dir / name)
        want = P.gen_spinor(geom.n_sites, 3, P.Layout(layout), seed=13, geom=geom)
        assert int(f.layout) == layout and f.b == 3 and np.array_equal(f.data, want.data)
        P.write_spinor(tmp_path / name, want)
        assert (tmp_path / name).read_bytes() == (golden_dir / name).read_bytes()
