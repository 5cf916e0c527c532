"""GPU parity of the batched GMRES and the per-rhs BLAS.

GMRES bar (BASELINE.json north_star): the same Arnoldi iteration count as
the reference +-1 and a final true residual below the tolerance; the
residual history is compared with the reference's over the common prefix
(tests/test_gmres.py semantics), plus the reference's own fake-operator
tests (identity, scaled identity, zero rhs, initial guess, stagnation).
"""

import numpy as np
import pytest

from oracle import lqcd_oracle as O
from tests.golden_util import load_gmres

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2601_05816_b200")


def host_field(logical, layout, geom=None):
    n, s, b = logical.shape
    f = P.BlockSpinorField.zeros(n, b, layout, s, geom)
    f.set_ksi(logical)
    return f


# ---- BLAS (tests/test_blas.py) ---------------------------------------------------


@pytest.mark.parametrize("layout", [1, 2])
@pytest.mark.parametrize("b", [1, 3, 5, 12, 17])
def test_dot_and_norms(layout, b):
    x, y = O.gen_spinor(24, b, 10), O.gen_spinor(24, b, 11)
    fx, fy = host_field(x, layout), host_field(y, layout)
    ref = np.einsum("xkb,xkb->b", x.conj(), y)
    for strategy in ("naive", "deferred"):
        got = P.block_dot(fx, fy, strategy)
        assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()
    assert np.abs(P.block_norms(fx) - np.linalg.norm(x.reshape(-1, b), axis=0)).max() < 1e-12 * np.abs(x).max()


def test_axpy_scale_and_errors():
    x, y = O.gen_spinor(12, 3, 5), O.gen_spinor(12, 3, 6)
    fx, fy = host_field(x, 2), host_field(y, 2)
    alpha = np.array([1 + 2j, -0.5, 0.0])
    P.block_axpy(alpha, fx, fy)
    assert np.abs(fy.ksi() - (y + x * alpha)).max() < 1e-14
    fs = host_field(x, 1)
    P.block_scale(np.array([2.0, 0.0, 1j]), fs)
    assert np.abs(fs.ksi() - x * np.array([2.0, 0.0, 1j])).max() < 1e-14
    with pytest.raises(ValueError):
        P.block_dot(host_field(x, 1), host_field(y, 2))
    with pytest.raises(ValueError):
        P.block_dot(fx, fx, "fancy")
    z = P.BlockSpinorField.zeros(8, 2, 1)
    assert np.array_equal(P.block_norms(z), np.zeros(2))


# ---- fake-operator GMRES (tests/test_gmres.py:38-69, 163-172) ------------------------


def test_identity_one_iteration():
    eta = P.gen_spinor(16, 3, 2, seed=1)
    res = P.gmres_solve(P.matrix_op(np.eye(192)), eta, None, P.GmresConfig(tol=1e-10))
    assert res.iterations == 1 and res.converged.all() and res.breakdown.all()
    assert np.abs(res.psi.ksi() - eta.ksi()).max() < 1e-12


def test_scaled_identity_and_zero_rhs():
    eta = P.gen_spinor(16, 2, 1, seed=2)
    res = P.gmres_solve(P.matrix_op(2.0 * np.eye(192)), eta, None, P.GmresConfig(tol=1e-10))
    assert np.abs(res.psi.ksi() - 0.5 * eta.ksi()).max() < 1e-12
    z = P.BlockSpinorField.zeros(16, 2, 1)
    res = P.gmres_solve(P.matrix_op(np.eye(192)), z, None, P.GmresConfig())
    assert np.isfinite(res.psi.data).all() and not res.psi.data.any() and res.converged.all()


def test_initial_guess_respected():
    rng = np.random.default_rng(3)
    a = np.diag(rng.uniform(1.0, 2.0, 48)).astype(np.complex128)
    eta = P.gen_spinor(4, 2, 1, seed=4)
    exact = P.BlockSpinorField.zeros_like(eta)
    exact.set_columns(np.linalg.solve(a, eta.columns()))
    res = P.gmres_solve(P.matrix_op(a), eta, exact, P.GmresConfig(tol=1e-10))
    assert res.iterations == 0
    assert np.abs(res.psi.ksi() - exact.ksi()).max() < 1e-12


def test_stagnation_flagged():
    n = 192
    perm = np.roll(np.eye(n), 1, axis=0)
    eta = P.BlockSpinorField.zeros(16, 1, 1)
    eta.data[0] = 1.0
    res = P.gmres_solve(P.matrix_op(perm), eta, None, P.GmresConfig(restart_len=5, restarts=2))
    assert res.stagnated and not res.converged.any()


# ---- Wilson GMRES vs the reference goldens --------------------------------------------


@pytest.mark.parametrize("oe", [False, True])
def test_nearunit_solve_matches_reference(oe):
    g = load_gmres()[f"nearunit_8444_{'oe' if oe else 'full'}"]
    dims = tuple(g["dims"])
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, g["eps"], g["link_seed"]), dims)
    eta = host_field(O.gen_spinor(geom.n_sites, g["b"], g["eta_seed"]), 2, geom)
    cfg = P.GmresConfig(restart_len=g["restart_len"], restarts=g["restarts"], tol=g["tol"])
    rep = P.solve_dirac(P.DiracParams(m0=g["m0"]), P.GaugeField(geom, links), None, eta, cfg, odd_even=oe)
    assert abs(rep.iterations - g["iterations"]) <= 1
    assert np.all(rep.full_relnorms <= g["tol"])
    ref_h = np.array(g["history"])
    k = min(len(ref_h), len(rep.result.history))
    got_h = np.array(rep.result.history[:k])
    assert np.all(np.abs(got_h - ref_h[:k]) <= 1e-6 * ref_h[:k])
    # solution agrees with the oracle solve
    psi, _, _ = O.solve_dirac(dims, g["m0"], links, None, eta.ksi(),
                              O.GmresConfig(restart_len=g["restart_len"], restarts=g["restarts"], tol=g["tol"]),
                              odd_even=oe)
    assert np.abs(rep.psi.ksi() - psi).max() / np.abs(psi).max() < 1e-8


def test_replicated_rhs_identical_histories():
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.near_unit_gauge(dims, 0.3, 31)
    col = O.gen_spinor(256, 1, 11)
    rep = host_field(np.repeat(col, 4, axis=2), 2, geom)
    res = P.gmres_solve(P.dirac_op(P.DiracParams(m0=1.0), P.GaugeField(geom, links), None), rep, None,
                        P.GmresConfig(tol=1e-8, restarts=40))
    for h in res.history:
        assert np.ptp(h) == 0.0
    cols = res.psi.ksi()
    assert np.abs(cols - cols[:, :, :1]).max() == 0.0


def test_batched_vs_independent_and_gamma_audit():
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    op = P.dirac_op(P.DiracParams(m0=1.0), P.GaugeField(geom, O.gen_gauge_random(dims, 81)), None)
    eta = host_field(O.gen_spinor(256, 4, 10), 1, geom)
    assert P.batched_vs_independent_audit(op, eta, None, P.GmresConfig(tol=1e-8, restarts=40)) <= 1e-8
    op2 = P.dirac_op(P.DiracParams(m0=-2.0), P.GaugeField(geom, O.gen_gauge_random(dims, 82)), None)
    eta2 = host_field(O.gen_spinor(256, 2, 12), 1, geom)
    assert P.gamma_residual_audit(op2, eta2, None, P.GmresConfig(restart_len=5, restarts=3)) <= 1e-8


def test_fixed_iteration_protocol_and_reorth():
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    op = P.dirac_op(P.DiracParams(m0=1.0), P.GaugeField(geom, O.gen_gauge_random(dims, 81)), None)
    eta = host_field(O.gen_spinor(256, 2, 7), 1, geom)
    res = P.gmres_solve(op, eta, None, P.GmresConfig(restart_len=10, restarts=10, fixed_iterations=True))
    assert res.iterations == 100 and len(res.history) == 100
    r1 = P.gmres_solve(op, eta, None, P.GmresConfig(tol=1e-10, restarts=40))
    r2 = P.gmres_solve(op, eta, None, P.GmresConfig(tol=1e-10, restarts=40, reorthogonalize=True))
    assert abs(r1.iterations - r2.iterations) <= 1 and r2.converged.all()


def test_gmres_matches_oracle_dirac_small():
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.gen_gauge_random(dims, 81)
    eta = O.gen_spinor(256, 4, 5)
    ocfg = O.GmresConfig(tol=1e-10, restarts=40)
    ref = O.gmres(lambda v: O.apply_dirac(dims, 1.0, links, None, v), eta, None, ocfg)
    res = P.gmres_solve(P.dirac_op(P.DiracParams(m0=1.0), P.GaugeField(geom, links), None),
                        host_field(eta, 1, geom), None, P.GmresConfig(tol=1e-10, restarts=40))
    assert abs(res.iterations - ref.iterations) <= 1
    assert res.converged.all()
    assert np.abs(res.psi.ksi() - ref.psi).max() / np.abs(ref.psi).max() < 1e-8


@pytest.mark.parametrize("with_clover", [False, True])
def test_tsplit_comm_single_rank_matches_single_gpu(with_clover):
    """TSplitComm with one rank (no process group) is the single-GPU path,
    with and without a clover term."""
    from paper_2601_05816_b200.tsplit import TSplitComm
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 11), dims)
    gauge = P.GaugeField(geom, links)
    clover = P.CloverField(geom, O.pack_clover(O.gen_clover_random(dims, 0.05, 3))) if with_clover else None
    eta = host_field(O.gen_spinor(512, 4, 13), 2, geom)
    comm = TSplitComm(geom)
    d1 = P.apply_dirac(P.DiracParams(m0=0.1), gauge, clover, eta, comm=comm).ksi()
    d0 = P.apply_dirac(P.DiracParams(m0=0.1), gauge, clover, eta).ksi()
    assert np.abs(d1 - d0).max() == 0.0
    cfg = P.GmresConfig(restart_len=30, restarts=20, tol=1e-10)
    for oe in (False, True):
        r1 = P.solve_dirac(P.DiracParams(m0=0.1), gauge, clover, eta, cfg, odd_even=oe, comm=comm)
        r0 = P.solve_dirac(P.DiracParams(m0=0.1), gauge, clover, eta, cfg, odd_even=oe)
        assert r1.iterations == r0.iterations
        assert np.all(r1.full_relnorms <= 1e-10)


@pytest.mark.parametrize("case", ["full", "oe", "oe_clover", "full_clover"])
def test_native_arnoldi_step_bitwise_equals_python_issued(case, monkeypatch):
    """b200wd_gmres_arnoldi (one ABI call per iteration) launches the same
    kernels in the same order as the Python-issued step: identical bits."""
    import paper_2601_05816_b200.gmres as G
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 11), dims)
    clover = None
    if case.endswith("clover"):
        clover = P.CloverField(geom, O.pack_clover(O.gen_clover_random(dims, 0.05, 3)))
    eta = host_field(O.gen_spinor(512, 4, 13), 2, geom)
    cfg = P.GmresConfig(restart_len=12, restarts=20, tol=1e-10)
    runs = []
    for native in (True, False):
        monkeypatch.setattr(G, "NATIVE_ARNOLDI", native)
        runs.append(P.solve_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), clover, eta, cfg,
                                  odd_even=case.startswith("oe")))
    a, b = runs
    assert a.iterations == b.iterations
    assert np.array_equal(np.array(a.result.history), np.array(b.result.history))
    assert np.array_equal(a.psi.ksi(), b.psi.ksi())
    assert np.all(a.full_relnorms <= 1e-10)


def test_operator_apply_matches_apply_device():
    """b200wd_operator_apply of the stage programs == the Python-issued applies."""
    import ctypes
    import torch
    from paper_2601_05816_b200 import _lib
    from paper_2601_05816_b200.device import stream_ptr, upload
    dims = (8, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    gauge = P.GaugeField(geom, O.gen_gauge_random(dims, 5))
    clover = P.CloverField(geom, O.pack_clover(O.gen_clover_random(dims, 0.05, 4)))
    for dtype in ("c128", "c64"):
        for cl in (None, clover):
            op = P.DiracOperator(P.DiracParams(m0=0.2), gauge, cl, dtype)
            v = upload(host_field(O.gen_spinor(geom.n_sites, 6, 2), 2, geom), dtype)
            scale = torch.linspace(0.5, 1.5, 6, dtype=torch.float64, device="cuda")
            ref = op.apply_device(v, None, scale)
            out = v.empty_like()
            nop = op.native_operator(v)
            _lib.call("b200wd_operator_apply", ctypes.byref(nop), 6, v.ptr, out.ptr, scale.data_ptr(), stream_ptr())
            assert torch.equal(out.data, ref.data)
            for keep in (0, 1):
                so = P.SchurOperator(P.DiracParams(m0=0.2), gauge, cl, keep_parity=keep, dtype=dtype)
                ve = upload(host_field(O.gen_spinor(geom.n_sites // 2, 6, 3), 2), dtype, parity=keep)
                ref = so.apply_device(ve, None, scale)
                out = ve.empty_like()
                nop = so.native_operator(ve)
                _lib.call("b200wd_operator_apply", ctypes.byref(nop), 6, ve.ptr, out.ptr, scale.data_ptr(),
                          stream_ptr())
                assert torch.equal(out.data, ref.data)
    bad = _lib.Operator()
    with pytest.raises(ValueError):
        _lib.call("b200wd_operator_apply", ctypes.byref(bad), 6, v.ptr, out.ptr, None, stream_ptr())


@pytest.mark.parametrize("b,oe", [(1, False), (5, True), (7, False)])
def test_gmres_runtime_nrhs_matches_oracle(b, oe):
    """Batched GMRES with nrhs outside the compiled set (runtime-b kernels)."""
    dims = (4, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 51), dims)
    eta = O.gen_spinor(geom.n_sites, b, 52)
    cfg = P.GmresConfig(restart_len=12, restarts=20, tol=1e-10)
    f = P.BlockSpinorField.zeros(geom.n_sites, b, P.Layout.COMPONENT_MAJOR, geom=geom)
    f.set_ksi(eta)
    rep = P.solve_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), None, f, cfg, odd_even=oe)
    psi, out, _ = O.solve_dirac(dims, 0.1, links, None, eta,
                                O.GmresConfig(restart_len=12, restarts=20, tol=1e-10), odd_even=oe)
    assert abs(rep.iterations - out.iterations) <= 1
    assert np.all(rep.full_relnorms <= 1e-10)
    assert np.abs(rep.psi.ksi() - psi).max() / np.abs(psi).max() < 1e-8


def test_solve_layouts_and_foreign_fields_agree():
    """The same solve from Layout 1 and Layout 2 host fields, and from a
    duck-typed foreign field object (the way lqcdlab's own dataclasses are
    accepted: n_sites, s, b, layout, data), gives identical results."""
    from types import SimpleNamespace
    dims = (4, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 71), dims)
    eta = O.gen_spinor(geom.n_sites, 6, 72)
    gauge = P.GaugeField(geom, links)
    cfg = P.GmresConfig(restart_len=10, restarts=30, tol=1e-10)
    reps = []
    for layout in (1, 2):
        f = P.BlockSpinorField.zeros(geom.n_sites, 6, P.Layout(layout), geom=geom)
        f.set_ksi(eta)
        reps.append(P.solve_dirac(P.DiracParams(m0=0.1), gauge, None, f, cfg, odd_even=True))
    f2 = P.BlockSpinorField.zeros(geom.n_sites, 6, P.Layout.COMPONENT_MAJOR, geom=geom)
    f2.set_ksi(eta)
    foreign = SimpleNamespace(n_sites=f2.n_sites, s=f2.s, b=f2.b, layout=2, data=f2.data.copy(), geom=geom)
    eta_dirac = P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, foreign)
    assert np.array_equal(eta_dirac.ksi(), P.apply_dirac(P.DiracParams(m0=0.1), gauge, None, f2).ksi())
    assert reps[0].iterations == reps[1].iterations
    assert np.array_equal(reps[0].psi.ksi(), reps[1].psi.ksi())
    assert reps[0].psi.layout == 1 and reps[1].psi.layout == 2


@pytest.mark.parametrize("case", ["full", "oe_clover", "fixed"])
def test_device_cycle_bitwise_equals_per_step(case, monkeypatch):
    """b200wd_gmres_cycle (a whole restart cycle enqueued with a device-side
    stop flag, one host round trip per cycle) runs the per-step call's kernels
    in the same order: identical iterations, histories and solutions, also
    when convergence falls mid-cycle (later kernels see the flag and exit)."""
    import paper_2601_05816_b200.gmres as G
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, 0.3, 81), dims)
    clover = P.CloverField(geom, O.pack_clover(O.gen_clover_random(dims, 0.05, 82))) if "clover" in case else None
    eta = host_field(O.gen_spinor(512, 6, 83), 2, geom)
    if case == "fixed":
        cfg = P.GmresConfig(restart_len=7, restarts=3, fixed_iterations=True)
    else:
        cfg = P.GmresConfig(restart_len=16, restarts=20, tol=1e-10)
    runs = []
    for cyc in (True, False):
        monkeypatch.setattr(G, "NATIVE_CYCLE", cyc)
        runs.append(P.solve_dirac(P.DiracParams(m0=0.1), P.GaugeField(geom, links), clover, eta, cfg,
                                  odd_even=case.startswith("oe")))
    a, b = runs
    assert a.iterations == b.iterations
    if case == "fixed":
        assert a.iterations == 21
    else:
        assert a.iterations % 16 != 0  # converged inside a cycle
    assert np.array_equal(np.array(a.result.history), np.array(b.result.history))
    assert np.array_equal(a.psi.ksi(), b.psi.ksi())


@pytest.mark.parametrize("oe", [False, True])
def test_cgs_extension_matches_reference_goldens(oe):
    """The classical Gram-Schmidt extension against the reference's MGS goldens
    (8x4^3 near-unit, b=12, GMRES(30), tol 1e-10): iterations +-1, residual below
    tol, solution equal to the oracle's to 1e-8."""
    g = load_gmres()[f"nearunit_8444_{'oe' if oe else 'full'}"]
    dims = tuple(g["dims"])
    geom = P.LatticeGeometry(dims)
    links = O.flip_time_boundary(O.near_unit_gauge(dims, g["eps"], g["link_seed"]), dims)
    eta = host_field(O.gen_spinor(geom.n_sites, g["b"], g["eta_seed"]), 2, geom)
    cfg = P.GmresConfig(restart_len=g["restart_len"], restarts=g["restarts"], tol=g["tol"], orthogonalization="cgs")
    rep = P.solve_dirac(P.DiracParams(m0=g["m0"]), P.GaugeField(geom, links), None, eta, cfg, odd_even=oe)
    assert abs(rep.iterations - g["iterations"]) <= 1
    assert np.all(rep.full_relnorms <= g["tol"])
    ref_h = np.array(g["history"])
    k = min(len(ref_h), len(rep.result.history))
    assert np.all(np.abs(np.array(rep.result.history[:k]) - ref_h[:k]) <= 1e-4 * ref_h[:k])
    psi, _, _ = O.solve_dirac(dims, g["m0"], links, None, eta.ksi(),
                              O.GmresConfig(restart_len=g["restart_len"], restarts=g["restarts"], tol=g["tol"]),
                              odd_even=oe)
    assert np.abs(rep.psi.ksi() - psi).max() / np.abs(psi).max() < 1e-8


def test_cgs_extension_rejects_unsupported_paths():
    m = P.matrix_op(np.eye(12 * 16, dtype=np.complex128))
    eta = host_field(np.ones((16, 12, 2), dtype=np.complex128), 2)
    with pytest.raises(ValueError, match="cgs"):
        P.gmres_solve(m, eta, None, P.GmresConfig(orthogonalization="cgs"))
