"""The reference's acceptance criteria (tests/test_acceptance.py) run against
the B200 package: 1 operator vs dense oracle, 2 free field, 3 layout
invariance, 4 batched vs independent, 5 gamma tracks the residual, 6 odd-even
iteration reduction, plus the remaining reference semantics tests
(monotone residual within a cycle, one-shot Schur wrappers, reduce -> solve ->
reconstruct solves the full system)."""

import numpy as np
import pytest

from oracle import lqcd_oracle as O

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2601_05816_b200")
SEED = 2024


@pytest.fixture(scope="module")
def lattice44():
    g = P.LatticeGeometry((4, 4, 4, 4))
    return g, P.gen_gauge(g, "random", seed=SEED), P.gen_clover(g, "random", scale=0.1, seed=SEED + 1)


@pytest.fixture(scope="module")
def lattice84():
    g = P.LatticeGeometry((8, 4, 4, 4))
    return g, P.gen_gauge(g, "random", seed=SEED + 2), P.gen_clover(g, "random", scale=0.1, seed=SEED + 3)


def test_criterion_01_operator_vs_dense(lattice44):
    g, u, c = lattice44
    dense = O.assemble_dirac_dense(g.dims, -0.5, u.data, c.blocks())
    worst = 0.0
    for b in (1, 2, 4, 8):
        for layout in (P.Layout.RHS_MAJOR, P.Layout.COMPONENT_MAJOR):
            psi = P.gen_spinor(g.n_sites, b, layout, seed=SEED + 10 + b, geom=g)
            eta = P.apply_dirac(P.DiracParams(m0=-0.5), u, c, psi)
            ref = dense @ psi.columns()
            worst = max(worst, np.linalg.norm(eta.columns() - ref) / np.linalg.norm(ref))
    assert worst <= 1e-12


def test_criterion_03_layout_invariance(lattice44):
    g, u, c = lattice44
    prm = P.DiracParams(m0=1.0)
    p1 = P.gen_spinor(g.n_sites, 4, 1, seed=SEED + 20, geom=g)
    p2 = p1.convert(2)
    e1, e2 = P.apply_dirac(prm, u, c, p1), P.apply_dirac(prm, u, c, p2)
    worst = np.abs(e1.ksi() - e2.ksi()).max() / np.abs(e1.ksi()).max()
    d1, d2 = P.block_dot(p1, e1), P.block_dot(p2, e2)
    worst = max(worst, np.abs(d1 - d2).max() / np.abs(d1).max())
    n1, n2 = P.block_norms(e1), P.block_norms(e2)
    worst = max(worst, np.abs(n1 - n2).max() / n1.max())
    assert worst <= 1e-13
    cfg = P.GmresConfig(restart_len=10, restarts=10, fixed_iterations=True)
    r1 = P.gen_spinor(g.n_sites, 4, 1, seed=SEED + 21, geom=g)
    s1 = P.gmres_solve(P.dirac_op(prm, u, c), r1, None, cfg)
    s2 = P.gmres_solve(P.dirac_op(prm, u, c), r1.convert(2), None, cfg)
    assert np.abs(s1.psi.ksi() - s2.psi.ksi()).max() / np.abs(s1.psi.ksi()).max() <= 1e-8


def test_criterion_04_05_batched_and_gamma(lattice44):
    g, u, c = lattice44
    op = P.dirac_op(P.DiracParams(m0=1.0), u, c)
    eta = P.gen_spinor(g.n_sites, 4, 1, seed=SEED + 30, geom=g)
    assert P.batched_vs_independent_audit(op, eta, None, P.GmresConfig(tol=1e-8, restarts=40)) <= 1e-8
    op2 = P.dirac_op(P.DiracParams(m0=-2.0), u, c)
    eta2 = P.gen_spinor(g.n_sites, 4, 1, seed=SEED + 40, geom=g)
    assert P.gamma_residual_audit(op2, eta2, None, P.GmresConfig(restart_len=10, restarts=10)) <= 1e-8


def test_criterion_06_odd_even_iteration_reduction(lattice44, lattice84):
    cfg = P.GmresConfig(tol=1e-8, restarts=60)
    for g, u, c in (lattice44, lattice84):
        eta = P.gen_spinor(g.n_sites, 4, 2, seed=SEED + 50, geom=g)
        d = P.solve_dirac(P.DiracParams(m0=1.0), u, c, eta, cfg, odd_even=False)
        s = P.solve_dirac(P.DiracParams(m0=1.0), u, c, eta, cfg, odd_even=True)
        assert s.iterations / d.iterations <= 2.0 / 3.0
        assert np.all(d.full_relnorms <= 1e-8) and np.all(s.full_relnorms <= 1e-8)
        assert np.abs(d.psi.ksi() - s.psi.ksi()).max() / np.abs(d.psi.ksi()).max() <= 1e-6


def test_history_monotone_within_cycle(lattice44):
    g, u, c = lattice44
    eta = P.gen_spinor(g.n_sites, 3, 2, seed=6, geom=g)
    res = P.gmres_solve(P.dirac_op(P.DiracParams(m0=1.0), u, c), eta, None, P.GmresConfig(tol=1e-8, restarts=40))
    h = np.array(res.history)
    for j in range(1, len(h)):
        if j % 10:
            assert np.all(h[j] <= h[j - 1] + 1e-14)


def test_reduce_dense_solve_reconstruct_and_wrappers(lattice44):
    g, u, c = lattice44
    prm = P.DiracParams(m0=-0.5)
    eta = P.gen_spinor(g.n_sites, 2, 2, seed=73, geom=g)
    s = P.SchurOperator(prm, u, c)
    reduced, elim = s.reduce_rhs(eta)
    dense = O.SchurOracle(g.dims, -0.5, u.data, c.blocks())
    # dense Schur matrix from the oracle's apply on unit vectors is too large; use the dense D instead
    D = O.assemble_dirac_dense(g.dims, -0.5, u.data, c.blocks())
    ev = (g.even_sites[:, None] * 12 + np.arange(12)).ravel()
    od = (g.odd_sites[:, None] * 12 + np.arange(12)).ravel()
    S = D[np.ix_(ev, ev)] - D[np.ix_(ev, od)] @ np.linalg.solve(D[np.ix_(od, od)], D[np.ix_(od, ev)])
    x = P.BlockSpinorField.zeros_like(reduced)
    x.set_columns(np.linalg.solve(S, reduced.columns()))
    psi = s.merge(x, s.reconstruct(x, elim))
    r = P.apply_dirac(prm, u, c, psi)
    assert np.linalg.norm(r.columns() - eta.columns()) / np.linalg.norm(eta.columns()) < 1e-12
    v = P.gen_spinor(g.n_sites // 2, 1, 1, seed=74)
    assert np.array_equal(P.apply_schur(prm, u, c, v).data, s.apply(v).data)
    x_odd = P.reconstruct_full(prm, u, c, x, elim)
    assert np.abs(x_odd.ksi() - s.reconstruct(x, elim).ksi()).max() == 0.0
    assert dense.n_sites == s.n_sites


@pytest.mark.parametrize("ranks", [1, 2, 4])
@pytest.mark.parametrize("with_clover", [False, True])
def test_multirank_executor_matches_single_rank(ranks, with_clover):
    """apply_dirac(..., comm=MultiRankExecutor(grid)) (halo.py:216-401): rank
    slabs with device halo exchange reproduce the single-rank apply."""
    dims = (8, 4, 4, 8)
    geom = P.LatticeGeometry(dims)
    gauge = P.gen_gauge(geom, "random", seed=61)
    clover = P.gen_clover(geom, "random", scale=0.1, seed=62) if with_clover else P.gen_clover(geom, "zero")
    psi = P.gen_spinor(geom.n_sites, 4, P.Layout.COMPONENT_MAJOR, seed=63, geom=geom)
    params = P.DiracParams(m0=0.1)
    ref = P.apply_dirac(params, gauge, clover, psi).ksi()
    got, ex = P.apply_dirac_multirank(params, gauge, clover, psi, P.RankGrid((ranks, 1, 1, 1)))
    assert np.linalg.norm(got.ksi() - ref) / np.linalg.norm(ref) < 1e-14
    assert len(ex.last_stats) == ranks
    via_comm = P.apply_dirac(params, gauge, clover, psi, comm=P.MultiRankExecutor(P.RankGrid((ranks, 1, 1, 1))))
    assert np.array_equal(via_comm.ksi(), got.ksi())


def test_multirank_executor_full_solve():
    """solve_dirac(..., comm=MultiRankExecutor(grid)) (gmres.py:353-385): the
    unpreconditioned solve applies D through the rank slabs."""
    dims = (8, 4, 4, 4)
    geom = P.LatticeGeometry(dims)
    gauge = P.flip_time_boundary(P.near_unit_gauge(geom, 0.3, 91))
    eta = P.gen_spinor(geom.n_sites, 3, P.Layout.COMPONENT_MAJOR, seed=92, geom=geom)
    cfg = P.GmresConfig(restart_len=20, restarts=20, tol=1e-10)
    params = P.DiracParams(m0=0.1)
    ref = P.solve_dirac(params, gauge, None, eta, cfg)
    got = P.solve_dirac(params, gauge, None, eta, cfg, comm=P.MultiRankExecutor(P.RankGrid((4, 1, 1, 1))))
    assert abs(got.iterations - ref.iterations) <= 1 and np.all(got.full_relnorms <= 1e-10)
    assert np.abs(got.psi.ksi() - ref.psi.ksi()).max() / np.abs(ref.psi.ksi()).max() < 1e-8
