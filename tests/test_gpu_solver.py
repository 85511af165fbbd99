"""Solver parity (gmres.hpp): the CUDA path against the CPU reference on the
same operator and right-hand side (b = A·1, x0 = 0).

Parity protocol: identical status, iteration, restart and
reduce counts and SyncCounter deltas; cycle-1 residual within 1e-10
relative; later cycles within the tolerance below, which is set from the
reference's own FMA/non-FMA self-divergence (up to 8.6e-7 relative at 128²,
3.9e-10 at 64²: rounding differences compound over restarts).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LATE_CYCLE_RTOL = 1e-5
ABS_FLOOR = 1e-13


def run_pair(kb, ref, grid, kind, shat, standard=False, dims=2):
    if dims == 2:
        a = ref.laplace2d(grid, grid)
        op = kb.Laplace2D(grid, grid)
    else:
        a = ref.laplace3d(grid, grid, grid)
        op = kb.Laplace3D(grid, grid, grid)
    b = ref.spmv(a, np.ones(a.n))
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat), big_step=shat)
    if standard:
        got = kb.standard_gmres(op, b, None, cfg)
    else:
        got = kb.sstep_gmres(op, b, None, cfg)
    want = ref.solve(a, b, None, ref.make_config(kind=kind, big_step=shat, shat=shat), standard=standard)
    return got, want


def assert_parity(got, want):
    assert int(got.status) == want.status
    assert got.iterations == want.iterations
    assert got.restarts == want.restarts
    assert got.sync.reduces == want.reduces
    assert got.sync.per_block == want.per_block
    assert got.sync.per_big_panel == want.per_big_panel
    assert len(got.cycle_residuals) == len(want.cycle_residuals)
    c_got, c_want = np.array(got.cycle_residuals), np.array(want.cycle_residuals)
    # Residuals are relative to r0; an explicit residual b − A·x is itself only
    # accurate to ~1e-15·r0, hence the absolute floor (ABS_FLOOR, units of r0).
    assert abs(c_got[0] - c_want[0]) <= 1e-10 * c_want[0] + ABS_FLOOR
    assert np.all(np.abs(c_got - c_want) <= LATE_CYCLE_RTOL * c_want + ABS_FLOOR)
    assert abs(got.initial_residual - want.initial_residual) <= 1e-12 * want.initial_residual


@pytest.mark.parametrize("grid", [16, 64, 100])
def test_pip2_solve_parity(kb, ctx, ref, grid):
    got, want = run_pair(kb, ref, grid, 2, 0)
    assert_parity(got, want)
    if grid == 100:  # SURVEY §8(c) anchors
        assert (got.iterations, got.restarts, got.sync.reduces) == (270, 4, 108)


@pytest.mark.parametrize("grid,shat", [(64, 60), (100, 60), (100, 20), (100, 30), (100, 5), (128, 60)])
def test_two_stage_solve_parity(kb, ctx, ref, grid, shat):
    got, want = run_pair(kb, ref, grid, 3, shat)
    assert_parity(got, want)
    if grid == 100 and shat == 60:
        assert (got.iterations, got.restarts, got.sync.reduces) == (300, 4, 65)
    if grid == 100 and shat == 20:
        assert (got.iterations, got.restarts, got.sync.reduces) == (280, 4, 70)


def test_two_stage_hat5_equals_pip2(kb, ctx, ref):
    got5, _ = run_pair(kb, ref, 64, 3, 5)
    gotp, _ = run_pair(kb, ref, 64, 2, 0)
    assert got5.iterations == gotp.iterations and got5.sync.reduces == gotp.sync.reduces


def test_laplace3d_two_stage_parity(kb, ctx, ref):
    got, want = run_pair(kb, ref, 16, 3, 60, dims=3)
    assert_parity(got, want)


def test_standard_gmres_parity(kb, ctx, ref):
    got, want = run_pair(kb, ref, 32, 1, 0, standard=True)
    assert_parity(got, want)


def test_solution_quality(kb, ctx, ref):
    a = ref.laplace2d(64, 64)
    op = kb.Laplace2D(64, 64)
    b = ref.spmv(a, np.ones(a.n))
    rep = kb.sstep_gmres(op, b, None, kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, 60)))
    r = b - ref.spmv(a, rep.solution)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1e-6 * (1 + 1e-9)
    assert abs(np.linalg.norm(r) / np.linalg.norm(b) - rep.final_relative_residual) < 1e-12


def test_csr_operator_solve_parity(kb, ctx, ref):
    a = ref.laplace2d(48, 48)
    op = kb.CsrOperator(a.row_ptr, a.col_idx, a.vals)
    b = ref.spmv(a, np.ones(a.n))
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, 60))
    got = kb.sstep_gmres(op, b, None, cfg)
    want = ref.solve(a, b, None, ref.make_config(kind=3))
    assert_parity(got, want)


def test_warm_start_and_max_iters(kb, ctx, ref):
    a = ref.laplace2d(64, 64)
    op = kb.Laplace2D(64, 64)
    b = ref.spmv(a, np.ones(a.n))
    x0 = np.full(a.n, 0.5)
    cfg = kb.SolverConfig(max_iters=120)
    got = kb.sstep_gmres(op, b, x0, cfg)
    want = ref.solve(a, b, x0, ref.make_config(max_iters=120))
    assert_parity(got, want)
    assert got.status == kb.SolveStatus.MAX_ITERS


def test_config_validation(kb, ctx):
    op = kb.Laplace2D(8, 8)
    b = np.ones(64)
    with pytest.raises(kb.DimensionMismatch):
        kb.sstep_gmres(op, b, None, kb.SolverConfig(restart_len=12, step=5))
    with pytest.raises(kb.DimensionMismatch):
        kb.sstep_gmres(op, b, None, kb.SolverConfig(big_step=7))
    with pytest.raises(ValueError):
        kb.sstep_gmres(op, b, None, kb.SolverConfig(rel_tol=0.0))


def test_zero_rhs_converges_immediately(kb, ctx):
    op = kb.Laplace2D(8, 8)
    rep = kb.sstep_gmres(op, np.zeros(64), None, kb.SolverConfig())
    assert rep.status == kb.SolveStatus.CONVERGED and rep.iterations == 0
