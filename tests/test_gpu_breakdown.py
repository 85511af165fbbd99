"""Breakdown and stagnation paths of the restart loop against the live
reference (gmres.hpp:315-343, 371-380; basis_store.hpp:178-208, 374-381)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def csr_from_dense_pattern(n, entries):
    rows = [[] for _ in range(n)]
    for i, j, v in entries:
        rows[i].append((j, v))
    rp = np.zeros(n + 1, np.int64)
    ci, vv = [], []
    for i in range(n):
        for j, v in sorted(rows[i]):
            ci.append(j)
            vv.append(v)
        rp[i + 1] = len(ci)
    return rp, np.array(ci, np.int64), np.array(vv)


def run_both(kb, ref, rp, ci, vv, b, kind, shat=0, standard=False):
    n = len(rp) - 1
    a = ref.Csr(n, rp, ci, vv)
    want = ref.solve(a, b, None, ref.make_config(kind=kind, big_step=shat, shat=shat), standard=standard)
    op = kb.CsrOperator(rp, ci, vv)
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat), big_step=shat)
    got = kb.standard_gmres(op, b, None, cfg) if standard else kb.sstep_gmres(op, b, None, cfg)
    return got, want


@pytest.mark.parametrize("kind,shat", [(2, 0), (3, 60), (3, 20), (1, 0)])
def test_identity_operator_lucky_breakdown(kb, ctx, ref, kind, shat):
    n = 300
    rp, ci, vv = csr_from_dense_pattern(n, [(i, i, 1.0) for i in range(n)])
    b = np.zeros(n)
    b[7] = 1.0  # exact data: every Gram entry is exactly 1, so pivot 2 fails identically everywhere
    got, want = run_both(kb, ref, rp, ci, vv, b, kind, shat)
    assert (int(got.status), got.iterations, got.restarts, got.sync.reduces, got.breakdown) == (
        want.status, want.iterations, want.restarts, want.reduces, want.breakdown)
    assert got.breakdown and int(got.status) == 0  # converged by lucky breakdown
    assert got.sync.per_block == [int(v) for v in want.per_block]
    assert abs(got.breakdown_kappa - want.breakdown_kappa) <= 1e-6 * max(1.0, abs(want.breakdown_kappa))
    np.testing.assert_allclose(got.solution, b, rtol=0, atol=1e-12)


@pytest.mark.parametrize("kind,shat", [(2, 0), (3, 60)])
def test_cyclic_shift_stagnates(kb, ctx, ref, kind, shat):
    # GMRES(60) makes no progress on a 200-cycle until m ≥ n: two ≤1 % cycles → Stagnation
    n = 200
    rp, ci, vv = csr_from_dense_pattern(n, [(i, (i + 1) % n, 1.0) for i in range(n)])
    b = np.zeros(n)
    b[0] = 1.0
    got, want = run_both(kb, ref, rp, ci, vv, b, kind, shat)
    assert int(got.status) == want.status == 3  # SolveStatus::Stagnation
    assert (got.iterations, got.restarts, got.sync.reduces) == (want.iterations, want.restarts, want.reduces)
    np.testing.assert_allclose(got.cycle_residuals, want.cycle_residuals, rtol=1e-12)


def test_standard_gmres_identity(kb, ctx, ref):
    n = 100
    rp, ci, vv = csr_from_dense_pattern(n, [(i, i, 2.0) for i in range(n)])
    b = np.zeros(n)
    b[3] = 2.0
    got, want = run_both(kb, ref, rp, ci, vv, b, 1, standard=True)
    assert (int(got.status), got.iterations, got.restarts, got.sync.reduces, got.breakdown) == (
        want.status, want.iterations, want.restarts, want.reduces, want.breakdown)


@pytest.mark.parametrize("k,kind,shat", [(9, 3, 60), (13, 3, 60), (14, 3, 60), (9, 2, 0), (13, 2, 0), (17, 2, 0)])
def test_mid_panel_breakdown_speculative_matches_synchronous(kb, ctx, ref, monkeypatch, k, kind, shat):
    """A Krylov space of dimension k (k distinct eigenvalues) ends inside the
    first big panel: the block that hits it fails its Cholesky after earlier
    blocks of the same panel were committed.  The speculative first stage
    (queued blocks, device factorisation) must roll back to that block and
    reproduce the synchronous path exactly."""
    n = 240
    rp, ci, vv = csr_from_dense_pattern(n, [(i, i, float(1 + i % k)) for i in range(n)])
    b = np.ones(n)
    reps = []
    for spec in ("1", "0"):
        monkeypatch.setenv("KRY_SPECULATE", spec)
        got, want = run_both(kb, ref, rp, ci, vv, b, kind, shat)
        reps.append(got)
    spec_rep, sync_rep = reps
    assert spec_rep.breakdown and sync_rep.breakdown
    assert (int(spec_rep.status), spec_rep.iterations, spec_rep.restarts, spec_rep.sync.reduces) == (
        int(sync_rep.status), sync_rep.iterations, sync_rep.restarts, sync_rep.sync.reduces)
    assert spec_rep.sync.per_block == sync_rep.sync.per_block
    assert spec_rep.cycle_residuals == sync_rep.cycle_residuals
    np.testing.assert_array_equal(spec_rep.solution, sync_rep.solution)
    # The reference hits the same rank deficiency.  Which of the ~ε pivots
    # fails first is a rounding-floor decision (randomised
    # sweep), so the counts are not compared here.
    assert want.breakdown


@pytest.mark.parametrize("grid,kind", [(64, 2), (100, 2), (16, 2)])
def test_speculative_pip2_matches_synchronous(kb, ctx, monkeypatch, grid, kind):
    """One-stage BCGS-PIP2 queued without host waits (both passes factorised
    on the device, replayed block by block with the per-block convergence
    check) reproduces the synchronous path bit for bit."""
    op = kb.Laplace2D(grid, grid)
    b = op.spmv(np.ones(op.n))
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), 0))
    reps = []
    for spec in ("1", "0"):
        monkeypatch.setenv("KRY_SPECULATE", spec)
        reps.append(kb.sstep_gmres(op, b, None, cfg))
    a, s = reps
    assert (int(a.status), a.iterations, a.restarts, a.sync.reduces) == (int(s.status), s.iterations, s.restarts,
                                                                        s.sync.reduces)
    assert a.sync.per_block == s.sync.per_block and a.cycle_residuals == s.cycle_residuals
    np.testing.assert_array_equal(a.solution, s.solution)


@pytest.mark.parametrize("grid,m,max_iters", [(24, 60, 600), (48, 60, 240), (40, 30, 300)])
def test_speculative_standard_gmres_matches_synchronous(kb, ctx, monkeypatch, grid, m, max_iters):
    """Standard GMRES (s = 1, BCGS2 with one column) queued without host waits
    (the four passes' coefficients formed on the device, replayed column by
    column with the per-column convergence check; synchronous once the
    prefix outgrows one Gram group) reproduces the synchronous path bit for
    bit."""
    op = kb.Laplace2D(grid, grid)
    b = op.spmv(np.ones(op.n))
    cfg = kb.SolverConfig(restart_len=m, max_iters=max_iters)
    reps = []
    for spec in ("1", "0"):
        monkeypatch.setenv("KRY_SPECULATE", spec)
        reps.append(kb.standard_gmres(op, b, None, cfg))
    a, s = reps
    assert (int(a.status), a.iterations, a.restarts, a.sync.reduces) == (int(s.status), s.iterations, s.restarts,
                                                                        s.sync.reduces)
    assert a.sync.per_block == s.sync.per_block and a.cycle_residuals == s.cycle_residuals
    np.testing.assert_array_equal(a.solution, s.solution)


def test_speculative_standard_gmres_lucky_breakdown(kb, ctx, monkeypatch):
    """A column that vanishes exactly (A = 0: the first SpMV output is the
    zero vector) fails its CholQR inside the queue; the solver redoes it on
    the synchronous path and ends exactly as the synchronous run does."""
    n = 64
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    op = kb.CsrOperator(rp, ci, np.zeros(n))
    b = np.linspace(1.0, 2.0, n)
    cfg = kb.SolverConfig(restart_len=10, max_iters=40)
    reps = []
    for spec in ("1", "0"):
        monkeypatch.setenv("KRY_SPECULATE", spec)
        reps.append(kb.standard_gmres(op, b, None, cfg))
    a, s = reps
    assert (int(a.status), a.iterations, a.restarts, a.sync.reduces, a.breakdown) == (
        int(s.status), s.iterations, s.restarts, s.sync.reduces, s.breakdown)
    np.testing.assert_array_equal(a.solution, s.solution)
