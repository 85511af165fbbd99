"""Kernel-level parity of the CUDA path against the CPU reference (oracle/_ref).

Protocol: SpMV/stencil bit-exact; Gram / BCGS-PIP outputs
within 1e-12 relative (Frobenius) of the reference on identical inputs;
Cholesky pivot outcomes identical.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(a - b)
    s = max(np.linalg.norm(b), 1e-300)
    return d / s


# ---- K1/K2: SpMV and MPK (spmv csr_matrix.hpp:69, mpk_monomial gmres.hpp:80) ----------
@pytest.mark.parametrize("nx,ny", [(2, 2), (3, 7), (12, 12), (100, 37), (512, 512)])
def test_laplace2d_stencil_bitwise(kb, ctx, ref, rng, nx, ny):
    a = ref.laplace2d(nx, ny)
    op = kb.Laplace2D(nx, ny)
    assert op.n == a.n
    x = rng.standard_normal(a.n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(a, x))


@pytest.mark.parametrize("dims", [(2, 2, 2), (5, 3, 4), (17, 9, 11), (64, 64, 64),
                                  # vectorised kernel: warps straddling grid rows, long z walks
                                  (6, 5, 7), (10, 33, 4), (130, 3, 19), (4, 2, 40)])
def test_laplace3d_stencil_bitwise(kb, ctx, ref, rng, dims):
    a = ref.laplace3d(*dims)
    op = kb.Laplace3D(*dims)
    x = rng.standard_normal(a.n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(a, x))


def random_csr(rng, n, per_row):
    rows = []
    for i in range(n):
        cols = np.unique(np.concatenate([[i], rng.integers(0, n, per_row)]))
        vals = rng.standard_normal(cols.size)
        vals[cols == i] += 4.0
        rows.append((cols, vals))
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([c.size for c, _ in rows])
    ci = np.concatenate([c for c, _ in rows]).astype(np.int64)
    vv = np.concatenate([v for _, v in rows])
    return rp, ci, vv


@pytest.mark.parametrize("n,per_row", [(1, 0), (40, 3), (1000, 7), (20000, 30)])
def test_csr_spmv_bitwise(kb, ctx, ref, rng, n, per_row):
    rp, ci, vv = random_csr(rng, n, per_row)
    a = ref.Csr(n, rp, ci, vv)
    op = kb.CsrOperator(rp, ci, vv)
    x = rng.standard_normal(n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(a, x))


# Column-sliced CSR (one pass per column range, running row sums carried
# between passes; kb_operator.cpp): still bit-identical, including rows with
# no entries in some slices, an empty row, the residual mode and the MPK.
@pytest.mark.parametrize("n,per_row,slices", [(20000, 30, 2), (20000, 30, 3), (5000, 4, 7), (300, 0, 5),
                                              (1, 0, 2)])
def test_csr_sliced_bitwise(kb, ctx, ref, rng, monkeypatch, n, per_row, slices):
    rp, ci, vv = random_csr(rng, n, per_row)
    if n > 2:  # empty the middle row
        i = n // 2
        lo, hi = rp[i], rp[i + 1]
        ci = np.concatenate([ci[:lo], ci[hi:]])
        vv = np.concatenate([vv[:lo], vv[hi:]])
        rp = rp.copy()
        rp[i + 1:] -= hi - lo
    a = ref.Csr(n, rp, ci, vv)
    monkeypatch.setenv("KRY_CSR_SLICES", str(slices))
    op = kb.CsrOperator(rp, ci, vv)
    x = rng.standard_normal(n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(a, x))
    start = x / np.linalg.norm(x)
    np.testing.assert_array_equal(op.mpk(start, 3), ref.mpk(a, start, 3))


def test_csr_laplace_matches_stencil(kb, ctx, ref, rng):
    a = ref.laplace2d(33, 21)
    csr = kb.CsrOperator(a.row_ptr, a.col_idx, a.vals)
    st = kb.Laplace2D(33, 21)
    x = rng.standard_normal(a.n)
    np.testing.assert_array_equal(csr.spmv(x), st.spmv(x))


@pytest.mark.parametrize("s", [1, 3, 5])
def test_mpk_bitwise(kb, ctx, ref, rng, s):
    a = ref.laplace2d(40, 30)
    op = kb.Laplace2D(40, 30)
    start = rng.standard_normal(a.n)
    start /= np.linalg.norm(start)
    np.testing.assert_array_equal(op.mpk(start, s), ref.mpk(a, start, s))


# The fused 2-D MPK (one pass, temporal blocking; k_ops.cu mpk2d_kernel):
# window seams (nx > 52), band seams (ny > 4s), odd nx (per-SpMV fallback),
# s up to 8, grids narrower than one window.
@pytest.mark.parametrize("nx,ny,s", [(130, 97, 5), (200, 64, 8), (52, 200, 2), (8, 300, 7), (131, 50, 5),
                                     (106, 41, 1), (64, 9, 6), (2, 2, 3),
                                     # a window's last lane on the grid's last column
                                     (110, 40, 5), (58, 30, 6), (104, 50, 8), (60, 33, 3), (62, 20, 1)])
def test_mpk_fused_bitwise(kb, ctx, ref, rng, monkeypatch, nx, ny, s):
    monkeypatch.setenv("KRY_FUSED_MPK", "2")  # below the size heuristic: force the one-pass kernel
    a = ref.laplace2d(nx, ny)
    op = kb.Laplace2D(nx, ny)
    start = rng.standard_normal(a.n)
    start /= np.linalg.norm(start)
    np.testing.assert_array_equal(op.mpk(start, s), ref.mpk(a, start, s))


# The fused 3-D MPK (k_ops.cu mpk3d_kernel: temporal blocking along z,
# 64 × 32 tiles shrinking by the level): tile seams in x (nx > 52) and y
# (ny > 22), z-band seams, odd nx (per-SpMV fallback), s up to 7 (s = 8
# falls back), grids smaller than one tile.
@pytest.mark.parametrize("nx,ny,nz,s", [(64, 64, 64, 5), (130, 50, 20, 5), (200, 40, 33, 7), (52, 33, 100, 5),
                                        (2, 2, 2, 1), (8, 300, 7, 3), (106, 23, 41, 2), (58, 45, 12, 6),
                                        (131, 20, 10, 5), (64, 64, 9, 8), (110, 22, 60, 4), (256, 256, 17, 5)])
def test_mpk3d_fused_bitwise(kb, ctx, ref, rng, monkeypatch, nx, ny, nz, s):
    monkeypatch.setenv("KRY_FUSED_MPK", "2")  # below the size heuristic: force the fused kernel
    a = ref.laplace3d(nx, ny, nz)
    op = kb.Laplace3D(nx, ny, nz)
    start = rng.standard_normal(a.n)
    start /= np.linalg.norm(start)
    np.testing.assert_array_equal(op.mpk(start, s), ref.mpk(a, start, s))


def prescaled(a):
    """D⁻¹A of a reference CSR on the host: a_ij / a_ii row by row."""
    from oracle import ref as R
    rows = np.repeat(np.arange(a.n), np.diff(a.row_ptr))
    d = a.vals[a.col_idx == rows]
    return R.Csr(a.n, a.row_ptr, a.col_idx, a.vals / d[rows])


@pytest.mark.parametrize("dims,shape,fused", [(2, (130, 97), "2"), (2, (131, 50), "2"), (2, (40, 30), "0"),
                                              (3, (58, 45, 12), "2"), (3, (17, 9, 11), "0"),
                                              (3, (64, 64, 64), "0")])
def test_jacobi_stencil_bitwise(kb, ctx, ref, rng, monkeypatch, dims, shape, fused):
    """Jacobi on the matrix-free Laplacians: the stencil and MPK kernels apply
    D⁻¹A (off-diagonal −1/d rounded, diagonal 1) bit-identically to the
    reference's spmv / mpk_monomial on the host pre-scaled CSR."""
    monkeypatch.setenv("KRY_FUSED_MPK", fused)
    a = ref.laplace2d(*shape) if dims == 2 else ref.laplace3d(*shape)
    op = (kb.Laplace2D if dims == 2 else kb.Laplace3D)(*shape)
    op.jacobi()
    assert op.is_jacobi
    aj = prescaled(a)
    x = rng.standard_normal(a.n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(aj, x))
    np.testing.assert_array_equal(op.mpk(x, 5), ref.mpk(aj, x, 5))


@pytest.mark.parametrize("dims,g,kind,shat", [(2, 64, 3, 60), (2, 100, 2, 0), (3, 16, 3, 60), (3, 24, 3, 20)])
def test_jacobi_stencil_solve_matches_reference(kb, ctx, ref, dims, g, kind, shat):
    """A Jacobi-preconditioned solve: the reference is handed D⁻¹A and D⁻¹b
    (b = A·1), the device gets A, b and kry_operator_jacobi."""
    a = ref.laplace2d(g, g) if dims == 2 else ref.laplace3d(g, g, g)
    b = ref.spmv(a, np.ones(a.n))
    want = ref.solve(prescaled(a), b / (4.0 if dims == 2 else 6.0), None,
                     ref.make_config(kind=kind, big_step=shat, shat=shat))
    op = (kb.Laplace2D(g, g) if dims == 2 else kb.Laplace3D(g, g, g)).jacobi()
    got = kb.sstep_gmres(op, b, None, kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat),
                                                     big_step=shat))
    assert (int(got.status), got.iterations, got.restarts, got.sync.reduces) == (
        want.status, want.iterations, want.restarts, want.reduces)
    assert abs(got.cycle_residuals[0] - want.cycle_residuals[0]) <= 1e-10 * want.cycle_residuals[0] + 1e-13
    assert abs(got.initial_residual - want.initial_residual) <= 1e-12 * want.initial_residual


def test_spmv_rejects_bad_length(kb, ctx):
    op = kb.Laplace2D(4, 4)
    with pytest.raises(kb.DimensionMismatch):
        op.spmv(np.ones(15))


def test_operator_dimension_errors(kb, ctx):
    with pytest.raises(kb.DimensionMismatch):
        kb.Laplace2D(1, 5)
    with pytest.raises(kb.DimensionMismatch):
        kb.Laplace3D(2, 2, 1)


# ---- K3: fused Gram [Q_prev V]ᵀV ---------------------------------------------------------
SHAPES = [(0, 1), (0, 6), (5, 6), (17, 3), (55, 6), (0, 21), (20, 21), (40, 21), (0, 31), (30, 31),
          (50, 11), (0, 61), (3, 61 - 3 - 1), (100, 6), (45, 16),
          # wide V beside a prefix: VᵀV alone + PᵀV in 32-column halves (m = 120, ŝ = 60 finalize)
          (60, 61), (60, 49), (7, 64)]


@pytest.mark.parametrize("c0,w", SHAPES)
@pytest.mark.parametrize("n", [7, 1000, 100003])
def test_gram_matches_reference(kb, ctx, ref, rng, n, c0, w):
    q = rng.standard_normal((n, c0))
    v = rng.standard_normal((n, w))
    rc, g = kb.gram(q if c0 else None, v)
    g_ref = ref.gram(v)
    assert rel(g, g_ref) < 1e-13
    np.testing.assert_array_equal(g, g.T)  # mirrored bit-exactly, like gram()
    if c0:
        assert rel(rc, ref.mat_mul_tn(q, v)) < 1e-13


def test_gram_deterministic(kb, ctx, rng):
    v = rng.standard_normal((300001, 6))
    q = rng.standard_normal((300001, 25))
    a = kb.gram(q, v)
    b = kb.gram(q, v)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


# ---- K4/K5: BCGS-PIP (block_ortho.hpp:152-189) -------------------------------------------
def orthonormal(rng, n, k):
    q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return np.asfortranarray(q)


@pytest.mark.parametrize("n,c0,w", [(120, 0, 5), (500, 6, 4), (4000, 55, 6), (20000, 0, 61), (20000, 40, 21),
                                    (5000, 50, 11), (100003, 25, 6), (20000, 60, 61)])
def test_bcgs_pip_matches_reference(kb, ctx, ref, rng, n, c0, w):
    q = orthonormal(rng, n, c0) if c0 else None
    v = rng.standard_normal((n, w))
    sync = kb.SyncCounter()
    res = kb.bcgs_pip(q, v, sync)
    q_ref, rc_ref, rj_ref, red = ref.bcgs_pip(q, v)
    assert sync.reduces == red == 1
    assert rel(res.q, q_ref) < 1e-12
    assert rel(res.r_jj, rj_ref) < 1e-12
    if c0:
        assert rel(res.r_col, rc_ref) < 1e-12
    assert np.all(np.diag(res.r_jj) > 0)


@pytest.mark.parametrize("n,c0,w", [(3000, 0, 70), (3000, 0, 81), (3000, 12, 75), (2000, 40, 129)])
def test_wide_blocks_match_reference(kb, ctx, ref, rng, n, c0, w):
    """Blocks wider than one 64-slot pass (finalize panels ŝ + 1 > 64):
    blocked Gram and blocked substitution (kb_ortho.cpp)."""
    q = orthonormal(rng, n, c0) if c0 else None
    v = rng.standard_normal((n, w))
    rc, g = kb.gram(q, v)
    assert rel(g, ref.gram(v)) < 1e-13
    if c0:
        assert rel(rc, ref.mat_mul_tn(q, v)) < 1e-13
    sync = kb.SyncCounter()
    res = kb.bcgs_pip(q, v, sync)
    q_ref, rc_ref, rj_ref, red = ref.bcgs_pip(q, v)
    assert rel(res.r_jj, rj_ref) < 1e-12
    assert rel(res.q, q_ref) < 1e-11
    if c0:
        assert rel(res.r_col, rc_ref) < 1e-12


def test_bcgs_pip_empty_prefix_is_cholqr(kb, ctx, rng):
    # BcgsPip.EmptyPrefixIsCholQrBitwise (tests/test_block_ortho.cpp:172-181)
    v = rng.standard_normal((120, 5))
    s1, s2 = kb.SyncCounter(), kb.SyncCounter()
    pip = kb.bcgs_pip(None, v, s1)
    chol = kb.cholqr(v, s2)
    np.testing.assert_array_equal(pip.q, chol.q)
    np.testing.assert_array_equal(np.triu(pip.r_jj), np.triu(chol.r))
    assert s1.reduces == 1


def test_bcgs_pip_rank_deficient_pivot(kb, ctx, ref, rng):
    v = rng.standard_normal((300, 4))
    v[:, 2] = 0.0  # exact zero column: pivot 3 fails for any reduction order
    sync = kb.SyncCounter()
    with pytest.raises(kb.NotPositiveDefinite) as e:
        kb.bcgs_pip(None, v, sync)
    with pytest.raises(ref.RefError) as er:
        ref.bcgs_pip(None, v)
    assert e.value.pivot == er.value.pivot == 3
    assert sync.reduces == 1


def test_bcgs_pip2_glued_matches_reference(kb, ctx, ref):
    # BcgsPip2.GluedWithinRangeStaysOrthogonal (tests/test_block_ortho.cpp:199-214)
    n, s, p = 20000, 5, 4
    glued = ref.gen_glued(n, p, s, 1e7, 1.0, 0.1, 16)
    sync = kb.SyncCounter()
    q_acc = np.zeros((n, 0), order="F")
    q_ref = np.zeros((n, 0), order="F")
    for j in range(p):
        blk = glued[:, j * s:(j + 1) * s]
        res = kb.bcgs_pip2(q_acc if q_acc.shape[1] else None, blk, sync)
        rq, rrc, rrj, _ = ref.bcgs_pip2(q_ref if q_ref.shape[1] else None, blk)
        assert rel(res.q, rq) < 1e-9
        q_acc = np.asfortranarray(np.hstack([q_acc, res.q]))
        q_ref = np.asfortranarray(np.hstack([q_ref, rq]))
    assert sync.reduces == 2 * p
    assert ref.ortho_error(q_acc) < 1e-13


def test_pip_partial_reports_partial_factor(kb, ctx, ref, rng):
    q = orthonormal(rng, 800, 6)
    v = rng.standard_normal((800, 5))
    v[:, 3] = 0.0  # zero column: the Pythagorean pivot 4 is exactly 0
    sync = kb.SyncCounter()
    out = kb.bcgs_pip_partial(q, v, sync)
    _, rc, rj, piv, _ = ref.bcgs_pip_partial(q, v)
    assert out.bad_pivot == piv
    assert out.q is None
    assert rel(out.r_col, rc) < 1e-12


# ---- Jacobi: D⁻¹A formed on the device ------------------------------
@pytest.mark.parametrize("n,slices", [(20000, 1), (20000, 3), (333, 2)])
def test_jacobi_csr_bitwise(kb, ctx, ref, rng, monkeypatch, n, slices):
    """kry_operator_jacobi on the configs[4] matrix: SpMV and MPK bit-identical
    to the reference's spmv / mpk_monomial on the host pre-scaled D⁻¹A
    (csr_matrix.hpp:69-79, gmres.hpp:80-90), unsliced and column-sliced."""
    from oracle import randsparse
    monkeypatch.setenv("KRY_CSR_SLICES", str(slices))
    op = kb.CsrOperator(*kb.gen_random_sparse(n, per_row=min(30, n)))
    assert not op.is_jacobi
    op.jacobi()
    op.jacobi()  # idempotent
    assert op.is_jacobi
    a = ref.Csr(n, *randsparse.random_sparse(n, 0, n, min(30, n), 1, 0.15, jacobi=True))
    x = rng.standard_normal(n)
    np.testing.assert_array_equal(op.spmv(x), ref.spmv(a, x))
    np.testing.assert_array_equal(op.mpk(x, 5), ref.mpk(a, x, 5))


def test_jacobi_rejects_missing_diagonal(kb, ctx, rng):
    # row 1 has no diagonal entry: refused, and the operator is left unscaled
    op = kb.CsrOperator(np.array([0, 2, 3]), np.array([0, 1, 0]), np.array([2.0, 1.0, 1.0]))
    with pytest.raises(ValueError):
        op.jacobi()
    assert not op.is_jacobi
    np.testing.assert_array_equal(op.spmv(np.array([1.0, 1.0])), np.array([3.0, 1.0]))
