"""The BCGS2 baseline pieces on the device: cholqr2, bcgs_project
and bcgs2 with the CholQR2 intra step (block_ortho.hpp:57-137) against the
reference (oracle/_ref) on the same inputs — the shapes and matrices of the
reference's own tests/test_block_ortho.cpp:57-170.

Protocol: identical reduce counts and Cholesky pivots; Q and R within 1e-12
relative (Frobenius) on well-conditioned inputs, within the reference's
κ-scaled rounding on the glued matrices."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def orthonormal(rng, n, k):
    q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return np.asfortranarray(q)


@pytest.mark.parametrize("n,w", [(400, 5), (4000, 1), (20000, 8), (100003, 16)])
def test_cholqr2_matches_reference(kb, ctx, ref, rng, n, w):
    v = rng.standard_normal((n, w)) @ np.diag(np.logspace(0, -3, w))
    sync = kb.SyncCounter()
    got = kb.cholqr2(v, sync)
    q, r, red = ref.cholqr2(v)
    assert sync.reduces == red == 2
    assert rel(got.q, q) < 1e-12 and rel(got.r, r) < 1e-12


def test_cholqr2_beyond_range_fails_like_reference(kb, ctx, ref):
    # CholQr2.BreaksDownBeyondRange (test_block_ortho.cpp:72-83): κ = 1e9
    v = ref.gen_logscaled(100000, 5, 1e9, 3)
    sync = kb.SyncCounter()
    try:
        got = kb.cholqr2(v, sync)
        failed = ref.ortho_error(got.q) > 1e-4
    except kb.NotPositiveDefinite:
        failed = True
    assert failed


@pytest.mark.parametrize("n,c0,w", [(30, 0, 3), (200, 6, 3), (300, 8, 4), (20000, 55, 6), (100003, 30, 5)])
def test_bcgs_project_matches_reference(kb, ctx, ref, rng, n, c0, w):
    q = orthonormal(rng, n, c0) if c0 else None
    v = np.asfortranarray(rng.standard_normal((n, w)))
    sync = kb.SyncCounter()
    vhat, rb = kb.bcgs_project(q, v, sync)
    rvhat, rrb, red = ref.bcgs_project(q, v)
    assert sync.reduces == red == (1 if c0 else 0)
    assert rb.shape == rrb.shape == (c0, w)
    if c0 == 0:
        np.testing.assert_array_equal(vhat, v)  # BcgsProject.EmptyPrefixCopies: exact copy
    else:
        assert rel(rb, rrb) < 1e-12 and rel(vhat, rvhat) < 1e-12
        assert np.abs(q.T @ vhat).max() < 1e-12 * np.linalg.norm(v)


@pytest.mark.parametrize("n,c0,w", [(150, 0, 4), (200, 4, 4), (20000, 0, 1), (20000, 30, 1), (20000, 25, 5),
                                    (100003, 40, 8)])
def test_bcgs2_matches_reference(kb, ctx, ref, rng, n, c0, w):
    q = orthonormal(rng, n, c0) if c0 else None
    v = np.asfortranarray(rng.standard_normal((n, w)))
    sync = kb.SyncCounter()
    got = kb.bcgs2(q, v, sync)
    rq, rc, rj, red = ref.bcgs2(q, v)
    # first block: the intra step only (2 reduces, 1 for one column); else 1 + intra + 1 + 1
    intra = 1 if w == 1 else 2
    assert sync.reduces == red == (intra if c0 == 0 else 3 + intra)
    assert rel(got.q, rq) < 1e-12 and rel(got.r_jj, rj) < 1e-12
    if c0:
        assert rel(got.r_col, rc) < 1e-12


def test_bcgs2_glued_accumulation_matches_reference(kb, ctx, ref):
    # Bcgs2.GluedAccumulationStaysOrthogonal (test_block_ortho.cpp:123-161): κ = 1e7
    n, s, p = 20000, 5, 4
    glued = ref.gen_glued(n, p, s, 1e7, 1.0, 0.1, 10)
    sync = kb.SyncCounter()
    q_acc = np.zeros((n, 0), order="F")
    reduces_ref = 0
    for j in range(p):
        blk = np.asfortranarray(glued[:, j * s:(j + 1) * s])
        prev = q_acc if q_acc.shape[1] else None
        res = kb.bcgs2(prev, blk, sync)
        rq, rc, rj, red = ref.bcgs2(prev, blk)  # the reference on the device's prefix: same inputs
        reduces_ref += red
        assert rel(res.q, rq) < 1e-9 and rel(res.r_jj, rj) < 1e-9
        recon = (prev @ res.r_col if prev is not None else 0.0) + res.q @ np.triu(res.r_jj)
        assert np.linalg.norm(recon - blk) <= 1e-13 * np.linalg.norm(blk)
        assert (np.diag(res.r_jj) >= 0).all()
        q_acc = np.asfortranarray(np.hstack([q_acc, res.q]))
    assert sync.reduces == reduces_ref == 2 + 5 * (p - 1)
    assert ref.ortho_error(q_acc) < 1e-13


def test_bcgs2_householder_intra_is_not_on_the_device(kb, ctx, rng):
    v = np.asfortranarray(rng.standard_normal((200, 4)))
    with pytest.raises(kb.Unsupported):
        kb.bcgs2(None, v, kb.SyncCounter(), intra="hhqr")
    # one column: both intra kinds are one normalisation (CholQR), on the device
    got = kb.bcgs2(None, v[:, :1], kb.SyncCounter(), intra="hhqr")
    assert abs(np.linalg.norm(got.q) - 1.0) < 1e-14


def test_bcgs2_breakdown_reports_pivot(kb, ctx, ref, rng):
    q = orthonormal(rng, 500, 6)
    v = np.asfortranarray(rng.standard_normal((500, 4)))
    v[:, 2] = 0.0  # zero column: the first intra CholQR's pivot 3 is exactly 0
    sync = kb.SyncCounter()
    with pytest.raises(kb.NotPositiveDefinite) as e:
        kb.bcgs2(q, v, sync)
    with pytest.raises(ref.RefError) as er:
        ref.bcgs2(q, v)
    assert e.value.pivot == er.value.pivot


def test_bcgs2_abi_errors(kb, ctx, rng):
    import ctypes as C
    v = np.asfortranarray(rng.standard_normal((100, 3)))
    q = np.zeros((100, 3), order="F")
    rc = np.zeros((1, 3), order="F")
    rj = np.zeros((3, 3), order="F")
    piv, red = C.c_int64(0), C.c_int64(0)
    P = kb._capi.P_dbl
    p = lambda a: a.ctypes.data_as(P)
    lib = kb.lib()
    # unknown intra kind, negative prefix, zero width: status codes, never a crash
    assert lib.kry_bcgs2(ctx.handle, 100, None, 0, p(v), 3, 7, p(q), p(rc), p(rj), C.byref(piv), C.byref(red)) != 0
    assert lib.kry_bcgs2(ctx.handle, 100, None, -1, p(v), 3, 1, p(q), p(rc), p(rj), C.byref(piv), C.byref(red)) != 0
    assert lib.kry_bcgs_project(ctx.handle, 100, None, 0, p(v), 0, p(q), p(rc), C.byref(red)) != 0
    assert lib.kry_cholqr2(ctx.handle, 0, p(v), 3, p(q), p(rj), C.byref(piv), C.byref(red)) != 0
    assert red.value == 0
