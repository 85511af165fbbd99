"""Basis-store parity (basis_store.hpp) — the reference's BasisStore tests
(tests/test_block_ortho.cpp:271-421) restated against the device store, plus
step-by-step comparison with the reference store on identical inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("kind", ["pip2", "bcgs2", "two"])
def test_raw_sequence_reconstruction(kb, ctx, ref, kind):
    # BasisStore.RawSequenceReconstruction (tests/test_block_ortho.cpp:331-380), MPK in the store.
    grid, m, s = 12, 12, 3
    a = ref.laplace2d(grid, grid)
    n = a.n
    op = kb.Laplace2D(grid, grid)
    b = ref.spmv(a, np.ones(n))
    v1 = b / np.linalg.norm(b)
    kinds = {"pip2": kb.OrthoKind.BCGS_PIP2, "bcgs2": kb.OrthoKind.BCGS2_CHOLQR2, "two": kb.OrthoKind.TWO_STAGE}
    store = kb.BasisStore(n, m, s, m)
    sync = kb.SyncCounter()
    scheme = kb.OrthoScheme(kinds[kind], m)
    raw = []
    for j in range(m // s):
        start = v1 if j == 0 else store.column(store.filled() - 1)
        blk = ref.mpk(a, start, s)
        raw.extend(blk[:, (0 if j == 0 else 1):].T)
        if kind == "two":
            oc = store.preprocess_block(blk, j != 0, sync)
        else:
            oc = store.append_block(blk, j != 0, scheme, sync)
        assert not oc.breakdown
    if kind == "two":
        store.finalize_big_panel(sync)
    raw = np.array(raw).T
    assert raw.shape[1] == store.filled()
    r = store.coefficients()
    q = store.all()
    recon = q @ np.triu(r[: q.shape[1], : q.shape[1]])
    assert np.linalg.norm(recon - raw) <= 1e-12 * np.linalg.norm(raw)
    assert np.all(np.diag(r)[: q.shape[1]] >= 0)


@pytest.mark.parametrize("kind,shat", [(2, 0), (3, 12), (3, 6), (3, 3), (1, 0)])
def test_store_matches_reference_step_by_step(kb, ctx, ref, kind, shat):
    """Same MPK-fed blocks into both stores: R, Q, records and sync deltas agree."""
    grid, m, s = 16, 12, 3
    a = ref.laplace2d(grid, grid)
    n = a.n
    b = ref.spmv(a, np.ones(n))
    v1 = b / np.linalg.norm(b)
    eff = shat if shat else m
    st = kb.BasisStore(n, m, s, eff)
    rs = ref.Store(n, m, s, eff)
    sync = kb.SyncCounter()
    rdeltas = []
    for j in range(m // s):
        start = v1 if j == 0 else rs.column(rs.info().filled - 1)
        blk = ref.mpk(a, start, s)
        if kind == 3:
            o = st.preprocess_block(blk, j != 0, sync)
            ro, d = rs.preprocess_block(blk, j != 0)
        else:
            o = st.append_block(blk, j != 0, kb.OrthoScheme(kb.OrthoKind(kind), 0), sync)
            ro, d = rs.append_block(blk, j != 0, kind)
        rdeltas.append(d)
        assert (o.committed, o.truncated, o.breakdown) == (ro.committed, bool(ro.truncated), bool(ro.breakdown))
        if kind == 3 and (rs.info().big_panel_full or j + 1 == m // s):
            st.finalize_big_panel(sync)
            rs.finalize_big_panel()
        assert st.filled() == rs.info().filled
        assert st.finalized_count() == rs.info().finalized
        assert st.big_panel_start() == rs.info().big_panel_start
        assert rel(st.coefficients(), rs.coefficients()) < 1e-10
        assert rel(st.all(), rs.all()) < 1e-10
    assert sync.per_block == rdeltas
    assert [int(p) for p in st.panel_states()] == rs.panel_states()
    for got, want in zip(st.block_records(), rs.block_records()):
        assert (got.c0, got.width, got.overlap) == want[:3]
        assert abs(got.carried_diag - want[4]) <= 1e-10 * max(1.0, abs(want[4]))
        if got.overlap:
            # carried = prefix coefficients of a column that is already orthogonal
            # to the prefix (O(ε) noise): compare on the column's own scale.
            assert np.max(np.abs(got.carried - want[3])) <= 1e-10 * max(1.0, abs(want[4]))
    k = st.filled() - 1
    assert rel(st.hessenberg(k), rs.hessenberg(k)) < 1e-9


def test_two_stage_sync_counts_overlap_feeding(kb, ctx, ref):
    # TwoStageSyncCounts intent: 12 preprocess + 1 finalize = 13 per cycle.
    grid, m, s = 40, 60, 5
    a = ref.laplace2d(grid, grid)
    n = a.n
    op = kb.Laplace2D(grid, grid)
    b = ref.spmv(a, np.ones(n))
    st = kb.BasisStore(n, m, s, m)
    sync = kb.SyncCounter()
    st.mpk(op, b / np.linalg.norm(b), 0, s)
    for j in range(m // s):
        if j:
            st.mpk(op, None, st.filled() - 1, s)
        o = st.append_inplace(s + 1, j != 0, kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, m), sync)
        assert not o.breakdown and sync.per_block[-1] == 1
    assert st.big_panel_full()
    st.finalize_big_panel(sync)
    assert sync.per_big_panel[-1] == 1
    assert sync.reduces == 13
    assert ref.ortho_error(st.all()) < 1e-12
    assert all(p == kb.PanelState.FINAL for p in st.panel_states())


def test_two_stage_equals_pip2_when_big_panel_is_panel(kb, ctx, ref):
    # TwoStageEqualsPip2WhenBigPanelIsPanel intent (tests/test_block_ortho.cpp:271-295), MPK feeding.
    grid, m, s = 20, 20, 5
    a = ref.laplace2d(grid, grid)
    n = a.n
    b = ref.spmv(a, np.ones(n))
    v1 = b / np.linalg.norm(b)
    p2 = kb.BasisStore(n, m, s, s)
    ts = kb.BasisStore(n, m, s, s)
    s1, s2 = kb.SyncCounter(), kb.SyncCounter()
    for j in range(m // s):
        blk = ref.mpk(a, v1 if j == 0 else p2.column(p2.filled() - 1), s)
        assert not p2.append_block(blk, j != 0, kb.OrthoScheme(kb.OrthoKind.BCGS_PIP2, 0), s1).breakdown
        assert not ts.preprocess_block(blk, j != 0, s2).breakdown
        ts.finalize_big_panel(s2)
    assert p2.filled() == ts.filled()
    assert np.max(np.abs(p2.all() - ts.all())) <= 1e-12
    assert np.max(np.abs(np.triu(p2.coefficients()) - np.triu(ts.coefficients()))) <= 1e-12
    assert s1.reduces == s2.reduces


def test_rank_collapse_truncates_with_seam(kb, ctx, rng):
    # BasisStore.RankCollapseTruncatesWithSeam (tests/test_block_ortho.cpp:382-406)
    n = 50
    v = np.zeros((n, 3), order="F")
    v[:, 0] = rng.standard_normal(n)
    v[:, 0] /= np.linalg.norm(v[:, 0])
    v[:, 1] = v[:, 0]
    v[:, 2] = v[:, 0]
    st = kb.BasisStore(n, 9, 3, 9)
    sync = kb.SyncCounter()
    oc = st.append_block(v, False, kb.OrthoScheme(kb.OrthoKind.BCGS_PIP2, 0), sync)
    assert oc.truncated and not oc.breakdown
    assert oc.committed == 1 and oc.pivot == 2
    assert st.has_seam_column()
    r = st.coefficients()
    assert abs(r[0, 1] - 1.0) <= 1e-12
    assert r[1, 1] == 0.0


def test_states_track_two_stage_lifecycle(kb, ctx, ref):
    # StatesTrackTwoStageLifecycle (tests/test_block_ortho.cpp:408-421)
    n, m, s, shat = 2000, 20, 5, 10
    glued = ref.gen_glued(n, m // s, s, 1e3, 1.0, 0.1, 23)
    st = kb.BasisStore(n, m, s, shat)
    sync = kb.SyncCounter()
    st.preprocess_block(glued[:, 0:s], False, sync)
    assert st.panel_states()[-1] == kb.PanelState.PREPROCESSED
    assert st.finalized_count() == 0 and st.filled() > 0
    st.preprocess_block(glued[:, s:2 * s], False, sync)
    st.finalize_big_panel(sync)
    assert st.finalized_count() == st.filled()
    assert all(p == kb.PanelState.FINAL for p in st.panel_states())


def test_store_config_errors(kb, ctx):
    with pytest.raises(kb.DimensionMismatch):
        kb.BasisStore(10, 12, 5, 0)  # s ∤ m
    with pytest.raises(kb.DimensionMismatch):
        kb.BasisStore(10, 12, 3, 4)  # s ∤ ŝ
    st = kb.BasisStore(10, 6, 3, 6)
    with pytest.raises(kb.DimensionMismatch):
        st.append_block(np.ones((10, 8)), False, kb.OrthoScheme(), kb.SyncCounter())  # capacity


@pytest.mark.parametrize("grid,kind,shat", [(64, 2, 0), (64, 3, 60), (100, 3, 20), (128, 3, 60), (128, 2, 0),
                                            (512, 2, 0), (512, 3, 60)])  # 512²: BASELINE configs[0]
def test_orthogonality_error_protocol(kb, ctx, ref, grid, kind, shat):
    """on the same MPK-fed blocks (one full m = 60 cycle),
    ‖I − QᵀQ‖₂ of the device store is ≤ max(1e-12, 10× the reference
    store's) and within 1e-10 absolute of it (ortho_error, spectral.hpp:104)."""
    m, s = 60, 5
    a = ref.laplace2d(grid, grid)
    n = a.n
    b = ref.spmv(a, np.ones(n))
    v1 = b / np.linalg.norm(b)
    eff = shat if shat else m
    st = kb.BasisStore(n, m, s, eff)
    rs = ref.Store(n, m, s, eff)
    sync = kb.SyncCounter()
    for j in range(m // s):
        blk = ref.mpk(a, v1 if j == 0 else rs.column(rs.info().filled - 1), s)
        if kind == 3:
            assert not st.preprocess_block(blk, j != 0, sync).breakdown
            rs.preprocess_block(blk, j != 0)
            if rs.info().big_panel_full or j + 1 == m // s:
                st.finalize_big_panel(sync)
                rs.finalize_big_panel()
        else:
            assert not st.append_block(blk, j != 0, kb.OrthoScheme(kb.OrthoKind(kind), 0), sync).breakdown
            rs.append_block(blk, j != 0, kind)
    e_gpu, e_cpu = ref.ortho_error(st.all()), ref.ortho_error(rs.all())
    assert e_gpu <= max(1e-12, 10.0 * e_cpu), (e_gpu, e_cpu)
    assert abs(e_gpu - e_cpu) <= 1e-10
