"""Pin the C restatement (oracle/krylov_oracle.c) before trusting it:
bit-exact against the golden fixtures generated from the reference
(tests/golden/) and against the live reference (oracle/_ref) on the same
inputs — SpMV, generators, MPK, Gram, Cholesky, BCGS-PIP/PIP2, the basis
store state machine (R, Q, records) and whole solves (status, counts,
SyncCounter deltas and every cycle residual).  CPU only."""
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "solver_golden.json")))
KG = np.load(os.path.join(ROOT, "tests", "golden", "kernels_golden.npz"))


@pytest.fixture(scope="module")
def orc():
    from oracle import orc as O
    if not O.available():
        pytest.fail("oracle/_lib/libkrylov_oracle.so missing: make -C oracle oracle")
    return O


def test_generators_match_reference(orc, ref):
    for nx, ny in [(2, 2), (9, 7), (30, 17)]:
        a, b = orc.laplace2d(nx, ny), ref.laplace2d(nx, ny)
        np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
        np.testing.assert_array_equal(a.col_idx, b.col_idx)
        np.testing.assert_array_equal(a.vals, b.vals)
    for d in [(2, 2, 2), (5, 4, 3), (9, 8, 7)]:
        a, b = orc.laplace3d(*d), ref.laplace3d(*d)
        np.testing.assert_array_equal(a.col_idx, b.col_idx)
        np.testing.assert_array_equal(a.vals, b.vals)


def test_kernels_match_golden(orc):
    a2 = orc.laplace2d(9, 7)
    np.testing.assert_array_equal(orc.spmv(a2, KG["lap2d_9x7_x"]), KG["lap2d_9x7_y"])
    a3 = orc.laplace3d(5, 4, 3)
    np.testing.assert_array_equal(orc.spmv(a3, KG["lap3d_5x4x3_x"]), KG["lap3d_5x4x3_y"])
    np.testing.assert_array_equal(orc.mpk(a2, KG["mpk_start"], 5), KG["mpk_V"])
    np.testing.assert_array_equal(orc.gram(KG["gram_v"]), KG["gram_out"])
    r, piv = orc.try_cholesky(KG["chol_s"])
    np.testing.assert_array_equal(np.triu(r), np.triu(KG["chol_r"]))
    r, piv = orc.try_cholesky(KG["chol_bad_s"])
    assert piv == int(KG["chol_bad_pivot"][0])
    q, rc, rj, red = orc.bcgs_pip(KG["pip_q"], KG["pip_v"])
    np.testing.assert_array_equal(q, KG["pip_out_q"])
    np.testing.assert_array_equal(rc, KG["pip_out_rcol"])
    np.testing.assert_array_equal(np.triu(rj), np.triu(KG["pip_out_rjj"]))
    q, rc, rj, red = orc.bcgs_pip2(KG["pip_q"], KG["pip_v"])
    np.testing.assert_array_equal(q, KG["pip2_out_q"])
    np.testing.assert_array_equal(rc, KG["pip2_out_rcol"])
    assert red == 2


def test_store_sequence_matches_golden(orc):
    st = orc.Store(144, 12, 3, 12)
    for j, blk in enumerate(KG["store_blocks"]):
        st.preprocess_block(blk, j != 0)
    st.finalize_big_panel()
    np.testing.assert_array_equal(st.coefficients(), KG["store_R"])
    np.testing.assert_array_equal(st.all(), KG["store_Q"])
    np.testing.assert_array_equal(st.hessenberg(st.info().filled - 1), KG["store_H"])


@pytest.mark.parametrize("kind,shat", [(2, 0), (3, 60), (3, 20), (1, 0)])
def test_store_matches_live_reference(orc, ref, kind, shat):
    a = ref.laplace2d(20, 20)
    b = ref.spmv(a, np.ones(a.n))
    v1 = b / np.linalg.norm(b)
    eff = shat or 60
    so, sr = orc.Store(a.n, 60, 5, eff), ref.Store(a.n, 60, 5, eff)
    for j in range(12):
        blk = ref.mpk(a, v1 if j == 0 else sr.column(sr.info().filled - 1), 5)
        if kind == 3:
            (oo, do), (orr, dr) = so.preprocess_block(blk, j != 0), sr.preprocess_block(blk, j != 0)
            if sr.info().big_panel_full or j == 11:
                so.finalize_big_panel()
                sr.finalize_big_panel()
        else:
            (oo, do), (orr, dr) = so.append_block(blk, j != 0, kind), sr.append_block(blk, j != 0, kind)
        assert do == dr and oo.committed == orr.committed
    np.testing.assert_array_equal(so.coefficients(), sr.coefficients())
    np.testing.assert_array_equal(so.all(), sr.all())


def test_rank_collapse_truncation_matches_reference(orc, ref):
    rng = np.random.default_rng(22)
    v = np.zeros((50, 3), order="F")
    v[:, 0] = rng.standard_normal(50)
    v[:, 0] /= np.linalg.norm(v[:, 0])
    v[:, 1] = v[:, 0]
    v[:, 2] = v[:, 0]
    so, sr = orc.Store(50, 9, 3, 9), ref.Store(50, 9, 3, 9)
    (oo, do), (orr, dr) = so.append_block(v, False, 2), sr.append_block(v, False, 2)
    assert (oo.committed, oo.truncated, oo.breakdown, oo.pivot, do) == (
        orr.committed, orr.truncated, orr.breakdown, orr.pivot, dr)
    assert oo.kappa_estimate == orr.kappa_estimate
    np.testing.assert_array_equal(so.coefficients(), sr.coefficients())


@pytest.mark.parametrize("key", sorted(GOLDEN))
def test_solver_matches_golden_bitwise(orc, ref, key):
    g = GOLDEN[key]
    if g["operator"] == "random":  # configs[4] generator, host pre-scaled (the reference's input)
        import os
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
        from make_golden import random_jacobi_system
        a, b = random_jacobi_system(g["grid"])
    else:
        if g["grid"] >= 200 or (g["dims"] == 3 and g["grid"] > 32):
            pytest.skip("long CPU solve")
        a = orc.laplace2d(g["grid"], g["grid"]) if g["dims"] == 2 else orc.laplace3d(g["grid"], g["grid"], g["grid"])
        b = orc.spmv(a, np.ones(a.n))
    x0 = None if g["x0"] is None else np.full(a.n, g["x0"])
    cfg = ref.make_config(kind=g["kind"], big_step=g["shat"], shat=g["shat"], max_iters=g["max_iters"])
    rep = orc.solve(a, b, x0, cfg, standard=g["standard"])
    assert (rep.status, rep.iterations, rep.restarts, rep.reduces) == (g["status"], g["iterations"], g["restarts"],
                                                                       g["reduces"])
    assert [int(v) for v in rep.per_block] == g["per_block"]
    assert [int(v) for v in rep.per_big_panel] == g["per_big_panel"]
    assert rep.cycle_residuals == g["cycle_residuals"]  # bit-exact
    assert rep.final_relative_residual == g["final_relative_residual"]
