"""The BASELINE configs[4] workload generator (kry_gen_random_sparse, host
code, no device needed) against its numpy restatement (oracle/randsparse.py,
SplitMix64 of rng.hpp:19-42): bit for bit, the CSR contract of
csr_matrix.hpp:25-38, rank-layout independence, and that the reference
solves the Jacobi-scaled system with restarts (not in one cycle)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_splitmix64_matches_the_reference_sequence():
    # rng.hpp:24-30 run sequentially from Seed{1}, restated in pure Python
    from oracle import randsparse
    state, want = 1, []
    for _ in range(8):
        state = (state + 0x9E3779B97F4A7C15) % 2**64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % 2**64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % 2**64
        want.append(z ^ (z >> 31))
    got = randsparse.splitmix64(1, np.arange(8, dtype=np.uint64))
    assert [int(v) for v in got] == want


@pytest.mark.parametrize("n,rb,nl,per_row,jac", [(20000, 0, 20000, 30, False), (20000, 777, 5000, 30, True),
                                                 (50, 0, 50, 50, True), (7, 0, 7, 1, False), (1, 0, 1, 1, True),
                                                 (100000, 99000, 1000, 8, True), (3, 1, 2, 3, False)])
def test_generator_matches_numpy_restatement(kb, n, rb, nl, per_row, jac):
    from oracle import randsparse
    got = kb.gen_random_sparse(n, rb, nl, per_row, seed=1, diag_factor=0.15, jacobi=jac)
    want = randsparse.random_sparse(n, rb, nl, per_row, seed=1, diag_factor=0.15, jacobi=jac)
    for g, w in zip(got, want):
        assert g.dtype == w.dtype and np.array_equal(g, w)


def test_generator_csr_contract_and_layout_independence(kb):
    n = 30000
    rp, ci, vv = kb.gen_random_sparse(n, per_row=30)
    assert rp[0] == 0 and rp[-1] == len(ci) == len(vv) == 30 * n
    rows = np.repeat(np.arange(n), 30)
    c = ci.reshape(n, 30)
    assert np.all(np.diff(c, axis=1) > 0) and c.min() >= 0 and c.max() < n  # strictly ascending, in range
    assert np.count_nonzero(ci == rows) == n  # one diagonal entry per row
    d = vv[ci == rows]
    off = np.abs(vv.reshape(n, 30)).sum(axis=1) - d
    assert np.allclose(d, 1.0 + 0.15 * off) and np.all(d < off)  # not diagonally dominant
    # two "ranks" generate the same rows as one
    a = kb.gen_random_sparse(n, 0, n // 3, 30)
    b = kb.gen_random_sparse(n, n // 3, n - n // 3, 30)
    assert np.array_equal(np.concatenate([a[1], b[1]]), ci) and np.array_equal(np.concatenate([a[2], b[2]]), vv)
    # Jacobi: every entry divided by its row's diagonal, diagonal exactly 1
    _, cj, vj = kb.gen_random_sparse(n, per_row=30, jacobi=True)
    assert np.array_equal(cj, ci) and np.array_equal(vj, vv / np.repeat(d, 30)) and np.all(vj[ci == rows] == 1.0)


def test_generator_errors(kb):
    with pytest.raises(kb.DimensionMismatch):
        kb.gen_random_sparse(10, 0, 10, 11)
    with pytest.raises(kb.DimensionMismatch):
        kb.gen_random_sparse(10, 5, 6, 3)
    with pytest.raises(ValueError):  # std::invalid_argument
        kb.gen_random_sparse(10, 0, 10, 3, diag_factor=-1.0)


def test_random_sparse_restarts_with_the_reference(ref):
    # configs[4] must exercise restarts: GMRES(60) two-stage needs 5 of them
    # at n = 20,000 on the Jacobi-scaled system (tests/golden/make_golden.py)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import random_jacobi_system
    a, b = random_jacobi_system(20000)
    rep = ref.solve(a, b, None, ref.make_config(kind=3, big_step=60, shat=60))
    assert rep.status == 0 and rep.restarts >= 3
