"""The synthetic workloads bench.py generates (BASELINE.json configs) are
valid reference inputs: CSR contract, determinism, diagonal dominance."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_random_sparse_rows_contract():
    from bench import random_sparse_rows
    rp, ci, vv = random_sparse_rows(5000, 0, 5000, 30, chunk=1024)
    n = 5000
    assert rp[0] == 0 and rp[-1] == len(ci) == len(vv) == 30 * n
    for i in range(0, n, 97):
        c, v = ci[rp[i]:rp[i + 1]], vv[rp[i]:rp[i + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < n  # strictly increasing, in range
        assert v[c == i][0] == 1.0  # Jacobi-scaled diagonal
        assert np.abs(v[c != i]).sum() < 1.0  # strictly diagonally dominant
    rp2, ci2, vv2 = random_sparse_rows(5000, 0, 5000, 30, chunk=1024)
    assert np.array_equal(ci, ci2) and np.array_equal(vv, vv2)  # deterministic


def test_random_sparse_solves_with_the_reference(ref):
    from bench import random_sparse_rows
    rp, ci, vv = random_sparse_rows(3000, 0, 3000, 30)
    a = ref.Csr(3000, rp, ci, vv)
    b = ref.spmv(a, np.ones(3000))
    rep = ref.solve(a, b, None, ref.make_config(kind=3))
    assert rep.status == 0 and rep.iterations <= 120
