"""TEST INFRASTRUCTURE — numpy restatement of the BASELINE configs[4] workload
generator (`kry_gen_random_sparse`, paper_2402_15033_b200/csrc/kb_matgen.cpp).

Used only as the checker: tests compare the library's generator with this
bit for bit, and tests/golden/make_golden.py builds the reference-side
(pre-scaled) matrix from it.  The reference has no random-sparse generator;
SURVEY §8(d) asks for one built on its SplitMix64
(/root/reference/proj/include/krylov/rng.hpp:19-42), which is restated here:
the t-th output (t = 0, 1, ...) of SplitMix64(Seed{seed}) is
mix(seed + (t+1)·0x9E3779B97F4A7C15), so any output can be computed directly
from its index.

Row i (global) with k = per_row − 1 off-diagonal entries consumes outputs
t = 2k·i … 2k·i + 2k − 1:
  * gap_j = 1 + (u_{2ki+j} >> 11) mod span, span = max(1, (n−1) // k);
    off-diagonal column c_j = (i + gap_0 + … + gap_j) mod n (distinct, ≠ i);
  * val_j = 2·((u_{2ki+k+j} >> 11)·2⁻⁵³) − 1  (uniform in [−1, 1));
  * diagonal a_ii = 1 + diag_factor·(|val_0| + … + |val_{k−1}|) (summed in j order);
stored in ascending column order (the wrapped columns < i, the diagonal,
then the columns > i).  Jacobi: a_ij / a_ii row by row.
"""
import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, t):
    """Outputs t (uint64 array of indices) of SplitMix64(Seed{seed}) — rng.hpp:24-30."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (t.astype(np.uint64) + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def random_sparse(n_global, row_begin, n_local, per_row, seed=1, diag_factor=0.25, jacobi=False):
    """CSR (int64 row_ptr from 0, int64 global columns, fp64 values) of rows
    [row_begin, row_begin + n_local)."""
    k = per_row - 1
    if per_row < 1 or k > n_global - 1:
        raise ValueError("per_row must be in [1, n_global]")
    rows = np.arange(row_begin, row_begin + n_local, dtype=np.int64)
    nnz = n_local * per_row
    rp = np.arange(n_local + 1, dtype=np.int64) * per_row
    if k == 0:
        return rp, rows.copy(), np.ones(n_local)
    span = max(1, (n_global - 1) // k)
    base = (rows * (2 * k))[:, None]
    j = np.arange(k, dtype=np.int64)[None, :]
    ug = splitmix64(seed, base + j)
    uv = splitmix64(seed, base + k + j)
    gaps = (ug >> np.uint64(11)) % np.uint64(span) + np.uint64(1)
    cum = np.cumsum(gaps.astype(np.int64), axis=1)
    cols = (rows[:, None] + cum) % n_global
    vals = (uv >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
    acc = np.zeros(n_local)
    for jj in range(k):  # sequential sum in j order
        acc = acc + np.abs(vals[:, jj])
    diag = 1.0 + diag_factor * acc
    if jacobi:
        vals = vals / diag[:, None]
        dval = diag / diag
    else:
        dval = diag
    # cum ascends, so the wrapped entries (i + cum ≥ n, columns < i) are the
    # last nw in j order: sorted row = wrapped (j ≥ k − nw), diagonal, the rest.
    wrapped = cols < rows[:, None]
    nw = wrapped.sum(axis=1)[:, None]
    pos = np.where(wrapped, j - (k - nw), nw + 1 + j)
    col = np.empty((n_local, per_row), dtype=np.int64)
    val = np.empty((n_local, per_row))
    r_idx = np.broadcast_to(np.arange(n_local)[:, None], (n_local, k))
    col[r_idx, pos] = cols
    val[r_idx, pos] = vals
    col[np.arange(n_local), nw[:, 0]] = rows
    val[np.arange(n_local), nw[:, 0]] = dval
    return rp, col.reshape(-1), val.reshape(-1)
