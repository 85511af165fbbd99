// Synthetic nonsymmetric random sparse rows — the BASELINE configs[4]
// workload.  The reference has no such generator; this one
// is built on the reference's SplitMix64 (rng.hpp:19-42) so the matrix is a
// function of (seed, n, per_row, diag_factor) alone, independent of the
// rank layout and of the thread count: output t of SplitMix64(Seed{seed})
// is mix(seed + (t+1)·γ), computed directly from t.
//
// Row i (global), k = per_row − 1 off-diagonals, consumes outputs
// [2k·i, 2k·i + 2k):
//   gap_j = 1 + (u_{2ki+j} >> 11) mod span,  span = max(1, (n−1)/k)
//   column_j = (i + gap_0 + … + gap_j) mod n     (distinct, never i)
//   val_j = 2·((u_{2ki+k+j} >> 11)·2⁻⁵³) − 1      (uniform in [−1, 1))
//   a_ii = 1 + diag_factor·Σ_j |val_j|             (j ascending)
// stored in ascending column order.  With jacobi, every entry is divided by
// a_ii (the left Jacobi scaling D⁻¹A the reference would be given).
// oracle/randsparse.py restates this in numpy (tests compare bit for bit).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "kb_common.hpp"

namespace kb {

namespace {
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

inline uint64_t splitmix_at(uint64_t seed, uint64_t t) {
    uint64_t z = seed + (t + 1) * kGamma;  // state after t+1 increments (rng.hpp:25)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void gen_rows(i64 n, i64 r0, i64 r1, i64 row_begin, i64 per_row, uint64_t seed, double diag_factor, bool jacobi,
              int64_t* col, double* vals) {
    const i64 k = per_row - 1;
    const uint64_t span = static_cast<uint64_t>(std::max<i64>(1, k > 0 ? (n - 1) / k : 1));
    std::vector<i64> c(static_cast<size_t>(k));
    std::vector<double> v(static_cast<size_t>(k));
    for (i64 r = r0; r < r1; ++r) {
        const i64 i = row_begin + r;
        const uint64_t base = static_cast<uint64_t>(i) * static_cast<uint64_t>(2 * k);
        i64 cum = 0, nw = 0;
        double acc = 0.0;
        for (i64 j = 0; j < k; ++j) {
            cum += static_cast<i64>((splitmix_at(seed, base + j) >> 11) % span + 1);
            i64 cj = i + cum;
            if (cj >= n) {
                cj -= n;
                ++nw;
            }
            c[j] = cj;
            v[j] = static_cast<double>(splitmix_at(seed, base + k + j) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
            acc = acc + std::fabs(v[j]);
        }
        const double d = 1.0 + diag_factor * acc;
        int64_t* co = col + r * per_row;
        double* vo = vals + r * per_row;
        // cum ascends: the nw wrapped entries (columns < i) are the last in j
        // order; ascending row = wrapped, diagonal, the rest.
        i64 o = 0;
        for (i64 j = k - nw; j < k; ++j, ++o) {
            co[o] = c[j];
            vo[o] = jacobi ? v[j] / d : v[j];
        }
        co[o] = i;
        vo[o] = jacobi ? d / d : d;
        ++o;
        for (i64 j = 0; j < k - nw; ++j, ++o) {
            co[o] = c[j];
            vo[o] = jacobi ? v[j] / d : v[j];
        }
    }
}
}  // namespace

void gen_random_sparse(i64 n_global, i64 row_begin, i64 n_local, i64 per_row, uint64_t seed, double diag_factor,
                       bool jacobi, int64_t* row_ptr, int64_t* col, double* vals) {
    if (n_global < 1 || per_row < 1 || per_row > n_global || row_begin < 0 || n_local < 0 ||
        row_begin + n_local > n_global)
        fail(KRY_DIMENSION_MISMATCH, "dimension mismatch: random sparse shape");
    if (!(diag_factor >= 0.0)) fail(KRY_INVALID_ARGUMENT, "diag_factor must be >= 0");
    for (i64 r = 0; r <= n_local; ++r) row_ptr[r] = r * per_row;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const i64 nt = std::max<i64>(1, std::min<i64>(hw, n_local / 65536));
    std::vector<std::thread> th;
    for (i64 t = 0; t < nt; ++t) {
        const i64 a = t * n_local / nt, b = (t + 1) * n_local / nt;
        th.emplace_back(gen_rows, n_global, a, b, row_begin, per_row, seed, diag_factor, jacobi, col, vals);
    }
    for (auto& x : th) x.join();
}

}  // namespace kb
