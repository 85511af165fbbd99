// krylov_b200/io.hpp — host-side input utilities of the drop-in C++ API:
// building a CsrMatrix from triplets, Matrix Market read / write and
// equilibration (the reference's csr_matrix.hpp:42-103 and
// matrix_market.hpp:18-76 interfaces, with its exception types, types.hpp:43-70)
// and the Laplacian generators of matgen.hpp:134-195.
// They prepare operators on the host (only gen_rhs_ones' SpMV runs on the
// GPU).  Used by tools/krylov_b200 (the CLI) and by the reference's
// own tests/test_sparse_core.cpp compiled against this API
// (tests/cpp/refcompat).
#pragma once

#include <algorithm>
#include <charconv>
#include <cmath>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "krylov.hpp"

namespace krylov_b200 {

class UnsupportedFormat : public std::runtime_error {
public:
    explicit UnsupportedFormat(const std::string& what) : std::runtime_error("unsupported format: " + what) {}
};
class MalformedEntry : public std::runtime_error {
public:
    MalformedEntry(std::size_t line, const std::string& what)
        : std::runtime_error("malformed entry at line " + std::to_string(line) + ": " + what), line(line) {}
    std::size_t line;
};
class IndexOutOfRange : public std::runtime_error {
public:
    IndexOutOfRange(std::size_t line, const std::string& what)
        : std::runtime_error("index out of range at line " + std::to_string(line) + ": " + what), line(line) {}
    std::size_t line;
};
class ZeroRowOrColumn : public std::runtime_error {
public:
    ZeroRowOrColumn(bool is_row, index_t index)
        : std::runtime_error(std::string(is_row ? "row " : "column ") + std::to_string(index) +
                             " has no nonzero entries"),
          is_row(is_row), index(index) {}
    bool is_row;
    index_t index;
};

// Matrix Market: "matrix coordinate real general|symmetric", square; '%'
// comment lines; 1-based indices; symmetric entries mirrored; duplicates summed.
inline CsrMatrix read_matrix_market(std::istream& in) {
    std::string line;
    std::size_t lineno = 0;
    if (!std::getline(in, line)) throw UnsupportedFormat("empty stream");
    ++lineno;
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket" || object != "matrix") throw UnsupportedFormat("missing %%MatrixMarket matrix header");
    if (format != "coordinate") throw UnsupportedFormat("format '" + format + "'");
    if (field != "real") throw UnsupportedFormat("field '" + field + "'");
    if (symmetry != "general" && symmetry != "symmetric") throw UnsupportedFormat("symmetry '" + symmetry + "'");
    const bool sym = symmetry == "symmetric";
    long long rows = -1, cols = -1, nnz = -1;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream ss(line);
        if (!(ss >> rows >> cols >> nnz) || rows < 0 || cols < 0 || nnz < 0) throw MalformedEntry(lineno, "size line");
        break;
    }
    if (rows < 0) throw MalformedEntry(lineno, "missing size line");
    if (rows != cols) throw UnsupportedFormat("rectangular matrix (square operator required)");
    std::vector<std::tuple<index_t, index_t, double>> trip;
    trip.reserve(static_cast<std::size_t>(sym ? 2 * nnz : nnz));
    long long seen = 0;
    while (seen < nnz && std::getline(in, line)) {
        ++lineno;
        if (line.empty() || line[0] == '%') continue;
        std::istringstream ss(line);
        long long r = 0, c = 0;
        double v = 0.0;
        if (!(ss >> r >> c >> v)) throw MalformedEntry(lineno, "expected 'row col value'");
        if (r < 1 || c < 1 || r > rows || c > cols) throw IndexOutOfRange(lineno, std::to_string(r) + " " + std::to_string(c));
        trip.emplace_back(static_cast<index_t>(r - 1), static_cast<index_t>(c - 1), v);
        if (sym && r != c) trip.emplace_back(static_cast<index_t>(c - 1), static_cast<index_t>(r - 1), v);
        ++seen;
    }
    if (seen < nnz) throw MalformedEntry(lineno, "fewer entries than announced");
    return CsrMatrix::from_triplets(static_cast<index_t>(rows), std::move(trip));
}

// Shortest round-trip decimal of every value: a written matrix reads back
// bit for bit.
inline void write_matrix_market(std::ostream& out, const CsrMatrix& a) {
    out << "%%MatrixMarket matrix coordinate real general\n" << a.n << ' ' << a.n << ' ' << a.nnz() << '\n';
    char buf[64];
    for (index_t i = 0; i < a.n; ++i)
        for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const auto r = std::to_chars(buf, buf + sizeof buf, a.vals[k]);
            out << (i + 1) << ' ' << (a.col_idx[k] + 1) << ' ' << std::string(buf, r.ptr) << '\n';
        }
}

// Two-sided scaling to unit maxima: every column divided by its largest
// |entry|, then every row by its largest |entry| (so row maxima are exactly
// 1).  ZeroRowOrColumn on an empty column or row.
inline CsrMatrix equilibrate(const CsrMatrix& a) {
    CsrMatrix e = a;
    std::vector<double> cmax(a.n, 0.0);
    for (index_t k = 0; k < e.nnz(); ++k) cmax[e.col_idx[k]] = std::max(cmax[e.col_idx[k]], std::abs(e.vals[k]));
    for (index_t j = 0; j < e.n; ++j)
        if (cmax[j] == 0.0) throw ZeroRowOrColumn(false, j);
    for (index_t k = 0; k < e.nnz(); ++k) e.vals[k] /= cmax[e.col_idx[k]];
    for (index_t i = 0; i < e.n; ++i) {
        double rmax = 0.0;
        for (index_t k = e.row_ptr[i]; k < e.row_ptr[i + 1]; ++k) rmax = std::max(rmax, std::abs(e.vals[k]));
        if (rmax == 0.0) throw ZeroRowOrColumn(true, i);
        for (index_t k = e.row_ptr[i]; k < e.row_ptr[i + 1]; ++k) e.vals[k] /= rmax;
    }
    return e;
}

// Dirichlet Laplacians on a grid, row-major node order, as CsrMatrix
// (matgen.hpp:134-195): 5-point (diagonal 4, neighbours −1), 9-point
// (diagonal 8/3, all eight neighbours −1/3), 7-point 3-D (diagonal 6,
// neighbours −1).  Columns ascend within each row.  (The solver's own
// matrix-free operators are Operator::laplace2d / laplace3d.)
inline CsrMatrix gen_laplace2d(index_t nx, index_t ny, int stencil = 5) {
    if (nx < 2 || ny < 2) throw DimensionMismatch("gen_laplace2d needs dimensions >= 2");
    if (stencil != 5 && stencil != 9) throw std::invalid_argument("gen_laplace2d stencil must be 5 or 9");
    CsrMatrix a;
    a.n = nx * ny;
    a.row_ptr.assign(1, 0);
    a.col_idx.reserve(a.n * static_cast<index_t>(stencil));
    a.vals.reserve(a.n * static_cast<index_t>(stencil));
    const double centre = stencil == 5 ? 4.0 : 8.0 / 3.0, nb = stencil == 5 ? -1.0 : -1.0 / 3.0;
    for (index_t iy = 0; iy < ny; ++iy)
        for (index_t ix = 0; ix < nx; ++ix) {
            for (index_t jy = iy == 0 ? 0 : iy - 1; jy <= std::min(iy + 1, ny - 1); ++jy)
                for (index_t jx = ix == 0 ? 0 : ix - 1; jx <= std::min(ix + 1, nx - 1); ++jx) {
                    const bool centre_node = jx == ix && jy == iy;
                    if (stencil == 5 && jx != ix && jy != iy) continue;  // no diagonals
                    a.col_idx.push_back(jy * nx + jx);
                    a.vals.push_back(centre_node ? centre : nb);
                }
            a.row_ptr.push_back(a.col_idx.size());
        }
    return a;
}

inline CsrMatrix gen_laplace3d(index_t nx, index_t ny, index_t nz) {
    if (nx < 2 || ny < 2 || nz < 2) throw DimensionMismatch("gen_laplace3d needs dimensions >= 2");
    CsrMatrix a;
    a.n = nx * ny * nz;
    a.row_ptr.assign(1, 0);
    a.col_idx.reserve(a.n * 7);
    a.vals.reserve(a.n * 7);
    const index_t plane = nx * ny;
    for (index_t iz = 0; iz < nz; ++iz)
        for (index_t iy = 0; iy < ny; ++iy)
            for (index_t ix = 0; ix < nx; ++ix) {
                const index_t r = iz * plane + iy * nx + ix;
                auto put = [&](bool present, index_t c, double v) {
                    if (!present) return;
                    a.col_idx.push_back(c);
                    a.vals.push_back(v);
                };
                put(iz > 0, r - plane, -1.0);
                put(iy > 0, r - nx, -1.0);
                put(ix > 0, r - 1, -1.0);
                put(true, r, 6.0);
                put(ix + 1 < nx, r + 1, -1.0);
                put(iy + 1 < ny, r + nx, -1.0);
                put(iz + 1 < nz, r + plane, -1.0);
                a.row_ptr.push_back(a.col_idx.size());
            }
    return a;
}

// b = A·1 (matgen.hpp:190), the SpMV on the GPU.
inline std::vector<double> gen_rhs_ones(const CsrMatrix& a) { return spmv(a, std::vector<double>(a.n, 1.0)); }

}  // namespace krylov_b200
