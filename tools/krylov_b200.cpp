// krylov_b200 — command-line drop-in for the reference CLI's `solve`
// subcommand (tools/krylov_main.cpp:126-150, 220-241): same flags, same
// report keys (harness.hpp:379-400 solve_report_json), same residual-history
// CSV (harness.hpp:402-410) and the same stderr summary line — but the solve
// runs on the B200 through include/krylov_b200/krylov.hpp.
//
//   krylov_b200 solve (--matrix A.mtx | --grid N [--stencil 5|9] | --grid3d N)
//                     [--scheme standard|bcgs2-cholqr2|bcgs-pip2|two-stage]
//                     [--m 60] [--s 5] [--shat 0] [--tol 1e-6] [--max-iters 500000]
//                     [--equilibrate] [--jacobi] --out report.json [--history hist.csv]
//
// Host-side input handling (Matrix Market reader, equilibrate, triplets) is
// the drop-in API's include/krylov_b200/io.hpp (the reference's
// matrix_market.hpp:18-76 and csr_matrix.hpp:42-103 interfaces).  --jacobi (B200 addition, BASELINE configs[4])
// row-scales A by its diagonal before the solve.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "krylov_b200/io.hpp"
#include "krylov_b200/krylov.hpp"

using namespace krylov_b200;

namespace {

struct Args {
    std::string matrix, scheme = "bcgs-pip2", out, history;
    index_t grid = 0, grid3d = 0;
    int stencil = 5;
    SolverConfig cfg;
    bool equilibrate = false, jacobi = false;
};

[[noreturn]] void usage(const std::string& why) {
    throw std::runtime_error(why + "\nusage: krylov_b200 solve (--matrix F | --grid N [--stencil 5|9] | --grid3d N) "
                                   "[--scheme S] [--m M] [--s S] [--shat H] [--tol T] [--max-iters K] "
                                   "[--equilibrate] [--jacobi] --out F [--history F]");
}

Args parse(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "solve") usage("a subcommand is required (only `solve` is on the B200 path)");
    Args a;
    for (int i = 2; i < argc; ++i) {
        const std::string k = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage("missing value for " + k);
            return argv[++i];
        };
        if (k == "--matrix") a.matrix = val();
        else if (k == "--grid") a.grid = std::stoull(val());
        else if (k == "--grid3d") a.grid3d = std::stoull(val());
        else if (k == "--stencil") a.stencil = std::stoi(val());
        else if (k == "--scheme") a.scheme = val();
        else if (k == "--m") a.cfg.restart_len = std::stoull(val());
        else if (k == "--s") a.cfg.step = std::stoull(val());
        else if (k == "--shat") a.cfg.big_step = std::stoull(val());
        else if (k == "--tol") a.cfg.rel_tol = std::stod(val());
        else if (k == "--max-iters") a.cfg.max_iters = std::stoull(val());
        else if (k == "--equilibrate") a.equilibrate = true;
        else if (k == "--jacobi") a.jacobi = true;
        else if (k == "--out") a.out = val();
        else if (k == "--history") a.history = val();
        else usage("unknown option " + k);
    }
    if (a.out.empty()) usage("--out is required");
    if (a.stencil != 5 && a.stencil != 9) usage("--stencil must be 5 or 9");
    static const char* schemes[] = {"standard", "bcgs2-hhqr", "bcgs2-cholqr2", "bcgs-pip2", "two-stage"};
    if (std::find(std::begin(schemes), std::end(schemes), a.scheme) == std::end(schemes))
        usage("unknown scheme '" + a.scheme + "'");
    return a;
}

CsrMatrix read_matrix_market(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open matrix file " + path);
    return krylov_b200::read_matrix_market(in);
}

CsrMatrix laplace2d_csr(index_t nx, index_t ny, int stencil) {  // matgen.hpp:134-164
    std::vector<std::tuple<index_t, index_t, double>> t;
    const double diag = stencil == 5 ? 4.0 : 8.0 / 3.0, off = stencil == 5 ? -1.0 : -1.0 / 3.0;
    for (index_t iy = 0; iy < ny; ++iy)
        for (index_t ix = 0; ix < nx; ++ix) {
            const index_t row = iy * nx + ix;
            t.emplace_back(row, row, diag);
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if ((dx == 0 && dy == 0) || (stencil == 5 && dx != 0 && dy != 0)) continue;
                    const long long jx = static_cast<long long>(ix) + dx, jy = static_cast<long long>(iy) + dy;
                    if (jx < 0 || jy < 0 || jx >= static_cast<long long>(nx) || jy >= static_cast<long long>(ny)) continue;
                    t.emplace_back(row, static_cast<index_t>(jy) * nx + static_cast<index_t>(jx), off);
                }
        }
    return CsrMatrix::from_triplets(nx * ny, std::move(t));
}

void jacobi_scale(CsrMatrix& a) {  // left diagonal scaling D⁻¹A
    for (index_t i = 0; i < a.n; ++i) {
        double d = 0.0;
        for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
            if (a.col_idx[k] == i) d = a.vals[k];
        if (d == 0.0) throw std::runtime_error("jacobi: zero diagonal in row " + std::to_string(i));
        for (index_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) a.vals[k] /= d;
    }
}

std::string num(double v) {  // shortest round-trip decimal
    if (std::isinf(v)) return v > 0 ? "Infinity" : "-Infinity";
    if (std::isnan(v)) return "NaN";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

std::string sci(double v) {  // harness.hpp fmt_sci
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.16e", v);
    return buf;
}

const char* status_name(SolveStatus s) {
    switch (s) {
        case SolveStatus::Converged: return "converged";
        case SolveStatus::MaxIters: return "max_iters";
        case SolveStatus::OrthoBreakdown: return "ortho_breakdown";
        case SolveStatus::Stagnation: return "stagnation";
    }
    return "?";
}

OrthoKind parse_kind(const std::string& s) {
    if (s == "bcgs2-hhqr") return OrthoKind::Bcgs2Hhqr;
    if (s == "bcgs2-cholqr2") return OrthoKind::Bcgs2Cholqr2;
    if (s == "two-stage") return OrthoKind::TwoStage;
    return OrthoKind::BcgsPip2;
}

int run(int argc, char** argv) {
    Args a = parse(argc, argv);
    const bool matrix_free = a.matrix.empty() && !a.equilibrate && !a.jacobi && (a.grid3d > 0 || a.stencil == 5);
    index_t n = 0;
    std::unique_ptr<Operator> op;
    if (matrix_free) {
        if (a.grid3d > 0) {
            op = std::make_unique<Operator>(Operator::laplace3d(a.grid3d, a.grid3d, a.grid3d));
        } else {
            if (a.grid == 0) throw std::runtime_error("either --matrix or --grid is required");
            op = std::make_unique<Operator>(Operator::laplace2d(a.grid, a.grid));
        }
    } else {
        CsrMatrix m;
        if (!a.matrix.empty()) m = read_matrix_market(a.matrix);
        else if (a.grid3d > 0) throw std::runtime_error("--grid3d with --equilibrate/--jacobi: use a .mtx file");
        else if (a.grid > 0) m = laplace2d_csr(a.grid, a.grid, a.stencil);
        else throw std::runtime_error("either --matrix or --grid is required");
        if (a.equilibrate) m = krylov_b200::equilibrate(m);
        if (a.jacobi) jacobi_scale(m);
        op = std::make_unique<Operator>(Operator::csr(m));
    }
    n = op->rows();
    std::vector<double> ones(n, 1.0);
    const std::vector<double> b = spmv(*op, ones);  // gen_rhs_ones (matgen.hpp:190-193)
    SolveReport rep;
    if (a.scheme == "standard") {
        rep = standard_gmres(*op, b, {}, a.cfg);
    } else {
        a.cfg.scheme = OrthoScheme{parse_kind(a.scheme), a.cfg.effective_big_step()};
        rep = sstep_gmres(*op, b, {}, a.cfg);
    }
    // solve_report_json (harness.hpp:379-400); keys in nlohmann's sorted order.
    std::map<std::string, std::string> j;
    j["scheme"] = "\"" + a.scheme + "\"";
    j["n"] = std::to_string(n);
    j["m"] = std::to_string(a.cfg.restart_len);
    j["s"] = std::to_string(a.cfg.step);
    j["shat"] = std::to_string(a.cfg.effective_big_step());
    j["rel_tol"] = num(a.cfg.rel_tol);
    j["status"] = std::string("\"") + status_name(rep.status) + "\"";
    j["iterations"] = std::to_string(rep.iterations);
    j["restarts"] = std::to_string(rep.restarts);
    j["initial_residual"] = num(rep.initial_residual);
    j["final_relative_residual"] = num(rep.final_relative_residual);
    j["breakdown"] = rep.breakdown ? "true" : "false";
    j["breakdown_kappa"] = num(rep.breakdown_kappa);
    j["total_reduces"] = std::to_string(rep.sync.reduces);
    j["reduces_per_iteration"] = num(rep.reduces_per_iteration);
    j["wall_seconds"] = num(rep.wall_seconds);
    std::string cyc = "[";
    for (size_t i = 0; i < rep.cycle_residuals.size(); ++i)
        cyc += (i ? ",\n    " : "\n    ") + num(rep.cycle_residuals[i]);
    cyc += rep.cycle_residuals.empty() ? "]" : "\n  ]";
    j["cycle_residuals"] = cyc;
    {
        std::ofstream f(a.out);
        if (!f) throw std::runtime_error("cannot open output file " + a.out);
        f << "{\n";
        size_t k = 0;
        for (const auto& [key, v] : j) f << "  \"" << key << "\": " << v << (++k < j.size() ? ",\n" : "\n");
        f << "}\n";
    }
    if (!a.history.empty()) {  // write_residual_history_csv (harness.hpp:402-410)
        std::ofstream f(a.history);
        if (!f) throw std::runtime_error("cannot open output file " + a.history);
        f << "scheme,m,s,shat,rel_tol,cycle,relative_residual\n";
        for (size_t c = 0; c < rep.cycle_residuals.size(); ++c)
            f << a.scheme << ',' << a.cfg.restart_len << ',' << a.cfg.step << ',' << a.cfg.effective_big_step() << ','
              << sci(a.cfg.rel_tol) << ',' << (c + 1) << ',' << sci(rep.cycle_residuals[c]) << '\n';
    }
    std::cerr << "status=" << status_name(rep.status) << " iters=" << rep.iterations
              << " relres=" << sci(rep.final_relative_residual) << " reduces=" << rep.sync.reduces << '\n';
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
