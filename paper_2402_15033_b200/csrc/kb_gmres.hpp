// s-step GMRES restart loop (gmres_impl, gmres.hpp:198-390) over the device
// basis store.  Control flow, convergence checks, update acceptance and the
// SolveReport bookkeeping follow the reference line for line; the vectors
// (x, r, b, the basis) stay in HBM and only scalars (norms, the Gram, R, y)
// cross to the host.
#pragma once

#include <vector>

#include "kb_operator.hpp"
#include "kb_store.hpp"

namespace kb {

struct Report {
    int status = KRY_STATUS_MAX_ITERS;
    i64 iterations = 0;
    i64 restarts = 0;
    double initial_residual = 0.0;
    double final_relative_residual = 0.0;
    std::vector<double> cycle_residuals;
    bool breakdown = false;
    double breakdown_kappa = 0.0;
    Sync sync;
    double reduces_per_iteration = 0.0;
    double wall_seconds = 0.0;
    // telemetry
    double mpk_bytes = 0.0, ortho_bytes = 0.0;
};

// d_b: n_local rhs (device); d_x0 may be null; d_x_out (n_local) may be null.
Report gmres(Ctx& ctx, Operator& op, const double* d_b, const double* d_x0, const kry_solver_config& cfg,
             bool standard_mode, double* d_x_out);

void validate_config(const kry_solver_config& cfg);

}  // namespace kb
