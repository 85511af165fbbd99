// s-step GMRES restart loop (gmres_impl, gmres.hpp:198-390) over the device
// basis store.  Control flow, convergence checks, update acceptance and the
// SolveReport bookkeeping follow the reference line for line; the vectors
// (x, r, b, the basis) stay in HBM and only scalars (norms, the Gram, R, y)
// cross to the host.
#pragma once

#include <memory>
#include <string>
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

// Device workspace of one solve (basis store + four vectors), kept by the
// C-ABI context so that repeated solves of the same shape reuse HBM instead
// of re-allocating (and re-zeroing) an n×(m+1) basis per call.
// Recorded launch sequences of the speculative queues (one per cycle
// position), replayed as CUDA graphs: a 512² cycle is ~70 (two-stage) to
// ~110 (PIP2) launches whose host-side cost would otherwise bound it.
struct GraphCache {
    struct Entry {
        uint64_t key;
        uint64_t gen;
        cudaGraphExec_t exec;
    };
    std::vector<Entry> entries;
    std::string sig;  // operator / scheme / switches the recordings belong to
    void clear() {
        for (auto& e : entries) cudaGraphExecDestroy(e.exec);
        entries.clear();
    }
    ~GraphCache() { clear(); }
};

struct Workspace {
    i64 n = -1, m = -1, s = -1, shat = -1;
    GraphCache graphs;
    std::unique_ptr<Store> store;
    DevBuf x, xn, r, rn;
    DevBuf bj;  // D⁻¹b of a Jacobi-preconditioned operator
    // host-output path: the solution update streams to the host while it is
    // computed (side stream, one event per row chunk)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t chunk_ev[8] = {}, copy_done = nullptr;
    Workspace() = default;
    Workspace(const Workspace&) = delete;
    Workspace& operator=(const Workspace&) = delete;
    ~Workspace();
};

// d_b: n_local rhs (device); d_x0 may be null (or alias d_x_out); d_x_out may
// be null.  h_x_out (host; pinned for the overlap to happen) receives the
// solution instead of d_x_out: every applied solution update is copied to
// it chunk by chunk as the update kernel produces it, so the final download
// overlaps the update and the acceptance check (re-downloaded if rejected).
Report gmres(Ctx& ctx, Operator& op, const double* d_b, const double* d_x0, const kry_solver_config& cfg,
             bool standard_mode, double* d_x_out, Workspace* ws = nullptr, double* h_x_out = nullptr);

void validate_config(const kry_solver_config& cfg);

}  // namespace kb
