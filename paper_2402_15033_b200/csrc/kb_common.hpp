// Shared internals of the B200 hot path: error type (maps onto the C ABI
// status codes, which map onto the reference's exception types), CUDA/NCCL
// checks, and the per-context launch counter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/krylov_b200.h"

namespace kb {

using i64 = int64_t;

// One exception type inside the library; the C ABI layer converts it to a
// status code (kb_capi.cpp).  `aux` carries the 1-based pivot for
// KRY_NOT_POSITIVE_DEFINITE and the column for KRY_SINGULAR_R.
struct Error : std::runtime_error {
    int code;
    i64 aux;
    Error(int c, const std::string& msg, i64 a = 0) : std::runtime_error(msg), code(c), aux(a) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg, i64 aux = 0) {
    throw Error(code, msg, aux);
}

inline void dim_check(bool ok, const char* what) {
    if (!ok) fail(KRY_DIMENSION_MISMATCH, std::string("dimension mismatch: ") + what);
}

#define KB_CUDA(expr)                                                                     \
    do {                                                                                  \
        cudaError_t kb_e_ = (expr);                                                       \
        if (kb_e_ != cudaSuccess)                                                         \
            ::kb::fail(KRY_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(kb_e_)); \
    } while (0)

// After every kernel launch: surface launch-configuration errors at once.
#define KB_LAUNCHED()                                                                     \
    do {                                                                                  \
        cudaError_t kb_e_ = cudaGetLastError();                                           \
        if (kb_e_ != cudaSuccess)                                                         \
            ::kb::fail(KRY_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(kb_e_)); \
    } while (0)

// CUDA-graph replay of a recorded launch sequence (kb_gmres.cpp): while the
// host re-runs a sequence whose kernels a cached graph already holds, the
// launch wrappers (launch_pdl) skip the launch; the host bookkeeping and the
// launch counters still run.
inline bool& launches_suppressed() {
    static thread_local bool on = false;
    return on;
}
// Bumped whenever a device buffer is (re)allocated: a recorded graph holds
// raw pointers, so it is replayed only while the generation is unchanged.
inline uint64_t& devbuf_generation() {
    static uint64_t g = 0;
    return g;
}

inline i64 ceil_div(i64 a, i64 b) { return (a + b - 1) / b; }
inline i64 round_up(i64 a, i64 b) { return ceil_div(a, b) * b; }

// Device leading dimension for n rows: even (16-byte column alignment for
// TMA) and a multiple of 32 rows (256-byte aligned columns).
inline i64 device_ld(i64 n) { return round_up(n < 1 ? 1 : n, 32); }

}  // namespace kb
