// Execution context: one device, one non-blocking stream, an optional NCCL
// communicator (one process per GPU; rows partitioned across ranks), the
// scratch buffers of the hot path and the CUDA-event phase timers.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <vector>

#include "kb_common.hpp"
#include "nvtx3/nvToolsExt.h"

namespace kb {

// RAII device allocation.
struct DevBuf {
    double* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    // Grow to at least `b` bytes (contents not preserved).
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        void* q = nullptr;
        KB_CUDA(cudaMalloc(&q, b));
        p = static_cast<double*>(q);
        bytes = b;
        ++devbuf_generation();
    }
    template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

// RAII pinned host allocation.
struct HostBuf {
    double* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { if (p) cudaFreeHost(p); }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
        void* q = nullptr;
        KB_CUDA(cudaMallocHost(&q, b));
        p = static_cast<double*>(q);
        bytes = b;
    }
};

enum Phase { PH_MPK = 0, PH_ORTHO, PH_GRAM, PH_UPDATE, PH_RESTART, PH_FUSED, PH_COUNT };

struct Ctx {
    int device = 0;
    int nranks = 1;
    int rank = 0;
    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    bool timing = false;
    int64_t launches = 0;
    int64_t allreduces = 0;
    double gram_bytes = 0.0, update_bytes = 0.0;  // algorithmic, this rank
    int64_t gram_launches = 0, update_launches = 0;
    double fused_bytes = 0.0;  // K6: necessary HBM bytes (k_fused.cu), this rank
    int64_t fused_launches = 0;

    // scratch
    DevBuf partials;      // reduce_grid() doubles + scalars
    DevBuf gram_partials; // per-CTA Gram partials
    DevBuf gram_packed;   // packed Gram tiles (all prefix groups)
    DevBuf coef;          // update coefficients (all passes)
    HostBuf h_packed, h_coef, h_scalar;

    // phase timers
    std::array<double, PH_COUNT> seconds{};
    std::vector<cudaEvent_t> pool;
    struct Pending { int phase; cudaEvent_t a, b; };
    std::vector<Pending> pending;

    Ctx(int dev, int nr, int rk, const void* nccl_id);
    ~Ctx();

    void sync();
    // KRY_HOST_PROFILE=1: time spent blocked in sync() (printed by gmres()).
    bool host_profile = false;
    double sync_wait_s = 0.0;
    int64_t sync_count = 0;
    // Timer: begin() returns a token; end(token) closes it.
    cudaEvent_t begin_phase();
    void end_phase(int phase, cudaEvent_t start);
    void resolve_timers();  // after a stream sync: accumulate elapsed times
    void drain_timers();    // accumulate the phases that already finished (no wait)

    // Σ over ranks, in place on the device (no-op for one rank): the
    // one-shot peer-memory allreduce (k_peer.cu) when the context mapped its
    // peers (KRY_PEER_ALLREDUCE=1, opt-in), else ncclAllReduce.
    void allreduce_sum(double* d, size_t count);
    bool peer = false;
    DevBuf peer_data, peer_flags;         // this rank's receive area and flags
    std::vector<void*> peer_opened;       // peers' areas mapped through CUDA IPC
    uint64_t peer_epoch = 0;
    void* peer_table = nullptr;           // PeerTable (host copy, kernel argument)
    void setup_peer();
    // Device scalar sum of r² style partials → host value (allreduced).
    double finalize_scalar(const double* d_partials, int count);
};

// Host thread-local: device of the current call.
void bind_device(Ctx& c);

// NVTX range for a profiler timeline (nsys / ncu --nvtx); a no-op unless a
// tool is attached.  Scoped: pushed on construction, popped on destruction.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace kb
