#include <cstdlib>
#include <chrono>
#include "kb_ctx.hpp"

#include <cstring>

#include "kb_kernels.hpp"

namespace kb {

#define KB_NCCL(expr)                                                                      \
    do {                                                                                   \
        ncclResult_t kb_r_ = (expr);                                                       \
        if (kb_r_ != ncclSuccess)                                                          \
            ::kb::fail(KRY_NCCL_ERROR, std::string(#expr) + ": " + ncclGetErrorString(kb_r_)); \
    } while (0)

Ctx::Ctx(int dev, int nr, int rk, const void* nccl_id) : device(dev), nranks(nr), rank(rk) {
    if (const char* e = std::getenv("KRY_HOST_PROFILE")) host_profile = std::atoi(e) != 0;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        fail(KRY_NO_DEVICE, "no CUDA device visible; the B200 path has no CPU fallback");
    }
    if (dev < 0 || dev >= count) fail(KRY_INVALID_ARGUMENT, "device index out of range");
    KB_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop;
    KB_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        fail(KRY_NO_DEVICE, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
    KB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    if (nranks > 1) {
        if (!nccl_id) fail(KRY_INVALID_ARGUMENT, "multi-rank context needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        KB_NCCL(ncclCommInitRank(&comm, nranks, id, rank));
    }
    partials.ensure(static_cast<size_t>(reduce_grid() + 64) * 8);
    h_scalar.ensure(64 * 8);
}

Ctx::~Ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& p : pending) {
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    if (comm) ncclCommDestroy(comm);
    if (stream) cudaStreamDestroy(stream);
}

void bind_device(Ctx& c) { KB_CUDA(cudaSetDevice(c.device)); }

void Ctx::sync() {
    drain_timers();  // elapsed-time queries of finished phases, while the GPU is still busy
    if (!host_profile) {
        KB_CUDA(cudaStreamSynchronize(stream));
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    KB_CUDA(cudaStreamSynchronize(stream));
    sync_wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ++sync_count;
}

cudaEvent_t Ctx::begin_phase() {
    if (!timing) return nullptr;
    cudaEvent_t e;
    if (pool.empty()) {
        KB_CUDA(cudaEventCreate(&e));
    } else {
        e = pool.back();
        pool.pop_back();
    }
    KB_CUDA(cudaEventRecord(e, stream));
    return e;
}

void Ctx::end_phase(int phase, cudaEvent_t start) {
    if (!timing || !start) return;
    cudaEvent_t e;
    if (pool.empty()) {
        KB_CUDA(cudaEventCreate(&e));
    } else {
        e = pool.back();
        pool.pop_back();
    }
    KB_CUDA(cudaEventRecord(e, stream));
    pending.push_back({phase, start, e});
}

void Ctx::drain_timers() {
    size_t done = 0;
    for (; done < pending.size(); ++done) {  // events complete in stream order
        const Pending& p = pending[done];
        if (cudaEventQuery(p.b) != cudaSuccess) break;
        float ms = 0.f;
        KB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        seconds[p.phase] += ms * 1e-3;
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    cudaGetLastError();  // cudaErrorNotReady from the query is not an error
    pending.erase(pending.begin(), pending.begin() + static_cast<std::ptrdiff_t>(done));
}

void Ctx::resolve_timers() {
    if (pending.empty()) return;
    KB_CUDA(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
        float ms = 0.f;
        KB_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        seconds[p.phase] += ms * 1e-3;
        pool.push_back(p.a);
        pool.push_back(p.b);
    }
    pending.clear();
}

void Ctx::allreduce_sum(double* d, size_t count) {
    if (nranks <= 1 || count == 0) return;
    KB_NCCL(ncclAllReduce(d, d, count, ncclDouble, ncclSum, comm, stream));
    ++allreduces;
}

double Ctx::finalize_scalar(const double* d_partials, int count) {
    double* d_out = partials.p + reduce_grid();
    launch_finalize_sum(stream, d_partials, count, d_out, launches);
    allreduce_sum(d_out, 1);
    KB_CUDA(cudaMemcpyAsync(h_scalar.p, d_out, 8, cudaMemcpyDeviceToHost, stream));
    sync();
    return h_scalar.p[0];
}

}  // namespace kb
