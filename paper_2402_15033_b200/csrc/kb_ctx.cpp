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
        // Opt-in (KRY_PEER_ALLREDUCE=1): parity-identical, but no faster than
        // NCCL's small-message allreduce over NVLink at N = 2 (8000²: 41.76
        // vs 41.72 ms per cycle; 2000²: 4.261 vs 4.258 ms).
        const char* e = std::getenv("KRY_PEER_ALLREDUCE");
        if (e && std::atoi(e) == 1 && nranks <= kPeerMaxRanks) setup_peer();
    }
    partials.ensure(static_cast<size_t>(reduce_grid() + 64) * 8);
    h_scalar.ensure(64 * 8);
}

void Ctx::setup_peer() {
    // Receive area + flags of this rank, exported through CUDA IPC; every
    // rank maps every peer's (one collective exchange of the handles).
    peer_data.ensure(static_cast<size_t>(2) * nranks * kPeerMaxDoubles * 8);
    peer_flags.ensure(static_cast<size_t>(2) * nranks * 8);
    KB_CUDA(cudaMemset(peer_flags.p, 0, static_cast<size_t>(2) * nranks * 8));
    cudaIpcMemHandle_t mine[2];
    KB_CUDA(cudaIpcGetMemHandle(&mine[0], peer_data.p));
    KB_CUDA(cudaIpcGetMemHandle(&mine[1], peer_flags.p));
    const size_t hb = sizeof(mine);
    DevBuf d;
    d.ensure(hb * nranks);
    KB_CUDA(cudaMemcpy(reinterpret_cast<char*>(d.p) + hb * rank, mine, hb, cudaMemcpyHostToDevice));
    KB_NCCL(ncclAllGather(reinterpret_cast<char*>(d.p) + hb * rank, d.p, hb, ncclChar, comm, stream));
    std::vector<cudaIpcMemHandle_t> all(2 * static_cast<size_t>(nranks));
    KB_CUDA(cudaMemcpyAsync(all.data(), d.p, hb * nranks, cudaMemcpyDeviceToHost, stream));
    KB_CUDA(cudaStreamSynchronize(stream));
    auto* t = new PeerTable{};
    for (int r = 0; r < nranks; ++r) {
        if (r == rank) {
            t->data[r] = peer_data.p;
            t->flags[r] = peer_flags.as<uint64_t>();
            continue;
        }
        void* pd = nullptr;
        void* pf = nullptr;
        if (cudaIpcOpenMemHandle(&pd, all[2 * r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&pf, all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            // no peer mapping on this system: every rank must agree, so fail
            // loudly rather than mix the two reduction paths
            cudaGetLastError();
            delete t;
            fail(KRY_CUDA_ERROR, "peer allreduce: cudaIpcOpenMemHandle failed (set KRY_PEER_ALLREDUCE=0)");
        }
        peer_opened.push_back(pd);
        peer_opened.push_back(pf);
        t->data[r] = static_cast<double*>(pd);
        t->flags[r] = static_cast<uint64_t*>(pf);
    }
    peer_table = t;
    peer = true;
    // every rank has mapped every peer before the first peer store
    KB_NCCL(ncclAllReduce(d.p, d.p, 1, ncclChar, ncclSum, comm, stream));
    KB_CUDA(cudaStreamSynchronize(stream));
}

Ctx::~Ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : peer_opened) cudaIpcCloseMemHandle(p);
    delete static_cast<PeerTable*>(peer_table);
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
    if (peer && count <= static_cast<size_t>(kPeerMaxDoubles)) {
        launch_peer_allreduce(stream, d, static_cast<int>(count), *static_cast<const PeerTable*>(peer_table), rank,
                              nranks, ++peer_epoch, launches);
    } else {
        KB_NCCL(ncclAllReduce(d, d, count, ncclDouble, ncclSum, comm, stream));
    }
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
