// One-shot deterministic allreduce of the small per-block reductions (the
// packed Gram, block_ortho.hpp:155's one reduce per BCGS-PIP, and the norm
// scalars) over NVLink peer memory, in place of an ncclAllReduce call.
//
// Every rank owns a receive area of 2 parities × nranks slots (CUDA IPC,
// mapped by every peer at context creation) and a flag array of the same
// shape.  One CTA per rank per call: (1) stores its vector into slot
// [parity][rank] of every rank's receive area (NVLink P2P stores through
// NVSwitch), (2) fences at system scope and raises flag [parity][rank] = epoch
// on every rank (release), (3) waits until all nranks flags of its own area
// reached the epoch (acquire), (4) sums the nranks slots in rank order — the
// same order on every rank, so the result is bit-identical everywhere (and
// independent of the NCCL algorithm / topology).  Parity double-buffering
// makes the areas reusable without a second handshake: a rank can only
// start epoch e + 2 after every rank has raised its flag for e + 1, i.e.
// after every rank finished reading epoch e.
#include <cuda_runtime.h>

#include "kb_common.hpp"
#include "kb_device.hpp"
#include "kb_kernels.hpp"

namespace kb {

namespace {

constexpr int kPeerThreads = 512;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kPeerThreads) peer_allreduce_kernel(double* __restrict__ d, int count,
                                                                    const PeerTable t, int rank, int nranks,
                                                                    uint64_t epoch) {
    KB_PDL_WAIT();
    const int par = static_cast<int>(epoch & 1);
    // 1. my contribution into slot [par][rank] of every rank's area
    for (int r = 0; r < nranks; ++r) {
        double* dst = t.data[r] + (static_cast<size_t>(par) * nranks + rank) * kPeerMaxDoubles;
        for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = d[i];
    }
    __threadfence_system();
    __syncthreads();
    // 2. raise my flag on every rank; 3. wait for every rank's flag in mine
    if (threadIdx.x < nranks) {
        st_release_sys(t.flags[threadIdx.x] + par * nranks + rank, epoch);
        const uint64_t* mine = t.flags[rank] + par * nranks + threadIdx.x;
        // a peer that never arrives (it failed, or took another code path)
        // must not hang the GPU: after ~10 s abort the context loudly
        const long long t0 = clock64();
        while (ld_acquire_sys(mine) < epoch) {
            if (clock64() - t0 > 20000000000LL) __trap();
        }
    }
    __syncthreads();
    // 4. Σ in rank order
    const double* area = t.data[rank] + static_cast<size_t>(par) * nranks * kPeerMaxDoubles;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += area[static_cast<size_t>(r) * kPeerMaxDoubles + i];
        d[i] = s;
    }
}

}  // namespace

void launch_peer_allreduce(cudaStream_t s, double* d, int count, const PeerTable& t, int rank, int nranks,
                           uint64_t epoch, int64_t& launches) {
    if (count > kPeerMaxDoubles || nranks > kPeerMaxRanks) fail(KRY_INTERNAL, "peer allreduce shape");
    launch_pdl(peer_allreduce_kernel, 1, kPeerThreads, 0, s, d, count, t, rank, nranks, epoch);
    KB_LAUNCHED();
    ++launches;
}

}  // namespace kb
