// Microbenchmark: random 8-byte gathers of x (n doubles) via the LSU
// (ld.global.cg) vs the TMA engine (cp.async.bulk.tensor.2d ... tile::gather4,
// x viewed as an [n/2][2] tensor of 16-byte rows).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_bench gather4_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

constexpr int kChunk = 256;  // indices per warp per round

__global__ void lsu_kernel(const double* __restrict__ x, const int* __restrict__ idx, long long m, double* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    double s = 0.0;
    for (long long base = warp * kChunk; base < m; base += nw * kChunk) {
        int c[kChunk / 32];
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) c[u] = idx[base + lane + 32 * u];
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) s += __ldcg(x + c[u]);
    }
    if (s == 12345.678) out[0] = s;
}

__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx, long long m,
                           double* out) {
    extern __shared__ __align__(128) double dyn[];  // per warp: 64 gather4 slots × 128 B (TMA needs 128-B aligned destinations)
    double* buf = dyn;  // [8][64][16]
    __shared__ alignas(8) unsigned long long bar[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    double s = 0.0;
    unsigned phase = 0;
    for (long long base = warp * kChunk; base < m; base += nw * kChunk) {
        int c[kChunk / 32];
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) c[u] = idx[base + lane + 32 * u];
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w])),
                         "r"(kChunk * 16) : "memory");
        __syncwarp();
        // row ids of the [n/2][2] view, staged for the issuing lanes (8 lanes × 8 gather4 × 4 rows)
        __shared__ int rows[8][kChunk];
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) rows[w][lane + 32 * u] = c[u] >> 1;
        __syncwarp();
        if (lane < 8) {
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const int e0 = (lane * 8 + g) * 4;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (w * 64 + e0 / 4) * 16)),
                    "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(rows[w][e0]), "r"(rows[w][e0 + 1]),
                    "r"(rows[w][e0 + 2]), "r"(rows[w][e0 + 3]), "r"(smem_u32(&bar[w]))
                    : "memory");
            }
        }
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(&bar[w])),
            "r"(phase)
            : "memory");
        phase ^= 1;
#pragma unroll
        for (int u = 0; u < kChunk / 32; ++u) {
            const int e = lane + 32 * u;  // gather4 slot e/4, row e%4 (16 B each)
            s += buf[(w * 64 + e / 4) * 16 + (e % 4) * 2 + (c[u] & 1)];
        }
        __syncwarp();
    }
    if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
    const long long n = argc > 1 ? atoll(argv[1]) : 20000000LL;
    const long long m = argc > 2 ? atoll(argv[2]) : 200000000LL;
    double* x;
    int* idx;
    double* out;
    cudaMalloc(&x, n * 8);
    cudaMalloc(&idx, m * 4);
    cudaMalloc(&out, 8);
    cudaMemset(x, 0, n * 8);
    std::vector<int> h(m);
    unsigned long long st = 88172645463325252ULL;
    for (long long i = 0; i < m; ++i) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        h[i] = static_cast<int>(st % n);
    }
    cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {2, static_cast<cuuint64_t>(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    int sms = 148;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        lsu_kernel<<<sms * 8, 256>>>(x, idx, m, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("lsu  %.3f ms  %.2f Ggather/s  err %s\n", ms, m / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        cudaEventRecord(a);
        cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 64 * 128);
        tma_kernel<<<sms * 3, 256, 8 * 64 * 128>>>(map, idx, m, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("tma  %.3f ms  %.2f Ggather/s  err %s\n", ms, m / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
