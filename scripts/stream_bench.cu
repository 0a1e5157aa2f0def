// Microbenchmark (not part of the library): raw streaming throughput of one SM / all
// SMs for the primitives the Top-K kernels use.
//   tma  : cp.async.bulk 1-D copies into an NSTAGE ring, thread 0 refills after a
//          CTA barrier (no other work).
//   ldg  : 128-bit ld.global.nc into registers, U float4 per thread in flight.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NSTAGE, int STAGE_BYTES>
__global__ void tma_stream(const float* rows, int n, float* sink)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * STAGE_BYTES);
    const float* x = rows + (size_t)blockIdx.x * n;
    const int nbytes = n * 4;
    const int ntiles = (nbytes + STAGE_BYTES - 1) / STAGE_BYTES;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int t) {
        const int s = t % NSTAGE;
        const uint32_t bytes = (uint32_t)min(STAGE_BYTES, nbytes - t * STAGE_BYTES);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bars + s)), "r"(bytes)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(smem + s * STAGE_BYTES)),
                     "l"(reinterpret_cast<const char*>(x) + (size_t)t * STAGE_BYTES), "r"(bytes), "r"(smem_u32(bars + s))
                     : "memory");
    };
    if (threadIdx.x == 0)
        for (int t = 0; t < NSTAGE && t < ntiles; ++t) issue(t);
    float acc = 0.f;
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % NSTAGE;
        uint32_t ok = 0;
        do {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(smem_u32(bars + s)), "r"((uint32_t)(t / NSTAGE) & 1u)
                : "memory");
        } while (!ok);
        acc += reinterpret_cast<const float*>(smem + s * STAGE_BYTES)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && t + NSTAGE < ntiles) issue(t + NSTAGE);
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int U>
__global__ void ldg_stream(const float* rows, int n, float* sink)
{
    const float4* x = reinterpret_cast<const float4*>(rows + (size_t)blockIdx.x * n);
    const int nv = n / 4;
    float acc = 0.f;
    for (int base = 0; base < nv; base += blockDim.x * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = base + u * blockDim.x + threadIdx.x;
            v[u] = i < nv ? __ldg(x + i) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 12345.f) sink[0] = acc;
}

int main()
{
    const int n = 100000;
    const int max_rows = 148 * 4;
    float* d;
    float* sink;
    cudaMalloc(&d, (size_t)max_rows * n * 4);
    cudaMemset(d, 0, (size_t)max_rows * n * 4);
    cudaMalloc(&sink, 4);
    float* flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, int rows, auto launch) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, 512 << 20);
            cudaEventRecord(e0);
            launch(rows);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double gb = (double)rows * n * 4 / 1e9;
        printf("%-28s rows %4d  %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA-row\n", name, rows, best * 1e3,
               gb / (best * 1e-3), (double)n * 4 / 1e9 / (best * 1e-3));
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) printf("  error %s\n", cudaGetErrorString(err));
    };
    cudaFuncSetAttribute(tma_stream<5, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 16384 + 64);
    cudaFuncSetAttribute(tma_stream<8, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 64);
    cudaFuncSetAttribute(tma_stream<4, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 64);
    cudaFuncSetAttribute(tma_stream<12, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384 + 64);
    for (int rows : {1, 148, 296, 592}) {
        timeit("tma 5x16KB", rows, [&](int r) { tma_stream<5, 16384><<<r, 256, 5 * 16384 + 64>>>(d, n, sink); });
        timeit("tma 8x16KB", rows, [&](int r) { tma_stream<8, 16384><<<r, 256, 8 * 16384 + 64>>>(d, n, sink); });
        timeit("tma 4x32KB", rows, [&](int r) { tma_stream<4, 32768><<<r, 256, 4 * 32768 + 64>>>(d, n, sink); });
        timeit("tma 12x16KB", rows, [&](int r) { tma_stream<12, 16384><<<r, 256, 12 * 16384 + 64>>>(d, n, sink); });
        timeit("ldg U4 256thr", rows, [&](int r) { ldg_stream<4><<<r, 256>>>(d, n, sink); });
        timeit("ldg U8 256thr", rows, [&](int r) { ldg_stream<8><<<r, 256>>>(d, n, sink); });
        timeit("ldg U4 512thr", rows, [&](int r) { ldg_stream<4><<<r, 512>>>(d, n, sink); });
        timeit("ldg U8 1024thr", rows, [&](int r) { ldg_stream<8><<<r, 1024>>>(d, n, sink); });
    }
    return 0;
}
