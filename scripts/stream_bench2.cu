// Microbenchmark (not part of the library): the GVR streaming collect loop alone —
// TMA ring -> threshold filter -> compaction into a shared-memory candidate buffer —
// across CTA geometries, to pick the kernel shape.  Rows are N(0,1) floats, the
// threshold keeps ~5 % (the f(T_c)/N range of the Eq. 1 rows).
//   lockstep : per tile, warp scan + CTA-wide scan of warp totals through shared memory
//              and two barriers; thread 0 refills after the second barrier.
//   decoupled: per tile, warp scan + one shared atomic per warp for the base; each warp
//              arrives on the stage's "empty" mbarrier; warp 0 refills.
// Occupancy is forced with dynamic shared-memory padding.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bench2 stream_bench2.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(bar), "r"(par)
                 : "memory");
    return ok;
}
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t par)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(bar), "r"(par)
                 : "memory");
    return ok;
}
__device__ __forceinline__ void issue(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ uint32_t warp_incl(uint32_t v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

constexpr int CAP = 8192;

template <int NT, int NSTAGE, int SF, bool DECOUPLED>
__global__ void __launch_bounds__(NT) collect(const float* rows, int n, float tf, int* out_cnt)
{
    constexpr int W = NT / 32;
    constexpr int EPT = SF / NT;  // floats per thread per tile
    constexpr int V = EPT / 4;
    static_assert(EPT % 4 == 0 && EPT <= 32, "");
    extern __shared__ __align__(128) unsigned char smem[];
    float* ring = reinterpret_cast<float*>(smem);
    uint32_t* bkey = reinterpret_cast<uint32_t*>(smem + NSTAGE * SF * 4);
    int32_t* bidx = reinterpret_cast<int32_t*>(bkey + CAP);
    uint64_t* full = reinterpret_cast<uint64_t*>(bidx + CAP);
    uint64_t* empty = full + NSTAGE;
    int* misc = reinterpret_cast<int*>(empty + NSTAGE);  // [0] fill, [32..] warp totals
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* x = rows + (size_t)blockIdx.x * n;
    const int ntiles = n / SF;
    if (tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            mbar_init(smem_u32(full + s), 1);
            mbar_init(smem_u32(empty + s), W);
        }
        misc[0] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int t = 0; t < NSTAGE && t < ntiles; ++t)
            issue(smem_u32(ring + t * SF), x + (size_t)t * SF, SF * 4, smem_u32(full + t));
    }
    __syncthreads();
    int fill = 0;
    uint32_t released = 0, issued = min(NSTAGE, ntiles);
    // element e of thread: vector j = e/4 at float offset 4*(lane + 32*(warp*V + j))
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % NSTAGE;
        const uint32_t par = (t / NSTAGE) & 1u;
        if (DECOUPLED && warp == 0) {
            while (!test_wait(smem_u32(full + s), par)) {
                if (tid == 0)
                    while (released < issued && test_wait(smem_u32(empty + released % NSTAGE), (released / NSTAGE) & 1u)) {
                        const uint32_t g = issued++;
                        ++released;
                        if ((int)g < ntiles)
                            issue(smem_u32(ring + (g % NSTAGE) * SF), x + (size_t)g * SF, SF * 4,
                                  smem_u32(full + g % NSTAGE));
                        else
                            --issued, released = issued;  // nothing more to issue
                    }
            }
        } else {
            while (!try_wait(smem_u32(full + s), par)) {
            }
        }
        const float* sp = ring + s * SF;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(sp + 4 * (lane + 32 * (warp * V + j)));
            mask |= (uint32_t)(v.x >= tf) << (4 * j);
            mask |= (uint32_t)(v.y >= tf) << (4 * j + 1);
            mask |= (uint32_t)(v.z >= tf) << (4 * j + 2);
            mask |= (uint32_t)(v.w >= tf) << (4 * j + 3);
        }
        const uint32_t cnt = __popc(mask);
        const uint32_t incl = warp_incl(cnt, lane);
        const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
        int base;
        if (DECOUPLED) {
            int b = 0;
            if (lane == 0 && wtot) b = atomicAdd(misc, (int)wtot);
            base = __shfl_sync(0xffffffffu, b, 0);
        } else {
            if (lane == 31) misc[32 + warp] = (int)incl;
            __syncthreads();
            int pre = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int c = misc[32 + w];
                pre += w < warp ? c : 0;
                tot += c;
            }
            base = fill + pre;
            fill += tot;
        }
        int pos = (base + (int)(incl - cnt)) & (CAP - 1);
        while (mask) {
            const int e = __ffs(mask) - 1;
            mask &= mask - 1;
            const int off = 4 * (lane + 32 * (warp * V + (e >> 2))) + (e & 3);
            const float v = sp[off];
            const uint32_t u = __float_as_uint(v);
            bkey[pos] = (int)u < 0 ? ~u : (u | 0x80000000u);
            bidx[pos] = t * SF + off;
            pos = (pos + 1) & (CAP - 1);
        }
        if (DECOUPLED) {
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)) : "memory");
        } else {
            __syncthreads();
            if (tid == 0 && t + NSTAGE < ntiles)
                issue(smem_u32(ring + s * SF), x + (size_t)(t + NSTAGE) * SF, SF * 4, smem_u32(full + s));
        }
    }
    __syncthreads();
    if (tid == 0) out_cnt[blockIdx.x] = DECOUPLED ? misc[0] : fill;
}

__global__ void init_normal(float* d, size_t n)
{
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + 12345;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const float u1 = ((z >> 40) + 1) * (1.0f / 16777217.0f), u2 = ((z & 0xffffff) + 0.5f) * (1.0f / 16777216.0f);
        d[i] = sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
    }
}

int main(int argc, char** argv)
{
    const int only = argc > 1 ? atoi(argv[1]) : -1;  // run one geometry (for ncu)
    int idx = 0;
    const int n = 98304;  // multiple of every tile size below
    const int max_rows = 148 * 4;
    float* d;
    int* cnt;
    cudaMalloc(&d, (size_t)max_rows * n * 4);
    init_normal<<<1024, 256>>>(d, (size_t)max_rows * n);
    cudaMalloc(&cnt, max_rows * 4);
    float* flush;
    cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const float tf = 1.645f;
    auto run = [&](const char* name, auto kern, int nt, int nstage, int sf, int cta_per_sm) {
        if (only >= 0 && idx++ != only) return;
        const int need = nstage * sf * 4 + CAP * 8 + 2 * nstage * 8 + 64 * 4;
        int smem = 227 * 1024 / cta_per_sm - 1024;
        if (smem < need) {
            printf("%-34s %d/SM: does not fit (%d > %d)\n", name, cta_per_sm, need, smem);
            return;
        }
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
        for (int rows : {148 * cta_per_sm, 488}) {
            float best = 1e9f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(flush, rep, 512 << 20);
                cudaEventRecord(e0);
                kern<<<rows, nt, smem>>>(d, n, tf, cnt);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            int c0;
            cudaMemcpy(&c0, cnt, 4, cudaMemcpyDeviceToHost);
            const double gb = (double)rows * n * 4 / 1e9;
            printf("%-34s %d/SM (occ %d) rows %4d  %7.1f us  %7.1f GB/s  cnt0 %d %s\n", name, cta_per_sm, occ, rows,
                   best * 1e3, gb / (best * 1e-3), c0, cudaGetErrorString(cudaGetLastError()));
        }
    };
#define RUN(NT, NS, SF, DEC, CPS) \
    run(DEC ? #NT " thr " #NS "x" #SF " decoupled" : #NT " thr " #NS "x" #SF " lockstep", collect<NT, NS, SF, DEC>, NT, NS, \
        SF, CPS)
    for (int cps : {1, 2, 3, 4}) {
        RUN(256, 4, 4096, false, cps);
        RUN(256, 4, 4096, true, cps);
        RUN(256, 3, 2048, false, cps);
        RUN(256, 3, 2048, true, cps);
        RUN(128, 4, 2048, false, cps);
        RUN(128, 4, 2048, true, cps);
        RUN(512, 4, 4096, false, cps);
        RUN(512, 4, 4096, true, cps);
        RUN(512, 3, 8192, false, cps);
        RUN(256, 6, 2048, false, cps);
        RUN(256, 6, 2048, true, cps);
    }
    return 0;
}
