// pipeline.cuh — TMA bulk-copy (cp.async.bulk) ring that streams a score row from HBM
// into shared memory (sm_100a async proxy, mbarrier transaction-count completion).
//
// The row body (16-byte aligned float4 run) is cut into ring tiles of STAGE_FLOATS
// fp32.  One elected thread arms a stage's mbarrier with the byte count and issues
// one 1-D bulk copy global -> shared per tile; all threads wait on the stage's parity.
// No registers hold in-flight data (the prefetch depth is set by shared memory), and
// tiles can be indexed dynamically: the rare candidates are picked out by index.
#pragma once
#include "row_tiles.cuh"

namespace gvr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t bar_full(int stage) { return smem_u32(g_smem + OFF_BAR + 8 * stage); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}

// Ring over the body of one row (non-persistent CTA): stage of tile t is t % NSTAGE
// and its mbarrier parity (t / NSTAGE) & 1.  Thread 0 primes NSTAGE tiles and refills
// the stage of tile t-1 with tile t-1+NSTAGE once every thread has passed tile t's
// block scan (all reads of tile t-1 are then complete).
struct Ring {
    const float* body;  // 16-byte aligned start of the row body
    int nfl;            // body floats (multiple of 4)
    int ntiles;
    uint64_t policy;

    __device__ __forceinline__ int tile_floats(int t) const { return min(STAGE_FLOATS, nfl - t * STAGE_FLOATS); }
    __device__ __forceinline__ int stage_of(int t) const { return t % NSTAGE; }
    __device__ __forceinline__ const float* stage_ptr(int t) const { return s_ring() + stage_of(t) * STAGE_FLOATS; }
    __device__ __forceinline__ void issue(int t) const
    {
        const int st = stage_of(t);
        const uint32_t bytes = (uint32_t)tile_floats(t) * 4u;
        const uint32_t bar = bar_full(st);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(smem_u32(s_ring() + st * STAGE_FLOATS), body + (size_t)t * STAGE_FLOATS, bytes, bar, policy);
    }
    __device__ __forceinline__ void wait(int t) const { mbar_wait(bar_full(stage_of(t)), (uint32_t)(t / NSTAGE) & 1u); }
};

__device__ __forceinline__ Ring make_ring(const float* body, int nfl)
{
    Ring r;
    r.body = body;
    r.nfl = nfl;
    r.ntiles = (nfl + STAGE_FLOATS - 1) / STAGE_FLOATS;
    r.policy = policy_evict_first();
    return r;
}

// Barrier init + prime (thread 0); the caller orders it with a CTA barrier before any
// consumer waits.
__device__ __forceinline__ void ring_start(const Ring& r)
{
    if (threadIdx.x == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(bar_full(s), 1);
        fence_mbar_init();
        for (int t = 0; t < NSTAGE && t < r.ntiles; ++t) r.issue(t);
    }
}

}  // namespace gvr
