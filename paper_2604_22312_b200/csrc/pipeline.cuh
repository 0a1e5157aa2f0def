// pipeline.cuh — TMA bulk-copy (cp.async.bulk) ring for streaming a score row from
// HBM into shared memory (sm_90+/sm_100a async proxy).
//
// The row body (16-byte aligned float4 run) is cut into ring tiles of STAGE_FLOATS
// fp32.  One elected thread arms a stage's mbarrier with the byte count and issues one
// 1-D bulk copy global -> shared per tile; consumers wait on the stage's mbarrier
// parity.  No registers hold in-flight data, so the prefetch depth is set by shared
// memory (NSTAGE-1 tiles ahead of the consumer), and tiles can be indexed dynamically
// (the rare candidates are picked out of shared memory by index).
#pragma once
#include "device_common.cuh"

namespace gvr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t bar_addr(int stage) { return smem_u32(g_smem + OFF_BAR + 8 * stage); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
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

// Ring state of one CTA.  `seq` counts tiles issued over the CTA's lifetime so stage
// and parity stay consistent across several passes over a row.
struct Ring {
    const float* body;  // 16B-aligned start of the row body
    int nfl;            // body length in floats (multiple of 4)
    int ntiles;
    uint32_t seq0;      // sequence number of this pass's tile 0
    uint64_t policy;

    __device__ __forceinline__ int tile_floats(int t) const { return min(STAGE_FLOATS, nfl - t * STAGE_FLOATS); }
    __device__ __forceinline__ int stage_of(int t) const { return (int)((seq0 + (uint32_t)t) % NSTAGE); }
    __device__ __forceinline__ uint32_t parity_of(int t) const { return ((seq0 + (uint32_t)t) / NSTAGE) & 1u; }
    __device__ __forceinline__ const float* stage_ptr(int t) const { return s_ring() + stage_of(t) * STAGE_FLOATS; }

    // issue tile t (one elected thread)
    __device__ __forceinline__ void issue(int t) const
    {
        const int st = stage_of(t);
        const uint32_t bytes = (uint32_t)tile_floats(t) * 4u;
        const uint32_t bar = bar_addr(st);
        mbar_arrive_expect_tx(bar, bytes);
        bulk_g2s(smem_u32(s_ring() + st * STAGE_FLOATS), body + (size_t)t * STAGE_FLOATS, bytes, bar, policy);
    }
    __device__ __forceinline__ void wait(int t) const { mbar_wait(bar_addr(stage_of(t)), parity_of(t)); }
};

// One-time barrier setup (thread 0), visible to the async proxy before first use.
__device__ __forceinline__ void ring_init_barriers(const Ctx& c)
{
    if (c.tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(bar_addr(s), 1);
        fence_mbar_init();
    }
}

__device__ __forceinline__ Ring make_ring(const float* body, int nfl, uint32_t seq0)
{
    Ring r;
    r.body = body;
    r.nfl = nfl;
    r.ntiles = (nfl + STAGE_FLOATS - 1) / STAGE_FLOATS;
    r.seq0 = seq0;
    r.policy = policy_evict_first();
    return r;
}

// Prime the first NSTAGE tiles (thread 0).  Ring memory must be free (generic-proxy
// accesses to it ordered before this call by a barrier).
__device__ __forceinline__ void ring_prime(const Ctx& c, const Ring& r)
{
    if (c.tid == 0) {
        fence_proxy_async();
        for (int t = 0; t < NSTAGE && t < r.ntiles; ++t) r.issue(t);
    }
}

}  // namespace gvr
