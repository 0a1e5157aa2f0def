// pipeline.cuh — TMA bulk-copy (cp.async.bulk) ring that streams a score row from HBM
// into shared memory (sm_100a async proxy, mbarrier transaction counts).
//
// The ring has NSTAGE stages of STAGE_FLOATS fp32; stages are contiguous in shared
// memory and are consumed ROUND_STAGES at a time ("rounds"), so one round is one
// contiguous block of ROUND_FLOATS floats.  Thread 0 arms a stage's "full" mbarrier with
// the byte count and issues one 1-D bulk copy global -> shared; the consumers wait on
// "full", process the round, meet at one CTA barrier, and thread 0 refills the round's
// stages with the tiles NSTAGE ahead.  No registers hold in-flight data; the ring is
// primed before Phase 1 so the first NSTAGE tiles load while the guess is evaluated.
#pragma once
#include "device_common.cuh"

namespace gvr {

constexpr int NSTAGE = 4;
constexpr int ROUND_STAGES = 2;
constexpr int STAGE_FLOATS = 4096;
constexpr int STAGE_BYTES = STAGE_FLOATS * 4;  // 16 KB
constexpr int ROUND_FLOATS = ROUND_STAGES * STAGE_FLOATS;
static_assert(NSTAGE % ROUND_STAGES == 0, "a round never wraps the ring");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// Generic-proxy shared-memory accesses (the ring aliased as a work area, the cluster
// exchange area) ordered before later async-proxy (TMA) writes to the same bytes: every
// thread that touched them fences, then a barrier, then the TMA issue.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
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

// Row plan: the body [head, head + nfl) is 16-byte aligned and a multiple of 4 floats;
// the <= 3 scalars before it and after it are handled separately.
struct RowPlan {
    const float* x;
    int idx0;  // row index of x[0] (0 for a whole row, the slice start for a cluster slice)
    int n;
    int head;    // scalar elements [0, head) before the first 16-byte boundary
    int nfl;     // body floats (multiple of 4), starting at x + head (16-byte aligned)
    int ntiles;  // 0 for rows that are not streamed (len <= k)
};

__device__ __forceinline__ RowPlan plan_row(const float* scores, int64_t stride, const int32_t* row_lens, int r, int k)
{
    RowPlan p;
    int n = (int)stride;
    if (row_lens) n = min(max(__ldg(row_lens + r), 0), (int)stride);
    p.x = scores + (int64_t)r * stride;
    p.idx0 = 0;
    p.n = n;
    const uintptr_t a = reinterpret_cast<uintptr_t>(p.x);
    int head = (int)(((16u - (uint32_t)(a & 15u)) & 15u) >> 2);
    if (head > n) head = n;
    p.head = head;
    p.nfl = 4 * ((n - head) >> 2);
    p.ntiles = n <= k ? 0 : (p.nfl + STAGE_FLOATS - 1) / STAGE_FLOATS;
    return p;
}

// Slice g of G of a row plan (cluster mode): the body is cut at multiples of 4 floats;
// slice 0 keeps the unaligned head scalars, slice G-1 the tail scalars.  Every slice of
// a streamed row is non-empty when the body holds at least 4*G floats.
__device__ __forceinline__ RowPlan slice_plan(const RowPlan& w, int g, int G)
{
    const int v = w.nfl >> 2;  // body float4s
    const int b0 = w.head + 4 * (int)(((int64_t)v * g) / G);
    const int b1 = w.head + 4 * (int)(((int64_t)v * (g + 1)) / G);
    RowPlan p;
    const int start = g == 0 ? 0 : b0;
    const int end = g == G - 1 ? w.n : b1;
    p.x = w.x + start;
    p.idx0 = start;
    p.n = end - start;
    p.head = g == 0 ? w.head : 0;
    p.nfl = b1 - b0;
    p.ntiles = w.ntiles == 0 ? 0 : (p.nfl + STAGE_FLOATS - 1) / STAGE_FLOATS;
    return p;
}

struct Ring {
    float* stages;   // NSTAGE * STAGE_FLOATS, contiguous
    uint64_t* bars;  // full[NSTAGE]
    uint64_t policy;
    __device__ __forceinline__ uint32_t full(int s) const { return smem_u32(bars + s); }
    __device__ __forceinline__ const float* stage(int s) const { return stages + s * STAGE_FLOATS; }
    // thread 0 only: load body tile t of row p into its stage (t % NSTAGE)
    __device__ __forceinline__ void issue(const RowPlan& p, int t) const
    {
        const int s = t % NSTAGE;
        const uint32_t bytes = (uint32_t)min(STAGE_FLOATS, p.nfl - t * STAGE_FLOATS) * 4u;
        mbar_arrive_expect_tx(full(s), bytes);
        bulk_g2s(smem_u32(stage(s)), p.x + p.head + (size_t)t * STAGE_FLOATS, bytes, full(s), policy);
    }
};

}  // namespace gvr
