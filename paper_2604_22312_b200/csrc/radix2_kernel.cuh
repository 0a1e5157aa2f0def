// radix2_kernel.cuh — the same-geometry radix-select baseline (
// DESIGN.md §2.5).
//
// The paper compares GVR with a radix select "under identical thread-level resources"
// (PAPER.md:800-802).  The one-CTA-per-row radix kernel (radix_kernel.cuh) re-reads the
// row from HBM on every round; this baseline instead runs on exactly the machinery of the
// GVR batch path, so the only difference is how the collect threshold is found:
//   * radix_hist_kernel — the first radix round as one HBM pass over the whole batch
//     (the filter kernel's persistent tile partition and TMA ring): a 2048-bin histogram
//     of the paper's 16-bit "half" digit (R18) — the top
//     11 bits of the fp16-rounded score's sortable key — per row segment in shared memory,
//     added into the row's global histogram at the segment's end.  Long rows are split
//     over several CTAs (the split-CTA radix of PAPER.md:140-142).
//   * radix_thresh_kernel — per row, the K-th-bin search over that histogram (the prefix
//     sum / find-threshold step) and T1 = the smallest fp32 key whose
//     half digit reaches the K-th bin.
//   * then gvr_filter_kernel (the second HBM pass, collecting {x >= T1}),
//     gvr_refine_kernel and gvr_fixup_kernel — the remaining radix rounds run on the
//     list in L2 (the refine's exact narrowing), as GVR's Phase 4 does.
// Two HBM passes per row where GVR's guess makes one; the result is exact for any T1 with
// f(T1) >= K (Lemma 1) and the refine verifies that count.
#pragma once
#include <cuda_fp16.h>

#include "filter_kernel.cuh"

namespace gvr {

constexpr int RH_NT = 256;
constexpr int RH_OFF_RING = 0;
constexpr int RH_OFF_BARS = F_NSTAGE * STAGE_BYTES;
constexpr int RH_OFF_HIST = RH_OFF_BARS + F_NSTAGE * 8;  // int32[NBINS] segment histogram
constexpr int RH_OFF_SCR = RH_OFF_HIST + NBINS * 4;
constexpr int RH_SMEM_BYTES = RH_OFF_SCR + GROUP_SCRATCH_BYTES;
static_assert(F_CTAS_PER_SM * (RH_SMEM_BYTES + 1024) <= 233472, "three histogram CTAs per SM");

// The 16-bit "half" digit: the top 11 bits of the sortable key of the
// fp16-rounded value (round to nearest: monotone non-decreasing in the fp32 value).
__device__ __forceinline__ int half_bin(float x)
{
    const uint32_t u = __half_as_ushort(__float2half_rn(x));
    const uint32_t k16 = u ^ ((u & 0x8000u) ? 0xffffu : 0x8000u);
    return (int)(k16 >> 5);
}

__global__ void __launch_bounds__(RH_NT, F_CTAS_PER_SM)
radix_hist_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                  CandLists cl, uint32_t* __restrict__ ghist)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const Ring ring{reinterpret_cast<float*>(smem + RH_OFF_RING), reinterpret_cast<uint64_t*>(smem + RH_OFF_BARS),
                    policy_evict_first()};
    int32_t* hist = reinterpret_cast<int32_t*>(smem + RH_OFF_HIST);
    FilterGroup c;
    c.init(threadIdx.x, smem + RH_OFF_SCR);
    const int b = blockIdx.x;
    const long long vb = cl_begin(cl, b), ve = cl_begin(cl, b + 1);
    RoundIter prod;
    prod.start(vb, ve, cl.tpr);
    if (c.tid == 0) {
        for (int s = 0; s < F_NSTAGE; ++s) mbar_init(ring.full(s), 1);
        fence_mbar_init();
        for (int issued = 0; issued < F_ROUNDS && prod.next(scores, stride, row_lens, k, cl.tpr); ++issued)
            issue_pair(ring, prod, issued);
    }
    for (int i = c.tid; i < NBINS; i += RH_NT) hist[i] = 0;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the cleared global histograms
    c.sync();
    RoundIter it;
    it.start(vb, ve, cl.tpr);
    const int lb = lane_base(c.warp, c.lane);
    for (int i = 0; it.next(scores, stride, row_lens, k, cl.tpr); ++i) {
        const RowPlan& p = it.p;
        const int body_end = p.head + p.nfl;
        int si = -1;
        if (it.t0 == 0 && c.tid < p.head) si = c.tid;
        if (it.t0 + it.nt == p.ntiles && c.tid >= 32 && c.tid < 32 + (p.n - body_end)) si = body_end + (c.tid - 32);
        const float sv = si >= 0 ? __ldg(p.x + si) : 0.f;
        const int s0 = ROUND_STAGES * (i % F_ROUNDS);
        const uint32_t par = (uint32_t)(i / F_ROUNDS) & 1u;
        mbar_wait(ring.full(s0), par);
        mbar_wait(ring.full(s0 + 1), par);
        const float* sp = ring.stage(s0);
        const int nf = min(it.nt * STAGE_FLOATS, p.nfl - it.t0 * STAGE_FLOATS);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (lb + 128 * j < nf) {
                const float4 v = *reinterpret_cast<const float4*>(sp + lb + 128 * j);
                atomicAdd(&hist[half_bin(v.x)], 1);
                atomicAdd(&hist[half_bin(v.y)], 1);
                atomicAdd(&hist[half_bin(v.z)], 1);
                atomicAdd(&hist[half_bin(v.w)], 1);
            }
        }
        if (si >= 0) atomicAdd(&hist[half_bin(sv)], 1);
        c.sync();  // the round's stages are consumed
        if (c.tid == 0 && prod.next(scores, stride, row_lens, k, cl.tpr)) issue_pair(ring, prod, i + F_ROUNDS);
        if (it.last) {
            // end of this CTA's segment of the row: its counts into the row's histogram
            uint32_t* gh = ghist + (size_t)it.r * NBINS;
            for (int q = c.tid; q < NBINS; q += RH_NT) {
                const int v = hist[q];
                if (v) {
                    atomicAdd(gh + q, (uint32_t)v);
                    hist[q] = 0;
                }
            }
            c.sync();
        }
    }
}

// Per row: the K-th bin of the half-digit histogram, scanned from the top, and T1 = the
// smallest fp32 key whose digit reaches it (binary search over the monotone digit).  Rows
// with no tiles go to the ready queue (the refine kernel emits them from the row itself).
__global__ void __launch_bounds__(256)
radix_thresh_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                    const uint32_t* __restrict__ ghist, GuessOut* __restrict__ gp, BatchQueue bq)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the histogram pass is complete
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ __align__(16) unsigned char scratch[GROUP_SCRATCH_BYTES];
    Group<256, 1> c;
    c.init(threadIdx.x, scratch);
    const int r = blockIdx.x;
    const RowPlan p = plan_row(scores, stride, row_lens, r, k);
    if (bq.queue && p.ntiles == 0 && c.tid == 0) st_release(bq.queue + atomicAdd(bq.qctl + Q_TAIL, 1), r + 1);
    if (p.n <= k) return;
    // thread t owns bins 2047 - 8t .. 2040 - 8t (descending digit order)
    const uint32_t* gh = ghist + (size_t)r * NBINS;
    int h[8];
    uint32_t loc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h[i] = (int)__ldcg(gh + (NBINS - 1 - 8 * c.tid - i));
        loc += (uint32_t)h[i];
    }
    uint32_t tot;
    const uint32_t above0 = group_excl_scan(c, loc, tot);
    {
        uint32_t above = above0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (above < (uint32_t)k && above + (uint32_t)h[i] >= (uint32_t)k) c.misc[0] = NBINS - 1 - 8 * c.tid - i;
            above += (uint32_t)h[i];
        }
    }
    c.sync();
    if (c.tid == 0) {
        const int bk = c.misc[0];
        uint64_t lo = 0, hi = 1ull << 32;  // invariant: digit(hi) >= bk (hi = 2^32: above every key)
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (half_bin(key2f((uint32_t)mid)) >= bk)
                hi = mid;
            else
                lo = mid;
        }
        GuessOut g{};
        g.Tc = hi > 0xffffffffull ? 0xffffffffu : (uint32_t)hi;
        g.tmin = 0u;
        g.top = 0xffffffffu;
        g.exit = GVR_P2_ALL;
        gp[r] = g;
        publish_tc(bq, r, g.Tc);
    }
}

}  // namespace gvr
