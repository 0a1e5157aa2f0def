// radix_kernel.cuh — in-house radix-select baseline (Sec. 2.2).
//
// One CTA of 256 threads per row (the paper runs its baseline one CTA per row,
// PAPER.md:707-710, 799-802).  Each round is a full-row histogram pass over global
// memory into a 2048-bin shared-memory histogram with atomicAdd, a
// K-th-bin search over the bin totals (the prefix-sum / find-threshold steps,
// PAPER.md:132-133), and a narrowing of the key prefix.  Digits are key bits [31:21],
// [20:10], [9:0] (the 11/11/10 schedule of PAPER.md:138; R18).  As soon as
// the threshold bucket holds <= 2048 elements the round loop exits early
// and one filter pass collects every element at or above the bucket
// into shared memory, where the exact ordered result is finished.  With all 32 bits
// resolved the K-th key is exact and ties are filled in index order.  Same 128-bit
// coalesced loads and ordered-output stage as GVR.
#pragma once
#include "select_global.cuh"

namespace gvr {

constexpr int RADIX_NT = 256;
constexpr int RADIX_CAP = SORT_MAX;  // early exit keeps < K + 2048 entries; tie fill uses [0, 2K)
using RadixGroup = Group<RADIX_NT, 1>;
constexpr int RADIX_OFF_BKEY = 0;
constexpr int RADIX_OFF_BIDX = RADIX_OFF_BKEY + RADIX_CAP * 4;
constexpr int RADIX_OFF_WORK = RADIX_OFF_BIDX + RADIX_CAP * 4;
constexpr int RADIX_CSORT = SORT_MAX;
constexpr int RADIX_OFF_SCRATCH = RADIX_OFF_WORK + work_bytes(RADIX_CSORT);
constexpr int RADIX_SMEM_BYTES = RADIX_OFF_SCRATCH + GROUP_SCRATCH_BYTES;
static_assert(RADIX_CAP >= 2 * KMAX, "tie fill uses B[0, 2K)");

__global__ void __launch_bounds__(RADIX_NT, 2)
radix_topk_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                  int32_t* __restrict__ out, float* out_val, gvr_row_stats* stats)
{
    extern __shared__ __align__(128) unsigned char smem[];
    RadixGroup c;
    c.init(threadIdx.x, smem + RADIX_OFF_SCRATCH);
    const Buf B{reinterpret_cast<uint32_t*>(smem + RADIX_OFF_BKEY), reinterpret_cast<int32_t*>(smem + RADIX_OFF_BIDX),
                RADIX_CAP};
    const Work Wk{reinterpret_cast<int32_t*>(smem + RADIX_OFF_WORK),
                  reinterpret_cast<int32_t*>(smem + RADIX_OFF_WORK + NBINS * 4),
                  reinterpret_cast<unsigned long long*>(smem + RADIX_OFF_WORK + 2 * NBINS * 4), RADIX_CSORT};
    const int r = blockIdx.x;
    int n = (int)stride;
    if (row_lens) n = min(max(row_lens[r], 0), (int)stride);
    const float* x = scores + (int64_t)r * stride;
    int32_t* o = out + (int64_t)r * k;
    float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
    const RowGeom g = make_geom(x, n);
    int passes = 0, cand = 0, done = GVR_DONE_RADIX;

    if (n <= k) {
        small_row_emit(c, B, Wk, g, k, o, ov);
        passes = 1;
        cand = n;
        done = GVR_DONE_TRIVIAL;
    } else {
        const RadixResult rr = radix_select_global(c, Wk, g, (uint32_t)k, true);
        passes = rr.rounds + 1;
        if (!rr.exact) {
            // early exit: everything >= the bucket's lower bound fits (< K + 2048)
            int fill = 0;
            const uint32_t lb = rr.prefix;
            for_each_tile<RADIX_NT>(g, c.tid, [&](auto& tl, int) {
                commit_unordered(c, B, tl, [&](uint32_t kk) { return kk >= lb; }, fill);
                return 0;
            });
            c.sync();
            cand = fill;
            emit_sorted(c, B, Wk, fill, 0u, 0u, fill, k, k, o, ov);
        } else {
            cand = (int)(rr.above + rr.bucket);
            if (rr.above + rr.bucket <= (uint32_t)SORT_MAX) {
                int fill = 0;
                const uint32_t T = rr.prefix;
                for_each_tile<RADIX_NT>(g, c.tid, [&](auto& tl, int) {
                    commit_unordered(c, B, tl, [&](uint32_t kk) { return kk >= T; }, fill);
                    return 0;
                });
                c.sync();
                emit_sorted(c, B, Wk, fill, 0u, 0u, fill, k, k, o, ov);
            } else {
                tiefill_emit(c, B, Wk, g, rr.prefix, rr.above, k, k, o, ov);
            }
        }
    }
    if (stats && c.tid == 0) {
        gvr_row_stats s;
        s.secant_iters = 0;
        s.snap_iters = 0;
        s.cand_count = cand;
        s.done_kind = done;
        s.global_passes = passes;
        s.raises = 0;
        s.buffer_count = 0;
        s.cluster = 1;
        s.phase2_exit = GVR_P2_ALL;
        s.sample_count = 0;
        s.tc_key = 0u;
        s.reserved = 0;
        stats[r] = s;
    }
}

}  // namespace gvr
