// filter_kernel.cuh — the batch path's streaming step.
//
// For batches of more than one wave the row-per-CTA streaming kernel loses a third of its
// time to things that are not streaming: each CTA's ring sits idle while it refines its
// row (Phases 2-4, ~15K cycles), and R rows on 2 x 148 slots leave a partial last wave.
// This kernel does only the HBM pass.  The batch's row bodies, cut into 16 KB tiles, form
// one virtual tile sequence (tpr tiles per row, rows shorter than row_stride leave empty
// virtual tiles); a persistent grid of G CTAs (3 per SM) takes contiguous, equal ranges of
// it, so every SM streams until the end and a row is covered by at most F_SEGS CTAs.
// Each CTA pulls its range through a TMA ring (two rounds of 2 x 16 KB), tests every
// element against its row's collect threshold T_c (Phase 1 output, gvr_guess_kernel)
// and appends the candidates — (sortable key, row index) — to its own region of global
// memory: the warp's inclusive scan of its pass counts and one shared atomicAdd per warp
// give every lane its write positions (ballot-free), and the writes go
// straight from the lanes to L2, with no shared staging and no global atomics.  At the end
// of each row segment the CTA records (cta, start, end) of that row's entries in its
// region; the refine step (gvr_refine_kernel) gathers a row's <= F_SEGS
// segments, and Lemma 1 makes {key >= T_c} enough for the exact Top-K
// whenever it holds at least K entries.
#pragma once
#include "gvr_kernel.cuh"

namespace gvr {

constexpr int F_NT = 256;
constexpr int F_CTAS_PER_SM = 3;   // 24 warps per SM: the collect loop is issue-latency bound
constexpr int F_ROUNDS = 2;        // rounds in flight: 64 KB of the row per CTA
constexpr int F_NSTAGE = F_ROUNDS * ROUND_STAGES;
constexpr int F_REG_MIN = 16384;   // smallest per-CTA candidate region (entries)
using FilterGroup = Group<F_NT, 1>;

constexpr int F_OFF_RING = 0;
constexpr int F_OFF_BARS = F_NSTAGE * STAGE_BYTES;
constexpr int F_OFF_CUR = F_OFF_BARS + F_NSTAGE * 8;  // region cursor, segment kmax
constexpr int F_OFF_SCR = F_OFF_CUR + 16;
constexpr int F_SMEM_BYTES = F_OFF_SCR + GROUP_SCRATCH_BYTES;
static_assert(F_CTAS_PER_SM * (F_SMEM_BYTES + 1024) <= 233472, "three filter CTAs per SM");

// Rounds of one CTA's range: up to two consecutive tiles of one row (a round always
// occupies two ring stages; a one-tile round arms its second stage with zero bytes so the
// stage phases stay in step).  Virtual tiles past a row's real tiles are skipped.
struct RoundIter {
    long long v, ve;
    int r, t;            // row and tile of virtual position v (tracked incrementally)
    int loaded = -1;     // row whose plan p holds
    RowPlan p;
    int t0 = 0, nt = 0;
    bool last = false;  // last round of this CTA's segment of row r
    __device__ __forceinline__ void start(long long vb, long long vend, int tpr)
    {
        v = vb;
        ve = vend;
        r = (int)(vb / tpr);
        t = (int)(vb - (long long)r * tpr);
    }
    __device__ __forceinline__ bool next(const float* scores, int64_t stride, const int32_t* row_lens, int k, int tpr)
    {
        while (v < ve) {
            if (loaded != r) {
                loaded = r;
                p = plan_row(scores, stride, row_lens, r, k);
            }
            if (t >= p.ntiles) {  // past the row's real tiles: on to the next row
                v += tpr - t;
                ++r;
                t = 0;
                continue;
            }
            t0 = t;
            nt = (int)min((long long)min(ROUND_STAGES, p.ntiles - t), ve - v);
            v += nt;
            t += nt;
            last = t >= p.ntiles || v >= ve;
            return true;
        }
        return false;
    }
};

// Candidate store with an L2 evict-last hint: the lists are re-read by the refine kernel
// right after the stream, whose own tiles are loaded evict-first.
__device__ __forceinline__ void st_cand(uint2* p, uint32_t key, uint32_t idx, uint64_t pol)
{
    asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(key), "r"(idx), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void issue_tile(const Ring& ring, const RowPlan& p, int t, int s)
{
    const uint32_t bytes = (uint32_t)min(STAGE_FLOATS, p.nfl - t * STAGE_FLOATS) * 4u;
    mbar_arrive_expect_tx(ring.full(s), bytes);
    bulk_g2s(smem_u32(ring.stage(s)), p.x + p.head + (size_t)t * STAGE_FLOATS, bytes, ring.full(s), ring.policy);
}

// thread 0: load round i (tiles it.t0 .. it.t0 + it.nt - 1 of row it.r) into its stage pair
__device__ __forceinline__ void issue_pair(const Ring& ring, const RoundIter& it, int i)
{
    const int s0 = ROUND_STAGES * (i % F_ROUNDS);
    issue_tile(ring, it.p, it.t0, s0);
    if (it.nt == 2)
        issue_tile(ring, it.p, it.t0 + 1, s0 + 1);
    else
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ring.full(s0 + 1)) : "memory");
}

__global__ void __launch_bounds__(F_NT, F_CTAS_PER_SM)
gvr_filter_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                  const GuessOut* __restrict__ gp, CandLists cl, BatchQueue bq)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const Ring ring{reinterpret_cast<float*>(smem + F_OFF_RING), reinterpret_cast<uint64_t*>(smem + F_OFF_BARS),
                    policy_evict_first()};
    int* cursor = reinterpret_cast<int*>(smem + F_OFF_CUR);
    uint32_t* seg_kmax = reinterpret_cast<uint32_t*>(smem + F_OFF_CUR + 4);
    FilterGroup c;
    c.init(threadIdx.x, smem + F_OFF_SCR);
    const int b = blockIdx.x;
    // diagnostics: stamps kept in registers, stored at exit if recording is on (the flag is
    // read last, off the critical path)
    const long long ts_entry = global_ns();
    long long ts_wait = 0;
    const long long vb = cl_begin(cl, b), ve = cl_begin(cl, b + 1);
    RoundIter prod;  // thread 0: two rounds ahead of the consumers
    prod.start(vb, ve, cl.tpr);
    int issued = 0;
    if (c.tid == 0) {
        for (int s = 0; s < F_NSTAGE; ++s) mbar_init(ring.full(s), 1);
        fence_mbar_init();
        *cursor = 0;
        *seg_kmax = 0u;
        // the row data does not depend on Phase 1: start the stream before waiting for it
        for (; issued < F_ROUNDS && prod.next(scores, stride, row_lens, k, cl.tpr); ++issued)
            issue_pair(ring, prod, issued);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // (r2) no wait for the whole Phase-1/2 grid: each row's threshold is taken from its
    // hand-off word (BatchQueue::tcw) once the guess kernel has published it
    const bool per_row = bq.tcw != nullptr;
    if (!per_row) asm volatile("griddepcontrol.wait;" ::: "memory");  // gp is complete and visible
    const uint32_t gen = per_row ? *bq.gen + 1u : 0u;
    c.sync();
    uint2* reg = cl.region + (long long)b * cl.reg;
    const int regcap = cl.reg;
    const uint64_t keep = policy_evict_last();
    RoundIter it;
    it.start(vb, ve, cl.tpr);
    const int lb = lane_base(c.warp, c.lane);
    int cur_r = -1, seg_start = 0;
    float Tf = 0.f;
    // T_c of the row after the current one, loaded a whole segment ahead of its use
    const int r_first = it.r;
    const int nrows = (int)(cl.V / cl.tpr);
    // row r's threshold from a (possibly early) read v of its hand-off word: spin until the
    // word carries this call's generation (acquire; the guess kernel stores it with release)
    auto tc_of = [&](int r, unsigned long long v) -> uint32_t {
        if (!per_row) return __ldcg(&gp[r].Tc);
        while ((uint32_t)(v >> 32) != gen) {
            __nanosleep(64);
            v = ld_acquire_u64(bq.tcw + r);
        }
        return (uint32_t)v;
    };
    auto tc_peek = [&](int r) -> unsigned long long { return per_row ? ld_relaxed_u64(bq.tcw + r) : 0ull; };
    unsigned long long tc_next = r_first < nrows ? tc_peek(r_first) : 0ull;
    uint32_t kmax = 0u;  // this thread's largest candidate key in the current segment
    for (int i = 0; it.next(scores, stride, row_lens, k, cl.tpr); ++i) {
        const RowPlan& p = it.p;
        if (it.r != cur_r) {
            const bool first = cur_r < 0;
            const uint32_t tc = tc_of(it.r, it.r == (first ? r_first : cur_r + 1) ? tc_next : tc_peek(it.r));
            if (first) ts_wait = global_ns();
            cur_r = it.r;
            Tf = key2f(tc);
            if (cur_r + 1 < nrows) tc_next = tc_peek(cur_r + 1);
        }
        // unaligned head scalars (round holding tile 0) and tail scalars (round holding the
        // last tile), loaded before the wait so their latency hides behind it
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
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 v = *reinterpret_cast<const float4*>(sp + lb + 128 * j);
            mask |= (uint32_t)pass_ge(v.x, Tf) << (4 * j);
            mask |= (uint32_t)pass_ge(v.y, Tf) << (4 * j + 1);
            mask |= (uint32_t)pass_ge(v.z, Tf) << (4 * j + 2);
            mask |= (uint32_t)pass_ge(v.w, Tf) << (4 * j + 3);
        }
        if (nf != ROUND_FLOATS) {
            uint32_t vm = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (lb + 128 * j < nf) vm |= 0xfu << (4 * j);
            mask &= vm;
        }
        const uint32_t cnt = (uint32_t)__popc(mask);
        const uint32_t incl = warp_incl_scan(cnt, c.lane);
        const uint32_t wtot = __shfl_sync(FULL, incl, 31);
        int base = 0;
        if (c.lane == 31 && wtot) base = atomicAdd(cursor, (int)wtot);
        base = __shfl_sync(FULL, base, 31);
        int pos = base + (int)(incl - cnt);
        const int ibase = p.idx0 + p.head + it.t0 * STAGE_FLOATS + lb;
        while (mask) {
            const int e = 31 - __clz(mask);
            mask ^= 1u << e;
            const int o = rel_off(e);
            const uint32_t u = __float_as_uint(sp[lb + o]);
            const uint32_t kv = u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);  // f2key
            if (pos < regcap) st_cand(reg + pos, kv, (uint32_t)(ibase + o), keep);
            kmax = max(kmax, kv);
            ++pos;
        }
        if (si >= 0 && pass_ge(sv, Tf)) {
            const int q = atomicAdd(cursor, 1);
            const uint32_t kv = f2key(sv);
            if (q < regcap) st_cand(reg + q, kv, (uint32_t)(p.idx0 + si), keep);
            kmax = max(kmax, kv);
        }
        if (it.last) {
            // end of this CTA's segment of row r: the segment's largest key, and every
            // thread's candidate writes ordered before the segment is counted as done
            const uint32_t wk = __reduce_max_sync(FULL, kmax);
            if (c.lane == 0 && wk) atomicMax(seg_kmax, wk);
            kmax = 0u;
        }
        c.sync();  // the round's stages are consumed and its reservations made
        if (c.tid == 0 && prod.next(scores, stride, row_lens, k, cl.tpr)) issue_pair(ring, prod, i + F_ROUNDS);
        if (it.last) {
            // record where the segment's entries are; the CTA finishing the row's last
            // segment puts the row in the ready queue of gvr_refine_kernel
            if (c.tid == 0) {
                const int end = *cursor;
                const long long v0 = (long long)cur_r * cl.tpr;
                const int b0 = cl_cta_of(cl, v0);
                cl.rec[(long long)cur_r * F_SEGS + (b - b0)] = make_int4(b, seg_start, end, (int)*seg_kmax);
                *seg_kmax = 0u;
                seg_start = end;
                if (bq.queue) {
                    const int ns = cl_cta_of(cl, v0 + p.ntiles - 1) - b0 + 1;
                    // the round barrier ordered every thread's candidate stores before this
                    // point; the fence makes them (and the record) visible device-wide
                    // before the count (the grid-barrier release pattern)
                    __threadfence();
                    if (atomicAdd(bq.segdone + cur_r, 1) == ns - 1) {
                        __threadfence();  // the other segments' records and entries happen-before the push
                        st_release(bq.queue + atomicAdd(bq.qctl + Q_TAIL, 1), cur_r + 1);
                    }
                }
            }
            c.sync();  // no reservation of the next segment before the cursor was read
        }
    }
    if (c.tid == 0 && b < FTS_MAX && *(volatile int*)&g_fts_on) {
        g_fts[b][0] = ts_entry;
        g_fts[b][1] = ts_wait;
        g_fts[b][2] = global_ns();
        g_fts[b][3] = sm_id();
    }
}

}  // namespace gvr
