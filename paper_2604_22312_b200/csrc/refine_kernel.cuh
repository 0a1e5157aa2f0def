// refine_kernel.cuh — the batch path's refine step: Phase 4 and the ordered output from the
// candidate lists gvr_filter_kernel leaves in L2.
//
// A persistent grid of four small CTAs per SM (37 KB of shared memory, <= 64 registers)
// launched behind the filter with programmatic dependent launch: one wave covers a decode
// batch, and CTAs that find room early start on the rows already complete.  CTAs pop rows
// from the ready queue in the // order their lists complete.  Per row (all of it exact key-space arithmetic):
//   * the row's <= F_SEGS list segments and their largest keys (filter records);
//   * Phase 4 fused with the ordered output (R28), over the
//     list itself, read from L2: a 2048-bin linear histogram of the keys >= T_c over
//     [T_c, kmax] (bin 0 = highest), the bin holding sorted position K-1 from the bin scan,
//     the entries of the bins up to it counting-sorted into shared memory as 64-bit
//     composites (key, ~index), each ranked inside its bin, and position j < K written to
//     out[j] — score descending, index ascending;
//   * rows this cannot finish — no tiles (len <= k or tiny rows), a list that overflowed its
//     region or holds fewer than K keys >= T_c (the guess overshot), a K-th bin crowded by
//     ties — go to the fixup list, worked off by gvr_topk_kernel in fixup mode.
// Phase 2 (the secant search) ran in gvr_guess_kernel over the row
// sample, so the list is {key >= T_c} with K <= f(T_c) ~ 1.3-2 K (R34-R36).
#pragma once
#ifdef GVR_DEBUG_BOUNDS
#include <cstdio>
#endif
#include "filter_kernel.cuh"

namespace gvr {

#ifndef GVR_RF_NBINS
#define GVR_RF_NBINS 2048
#endif
// (r2) Two geometries, chosen per call by the batch size (gvr_topk.cu): few rows — two
// 512-thread CTAs per SM, 8 held entries per thread (rows finish sooner); many rows — four
// 256-thread CTAs per SM, 16 held entries per thread (more rows in flight per SM).  Both
// hold 4,096 list entries per row in registers at 64 registers per thread.
template <int NT_, int HOLD_, int CPS_>
struct RefineGeo {
    static constexpr int NT = NT_;
    static constexpr int HOLD = HOLD_;
    static constexpr int CPS = CPS_;
};
using RefineFew = RefineGeo<512, 8, 2>;
using RefineMany = RefineGeo<256, 16, 4>;
constexpr int RF_MANY_ROWS = 1024;  // batches above this take RefineMany
constexpr int RF_NBINS = GVR_RF_NBINS;  // Phase-4 bins of the refine (finer than NBINS: shorter in-bin ranking)
constexpr int RF_CSORT = 2560;     // entries up to the K-th bin sorted in shared memory
constexpr int RF_MAXLIST = 1 << 22;  // longest list refined here
constexpr int RF_BIN_FAST = 16;    // largest bin ranked without narrowing first
constexpr int RF_ZOOM_MIN = 64;    // a lowest K-th bin above this is zoomed into from above
constexpr int RF_OFF_HIST = 0;                       // int32 bin counts
constexpr int RF_OFF_CUR = RF_OFF_HIST + RF_NBINS * 4;  // int32 bin cursors
constexpr int RF_OFF_CS = RF_OFF_CUR + RF_NBINS * 4;
constexpr int RF_PAD = 16;    // zero composites past the sorted prefix (fixed rank window)
constexpr int RF_OFF_ROW = RF_OFF_CS + (RF_CSORT + RF_PAD) * 8;
constexpr int RF_OFF_SCR = RF_OFF_ROW + 16;
constexpr int RF_SMEM_BYTES = RF_OFF_SCR + GROUP_SCRATCH_BYTES;
static_assert(RefineMany::CPS * (RF_SMEM_BYTES + 1024) <= 233472, "refine CTAs per SM");


// ---- Phase 4 over a row's list, instruction-lean (r2): the list is loaded once into
// registers (HOLD slots per thread: flat slot j = tid + NT u of the row's
// concatenated segments), every histogram level and the scatter run from the registers,
// and the shared-memory atomics are predicated instead of branched around.

// A row's list: its <= F_SEGS segments of the filter regions as one flat sequence.
// tab (shared memory, written by the records step): {p_s, o_s} per segment s — the
// first flat slot of segment s (a trailing empty segment starts at `total`) and region
// position minus flat slot.  map() copies it into registers for a batch of loads.
struct ListSrc {
    const uint2* region;
    const int32_t* tab;
    struct Map {
        const uint2* region;
        int o0, p1, o1, p2, o2, p3, o3;
        __device__ __forceinline__ uint2 load(int j) const
        {
            int pos = j + o0;
            pos = j >= p1 ? j + o1 : pos;
            pos = j >= p2 ? j + o2 : pos;
            pos = j >= p3 ? j + o3 : pos;
            return __ldcg(region + pos);
        }
    };
    __device__ __forceinline__ Map map() const
    {
        static_assert(F_SEGS == 4, "four list segments");
        const int4 t0 = reinterpret_cast<const int4*>(tab)[0], t1 = reinterpret_cast<const int4*>(tab)[1];
        return Map{region, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
    }
};
// A row with len <= k: the row itself (key, position).
struct RowSrc {
    const float* x;
    struct Map {
        const float* x;
        __device__ __forceinline__ uint2 load(int j) const { return make_uint2(f2key(__ldg(x + j)), (uint32_t)j); }
    };
    __device__ __forceinline__ Map map() const { return Map{x}; }
};

// floor(2^32 RF_NBINS / range), saturated: d -> floor(d scale / 2^32) maps [0, range) onto the bins
__device__ __forceinline__ uint32_t rf_scale(uint64_t range)
{
    const unsigned long long q = (((unsigned long long)RF_NBINS) << 32) / range;
    return q > 0xffffffffull ? 0xffffffffu : (uint32_t)q;
}
// Descending linear bin of key >= lo over [lo, lo + range): bin 0 holds the largest keys.
__device__ __forceinline__ int rbin(uint32_t key, uint32_t lo, uint32_t scale)
{
    // (unsigned clamp: after a zoom, keys far above the binned range give products >= 2^31)
    return (RF_NBINS - 1) - (int)min(__umulhi(key - lo, scale), (uint32_t)(RF_NBINS - 1));
}
__device__ __forceinline__ void red_inc_if(int32_t* p, bool pred)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.shared.add.u32 [%0], 1;\n\t}" ::"r"(smem_u32(p)),
                 "r"((uint32_t)pred)
                 : "memory");
}
// if pred: cs[cur[b]++] = (key << 32) | ~idx
__device__ __forceinline__ void scatter_if(int32_t* curb, unsigned long long* cs, uint32_t key, uint32_t idx, bool pred)
{
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 s, a;\n\tmov.u32 s, 0;\n\tsetp.ne.u32 q, %2, 0;\n\t"
        "@q atom.shared.add.u32 s, [%0], 1;\n\tshl.b32 a, s, 3;\n\tadd.u32 a, a, %1;\n\t"
        "@q st.shared.v2.u32 [a], {%3, %4};\n\t}" ::"r"(smem_u32(curb)),
        "r"(smem_u32(cs)), "r"((uint32_t)pred), "r"(~idx), "r"(key)
        : "memory");
}

// Phase 4 fused with the ordered output (R28, R32) over
// `total` entries of src, keys >= lo selected: 2048-bin linear histogram over
// [lo, kmax] (bin 0 = highest), the bin holding position take-1 from the bin scan,
// narrowing (<= 3 levels) when the bins up to it are crowded, then the entries up to
// that bin counting-sorted into cs as 64-bit composites and ranked inside their bins;
// position j < take goes to o[j] / ov[j].  Returns false (group-uniform) when the row
// cannot be finished here.  ftc = f(lo) of the first level; levels = histogram passes.
template <class Geo, class Src>
__device__ __forceinline__ bool refine_phase4(Group<Geo::NT, 1>& c, const Src& src, int total, uint32_t lo, uint32_t kmax,
                                              int take, int32_t* hist, int32_t* cur, unsigned long long* cs,
                                              int32_t* o, float* ov, int& ftc, int& levels, int& next_slot,
                                              int32_t* qhead, bool timing, long long (&ts)[TS_N])
{
    constexpr int BPT = RF_NBINS / Geo::NT;
    // held slots of this thread: u < nv
    const int nv = total > c.tid ? min(Geo::HOLD, (total - c.tid + Geo::NT - 1) / Geo::NT) : 0;
    uint2 e[Geo::HOLD];
    {
        const auto m = src.map();
#pragma unroll
        for (int u = 0; u < Geo::HOLD; ++u) e[u] = u < nv ? m.load(c.tid + u * Geo::NT) : make_uint2(0u, 0u);
    }
    uint32_t scale = 0u, off0 = 0u;
    uint32_t hi = kmax;  // binned range [lo, hi]; keys above hi saturate into bin 0
    const int b0 = c.tid * BPT;
    int h[BPT];
    int bk = -1, nsel = 0;
    bool ok = false;
    for (int lvl = 0; lvl < 3; ++lvl) {
        levels = lvl + 1;
#pragma unroll
        for (int i = 0; i < BPT / 4; ++i) reinterpret_cast<int4*>(hist + b0)[i] = make_int4(0, 0, 0, 0);
        if (c.tid == 0) {
            c.misc[12] = -1;  // K-th bin: set below by the thread that holds it
            c.misc[14] = (int)rf_scale((uint64_t)hi - lo + 1ull);  // one 64-bit division per level
        }
        c.sync();
        scale = (uint32_t)c.misc[14];
        uint32_t f = 0;
#pragma unroll
        for (int u = 0; u < Geo::HOLD; ++u) {
            if (u * Geo::NT >= total) break;  // group-uniform
            const bool in = u < nv && e[u].x >= lo;
#ifdef GVR_DEBUG_BOUNDS  // debug builds: every bin in range (nvcc -DGVR_DEBUG_BOUNDS)
            if (in && (rbin(e[u].x, lo, scale) < 0 || rbin(e[u].x, lo, scale) >= RF_NBINS)) {
                printf("refine: bin out of range, lo %u hi %u scale %u key %u\n", lo, hi, scale, e[u].x);
                __trap();
            }
#endif
            red_inc_if(hist + rbin(e[u].x, lo, scale), in);
            f += in ? 1u : 0u;
        }
        for (int j = c.tid + Geo::HOLD * Geo::NT; j < total; j += Geo::NT) {  // entries past the held slots
            const uint32_t kv = src.map().load(j).x;                       // (rare: lists > HOLD NT)
            red_inc_if(hist + rbin(kv, lo, scale), kv >= lo);
            f += kv >= lo ? 1u : 0u;
        }
        f = group_red1<R_ADD>(c, f);  // its barrier also completes the histogram
        if (lvl == 0) {
            ftc = (int)f;
            if (timing) ts[TS_STREAM] = clock64();
        }
        uint32_t loc = 0;
#pragma unroll
        for (int i = 0; i < BPT / 4; ++i) {
            const int4 hv = reinterpret_cast<const int4*>(hist + b0)[i];
            h[4 * i] = hv.x, h[4 * i + 1] = hv.y, h[4 * i + 2] = hv.z, h[4 * i + 3] = hv.w;
        }
#pragma unroll
        for (int i = 0; i < BPT; ++i) loc += (uint32_t)h[i];
        uint32_t lmx = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) lmx = max(lmx, (uint32_t)h[i]);
        uint32_t tot, mx_before;
        off0 = group_excl_scan_pmax(c, loc, lmx, tot, mx_before);
        {
            // the thread holding position take-1 also knows the largest bin up to it
            uint32_t off = off0, m = mx_before;
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                m = max(m, (uint32_t)h[i]);
                if ((uint32_t)(take - 1) >= off && (uint32_t)(take - 1) < off + (uint32_t)h[i]) {
                    c.misc[12] = b0 + i;
                    c.misc[13] = (int)(off + (uint32_t)h[i]);
                    c.misc[15] = (int)m;
                    c.misc[16] = h[i];
                }
                off += (uint32_t)h[i];
            }
        }
        c.sync();
        bk = ftc >= take ? c.misc[12] : -1;
        nsel = c.misc[13];
        const uint32_t mx = bk >= 0 ? (uint32_t)c.misc[15] : 0u;
        ok = bk >= 0 && nsel <= RF_CSORT && mx <= (uint32_t)CSORT_BIN_MAX;  // group-uniform
        // narrow also when the ranking would loop over bins of more than RF_BIN_FAST
        if (bk < 0 || lvl == 2 || (ok && mx <= (uint32_t)RF_BIN_FAST)) break;
        // lower edge of bin bk: the smallest d with floor(d scale / 2^32) = RF_NBINS - 1 - bk
        const uint64_t L = (uint64_t)(RF_NBINS - 1 - bk);
        const uint64_t dmin = ((L << 32) + scale - 1ull) / scale;
        if (dmin == 0ull) {
            // the K-th bin is the lowest.  Moderately crowded: ranked as it is.  Heavily
            // crowded (a few keys far above the rest stretch the range): zoom into that bin
            // from above (its top edge becomes hi; the keys above saturate into bin 0)
            // (only when the keys above that bin are few: they all land in bin 0)
            if (mx <= (uint32_t)RF_ZOOM_MIN || nsel - c.misc[16] > RF_PAD) break;
            const uint64_t dtop = ((1ull << 32) + scale - 1ull) / scale;  // first d of the next bin up
            if (dtop <= 1ull) break;
            hi = lo + (uint32_t)(dtop - 1ull);
            continue;
        }
        lo += (uint32_t)dmin;
    }
    if (timing) ts[TS_PHASE23] = clock64();
    if (!ok) return false;
    {
        // bin starts; they become the bin ends after the scatter
        int st[BPT];
        int off = (int)off0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            st[i] = off;
            off += h[i];
        }
#pragma unroll
        for (int i = 0; i < BPT / 4; ++i)
            reinterpret_cast<int4*>(cur + b0)[i] = make_int4(st[4 * i], st[4 * i + 1], st[4 * i + 2], st[4 * i + 3]);
    }
    if (c.tid < RF_PAD) cs[nsel + c.tid] = 0ull;  // the rank window may run past the last bin
    c.sync();
    // ---- counting sort of the bins up to the K-th bin (composites)
#pragma unroll
    for (int u = 0; u < Geo::HOLD; ++u) {
        if (u * Geo::NT >= total) break;
        const int b = rbin(e[u].x, lo, scale);
        scatter_if(cur + b, cs, e[u].x, e[u].y, u < nv && e[u].x >= lo && b <= bk);
    }
    for (int j = c.tid + Geo::HOLD * Geo::NT; j < total; j += Geo::NT) {
        const uint2 x = src.map().load(j);
        const int b = rbin(x.x, lo, scale);
        scatter_if(cur + b, cs, x.x, x.y, x.x >= lo && b <= bk);
    }
    c.sync();
#ifdef GVR_DEBUG_BOUNDS  // debug builds: the scatter filled every bin up to the K-th exactly
    {
        int off = (int)off0;
        for (int i = 0; i < BPT; ++i) {
            if (b0 + i <= bk && cur[b0 + i] != off + h[i]) {
                printf("refine: bin %d filled to %d, expected %d\n", b0 + i, cur[b0 + i], off + h[i]);
                __trap();
            }
            off += h[i];
        }
    }
#endif
    if (timing) ts[TS_PHASE4] = clock64();
    if (c.tid == 0 && qhead) next_slot = atomicAdd(qhead, 1);
    // ---- rank inside the bin; positions < take are the ordered output.  Bins are
    // contiguous in cs in descending key order, so counting the larger composites over a
    // fixed window from the bin start (later bins and the zero padding are all smaller)
    // ranks every entry of a bin of at most RF_PAD entries without a per-compare bound.
    auto rank_of = [&](int j, unsigned long long& v) -> int {
        v = cs[j];
        const int b = rbin(comp_key(v), lo, scale);
        const int cnt = hist[b];
        const int st = cur[b] - cnt;
        const int wmax = (int)__reduce_max_sync(__activemask(), (uint32_t)cnt);
        int rank = 0;
        if (wmax <= RF_PAD) {
#pragma unroll
            for (int t = 0; t < RF_PAD; t += 4) {
                if (t >= wmax) break;
                rank += (cs[st + t] > v ? 1 : 0) + (cs[st + t + 1] > v ? 1 : 0) + (cs[st + t + 2] > v ? 1 : 0) +
                        (cs[st + t + 3] > v ? 1 : 0);
            }
        } else {
            for (int t = 0; t < cnt; ++t) rank += cs[st + t] > v ? 1 : 0;
        }
        return st + rank;
    };
    if (ov) {
        for (int j = c.tid; j < nsel; j += Geo::NT) {
            unsigned long long v;
            const int pos = rank_of(j, v);
            if (pos < take) {
                o[pos] = comp_idx(v);
                ov[pos] = key2f(comp_key(v));
            }
        }
    } else {
        for (int j = c.tid; j < nsel; j += Geo::NT) {  // indices only: one predicated store
            unsigned long long v;
            const int pos = rank_of(j, v);
            asm volatile("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %1, %2;\n\t@q st.global.b32 [%0], %3;\n\t}" ::"l"(o + pos),
                         "r"(pos), "r"(take), "r"(comp_idx(v))
                         : "memory");
        }
    }
    return true;
}

template <bool TIMING, class Geo>
__global__ void __launch_bounds__(Geo::NT, Geo::CPS)
gvr_refine_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                  int num_rows, int32_t* out, float* out_val, gvr_row_stats* stats, const GuessOut* gp, CandLists cl,
                  BatchQueue bq, long long* phase_ts, bool fused = false, int32_t* ctl = nullptr)
{
    // the fixup grid may be scheduled now: it waits for this grid's release flag (ctl)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // fused (the indexer path, indexer_kernel.cuh): the score rows do not exist, so rows
    // that need them — len <= k, the ties fill — go to the fixup list, which materialises them
    // phase_ts (optional, [num_rows][TS_N]): clock64 at the pop, after the segment records,
    // after the histogram pass, after the K-th bin search, after the scatter, at the end;
    // then globaltimer at the pop and the end, and the SM id.
    extern __shared__ __align__(128) unsigned char smem[];
    int32_t* hist = reinterpret_cast<int32_t*>(smem + RF_OFF_HIST);
    int32_t* cur = reinterpret_cast<int32_t*>(smem + RF_OFF_CUR);
    unsigned long long* cs = reinterpret_cast<unsigned long long*>(smem + RF_OFF_CS);
    int* sh_row = reinterpret_cast<int*>(smem + RF_OFF_ROW);
    Group<Geo::NT, 1> c;
    c.init(threadIdx.x, smem + RF_OFF_SCR);
    const int K = k;
    // thread 0 claims the next queue slot during the current row's last step (ranking),
    // so the claim's round trip is off the critical path without hoarding rows early
    int next_slot = -1;
    for (;;) {
        if (c.tid == 0) {
            const int slot = next_slot >= 0 ? next_slot : atomicAdd(bq.qctl + Q_HEAD, 1);
            next_slot = -1;
            int r = -1;
            if (slot < num_rows) {
                int v;
                while ((v = ld_acquire(bq.queue + slot)) == 0) __nanosleep(100);
                r = v - 1;
                bq.queue[slot] = 0;
            }
            *sh_row = r;
        }
        c.sync();
        const int r = *sh_row;
        if (r < 0) break;
        const bool timing = TIMING && phase_ts != nullptr;  // (the TIMING=false instance has no stamps)
        long long tsr[TS_N] = {timing ? clock64() : 0ll, 0, 0, 0, 0, 0, timing ? global_ns() : 0ll, 0, 0};
        // the segment records, the row length and T_c are loaded together (the records of
        // slots past the row's segment count are stale and ignored)
        const int4 erec = c.warp == 0 && c.lane < F_SEGS ? __ldcg(cl.rec + (long long)r * F_SEGS + c.lane)
                                                         : make_int4(0, 0, 0, 0);
        const uint4 g0 = __ldcg(reinterpret_cast<const uint4*>(gp + r));      // Tc, tie, tmin, top
        const uint4 g1 = __ldcg(reinterpret_cast<const uint4*>(gp + r) + 1);  // T0, iters | exit, ...
        uint32_t Tc = g0.x;
        const uint32_t tie = g0.y;
        const RowPlan p = plan_row(scores, stride, row_lens, r, k);
        // ---- the row's list segments (filter records)
        int total = -1;
        uint32_t kmax = 0u;
        if (p.ntiles > 0 && c.warp == 0) {
            const long long v0 = (long long)r * cl.tpr;
            const int b0 = cl_cta_of(cl, v0);
            const int ns = cl_cta_of(cl, v0 + p.ntiles - 1) - b0 + 1;
            int gsv = 0, n = 0, bad = ns > F_SEGS ? 1 : 0;
            uint32_t km = 0u;
            if (c.lane < ns && c.lane < F_SEGS) {
                const int4 e = erec;
                bad = (e.x != b0 + c.lane || e.y < 0 || e.z < e.y || e.z > cl.reg) ? 1 : 0;
                gsv = e.x * cl.reg + e.y;
                n = e.z - e.y;
                km = (uint32_t)e.w;
            }
            bad = __any_sync(FULL, bad);
            const int tot = (int)__reduce_add_sync(FULL, (uint32_t)n);
            km = __reduce_max_sync(FULL, km);
            // the flat-slot table of the list (ListSrc): segment s starts at flat slot
            // p_s = n_0 + ... + n_{s-1}; its region positions are flat slot + o_s
            uint32_t ps = n;
#pragma unroll
            for (int o = 1; o < F_SEGS; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, ps, o);
                if (c.lane >= o) ps += y;
            }
            ps -= (uint32_t)n;
            if (c.lane < F_SEGS) {
                c.misc[24 + 2 * c.lane] = (int)ps;
                c.misc[25 + 2 * c.lane] = gsv - (int)ps;
            }
            if (c.lane == 0) {
                c.misc[22] = bad ? -1 : tot;
                c.misc[23] = (int)km;
                bq.segdone[r] = 0;  // popped: reset for the next call
            }
        }
        c.sync();
        if (p.ntiles > 0) {
            total = c.misc[22];
            kmax = (uint32_t)c.misc[23];
        }
        bool ok = p.ntiles > 0 && p.n > k && total >= K && total <= RF_MAXLIST && kmax >= Tc;
        // a Phase-2 ties exit collected the keys strictly above the tied key (R37): when
        // they are fewer than K, all of them lead the output and the tie's lowest indices
        // follow (an ordered scan of the row below)
        const int p2exit = (int)(int16_t)(g1.y >> 16);
        const bool tie_fill = p.ntiles > 0 && p.n > k && p2exit == GVR_P2_TIES && tie < 0xffffffffu &&
                              Tc == tie + 1u && total >= 0 && total < K;
        if (tie_fill) ok = !fused && (total == 0 || kmax >= Tc);
        // a row with len <= k: every element is selected (take = len), binned over its own
        // key range [min, max], then -1 padding (R5)
        const bool trivial = p.n <= k;
        const float* rowx = nullptr;
        int take = tie_fill ? total : K;
        if (trivial && fused) ok = false;
        if (trivial && !fused) {
            uint32_t mn = 0xffffffffu, mx2 = 0u;
            for (int q = c.tid; q < p.n; q += Geo::NT) {
                const uint32_t kv = f2key(__ldg(p.x + q));
                mn = min(mn, kv);
                mx2 = max(mx2, kv);
            }
            group_red2<R_MIN, R_MAX>(c, mn, mx2);
            rowx = p.x;
            total = p.n;
            take = p.n;
            Tc = mn;
            kmax = mx2;
            ok = p.n > 0;
        }
        if (timing) tsr[TS_PHASE1] = clock64();
        int ftc = 0, levels = 0;
        if (ok && take > 0) {
            int32_t* o = out + (int64_t)r * k;
            float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
            if (rowx) {
                ok = refine_phase4<Geo>(c, RowSrc{rowx}, total, Tc, kmax, take, hist, cur, cs, o, ov, ftc, levels,
                                   next_slot, bq.qctl + Q_HEAD, timing, tsr);
            } else {
                ok = refine_phase4<Geo>(c, ListSrc{cl.region, c.misc + 24}, total, Tc, kmax, take, hist, cur, cs, o, ov, ftc, levels, next_slot,
                                   bq.qctl + Q_HEAD, timing, tsr);
            }
            if (ok && !tie_fill)
                for (int j = take + c.tid; j < k; j += Geo::NT) {  // len < k: -1 padding
                    o[j] = -1;
                    if (ov) ov[j] = 0.f;
                }
        }
        if (ok && tie_fill) {
            // positions [take, K): the first K - take elements of the row equal to the tied
            // key, in index order — thread t scans 8 consecutive elements per step, an
            // exclusive scan orders the matches; fewer than needed: the tie is not the K-th
            // key after all and the row goes to the fixup list
            int32_t* o = out + (int64_t)r * k;
            float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
            const int need = K - take;
            int found = 0;
            for (int base = 0; base < p.n && found < need; base += 8 * Geo::NT) {
                const int i0 = base + 8 * c.tid;
                uint32_t hit = 0u;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (i0 + j < p.n && f2key(__ldg(p.x + i0 + j)) == tie) hit |= 1u << j;
                uint32_t tot;
                uint32_t pos = (uint32_t)(take + found) + group_excl_scan(c, (uint32_t)__popc(hit), tot);
                for (; hit; hit &= hit - 1u, ++pos)
                    if (pos < (uint32_t)K) {
                        o[pos] = i0 + __ffs(hit) - 1;
                        if (ov) ov[pos] = key2f(tie);
                    }
                found += (int)tot;
            }
            ok = found >= need;
            levels = 0;
            ftc = total;
        }
        if (trivial && p.n == 0 && !fused) {
            int32_t* o = out + (int64_t)r * k;
            for (int j = c.tid; j < k; j += Geo::NT) {
                o[j] = -1;
                if (out_val) out_val[(int64_t)r * k + j] = 0.f;
            }
            ok = true;
        }
        if (c.tid == 0) {
            if (!ok) {
                // a complete list with fewer than K keys >= T_c: the fixup streams the row at
                // the second-pass threshold directly (flag bit 31)
                const bool short_list = p.ntiles > 0 && p.n > k && total >= 0 && total < K;
                bq.fixlist[atomicAdd(bq.qctl + Q_NFIX, 1)] = (int32_t)((uint32_t)r | (short_list ? 0x80000000u : 0u));
            } else if (stats) {
                const GuessOut g = trivial ? GuessOut{} : gp[r];
                gvr_row_stats s;
                s.secant_iters = g.iters;  // Phase-2 probes (gvr_guess_kernel)
                s.snap_iters = 0;
                s.cand_count = trivial ? p.n : ftc;
                s.done_kind = trivial ? GVR_DONE_TRIVIAL : tie_fill ? GVR_DONE_TIEFILL : GVR_DONE_CONVERGED;
                s.global_passes = tie_fill ? 2 : 1;  // the tie scan reads (part of) the row again
                s.raises = levels > 1 ? levels - 1 : 0;  // Phase-4 histogram narrowings (R32)
                s.buffer_count = trivial ? 0 : ftc;
                s.cluster = 1;
                s.phase2_exit = g.exit;
                s.sample_count = g.scount;
                s.tc_key = g.Tc;
                s.reserved = 0;
                stats[r] = s;
            }
            if (timing && ok) {
                tsr[TS_END] = clock64();
                tsr[TS_GEND] = global_ns();
                tsr[TS_SMID] = sm_id();
                for (int i = 0; i < TS_N; ++i) phase_ts[(int64_t)r * TS_N + i] = tsr[i];
            }
        }
        c.sync();  // smem (row slot, histogram, sort buffer) is reused for the next row
    }
    // the last CTA to finish releases the fixup grid (its list is complete)
    if (c.tid == 0 && ctl) {
        __threadfence();
        if (atomicAdd(bq.qctl + Q_RDONE, 1) == (int)gridDim.x - 1) {
            __threadfence();
            st_release(ctl + CTL_RDONE, 1);
        }
    }
}

}  // namespace gvr
