// gvr_kernel.cuh — Guess-Verify-Refine exact Top-K on sm_100a.
//
// One CTA of 256 threads per row, two CTAs per SM (115.6 KB of shared memory each), so
// one CTA streams while the other evaluates its guess or refines.
//
// Method: PAPER.md Sec. 4 (lines 379-690).  Per row:
//   Phase 1 (Guess): x at the previous step's Top-K positions ->
//     pmin / pmax / pmean (Eq. 4).
//   Phase 2: the secant search of Eq. 6 for a collect threshold T_c
//     whose count lies in a target window — T0 = pmean first, then the Phase-1 bracket
//     end on the far side, then Eq.-6 steps (first one damped <= 0.5, key-space bisection
//     at float precision limits).  Each count f(T) is taken over a fixed 4096-value row
//     sample held in registers (16 contiguous floats per thread), not over the row in
//     HBM: the window is the sample image of [K, C] with a margin that keeps
//     f(T_c) >= K (R34-R36).  Phases 1-2 run in gvr_guess_kernel on the batch
//     paths and inside the row's CTA on the fused / cluster paths (phase12()).
//   Streaming pass (B200 re-design of the Phase-3 collector): the row
//     body is read from HBM exactly once, in rounds of 2 x 16 KB TMA tiles; every element
//     whose key is >= T_c is appended to B (warp scan + one shared atomic per warp:
//     ballot-free).  B holds {x >= T_c}, so f(T) for every T >= T_c is
//     counted from B alone (Lemma 1).  If B would overflow, T_c is
//     raised by a key-space histogram search over B (R23) to a threshold that still keeps
//     >= K elements.
//   Phase 3: ballot-free compaction of B to {x >= T} reusing the
//     per-thread counts of the last count pass (count cache).
//   Phase 4: 2048-bin histogram over the candidate key range,
//     warp-parallel K-th-bin search, snap iterations (count_ge, count_gt, snap_up,
//     snap_down) until n>(T) < K <= n>=(T) — run by one warp over the K-th bin's members
//     (every snap step stays inside that bin, so T* and the step count equal a scan over
//     all candidates); exact narrowing of the bin if it is too large.
//   Ordered output: candidates >= T* sorted by (key desc, index asc), first K written.
//   Fallbacks (R12/R13): massive ties or an
//     overshooting threshold (f(T_c) < K) -> a second stream at a lower threshold, exact
//     radix select + ordered tie fill from global memory.
#pragma once
#include <cooperative_groups.h>

#include "pipeline.cuh"
#include "select_global.cuh"

namespace gvr {

struct GvrParams {
    float window_z;  // Phase-2 window lower edge: mu + z sqrt(mu) sample hits (R35)
    int max_secant;  // secant steps before pure bisection (R11)
    int guess_stride;  // Phase-1 statistics over every guess_stride-th guessed position (R29)
};

constexpr int GVR_NT = 256;
constexpr int GVR_CAP = 6016;   // candidate buffer capacity (C = 6144 less the raise histogram)
constexpr int RAISE_BINS = 256;  // raise_threshold histogram (one bin per thread)
constexpr int GVR_CSORT = SORT_MAX;  // counting-sort capacity (K plus ties at T*)
using GvrGroup = Group<GVR_NT, 1>;

// Shared-memory layout (dynamic).  The refine work area aliases the ring, which is idle
// once the stream is done.
constexpr int G_OFF_RING = 0;
constexpr int G_OFF_B = G_OFF_RING + NSTAGE * STAGE_BYTES;  // {key[CAP], idx[CAP]}
constexpr int G_OFF_WORK = G_OFF_RING;
constexpr int G_OFF_RHIST = G_OFF_B + GVR_CAP * 8;          // raise histogram [RAISE_BINS]
constexpr int G_OFF_BARS = G_OFF_RHIST + RAISE_BINS * 4;    // full[NSTAGE]
constexpr int G_OFF_SCR = G_OFF_BARS + NSTAGE * 8;
constexpr int GVR_SMEM_BYTES = G_OFF_SCR + GROUP_SCRATCH_BYTES;
static_assert(work_bytes(GVR_CSORT) <= NSTAGE * STAGE_BYTES, "work area fits in the ring");
static_assert(GVR_SMEM_BYTES + 1024 <= 233472 / 2, "two CTAs per SM");
static_assert(GVR_CAP >= 2 * KMAX && GVR_CAP <= NCHUNK_MAX * CHUNK_SLOTS * GVR_NT, "buffer capacity");
static_assert(GVR_CAP * 8 >= SORT_MAX * 8, "bitonic fallback aliases the buffer");
static_assert(ROUND_FLOATS == 32 * GVR_NT, "32 elements per thread per round");
static_assert(RAISE_BINS == GVR_NT, "one raise bin per thread");

// Phase timestamps (written when phase_ts != nullptr): the paper's GVR_PHASE_TIMING
// instrumentation.
enum { TS_START = 0, TS_PHASE1, TS_STREAM, TS_PHASE23, TS_PHASE4, TS_END, TS_GSTART, TS_GEND, TS_SMID, TS_N };

__device__ __forceinline__ long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return (long long)t;
}
__device__ __forceinline__ long long sm_id()
{
    uint32_t s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return (long long)s;
}

// Diagnostics (gvr_cta_timeline), recorded while g_fts_on is set: per gvr_filter_kernel CTA
// b < FTS_MAX globaltimer at entry, after the Phase-1/2 wait and at exit, and its SM id;
// per gvr_guess_kernel CTA (row) globaltimer at entry and exit and its SM id.
constexpr int FTS_MAX = 4096;
__device__ int g_fts_on;
__device__ long long g_fts[FTS_MAX][4];
__device__ long long g_gts[FTS_MAX][4];

// What Phases 1-2 (phase12) hand to the streaming step, per row (32 bytes).
struct GuessOut {
    uint32_t Tc;     // collect threshold key (Phase 2 result)
    uint32_t tie;    // Phase-2 ties exit: the tied sample key (the lo anchor), else 0
    uint32_t tmin;   // second-pass threshold: pmin when all k guesses were gathered and
                     // valid (then f(pmin) >= k for distinct guesses), else 0 (everything)
    uint32_t top;    // max(pmax, sample max) key
    uint32_t T0;     // f2key(pmean), the Phase-2 start
    int16_t iters;   // Phase-2 probes I
    int16_t exit;    // gvr_phase2_exit
    int32_t scount;  // sample hits at T_c
    int32_t t0_ok;   // pmean finite
};
static_assert(sizeof(GuessOut) == 32, "GuessOut layout");

// Batch path (filter_kernel.cuh): where gvr_filter_kernel left each row's candidates.
constexpr int F_SEGS = 4;  // most filter CTAs covering one row (host-enforced)
// Partition of the virtual tile sequence [0, V) over G CTAs: CTA b owns [V b / G, V (b+1) / G).
struct CandLists {
    uint2* region;  // [G][reg]: (key, idx) entries, CTA b from region + b * reg
    int4* rec;      // [num_rows][F_SEGS]: {cta, start, end, 0}, slot = cta - cta_of(first tile)
    long long V;    // num_rows * tpr
    int G;          // filter CTAs
    int tpr;        // virtual tiles per row = ceil(row_stride / STAGE_FLOATS)
    int reg;        // region capacity per CTA (entries); entries past it are dropped
};

__host__ __device__ __forceinline__ long long cl_begin(const CandLists& cl, int b) { return cl.V * b / cl.G; }
// The CTA whose range holds virtual tile v: the largest b with floor(V b / G) <= v.
__host__ __device__ __forceinline__ int cl_cta_of(const CandLists& cl, long long v)
{
    return (int)(((v + 1) * cl.G + cl.V - 1) / cl.V) - 1;
}

// Batch filter path hand-over between the kernels (scratch; every word is zero between
// calls).  Rows enter the ready queue when their candidate list is complete (the filter
// CTA finishing a row's last segment pushes it; gvr_guess_kernel pushes rows with no
// tiles); gvr_refine_kernel pops them in that order and appends the rows it cannot
// finish to the fixup list, which gvr_topk_kernel (fixup mode) works off last.
enum { Q_HEAD = 0, Q_TAIL = 1, Q_NFIX = 2, Q_RDONE = 3, Q_WORDS = 4 };
constexpr int CTL_RDONE = 3;  // ctl word: set (release) by the last refine CTA to finish
struct BatchQueue {
    int32_t* qctl;     // [Q_WORDS]
    int32_t* queue;    // [num_rows]: row + 1 once pushed, reset to 0 when popped
    int32_t* segdone;  // [num_rows]: finished filter segments, reset when popped
    int32_t* fixlist;  // [num_rows]
    // (r2) per-row threshold hand-off from Phases 1-2 to the filter kernel: tcw[r] =
    // (generation << 32) | T_c, stored with release once row r's GuessOut is written; the
    // generation is *gen + 1, *gen counting the lease's completed filter-path calls (the
    // fixup's last CTA increments it).  The filter waits per row, not for the whole grid.
    uint32_t* gen;
    unsigned long long* tcw;  // [num_rows]
};
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Publish row r's threshold (thread 0, after gp[r] is written).
__device__ __forceinline__ void publish_tc(const BatchQueue& bq, int r, uint32_t Tc)
{
    if (bq.tcw) st_release_u64(bq.tcw + r, ((unsigned long long)(*bq.gen + 1u) << 32) | Tc);
}

__device__ __forceinline__ int ld_relaxed(const int32_t* p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire(const int32_t* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// What the streaming pass hands to Phases 2-4.
struct RowMeta {
    int fill;         // entries in B
    uint32_t Tc;      // collect threshold (after raises)
    uint32_t ftc;     // f(T_c) = fill - extras
    uint32_t kmax;    // max key in B
    uint32_t extras;  // superset entries (NaN / -0 against +0) with key < T_c
};

// Secant step of Eq. 6 in value space between the anchors
// (lo, f(lo) = clo > target) and (hi, f(hi) = chi < target); hi is exclusive and may
// be 2^32.  First-step damping caps the interpolation fraction at 0.5 (PAPER.md:565,
// 540-541).  If the result is not strictly inside (lo, hi) in key space (float
// precision limits, +/-Inf or NaN anchors) the key-space midpoint is used instead.
// Requires hi - lo >= 2.  Arithmetic is explicit round-to-nearest fp32 (R19).
__device__ __forceinline__ uint32_t secant_step(uint64_t lo, uint32_t clo, uint64_t hi, uint32_t chi,
                                                float target, bool damp, bool bisect)
{
    if (!bisect && hi <= 0xffffffffull) {
        const float flo = key2f((uint32_t)lo);
        const float fhi = key2f((uint32_t)hi);
        float frac = __fdiv_rn(__fsub_rn((float)clo, target), (float)(clo - chi));
        if (damp) frac = fminf(frac, 0.5f);
        const float tf = __fadd_rn(flo, __fmul_rn(frac, __fsub_rn(fhi, flo)));
        if (isfinite(tf)) {
            const uint32_t kt = f2key(tf);
            if ((uint64_t)kt > lo && (uint64_t)kt < hi) return kt;
        }
    }
    return (uint32_t)(lo + ((hi - lo) >> 1));
}


// Round geometry: warp w owns floats [1024 w, 1024 (w+1)) of the 8192-float round
// block; lane l's float4 j (0..7) is at 1024 w + 128 j + 4 l, so every warp load is 512
// contiguous bytes (conflict-free).  Element e = 4 j + c of the 32-bit pass mask sits at
// lane_base + rel_off(e).
__device__ __forceinline__ int lane_base(int warp, int lane) { return 1024 * warp + 4 * lane; }
__device__ __forceinline__ int rel_off(int e) { return ((e & ~3) << 5) | (e & 3); }

// Raise the collect threshold when B would overflow.  Called by the
// whole group after a round in which some warps could not reserve space: B[0, fill)
// plus the round elements held by those warps (held mask, elements at sp[lb +
// rel_off(e)]) exceed the capacity.  Finds a key T > Tc whose count over B and the held
// elements lies in [K, cap/2], as close as possible to f_target*phi (phi = streamed
// fraction of the row, so the count extrapolates to f_target at the row's end), by a
// key-space radix search: a 256-bin histogram of [base, base + width) per level, suffix
// counts at the bin edges, then either an acceptable edge or narrowing into the bin
// where the count crosses K.  Compacts B to {key >= T} and returns 0, or returns 1 if
// no such T exists (massive ties).  mx = max key over B and the held elements.
__device__ __noinline__ int raise_threshold(GvrGroup& c, const Buf& B, int32_t* hist, const float* sp, int lb,
                                            uint32_t held, uint32_t& Tc, int& fill, uint32_t mx, float phi, int K,
                                            int& raises, uint32_t& tie_key)
{
    const uint32_t acc_hi = (uint32_t)B.cap / 2;
    const float ft = 0.5f * (float)(K + CWIN);
    const uint32_t target = (uint32_t)fminf(fmaxf(ft * phi, (float)K), (float)acc_hi);
    uint32_t base = Tc, above = 0;
    uint64_t width = (uint64_t)mx - Tc + 1ull;
    uint32_t T = 0;
    int rc = 1;
    for (int level = 0; level < 5; ++level) {
        const int s = width > (uint64_t)RAISE_BINS ? 64 - __clzll((long long)(width - 1)) - 8 : 0;
        hist[c.tid] = 0;
        c.sync();
        for (int p = c.tid; p < fill; p += GVR_NT) {
            const uint32_t kk = B.key[p];
            if (kk >= base && (uint64_t)(kk - base) < width) atomicAdd(&hist[(kk - base) >> s], 1);
        }
        for (uint32_t m = held; m; m &= m - 1) {
            const uint32_t kk = f2key(sp[lb + rel_off(__ffs(m) - 1)]);
            if (kk >= base && (uint64_t)(kk - base) < width) atomicAdd(&hist[(kk - base) >> s], 1);
        }
        c.sync();
        // thread t owns bin b = 255 - t: S_b = count(key >= edge(b)) = above + sum_{b' >= b} hist
        const int b = RAISE_BINS - 1 - c.tid;
        const uint32_t h = (uint32_t)hist[b];
        uint32_t tot;
        const uint32_t Sb = above + group_excl_scan(c, h, tot) + h;
        // edges with S >= target / S >= K form prefixes [0, m) of the bins
        uint32_t m_t = Sb >= target ? 1u : 0u, m_k = Sb >= (uint32_t)K ? 1u : 0u;
        group_red2<R_ADD, R_ADD>(c, m_t, m_k);
        const int bt = (int)m_t - 1, bk = (int)m_k - 1;
        if (b == bt) c.misc[20] = (int)Sb;
        if (b == bk) c.misc[21] = (int)Sb;
        if (b == bk + 1) c.misc[22] = (int)Sb;
        c.sync();
        const uint32_t St = bt >= 0 ? (uint32_t)c.misc[20] : 0u;
        const uint32_t Sk = (uint32_t)c.misc[21];
        const uint32_t Snext = bk + 1 < RAISE_BINS ? (uint32_t)c.misc[22] : above;
        c.sync();
        if (bk < 0) break;  // cannot happen: S at the lowest edge is >= K
        if (bt >= 0 && St <= acc_hi) {
            T = base + ((uint32_t)bt << s);
            rc = 0;
            break;
        }
        if (Sk <= acc_hi) {
            T = base + ((uint32_t)bk << s);
            rc = 0;
            break;
        }
        if (s == 0) {  // one key value holds the crossing: keep it if B can hold it
            if (Sk <= (uint32_t)B.cap && base + (uint32_t)bk != Tc) {
                T = base + (uint32_t)bk;
                rc = 0;
            } else if (base + (uint32_t)bk < 0xffffffffu) {
                // massive ties at v = base + bk (more than the buffer holds, fewer than K
                // above it so far): keep collecting only keys > v.  If the row ends with
                // fewer than K keys > v, v is the K-th key and the caller runs the ordered
                // tie fill (R13); otherwise later raises continue as usual.
                tie_key = base + (uint32_t)bk;
                T = tie_key + 1u;
                rc = 0;
            }
            break;
        }
        base += (uint32_t)bk << s;
        width = 1ull << s;
        above = Snext;
    }
    if (rc == 0) {
        const ChunkCounts cc = count_chunks_ge(c, B, fill, T);
        fill = compact_ge(c, B, fill, T, cc);
        Tc = T;
        ++raises;
    }
    return rc;
}

// Append the elements of `mask` (round elements at sp[lb + rel_off(e)], row index
// ibase + rel_off(e)) to B at pos, pos+1, ...
__device__ __forceinline__ void write_candidates(const Buf& B, const float* sp, int lb, int ibase, uint32_t mask,
                                                 int pos, uint32_t Tc, uint32_t& kmax, uint32_t& extras)
{
    while (mask) {
        const int e = 31 - __clz(mask);
        mask ^= 1u << e;
        const int o = rel_off(e);
        const uint32_t u = __float_as_uint(sp[lb + o]);
        const uint32_t kv = u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);  // f2key
        kmax = max(kmax, kv);
        extras += kv < Tc;  // superset entry (NaN / -0 against +0)
        B.key[pos] = kv;
        B.idx[pos] = ibase + o;
        ++pos;
    }
}

// The streaming pass of one row (row body through the ring; the <= 6 unaligned head /
// tail scalars exactly).  Collects B ⊇ {key >= Tc}, superset only by NaN / -0-against-+0
// entries counted in `extras`.  Returns 0, or 1 on massive ties (the remaining tiles are
// still waited for, so no copy is in flight when the ring is reused).  pbits: the phase
// parity of each stage's mbarrier before this pass (bit s for stage s); the ring's
// barriers are initialised once per CTA and their phases carried across passes and rows
// (no mbarrier re-initialisation while copies of earlier passes are tracked), updated here
// by the number of tiles each stage received.
__device__ __forceinline__ int stream_row(GvrGroup& c, const Ring& ring, const RowPlan& p, const Buf& B,
                                          int32_t* rhist, uint32_t& Tc, int& fill, int K, int& raises, uint32_t& kmax,
                                          uint32_t& extras, uint32_t& tie_key, uint32_t& pbits)
{
    int* fillp = c.misc + 16;     // reservation cursor
    int* failbase = c.misc + 17;  // lowest failed reservation of the round
    const int body_end = p.head + p.nfl;
    {  // scalar head [0, head) and tail [body_end, n)
        const int tail = p.n - body_end;
        int i = -1;
        if (c.tid < p.head)
            i = c.tid;
        else if (c.tid < p.head + tail)
            i = body_end + (c.tid - p.head);
        const uint32_t kv = i >= 0 ? f2key(__ldg(p.x + i)) : 0u;
        const uint32_t pass = (i >= 0 && kv >= Tc) ? 1u : 0u;
        uint32_t tot;
        const uint32_t ex = group_excl_scan(c, pass, tot);
        if (pass) {
            B.key[ex] = kv;
            B.idx[ex] = p.idx0 + i;
            kmax = max(kmax, kv);
        }
        if (c.tid == 0) {
            *fillp = (int)tot;
            *failbase = 0x7fffffff;
        }
        c.sync();
    }
    const int lb = lane_base(c.warp, c.lane);
    const float inv_n = 1.0f / (float)p.n;
    const int nrounds = (p.ntiles + ROUND_STAGES - 1) / ROUND_STAGES;
    float Tf = key2f(Tc);
    int rc = 0;
    for (int rd = 0; rd < nrounds; ++rd) {
        const int t0 = rd * ROUND_STAGES;
        const int s0 = t0 % NSTAGE;
        const uint32_t lap = (uint32_t)(t0 / NSTAGE);
        const int nf = min(ROUND_FLOATS, p.nfl - t0 * STAGE_FLOATS);  // floats in this round
        mbar_wait(ring.full(s0), (lap ^ (pbits >> s0)) & 1u);
        if (t0 + 1 < p.ntiles) mbar_wait(ring.full(s0 + 1), (lap ^ (pbits >> (s0 + 1))) & 1u);
        const float* sp = ring.stage(s0);
        const int ibase = p.idx0 + p.head + t0 * STAGE_FLOATS + lb;
        bool failed_here = false;
        uint32_t mask = 0;
        if (rc == 0) {
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
            if (c.lane == 31 && wtot) base = atomicAdd(fillp, (int)wtot);
            base = __shfl_sync(FULL, base, 31);
            if (wtot && base + (int)wtot > B.cap) {  // warp-uniform: no room, hold the round
                failed_here = true;
                if (c.lane == 0) atomicMin(failbase, base);
            } else {
                write_candidates(B, sp, lb, ibase, mask, base + (int)(incl - cnt), Tc, kmax, extras);
            }
        }
        if (c.sync_or(failed_here)) {
            // B would overflow: raise T_c over B and the held elements, then the held
            // warps filter their elements again and append them.
            int f = min(*fillp, *failbase);
            const float phi = (float)(p.n - p.nfl + t0 * STAGE_FLOATS + nf) * inv_n;
            const uint32_t held = failed_here ? mask : 0u;
            uint32_t mx = kmax;
            for (uint32_t m = held; m; m &= m - 1) mx = max(mx, f2key(sp[lb + rel_off(__ffs(m) - 1)]));
            mx = group_red1<R_MAX>(c, mx);
            const int rr = raise_threshold(c, B, rhist, sp, lb, held, Tc, f, mx, phi, K, raises, tie_key);
            if (rr) {
                rc = 1;
            } else {
                extras = 0;  // the compaction was exact
                Tf = key2f(Tc);
                if (c.tid == 0) {
                    *fillp = f;
                    *failbase = 0x7fffffff;
                }
                c.sync();
                if (failed_here) {
                    uint32_t m2 = 0;
                    for (uint32_t m = mask; m; m &= m - 1) {
                        const int e = __ffs(m) - 1;
                        if (f2key(sp[lb + rel_off(e)]) >= Tc) m2 |= 1u << e;
                    }
                    const uint32_t cnt = (uint32_t)__popc(m2);
                    const uint32_t incl = warp_incl_scan(cnt, c.lane);
                    const uint32_t wtot = __shfl_sync(FULL, incl, 31);
                    int base = 0;
                    if (c.lane == 31 && wtot) base = atomicAdd(fillp, (int)wtot);
                    base = __shfl_sync(FULL, base, 31);
                    write_candidates(B, sp, lb, ibase, m2, base + (int)(incl - cnt), Tc, kmax, extras);
                }
            }
            c.sync();
        }
        if (c.tid == 0)
#pragma unroll
            for (int q = 0; q < ROUND_STAGES; ++q)
                if (t0 + q + NSTAGE < p.ntiles) ring.issue(p, t0 + q + NSTAGE);
    }
    fill = *fillp;
#pragma unroll
    for (int st = 0; st < NSTAGE; ++st)  // tiles t = st, st + NSTAGE, ... each completed one phase
        if (p.ntiles > st) pbits ^= ((uint32_t)((p.ntiles - 1 - st) / NSTAGE + 1) & 1u) << st;
    c.sync();  // every thread has read the cursor before the scratch is reused
    return rc;
}

// Phases 3-4 and the ordered output of one streamed row (Phase 2 ran before the stream,
// phase12): B holds f(T_c) <= capacity entries, so no further threshold search is needed.
// st = {unused, snap_iters, cand_count, needs_tiefill}.
__device__ __forceinline__ void refine_row(GvrGroup& c, const Buf& B, const Work& Wk, const RowMeta& meta,
                                           int k, int32_t* o, float* ov, int (&st)[4], long long* ts)
{
    const int K = k;
    const int fill = meta.fill;
    const uint32_t kmax = meta.kmax;
    const uint32_t extras = meta.extras;
    const uint32_t T = meta.Tc;
    ChunkCounts cc;
    // ---------------- Phase 3: ballot-free compaction
    int cand = fill;
    if (extras != 0u) {
        cc = count_chunks_ge(c, B, fill, T);
        cand = compact_ge(c, B, fill, T, cc);
    }
    st[2] = cand;
    if (ts) ts[TS_PHASE23] = clock64();
    // ---------------- Phase 4 fused with the ordered output (R28): histogram over the
    // candidates, K-th bin from its scan, the bins up to it sorted -> T* and the result
    if (cand > K) {
        uint32_t ts_sorted = 0;
        if (select_sorted(c, B, Wk, cand, T, kmax, K, k, o, ov, &ts_sorted)) {
            if (ts) {
                ts[TS_PHASE4] = clock64();
            }
            st[3] = 0;
            return;
        }
    }
    // ---------------- Phase 4: exact refinement — the snap-based path,
    // taken when the K-th bin is crowded (ties) or the prefix exceeds the sort capacity
    // every candidate key lies in [T, kmax] (kmax tracked while collecting)
    uint32_t Tstar = T, nge = (uint32_t)cand;
    if (cand != K) {
        int32_t* hist = Wk.hist;
        uint32_t* list = Wk.list();
        uint32_t base = T;
        uint64_t width = (uint64_t)kmax - T + 1ull;  // keys in [base, base + width)
        int s = shift_for_width(width);
        uint32_t krem = (uint32_t)K, above = 0;
        for (int level = 0; level < 5; ++level) {
            zero_ints(c, hist, NBINS);
            if (c.tid == 0) c.misc[4] = 0;
            c.sync();
            for (int p0 = c.tid; p0 < cand; p0 += 4 * GVR_NT) {
                uint32_t kk[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) kk[u] = p0 + u * GVR_NT < cand ? B.key[p0 + u * GVR_NT] : 0u;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (p0 + u * GVR_NT < cand && kk[u] >= base && (uint64_t)(kk[u] - base) < width)
                        atomicAdd(&hist[(kk[u] - base) >> s], 1);
            }
            c.sync();
            int b;
            uint32_t a;
            kth_bin(c, hist, NBINS, krem, b, a);
            const uint32_t hb = (uint32_t)hist[b];
            const uint32_t lo_b = base + ((uint32_t)b << s);
            above += a;
            krem -= a;
            if (s == 0) {
                Tstar = lo_b;
                nge = above + hb;
                break;
            }
            const uint64_t bw = 1ull << s;
            if (hb <= (uint32_t)LIST_MAX) {
                for (int p0 = c.tid; p0 < cand; p0 += 4 * GVR_NT) {
                    uint32_t kk[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) kk[u] = p0 + u * GVR_NT < cand ? B.key[p0 + u * GVR_NT] : 0u;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (p0 + u * GVR_NT < cand && kk[u] >= lo_b && (uint64_t)(kk[u] - lo_b) < bw)
                            list[atomicAdd(&c.misc[4], 1)] = kk[u];
                }
                c.sync();
                if (c.warp == 0) {
                    // snap iterations, T starts at the bin's lower edge
                    uint32_t Ts = lo_b, ge_f = 0;
                    int S = 0;
                    for (;;) {
                        uint32_t ge = 0, gt = 0, up = 0xffffffffu, dn = 0u;
                        for (int i = c.lane; i < (int)hb; i += 32) {
                            const uint32_t kk = list[i];
                            ge += kk >= Ts;
                            gt += kk > Ts;
                            if (kk > Ts) up = min(up, kk);
                            if (kk < Ts) dn = max(dn, kk);
                        }
                        ge = above + __reduce_add_sync(FULL, ge);
                        gt = above + __reduce_add_sync(FULL, gt);
                        up = __reduce_min_sync(FULL, up);
                        dn = __reduce_max_sync(FULL, dn);
                        ++S;
                        if (ge < (uint32_t)K && dn >= lo_b)
                            Ts = dn;
                        else if (gt >= (uint32_t)K)
                            Ts = up;
                        else {
                            ge_f = ge;
                            break;
                        }
                    }
                    if (c.lane == 0) {
                        c.misc[6] = (int32_t)Ts;
                        c.misc[7] = (int32_t)ge_f;
                        c.misc[8] = S;
                    }
                }
                c.sync();
                Tstar = (uint32_t)c.misc[6];
                nge = (uint32_t)c.misc[7];
                st[1] += c.misc[8];
                c.sync();
                break;
            }
            // exact narrowing inside bin b (every thread has read hist[b] before the next
            // level clears the histogram)
            base = lo_b;
            width = bw;
            s = s > 11 ? s - 11 : 0;
            c.sync();
        }
    } else {
        uint32_t kmin = 0xffffffffu;
        for (int q = c.tid; q < cand; q += GVR_NT) kmin = min(kmin, B.key[q]);
        Tstar = group_red1<R_MIN>(c, kmin);
    }
    if (ts) ts[TS_PHASE4] = clock64();
    // ---------------- ordered output
    if (nge > (uint32_t)SORT_MAX) {
        st[3] = 1;  // the caller runs the ordered tie fill from global memory
        uint32_t ngt = 0;
        for (int q = c.tid; q < cand; q += GVR_NT) ngt += B.key[q] > Tstar;
        ngt = group_red1<R_ADD>(c, ngt);
        if (c.tid == 0) {
            c.misc[10] = (int32_t)Tstar;
            c.misc[11] = (int32_t)ngt;
        }
        c.sync();
    } else {
        st[3] = 0;
        emit_sorted(c, B, Wk, cand, Tstar, kmax, (int)nge, K, k, o, ov);
    }
}


// Isolated 4-byte gather (guess values, row samples): read-only path without L1
// allocation and a 64-B L2 fetch size.  With plain __ldg every miss pulled ~3.3 sectors
// (ncu: 3.6M L2 sectors, 108 MB DRAM for 1.25M requested sectors); with the hint 65 MB,
// and the guess kernel finishes ~3 us sooner on cfg2.
__device__ __forceinline__ float ld_gather(const float* p)
{
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
// Row-sample chunk load (Phase 2): 16 contiguous bytes of a 64-byte chunk, no L1 allocation.
__device__ __forceinline__ float4 ldg_sample(const float4* p)
{
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// Deterministic fp32 sum of one channel over the group: fixed xor-shuffle tree per warp,
// then the same tree over the warp sums (lanes >= W contribute 0) — the order the CPU
// replay (oracle/phase2_replay.py) follows.
template <class G>
__device__ __forceinline__ float group_fsum1(G& c, float a)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = __fadd_rn(a, __shfl_xor_sync(FULL, a, o));
    float* s = c.redf + c.par * 2 * G::W;
    if (c.lane == 0) s[c.warp] = a;
    c.sync();
    a = c.lane < G::W ? s[c.lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = __fadd_rn(a, __shfl_xor_sync(FULL, a, o));
    c.par ^= 1;
    return a;
}

// Phase-2 constants (R34-R36).
constexpr int P2_CHUNK = 16;                 // sample floats per thread (one 64-byte read)
constexpr int P2_S = 256 * P2_CHUNK;         // sample values: one chunk per thread
#ifndef GVR_P2_RUN
#define GVR_P2_RUN 16
#endif
constexpr int P2_RUN = GVR_P2_RUN;           // floats per contiguous sample run (P2_RUN / 16 threads)
constexpr int P2_TPR = P2_RUN / P2_CHUNK;    // threads per run
constexpr int P2_NRUN = 256 / P2_TPR;        // runs per row sample
static_assert(P2_RUN % P2_CHUNK == 0 && 256 % P2_TPR == 0, "sample runs");
// Offset (from the 16-byte aligned body start) of thread t's 16 sample floats: run
// g = t / P2_TPR starts at P2_RUN floor(g nrun / P2_NRUN), nrun = floor(body / P2_RUN),
// and thread t reads its 16 floats at 16 (t % P2_TPR) inside it (R34).
__host__ __device__ __forceinline__ int sample_off(int t, int body)
{
    const int nrun = body / P2_RUN;
    return P2_RUN * (int)(((int64_t)(t / P2_TPR) * nrun) / P2_NRUN) + P2_CHUNK * (t % P2_TPR);
}
constexpr int P2_MAX_ITERS = 12;             // probes before the Phase-2 fallback (R12)
constexpr float P2_Z_DEFAULT = 4.5f;

// Phases 1-2 for one row by a 256-thread group (R7, R8-R12,
// R19, R29, R34-R36).  Every fp32 operation is explicit round-to-nearest in a fixed
// order, so the CPU replay reproduces T_c, I and the exit kind bit for bit.
//   Phase 1: the guessed values x[q], q = prev[m] for the guessed ranks m of slots
//     i = t + 256 j (thread t): m_i = 8 gs floor(i / 8) + i % 8 < k (R29; load_guess_idx)
//     -> pmin / pmax (keys), pmean = sum / count (Eq. 4).
//     No valid guess -> the statistics of the row sample.
//   Sample: thread t's 16 contiguous floats of the 16-byte aligned body at sample_off(t):
//     256 chunks of 16 floats spread over the row (R34), in registers, as keys.
//   Phase 2: window [L, H] in sample hits, L = ceil(mu + z sqrt(mu)) with mu = k S / n
//     the expected hits at the K-th value, H = L + ceil(L / 2), target (L + H) / 2;
//     anchors exact for the sample: (min key, S), (max key + 1, 0) (R8).  Probe T0 =
//     pmean, then the bracket end pmin (f(T0) below the window) or
//     pmax (above), then Eq. 6 steps (secant_step) — a probe with L <= hits <= H ends
//     the search.  Adjacent anchors (ties) or P2_MAX_ITERS probes -> the lo anchor, whose
//     hits are above the window.
// The rank-th largest of the group's 16 register keys per thread (1 <= rank <= 4096):
// most-significant-digit radix select, 8 bits per level over a 256-bin shared histogram
// (sh: 256 ints of the caller's shared memory).
template <class G>
__device__ __forceinline__ uint32_t sample_rank_key16(G& c, const uint32_t (&sk)[16], int32_t* sh, uint32_t rank)
{
    uint32_t prefix = 0u, pmask = 0u, rem = rank;
    for (int level = 0; level < 4; ++level) {
        const int shift = 24 - 8 * level;
        sh[c.tid] = 0;
        c.sync();
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if ((sk[q] & pmask) == prefix) atomicAdd(&sh[(sk[q] >> shift) & 255u], 1);
        c.sync();
        const int bin = 255 - c.tid;  // thread t owns bin 255 - t: descending digit order
        const uint32_t h = (uint32_t)sh[bin];
        uint32_t tot;
        const uint32_t ex = group_excl_scan(c, h, tot);
        if (ex < rem && ex + h >= rem) {
            c.misc[0] = bin;
            c.misc[1] = (int)ex;
        }
        c.sync();
        prefix |= (uint32_t)c.misc[0] << shift;
        pmask |= 255u << shift;
        rem -= (uint32_t)c.misc[1];
        c.sync();
    }
    return prefix;
}

// The guess indices Phase 1 reads (they do not depend on the row length, so callers issue
// these loads first): slot i = tid + 256 j holds guessed rank m_i = 8 gs (i / 8) + i % 8
// when m_i < k — blocks of 8 consecutive ranks every 8 gs ranks, one 32-byte sector of
// indices per block (gs = guess_stride; 1 = every rank; R29); -1 for unused slots.
constexpr int GUESS_PER_THREAD = KMAX / 256;
template <class G>
__device__ __forceinline__ void load_guess_idx(const G& c, const int32_t* pr, int k, const GvrParams& prm,
                                               int32_t (&gi)[GUESS_PER_THREAD])
{
    static_assert(G::N == 256, "eight guess slots per thread");
    const int gs = prm.guess_stride;
#pragma unroll
    for (int j = 0; j < GUESS_PER_THREAD; ++j) gi[j] = -1;
#pragma unroll
    for (int j = 0; j < GUESS_PER_THREAD; ++j) {
        if (j * G::N * gs >= k) break;  // group-uniform: slot j's smallest rank is 256 gs j
        const int i = c.tid + j * G::N;
        const int m = 8 * gs * (i >> 3) + (i & 7);
        if (pr && m < k) gi[j] = __ldg(pr + m);
    }
}

// Phases 1-2 from the values: gv[j] the guessed value of slot j (valid bit j), sv the
// thread's 16 sample values; n the row length.  Shared by phase12 (values read from the
// score row) and the fused indexer path (values computed from the keys, indexer_kernel.cuh).
template <class G>
__device__ __forceinline__ GuessOut phase12_core(G& c, int n, const float (&gv)[GUESS_PER_THREAD], uint32_t valid,
                                                 const float (&sv)[P2_CHUNK], int k, const GvrParams& prm,
                                                 int32_t* sh256, long long* ts = nullptr)
{
    constexpr int GPT = GUESS_PER_THREAD;
    GuessOut g;
    uint32_t sk[P2_CHUNK];
    uint32_t smin = 0xffffffffu, smax = 0u;
#pragma unroll
    for (int q = 0; q < P2_CHUNK; ++q) {
        sk[q] = f2key(sv[q]);
        smin = min(smin, sk[q]);
        smax = max(smax, sk[q]);
    }
    // ---- Phase 1 (Eq. 4)
    uint32_t kmn = 0xffffffffu, kmx = 0u, cnt = 0u;
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
        if ((valid >> j) & 1u) {
            const uint32_t kv = f2key(gv[j]);
            kmn = min(kmn, kv);
            kmx = max(kmx, kv);
            ++cnt;
        }
        sum = __fadd_rn(sum, gv[j]);  // invalid slots add +0
    }
    group_red4<R_MIN, R_MAX, R_ADD, R_MAX>(c, kmn, kmx, cnt, smax);
    if (ts && c.tid == 0) ts[2] = global_ns();  // (diagnostics) every load has arrived
    smin = group_red1<R_MIN>(c, smin);
    bool complete = cnt == (uint32_t)k && prm.guess_stride == 1;
    if (cnt == 0) {  // no valid guess: statistics of the row sample (R7)
        sum = 0.f;
#pragma unroll
        for (int q = 0; q < P2_CHUNK; ++q) sum = __fadd_rn(sum, sv[q]);
        kmn = smin;
        kmx = smax;
        cnt = P2_S;
        complete = false;
    }
    sum = group_fsum1(c, sum);
    const float pmean = __fdiv_rn(sum, (float)cnt);
    if (ts && c.tid == 0) ts[3] = global_ns();  // (diagnostics) Phase 1 done
    // ---- Phase 2 over the sample (Eq. 6)
    const float mu = __fdiv_rn((float)(k * P2_S), (float)n);
    const int L = min(max((int)ceilf(__fadd_rn(mu, __fmul_rn(prm.window_z, __fsqrt_rn(mu)))), 1), P2_S);
    const int H = min(L + (L + 1) / 2, P2_S);
    const float ft = __fmul_rn((float)(L + H), 0.5f);
    uint32_t klo = smin, clo = P2_S, chi = 0;
    uint64_t khi = (uint64_t)smax + 1ull;
    int it = 0;
    uint32_t hits = 0;
    auto probe = [&](uint32_t T) -> bool {  // group-uniform
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < P2_CHUNK; ++q) m += sk[q] >= T ? 1u : 0u;
        hits = group_red1<R_ADD>(c, m);
        ++it;
        if (hits >= (uint32_t)L && hits <= (uint32_t)H) return true;
        if (hits > (uint32_t)H) {
            klo = T;
            clo = hits;
        } else {
            khi = T;
            chi = hits;
        }
        return false;
    };
    int exitk = GVR_P2_WINDOW;
    uint32_t T = 0;
    bool found = false;
    if (isfinite(pmean)) {
        const uint32_t t0 = f2key(pmean);
        if (t0 > klo && (uint64_t)t0 < khi) {
            T = t0;
            found = probe(t0);
            if (!found) {
                const uint32_t t1 = hits < (uint32_t)L ? kmn : kmx;
                if (t1 > klo && (uint64_t)t1 < khi) {
                    T = t1;
                    found = probe(t1);
                }
            }
        }
    }
    for (int secants = 0; !found; ++secants) {
        if (khi - klo < 2) {
            exitk = GVR_P2_TIES;
            break;
        }
        if (it >= P2_MAX_ITERS) {
            exitk = GVR_P2_EXHAUSTED;
            break;
        }
        T = secant_step(klo, clo, khi, chi, ft, secants == 0, secants >= prm.max_secant);
        found = probe(T);
    }
    g.tie = 0u;
    if (!found && exitk == GVR_P2_EXHAUSTED) {
        // no probe landed in the window: the exact finisher over the sample (R12) — the
        // sample key of rank ceil(f_t), whose hits are at least that rank
        T = sample_rank_key16(c, sk, sh256, (uint32_t)((L + H + 1) / 2));
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < P2_CHUNK; ++q) m += sk[q] >= T ? 1u : 0u;
        hits = group_red1<R_ADD>(c, m);
        if (hits > (uint32_t)H) {
            // that key is a tie group reaching past the window (R37): a ties exit at it
            exitk = GVR_P2_TIES;
            g.tie = T;
        }
    } else if (!found) {
        // ties: the anchors are adjacent keys — the lo anchor's key holds a tie group that
        // spans the window (its hits are above it, the next key's below)
        T = klo;
        hits = clo;
        g.tie = klo;
    }
    g.Tc = T;
    g.T0 = f2key(pmean);
    g.t0_ok = isfinite(pmean) ? 1 : 0;
    g.tmin = (complete && kmn < T) ? kmn : 0u;
    g.top = max(kmx, smax);
    g.iters = (int16_t)it;
    g.exit = (int16_t)exitk;
    g.scount = (int32_t)hits;
    return g;
}

template <class G>
__device__ __forceinline__ GuessOut phase12(G& c, const RowPlan& p, const int32_t (&gi)[GUESS_PER_THREAD], int k,
                                            const GvrParams& prm, int32_t* sh256, long long* ts = nullptr)
{
    static_assert(G::N == 256, "one sample chunk per thread");
    constexpr int GPT = GUESS_PER_THREAD;  // 8 guessed positions per thread
    if (p.n <= GVR_CAP) {  // the whole row fits in B: collect everything, no search
        GuessOut g;
        g.Tc = 0u;
        g.tie = 0u;
        g.T0 = 0u;
        g.tmin = 0u;
        g.top = 0xffffffffu;
        g.t0_ok = 0;
        g.iters = 0;
        g.exit = GVR_P2_ALL;
        g.scount = 0;
        return g;
    }
    // ---- loads: the sample chunk, then the guessed values
    const float4* sp4 = reinterpret_cast<const float4*>(p.x + p.head + sample_off(c.tid, p.nfl));
    float sv[P2_CHUNK];
#pragma unroll
    for (int q = 0; q < P2_CHUNK / 4; ++q) {
        const float4 v = ldg_sample(sp4 + q);
        sv[4 * q] = v.x;
        sv[4 * q + 1] = v.y;
        sv[4 * q + 2] = v.z;
        sv[4 * q + 3] = v.w;
    }
    float gv[GPT];
    uint32_t valid = 0;
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
        gv[j] = 0.f;
        if (gi[j] >= 0 && gi[j] < p.n) {
            gv[j] = ld_gather(p.x + gi[j]);
            valid |= 1u << j;
        }
    }
    return phase12_core(c, p.n, gv, valid, sv, k, prm, sh256, ts);
}


// ---------------- Phases 1-2 for the batch paths
// One 256-thread CTA per row, all rows resident at once: with every row's gathers in
// flight together and no streaming traffic in the memory queues, the dependent round
// trips (guess indices, then the values and the sample) cost one short kernel instead of
// stalling each row's streaming CTA.
constexpr int GUESS_NT = 256;
using GuessGroup = Group<GUESS_NT, 1>;

// Row order of the row path (batch_path = 1): rows whose Phase 2 did not end in its
// window (ties, exhausted) first, so the expensive rows start in the first wave.
struct RowSched {
    int32_t* order;    // [num_rows]: CTA b of the streaming kernel processes row order[b]
    int32_t* cursors;  // [3]: front / back fill counts, finished streaming CTAs (zero at launch)
};

__global__ void __launch_bounds__(GUESS_NT)
gvr_guess_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens,
                 const int32_t* prev, int k, int num_rows, GvrParams prm, GuessOut* __restrict__ gp, RowSched sched,
                 BatchQueue bq)
{
    // the streaming kernel may be scheduled now; it waits for this grid before reading
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ __align__(16) unsigned char scratch[GROUP_SCRATCH_BYTES];
    GuessGroup c;
    c.init(threadIdx.x, scratch);
    const int r = blockIdx.x;
    // diagnostics: stamps kept locally, stored at exit if recording is on (flag read last)
    long long gts_l[4] = {global_ns(), 0, 0, 0};
    int32_t gi[GUESS_PER_THREAD];  // issued first: the guess indices do not depend on the row length
    load_guess_idx(c, prev ? prev + (int64_t)r * k : nullptr, k, prm, gi);
    const RowPlan p = plan_row(scores, stride, row_lens, r, k);
    // batch filter path: a row with no tiles never reaches the filter kernel; it goes to
    // the ready queue now (the refine kernel emits it from the row itself)
    if (bq.queue && p.ntiles == 0 && c.tid == 0) st_release(bq.queue + atomicAdd(bq.qctl + Q_TAIL, 1), r + 1);
    if (p.n <= k) {  // trivial row: no guess needed (block-uniform); scheduled last
        if (c.tid == 0 && !bq.queue) sched.order[num_rows - 1 - atomicAdd(sched.cursors + 1, 1)] = r;
        return;
    }
    __shared__ int32_t sh[256];
    GuessOut g = phase12(c, p, gi, k, prm, sh, gts_l);
    // filter path, a ties exit: collect the keys strictly above the tie; when they are
    // fewer than K the refine kernel fills the rest with the tie's lowest indices (R37)
    if (bq.queue && g.exit == GVR_P2_TIES && g.tie < 0xffffffffu) g.Tc = g.tie + 1u;
    if (c.tid == 0 && r < FTS_MAX && *(volatile int*)&g_fts_on) {
        g_gts[r][0] = gts_l[0];
        g_gts[r][1] = global_ns();
        g_gts[r][2] = gts_l[2];
        g_gts[r][3] = gts_l[3];
    }
    if (c.tid == 0) {
        gp[r] = g;
        publish_tc(bq, r, g.Tc);  // release: gp[r] is visible to whoever sees this word
        if (!bq.queue) {
            if (g.exit == GVR_P2_TIES || g.exit == GVR_P2_EXHAUSTED)
                sched.order[atomicAdd(sched.cursors, 1)] = r;
            else
                sched.order[num_rows - 1 - atomicAdd(sched.cursors + 1, 1)] = r;
        }
    }
}

// Split / fixup mode: the last CTA of the grid resets the scheduling cursors and the batch
// queue's control words for the next call.
__device__ __forceinline__ void fixup_done(int32_t* ctl, const BatchQueue& bq, int tid)
{
    if (tid == 0 && ctl && atomicAdd(ctl + 2, 1) == (int)gridDim.x - 1) {
        ctl[0] = 0;
        ctl[1] = 0;
        ctl[2] = 0;
        ctl[CTL_RDONE] = 0;
        if (bq.qctl)
            for (int i = 0; i < Q_WORDS; ++i) bq.qctl[i] = 0;
        if (bq.gen) *bq.gen += 1u;  // this call's thresholds are stale from now on
    }
}

// The fixup kernels' start: thread 0 waits for the last refine CTA's release flag.
__device__ __forceinline__ void fixup_wait(int32_t* ctl)
{
    __shared__ int go;
    if (threadIdx.x == 0) {
        while (ld_acquire(ctl + CTL_RDONE) == 0) __nanosleep(128);
        go = 1;
    }
    __syncthreads();
    (void)go;
}

// One row, the whole path: Phases 1-2 (or their hand-off), the streaming pass, Phases 3-4
// and the ordered output, with every fallback.  A CTA calls it once per row (reinit: the
// ring barriers were used by a previous row of this CTA).  short_known: an earlier pass
// (the filter kernel) already found f(T_c) < K, so the row is streamed at once at the
// second-pass threshold (R30).
__device__ __forceinline__ void topk_row(const float* __restrict__ scores, int64_t stride,
                                      const int32_t* __restrict__ row_lens, int k, int32_t* out, float* out_val,
                                      gvr_row_stats* stats, const GvrParams& prm, const GuessOut* __restrict__ gp,
                                      const int32_t* prev, long long* phase_ts, int r, bool reinit,
                                      uint32_t& pbits, bool short_known = false)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const Ring ring{reinterpret_cast<float*>(smem + G_OFF_RING), reinterpret_cast<uint64_t*>(smem + G_OFF_BARS),
                    policy_evict_first()};
    const Buf B{reinterpret_cast<uint32_t*>(smem + G_OFF_B), reinterpret_cast<int32_t*>(smem + G_OFF_B + GVR_CAP * 4),
                GVR_CAP};
    const Work Wk{reinterpret_cast<int32_t*>(smem + G_OFF_WORK), reinterpret_cast<int32_t*>(smem + G_OFF_WORK + NBINS * 4),
                  reinterpret_cast<unsigned long long*>(smem + G_OFF_WORK + 2 * NBINS * 4), GVR_CSORT};
    GvrGroup c;
    c.init(threadIdx.x, smem + G_OFF_SCR);
    const int K = k;
    const RowPlan p = plan_row(scores, stride, row_lens, r, k);
    const long long ts0 = phase_ts ? clock64() : 0ll;
    if (reinit) {
        fence_proxy_async_smem();  // the previous row's work area (aliasing the ring) before the TMA refill
        c.sync();                  // every wait on the previous row's barriers is over
    }
    if (c.tid == 0) {
        if (!reinit) {  // the CTA's first row: the barriers start at phase 0
            for (int s = 0; s < NSTAGE; ++s) mbar_init(ring.full(s), 1);
            fence_mbar_init();
        }
        for (int t = 0; t < NSTAGE && t < p.ntiles; ++t) ring.issue(p, t);  // the first 64 KB load during Phase 1
    }
    const RowGeom g = make_geom(p.x, p.n);
    int32_t* o = out + (int64_t)r * k;
    float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
    int st[4] = {0, 0, 0, 0};
    int done_kind = GVR_DONE_CONVERGED, passes = 1, raises = 0, ftc_stat = 0;
    long long tsr[TS_N] = {ts0, 0, 0, 0, 0, 0, phase_ts ? global_ns() : 0ll, 0, 0};
    GuessOut gq{};
    if (p.n <= k) {
        c.sync();
        small_row_emit(c, B, Wk, g, k, o, ov);
        done_kind = GVR_DONE_TRIVIAL;
        st[2] = p.n;
    } else {
        // ---------------- Phases 1-2: in gvr_guess_kernel (batch paths) or here (fused)
        if (gp) {
            gq = gp[r];
        } else {
            int32_t gi[GUESS_PER_THREAD];
            load_guess_idx(c, prev ? prev + (int64_t)r * k : nullptr, k, prm, gi);
            gq = phase12(c, p, gi, k, prm, reinterpret_cast<int32_t*>(smem + G_OFF_RHIST));
        }
        RowMeta m;
        m.Tc = short_known ? gq.tmin : gq.Tc;
        if (short_known) passes = 2;
        if (phase_ts) tsr[TS_PHASE1] = clock64();
        // ---------------- streaming pass (HBM read once, TMA ring)
        uint32_t kmax = 0u, extras = 0u, tie_key = 0u;
        const int rc = stream_row(c, ring, p, B, reinterpret_cast<int32_t*>(smem + G_OFF_RHIST), m.Tc, m.fill, K, raises,
                                  kmax, extras, tie_key, pbits);
        group_red2<R_MAX, R_ADD>(c, kmax, extras);
        m.kmax = kmax;
        m.extras = extras;
        m.ftc = (uint32_t)m.fill - extras;
        if (phase_ts) tsr[TS_STREAM] = clock64();
        if (rc == 0 && m.ftc < (uint32_t)K && tie_key != 0u) {
            // massive ties at tie_key and fewer than K keys above it in the whole row:
            // tie_key is the K-th key; ordered tie fill (one more pass, R13)
            done_kind = GVR_DONE_TIEFILL;
            ++passes;
            tiefill_emit(c, B, Wk, g, tie_key, m.ftc, K, k, o, ov);
        } else if (rc == 0 && m.ftc < (uint32_t)K && short_known) {
            // the second-pass threshold was short as well (only massive ties can do that):
            // exact radix select + ordered tie fill
            const RadixResult rr = radix_select_global(c, Wk, g, (uint32_t)K, false);
            passes += rr.rounds + 1;
            done_kind = GVR_DONE_TIEFILL;
            tiefill_emit(c, B, Wk, g, rr.prefix, rr.above, K, k, o, ov);
        } else if (rc == 0 && m.ftc < (uint32_t)K) {
            // f(T_c) < K (the threshold overshot the K-th value): stream the row once more at
            // a threshold that cannot undershoot — pmin of a complete guess, else -inf —
            // with the usual raises keeping >= K (R30); bounded at two HBM passes
            fence_proxy_async_smem();
            c.sync();
            if (c.tid == 0)
                for (int t = 0; t < NSTAGE && t < p.ntiles; ++t) ring.issue(p, t);
            m.Tc = gq.tmin;
            kmax = 0u;
            extras = 0u;
            uint32_t tie2 = 0u;
            const int rc2 = stream_row(c, ring, p, B, reinterpret_cast<int32_t*>(smem + G_OFF_RHIST), m.Tc, m.fill, K,
                                       raises, kmax, extras, tie2, pbits);
            group_red2<R_MAX, R_ADD>(c, kmax, extras);
            m.kmax = kmax;
            m.extras = extras;
            m.ftc = (uint32_t)m.fill - extras;
            ++passes;
            if (rc2 == 0 && m.ftc < (uint32_t)K && tie2 != 0u) {
                done_kind = GVR_DONE_TIEFILL;
                ++passes;
                tiefill_emit(c, B, Wk, g, tie2, m.ftc, K, k, o, ov);
            } else if (rc2 == 0 && m.ftc >= (uint32_t)K) {
                ftc_stat = (int)m.ftc;
                refine_row(c, B, Wk, m, k, o, ov, st, phase_ts ? tsr : nullptr);
                if (st[3]) {
                    done_kind = GVR_DONE_TIEFILL;
                    ++passes;
                    tiefill_emit(c, B, Wk, g, (uint32_t)c.misc[10], (uint32_t)c.misc[11], K, k, o, ov);
                }
            } else {
                const RadixResult rr = radix_select_global(c, Wk, g, (uint32_t)K, false);
                passes += rr.rounds + 1;
                done_kind = GVR_DONE_TIEFILL;
                tiefill_emit(c, B, Wk, g, rr.prefix, rr.above, K, k, o, ov);
            }
        } else if (rc) {
            // massive ties: exact radix select + ordered tie fill from global memory
            // (R12/R13)
            const RadixResult rr = radix_select_global(c, Wk, g, (uint32_t)K, false);
            passes += rr.rounds + 1;
            done_kind = GVR_DONE_TIEFILL;
            tiefill_emit(c, B, Wk, g, rr.prefix, rr.above, K, k, o, ov);
        } else {
            ftc_stat = (int)m.ftc;
            refine_row(c, B, Wk, m, k, o, ov, st, phase_ts ? tsr : nullptr);
            if (st[3]) {
                // huge tie group at T*: ordered tie fill from global memory (R13)
                done_kind = GVR_DONE_TIEFILL;
                ++passes;
                tiefill_emit(c, B, Wk, g, (uint32_t)c.misc[10], (uint32_t)c.misc[11], K, k, o, ov);
            }
        }
    }
    if (c.tid == 0) {
        if (stats) {
            gvr_row_stats s;
            s.secant_iters = gq.iters;
            s.snap_iters = st[1];
            s.cand_count = st[2];
            s.done_kind = done_kind;
            s.global_passes = passes;
            s.raises = raises;
            s.buffer_count = ftc_stat;
            s.cluster = 1;
            s.phase2_exit = gq.exit;
            s.sample_count = gq.scount;
            s.tc_key = gq.Tc;
            s.reserved = 0;
            stats[r] = s;
        }
        if (phase_ts) {
            tsr[TS_END] = clock64();
            tsr[TS_GEND] = global_ns();
            tsr[TS_SMID] = sm_id();
            for (int i = 0; i < TS_N; ++i) phase_ts[(int64_t)r * TS_N + i] = tsr[i];
        }
    }
}

__global__ void __launch_bounds__(GVR_NT, 2)
gvr_topk_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm, const GuessOut* __restrict__ gp,
                const int32_t* __restrict__ order, const int32_t* prev, long long* phase_ts, int32_t* ctl)
{
    // Split mode (gp != nullptr): Phase 1 ran in gvr_guess_kernel and CTA b processes row
    // order[b]; it runs under programmatic dependent launch: wait for the guess grid (its
    // writes are visible after this) before reading the row order and the hand-off.
    // Fused mode (gp == nullptr, batches of at most one wave): CTA b processes row b and
    // runs Phase 1 itself while its first tiles load.
    if (gp) asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t pbits = 0u;
    topk_row(scores, stride, row_lens, k, out, out_val, stats, prm, gp, prev, phase_ts,
             gp ? order[blockIdx.x] : (int)blockIdx.x, false, pbits);
    fixup_done(ctl, BatchQueue{}, threadIdx.x);
}

// Batch filter path, last step: the rows gvr_refine_kernel could not finish from their
// candidate lists (an overflowed or too short list, massive ties, rows with no tiles) are
// streamed and refined in full — CTA b takes fixup-list entries b, b + G, ...  One CTA per
// SM (the loop needs more registers than the row kernel's two-per-SM budget); the list is
// usually empty.  The last CTA resets the batch queue's control words.
__global__ void __launch_bounds__(GVR_NT, 2)
gvr_fixup_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                 int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm, const GuessOut* __restrict__ gp,
                 const int32_t* prev, long long* phase_ts, int32_t* ctl, BatchQueue bq)
{
    // The refine grid's fixup list is complete once its last CTA sets the flag (this grid
    // is launched only after every refine CTA has started, so spinning cannot starve it);
    // an empty list lets the CTAs leave before the refine grid has even retired.
    fixup_wait(ctl);
    const int nfix = ld_relaxed(bq.qctl + Q_NFIX);
    uint32_t pbits = 0u;  // stage phase parities carried across this CTA's rows
    for (int li = (int)blockIdx.x; li < nfix; li += (int)gridDim.x)
    {
        const uint32_t e = (uint32_t)__ldcg(bq.fixlist + li);  // row | (f(T_c) < K known) << 31
        topk_row(scores, stride, row_lens, k, out, out_val, stats, prm, gp, prev, phase_ts, (int)(e & 0x7fffffffu),
                 li != (int)blockIdx.x, pbits, (e >> 31) != 0u);
    }
    fixup_done(ctl, bq, threadIdx.x);
}

// =====================================================================================
// Cluster of G CTAs per row (BASELINE.json "one CTA or cluster per row chosen
// by N"): for few, long rows one CTA streams too slowly (≈ 20 GB/s), so the row is cut
// into G slices (slice_plan), each streamed by one CTA of a thread-block cluster into its
// own buffer B_g with the common collect threshold T_c (Phase 1 is evaluated by every
// CTA, identically).  A CTA that overflows raises its own threshold, keeping >= K of its
// slice, so T_m = max_g T_c,g still satisfies f(T_m) >= K and, by Lemma 1, every element
// >= T_m of the row sits in some B_g.  The CTAs then exchange (T_c,g, kmax_g) through the
// leader's shared memory (DSMEM), count their entries >= T_m, and — after a cluster-wide
// radix search for a higher threshold if the union would not fit — push them into the
// leader's B (st.shared::cluster).  The leader finishes Phases 2-4 and the ordered output.
namespace cg = cooperative_groups;

constexpr int CX_OFF = 60 * 1024;  // cluster exchange area inside the (idle) ring
enum { CX_TC = 0, CX_KMAX = 1, CX_RC = 2, CX_N = 3, CX_STRIDE = 4, CX_DEC = 32 };
static_assert(CX_OFF + (CX_DEC + 8) * 4 <= NSTAGE * STAGE_BYTES, "exchange area fits in the ring");

// Cluster-wide threshold search: every CTA histograms its own B over [base, base+width)
// (256 bins), the leader sums the G histograms through DSMEM, picks a bin edge whose
// count over the whole cluster lies in [K, cap] (nearest f_target) or narrows into the
// crossing bin, and publishes the decision in its exchange area.  Returns the new
// threshold, or 0xffffffff... flagged through ok = false when none exists (massive ties).
__device__ __noinline__ uint32_t cluster_threshold(GvrGroup& c, const Buf& B, int fill, int32_t* hist, int32_t* lcx,
                                                   uint32_t Tm, uint32_t kmx, int K, bool& ok)
{
    cg::cluster_group cl = cg::this_cluster();
    const int G = (int)cl.num_blocks();
    const bool leader = cl.block_rank() == 0;
    const uint32_t cap = (uint32_t)B.cap;
    const uint32_t target = min((uint32_t)((K + CWIN) / 2), cap);
    uint32_t base = Tm, above = 0;
    uint64_t width = (uint64_t)kmx - Tm + 1ull;
    ok = false;
    uint32_t T = Tm;
    for (int level = 0; level < 5; ++level) {
        const int s = width > (uint64_t)RAISE_BINS ? 64 - __clzll((long long)(width - 1)) - 8 : 0;
        hist[c.tid] = 0;
        c.sync();
        for (int p = c.tid; p < fill; p += GVR_NT) {
            const uint32_t kk = B.key[p];
            if (kk >= base && (uint64_t)(kk - base) < width) atomicAdd(&hist[(kk - base) >> s], 1);
        }
        cl.sync();  // every CTA's histogram complete and visible
        if (leader) {
            const int b = RAISE_BINS - 1 - c.tid;
            uint32_t h = 0;
            for (int q = 0; q < G; ++q) h += (uint32_t)cl.map_shared_rank(hist, q)[b];
            uint32_t tot;
            const uint32_t Sb = above + group_excl_scan(c, h, tot) + h;
            uint32_t m_t = Sb >= target ? 1u : 0u, m_k = Sb >= (uint32_t)K ? 1u : 0u;
            group_red2<R_ADD, R_ADD>(c, m_t, m_k);
            const int bt = (int)m_t - 1, bk = (int)m_k - 1;
            if (b == bt) c.misc[20] = (int)Sb;
            if (b == bk) c.misc[21] = (int)Sb;
            if (b == bk + 1) c.misc[22] = (int)Sb;
            c.sync();
            if (c.tid == 0) {
                const uint32_t St = bt >= 0 ? (uint32_t)c.misc[20] : 0u;
                const uint32_t Sk = (uint32_t)c.misc[21];
                const uint32_t Snext = bk + 1 < RAISE_BINS ? (uint32_t)c.misc[22] : above;
                int dec = 0;  // 0 narrow, 1 done, 2 fail
                uint32_t Tn = 0;
                if (bk < 0) {
                    dec = 2;
                } else if (bt >= 0 && St <= cap) {
                    dec = 1;
                    Tn = base + ((uint32_t)bt << s);
                } else if (Sk <= cap) {
                    dec = 1;
                    Tn = base + ((uint32_t)bk << s);
                } else if (s == 0) {
                    dec = 2;
                } else {
                    Tn = base + ((uint32_t)bk << s);  // new base
                }
                lcx[CX_DEC + 0] = dec;
                lcx[CX_DEC + 1] = (int32_t)Tn;
                lcx[CX_DEC + 2] = s;
                lcx[CX_DEC + 3] = (int32_t)Snext;
            }
        }
        cl.sync();  // decision published
        const int dec = lcx[CX_DEC + 0];
        const uint32_t Tn = (uint32_t)lcx[CX_DEC + 1];
        const int sw = lcx[CX_DEC + 2];
        const uint32_t Snext = (uint32_t)lcx[CX_DEC + 3];
        cl.sync();  // everyone read it before the next level overwrites the histograms
        if (dec == 1) {
            ok = true;
            T = Tn;
            break;
        }
        if (dec == 2) break;
        base = Tn;
        width = 1ull << sw;
        above = Snext;
    }
    return T;
}

__global__ void __launch_bounds__(GVR_NT, 2)
gvr_topk_cluster_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                        int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm, const int32_t* prev,
                        long long* phase_ts)
{
    extern __shared__ __align__(128) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int G = (int)cl.num_blocks();
    const int g = (int)cl.block_rank();
    const int r = (int)blockIdx.x / G;
    const Ring ring{reinterpret_cast<float*>(smem + G_OFF_RING), reinterpret_cast<uint64_t*>(smem + G_OFF_BARS),
                    policy_evict_first()};
    const Buf B{reinterpret_cast<uint32_t*>(smem + G_OFF_B), reinterpret_cast<int32_t*>(smem + G_OFF_B + GVR_CAP * 4),
                GVR_CAP};
    const Work Wk{reinterpret_cast<int32_t*>(smem + G_OFF_WORK), reinterpret_cast<int32_t*>(smem + G_OFF_WORK + NBINS * 4),
                  reinterpret_cast<unsigned long long*>(smem + G_OFF_WORK + 2 * NBINS * 4), GVR_CSORT};
    int32_t* rhist = reinterpret_cast<int32_t*>(smem + G_OFF_RHIST);
    int32_t* cx = reinterpret_cast<int32_t*>(smem + G_OFF_RING + CX_OFF);
    GvrGroup c;
    c.init(threadIdx.x, smem + G_OFF_SCR);
    const int K = k;
    const RowPlan pw = plan_row(scores, stride, row_lens, r, k);
    const RowPlan p = slice_plan(pw, g, G);
    const long long ts0 = phase_ts ? clock64() : 0ll;
    if (c.tid == 0) {
        for (int s = 0; s < NSTAGE; ++s) mbar_init(ring.full(s), 1);
        fence_mbar_init();
        for (int t = 0; t < NSTAGE && t < p.ntiles; ++t) ring.issue(p, t);
    }
    const RowGeom geo = make_geom(pw.x, pw.n);
    int32_t* o = out + (int64_t)r * k;
    float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
    int st[4] = {0, 0, 0, 0};
    int done_kind = GVR_DONE_CONVERGED, passes = 1, raises = 0, ftc_stat = 0;
    long long tsr[TS_N] = {ts0, 0, 0, 0, 0, 0, phase_ts ? global_ns() : 0ll, 0, 0};
    GuessOut gq{};
    if (pw.n <= k) {  // cluster-uniform: the leader emits the whole row
        if (g != 0) return;
        c.sync();
        small_row_emit(c, B, Wk, geo, k, o, ov);
        done_kind = GVR_DONE_TRIVIAL;
        st[2] = pw.n;
    } else {
        // ---------------- Phase 1 (every CTA, identical result) and the slice stream
        int32_t gi[GUESS_PER_THREAD];
        load_guess_idx(c, prev ? prev + (int64_t)r * k : nullptr, k, prm, gi);
        gq = phase12(c, pw, gi, k, prm, rhist);
        if (phase_ts) tsr[TS_PHASE1] = clock64();
        uint32_t Tc = gq.Tc, kmax = 0u, extras = 0u, Tm = 0u, kmx = 0u, T = 0u, tot = 0, pre = 0;
        int fill = 0, raises_all = 0;
        bool ok = false;
        ChunkCounts cc;
        int32_t* lcx = cl.map_shared_rank(cx, 0);
        uint32_t pbits = 0u;  // stage phase parities (stream_row)
        for (int pass = 0;; ++pass) {
            if (pass == 1) {
                // f(T_m) < K: every slice is streamed once more at a threshold that cannot
                // undershoot (R30)
                fence_proxy_async_smem();  // the exchange area (inside the ring) before the TMA refill
                c.sync();
                if (c.tid == 0)
                    for (int t = 0; t < NSTAGE && t < p.ntiles; ++t) ring.issue(p, t);
                Tc = gq.tmin;
                kmax = 0u;
                extras = 0u;
                fill = 0;
                ++passes;
            }
            uint32_t tie_unused = 0u;  // cluster slices: ties end in the leader's fallback
            const int rc = stream_row(c, ring, p, B, rhist, Tc, fill, K, raises, kmax, extras, tie_unused, pbits);
            group_red2<R_MAX, R_ADD>(c, kmax, extras);
            // ---------------- merge across the cluster (DSMEM)
            cl.sync();  // every slice streamed; rings idle
            if (c.tid == 0) {
                lcx[g * CX_STRIDE + CX_TC] = (int32_t)Tc;
                lcx[g * CX_STRIDE + CX_KMAX] = (int32_t)kmax;
                lcx[g * CX_STRIDE + CX_RC] = rc | (raises << 1);
            }
            cl.sync();
            Tm = 0u;
            kmx = 0u;
            int any_rc = 0;
            raises_all = 0;
            for (int q = 0; q < G; ++q) {
                Tm = max(Tm, (uint32_t)lcx[q * CX_STRIDE + CX_TC]);
                kmx = max(kmx, (uint32_t)lcx[q * CX_STRIDE + CX_KMAX]);
                any_rc |= lcx[q * CX_STRIDE + CX_RC] & 1;
                raises_all += lcx[q * CX_STRIDE + CX_RC] >> 1;
            }
            ok = any_rc == 0;
            T = Tm;
            tot = pre = 0;
            if (ok) {
                cc = count_chunks_ge(c, B, fill, T);
                uint32_t ng = group_red1<R_ADD>(c, chunk_total(cc));
                cl.sync();  // the exchange slots are read before they are rewritten
                if (c.tid == 0) lcx[g * CX_STRIDE + CX_N] = (int32_t)ng;
                cl.sync();
                for (int q = 0; q < G; ++q) {
                    const uint32_t nq = (uint32_t)lcx[q * CX_STRIDE + CX_N];
                    tot += nq;
                    if (q < g) pre += nq;
                }
                if (tot > (uint32_t)B.cap) {
                    // the union does not fit the leader's buffer: raise the threshold cluster-wide
                    T = cluster_threshold(c, B, fill, rhist, lcx, Tm, kmx, K, ok);
                    if (ok) {
                        ++raises_all;
                        cc = count_chunks_ge(c, B, fill, T);
                        ng = group_red1<R_ADD>(c, chunk_total(cc));
                        if (c.tid == 0) lcx[g * CX_STRIDE + CX_N] = (int32_t)ng;
                        cl.sync();
                        tot = pre = 0;
                        for (int q = 0; q < G; ++q) {
                            const uint32_t nq = (uint32_t)lcx[q * CX_STRIDE + CX_N];
                            tot += nq;
                            if (q < g) pre += nq;
                        }
                    }
                }
            }
            const bool under = ok && tot < (uint32_t)K;  // cluster-uniform
            ok = ok && !under;
            if (!under || pass == 1) break;
            cl.sync();  // the exchange area (inside the rings) is read before the rings refill
        }
        if (ok) {
            // the leader compacts its own entries in place, then the others append theirs
            if (g == 0) fill = compact_ge(c, B, fill, T, cc);
            cl.sync();
            if (g != 0) {
                uint32_t* dkey = cl.map_shared_rank(B.key, 0);
                int32_t* didx = cl.map_shared_rank(B.idx, 0);
                push_ge(c, B, fill, T, cc, dkey, didx, (int)pre);
            }
            cl.sync();  // every push has landed in the leader's buffer
            if (g != 0) return;
            if (phase_ts) tsr[TS_STREAM] = clock64();
            RowMeta m;
            m.fill = (int)tot;
            m.Tc = T;
            m.ftc = tot;
            m.kmax = kmx;
            m.extras = 0u;  // the merge compared exact keys
            ftc_stat = (int)tot;
            refine_row(c, B, Wk, m, k, o, ov, st, phase_ts ? tsr : nullptr);
            if (st[3]) {
                done_kind = GVR_DONE_TIEFILL;
                ++passes;
                tiefill_emit(c, B, Wk, geo, (uint32_t)c.misc[10], (uint32_t)c.misc[11], K, k, o, ov);
            }
        } else {
            // massive ties or f(T_m) < K: the leader selects from global memory
            cl.sync();
            if (g != 0) return;
            const RadixResult rr = radix_select_global(c, Wk, geo, (uint32_t)K, false);
            passes += rr.rounds + 1;
            done_kind = GVR_DONE_TIEFILL;
            tiefill_emit(c, B, Wk, geo, rr.prefix, rr.above, K, k, o, ov);
        }
        raises = raises_all;
    }
    if (c.tid == 0) {
        if (stats) {
            gvr_row_stats sr;
            sr.secant_iters = gq.iters;
            sr.snap_iters = st[1];
            sr.cand_count = st[2];
            sr.done_kind = done_kind;
            sr.global_passes = passes;
            sr.raises = raises;
            sr.buffer_count = ftc_stat;
            sr.cluster = G;
            sr.phase2_exit = gq.exit;
            sr.sample_count = gq.scount;
            sr.tc_key = gq.Tc;
            sr.reserved = 0;
            stats[r] = sr;
        }
        if (phase_ts) {
            tsr[TS_END] = clock64();
            tsr[TS_GEND] = global_ns();
            tsr[TS_SMID] = sm_id();
            for (int i = 0; i < TS_N; ++i) phase_ts[(int64_t)r * TS_N + i] = tsr[i];
        }
    }
}

}  // namespace gvr
