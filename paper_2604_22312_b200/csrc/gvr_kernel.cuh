// gvr_kernel.cuh — Guess-Verify-Refine exact Top-K on sm_100a: one 256-thread CTA per
// row, two CTAs per SM (one streams while the other refines), TMA bulk-copy ring.
//
// Method: PAPER.md Sec. 4 (lines 379-690).  Per row, as executed here:
//   Phase 1 (Guess): x at the previous step's Top-K positions ->
//     pmin / pmax / pmean (Eq. 4) plus the second moment (the first ring tiles are
//     already in flight).
//   Streaming pass (B200 re-design of the Phase-2 count pass fused with the Phase-3
//     collector): the row body is read from HBM exactly once by TMA
//     bulk copies into a 3 x 16 KB shared-memory ring (pipeline.cuh); every thread
//     appends its elements (16 per tile) whose key is >= the collect
//     threshold T_c to the candidate buffer B in shared memory (ballot-free, block-scan
//     offsets).  B holds {x >= T_c}, so f(T) for every T >= T_c is counted from B alone
//     (Lemma 1).  If B would overflow, T_c is raised by a secant
//     search over B (Eq. 6) to a threshold that still keeps >= K elements.
//   Phase 2: secant search of Eq. 6 toward f_target inside the
//     window K <= f(T) <= C, starting from T0 = pmean, with first-step damping and
//     bisection fallback — counts from B (shared memory), not from HBM.
//   Phase 3: ballot-free compaction of B to {x >= T} reusing the
//     per-thread counts of the last count pass (count cache).
//   Phase 4: 2048-bin histogram over the candidate key range,
//     warp-parallel K-th-bin search, snap iterations (count_ge, count_gt, snap_up,
//     snap_down) until n>(T) < K <= n>=(T) — run by one warp over the K-th bin's members
//     (every snap step stays inside that bin, so T* and the step count equal a scan over
//     all candidates); exact narrowing of the bin if it is too large.
//   Ordered output: candidates >= T* sorted by (key desc, index asc), first K written.
//   Fallbacks (R12/R13): massive ties or an
//     underflowing guess (f(T_c) < K) -> exact radix select + ordered tie fill from
//     global memory.
#pragma once
#include "select_global.cuh"

namespace gvr {

struct GvrParams {
    float collect_sigma;
    int max_secant;
};

struct RowStats {
    int secant, snap, cand, done, passes, raises, bufcnt;
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

// Element e (0..15) of a consumer thread's share of a ring tile sits at stage float
// 4*(tid + (e>>2)*NT) + (e&3): float4 j = e>>2 of the thread is vector tid + j*NT.
__device__ __forceinline__ int tile_pos(int tid, int e) { return 4 * (tid + (e >> 2) * NT) + (e & 3); }

// Raise the collect threshold when B would overflow.  B[0, fill) and
// the tile's elements >= Tc together exceed CAP.  Find T > Tc whose count over B plus
// the tile lies in [K, CAP/2] by Eq. 6 secant steps aimed at K <= f_target*phi <= CAP/2
// (phi = streamed fraction of the row), compact B to {key >= T} and return 0; return 1
// if no such T exists (massive ties).  The tile is re-read from the ring stage.
__device__ __noinline__ int raise_threshold(const float* sp, uint32_t vmask, uint32_t& Tc, int& fill,
                                            uint32_t c_at_tc, float phi, int K, int max_secant, int& raises,
                                            int& par)
{
    Ctx c = make_ctx();
    c.par = par;
    uint32_t mx = buffer_max_local(c, fill);
    for (int e = 0; e < 16; ++e)
        if ((vmask >> e) & 1u) mx = max(mx, f2key(sp[tile_pos(c.tid, e)]));
    mx = block_red1<R_MAX>(c, mx);
    uint64_t lo = Tc, hi = (uint64_t)mx + 1ull;  // exclusive upper anchor
    uint32_t clo = c_at_tc, chi = 0;
    const uint32_t acc_hi = CAP / 2;
    const float ft = 0.5f * (float)(K + CWIN);
    const float target = fminf(fmaxf(ft * phi, (float)K), (float)acc_hi);
    uint32_t T = Tc;
    ChunkCounts cc;
    int rc = 0;
    for (int it = 0;; ++it) {
        if (it >= 64) {  // safety bound (bisection needs <= 32 steps)
            rc = 1;
            break;
        }
        if (hi - lo < 2) {
            // adjacent keys: no threshold in [K, CAP/2]; lo still fits if clo <= CAP
            if (clo > (uint32_t)CAP || lo == (uint64_t)Tc) {
                rc = 1;
                break;
            }
            T = (uint32_t)lo;
            cc = count_chunks_ge(c, fill, T);
            break;
        }
        T = secant_step(lo, clo, hi, chi, target, it == 0, it >= max_secant);
        cc = count_chunks_ge(c, fill, T);
        uint32_t cnt = chunk_total(cc);
        for (int e = 0; e < 16; ++e)
            if (((vmask >> e) & 1u) && f2key(sp[tile_pos(c.tid, e)]) >= T) ++cnt;
        cnt = block_red1<R_ADD>(c, cnt);
        if (cnt >= (uint32_t)K && cnt <= acc_hi) break;
        if (cnt > acc_hi) {
            lo = T;
            clo = cnt;
        } else {
            hi = T;
            chi = cnt;
        }
    }
    if (rc == 0) {
        fill = compact_ge(c, fill, T, cc);
        Tc = T;
        ++raises;
    }
    par = c.par;
    return rc;
}

// Streaming pass over one row: scalar head/tail exactly, then the body tiles from the
// ring.  Collects B ⊇ {key >= Tc} (superset only by NaN / -0-against-+0 entries, which
// every later step filters by key), raising Tc on overflow.  Returns 0, or 1 on massive
// ties.
__device__ __forceinline__ int stream_collect(Ctx& c, const RowGeom& g, const Ring& ring, int t_start, uint32_t& Tc,
                                              int& fill, int K, const GvrParams& prm, RowStats& st, uint32_t& kmax_local,
                                              uint32_t& extras)
{
    uint32_t* bkey = s_bkey();
    int32_t* bidx = s_bidx();
    if (t_start == 0) {  // scalar head [0, head) and tail [body_end, n): <= 6 elements, exact key test
        fill = 0;
        int i = -1;
        if (c.tid < g.head)
            i = c.tid;
        else if (c.tid < g.head + g.tail)
            i = g.body_end + (c.tid - g.head);
        const uint32_t kv = i >= 0 ? f2key(__ldg(g.x + i)) : 0u;
        const uint32_t pass = (i >= 0 && kv >= Tc) ? 1u : 0u;
        uint32_t tot;
        const uint32_t ex = block_excl_scan(c, pass, tot);
        if (pass) {
            bkey[ex] = kv;
            bidx[ex] = i;
        }
        fill = (int)tot;
    }
    const float inv_n = 1.0f / (float)g.n;
    float Tf = key2f(Tc);
    for (int t = t_start; t < ring.ntiles; ++t) {
        ring.wait(t);
        const float* sp = ring.stage_ptr(t);
        const int nf = ring.tile_floats(t);
        uint32_t vmask = 0xffffu;
        if (nf != STAGE_FLOATS) {
            vmask = 0u;
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (tile_pos(c.tid, e) < nf) vmask |= 1u << e;
        }
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float4 v = reinterpret_cast<const float4*>(sp)[c.tid + j * NT];
            if (pass_ge(v.x, Tf)) mask |= 1u << (4 * j);
            if (pass_ge(v.y, Tf)) mask |= 2u << (4 * j);
            if (pass_ge(v.z, Tf)) mask |= 4u << (4 * j);
            if (pass_ge(v.w, Tf)) mask |= 8u << (4 * j);
        }
        mask &= vmask;
        uint32_t tot;
        uint32_t ex = block_excl_scan(c, (uint32_t)__popc(mask), tot);
        // every thread is past tile t-1: refill its stage with tile t-1+NSTAGE
        if (c.tid == 0 && t >= 1 && t - 1 + NSTAGE < ring.ntiles) ring.issue(t - 1 + NSTAGE);
        if (fill + (int)tot > CAP) {  // block-uniform
            const float phi = (float)(g.head + g.tail + t * STAGE_FLOATS + nf) * inv_n;
            if (raise_threshold(sp, vmask, Tc, fill, (uint32_t)fill + tot, phi, K, prm.max_secant, st.raises, c.par))
                return 1;
            extras = 0;  // the compaction was exact
            Tf = key2f(Tc);
            mask = 0;
            for (int e = 0; e < 16; ++e)
                if (((vmask >> e) & 1u) && f2key(sp[tile_pos(c.tid, e)]) >= Tc) mask |= 1u << e;
            ex = block_excl_scan(c, (uint32_t)__popc(mask), tot);
        }
        // write the (few) candidates, picked out of the stage by index
        int pos = fill + (int)ex;
        const int ebase = g.head + t * STAGE_FLOATS;
        while (mask) {
            const int e = __ffs(mask) - 1;
            mask &= mask - 1;
            const int q = tile_pos(c.tid, e);
            const uint32_t kv = f2key(sp[q]);
            kmax_local = max(kmax_local, kv);
            extras += kv < Tc;  // superset entry (NaN / -0 against +0)
            bkey[pos] = kv;
            bidx[pos] = ebase + q;
            ++pos;
        }
        fill += (int)tot;
    }
    return 0;
}

// Capture the scalar head/tail and the whole first ring tile into B unfiltered (the
// collect threshold is not known yet: Phase 1's gathers are still in flight).  Tile 0
// keeps its stage layout, so B[0, nf0) is contiguous; the <= 6 scalars follow.
// Returns the fill.
__device__ __forceinline__ int capture_first_tile(Ctx& c, const RowGeom& g, const Ring& ring, uint32_t& kmax_local)
{
    uint32_t* bkey = s_bkey();
    int32_t* bidx = s_bidx();
    int nf0 = 0;
    if (ring.ntiles > 0) {
        ring.wait(0);
        nf0 = ring.tile_floats(0);
        const float4* sp = reinterpret_cast<const float4*>(ring.stage_ptr(0));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int v = c.tid + j * NT;
            if (4 * v < nf0) {
                const float4 f = sp[v];
                const uint4 kk = make_uint4(f2key(f.x), f2key(f.y), f2key(f.z), f2key(f.w));
                kmax_local = max(kmax_local, max(max(kk.x, kk.y), max(kk.z, kk.w)));
                reinterpret_cast<uint4*>(bkey)[v] = kk;
                const int i0 = g.head + 4 * v;
                reinterpret_cast<int4*>(bidx)[v] = make_int4(i0, i0 + 1, i0 + 2, i0 + 3);
            }
        }
    }
    const int ns = g.head + g.tail;  // <= 6
    if (c.tid < ns) {
        const int i = c.tid < g.head ? c.tid : g.body_end + (c.tid - g.head);
        const uint32_t kv = f2key(__ldg(g.x + i));
        kmax_local = max(kmax_local, kv);
        bkey[nf0 + c.tid] = kv;
        bidx[nf0 + c.tid] = i;
    }
    return nf0 + ns;
}

// Phase 4 over the candidates B[0, cand): returns T*, the exact
// K-th largest key, and n>=(T*).  Level 0: 2048-bin histogram over [kmin, kmax] with
// power-of-two bin width, warp-parallel K-th-bin search, T = lower edge of the K-th
// bin, then snap iterations until n>(T) < K <= n>=(T).  All snap steps stay inside
// the K-th bin, so they are computed by one warp over that bin's members plus the
// count above the bin.  A bin too large for the member list is re-histogrammed.
__device__ __forceinline__ uint32_t refine_exact(Ctx& c, int cand, int K, uint32_t kmin, uint32_t kmax, uint32_t& nge_out,
                                                 RowStats& st)
{
    const uint32_t* bkey = s_bkey();
    int32_t* hist = s_hist();
    uint32_t* list = s_list();
    int32_t* misc = s_misc();
    uint32_t base = kmin;
    uint64_t width = (uint64_t)kmax - kmin + 1ull;  // keys in [base, base + width)
    int s = shift_for_width(width);
    uint32_t krem = (uint32_t)K, above = 0;
    for (int level = 0; level < 5; ++level) {
        zero_hist(c, hist, NBINS);
        if (c.tid == 0) misc[4] = 0;
        csync();
        for (int p = c.tid; p < cand; p += NT) {
            const uint32_t k = bkey[p];
            if (k >= base && (uint64_t)(k - base) < width) atomicAdd(&hist[(k - base) >> s], 1);
        }
        csync();
        int b;
        uint32_t a;
        kth_bin(c, NBINS, krem, b, a);
        const uint32_t hb = (uint32_t)hist[b];
        const uint32_t lo_b = base + ((uint32_t)b << s);
        above += a;
        krem -= a;
        if (s == 0) {
            nge_out = above + hb;
            return lo_b;
        }
        const uint64_t bw = 1ull << s;
        if (hb <= (uint32_t)LIST_MAX) {
            for (int p = c.tid; p < cand; p += NT) {
                const uint32_t k = bkey[p];
                if (k >= lo_b && (uint64_t)(k - lo_b) < bw) list[atomicAdd(&misc[4], 1)] = k;
            }
            csync();
            if (c.warp == 0) {
                // snap iterations, T starts at the bin's lower edge
                uint32_t T = lo_b, nge = 0;
                int S = 0;
                for (;;) {
                    uint32_t ge = 0, gt = 0, up = 0xffffffffu, dn = 0u;
                    for (int i = c.lane; i < (int)hb; i += 32) {
                        const uint32_t k = list[i];
                        ge += k >= T;
                        gt += k > T;
                        if (k > T) up = min(up, k);
                        if (k < T) dn = max(dn, k);
                    }
                    ge = above + __reduce_add_sync(FULL, ge);
                    gt = above + __reduce_add_sync(FULL, gt);
                    up = __reduce_min_sync(FULL, up);
                    dn = __reduce_max_sync(FULL, dn);
                    ++S;
                    if (ge < (uint32_t)K && dn >= lo_b)
                        T = dn;
                    else if (gt >= (uint32_t)K)
                        T = up;
                    else {
                        nge = ge;
                        break;
                    }
                }
                if (c.lane == 0) {
                    misc[6] = (int32_t)T;
                    misc[7] = (int32_t)nge;
                    misc[8] = S;
                }
            }
            csync();
            nge_out = (uint32_t)misc[7];
            st.snap += misc[8];
            const uint32_t Tstar = (uint32_t)misc[6];
            csync();  // misc reused by the caller
            return Tstar;
        }
        // exact narrowing inside bin b
        base = lo_b;
        width = bw;
        s = s > 11 ? s - 11 : 0;
    }
    nge_out = 0;
    return base;  // unreachable: s reaches 0 within 3 narrowing levels
}

// Phase timestamps: clock64() at phase boundaries, written by thread 0 when `phase_ts`
// is non-null (the paper's -DGVR_PHASE_TIMING instrumentation).
enum { TS_START = 0, TS_PHASE1, TS_STREAM, TS_PHASE23, TS_PHASE4, TS_END, TS_N };

__global__ void __launch_bounds__(NT, 2)
gvr_topk_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens,
                const int32_t* prev, int k, int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm,
                long long* phase_ts)
{
    long long ts[TS_N] = {0, 0, 0, 0, 0, 0};
    if (phase_ts) ts[TS_START] = clock64();
    Ctx c = make_ctx();
    const int r = blockIdx.x;
    int n = (int)stride;
    if (row_lens) n = min(max(__ldg(row_lens + r), 0), (int)stride);
    const float* x = scores + (int64_t)r * stride;
    int32_t* o = out + (int64_t)r * k;
    float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
    const RowGeom g = make_geom(x, n);
    RowStats st = {0, 0, 0, GVR_DONE_CONVERGED, 0, 0, 0};
    const int K = k;

    if (n <= k) {
        // no selection needed; the guess is irrelevant (every element is emitted)
        small_row_emit(c, g, k, o, ov);
        st.done = GVR_DONE_TRIVIAL;
        st.passes = 1;
        st.cand = n;
    } else {
        // start streaming the row body before Phase 1 (TMA ring, pipeline.cuh)
        const Ring ring = make_ring(x + g.head, 4 * g.nvec);
        ring_start(ring);

        // ---------------- Phase 1: guess statistics (Eq. 4)
        // The gathers are issued now and consumed after the first ring tile has been
        // captured, so their latency overlaps the first TMA transfer.
        constexpr int GPT = KMAX / NT;  // guesses per thread
        float gv[GPT];
        uint32_t gok = 0;
        {
            int32_t gi[GPT];
            const int32_t* pr = prev ? prev + (int64_t)r * k : nullptr;
#pragma unroll
            for (int j = 0; j < GPT; ++j) {
                const int q = c.tid + j * NT;
                gi[j] = -1;
                if (pr && q < k) asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(gi[j]) : "l"(pr + q));
            }
#pragma unroll
            for (int j = 0; j < GPT; ++j) {
                gv[j] = 0.f;
                if (gi[j] >= 0 && gi[j] < n) {
                    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(gv[j]) : "l"(x + gi[j]));
                    gok |= 1u << j;
                }
            }
        }
        csync();  // ring barriers initialised before anyone waits on them
        uint32_t kmax_local = 0u, extras = 0u;
        int fill = capture_first_tile(c, g, ring, kmax_local);
        uint32_t kmn = 0xffffffffu, kmx = 0u, cnt = 0u, unused = 0u;
        float sum = 0.f, sq = 0.f;
#pragma unroll
        for (int j = 0; j < GPT; ++j) {
            if ((gok >> j) & 1u) {
                const float v = gv[j];
                const uint32_t kv = f2key(v);
                kmn = min(kmn, kv);
                kmx = max(kmx, kv);
                ++cnt;
                sum += v;
                sq += v * v;
            }
        }
        block_red4<R_MIN, R_MAX, R_ADD, R_ADD>(c, kmn, kmx, cnt, unused);
        if (cnt == 0) {
            // no valid guess: deterministic stride sample of M values
            kmn = 0xffffffffu;
            kmx = 0u;
            sum = sq = 0.f;
            const int M = min(KMAX, n);
            for (int j = c.tid; j < M; j += NT) {
                const int q = (int)(((int64_t)j * n) / M);
                const float v = __ldg(x + q);
                const uint32_t kv = f2key(v);
                kmn = min(kmn, kv);
                kmx = max(kmx, kv);
                ++cnt;
                sum += v;
                sq += v * v;
            }
            block_red4<R_MIN, R_MAX, R_ADD, R_ADD>(c, kmn, kmx, cnt, unused);
        }
        block_fsum2(c, sum, sq);
        const float pmean = sum / (float)cnt;
        const float var = fmaxf(sq / (float)cnt - pmean * pmean, 0.f);
        const float tcf = pmean - prm.collect_sigma * sqrtf(var);
        uint32_t Tc = isfinite(tcf) ? f2key(tcf) : kmn;
        if (n <= CAP) Tc = 0u;  // the whole row fits in B
        const uint32_t T0 = f2key(pmean);
        const bool t0_ok = isfinite(pmean);

        // ---------------- streaming pass (HBM read once, TMA ring)
        if (phase_ts) ts[TS_PHASE1] = clock64();
        ++st.passes;
        if (Tc != 0u) {  // apply T_c to the captured first tile
            const ChunkCounts c0 = count_chunks_ge(c, fill, Tc);
            fill = compact_ge(c, fill, Tc, c0);
        }
        const int rc = stream_collect(c, g, ring, 1, Tc, fill, K, prm, st, kmax_local, extras);
        uint32_t kmax = kmax_local;
        block_red2<R_MAX, R_ADD>(c, kmax, extras);  // also: B complete and visible
        const uint32_t ftc = rc == 0 ? (uint32_t)fill - extras : 0u;  // exact f(T_c)
        if (phase_ts) ts[TS_STREAM] = clock64();
        ChunkCounts cc;
        if (rc != 0 || ftc < (uint32_t)K) {
            // massive ties, or f(T_c) < K (the guess overshot): exact radix select +
            // ordered tie fill from global memory (R12/R13)
            const RadixResult rr = radix_select_global(c, g, (uint32_t)K, false);
            st.passes += rr.rounds + 1;
            st.done = GVR_DONE_TIEFILL;
            tiefill_emit(c, g, rr.prefix, rr.above, K, k, o, ov);
        } else {
            st.bufcnt = (int)ftc;
            st.secant = 1;  // f(T_c) was counted during the stream
            // ---------------- Phase 2: secant search over B
            uint32_t T = Tc;
            if (ftc > (uint32_t)CWIN) {
                uint64_t lo = Tc, hi = (uint64_t)kmax + 1ull;  // kmax = max key in B
                uint32_t clo = ftc, chi = 0;
                const float target = 0.5f * (float)(K + CWIN);  // f_target
                bool have_t0 = t0_ok && (uint64_t)T0 > lo && (uint64_t)T0 < hi;
                bool first_secant = true;
                for (int it = 0;; ++it) {
                    if (hi - lo < 2 || it >= 64) {
                        T = (uint32_t)lo;  // f(lo) <= CAP: B itself is a valid candidate set
                        cc = count_chunks_ge(c, fill, T);
                        break;
                    }
                    if (have_t0) {
                        T = T0;  // Phase 2 starts at T0 = pmean
                        have_t0 = false;
                    } else {
                        T = secant_step(lo, clo, hi, chi, target, first_secant, it >= prm.max_secant);
                        first_secant = false;
                    }
                    cc = count_chunks_ge(c, fill, T);
                    const uint32_t f = block_red1<R_ADD>(c, chunk_total(cc));
                    ++st.secant;
                    if (f >= (uint32_t)K && f <= (uint32_t)CWIN) break;
                    if (f > (uint32_t)CWIN) {
                        lo = T;
                        clo = f;
                    } else {
                        hi = T;
                        chi = f;
                    }
                }
            }
            // ---------------- Phase 3: ballot-free compaction
            int cand = fill;
            if (T != Tc) {
                cand = compact_ge(c, fill, T, cc);
            } else if (extras != 0u) {
                cc = count_chunks_ge(c, fill, T);
                cand = compact_ge(c, fill, T, cc);
            }
            st.cand = cand;
            if (phase_ts) ts[TS_PHASE23] = clock64();
            // ---------------- Phase 4: exact refinement
            // every candidate key lies in [T, kmax] (kmax tracked while collecting)
            uint32_t Tstar = T, nge = (uint32_t)cand;
            if (cand != K) {
                Tstar = refine_exact(c, cand, K, T, kmax, nge, st);
            } else {
                uint32_t kmin = 0xffffffffu;
                for (int q = c.tid; q < cand; q += NT) kmin = min(kmin, s_bkey()[q]);
                Tstar = block_red1<R_MIN>(c, kmin);
            }
            if (phase_ts) ts[TS_PHASE4] = clock64();
            // ---------------- ordered output
            if (nge > (uint32_t)SORT_MAX) {
                // huge tie group at T*: ordered tie fill from global memory (R13)
                uint32_t ngt = 0;
                for (int q = c.tid; q < cand; q += NT) ngt += s_bkey()[q] > Tstar;
                ngt = block_red1<R_ADD>(c, ngt);
                st.done = GVR_DONE_TIEFILL;
                ++st.passes;
                tiefill_emit(c, g, Tstar, ngt, K, k, o, ov);
            } else {
                emit_sorted(c, cand, Tstar, kmax, (int)nge, K, k, o, ov);
            }
        }
    }
    if (phase_ts && c.tid == 0) {
        ts[TS_END] = clock64();
        for (int i = 0; i < TS_N; ++i) phase_ts[(int64_t)r * TS_N + i] = ts[i];
    }
    if (stats && c.tid == 0) {
        gvr_row_stats s;
        s.secant_iters = st.secant;
        s.snap_iters = st.snap;
        s.cand_count = st.cand;
        s.done_kind = st.done;
        s.global_passes = st.passes;
        s.raises = st.raises;
        s.buffer_count = st.bufcnt;
        s.cluster = 1;
        stats[r] = s;
    }
}

}  // namespace gvr
