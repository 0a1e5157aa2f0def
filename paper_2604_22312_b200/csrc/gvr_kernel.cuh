// gvr_kernel.cuh — Guess-Verify-Refine exact Top-K, one CTA per row (sm_100a).
//
// Method: PAPER.md Sec. 4 (lines 379-690).  Phases as executed here:
//   Phase 1 (Guess): gather x at the previous step's Top-K
//     positions; pmin / pmax / pmean (Eq. 4) plus the second moment.
//   Streaming pass (B200 re-design of the Phase-2 count pass fused with the Phase-3
//     collector): the row body is read from HBM exactly once by TMA
//     bulk copies into a 3-stage shared-memory ring (pipeline.cuh); every element whose
//     key is >= the collect threshold T_c is appended (ballot-free, block-scan offsets)
//     to the candidate buffer B in shared memory.  B therefore holds {x >= T_c} and
//     f(T) for every T >= T_c can be counted from B alone (Lemma 1).
//     If B would overflow, T_c is raised by a secant search over B (Eq. 6) to a
//     threshold that still keeps >= K elements (so f(T_c) >= K at the end of the row).
//   Phase 2: secant search of Eq. 6 toward f_target inside the
//     window K <= f(T) <= C, starting from T0 = pmean, with first-step damping and
//     bisection fallback — the counts come from B (shared memory), not from HBM.
//   Phase 3: ballot-free compaction of B to {x >= T} reusing the
//     per-thread counts of the last count pass (count cache).
//   Phase 4: 2048-bin histogram over the candidate key range,
//     warp-parallel K-th-bin search, then the snap iterations (count_ge, count_gt,
//     snap_up, snap_down) until n>(T) < K <= n>=(T) — run by one warp over the
//     members of the K-th bin (every snap step stays inside that bin, so the result
//     and the number of steps equal a scan over all candidates); exact narrowing of
//     the bin if it is too large.
//   Ordered output: the candidates >= T* are sorted by (key desc, index asc)
//     (counting sort) and the first K indices are written (BASELINE.json tie rule).
//   Fallbacks (R12/R13): underflow -> second
//     streaming pass with T_c = -inf; massive ties -> exact radix select + ordered tie
//     fill from global memory.
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

// One ring tile held by a thread: 8 fp32 values (two float4 of the stage) and the
// valid-element mask.  Element e sits at stage float 4*(tid + (e>>2)*NT) + (e&3).
struct RingTile {
    float x[8];
    uint32_t vmask;
    __device__ __forceinline__ static int pos(int tid, int e) { return 4 * (tid + (e >> 2) * NT) + (e & 3); }
};

// Raise the collect threshold when B would overflow (B200 design).
// B[0, fill) and the tile's elements >= Tc together exceed CAP.  Find T > Tc whose
// count over B plus the tile lies in [K, CAP/2] by Eq. 6 secant steps aimed at
// K <= f_target*phi <= CAP/2 (phi = streamed fraction of the row), compact B to
// {key >= T} and return 0; return 1 if no such T exists (massive ties).
__device__ __noinline__ int raise_threshold(Ctx& c, const RingTile& tl, uint32_t& Tc, int& fill, uint32_t c_at_tc,
                                            float phi, int K, int max_secant, int& raises)
{
    uint32_t tk[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) tk[e] = ((tl.vmask >> e) & 1u) ? f2key(tl.x[e]) : 0u;
    // exclusive upper anchor: 1 + max key over B and the tile
    uint32_t mx = buffer_max_local(c, fill);
#pragma unroll
    for (int e = 0; e < 8; ++e) mx = max(mx, tk[e]);
    mx = block_red1<R_MAX>(c, mx);
    uint64_t lo = Tc, hi = (uint64_t)mx + 1ull;
    uint32_t clo = c_at_tc, chi = 0;
    const uint32_t acc_hi = CAP / 2;
    const float ft = 0.5f * (float)(K + CWIN);
    const float target = fminf(fmaxf(ft * phi, (float)K), (float)acc_hi);
    uint32_t T = Tc;
    ChunkCounts cc;
    for (int it = 0;; ++it) {
        if (it >= 64) return 1;  // safety bound (bisection needs <= 32 steps)
        if (hi - lo < 2) {
            // adjacent keys: no threshold in [K, CAP/2]; lo still fits if clo <= CAP
            if (clo > (uint32_t)CAP || lo == (uint64_t)Tc) return 1;
            T = (uint32_t)lo;
            cc = count_chunks_ge(c, fill, T);
            break;
        }
        T = secant_step(lo, clo, hi, chi, target, it == 0, it >= max_secant);
        cc = count_chunks_ge(c, fill, T);
        uint32_t cnt = chunk_total(cc);
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (((tl.vmask >> e) & 1u) && tk[e] >= T) ++cnt;
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
    fill = compact_ge(c, fill, T, cc);
    Tc = T;
    ++raises;
    return 0;
}

// Streaming pass over the row: scalar head/tail exactly, then the body through the
// TMA ring.  Collects B ⊇ {key >= Tc} (superset only by NaN / -0 against +0 entries,
// which every later step filters by key), raising Tc on overflow.  Returns 0, or 1 on
// massive ties.
__device__ __forceinline__ int stream_collect(Ctx& c, const RowGeom& g, const Ring& ring, uint32_t& Tc, int& fill,
                                              int K, const GvrParams& prm, RowStats& st)
{
    uint32_t* bkey = s_bkey();
    int32_t* bidx = s_bidx();
    ++st.passes;
    fill = 0;
    {  // scalar head [0, head) and tail [body_end, n): <= 6 elements, exact key test
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
    for (int t = 0; t < ring.ntiles; ++t) {
        ring.wait(t);
        const float* sp = ring.stage_ptr(t);
        const int nf = ring.tile_floats(t);
        RingTile tl;
        {
            const float4 a = reinterpret_cast<const float4*>(sp)[c.tid];
            const float4 b = reinterpret_cast<const float4*>(sp)[c.tid + NT];
            tl.x[0] = a.x; tl.x[1] = a.y; tl.x[2] = a.z; tl.x[3] = a.w;
            tl.x[4] = b.x; tl.x[5] = b.y; tl.x[6] = b.z; tl.x[7] = b.w;
        }
        if (nf == STAGE_FLOATS) {
            tl.vmask = 0xffu;
        } else {
            tl.vmask = 0u;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (RingTile::pos(c.tid, e) < nf) tl.vmask |= 1u << e;
        }
        uint32_t mask = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (pass_ge(tl.x[e], Tf)) mask |= 1u << e;
        mask &= tl.vmask;
        uint32_t tot;
        uint32_t ex = block_excl_scan(c, (uint32_t)__popc(mask), tot);
        // every thread is past tile t-1: refill its stage with tile t-1+NSTAGE
        if (c.tid == 0 && t >= 1 && t - 1 + NSTAGE < ring.ntiles) {
            fence_proxy_async();
            ring.issue(t - 1 + NSTAGE);
        }
        if (fill + (int)tot > CAP) {  // block-uniform
            const float phi = (float)(g.head + g.tail + t * STAGE_FLOATS + nf) * inv_n;
            if (raise_threshold(c, tl, Tc, fill, (uint32_t)fill + tot, phi, K, prm.max_secant, st.raises))
                return 1;
            Tf = key2f(Tc);
            mask = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (((tl.vmask >> e) & 1u) && f2key(tl.x[e]) >= Tc) mask |= 1u << e;
            ex = block_excl_scan(c, (uint32_t)__popc(mask), tot);
        }
        // write the (few) candidates, picked out of the stage by index
        int pos = fill + (int)ex;
        const int ebase = g.head + t * STAGE_FLOATS;
        while (mask) {
            const int e = __ffs(mask) - 1;
            mask &= mask - 1;
            const int p = RingTile::pos(c.tid, e);
            bkey[pos] = f2key(sp[p]);
            bidx[pos] = ebase + p;
            ++pos;
        }
        fill += (int)tot;
    }
    return 0;
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
        __syncthreads();
        for (int p = c.tid; p < cand; p += NT) {
            const uint32_t k = bkey[p];
            if (k >= base && (uint64_t)(k - base) < width) atomicAdd(&hist[(k - base) >> s], 1);
        }
        __syncthreads();
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
            __syncthreads();
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
            __syncthreads();
            nge_out = (uint32_t)misc[7];
            st.snap += misc[8];
            return (uint32_t)misc[6];
        }
        // exact narrowing inside bin b
        base = lo_b;
        width = bw;
        s = s > 11 ? s - 11 : 0;
    }
    nge_out = 0;
    return base;  // unreachable: s reaches 0 within 3 narrowing levels
}

__global__ void __launch_bounds__(NT, 2)
gvr_topk_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens,
                const int32_t* prev, int k, int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm)
{
    Ctx c = make_ctx();
    const int r = blockIdx.x;
    int n = (int)stride;
    if (row_lens) n = min(max(row_lens[r], 0), (int)stride);
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
        ring_init_barriers(c);
        __syncthreads();
        Ring ring = make_ring(x + g.head, 4 * g.nvec, 0u);
        ring_prime(c, ring);

        // ---------------- Phase 1: guess statistics (Eq. 4)
        uint32_t kmn = 0xffffffffu, kmx = 0u, cnt = 0u, unused = 0u;
        float sum = 0.f, sq = 0.f;
        if (prev) {
            const int32_t* pr = prev + (int64_t)r * k;
            for (int j = c.tid; j < k; j += NT) {
                const int p = pr[j];
                if (p >= 0 && p < n) {
                    const float v = __ldg(x + p);
                    const uint32_t kv = f2key(v);
                    kmn = min(kmn, kv);
                    kmx = max(kmx, kv);
                    ++cnt;
                    sum += v;
                    sq += v * v;
                }
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
                const int p = (int)(((int64_t)j * n) / M);
                const float v = __ldg(x + p);
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

        // ---------------- streaming pass (HBM read once)
        int fill = 0;
        int rc = stream_collect(c, g, ring, Tc, fill, K, prm, st);
        __syncthreads();
        ChunkCounts cc = count_chunks_ge(c, fill, Tc);
        uint32_t ftc = rc == 0 ? block_red1<R_ADD>(c, chunk_total(cc)) : 0u;
        if (rc == 0 && ftc < (uint32_t)K) {
            // underflow: f(T_c) < K; stream again with T_c = -inf (always >= K)
            Tc = 0u;
            Ring ring2 = make_ring(x + g.head, 4 * g.nvec, (uint32_t)ring.ntiles);
            ring_prime(c, ring2);
            rc = stream_collect(c, g, ring2, Tc, fill, K, prm, st);
            __syncthreads();
            cc = count_chunks_ge(c, fill, Tc);
            ftc = rc == 0 ? block_red1<R_ADD>(c, chunk_total(cc)) : 0u;
        }
        if (rc != 0) {
            // massive ties: exact radix select + ordered tie fill (R13)
            __syncthreads();
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
                const uint32_t mx = block_red1<R_MAX>(c, buffer_max_local(c, fill));
                uint64_t lo = Tc, hi = (uint64_t)mx + 1ull;
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
            if (T != Tc || ftc != (uint32_t)fill) cand = compact_ge(c, fill, T, cc);
            st.cand = cand;
            // ---------------- Phase 4: exact refinement
            uint32_t kmin = 0xffffffffu, kmax = 0u;
            const uint32_t* bkey = s_bkey();
            for (int p = c.tid; p < cand; p += NT) {
                const uint32_t kv = bkey[p];
                kmin = min(kmin, kv);
                kmax = max(kmax, kv);
            }
            block_red2<R_MIN, R_MAX>(c, kmin, kmax);
            uint32_t Tstar = kmin, nge = (uint32_t)cand;
            if (cand != K) Tstar = refine_exact(c, cand, K, kmin, kmax, nge, st);
            // ---------------- ordered output
            emit_sorted(c, cand, Tstar, (int)nge, K, k, o, ov);
        }
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
