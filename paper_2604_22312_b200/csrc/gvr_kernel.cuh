// gvr_kernel.cuh — Guess-Verify-Refine exact Top-K, one CTA per row (sm_100a).
//
// Method: PAPER.md Sec. 4 (lines 379-690).  Phases as executed here:
//   Phase 1 (Guess): gather x at the previous step's Top-K
//     positions; pmin / pmax / pmean (Eq. 4) plus the second moment.
//   Streaming pass (B200 re-design of the Phase-2 count pass fused with the Phase-3
//     collector): the row is read from HBM exactly once, in
//     coalesced float4 tiles held in registers; every element >= the collect
//     threshold T_c is appended (ballot-free, block-scan offsets) to the candidate
//     buffer B in shared memory.  B therefore holds {x >= T_c} and f(T) for every
//     T >= T_c can be counted from B alone (Lemma 1).  If B would
//     overflow, T_c is raised by a secant search over B (Eq. 6) to a threshold that
//     still keeps >= K elements (so f(T_c) >= K at the end of the row).
//   Phase 2: secant search of Eq. 6 toward f_target inside the
//     window K <= f(T) <= C, starting from T0 = pmean, with first-step damping and
//     bisection fallback — the counts come from B (shared memory), not from HBM.
//   Phase 3: ballot-free compaction of B to {x >= T} reusing the
//     per-thread counts of the last count pass (count cache).
//   Phase 4: 2048-bin histogram over the candidate key range,
//     warp-parallel K-th-bin search, snap iterations until n>(T) < K <= n>=(T),
//     exact hierarchical narrowing if the snap budget runs out.
//   Ordered output: the candidates >= T* are sorted by (key desc, index asc) and the
//     first K indices are written (BASELINE.json tie rule; R1/R2).
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

// Raise the collect threshold when B would overflow (B200 design).
// B[0, fill) and the tile's keys >= Tc together exceed CAP.  Find T > Tc whose count
// over B plus the tile lies in [K, CAP/2] by Eq. 6 secant steps aimed at
// K <= f_target*phi <= CAP/2 (phi = streamed fraction of the row), compact B to
// {key >= T} and return 0; return 1 if no such T exists (massive ties).
template <class Tile>
__device__ __forceinline__ int raise_threshold(Ctx& c, const Tile& tl, uint32_t& Tc, int& fill, uint32_t c_at_tc,
                                               float phi, int K, const GvrParams& prm, RowStats& st)
{
    // exclusive upper anchor: 1 + max key over B and the tile
    uint32_t mx = buffer_max_local(c, fill);
#pragma unroll
    for (int e = 0; e < Tile::E; ++e)
        if (tl.valid(e) && tl.key[e] >= Tc) mx = max(mx, tl.key[e]);
    mx = block_red1<R_MAX>(c, mx);
    uint64_t lo = Tc, hi = (uint64_t)mx + 1ull;
    uint32_t clo = c_at_tc, chi = 0;
    const uint32_t acc_hi = CAP / 2;
    const float ft = 0.5f * (float)(K + CWIN);
    const float target = fminf(fmaxf(ft * phi, (float)K), (float)acc_hi);
    uint32_t T = Tc;
    ChunkCounts cc;
    for (int it = 0;; ++it) {
        if (hi - lo < 2) {
            // adjacent keys: no threshold in [K, CAP/2]; lo still fits if clo <= CAP
            if (clo > (uint32_t)CAP || lo == (uint64_t)Tc) return 1;
            T = (uint32_t)lo;
            cc = count_chunks_ge(c, fill, T);
            break;
        }
        T = secant_step(lo, clo, hi, chi, target, it == 0, it >= prm.max_secant);
        cc = count_chunks_ge(c, fill, T);
        uint32_t cnt = chunk_total(cc);
#pragma unroll
        for (int e = 0; e < Tile::E; ++e)
            if (tl.valid(e) && tl.key[e] >= T) ++cnt;
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
    ++st.raises;
    return 0;
}

// Streaming pass: read the row once, collect {key >= Tc} into B, raising Tc on
// overflow.  Returns 0 (B = {key >= Tc}, fill = f(Tc) <= CAP) or 1 (massive ties).
__device__ __forceinline__ int stream_collect(Ctx& c, const RowGeom& g, uint32_t& Tc, int& fill, int K,
                                              const GvrParams& prm, RowStats& st)
{
    ++st.passes;
    fill = 0;
    const float inv_n = 1.0f / (float)g.n;
    return for_each_tile(g, c.tid, [&](auto& tl, int streamed) -> int {
        using T_ = std::remove_reference_t<decltype(tl)>;
        uint32_t cnt = 0;
#pragma unroll
        for (int e = 0; e < T_::E; ++e)
            if (tl.valid(e) && tl.key[e] >= Tc) ++cnt;
        uint32_t tot;
        uint32_t ex = block_excl_scan(c, cnt, tot);
        if (fill + (int)tot > CAP) {  // block-uniform
            if (raise_threshold(c, tl, Tc, fill, (uint32_t)fill + tot, (float)streamed * inv_n, K, prm, st))
                return 1;
            cnt = 0;
#pragma unroll
            for (int e = 0; e < T_::E; ++e)
                if (tl.valid(e) && tl.key[e] >= Tc) ++cnt;
            ex = block_excl_scan(c, cnt, tot);
        }
        int pos = fill + (int)ex;
#pragma unroll
        for (int e = 0; e < T_::E; ++e) {
            if (tl.valid(e) && tl.key[e] >= Tc) {
                c.bkey[pos] = tl.key[e];
                c.bidx[pos] = tl.idx(e);
                ++pos;
            }
        }
        fill += (int)tot;
        return 0;
    });
}

// Phase 4 over the candidates B[0, cand): returns T*, the exact
// K-th largest key.  Level 0: 2048-bin histogram over [kmin, kmax] with power-of-two
// bin width, warp-parallel K-th-bin search, lower-edge T, then snap iterations
// (count_ge, count_gt, snap_up, snap_down in one scan) until n>(T) < K <= n>=(T).
// If the snap budget is exhausted, the K-th bin is re-histogrammed (exact narrowing).
__device__ __forceinline__ uint32_t refine_exact(Ctx& c, int cand, int K, uint32_t kmin, uint32_t kmax, RowStats& st)
{
    constexpr int S_MAX = 32;
    uint32_t base = kmin;
    uint64_t width = (uint64_t)kmax - kmin + 1ull;  // keys in [base, base + width)
    int s = 0;
    while ((width - 1) >> s >= (uint64_t)NBINS) ++s;
    uint32_t krem = (uint32_t)K;
    bool first = true;
    for (;;) {
        zero_hist(c, NBINS);
        __syncthreads();
        for (int p = c.tid; p < cand; p += NT) {
            const uint32_t k = c.bkey[p];
            if (k >= base && (uint64_t)(k - base) < width) atomicAdd(&c.hist[(k - base) >> s], 1);
        }
        __syncthreads();
        int b;
        uint32_t a;
        kth_bin(c, NBINS, krem, b, a);
        uint32_t T = base + ((uint32_t)b << s);
        if (s == 0) return T;
        if (first) {
            first = false;
            // snap iterations
            for (int it = 0; it < S_MAX; ++it) {
                uint32_t nge = 0, ngt = 0, up = 0xffffffffu, dn = 0u;
                for (int p = c.tid; p < cand; p += NT) {
                    const uint32_t k = c.bkey[p];
                    nge += k >= T;
                    ngt += k > T;
                    if (k > T) up = min(up, k);
                    if (k < T) dn = max(dn, k);
                }
                block_red4<R_ADD, R_ADD, R_MIN, R_MAX>(c, nge, ngt, up, dn);
                ++st.snap;
                if (nge < (uint32_t)K)
                    T = dn;
                else if (ngt >= (uint32_t)K)
                    T = up;
                else
                    return T;
            }
        }
        // exact narrowing inside bin b
        krem -= a;
        base = base + ((uint32_t)b << s);
        width = 1ull << s;
        s = s > 11 ? s - 11 : 0;
    }
}

__global__ void __launch_bounds__(NT, 2)
gvr_topk_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens,
                const int32_t* prev, int k, int32_t* out, float* out_val, gvr_row_stats* stats, GvrParams prm)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Ctx c = make_ctx(smem_raw);
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
        int rc = stream_collect(c, g, Tc, fill, K, prm, st);
        if (rc == 0 && fill < K) {
            // underflow: f(T_c) < K; stream again with T_c = -inf (always >= K)
            Tc = 0u;
            rc = stream_collect(c, g, Tc, fill, K, prm, st);
        }
        __syncthreads();
        if (rc != 0) {
            // massive ties: exact radix select + ordered tie fill (R13)
            const RadixResult rr = radix_select_global(c, g, (uint32_t)K, false);
            st.passes += rr.rounds + 1;
            st.done = GVR_DONE_TIEFILL;
            tiefill_emit(c, g, rr.prefix, rr.above, K, k, o, ov);
        } else {
            st.bufcnt = fill;
            st.secant = 1;  // f(T_c) was counted during the stream
            // ---------------- Phase 2: secant search over B
            uint32_t T = Tc;
            int cand = fill;
            if (fill > CWIN) {
                uint32_t mx = block_red1<R_MAX>(c, buffer_max_local(c, fill));
                uint64_t lo = Tc, hi = (uint64_t)mx + 1ull;
                uint32_t clo = (uint32_t)fill, chi = 0;
                const float target = 0.5f * (float)(K + CWIN);  // f_target
                ChunkCounts cc;
                bool have_t0 = t0_ok && (uint64_t)T0 > lo && (uint64_t)T0 < hi;
                for (int it = 0;; ++it) {
                    if (hi - lo < 2) {
                        T = (uint32_t)lo;  // f(lo) <= fill <= CAP: B itself is a valid set
                        cc = count_chunks_ge(c, fill, T);
                        break;
                    }
                    if (have_t0) {
                        T = T0;  // Phase 2 starts at T0 = pmean
                        have_t0 = false;
                    } else {
                        T = secant_step(lo, clo, hi, chi, target, it <= 1, it >= prm.max_secant);
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
                // ---------------- Phase 3: ballot-free compaction
                cand = compact_ge(c, fill, T, cc);
            }
            st.cand = cand;
            // ---------------- Phase 4: exact refinement
            uint32_t kmin = 0xffffffffu, kmax = 0u;
            for (int p = c.tid; p < cand; p += NT) {
                const uint32_t kv = c.bkey[p];
                kmin = min(kmin, kv);
                kmax = max(kmax, kv);
            }
            block_red2<R_MIN, R_MAX>(c, kmin, kmax);
            uint32_t Tstar = kmin;
            if (cand != K) Tstar = refine_exact(c, cand, K, kmin, kmax, st);
            // ---------------- ordered output
            uint32_t nge = 0, ngt = 0;
            ChunkCounts cc2 = count_chunks_ge(c, cand, Tstar);
            nge = chunk_total(cc2);
            for (int p = c.tid; p < cand; p += NT) ngt += c.bkey[p] > Tstar;
            block_red2<R_ADD, R_ADD>(c, nge, ngt);
            if (nge > (uint32_t)SORT_MAX) {
                // huge tie group at T*: ordered tie fill from global memory
                st.done = GVR_DONE_TIEFILL;
                ++st.passes;
                tiefill_emit(c, g, Tstar, ngt, K, k, o, ov);
            } else {
                const int m = compact_ge(c, cand, Tstar, cc2);
                sort_and_emit(c, m, K, k, o, ov);
            }
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
