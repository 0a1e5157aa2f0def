// select_global.cuh — distribution-agnostic pieces that read the row from global
// memory: the radix select of the exact K-th key (Sec. 2.2),
// the ordered tie fill (PAPER.md:417-420 caveat, 647-648 partition; R13),
// and the small-row (len <= k) path.  Used by the radix baseline entry point and as
// the GVR fallback for massive ties or an overshooting guess.
#pragma once
#include "row_tiles.cuh"

namespace gvr {

// Commit the entries of a tile whose key satisfies pred into B at fill (unordered,
// ballot-free offsets from one group scan).  The caller guarantees capacity.
template <class G, class Tile, class Pred>
__device__ __forceinline__ void commit_unordered(G& c, const Buf& B, const Tile& tl, Pred pred, int& fill)
{
    uint32_t cnt = 0;
#pragma unroll
    for (int e = 0; e < Tile::E; ++e)
        if (tl.valid(e) && pred(tl.key[e])) ++cnt;
    uint32_t tot;
    int pos = fill + (int)group_excl_scan(c, cnt, tot);
#pragma unroll
    for (int e = 0; e < Tile::E; ++e) {
        if (tl.valid(e) && pred(tl.key[e])) {
            B.key[pos] = tl.key[e];
            B.idx[pos] = tl.idx(e);
            ++pos;
        }
    }
    fill += (int)tot;
}

// Exact K-th largest key of the row and the number of keys strictly above it, by three
// 2048/2048/1024-bin radix rounds over key bits [31:21], [20:10], [9:0] with
// shared-memory histograms.  If `early` is set, stops after the
// first round whose threshold bucket holds <= RADIX_EARLY elements
// and reports the bucket's lower bound instead (`exact` = false).
struct RadixResult {
    uint32_t prefix;  // exact K-th key (exact) or lower bound of the threshold bucket
    uint32_t above;   // # keys strictly above the bucket / the K-th key
    uint32_t bucket;  // # keys in the bucket
    int rounds;
    bool exact;
};

template <class G>
__device__ __forceinline__ RadixResult radix_select_global(G& c, const Work& Wk, const RowGeom& g, uint32_t K,
                                                           bool early)
{
    RadixResult rr;
    uint32_t prefix = 0, pmask = 0, krem = K, above = 0;
    rr.exact = false;
    rr.rounds = 0;
    rr.bucket = 0;
    int32_t* hist = Wk.hist;
    for (int round = 0; round < 3; ++round) {
        const int shift = round == 0 ? 21 : (round == 1 ? 10 : 0);
        const int bits = round == 2 ? 10 : 11;
        const uint32_t dmask = (1u << bits) - 1u;
        const int nb = 1 << bits;
        zero_ints(c, hist, nb);
        c.sync();
        for_each_tile<G::N>(g, c.tid, [&](auto& tl, int) {
#pragma unroll
            for (int e = 0; e < tl.E; ++e) {
                const uint32_t k = tl.key[e];
                if (tl.valid(e) && (k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & dmask], 1);
            }
            return 0;
        });
        c.sync();
        int b;
        uint32_t a;
        kth_bin(c, hist, nb, krem, b, a);
        const uint32_t cb = (uint32_t)hist[b];
        above += a;
        krem -= a;
        prefix |= (uint32_t)b << shift;
        pmask |= dmask << shift;
        rr.rounds = round + 1;
        rr.bucket = cb;
        c.sync();
        if (round == 2) {
            rr.exact = true;
            break;
        }
        if (early && cb <= (uint32_t)RADIX_EARLY) break;
    }
    rr.prefix = prefix;
    rr.above = above;
    return rr;
}

// Ordered tie fill: the row's K-th largest key is Tstar with n_gt keys strictly above
// it (n_gt < K).  Emits all keys > Tstar plus the (K - n_gt) lowest-index keys equal to
// Tstar, sorted, as the row's output.  One pass in index order; ties are ranked by a
// group scan per float4 column so that they are taken in index order.
template <class G>
__device__ __forceinline__ void tiefill_emit(G& c, const Buf& B, const Work& Wk, const RowGeom& g, uint32_t Tstar,
                                             uint32_t n_gt, int K, int k, int32_t* out, float* out_val)
{
    const uint32_t need = (uint32_t)K - n_gt;
    int fill_gt = 0;
    uint32_t ties = 0;
    const int tie_base = KMAX;  // ties go to B[KMAX, KMAX + need)
    for_each_tile<G::N>(g, c.tid, [&](auto& tl, int) {
        // keys strictly above Tstar (unordered)
        commit_unordered(c, B, tl, [&](uint32_t kk) { return kk > Tstar; }, fill_gt);
        if (ties < need) {
            // ties, ranked in index order: for a MainTile the four lanes of float4 slot j
            // of all threads form one index-ordered column
            constexpr int COLS = (std::remove_reference_t<decltype(tl)>::E + 3) / 4;
#pragma unroll
            for (int j = 0; j < COLS; ++j) {
                uint32_t cnt = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = 4 * j + q;
                    if (e < tl.E && tl.valid(e) && tl.key[e] == Tstar) ++cnt;
                }
                uint32_t tot;
                uint32_t r = ties + group_excl_scan(c, cnt, tot);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = 4 * j + q;
                    if (e < tl.E && tl.valid(e) && tl.key[e] == Tstar) {
                        if (r < need) {
                            B.key[tie_base + r] = Tstar;
                            B.idx[tie_base + r] = tl.idx(e);
                        }
                        ++r;
                    }
                }
                ties += tot;
            }
        }
        return 0;
    });
    c.sync();
    // move the ties behind the > Tstar entries
    for (int i = c.tid; i < (int)need; i += G::N) {
        B.key[n_gt + i] = B.key[tie_base + i];
        B.idx[n_gt + i] = B.idx[tie_base + i];
    }
    c.sync();
    emit_sorted(c, B, Wk, K, 0u, 0u, K, K, k, out, out_val);
}

// Rows with len <= k: every element, sorted, then -1 padding (R5).
template <class G>
__device__ __forceinline__ void small_row_emit(G& c, const Buf& B, const Work& Wk, const RowGeom& g, int k,
                                               int32_t* out, float* out_val)
{
    int fill = 0;
    for_each_tile<G::N>(g, c.tid, [&](auto& tl, int) {
        commit_unordered(c, B, tl, [](uint32_t) { return true; }, fill);
        return 0;
    });
    c.sync();
    emit_sorted(c, B, Wk, g.n, 0u, 0u, g.n, g.n, k, out, out_val);
}

}  // namespace gvr
