// device_common.cuh — shared device building blocks of the GVR / radix Top-K kernels
// (sm_100a): the sortable key transform, thread groups with their own named barrier
// (a CTA may run several groups concurrently), group reductions and scans, the
// candidate-buffer count cache and in-place compaction, the K-th-bin search, and the
// ordered-output stage.
//
// PAPER.md references are to /root/reference/PAPER.md (arXiv 2604.22312).
#pragma once
#include <cstdint>
#include <new>
#include <type_traits>
#include <cuda_runtime.h>
#include "../../include/gvr_topk.h"

namespace gvr {

// ---------------------------------------------------------------------------------
// Constants.
constexpr int KMAX = GVR_MAX_K;         // 2048
constexpr int CWIN = GVR_WINDOW_C;      // Lemma-1 window upper bound C
constexpr int NBINS = 2048;             // Phase-4 / radix histogram bins
constexpr int CHUNK_SLOTS = 8;          // buffer slots per thread per compaction chunk
constexpr int NCHUNK_MAX = 4;           // chunks per count cache (capacity <= 4 * 8 * group size)
constexpr int VEC = 4;                  // float4 loads per thread per register tile
constexpr int SORT_MAX = 4096;          // largest bitonic ordered-output sort (64-bit composites)
constexpr int CSORT_BIN_MAX = 256;      // counting sort: largest bin ranked in place
constexpr int LIST_MAX = 64;            // Phase 4: largest K-th-bin snapped over (else narrowed)
constexpr int RADIX_EARLY = 2048;       // radix early exit
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------------
// Sortable FP32 key: monotone uint32, negative -> flip all bits,
// non-negative -> flip the sign bit.
__device__ __forceinline__ uint32_t f2key(float f)
{
    uint32_t u = __float_as_uint(f);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k)
{
    uint32_t u = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
    return __uint_as_float(u);
}
// Ordered-output composite: larger composite = earlier in (key desc, idx asc).
__device__ __forceinline__ unsigned long long make_comp(uint32_t key, int32_t idx)
{
    return ((unsigned long long)key << 32) | (unsigned long long)(~(uint32_t)idx);
}
__device__ __forceinline__ int32_t comp_idx(unsigned long long cv) { return (int32_t)(~(uint32_t)(cv & 0xffffffffull)); }
__device__ __forceinline__ uint32_t comp_key(unsigned long long cv) { return (uint32_t)(cv >> 32); }

// Float-domain superset test of key(x) >= key(tf): !(x < tf) holds for every x whose
// key is >= key(tf) (key order refines float order; NaN x and NaN tf pass).  Elements
// that pass spuriously (NaN, -0 against +0) are harmless: every later count and the
// output use exact key comparisons.
__device__ __forceinline__ bool pass_ge(float x, float tf) { return !(x < tf); }

// Streaming 128-bit load: read-only path, no L1 allocation, 256B L2 prefetch.
__device__ __forceinline__ float4 ldg_stream(const float4* p)
{
    float4 v;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(p));
    return v;
}

// ---------------------------------------------------------------------------------
// A group of N threads (N/32 warps) synchronising on named barrier BAR.  Reductions
// alternate between two scratch slots (par) so back-to-back calls need one barrier.
constexpr int GROUP_SCRATCH_BYTES = 2 * 4 * 16 * 4 + 2 * 2 * 16 * 4 + 32 * 4;  // up to 16 warps

template <int N_, int BAR_>
struct Group {
    static constexpr int N = N_;
    static constexpr int W = N_ / 32;
    static constexpr int BAR = BAR_;
    static_assert(W <= 16 && N_ % 32 == 0, "group size");
    int tid, lane, warp, par;
    uint32_t* red;  // [2][4][W]
    float* redf;    // [2][2][W]
    int32_t* misc;  // [32]

    __device__ __forceinline__ void init(int local_tid, unsigned char* scratch)
    {
        tid = local_tid;
        lane = local_tid & 31;
        warp = local_tid >> 5;
        par = 0;
        red = reinterpret_cast<uint32_t*>(scratch);
        redf = reinterpret_cast<float*>(scratch + 2 * 4 * 16 * 4);
        misc = reinterpret_cast<int32_t*>(scratch + 2 * 4 * 16 * 4 + 2 * 2 * 16 * 4);
    }
    __device__ __forceinline__ void sync() const { asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(N) : "memory"); }
    // barrier + group-wide OR of p in one instruction (BAR.RED.OR)
    __device__ __forceinline__ bool sync_or(bool p) const
    {
        uint32_t r;
        asm volatile(
            "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbarrier.cta.red.or.pred q, %2, %3, p;\n\t"
            "selp.u32 %0, 1, 0, q;\n\t}"
            : "=r"(r)
            : "r"((uint32_t)p), "n"(BAR), "n"(N)
            : "memory");
        return r != 0;
    }
};

// Candidate buffer B: parallel key / index arrays of capacity cap.
struct Buf {
    uint32_t* key;
    int32_t* idx;
    int cap;
    __device__ __forceinline__ unsigned long long* comp() const { return reinterpret_cast<unsigned long long*>(key); }
};

// Work area: NBINS-int histogram, NBINS-int aux (cursors / K-th-bin member list,
// which may run on into csort), csort_cap composites for the counting sort.
struct Work {
    int32_t* hist;
    int32_t* aux;
    unsigned long long* csort;
    int csort_cap;
    __device__ __forceinline__ uint32_t* list() const { return reinterpret_cast<uint32_t*>(aux); }
};
__host__ __device__ constexpr int work_bytes(int csort_cap) { return 2 * NBINS * 4 + csort_cap * 8; }
static_assert(LIST_MAX * 4 <= NBINS * 4, "list fits aux");

// ---------------------------------------------------------------------------------
// Group reductions.
enum { R_ADD = 0, R_MIN = 1, R_MAX = 2 };

template <int OP> __device__ __forceinline__ uint32_t wred(uint32_t v)
{
    if (OP == R_ADD) return __reduce_add_sync(FULL, v);
    if (OP == R_MIN) return __reduce_min_sync(FULL, v);
    return __reduce_max_sync(FULL, v);
}
template <int OP> __device__ __forceinline__ uint32_t rident() { return OP == R_MIN ? 0xffffffffu : 0u; }

template <int O0, int O1, int O2, int O3, class G>
__device__ __forceinline__ void group_red4(G& c, uint32_t& a, uint32_t& b, uint32_t& d, uint32_t& e)
{
    a = wred<O0>(a);
    b = wred<O1>(b);
    d = wred<O2>(d);
    e = wred<O3>(e);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[G::W + c.warp] = b;
        s[2 * G::W + c.warp] = d;
        s[3 * G::W + c.warp] = e;
    }
    c.sync();
    const bool in = c.lane < G::W;
    a = wred<O0>(in ? s[c.lane] : rident<O0>());
    b = wred<O1>(in ? s[G::W + c.lane] : rident<O1>());
    d = wred<O2>(in ? s[2 * G::W + c.lane] : rident<O2>());
    e = wred<O3>(in ? s[3 * G::W + c.lane] : rident<O3>());
    c.par ^= 1;
}

template <int O0, int O1, class G>
__device__ __forceinline__ void group_red2(G& c, uint32_t& a, uint32_t& b)
{
    a = wred<O0>(a);
    b = wred<O1>(b);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[G::W + c.warp] = b;
    }
    c.sync();
    const bool in = c.lane < G::W;
    a = wred<O0>(in ? s[c.lane] : rident<O0>());
    b = wred<O1>(in ? s[G::W + c.lane] : rident<O1>());
    c.par ^= 1;
}

template <int O0, class G>
__device__ __forceinline__ uint32_t group_red1(G& c, uint32_t a)
{
    a = wred<O0>(a);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 0) s[c.warp] = a;
    c.sync();
    a = wred<O0>(c.lane < G::W ? s[c.lane] : rident<O0>());
    c.par ^= 1;
    return a;
}

// Deterministic fp32 sums of two channels (fixed shuffle tree + fixed warp order).
template <class G>
__device__ __forceinline__ void group_fsum2(G& c, float& a, float& b)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        b += __shfl_xor_sync(FULL, b, o);
    }
    float* s = c.redf + c.par * 2 * G::W;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[G::W + c.warp] = b;
    }
    c.sync();
    a = c.lane < G::W ? s[c.lane] : 0.f;
    b = c.lane < G::W ? s[G::W + c.lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        b += __shfl_xor_sync(FULL, b, o);
    }
    c.par ^= 1;
}

// Inclusive warp scan (shuffles).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane)
{
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

// Exclusive group scan of one u32 per thread (thread order); returns the thread's
// offset and the total.  Warp shuffles + one barrier: the ballot-free offset
// computation of PAPER.md:600-604.
template <class G>
__device__ __forceinline__ uint32_t group_excl_scan(G& c, uint32_t v, uint32_t& total)
{
    const uint32_t x = warp_incl_scan(v, c.lane);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 31) s[c.warp] = x;
    c.sync();
    const uint32_t w = c.lane < G::W ? s[c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    total = __reduce_add_sync(FULL, w);
    c.par ^= 1;
    return before + x - v;
}

// Exclusive scan of v plus the exclusive prefix max of m (the max of m over the threads
// before this one, 0 for thread 0), with one barrier.
template <class G>
__device__ __forceinline__ uint32_t group_excl_scan_pmax(G& c, uint32_t v, uint32_t m, uint32_t& total,
                                                         uint32_t& m_before)
{
    uint32_t x = v, y = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t xv = __shfl_up_sync(FULL, x, o);
        const uint32_t yv = __shfl_up_sync(FULL, y, o);
        if (c.lane >= o) {
            x += xv;
            y = max(y, yv);
        }
    }
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 31) {
        s[c.warp] = x;
        s[G::W + c.warp] = y;
    }
    c.sync();
    const uint32_t w = c.lane < G::W ? s[c.lane] : 0u;
    const uint32_t wm = c.lane < G::W ? s[G::W + c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    const uint32_t mb_warps = __reduce_max_sync(FULL, c.lane < c.warp ? wm : 0u);
    total = __reduce_add_sync(FULL, w);
    const uint32_t mb_lanes = __shfl_up_sync(FULL, y, 1);  // inclusive max of the lanes before
    m_before = max(mb_warps, c.lane > 0 ? mb_lanes : 0u);
    c.par ^= 1;
    return before + x - v;
}

// Exclusive scan of v plus the group max of m, with one barrier.
template <class G>
__device__ __forceinline__ uint32_t group_excl_scan_max(G& c, uint32_t v, uint32_t m, uint32_t& total, uint32_t& mall)
{
    const uint32_t x = warp_incl_scan(v, c.lane);
    const uint32_t wm = __reduce_max_sync(FULL, m);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 31) {
        s[c.warp] = x;
        s[G::W + c.warp] = wm;
    }
    c.sync();
    const uint32_t w = c.lane < G::W ? s[c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    total = __reduce_add_sync(FULL, w);
    mall = __reduce_max_sync(FULL, c.lane < G::W ? s[G::W + c.lane] : 0u);
    c.par ^= 1;
    return before + x - v;
}

// ---------------------------------------------------------------------------------
// Count cache over B (the "count cache" of PAPER.md:588-597, applied to the shared-
// memory buffer): slot p of chunk ch for thread t is ch*CHUNK + j*N + t with
// CHUNK = 8*N; per-chunk counts of the last count pass let the following compaction
// skip the recount.
struct ChunkCounts {
    uint32_t c[NCHUNK_MAX];
};

template <class G>
__device__ __forceinline__ ChunkCounts count_chunks_ge(const G& c, const Buf& B, int fill, uint32_t T)
{
    constexpr int CHUNK = G::N * CHUNK_SLOTS;
    ChunkCounts cc;
#pragma unroll
    for (int ch = 0; ch < NCHUNK_MAX; ++ch) {
        uint32_t n = 0;
        if (ch * CHUNK < fill) {  // group-uniform: skip empty chunks
#pragma unroll
            for (int j = 0; j < CHUNK_SLOTS; ++j) {
                const int p = ch * CHUNK + j * G::N + c.tid;
                if (p < fill && B.key[p] >= T) ++n;
            }
        }
        cc.c[ch] = n;
    }
    return cc;
}

__device__ __forceinline__ uint32_t chunk_total(const ChunkCounts& cc)
{
    uint32_t s = 0;
#pragma unroll
    for (int ch = 0; ch < NCHUNK_MAX; ++ch) s += cc.c[ch];
    return s;
}

// In-place, order-free compaction of B[0, fill) to the entries with key >= T, using
// the cached per-chunk counts of the last count pass at T.  Chunk ch writes only to
// positions below (ch+1)*CHUNK, and every thread has loaded its chunk-ch slots before
// the scan barrier, so no slot is overwritten before it is read.  Returns new fill.
template <class G>
__device__ __forceinline__ int compact_ge(G& c, const Buf& B, int fill, uint32_t T, const ChunkCounts& cc)
{
    constexpr int CHUNK = G::N * CHUNK_SLOTS;
    int out_base = 0;
#pragma unroll
    for (int ch = 0; ch < NCHUNK_MAX; ++ch) {
        if (ch * CHUNK >= fill) break;  // group-uniform
        uint32_t kk[CHUNK_SLOTS];
        int32_t ii[CHUNK_SLOTS];
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * G::N + c.tid;
            kk[j] = 0u;
            ii[j] = 0;
            if (p < fill) {
                kk[j] = B.key[p];
                ii[j] = B.idx[p];
            }
        }
        uint32_t tot;
        int pos = out_base + (int)group_excl_scan(c, cc.c[ch], tot);
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * G::N + c.tid;
            if (p < fill && kk[j] >= T) {
                B.key[pos] = kk[j];
                B.idx[pos] = ii[j];
                ++pos;
            }
        }
        out_base += (int)tot;
    }
    c.sync();
    return out_base;
}

// Append the entries of B[0, fill) with key >= T to another buffer (dkey / didx, e.g. a
// cluster peer's shared memory) at base, base+1, ..., using the cached per-chunk counts
// of the last count pass at T.  Order-free.
template <class G>
__device__ __forceinline__ void push_ge(G& c, const Buf& B, int fill, uint32_t T, const ChunkCounts& cc, uint32_t* dkey,
                                        int32_t* didx, int base)
{
    constexpr int CHUNK = G::N * CHUNK_SLOTS;
    int out_base = base;
#pragma unroll
    for (int ch = 0; ch < NCHUNK_MAX; ++ch) {
        if (ch * CHUNK >= fill) break;  // group-uniform
        uint32_t tot;
        int pos = out_base + (int)group_excl_scan(c, cc.c[ch], tot);
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * G::N + c.tid;
            if (p < fill) {
                const uint32_t kk = B.key[p];
                if (kk >= T) {
                    dkey[pos] = kk;
                    didx[pos] = B.idx[p];
                    ++pos;
                }
            }
        }
        out_base += (int)tot;
    }
}

// ---------------------------------------------------------------------------------
// K-th bin search: find bin b with
//   sum(hist[b+1..nb)) < krem <= sum(hist[b..nb)).
// Each warp owns nb/W consecutive bins, warp totals are combined from the top, the
// owning lane resolves the exact bin.  Requires 1 <= krem <= sum(hist).
template <class G>
__device__ __forceinline__ void kth_bin(G& c, const int32_t* hist, int nb, uint32_t krem, int& b_out,
                                        uint32_t& above_out)
{
    const int per = nb / G::W;
    const int q = per / 32;
    const int base = c.warp * per + c.lane * q;
    uint32_t ls = 0;
    for (int i = 0; i < q; ++i) ls += (uint32_t)hist[base + i];
    const uint32_t wt = __reduce_add_sync(FULL, ls);
    uint32_t* s = c.red + c.par * 4 * G::W;
    if (c.lane == 0) s[c.warp] = wt;
    c.sync();
    const uint32_t v = c.lane < G::W ? s[c.lane] : 0u;
    const uint32_t above_w = __reduce_add_sync(FULL, (c.lane > c.warp && c.lane < G::W) ? v : 0u);
    uint32_t x = ls;  // inclusive suffix over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(FULL, x, o);
        if (c.lane + o < 32) x += y;
    }
    const uint32_t above_g = above_w + x - ls;
    if (ls > 0 && above_g < krem && krem <= above_g + ls) {
        uint32_t a = above_g;
        for (int i = q - 1; i >= 0; --i) {
            const uint32_t h = (uint32_t)hist[base + i];
            if (a + h >= krem) {
                c.misc[0] = base + i;
                c.misc[1] = (int32_t)a;
                break;
            }
            a += h;
        }
    }
    c.sync();
    b_out = c.misc[0];
    above_out = (uint32_t)c.misc[1];
    c.par ^= 1;
    c.sync();  // misc may be reused immediately
}

template <class G>
__device__ __forceinline__ void zero_ints(const G& c, int32_t* h, int nb)
{
    for (int i = c.tid; i < nb; i += G::N) h[i] = 0;
}

// Smallest s with (width - 1) >> s < NBINS (width in [1, 2^32]).
__device__ __forceinline__ int shift_for_width(uint64_t width)
{
    const uint32_t w = (uint32_t)(width - 1ull);
    const int bits = 32 - __clz(w);
    return bits > 11 ? bits - 11 : 0;
}

// Linear bin of d = key - lo over [0, range) using all NBINS bins:
// (d * scale) >> 32 with scale = floor(2^32 * NBINS / range), monotone in d.
__device__ __forceinline__ uint32_t bin_scale(uint64_t range)
{
    const unsigned long long q = (((unsigned long long)NBINS) << 32) / range;
    return q > 0xffffffffull ? 0xffffffffu : (uint32_t)q;
}
__device__ __forceinline__ int lin_bin(uint32_t d, uint32_t scale)
{
    return min((int)(((uint64_t)d * scale) >> 32), NBINS - 1);
}

// ---------------------------------------------------------------------------------
// Ordered output (not part of the paper, whose output is an unordered partition with
// non-deterministic ties): the selected entries are sorted by
// the 64-bit composite (key << 32 | ~idx) descending = (score desc, index asc).

// Bitonic fallback: P (power of two, <= SORT_MAX) composites in the aliasing array.
template <class G>
__device__ __forceinline__ void bitonic_sort_desc(G& c, unsigned long long* a, int P)
{
    for (int kk = 2; kk <= P; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = c.tid; i < (P >> 1); i += G::N) {
                const int lo = 2 * i - (i & (j - 1));
                const int hi = lo + j;
                const bool desc = (lo & kk) == 0;
                const unsigned long long A = a[lo], Bv = a[hi];
                if ((A < Bv) == desc) {
                    a[lo] = Bv;
                    a[hi] = A;
                }
            }
            c.sync();
        }
    }
}

__device__ __forceinline__ int pow2_at_least(int m)
{
    int p = 64;
    while (p < m) p <<= 1;
    return p;
}

// Emit the entries of B[0, fill) with key >= Tsel (n_sel of them, n_sel <= SORT_MAX),
// sorted, as the row's first `take` outputs, then -1 padding up to k.
// Counting sort: a 2048-bin linear histogram over [Tsel, kmax] (bin 0 = highest keys),
// bin offsets by one group scan, scatter with per-bin cursors, then every entry is
// ranked among the (few) entries that share its bin, in parallel.  Falls back to the
// bitonic sort (in B's memory) when the selection or a bin is too large.
// kmax_sel = 0 means "unknown" (computed here).
template <class G>
__device__ __forceinline__ void emit_sorted(G& c, const Buf& B, const Work& Wk, int fill, uint32_t Tsel,
                                            uint32_t kmax_sel, int n_sel, int take, int k, int32_t* out,
                                            float* out_val)
{
    int32_t* hist = Wk.hist;
    int32_t* cur = Wk.aux;
    zero_ints(c, hist, NBINS);
    uint32_t kmx = kmax_sel;
    if (kmx == 0u) {
        for (int p = c.tid; p < fill; p += G::N) {
            const uint32_t kv = B.key[p];
            if (kv >= Tsel) kmx = max(kmx, kv);
        }
        kmx = group_red1<R_MAX>(c, kmx);  // (barrier also orders the zeroing)
    } else {
        c.sync();
    }
    const uint32_t scale = bin_scale((uint64_t)kmx - Tsel + 1ull);
    bool counting = n_sel <= Wk.csort_cap;
    if (counting) {
        // loads run ahead of the (aliasing) shared atomics: UNR entries per thread per step
        constexpr int UNR = 4;
        for (int p0 = c.tid; p0 < fill; p0 += UNR * G::N) {
            uint32_t kv[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) kv[u] = p0 + u * G::N < fill ? B.key[p0 + u * G::N] : 0u;
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                if (p0 + u * G::N < fill && kv[u] >= Tsel) atomicAdd(&hist[(NBINS - 1) - lin_bin(kv[u] - Tsel, scale)], 1);
        }
        c.sync();
        constexpr int BPT = NBINS / G::N;  // consecutive bins per thread
        const int b0 = c.tid * BPT;
        int h[BPT];
        uint32_t loc = 0, mx = 0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            h[i] = hist[b0 + i];
            loc += (uint32_t)h[i];
            mx = max(mx, (uint32_t)h[i]);
        }
        uint32_t tot;
        uint32_t off = group_excl_scan_max(c, loc, mx, tot, mx);
        counting = mx <= (uint32_t)CSORT_BIN_MAX;
        if (counting) {
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                cur[b0 + i] = (int)off;  // bin start; becomes the bin end after the scatter
                off += (uint32_t)h[i];
            }
            c.sync();
            unsigned long long* cs = Wk.csort;
            for (int p0 = c.tid; p0 < fill; p0 += UNR * G::N) {
                uint32_t kv[UNR];
                int32_t ix[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int p = p0 + u * G::N;
                    kv[u] = p < fill ? B.key[p] : 0u;
                    ix[u] = p < fill ? B.idx[p] : 0;
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    if (p0 + u * G::N < fill && kv[u] >= Tsel) {
                        const int b = (NBINS - 1) - lin_bin(kv[u] - Tsel, scale);
                        const int slot = atomicAdd(&cur[b], 1);
                        cs[slot] = make_comp(kv[u], ix[u]);
                    }
                }
            }
            c.sync();
            // rank every entry inside its (small) bin in parallel: final position = bin
            // start + #entries of the bin with a larger composite; B is free now
            int32_t* fidx = B.idx;
            float* fval = reinterpret_cast<float*>(B.key);
            for (int j = c.tid; j < n_sel; j += G::N) {
                const unsigned long long v = cs[j];
                const int b = (NBINS - 1) - lin_bin(comp_key(v) - Tsel, scale);
                const int cnt = hist[b];
                const int st = cur[b] - cnt;
                int rank = 0;
#pragma unroll 4
                for (int i = st; i < st + cnt; ++i) rank += cs[i] > v;
                const int pos = st + rank;
                if (pos < take) {
                    fidx[pos] = comp_idx(v);
                    fval[pos] = key2f(comp_key(v));
                }
            }
            c.sync();
            for (int j = c.tid; j < k; j += G::N) {
                const bool in = j < take;
                out[j] = in ? fidx[j] : -1;
                if (out_val) out_val[j] = in ? fval[j] : 0.f;
            }
            c.sync();  // B is reused by the caller
            return;
        }
    }
    // bitonic fallback: compact the selection, then sort composites in B's memory
    constexpr int PER = SORT_MAX / G::N;
    unsigned long long v[PER];
    ChunkCounts cc = count_chunks_ge(c, B, fill, Tsel);
    const int m = compact_ge(c, B, fill, Tsel, cc);
    const int P = pow2_at_least(m);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * G::N + c.tid;
        v[j] = 0ull;
        if (p < m) v[j] = make_comp(B.key[p], B.idx[p]);
    }
    c.sync();  // all reads of B done before the aliasing writes
    unsigned long long* comp = B.comp();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * G::N + c.tid;
        if (p < P) comp[p] = v[j];
    }
    c.sync();
    bitonic_sort_desc(c, comp, P);
    for (int j = c.tid; j < k; j += G::N) {
        int32_t idx = -1;
        float val = 0.f;
        if (j < take) {
            idx = comp_idx(comp[j]);
            val = key2f(comp_key(comp[j]));
        }
        out[j] = idx;
        if (out_val) out_val[j] = val;
    }
    c.sync();
}

// Phase 4 fused with the ordered output (R28): the candidates B[0, fill) (all
// keys in [Tlo, kmx]) are counting-sorted into NBINS linear bins (bin 0 = highest keys),
// the bin holding sorted position take-1 is found from the bin scan — the paper's K-th
// bin search over the 2048-bin histogram — and only the bins up to it
// are scattered and ranked (entries ranked inside their bin by the 64-bit composite, so
// the K-th key T* is read off the sorted order instead of being snapped to).  The first
// `take` entries are written, then -1 padding up to k.  Returns false without writing
// when the prefix up to the K-th bin exceeds the sort capacity or one of its bins holds
// more than CSORT_BIN_MAX entries (massive ties); the caller then runs the snap-based
// Phase 4 and emit_sorted.  On success *tstar_out = T*.
template <class G>
__device__ __forceinline__ bool select_sorted(G& c, const Buf& B, const Work& Wk, int fill, uint32_t Tlo, uint32_t kmx,
                                              int take, int k, int32_t* out, float* out_val, uint32_t* tstar_out)
{
    int32_t* hist = Wk.hist;
    int32_t* cur = Wk.aux;
    zero_ints(c, hist, NBINS);
    c.sync();
    const uint32_t scale = bin_scale((uint64_t)kmx - Tlo + 1ull);
    constexpr int UNR = 4;
    for (int p0 = c.tid; p0 < fill; p0 += UNR * G::N) {
        uint32_t kv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) kv[u] = p0 + u * G::N < fill ? B.key[p0 + u * G::N] : 0u;
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (p0 + u * G::N < fill) atomicAdd(&hist[(NBINS - 1) - lin_bin(kv[u] - Tlo, scale)], 1);
    }
    c.sync();
    constexpr int BPT = NBINS / G::N;
    const int b0 = c.tid * BPT;
    int h[BPT];
    uint32_t loc = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
        h[i] = hist[b0 + i];
        loc += (uint32_t)h[i];
    }
    uint32_t tot;
    const uint32_t off0 = group_excl_scan(c, loc, tot);
    // the bin bk that holds sorted position take-1, and the end of the prefix up to it
    {
        uint32_t off = off0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            if ((uint32_t)(take - 1) >= off && (uint32_t)(take - 1) < off + (uint32_t)h[i]) {
                c.misc[12] = b0 + i;
                c.misc[13] = (int)(off + (uint32_t)h[i]);
            }
            off += (uint32_t)h[i];
        }
    }
    c.sync();
    const int bk = c.misc[12];
    const int nsel = c.misc[13];
    uint32_t mx = 0;
#pragma unroll
    for (int i = 0; i < BPT; ++i)
        if (b0 + i <= bk) mx = max(mx, (uint32_t)h[i]);
    mx = group_red1<R_MAX>(c, mx);
    if (nsel > Wk.csort_cap || mx > (uint32_t)CSORT_BIN_MAX) return false;  // group-uniform
    {
        uint32_t off = off0;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            cur[b0 + i] = (int)off;  // bin start; becomes the bin end after the scatter
            off += (uint32_t)h[i];
        }
    }
    c.sync();
    unsigned long long* cs = Wk.csort;
    for (int p0 = c.tid; p0 < fill; p0 += UNR * G::N) {
        uint32_t kv[UNR];
        int32_t ix[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int p = p0 + u * G::N;
            kv[u] = p < fill ? B.key[p] : 0u;
            ix[u] = p < fill ? B.idx[p] : 0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (p0 + u * G::N < fill) {
                const int b = (NBINS - 1) - lin_bin(kv[u] - Tlo, scale);
                if (b <= bk) cs[atomicAdd(&cur[b], 1)] = make_comp(kv[u], ix[u]);
            }
        }
    }
    c.sync();
    int32_t* fidx = B.idx;  // B is free now
    float* fval = reinterpret_cast<float*>(B.key);
    for (int j = c.tid; j < nsel; j += G::N) {
        const unsigned long long v = cs[j];
        const int b = (NBINS - 1) - lin_bin(comp_key(v) - Tlo, scale);
        const int cnt = hist[b];
        const int st = cur[b] - cnt;
        // rank inside the bin; the warp's largest bin picks a fully unrolled, predicated
        // variant so the loads issue back to back instead of one dependent trip at a time
        const int wmax = (int)__reduce_max_sync(__activemask(), (uint32_t)cnt);
        int rank = 0;
        if (wmax <= 4) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < cnt) rank += cs[st + t] > v;
        } else if (wmax <= 8) {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (t < cnt) rank += cs[st + t] > v;
        } else {
            for (int i2 = st; i2 < st + cnt; ++i2) rank += cs[i2] > v;
        }
        const int pos = st + rank;
        if (pos < take) {
            fidx[pos] = comp_idx(v);
            fval[pos] = key2f(comp_key(v));
            if (pos == take - 1) c.misc[14] = (int)comp_key(v);
        }
    }
    c.sync();
    *tstar_out = (uint32_t)c.misc[14];
    for (int j = c.tid; j < k; j += G::N) {
        const bool in = j < take;
        out[j] = in ? fidx[j] : -1;
        if (out_val) out_val[j] = in ? fval[j] : 0.f;
    }
    c.sync();  // B is reused by the caller
    return true;
}

}  // namespace gvr
