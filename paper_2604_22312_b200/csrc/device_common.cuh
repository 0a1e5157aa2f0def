// device_common.cuh — shared device building blocks of the GVR / radix Top-K kernels
// (sm_100a): shared-memory layout, the sortable key transform, block reductions and
// scans over 16 warps, the candidate-buffer count cache and in-place compaction, the
// K-th-bin search, and the ordered-output stage.
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
// Geometry and capacities.
constexpr int NT = 256;                 // threads per CTA (the paper uses 512)
constexpr int NW = NT / 32;             // 8 warps (the paper's K-th-bin search uses 16)
constexpr int KMAX = GVR_MAX_K;         // 2048
constexpr int CWIN = GVR_WINDOW_C;      // Lemma-1 window upper bound C
constexpr int CHUNK_SLOTS = 8;          // buffer slots per thread per compaction chunk
constexpr int CHUNK = NT * CHUNK_SLOTS; // 2048 entries per chunk
constexpr int NCHUNK = 4;
constexpr int CAP = CHUNK * NCHUNK;     // 8192: capacity of the streamed candidate buffer B
constexpr int NBINS = 2048;             // Phase-4 / radix histogram bins
constexpr int VEC = 4;                  // float4 loads per thread per register tile
constexpr int TILE_VEC = NT * VEC;      // float4s per register tile (8192 elements)
constexpr int SORT_MAX = 4096;          // largest bitonic ordered-output sort (64-bit composites)
constexpr int CSORT_MAX = 4096;         // largest counting-sort ordered output
constexpr int CSORT_BIN_MAX = 32;       // counting sort: largest bin ranked in place
constexpr int LIST_MAX = 4096;          // Phase 4: largest K-th-bin member list
constexpr int RADIX_EARLY = 2048;       // radix early exit
constexpr unsigned FULL = 0xffffffffu;

// TMA bulk-copy ring: NSTAGE stages of STAGE_FLOATS fp32 (16 per thread).
constexpr int NSTAGE = 3;
constexpr int STAGE_FLOATS = NT * 16;          // 4096
constexpr int STAGE_BYTES = STAGE_FLOATS * 4;  // 16 KB

static_assert(CAP >= CWIN, "buffer must hold the Lemma-1 window");
static_assert(NBINS % NT == 0 && NBINS / NW % 32 == 0, "bin partitioning");
static_assert(SORT_MAX <= CAP, "bitonic sort array aliases the buffer");

// Shared-memory layout (dynamic): B = {bkey, bidx} is the candidate buffer (the 64-bit
// bitonic sort array aliases it).  The TMA ring is idle once a row has been streamed
// and then hosts the work area: histograms, the K-th-bin member list, counting sort.
constexpr int OFF_BKEY = 0;
constexpr int OFF_BIDX = OFF_BKEY + CAP * 4;
constexpr int OFF_RING = OFF_BIDX + CAP * 4;               // 64 KB, 128-B aligned
constexpr int OFF_WORK = OFF_RING;
constexpr int OFF_HIST = OFF_WORK;                         // int32 [NBINS]     (ring alias)
constexpr int OFF_AUX = OFF_WORK + NBINS * 4;              // int32 [NBINS]     (ring alias)
constexpr int OFF_CSORT = OFF_WORK + 2 * NBINS * 4;        // u64 [CSORT_MAX]   (ring alias)
constexpr int OFF_LIST = OFF_AUX;                          // u32 [LIST_MAX]    (Phase 4 only)
constexpr int WORK_BYTES = 2 * NBINS * 4 + CSORT_MAX * 8;  // 48 KB
constexpr int OFF_BAR = OFF_RING + NSTAGE * STAGE_BYTES;   // u64 [NSTAGE] mbarriers
constexpr int OFF_RED = OFF_BAR + 64;                      // u32 [2][4][NW]
constexpr int OFF_REDF = OFF_RED + 2 * 4 * NW * 4;         // f32 [2][2][NW]
constexpr int OFF_MISC = OFF_REDF + 2 * 2 * NW * 4;        // int32 [32]
constexpr int SMEM_BYTES = OFF_MISC + 32 * 4;              // 115,264 B -> 2 CTAs per SM
static_assert(WORK_BYTES <= NSTAGE * STAGE_BYTES, "work area fits the idle ring");
static_assert(OFF_LIST + LIST_MAX * 4 <= OFF_WORK + WORK_BYTES, "list fits the work area");
static_assert(2 * (SMEM_BYTES + 1024) <= 233472, "two CTAs per SM");

// Named barrier 1 over the CTA's NT threads.
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

extern __shared__ __align__(128) unsigned char g_smem[];

__device__ __forceinline__ uint32_t* s_bkey() { return reinterpret_cast<uint32_t*>(g_smem + OFF_BKEY); }
__device__ __forceinline__ int32_t* s_bidx() { return reinterpret_cast<int32_t*>(g_smem + OFF_BIDX); }
__device__ __forceinline__ unsigned long long* s_comp() { return reinterpret_cast<unsigned long long*>(g_smem + OFF_BKEY); }
__device__ __forceinline__ int32_t* s_hist() { return reinterpret_cast<int32_t*>(g_smem + OFF_HIST); }
__device__ __forceinline__ int32_t* s_aux() { return reinterpret_cast<int32_t*>(g_smem + OFF_AUX); }
__device__ __forceinline__ unsigned long long* s_csort() { return reinterpret_cast<unsigned long long*>(g_smem + OFF_CSORT); }
__device__ __forceinline__ uint32_t* s_list() { return reinterpret_cast<uint32_t*>(g_smem + OFF_LIST); }
__device__ __forceinline__ float* s_ring() { return reinterpret_cast<float*>(g_smem + OFF_RING); }
__device__ __forceinline__ uint32_t* s_red() { return reinterpret_cast<uint32_t*>(g_smem + OFF_RED); }
__device__ __forceinline__ float* s_redf() { return reinterpret_cast<float*>(g_smem + OFF_REDF); }
__device__ __forceinline__ int32_t* s_misc() { return reinterpret_cast<int32_t*>(g_smem + OFF_MISC); }

struct Ctx {
    int tid, lane, warp, par;
};

__device__ __forceinline__ Ctx make_ctx()
{
    Ctx c;
    c.tid = threadIdx.x;
    c.lane = threadIdx.x & 31;
    c.warp = threadIdx.x >> 5;
    c.par = 0;
    return c;
}

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
// Block reductions.  Every call costs one csync(); scratch slots alternate
// (c.par) so back-to-back calls need no second barrier.
enum { R_ADD = 0, R_MIN = 1, R_MAX = 2 };

template <int OP> __device__ __forceinline__ uint32_t wred(uint32_t v)
{
    if (OP == R_ADD) return __reduce_add_sync(FULL, v);
    if (OP == R_MIN) return __reduce_min_sync(FULL, v);
    return __reduce_max_sync(FULL, v);
}
template <int OP> __device__ __forceinline__ uint32_t rident()
{
    return OP == R_MIN ? 0xffffffffu : 0u;
}

template <int O0, int O1, int O2, int O3>
__device__ __forceinline__ void block_red4(Ctx& c, uint32_t& a, uint32_t& b, uint32_t& d, uint32_t& e)
{
    a = wred<O0>(a);
    b = wred<O1>(b);
    d = wred<O2>(d);
    e = wred<O3>(e);
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
        s[2 * NW + c.warp] = d;
        s[3 * NW + c.warp] = e;
    }
    csync();
    const bool in = c.lane < NW;
    a = wred<O0>(in ? s[c.lane] : rident<O0>());
    b = wred<O1>(in ? s[NW + c.lane] : rident<O1>());
    d = wred<O2>(in ? s[2 * NW + c.lane] : rident<O2>());
    e = wred<O3>(in ? s[3 * NW + c.lane] : rident<O3>());
    c.par ^= 1;
}

template <int O0, int O1>
__device__ __forceinline__ void block_red2(Ctx& c, uint32_t& a, uint32_t& b)
{
    a = wred<O0>(a);
    b = wred<O1>(b);
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
    }
    csync();
    const bool in = c.lane < NW;
    a = wred<O0>(in ? s[c.lane] : rident<O0>());
    b = wred<O1>(in ? s[NW + c.lane] : rident<O1>());
    c.par ^= 1;
}

template <int O0>
__device__ __forceinline__ uint32_t block_red1(Ctx& c, uint32_t a)
{
    a = wred<O0>(a);
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 0) s[c.warp] = a;
    csync();
    a = wred<O0>(c.lane < NW ? s[c.lane] : rident<O0>());
    c.par ^= 1;
    return a;
}

// Deterministic fp32 sums of two channels (fixed shuffle tree + fixed warp order).
__device__ __forceinline__ void block_fsum2(Ctx& c, float& a, float& b)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        b += __shfl_xor_sync(FULL, b, o);
    }
    float* s = s_redf() + c.par * 2 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
    }
    csync();
    a = c.lane < NW ? s[c.lane] : 0.f;
    b = c.lane < NW ? s[NW + c.lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(FULL, a, o);
        b += __shfl_xor_sync(FULL, b, o);
    }
    c.par ^= 1;
}

// Exclusive block scan of one u32 per thread (thread order); returns the thread's
// offset and the block total.  Warp shuffles + one barrier: the ballot-free offset
// computation of PAPER.md:600-604.
__device__ __forceinline__ uint32_t block_excl_scan(Ctx& c, uint32_t v, uint32_t& total)
{
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, x, o);
        if (c.lane >= o) x += y;
    }
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 31) s[c.warp] = x;
    csync();
    const uint32_t w = c.lane < NW ? s[c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    total = __reduce_add_sync(FULL, w);
    c.par ^= 1;
    return before + x - v;
}

// Exclusive scan of v plus the block max of m, with one barrier.
__device__ __forceinline__ uint32_t block_excl_scan_max(Ctx& c, uint32_t v, uint32_t m, uint32_t& total,
                                                        uint32_t& mall)
{
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, x, o);
        if (c.lane >= o) x += y;
    }
    const uint32_t wm = __reduce_max_sync(FULL, m);
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 31) {
        s[c.warp] = x;
        s[NW + c.warp] = wm;
    }
    __syncwarp();
    csync();
    const uint32_t w = c.lane < NW ? s[c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    total = __reduce_add_sync(FULL, w);
    mall = __reduce_max_sync(FULL, c.lane < NW ? s[NW + c.lane] : 0u);
    c.par ^= 1;
    return before + x - v;
}

// ---------------------------------------------------------------------------------
// Candidate buffer B: slot p of chunk ch for thread t is ch*CHUNK + j*NT + t.  Counting
// passes cache per-chunk counts (the "count cache" of PAPER.md:588-597, applied to the
// shared-memory buffer) so that the following compaction needs no recount.
struct ChunkCounts {
    uint32_t c[NCHUNK];
};

__device__ __forceinline__ ChunkCounts count_chunks_ge(const Ctx& c, int fill, uint32_t T)
{
    const uint32_t* bkey = s_bkey();
    ChunkCounts cc;
#pragma unroll
    for (int ch = 0; ch < NCHUNK; ++ch) {
        uint32_t n = 0;
        if (ch * CHUNK < fill) {  // block-uniform: skip empty chunks
#pragma unroll
            for (int j = 0; j < CHUNK_SLOTS; ++j) {
                const int p = ch * CHUNK + j * NT + c.tid;
                if (p < fill && bkey[p] >= T) ++n;
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
    for (int ch = 0; ch < NCHUNK; ++ch) s += cc.c[ch];
    return s;
}

// In-place, order-free compaction of B[0, fill) to the entries with key >= T, using
// the cached per-chunk counts of the last count pass at T.  Chunk ch writes only to
// positions below (ch+1)*CHUNK, and every thread has loaded its chunk-ch slots before
// the scan barrier, so no slot is overwritten before it is read.  Returns new fill.
__device__ __forceinline__ int compact_ge(Ctx& c, int fill, uint32_t T, const ChunkCounts& cc)
{
    uint32_t* bkey = s_bkey();
    int32_t* bidx = s_bidx();
    int out_base = 0;
#pragma unroll
    for (int ch = 0; ch < NCHUNK; ++ch) {
        if (ch * CHUNK >= fill) break;  // block-uniform
        uint32_t kk[CHUNK_SLOTS];
        int32_t ii[CHUNK_SLOTS];
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * NT + c.tid;
            kk[j] = 0u;
            ii[j] = 0;
            if (p < fill) {
                kk[j] = bkey[p];
                ii[j] = bidx[p];
            }
        }
        uint32_t tot;
        int pos = out_base + (int)block_excl_scan(c, cc.c[ch], tot);
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * NT + c.tid;
            if (p < fill && kk[j] >= T) {
                bkey[pos] = kk[j];
                bidx[pos] = ii[j];
                ++pos;
            }
        }
        out_base += (int)tot;
    }
    csync();
    return out_base;
}

// Max key over B[0, fill) (thread-local part).
__device__ __forceinline__ uint32_t buffer_max_local(const Ctx& c, int fill)
{
    const uint32_t* bkey = s_bkey();
    uint32_t m = 0;
    for (int p = c.tid; p < fill; p += NT) m = max(m, bkey[p]);
    return m;
}

// ---------------------------------------------------------------------------------
// K-th bin search: find bin b with
//   sum(hist[b+1..nb)) < krem <= sum(hist[b..nb)).
// Each warp owns nb/NW consecutive bins, warp totals are combined from the top, the
// owning lane resolves the exact bin.  Requires 1 <= krem <= sum(hist).
__device__ __forceinline__ void kth_bin(Ctx& c, int nb, uint32_t krem, int& b_out, uint32_t& above_out)
{
    const int32_t* hist = s_hist();
    int32_t* misc = s_misc();
    const int per = nb / NW;  // 128 or 64
    const int q = per / 32;   // 4 or 2
    const int base = c.warp * per + c.lane * q;
    uint32_t ls = 0;
    for (int i = 0; i < q; ++i) ls += (uint32_t)hist[base + i];
    const uint32_t wt = __reduce_add_sync(FULL, ls);
    uint32_t* s = s_red() + c.par * 4 * NW;
    if (c.lane == 0) s[c.warp] = wt;
    csync();
    const uint32_t v = c.lane < NW ? s[c.lane] : 0u;
    const uint32_t above_w = __reduce_add_sync(FULL, (c.lane > c.warp && c.lane < NW) ? v : 0u);
    uint32_t x = ls;  // inclusive suffix over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_down_sync(FULL, x, o);
        if (c.lane + o < 32) x += y;
    }
    const uint32_t above_g = above_w + x - ls;
    if (ls > 0 && above_g < krem && krem <= above_g + ls) {
        uint32_t a = above_g;
        for (int i = q - 1; i >= 0; --i) {
            const uint32_t h = (uint32_t)hist[base + i];
            if (a + h >= krem) {
                misc[0] = base + i;
                misc[1] = (int32_t)a;
                break;
            }
            a += h;
        }
    }
    csync();
    b_out = misc[0];
    above_out = (uint32_t)misc[1];
    c.par ^= 1;
    csync();  // misc may be reused immediately
}

__device__ __forceinline__ void zero_hist(const Ctx& c, int32_t* h, int nb)
{
    for (int i = c.tid; i < nb; i += NT) h[i] = 0;
}

// Smallest s with (width - 1) >> s < NBINS (width in [1, 2^32]).
__device__ __forceinline__ int shift_for_width(uint64_t width)
{
    const uint32_t w = (uint32_t)(width - 1ull);
    const int bits = 32 - __clz(w);  // bits needed for w
    return bits > 11 ? bits - 11 : 0;
}

// ---------------------------------------------------------------------------------
// Ordered output (not part of the paper, whose output is an unordered partition with
// non-deterministic ties): the selected entries are sorted by
// the 64-bit composite (key << 32 | ~idx) descending = (score desc, index asc).

// Bitonic fallback: P (power of two, <= SORT_MAX) composites in the aliasing array.
__device__ __forceinline__ void bitonic_sort_desc(Ctx& c, int P)
{
    unsigned long long* a = s_comp();
    for (int kk = 2; kk <= P; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = c.tid; i < (P >> 1); i += NT) {
                const int lo = 2 * i - (i & (j - 1));
                const int hi = lo + j;
                const bool desc = (lo & kk) == 0;
                const unsigned long long A = a[lo], B = a[hi];
                if ((A < B) == desc) {
                    a[lo] = B;
                    a[hi] = A;
                }
            }
            csync();
        }
    }
}

__device__ __forceinline__ int pow2_at_least(int m)
{
    int p = 64;
    while (p < m) p <<= 1;
    return p;
}

__device__ __forceinline__ void write_output(const Ctx& c, const unsigned long long* sorted, int take, int k,
                                             int32_t* out, float* out_val)
{
    for (int j = c.tid; j < k; j += NT) {
        int32_t idx = -1;
        float val = 0.f;
        if (j < take) {
            const unsigned long long cv = sorted[j];
            idx = comp_idx(cv);
            val = key2f(comp_key(cv));
        }
        out[j] = idx;
        if (out_val) out_val[j] = val;
    }
}

// Linear bin of d = key - Tsel over [0, range) with all NBINS bins in use:
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

// Emit the entries of B[0, fill) with key >= Tsel (n_sel of them, n_sel <= SORT_MAX),
// sorted, as the row's first `take` outputs, then -1 padding up to k.
// Counting sort: a 2048-bin linear histogram over [Tsel, kmax] (bin 0 = highest keys), bin
// offsets by one block scan, scatter with per-bin cursors, then every entry is ranked
// among the (few) entries that share its bin, in parallel.  Falls back to the bitonic sort when the
// selection or a bin is too large.
__device__ __forceinline__ void emit_sorted(Ctx& c, int fill, uint32_t Tsel, uint32_t kmax_sel, int n_sel, int take,
                                            int k, int32_t* out, float* out_val)
{
    uint32_t* bkey = s_bkey();
    int32_t* bidx = s_bidx();
    int32_t* hist = s_hist();
    int32_t* cur = s_aux();
    zero_hist(c, hist, NBINS);
    uint32_t kmx = kmax_sel;
    if (kmx == 0u) {  // not known by the caller
        for (int p = c.tid; p < fill; p += NT) {
            const uint32_t kv = bkey[p];
            if (kv >= Tsel) kmx = max(kmx, kv);
        }
        kmx = block_red1<R_MAX>(c, kmx);  // (barrier also orders the zeroing)
    } else {
        csync();
    }
    const uint32_t scale = bin_scale((uint64_t)kmx - Tsel + 1ull);
    bool counting = n_sel <= CSORT_MAX;
    if (counting) {
        for (int p = c.tid; p < fill; p += NT) {
            const uint32_t kv = bkey[p];
            if (kv >= Tsel) atomicAdd(&hist[(NBINS - 1) - lin_bin(kv - Tsel, scale)], 1);
        }
        csync();
        // exclusive scan over bins (BPT consecutive bins per thread)
        constexpr int BPT = NBINS / NT;
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
        uint32_t off = block_excl_scan_max(c, loc, mx, tot, mx);
        counting = mx <= (uint32_t)CSORT_BIN_MAX;
        if (counting) {
#pragma unroll
            for (int i = 0; i < BPT; ++i) {
                cur[b0 + i] = (int)off;  // bin start; becomes the bin end after the scatter
                off += (uint32_t)h[i];
            }
            csync();
            unsigned long long* cs = s_csort();
            for (int p = c.tid; p < fill; p += NT) {
                const uint32_t kv = bkey[p];
                if (kv >= Tsel) {
                    const int b = (NBINS - 1) - lin_bin(kv - Tsel, scale);
                    const int slot = atomicAdd(&cur[b], 1);
                    cs[slot] = make_comp(kv, bidx[p]);
                }
            }
            csync();
            // rank every entry inside its (small) bin in parallel: final position =
            // bin start + #entries of the bin with a larger composite; B is free now
            int32_t* fidx = s_bidx();
            float* fval = reinterpret_cast<float*>(s_bkey());
            for (int j = c.tid; j < n_sel; j += NT) {
                const unsigned long long v = cs[j];
                const int b = (NBINS - 1) - lin_bin(comp_key(v) - Tsel, scale);
                const int cnt = hist[b];
                const int st = cur[b] - cnt;
                int rank = 0;
                for (int i = st; i < st + cnt; ++i) rank += cs[i] > v;
                const int pos = st + rank;
                if (pos < take) {
                    fidx[pos] = comp_idx(v);
                    fval[pos] = key2f(comp_key(v));
                }
            }
            csync();
            for (int j = c.tid; j < k; j += NT) {
                const bool in = j < take;
                out[j] = in ? fidx[j] : -1;
                if (out_val) out_val[j] = in ? fval[j] : 0.f;
            }
            return;
        }
    }
    // bitonic fallback: gather the selection into the aliasing composite array
    constexpr int PER = SORT_MAX / NT;  // 16
    unsigned long long v[PER];
    // compact the selected entries of this thread's slots first (order-free)
    ChunkCounts cc = count_chunks_ge(c, fill, Tsel);
    const int m = compact_ge(c, fill, Tsel, cc);
    const int P = pow2_at_least(m);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * NT + c.tid;
        v[j] = 0ull;
        if (p < m) v[j] = make_comp(bkey[p], bidx[p]);
    }
    csync();  // all reads of B done before the aliasing writes
    unsigned long long* comp = s_comp();
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * NT + c.tid;
        if (p < P) comp[p] = v[j];
    }
    csync();
    bitonic_sort_desc(c, P);
    write_output(c, comp, take, k, out, out_val);
}

}  // namespace gvr
