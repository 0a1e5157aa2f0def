// device_common.cuh — shared device building blocks of the GVR / radix Top-K kernels
// (sm_100a).  Block-level reductions and scans over 16 warps, the sortable key
// transform, the shared-memory candidate buffer layout, the in-place chunked
// compaction, the K-th-bin search, and the ordered-output block sort.
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
constexpr int NT = 512;                 // threads per CTA
constexpr int NW = NT / 32;             // 16 warps
constexpr int KMAX = GVR_MAX_K;         // 2048
constexpr int CWIN = GVR_WINDOW_C;      // Lemma-1 window upper bound C
constexpr int CHUNK_SLOTS = 8;          // buffer slots per thread per compaction chunk
constexpr int CHUNK = NT * CHUNK_SLOTS; // 4096 entries per chunk
constexpr int NCHUNK = 3;
constexpr int CAP = CHUNK * NCHUNK;     // 12288: capacity of the streamed candidate buffer B
constexpr int NBINS = 2048;             // Phase-4 / radix histogram bins
constexpr int VEC = 4;                  // float4 loads per thread per tile
constexpr int TILE_VEC = NT * VEC;      // float4s per tile (8192 elements)
constexpr int SORT_MAX = 8192;          // largest ordered-output sort (64-bit composites)
constexpr int RADIX_EARLY = 2048;       // radix early exit
constexpr unsigned FULL = 0xffffffffu;

static_assert(CAP >= CWIN, "buffer must hold the Lemma-1 window");
static_assert(SORT_MAX * 8 <= CAP * 8, "sort array aliases the buffer");

// Shared-memory layout (dynamic).  B = {bkey, bidx} is the candidate buffer; the
// 64-bit sort array aliases its first SORT_MAX*8 bytes.
constexpr int OFF_BKEY = 0;
constexpr int OFF_BIDX = OFF_BKEY + CAP * 4;
constexpr int OFF_HIST = OFF_BIDX + CAP * 4;
constexpr int OFF_RED = OFF_HIST + NBINS * 4;      // u32 [2][4][NW]
constexpr int OFF_REDF = OFF_RED + 2 * 4 * NW * 4; // f32 [2][2][NW]
constexpr int OFF_MISC = OFF_REDF + 2 * 2 * NW * 4;
constexpr int SMEM_BYTES = OFF_MISC + 32 * 4;      // 107,392 B -> 2 CTAs per SM

struct Ctx {
    int tid, lane, warp, par;
    uint32_t* bkey;
    int32_t* bidx;
    unsigned long long* comp;
    int32_t* hist;
    uint32_t* red;
    float* redf;
    int32_t* misc;
};

__device__ __forceinline__ Ctx make_ctx(unsigned char* smem)
{
    Ctx c;
    c.tid = threadIdx.x;
    c.lane = threadIdx.x & 31;
    c.warp = threadIdx.x >> 5;
    c.par = 0;
    c.bkey = reinterpret_cast<uint32_t*>(smem + OFF_BKEY);
    c.bidx = reinterpret_cast<int32_t*>(smem + OFF_BIDX);
    c.comp = reinterpret_cast<unsigned long long*>(smem + OFF_BKEY);
    c.hist = reinterpret_cast<int32_t*>(smem + OFF_HIST);
    c.red = reinterpret_cast<uint32_t*>(smem + OFF_RED);
    c.redf = reinterpret_cast<float*>(smem + OFF_REDF);
    c.misc = reinterpret_cast<int32_t*>(smem + OFF_MISC);
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
// Block reductions.  Every call costs one __syncthreads(); scratch slots alternate
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
    uint32_t* s = c.red + c.par * 4 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
        s[2 * NW + c.warp] = d;
        s[3 * NW + c.warp] = e;
    }
    __syncthreads();
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
    uint32_t* s = c.red + c.par * 4 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
    }
    __syncthreads();
    const bool in = c.lane < NW;
    a = wred<O0>(in ? s[c.lane] : rident<O0>());
    b = wred<O1>(in ? s[NW + c.lane] : rident<O1>());
    c.par ^= 1;
}

template <int O0>
__device__ __forceinline__ uint32_t block_red1(Ctx& c, uint32_t a)
{
    a = wred<O0>(a);
    uint32_t* s = c.red + c.par * 4 * NW;
    if (c.lane == 0) s[c.warp] = a;
    __syncthreads();
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
    float* s = c.redf + c.par * 2 * NW;
    if (c.lane == 0) {
        s[c.warp] = a;
        s[NW + c.warp] = b;
    }
    __syncthreads();
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
    uint32_t* s = c.red + c.par * 4 * NW;
    if (c.lane == 31) s[c.warp] = x;
    __syncthreads();
    const uint32_t w = c.lane < NW ? s[c.lane] : 0u;
    const uint32_t before = __reduce_add_sync(FULL, c.lane < c.warp ? w : 0u);
    total = __reduce_add_sync(FULL, w);
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
    ChunkCounts cc;
#pragma unroll
    for (int ch = 0; ch < NCHUNK; ++ch) {
        uint32_t n = 0;
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * NT + c.tid;
            if (p < fill && c.bkey[p] >= T) ++n;
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
                kk[j] = c.bkey[p];
                ii[j] = c.bidx[p];
            }
        }
        uint32_t tot;
        int pos = out_base + (int)block_excl_scan(c, cc.c[ch], tot);
#pragma unroll
        for (int j = 0; j < CHUNK_SLOTS; ++j) {
            const int p = ch * CHUNK + j * NT + c.tid;
            if (p < fill && kk[j] >= T) {
                c.bkey[pos] = kk[j];
                c.bidx[pos] = ii[j];
                ++pos;
            }
        }
        out_base += (int)tot;
    }
    __syncthreads();
    return out_base;
}

// Max key over B[0, fill).
__device__ __forceinline__ uint32_t buffer_max_local(const Ctx& c, int fill)
{
    uint32_t m = 0;
    for (int p = c.tid; p < fill; p += NT) m = max(m, c.bkey[p]);
    return m;
}

// ---------------------------------------------------------------------------------
// K-th bin search: find bin b with
//   sum(hist[b+1..nb)) < krem <= sum(hist[b..nb)).
// Each warp owns nb/NW consecutive bins, warp totals are combined from the top, the
// owning lane resolves the exact bin.  Requires 1 <= krem <= sum(hist).
__device__ __forceinline__ void kth_bin(Ctx& c, int nb, uint32_t krem, int& b_out, uint32_t& above_out)
{
    const int per = nb / NW;  // 128 or 64
    const int q = per / 32;   // 4 or 2
    const int base = c.warp * per + c.lane * q;
    uint32_t ls = 0;
    for (int i = 0; i < q; ++i) ls += (uint32_t)c.hist[base + i];
    const uint32_t wt = __reduce_add_sync(FULL, ls);
    uint32_t* s = c.red + c.par * 4 * NW;
    if (c.lane == 0) s[c.warp] = wt;
    __syncthreads();
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
            const uint32_t h = (uint32_t)c.hist[base + i];
            if (a + h >= krem) {
                c.misc[0] = base + i;
                c.misc[1] = (int32_t)a;
                break;
            }
            a += h;
        }
    }
    __syncthreads();
    b_out = c.misc[0];
    above_out = (uint32_t)c.misc[1];
    c.par ^= 1;
    __syncthreads();  // misc may be reused immediately
}

__device__ __forceinline__ void zero_hist(const Ctx& c, int nb)
{
    for (int i = c.tid; i < nb; i += NT) c.hist[i] = 0;
}

// ---------------------------------------------------------------------------------
// Ordered output: bitonic sort of P (power of two, <= SORT_MAX) 64-bit composites in
// shared memory, descending, so that position j holds the j-th element of the
// (score desc, index asc) order.
__device__ __forceinline__ void bitonic_sort_desc(Ctx& c, int P)
{
    unsigned long long* a = c.comp;
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
            __syncthreads();
        }
    }
}

__device__ __forceinline__ int pow2_at_least(int m)
{
    int p = 64;
    while (p < m) p <<= 1;
    return p;
}

// Build composites from B[0, m) into the aliasing sort array, sort, and write the
// first `take` entries as the row's output (indices, optional values) followed by -1
// padding up to k.  m <= SORT_MAX.
__device__ __forceinline__ void sort_and_emit(Ctx& c, int m, int take, int k, int32_t* out,
                                              float* out_val)
{
    const int P = pow2_at_least(m);
    constexpr int PER = SORT_MAX / NT;  // 16
    unsigned long long v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * NT + c.tid;
        v[j] = 0ull;
        if (p < m) v[j] = make_comp(c.bkey[p], c.bidx[p]);
    }
    __syncthreads();  // all reads of B done before the aliasing writes
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int p = j * NT + c.tid;
        if (p < P) c.comp[p] = v[j];
    }
    __syncthreads();
    bitonic_sort_desc(c, P);
    for (int j = c.tid; j < k; j += NT) {
        int32_t idx = -1;
        float val = 0.f;
        if (j < take) {
            const unsigned long long cv = c.comp[j];
            idx = (int32_t)(~(uint32_t)(cv & 0xffffffffull));
            val = key2f((uint32_t)(cv >> 32));
        }
        out[j] = idx;
        if (out_val) out_val[j] = val;
    }
}

}  // namespace gvr
