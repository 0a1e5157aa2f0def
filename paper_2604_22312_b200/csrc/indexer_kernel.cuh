// indexer_kernel.cuh — the DSA indexer scores (Eq. 1, lines 78-81) on tensor
// cores, and the fused indexer -> GVR Top-K path.
//
//   I_t[i] = sum_j W_j * ReLU(Q_j . K_i),  j < 64 heads, Q_j, K_i in R^128 (bf16 inputs,
//   fp32 accumulation; the keys already RoPE'd, as the indexer cache holds them).
//
// Per 64-key tile the 64 x 64 head-by-key dot products are one bf16 MMA block (mma.sync
// m16n8k16, fp32 accumulators): warp w owns heads 16 (w & 3) .. + 15 and keys 32 (w >> 2)
// .. + 31 (4 n-tiles of 8 keys, 8 k-steps of 16 dims); its Q fragments stay in registers
// for the whole row.  The epilogue applies ReLU and the head weights, sums the warp's 16
// heads with a fixed shuffle tree and the 4 head blocks in a fixed order — one function
// (score_tile) used by every path, so the fused and the materialising kernels produce the
// same fp32 scores bit for bit.  Keys and Q are staged into shared memory with cp.async
// (16-byte chunks, XOR-swizzled by row so ldmatrix is conflict-free).
//
// The op is memory bound on the key cache (256 B per key for 2 x 64 x 128 FLOP: 64 FLOP/B,
// under B200's ridge for any tensor-core path), so mma.sync suffices here.
//
// Fused path (gvr_indexer_topk_batched): indexer_guess_kernel computes the scores at the
// guessed positions and at the 4096 row-sample positions and runs Phases 1-2 on them
// (phase12_core); indexer_filter_kernel streams the key cache once (persistent CTAs, the
// filter kernel's tile partition with 256-key steps), computes each step's 256 scores and
// collects those >= T_c into the candidate lists; gvr_refine_kernel selects each row from
// its list.  The score row never exists in memory.  Rows the lists cannot finish (and
// rows of <= k keys) are materialised into the caller's scratch row by the fixup kernel
// (indexer_fixup_kernel) and finished by the row path.
#pragma once
#include <cuda_bf16.h>

#include "refine_kernel.cuh"

namespace gvr {

constexpr int IX_D = 128;     // head dim of the indexer (DSV3.2)
constexpr int IX_H = 64;      // indexer heads
constexpr int IX_TILE = 64;   // keys per MMA tile
constexpr int IX_NT = 256;    // 8 warps
constexpr int IX_STEP = 4;    // tiles per filter step (256 keys, 64 KB of keys)
static_assert(IX_NT == 8 * 32, "eight warps: 4 head blocks x 2 key halves");

struct IndexerArgs {
    const __nv_bfloat16* keys;  // [num_sets][n_max][128], row-major
    int64_t n_max;              // keys per set
    const int32_t* row_set;     // [num_rows]: the key set of each row
    const __nv_bfloat16* q;     // [num_rows][64][128]
    const float* w;             // [num_rows][64]
};

// ---- shared-memory tiles: 64 rows x 256 B, 16-byte chunk c of row r at chunk c ^ (r & 7)
__device__ __forceinline__ uint32_t swz(int row, int chunk) { return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4)); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid)
{
    const int sz = valid ? 16 : 0;  // 0: zero-fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Stage 64 rows of 128 bf16 into a swizzled tile: row i from src_row(i) (nullptr: zeros).
template <class RowFn>
__device__ __forceinline__ void load_tile64(uint32_t tile, int tid, RowFn&& src_row)
{
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int q = tid + u * IX_NT;  // 1024 chunks of 16 B
        const int row = q >> 4, ch = q & 15;
        const __nv_bfloat16* s = src_row(row);
        cp_async16(tile + swz(row, ch), s ? (const void*)(s + ch * 8) : (const void*)src_row(-1), s != nullptr);
    }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3)
{
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// The warp's Q fragments (heads 16 hb .. + 15, all 8 k-steps) from the swizzled Q tile.
struct QFrag {
    uint32_t a[8][4];
};
__device__ __forceinline__ void load_qfrag(QFrag& f, uint32_t qtile, int warp, int lane)
{
    const int hb = warp & 3;
    const int row = 16 * hb + (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
    for (int s = 0; s < 8; ++s) ldsm_x4(qtile + swz(row, 2 * s + (lane >> 4)), f.a[s][0], f.a[s][1], f.a[s][2], f.a[s][3]);
}

// Scores of the 64 keys of a staged key tile: out[i] for key i of the tile.  Every warp's
// partial sums go to part[4][64]; the caller synchronises before and after (out and part
// are shared).  W: the 64 head weights in shared memory.
__device__ __forceinline__ void score_tile(const QFrag& f, uint32_t ktile, const float* W, float* part, int warp,
                                           int lane)
{
    const int hb = warp & 3, kh = warp >> 2;
    float acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {  // two n-tiles of 8 keys per ldmatrix.x4
            const int key = 32 * kh + 16 * jj + (lane & 7) + ((lane >> 4) << 3);
            const int ch = 2 * s + ((lane >> 3) & 1);
            uint32_t b0, b1, b2, b3;
            ldsm_x4(ktile + swz(key, ch), b0, b1, b2, b3);
            mma_bf16(acc[2 * jj], f.a[s], b0, b1);
            mma_bf16(acc[2 * jj + 1], f.a[s], b2, b3);
        }
    }
    // epilogue: ReLU, head weights, sum over the warp's 16 heads (rows g and g + 8 of the
    // m16 tile in this thread, then the 8 row groups by a fixed xor-shuffle tree)
    const int g = lane >> 2, t = lane & 3;
    const float w0 = W[16 * hb + g], w1 = W[16 * hb + g + 8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float v0 = __fmaf_rn(w1, fmaxf(acc[j][2], 0.f), __fmul_rn(w0, fmaxf(acc[j][0], 0.f)));
        float v1 = __fmaf_rn(w1, fmaxf(acc[j][3], 0.f), __fmul_rn(w0, fmaxf(acc[j][1], 0.f)));
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            v0 = __fadd_rn(v0, __shfl_xor_sync(FULL, v0, o));
            v1 = __fadd_rn(v1, __shfl_xor_sync(FULL, v1, o));
        }
        if (g == 0) {
            const int key = 32 * kh + 8 * j + 2 * t;
            part[hb * IX_TILE + key] = v0;
            part[hb * IX_TILE + key + 1] = v1;
        }
    }
}
// key i's score from the 4 head blocks' partial sums (fixed order)
__device__ __forceinline__ float tile_score(const float* part, int i)
{
    return __fadd_rn(__fadd_rn(__fadd_rn(part[i], part[IX_TILE + i]), part[2 * IX_TILE + i]), part[3 * IX_TILE + i]);
}

// shared-memory layout of the indexer kernels
constexpr int IX_OFF_Q = 0;                               // Q tile, 16 KB
constexpr int IX_OFF_K = IX_OFF_Q + 16384;                // 2 x IX_STEP key tiles, 128 KB
constexpr int IX_OFF_W = IX_OFF_K + 2 * IX_STEP * 16384;  // head weights, 256 B
constexpr int IX_OFF_PART = IX_OFF_W + IX_H * 4;          // partial sums [4][64]
constexpr int IX_OFF_SC = IX_OFF_PART + 4 * IX_TILE * 4;  // scores of a step [256] / guess scratch
constexpr int IX_OFF_CUR = IX_OFF_SC + IX_STEP * IX_TILE * 4;
constexpr int IX_OFF_SCR = IX_OFF_CUR + 16;
constexpr int IX_SMEM_BYTES = IX_OFF_SCR + GROUP_SCRATCH_BYTES;

// Stage row r's Q (cp.async, swizzled) and W, and wait for them.
__device__ __forceinline__ void load_row_q(const IndexerArgs& ia, int r, uint32_t qtile, float* W, int tid)
{
    const __nv_bfloat16* qr = ia.q + (int64_t)r * IX_H * IX_D;
    load_tile64(qtile, tid, [&](int row) { return row < 0 ? qr : qr + row * IX_D; });
    cp_async_commit();
    if (tid < IX_H) W[tid] = __ldg(ia.w + (int64_t)r * IX_H + tid);
}

// ---------------------------------------------------------------------------------
// Materialised scores: out[r][i] for i < row_lens[r] (the unfused indexer, and the fixup's
// score row).  Grid: (tiles, rows); CTA (x, r) scores tiles x, x + gridDim.x, ... of row r.
__global__ void __launch_bounds__(IX_NT)
indexer_scores_kernel(IndexerArgs ia, const int32_t* __restrict__ row_lens, float* __restrict__ out,
                      int64_t out_stride)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t sbase = smem_u32(smem);
    float* W = reinterpret_cast<float*>(smem + IX_OFF_W);
    float* part = reinterpret_cast<float*>(smem + IX_OFF_PART);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = blockIdx.y;
    const int n = row_lens ? min(max(__ldg(row_lens + r), 0), (int)ia.n_max) : (int)ia.n_max;
    const __nv_bfloat16* kb = ia.keys + (int64_t)__ldg(ia.row_set + r) * ia.n_max * IX_D;
    load_row_q(ia, r, sbase + IX_OFF_Q, W, tid);
    cp_async_wait<0>();
    __syncthreads();
    QFrag f;
    load_qfrag(f, sbase + IX_OFF_Q, warp, lane);
    const int ntiles = (n + IX_TILE - 1) / IX_TILE;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint32_t kt = sbase + IX_OFF_K;
        load_tile64(kt, tid, [&](int row) {
            const int key = t * IX_TILE + row;
            return row < 0 ? kb : (key < n ? kb + (int64_t)key * IX_D : nullptr);
        });
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        score_tile(f, kt, W, part, warp, lane);
        __syncthreads();
        if (tid < IX_TILE && t * IX_TILE + tid < n) out[(int64_t)r * out_stride + t * IX_TILE + tid] = tile_score(part, tid);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------
// A pipeline of 64-key tiles through NBUF shared buffers (cp.async groups, one per tile):
// tile u's rows come from rows(u, i) (key index or -1 for zeros); consume(u) runs after
// the tile's scores are in part[] (all threads, between barriers).
template <int NBUF, class Rows, class Consume>
__device__ __forceinline__ void score_tiles(const QFrag& f, uint32_t kbuf, const float* W, float* part,
                                            const __nv_bfloat16* kb, int ntiles_u, Rows&& rows, Consume&& consume,
                                            int tid, int warp, int lane)
{
    auto issue = [&](int u) {
        const uint32_t dst = kbuf + (uint32_t)(u % NBUF) * 16384u;
        load_tile64(dst, tid, [&](int row) {
            if (row < 0) return kb;
            const int key = rows(u, row);
            return key >= 0 ? kb + (int64_t)key * IX_D : (const __nv_bfloat16*)nullptr;
        });
    };
#pragma unroll
    for (int u = 0; u < NBUF - 1; ++u) {
        if (u < ntiles_u) issue(u);
        cp_async_commit();
    }
    for (int u = 0; u < ntiles_u; ++u) {
        if (u + NBUF - 1 < ntiles_u) issue(u + NBUF - 1);
        cp_async_commit();
        cp_async_wait<NBUF - 1>();  // tile u has landed
        __syncthreads();
        score_tile(f, kbuf + (uint32_t)(u % NBUF) * 16384u, W, part, warp, lane);
        __syncthreads();
        consume(u);
        __syncthreads();  // part[] and the buffer are reused
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------
// Fused Phases 1-2 (gvr_indexer_topk_batched): one CTA per row computes the scores at the
// guessed positions and at the 4096 row-sample positions (sample_off: 256 chunks of 16
// consecutive keys spread over the row — the score path's sample with head 0)
// and runs phase12_core on them.  Rows with no tiles go to the ready queue.
constexpr int IXG_OFF_Q = 0;
constexpr int IXG_OFF_K = 16384;                       // 4 tile buffers
constexpr int IXG_OFF_W = IXG_OFF_K + 4 * 16384;
constexpr int IXG_OFF_PART = IXG_OFF_W + IX_H * 4;
constexpr int IXG_OFF_SS = IXG_OFF_PART + 4 * IX_TILE * 4;  // sample scores [4096]
constexpr int IXG_OFF_GS = IXG_OFF_SS + P2_S * 4;           // guess scores [2048]
constexpr int IXG_OFF_GI = IXG_OFF_GS + KMAX * 4;           // guess positions [2048]
constexpr int IXG_OFF_SH = IXG_OFF_GI + KMAX * 4;           // 256-bin histogram
constexpr int IXG_OFF_SCR = IXG_OFF_SH + 256 * 4;
constexpr int IXG_SMEM_BYTES = IXG_OFF_SCR + GROUP_SCRATCH_BYTES;

__global__ void __launch_bounds__(IX_NT)
indexer_guess_kernel(IndexerArgs ia, const float* __restrict__ scratch, const int32_t* __restrict__ row_lens,
                     const int32_t* prev, int k, GvrParams prm, GuessOut* __restrict__ gp, BatchQueue bq)
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t sbase = smem_u32(smem);
    float* W = reinterpret_cast<float*>(smem + IXG_OFF_W);
    float* part = reinterpret_cast<float*>(smem + IXG_OFF_PART);
    float* ss = reinterpret_cast<float*>(smem + IXG_OFF_SS);
    float* gsc = reinterpret_cast<float*>(smem + IXG_OFF_GS);
    int32_t* gpos = reinterpret_cast<int32_t*>(smem + IXG_OFF_GI);
    Group<IX_NT, 1> c;
    c.init(threadIdx.x, smem + IXG_OFF_SCR);
    const int tid = c.tid, warp = c.warp, lane = c.lane;
    const int r = blockIdx.x;
    int32_t gi[GUESS_PER_THREAD];
    load_guess_idx(c, prev ? prev + (int64_t)r * k : nullptr, k, prm, gi);
    const RowPlan p = plan_row(scratch, ia.n_max, row_lens, r, k);
    if (bq.queue && p.ntiles == 0 && tid == 0) st_release(bq.queue + atomicAdd(bq.qctl + Q_TAIL, 1), r + 1);
    if (p.n <= k) return;
    GuessOut g;
    if (p.n <= GVR_CAP) {  // collect everything, no search
        g = GuessOut{};
        g.top = 0xffffffffu;
        g.exit = GVR_P2_ALL;
    } else {
        const int n = p.n;
        const __nv_bfloat16* kb = ia.keys + (int64_t)__ldg(ia.row_set + r) * ia.n_max * IX_D;
        load_row_q(ia, r, sbase + IXG_OFF_Q, W, tid);
#pragma unroll
        for (int j = 0; j < GUESS_PER_THREAD; ++j) gpos[tid + j * IX_NT] = (gi[j] >= 0 && gi[j] < n) ? gi[j] : -1;
        cp_async_wait<0>();
        __syncthreads();
        QFrag f;
        load_qfrag(f, sbase + IXG_OFF_Q, warp, lane);
        // guessed slots used: blocks of 8 ranks every 8 gs ranks while the rank is < k
        const int gs = prm.guess_stride;
        const int nslots = min(KMAX, 8 * ((k + 8 * gs - 1) / (8 * gs)));
        const int gtiles = (nslots + IX_TILE - 1) / IX_TILE;
        score_tiles<4>(
            f, sbase + IXG_OFF_K, W, part, kb, P2_S / IX_TILE + gtiles,
            [&](int u, int i) {
                if (u < P2_S / IX_TILE) {  // sample tile: chunks 4u .. 4u + 3
                    const int cidx = 4 * u + (i >> 4);  // the thread whose sample value this is
                    return sample_off(cidx, n) + (i & 15);
                }
                const int slot = (u - P2_S / IX_TILE) * IX_TILE + i;
                return slot < nslots ? gpos[slot] : -1;
            },
            [&](int u) {
                if (tid < IX_TILE) {
                    const float v = tile_score(part, tid);
                    if (u < P2_S / IX_TILE)
                        ss[u * IX_TILE + tid] = v;
                    else
                        gsc[(u - P2_S / IX_TILE) * IX_TILE + tid] = v;
                }
            },
            tid, warp, lane);
        __syncthreads();
        float sv[P2_CHUNK], gv[GUESS_PER_THREAD];
        uint32_t valid = 0u;
#pragma unroll
        for (int q2 = 0; q2 < P2_CHUNK; ++q2) sv[q2] = ss[P2_CHUNK * tid + q2];
#pragma unroll
        for (int j = 0; j < GUESS_PER_THREAD; ++j) {
            const int slot = tid + j * IX_NT;
            gv[j] = 0.f;
            if (slot < nslots && gpos[slot] >= 0) {
                gv[j] = gsc[slot];
                valid |= 1u << j;
            }
        }
        g = phase12_core(c, n, gv, valid, sv, k, prm, reinterpret_cast<int32_t*>(smem + IXG_OFF_SH));
        if (bq.queue && g.exit == GVR_P2_TIES && g.tie < 0xffffffffu) g.Tc = g.tie + 1u;
    }
    if (tid == 0) gp[r] = g;
}

// ---------------------------------------------------------------------------------
// Fused HBM pass: the key cache streamed once.  The batch's rows form the score filter's
// virtual tile sequence (tpr tiles of 4096 keys per row, the row plan of the scratch
// layout); a persistent grid of one CTA per SM takes contiguous equal ranges, so a row is
// covered by at most F_SEGS CTAs.  Each tile is scored in steps of 256 keys (4 MMA tiles,
// double-buffered cp.async), each step's scores tested against T_c and the candidates
// (key, index) appended to the CTA's region — the lists the refine kernel reads.
// One virtual 4096-key tile at a time of a CTA's range (the filter kernel's RoundIter with
// one tile per step); t0 = the tile, last = the last tile of this CTA's part of row r.
struct IxTileIter {
    long long v, ve;
    int r, t, loaded = -1, t0 = 0, nt = 0;
    RowPlan p;
    bool last = false;
    __device__ __forceinline__ void start(long long vb, long long vend, int tpr)
    {
        v = vb;
        ve = vend;
        r = (int)(vb / tpr);
        t = (int)(vb - (long long)r * tpr);
    }
    __device__ __forceinline__ bool next(const float* base, int64_t stride, const int32_t* row_lens, int k, int tpr)
    {
        while (v < ve) {
            if (loaded != r) {
                loaded = r;
                p = plan_row(base, stride, row_lens, r, k);
            }
            if (t >= p.ntiles) {
                v += tpr - t;
                ++r;
                t = 0;
                continue;
            }
            t0 = t;
            nt = 1;
            ++v;
            ++t;
            last = t >= p.ntiles || v >= ve;
            return true;
        }
        return false;
    }
};

constexpr int IXF_OFF_Q = 0;
constexpr int IXF_OFF_K = 16384;  // 2 steps x 4 tiles
constexpr int IXF_OFF_W = IXF_OFF_K + 2 * IX_STEP * 16384;
constexpr int IXF_OFF_PART = IXF_OFF_W + IX_H * 4;
constexpr int IXF_OFF_SC = IXF_OFF_PART + 4 * IX_TILE * 4;
constexpr int IXF_OFF_CUR = IXF_OFF_SC + IX_STEP * IX_TILE * 4;
constexpr int IXF_OFF_SCR = IXF_OFF_CUR + 16;
constexpr int IXF_SMEM_BYTES = IXF_OFF_SCR + GROUP_SCRATCH_BYTES;

__global__ void __launch_bounds__(IX_NT, 1)
indexer_filter_kernel(IndexerArgs ia, const float* __restrict__ scratch, const int32_t* __restrict__ row_lens, int k,
                      const GuessOut* __restrict__ gp, CandLists cl, BatchQueue bq)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t sbase = smem_u32(smem);
    float* W = reinterpret_cast<float*>(smem + IXF_OFF_W);
    float* part = reinterpret_cast<float*>(smem + IXF_OFF_PART);
    float* sc = reinterpret_cast<float*>(smem + IXF_OFF_SC);
    int* cursor = reinterpret_cast<int*>(smem + IXF_OFF_CUR);
    uint32_t* seg_kmax = reinterpret_cast<uint32_t*>(smem + IXF_OFF_CUR + 4);
    Group<IX_NT, 1> c;
    c.init(threadIdx.x, smem + IXF_OFF_SCR);
    const int tid = c.tid, warp = c.warp, lane = c.lane;
    const int b = blockIdx.x;
    if (tid == 0) {
        *cursor = 0;
        *seg_kmax = 0u;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // gp (Phases 1-2) is complete and visible
    __syncthreads();
    uint2* reg = cl.region + (long long)b * cl.reg;
    const int regcap = cl.reg;
    const uint64_t keep = policy_evict_last();
    IxTileIter it;
    it.start(cl_begin(cl, b), cl_begin(cl, b + 1), cl.tpr);
    int cur_r = -1, seg_start = 0;
    uint32_t tck = 0u;
    QFrag f;
    const __nv_bfloat16* kb = nullptr;
    while (it.next(scratch, ia.n_max, row_lens, k, cl.tpr)) {
        const RowPlan& p = it.p;
        if (it.r != cur_r) {  // a new row: its query, weights and threshold
            cur_r = it.r;
            tck = __ldcg(&gp[cur_r].Tc);
            kb = ia.keys + (int64_t)__ldg(ia.row_set + cur_r) * ia.n_max * IX_D;
            __syncthreads();  // the previous row's fragments are out of use
            load_row_q(ia, cur_r, sbase + IXF_OFF_Q, W, tid);
            cp_async_wait<0>();
            __syncthreads();
            load_qfrag(f, sbase + IXF_OFF_Q, warp, lane);
        }
        const int key0 = it.t0 * STAGE_FLOATS;
        const int key1 = (it.t0 + it.nt == p.ntiles) ? p.n : key0 + it.nt * STAGE_FLOATS;  // last tile: the tail too
        const int nsteps = (key1 - key0 + IX_STEP * IX_TILE - 1) / (IX_STEP * IX_TILE);
        const float Tf = key2f(tck);
        uint32_t kmax = 0u;
        score_tiles<2 * IX_STEP>(
            f, sbase + IXF_OFF_K, W, part, kb, nsteps * IX_STEP,
            [&](int u, int i) {
                const int key = key0 + u * IX_TILE + i;
                return key < key1 ? key : -1;
            },
            [&](int u) {
                if (tid < IX_TILE) sc[(u % IX_STEP) * IX_TILE + tid] = tile_score(part, tid);
                if ((u % IX_STEP) == IX_STEP - 1 || u == nsteps * IX_STEP - 1) {
                    __syncthreads();
                    // collect the step's scores (ballot-free: warp scan + one atomic per warp)
                    const int s0 = key0 + (u / IX_STEP) * IX_STEP * IX_TILE;
                    const int key = s0 + tid;
                    const float v = sc[tid];
                    const bool pass = key < key1 && key < s0 + ((u % IX_STEP) + 1) * IX_TILE && pass_ge(v, Tf);
                    const uint32_t cnt = pass ? 1u : 0u;
                    const uint32_t incl = warp_incl_scan(cnt, lane);
                    const uint32_t wtot = __shfl_sync(FULL, incl, 31);
                    int base = 0;
                    if (lane == 31 && wtot) base = atomicAdd(cursor, (int)wtot);
                    base = __shfl_sync(FULL, base, 31);
                    if (pass) {
                        const uint32_t kv = f2key(v);
                        const int pos = base + (int)(incl - cnt);
                        if (pos < regcap) st_cand(reg + pos, kv, (uint32_t)key, keep);
                        kmax = max(kmax, kv);
                    }
                }
            },
            tid, warp, lane);
        if (it.last) {
            const uint32_t wk = __reduce_max_sync(FULL, kmax);
            if (lane == 0 && wk) atomicMax(seg_kmax, wk);
            __syncthreads();
            if (tid == 0) {
                const int end = *cursor;
                const long long v0 = (long long)cur_r * cl.tpr;
                const int b0 = cl_cta_of(cl, v0);
                cl.rec[(long long)cur_r * F_SEGS + (b - b0)] = make_int4(b, seg_start, end, (int)*seg_kmax);
                *seg_kmax = 0u;
                seg_start = end;
                const int ns = cl_cta_of(cl, v0 + p.ntiles - 1) - b0 + 1;
                __threadfence();
                if (atomicAdd(bq.segdone + cur_r, 1) == ns - 1) {
                    __threadfence();
                    st_release(bq.queue + atomicAdd(bq.qctl + Q_TAIL, 1), cur_r + 1);
                }
            }
            __syncthreads();
        } else {
            const uint32_t wk = __reduce_max_sync(FULL, kmax);
            if (lane == 0 && wk) atomicMax(seg_kmax, wk);
        }
    }
}

// ---------------------------------------------------------------------------------
// Fixup of the fused path: each listed row's scores are materialised into its scratch row
// (the same score_tile arithmetic), then the row path finishes it from there.  One CTA per
// SM with the row kernel's shared memory; the list is usually empty.
__global__ void __launch_bounds__(GVR_NT, 1)
indexer_fixup_kernel(IndexerArgs ia, float* scratch, const int32_t* __restrict__ row_lens, int k, int32_t* out,
                     float* out_val, gvr_row_stats* stats, GvrParams prm, const GuessOut* __restrict__ gp,
                     const int32_t* prev, int32_t* ctl, BatchQueue bq)
{
    fixup_wait(ctl);  // the refine grid's fixup list is complete
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t sbase = smem_u32(smem);
    // materialisation area (inside the row kernel's layout; idle between rows)
    float* W = reinterpret_cast<float*>(smem + 16384 + 4 * 16384);
    float* part = W + IX_H;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nfix = ld_relaxed(bq.qctl + Q_NFIX);
    uint32_t pbits = 0u;
    for (int li = (int)blockIdx.x; li < nfix; li += (int)gridDim.x) {
        const uint32_t e = (uint32_t)__ldcg(bq.fixlist + li);
        const int r = (int)(e & 0x7fffffffu);
        const int n = row_lens ? min(max(__ldg(row_lens + r), 0), (int)ia.n_max) : (int)ia.n_max;
        float* srow = scratch + (int64_t)r * ia.n_max;
        const __nv_bfloat16* kb = ia.keys + (int64_t)__ldg(ia.row_set + r) * ia.n_max * IX_D;
        __syncthreads();  // the previous row is done with the shared memory
        load_row_q(ia, r, sbase, W, tid);
        cp_async_wait<0>();
        __syncthreads();
        QFrag f;
        load_qfrag(f, sbase, warp, lane);
        score_tiles<4>(
            f, sbase + 16384, W, part, kb, (n + IX_TILE - 1) / IX_TILE,
            [&](int u, int i) {
                const int key = u * IX_TILE + i;
                return key < n ? key : -1;
            },
            [&](int u) {
                if (tid < IX_TILE && u * IX_TILE + tid < n) srow[u * IX_TILE + tid] = tile_score(part, tid);
            },
            tid, warp, lane);
        // the score row (generic stores) and the shared memory (cp.async) before the row
        // path's bulk copies read / refill them
        asm volatile("fence.proxy.async.global;" ::: "memory");
        fence_proxy_async_smem();
        __syncthreads();
        topk_row(scratch, ia.n_max, row_lens, k, out, out_val, stats, prm, gp, prev, nullptr, r,
                 li != (int)blockIdx.x, pbits, (e >> 31) != 0u);
    }
    fixup_done(ctl, bq, threadIdx.x);
}

}  // namespace gvr
