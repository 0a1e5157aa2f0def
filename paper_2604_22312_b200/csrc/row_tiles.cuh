// row_tiles.cuh — coalesced register streaming of one fp32 score row in index order
// (used by the radix baseline and the distribution-agnostic fallbacks; the GVR hot
// loop streams through the TMA ring of pipeline.cuh instead).
//
// A row x[0, n) is split into an unaligned scalar head (elements before the first
// 16-byte boundary, < 4), a body of float4 vectors and a scalar tail (< 4).  The body
// is consumed in tiles of N*VEC float4 (N threads x VEC float4): float4 j of thread t
// is vector t + j*N, so every warp load is 512 contiguous bytes (128-bit vectorised,
// coalesced).  The next tile is loaded into registers while the current one is
// processed (register double buffer).
#pragma once
#include "device_common.cuh"

namespace gvr {

struct RowGeom {
    const float* x;
    int n;
    int head;      // scalar elements [0, head)
    int nvec;      // float4 vectors starting at element `head`
    int body_end;  // head + 4*nvec
    int tail;      // scalar elements [body_end, n)
};

__device__ __forceinline__ RowGeom make_geom(const float* x, int n)
{
    RowGeom g;
    g.x = x;
    g.n = n;
    const uintptr_t a = reinterpret_cast<uintptr_t>(x);
    int head = (int)(((16u - (uint32_t)(a & 15u)) & 15u) >> 2);
    if (head > n) head = n;
    g.head = head;
    g.nvec = (n - head) >> 2;
    g.body_end = head + 4 * g.nvec;
    g.tail = n - g.body_end;
    return g;
}

// One body tile held in registers: 4*VEC keys per thread.
template <int N>
struct MainTile {
    static constexpr int E = 4 * VEC;
    uint32_t key[E];
    int vbase;  // first vector index of this thread's slot j=0
    int nvec;
    int head;
    __device__ __forceinline__ bool valid(int e) const { return vbase + (e >> 2) * N < nvec; }
    __device__ __forceinline__ int idx(int e) const { return head + 4 * (vbase + (e >> 2) * N) + (e & 3); }
};

// One scalar element per thread (head or tail).
struct ScalarTile {
    static constexpr int E = 1;
    uint32_t key[1];
    int i;  // element index, or -1
    __device__ __forceinline__ bool valid(int) const { return i >= 0; }
    __device__ __forceinline__ int idx(int) const { return i; }
};

template <int N>
__device__ __forceinline__ void load_tile(const RowGeom& g, int t, int tid, float4 (&v)[VEC])
{
    const float4* xv = reinterpret_cast<const float4*>(g.x + g.head);
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
        const int vi = t * N * VEC + j * N + tid;
        v[j] = vi < g.nvec ? ldg_stream(xv + vi) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

template <int N>
__device__ __forceinline__ void to_tile(const RowGeom& g, int t, int tid, const float4 (&v)[VEC], MainTile<N>& mt)
{
    mt.vbase = t * N * VEC + tid;
    mt.nvec = g.nvec;
    mt.head = g.head;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
        mt.key[4 * j + 0] = f2key(v[j].x);
        mt.key[4 * j + 1] = f2key(v[j].y);
        mt.key[4 * j + 2] = f2key(v[j].z);
        mt.key[4 * j + 3] = f2key(v[j].w);
    }
}

// Visit every element of the row in index order, one tile at a time:
//   f(tile, elements_streamed_after_this_tile) -> int (non-zero aborts).
// All threads of the group call f for every tile (group-uniform control flow).
template <int N, class F>
__device__ __forceinline__ int for_each_tile(const RowGeom& g, int tid, F&& f)
{
    if (g.head > 0) {
        ScalarTile s;
        s.i = tid < g.head ? tid : -1;
        s.key[0] = s.i >= 0 ? f2key(__ldg(g.x + s.i)) : 0u;
        const int rc = f(s, g.head);
        if (rc) return rc;
    }
    const int ntiles = (g.nvec + N * VEC - 1) / (N * VEC);
    if (ntiles > 0) {
        float4 cur[VEC], nxt[VEC];
        load_tile<N>(g, 0, tid, cur);
        for (int t = 0; t < ntiles; ++t) {
            if (t + 1 < ntiles) load_tile<N>(g, t + 1, tid, nxt);
            MainTile<N> mt;
            to_tile<N>(g, t, tid, cur, mt);
            const int vend = min(g.nvec, (t + 1) * N * VEC);
            const int rc = f(mt, g.head + 4 * vend);
            if (rc) return rc;
#pragma unroll
            for (int j = 0; j < VEC; ++j) cur[j] = nxt[j];
        }
    }
    if (g.tail > 0) {
        ScalarTile s;
        s.i = tid < g.tail ? g.body_end + tid : -1;
        s.key[0] = s.i >= 0 ? f2key(__ldg(g.x + s.i)) : 0u;
        const int rc = f(s, g.n);
        if (rc) return rc;
    }
    return 0;
}

}  // namespace gvr
