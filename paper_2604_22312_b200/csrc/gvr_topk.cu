// gvr_topk.cu — C ABI of libgvrtopk.so (declared in include/gvr_topk.h): argument
// validation, launch configuration and the host-buffer workspace entry point.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <type_traits>

#include "../../include/gvr_topk.h"
#include "gvr_kernel.cuh"
#include "refine_kernel.cuh"
#include "radix_kernel.cuh"
#include "radix2_kernel.cuh"
#include "indexer_kernel.cuh"

namespace {

using namespace gvr;

thread_local cudaError_t g_last_cuda_error = cudaSuccess;

constexpr int kVersion = 1 * 10000 + 0 * 100 + 0;

bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb)
{
    const char* pa = static_cast<const char*>(a);
    const char* pb = static_cast<const char*>(b);
    return pa < pb + nb && pb < pa + na;
}

gvr_status validate(const float* scores, int64_t row_stride, int32_t num_rows, int32_t k, const int32_t* out)
{
    if (num_rows < 0 || k < 1 || row_stride < 1) return GVR_ERR_INVALID_ARGUMENT;
    if (k > GVR_MAX_K) return GVR_ERR_UNSUPPORTED;
    if (row_stride > 0x7fffffffLL) return GVR_ERR_UNSUPPORTED;
    if (num_rows > 0 && (scores == nullptr || out == nullptr)) return GVR_ERR_INVALID_ARGUMENT;
    return GVR_OK;
}

// Stream-ordered scratch for the guess-kernel hand-off: a private memory pool per device
// that never trims (release threshold = max), so steady-state calls reuse the same pages
// instead of re-mapping them after every synchronisation, as the default pool would.
cudaMemPool_t scratch_pool()
{
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) return nullptr;
        unsigned long long thr = ~0ull;
        (void)cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        pools[dev] = p;
    }
    return pools[dev];
}

// Per-(device, stream) scratch of the batch path, grown stream-ordered from scratch_pool()
// and then reused: steady-state calls allocate nothing (CUDA-Graph friendly).  Calls on
// one stream are serialised by the stream, so one buffer per stream is race-free.
//  * Slots are keyed by cudaStreamGetId, which is unique per stream — also for the
//    per-thread default stream, whose handle value is the same on every host thread.
//  * The lease holds the cache's lock until the caller has enqueued its kernels (the
//    ScratchLease destructor), so no other host thread can grow the slot and free the
//    buffer between the lookup and the launches.
//  * A stream being captured never uses (or changes) the cache: the call takes a
//    graph-owned allocation / free pair recorded in the graph, zeroed by a memset node,
//    so every graph owns its scratch and a later eager call cannot free it under it.
//  * A failed call leaves the slot marked dirty; the next lease clears its zero region.
//
// Layout: a zero region at fixed offsets — ctl[4] | qctl[4] | queue[rows_cap] |
// segdone[rows_cap] | gen, pad | tcw[rows_cap] (8 B) — whose words are zero between calls
// (each kernel resets what it used; gen counts completed filter-path calls and tcw[r]
// carries the generation it was written for, so neither needs a reset), sized by the lease's row capacity so that calls with fewer rows leave the tail
// untouched; then the per-call arrays (zero_region_bytes(rows_cap) onwards).
struct ScratchSlot {
    void* ptr = nullptr;
    size_t size = 0;
    int64_t rows_cap = 0;
    bool dirty = false;  // a call failed after taking the lease: re-zero before reuse
};

struct ScratchLease {
    unsigned char* ptr = nullptr;
    int64_t rows_cap = 0;
    bool temporary = false;         // free after the launch (capture-time allocation)
    bool fresh = false;             // newly allocated or dirty: its zero region must be cleared
    ScratchSlot* slot = nullptr;    // the cached slot (nullptr for a temporary)
    std::unique_lock<std::mutex> lock;
    void fail()
    {
        if (slot) slot->dirty = true;
    }
};

size_t zero_region_bytes(int64_t rows_cap) { return (40 + 16 * (size_t)rows_cap + 255) & ~(size_t)255; }

std::mutex& scratch_mutex()
{
    static std::mutex mu;
    return mu;
}

// bytes_after(rows_cap): bytes needed past the zero region for this call
template <class F>
cudaError_t acquire_scratch(cudaStream_t stream, int64_t rows, F bytes_after, ScratchLease& lease)
{
    static std::map<std::pair<int, unsigned long long>, ScratchSlot> cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(stream, &cap)) != cudaSuccess) return e;
    if (cap != cudaStreamCaptureStatusNone) {
        const size_t need = zero_region_bytes(rows) + bytes_after(rows);
        lease.temporary = true;
        lease.fresh = true;
        lease.rows_cap = rows;
        return cudaMallocFromPoolAsync(reinterpret_cast<void**>(&lease.ptr), need, pool, stream);
    }
    unsigned long long sid = 0;
    if ((e = cudaStreamGetId(stream, &sid)) != cudaSuccess) return e;
    lease.lock = std::unique_lock<std::mutex>(scratch_mutex());
    ScratchSlot& slot = cache[std::make_pair(dev, sid)];
    lease.slot = &slot;
    if (slot.ptr && slot.rows_cap >= rows && slot.size >= zero_region_bytes(slot.rows_cap) + bytes_after(slot.rows_cap)) {
        lease.ptr = static_cast<unsigned char*>(slot.ptr);
        lease.rows_cap = slot.rows_cap;
        lease.fresh = slot.dirty;
        slot.dirty = false;
        return cudaSuccess;
    }
    const int64_t rc = rows > slot.rows_cap ? rows : slot.rows_cap;
    const size_t need = zero_region_bytes(rc) + bytes_after(rc);
    const size_t grow = need > 2 * slot.size ? need : 2 * slot.size;
    void* p = nullptr;
    if ((e = cudaMallocFromPoolAsync(&p, grow, pool, stream)) != cudaSuccess) return e;
    if (slot.ptr) (void)cudaFreeAsync(slot.ptr, stream);  // stream-ordered after earlier users
    slot.ptr = p;
    slot.size = grow;
    slot.rows_cap = rc;
    slot.dirty = false;
    lease.ptr = static_cast<unsigned char*>(p);
    lease.rows_cap = rc;
    lease.fresh = true;
    return cudaSuccess;
}

// Largest batch handled by the single-launch fused path: one wave of the streaming
// kernel (resident CTAs per SM x SMs), where the guess kernel's row ordering cannot help
// and its extra launch and hand-off only add latency.
// gvr_fixup_kernel's grid: two CTAs per SM (the list is usually empty and every CTA then
// exits at once; a batch of massive ties fills it).

int fused_max_rows()
{
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        (void)cudaGetLastError();
        return 0;
    }
    if (!cached[dev]) {
        int sms = 0, per_sm = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaFuncSetAttribute(gvr_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GVR_SMEM_BYTES) !=
                cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gvr_topk_kernel, GVR_NT, GVR_SMEM_BYTES) !=
                cudaSuccess) {
            (void)cudaGetLastError();
            return 0;
        }
        cached[dev] = sms * per_sm > 0 ? sms * per_sm : -1;
    }
    return cached[dev] > 0 ? cached[dev] : 0;
}

template <class Kern>
gvr_status set_smem(Kern kern, int bytes)
{
    // Opt in to > 48 KB dynamic shared memory; idempotent and cheap.
    // Every kernel also prefers the largest shared-memory carveout, so that CTAs of
    // consecutive kernels (programmatic dependent launch) can share an SM: the filter's
    // two CTAs leave room for a refine CTA only if the SM is not configured smaller.
    if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared) !=
            cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return GVR_OK;
}


// The refine kernel's four instances (phase stamps on/off x the two geometries).
gvr_status set_refine_smem()
{
    gvr_status st;
    if ((st = set_smem(gvr_refine_kernel<false, RefineFew>, RF_SMEM_BYTES)) != GVR_OK ||
        (st = set_smem(gvr_refine_kernel<true, RefineFew>, RF_SMEM_BYTES)) != GVR_OK ||
        (st = set_smem(gvr_refine_kernel<false, RefineMany>, RF_SMEM_BYTES)) != GVR_OK ||
        (st = set_smem(gvr_refine_kernel<true, RefineMany>, RF_SMEM_BYTES)) != GVR_OK)
        return st;
    return GVR_OK;
}

// Launch the refine kernel in the geometry the batch size picks (refine_kernel.cuh):
// go(kernel, grid, threads) performs the launch with the call's arguments.
template <class Go>
cudaError_t launch_refine(int64_t num_rows, int sms, bool timing, Go&& go)
{
    if (num_rows > RF_MANY_ROWS) {
        const int grid = (int)std::min<int64_t>(num_rows, (int64_t)RefineMany::CPS * sms);
        return timing ? go(gvr_refine_kernel<true, RefineMany>, grid, RefineMany::NT)
                      : go(gvr_refine_kernel<false, RefineMany>, grid, RefineMany::NT);
    }
    const int grid = (int)std::min<int64_t>(num_rows, (int64_t)RefineFew::CPS * sms);
    return timing ? go(gvr_refine_kernel<true, RefineFew>, grid, RefineFew::NT)
                  : go(gvr_refine_kernel<false, RefineFew>, grid, RefineFew::NT);
}

gvr_status launch_status()
{
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) g_last_cuda_error = e;
    return e == cudaSuccess ? GVR_OK : GVR_ERR_CUDA;
}

}  // namespace

extern "C" {

const char* gvr_status_string(gvr_status s)
{
    switch (s) {
    case GVR_OK: return "GVR_OK";
    case GVR_ERR_INVALID_ARGUMENT: return "GVR_ERR_INVALID_ARGUMENT";
    case GVR_ERR_UNSUPPORTED: return "GVR_ERR_UNSUPPORTED";
    case GVR_ERR_CUDA: return "GVR_ERR_CUDA";
    default: return "GVR_ERR_UNKNOWN";
    }
}

int32_t gvr_version(void) { return kVersion; }

gvr_status gvr_cta_timeline(int32_t kernel, int32_t enable, int64_t* host_out, int32_t max_ctas, int32_t* n_out)
{
    if (kernel != 0 && kernel != 1) return GVR_ERR_INVALID_ARGUMENT;
    const int on = enable ? 1 : 0;
    if (!enable) {
        if (!host_out || max_ctas < 0) return GVR_ERR_INVALID_ARGUMENT;
        const int n = min((int)max_ctas, FTS_MAX);
        if (cudaDeviceSynchronize() != cudaSuccess ||
            (kernel == 0 ? cudaMemcpyFromSymbol(host_out, g_fts, (size_t)n * 4 * sizeof(long long))
                         : cudaMemcpyFromSymbol(host_out, g_gts, (size_t)n * 4 * sizeof(long long))) != cudaSuccess) {
            g_last_cuda_error = cudaGetLastError();
            return GVR_ERR_CUDA;
        }
        if (n_out) *n_out = n;
    }
    if (cudaMemcpyToSymbol(g_fts_on, &on, sizeof(int)) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return GVR_OK;
}

gvr_status gvr_kernel_info(int32_t* gvr_ctas_per_sm, int32_t* gvr_threads, int32_t* gvr_smem_bytes,
                           int32_t* radix_ctas_per_sm, int32_t* radix_threads, int32_t* radix_smem_bytes)
{
    gvr_status st;
    if ((st = set_smem(gvr_topk_kernel, GVR_SMEM_BYTES)) != GVR_OK) return st;
    if ((st = set_smem(radix_topk_kernel, RADIX_SMEM_BYTES)) != GVR_OK) return st;
    int a = 0, b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, gvr_topk_kernel, GVR_NT, GVR_SMEM_BYTES) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, radix_topk_kernel, RADIX_NT, RADIX_SMEM_BYTES) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    if (gvr_ctas_per_sm) *gvr_ctas_per_sm = a;
    if (gvr_threads) *gvr_threads = GVR_NT;
    if (gvr_smem_bytes) *gvr_smem_bytes = GVR_SMEM_BYTES;
    if (radix_ctas_per_sm) *radix_ctas_per_sm = b;
    if (radix_threads) *radix_threads = RADIX_NT;
    if (radix_smem_bytes) *radix_smem_bytes = RADIX_SMEM_BYTES;
    return GVR_OK;
}

const char* gvr_last_cuda_error(void) { return cudaGetErrorString(g_last_cuda_error); }

// radix2: the same-geometry radix baseline (radix2_kernel.cuh) — the batch filter path
// with its Phase 1-2 guess kernel replaced by a histogram pass over the batch and a
// per-row threshold kernel; used for every batch size.
static gvr_status gvr_launch(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                             const int32_t* prev_topk, int32_t k, int32_t* out_idx, cudaStream_t stream,
                             const gvr_options* opt, float* out_val, gvr_row_stats* stats, long long* phase_ts,
                             cudaEvent_t const* ev = nullptr, bool radix2 = false)
{
    gvr_status st = validate(scores, row_stride, num_rows, k, out_idx);
    if (st != GVR_OK) return st;
    if (num_rows == 0) return GVR_OK;
    const size_t bytes = (size_t)num_rows * (size_t)k * sizeof(int32_t);
    if (prev_topk && prev_topk != out_idx && ranges_overlap(prev_topk, bytes, out_idx, bytes))
        return GVR_ERR_INVALID_ARGUMENT;
    GvrParams prm;
    prm.window_z = P2_Z_DEFAULT;  // DESIGN.md R35
    prm.max_secant = 8;
#ifndef GVR_DEFAULT_GUESS_STRIDE
#define GVR_DEFAULT_GUESS_STRIDE 8  // DESIGN.md R29
#endif
    prm.guess_stride = GVR_DEFAULT_GUESS_STRIDE;
    if (opt) {
        if (opt->guess_stride > 0) prm.guess_stride = opt->guess_stride;
        // 0 / NaN = default; a negative z aims below the K-th value (tests of R30)
        if (opt->window_z == opt->window_z && opt->window_z != 0.f) prm.window_z = opt->window_z;
        if (opt->max_secant_iters > 0) prm.max_secant = opt->max_secant_iters;
    }
    if ((st = set_smem(gvr_topk_kernel, GVR_SMEM_BYTES)) != GVR_OK) return st;
    auto mark = [&](int i) {
        if (ev && ev[i]) (void)cudaEventRecord(ev[i], stream);
    };
    // Cluster geometry: G CTAs per row when the batch is small and the
    // rows long — G = the largest power of two <= 8 with >= 16K elements per slice and
    // num_rows * G within one wave; gvr_options.force_cluster (1, 2, 4, 8) overrides.
    int G = 1;
    const int wave = radix2 ? 0 : fused_max_rows();
    if (radix2) {
        G = 1;
    } else if (opt && opt->force_cluster > 0) {
        G = opt->force_cluster;
        if (G != 1 && G != 2 && G != 4 && G != 8) return GVR_ERR_UNSUPPORTED;
    } else {
        while (G < 8 && row_stride / (2 * G) >= 16384 && (int64_t)num_rows * 2 * G <= wave) G *= 2;
    }
    if (G > 1) {
        if ((st = set_smem(gvr_topk_cluster_kernel, GVR_SMEM_BYTES)) != GVR_OK) return st;
        if ((int64_t)num_rows * G > 0x7fffffffLL) return GVR_ERR_UNSUPPORTED;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(num_rows * G));
        cfg.blockDim = dim3(GVR_NT);
        cfg.dynamicSmemBytes = GVR_SMEM_BYTES;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = (unsigned)G;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        mark(0);
        mark(1);
        const cudaError_t e = cudaLaunchKernelEx(&cfg, gvr_topk_cluster_kernel, scores, row_stride, row_lens, (int)k,
                                                 out_idx, out_val, stats, prm, prev_topk, phase_ts);
        mark(2);
        mark(3);
        if (e != cudaSuccess) {
            g_last_cuda_error = e;
            (void)cudaGetLastError();
            return GVR_ERR_CUDA;
        }
        return launch_status();
    }
    if (num_rows <= wave && !radix2) {
        // one wave: a single launch, Phase 1 inside each row's CTA (no hand-off, no
        // scratch); the gathers overlap the CTA's first tile loads
        mark(0);
        mark(1);
        gvr_topk_kernel<<<num_rows, GVR_NT, GVR_SMEM_BYTES, stream>>>(scores, row_stride, row_lens, k, out_idx, out_val,
                                                                      stats, prm, nullptr, nullptr, prev_topk, phase_ts,
                                                                      nullptr);
        mark(2);
        mark(3);
        return launch_status();
    }
    // Batch path (more than one wave).  Phase 1 for every row (gvr_guess_kernel, one small
    // CTA per row), then either
    //  * the filter path (default): gvr_filter_kernel streams the whole
    //    batch once (persistent, three CTAs per SM) into per-CTA candidate lists and queues
    //    each row when its list is complete; gvr_refine_kernel (four small CTAs per SM)
    //    selects every queued row from its list; the few rows it cannot finish are
    //    streamed and refined by gvr_topk_kernel in fixup mode; or
    //  * the row path (gvr_options.batch_path = 1): gvr_topk_kernel streams and refines one
    //    row per CTA, two CTAs per SM.
    // The kernels follow each other under programmatic dependent launch.  Scratch: the
    // stream's cached lease (acquire_scratch).
    CandLists cl{};
    BatchQueue bq{};
    bool filt = radix2 || !(opt && opt->batch_path == 1);
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess || sms < 1) {
        int dev = 0;
        (void)cudaGetLastError();
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                       cudaSuccess) {
            g_last_cuda_error = cudaGetLastError();
            return GVR_ERR_CUDA;
        }
    }
    // per-call arrays after the zero region: GuessOut[R] | order[R] | fixlist[R] |
    // rec[R][F_SEGS] | [radix2: hist[R][NBINS]] | region[G][reg]
    const size_t gp_bytes = (size_t)num_rows * sizeof(GuessOut);
    const size_t order_off = gp_bytes;
    const size_t fix_off = order_off + (size_t)num_rows * 4;
    const size_t rec_off = (fix_off + (size_t)num_rows * 4 + 255) & ~(size_t)255;
    size_t after_bytes = fix_off;
    size_t region_off = 0, hist_off = 0;
    if (filt) {
        const int tpr = (int)((row_stride + STAGE_FLOATS - 1) / STAGE_FLOATS);
        const long long V = (long long)num_rows * tpr;
        const int min_tiles = (tpr + 2) / 3;  // >= ceil(tpr / 3) tiles per CTA: <= F_SEGS CTAs per row
        long long G = (long long)F_CTAS_PER_SM * sms;  // persistent: every filter CTA resident
        if (G > V / min_tiles) G = V / min_tiles;
        const long long per = (V + G - 1) / (G > 0 ? G : 1);
        long long reg = per * STAGE_FLOATS / 8;  // room for 1/8 of the elements
        if (reg < F_REG_MIN) reg = F_REG_MIN;
        if (G < 1 || G * reg > 0x7fffffffLL) {
            if (radix2) return GVR_ERR_UNSUPPORTED;
            filt = false;
        } else {
            cl.V = V;
            cl.G = (int)G;
            cl.tpr = tpr;
            cl.reg = (int)reg;
            hist_off = (rec_off + (size_t)num_rows * F_SEGS * sizeof(int4) + 255) & ~(size_t)255;
            region_off = hist_off + (radix2 ? (size_t)num_rows * NBINS * sizeof(uint32_t) : 0);
            after_bytes = region_off + (size_t)G * (size_t)reg * sizeof(uint2);
        }
    }
    if (radix2 && (st = set_smem(radix_hist_kernel, RH_SMEM_BYTES)) != GVR_OK) return st;
    if (filt && ((st = set_smem(gvr_filter_kernel, F_SMEM_BYTES)) != GVR_OK ||
                 (st = set_refine_smem()) != GVR_OK ||
                 (st = set_smem(gvr_fixup_kernel, GVR_SMEM_BYTES)) != GVR_OK))
        return st;
    ScratchLease lease;
    if (acquire_scratch(stream, num_rows, [&](int64_t) { return after_bytes; }, lease) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    unsigned char* scratch = lease.ptr;
    unsigned char* per_call = scratch + zero_region_bytes(lease.rows_cap);
    int32_t* ctl = reinterpret_cast<int32_t*>(scratch);
    GuessOut* gp = reinterpret_cast<GuessOut*>(per_call);
    RowSched sched{reinterpret_cast<int32_t*>(per_call + order_off), ctl};
    if (filt) {
        bq.qctl = reinterpret_cast<int32_t*>(scratch + 16);
        bq.queue = bq.qctl + 4;
        bq.segdone = bq.queue + lease.rows_cap;
        bq.fixlist = reinterpret_cast<int32_t*>(per_call + fix_off);
        bq.gen = reinterpret_cast<uint32_t*>(bq.segdone + lease.rows_cap);
        bq.tcw = reinterpret_cast<unsigned long long*>(scratch + 40 + 8 * (size_t)lease.rows_cap);
        cl.rec = reinterpret_cast<int4*>(per_call + rec_off);
        cl.region = reinterpret_cast<uint2*>(per_call + region_off);
    }
    if (lease.fresh && cudaMemsetAsync(scratch, 0, zero_region_bytes(lease.rows_cap), stream) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        if (lease.temporary) (void)cudaFreeAsync(scratch, stream);
        lease.fail();
        return GVR_ERR_CUDA;
    }
    // programmatic dependent launch: each kernel is scheduled while its predecessor runs
    // (the refine CTAs become resident beside the filter CTAs); kernels that read their
    // predecessor's output wait for it (griddepcontrol.wait) or for a per-row flag.
    // Serialised when per-kernel events are recorded between them.
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    static const bool no_pdl = getenv("GVR_NO_PDL") != nullptr;  // experiments: serialise the kernels
    // fixup grid: one CTA per SM — the list is usually empty, and an empty fixup grid costs
    // its CTAs' scheduling and drain after the refine (2 per SM: cfg2 +1 us; a batch that
    // sends every row to the fixup takes ~2x longer at 1 per SM, still <= 2 passes per row)
    static const int fixup_per_sm = getenv("GVR_FIXUP_PER_SM") ? atoi(getenv("GVR_FIXUP_PER_SM")) : 1;  // experiments
    const int fixup_ctas = fixup_per_sm > 0 ? fixup_per_sm * sms : 16;
    pdl[0].val.programmaticStreamSerializationAllowed = (ev || no_pdl) ? 0 : 1;
    auto launch = [&](auto kern, int grid, int threads, int smem_bytes, auto... args) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = (size_t)smem_bytes;
        cfg.stream = stream;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, args...);
    };
    cudaError_t e = cudaSuccess;
    mark(0);
    if (radix2) {
        uint32_t* ghist = reinterpret_cast<uint32_t*>(per_call + hist_off);
        e = cudaMemsetAsync(ghist, 0, (size_t)num_rows * NBINS * sizeof(uint32_t), stream);
        if (e == cudaSuccess)
            e = launch(radix_hist_kernel, cl.G, RH_NT, RH_SMEM_BYTES, scores, row_stride, row_lens, (int)k, cl,
                       ghist);
        const uint32_t* ghc = ghist;
        if (e == cudaSuccess)
            e = launch(radix_thresh_kernel, (int)num_rows, 256, 0, scores, row_stride, row_lens, (int)k, ghc, gp, bq);
        if (e != cudaSuccess) {
            g_last_cuda_error = e;
            (void)cudaGetLastError();
            lease.fail();
            if (lease.temporary) (void)cudaFreeAsync(scratch, stream);
            return GVR_ERR_CUDA;
        }
    } else {
        gvr_guess_kernel<<<num_rows, GUESS_NT, 0, stream>>>(scores, row_stride, row_lens, prev_topk, k, num_rows, prm,
                                                            gp, sched, bq);
    }
    mark(1);
    const GuessOut* gpc = gp;
    const int32_t* orderc = sched.order;
    const int32_t* nop = nullptr;
    if (filt) {
        e = launch(gvr_filter_kernel, cl.G, F_NT, F_SMEM_BYTES, scores, row_stride, row_lens, (int)k, gpc, cl, bq);
        mark(2);
        if (e == cudaSuccess)
            e = launch_refine(num_rows, sms, phase_ts != nullptr, [&](auto kern, int grid, int threads) {
                return launch(kern, grid, threads, RF_SMEM_BYTES, scores, row_stride, row_lens, (int)k, (int)num_rows,
                              out_idx, out_val, stats, gpc, cl, bq, phase_ts, false, ctl);
            });
        if (e == cudaSuccess)
            e = launch(gvr_fixup_kernel, min((int)num_rows, fixup_ctas), GVR_NT, GVR_SMEM_BYTES, scores, row_stride, row_lens,
                       (int)k, out_idx, out_val, stats, prm, gpc, prev_topk, phase_ts, ctl, bq);
    } else {
        e = launch(gvr_topk_kernel, (int)num_rows, GVR_NT, GVR_SMEM_BYTES, scores, row_stride, row_lens, (int)k, out_idx,
                   out_val, stats, prm, gpc, orderc, nop, phase_ts, ctl);
        mark(2);
    }
    if (e != cudaSuccess) {
        g_last_cuda_error = e;
        (void)cudaGetLastError();
    }
    mark(3);
    const gvr_status ls = e != cudaSuccess ? GVR_ERR_CUDA : launch_status();
    if (ls != GVR_OK) lease.fail();  // kernels of this call may not have reset the zero region
    if (lease.temporary && cudaFreeAsync(scratch, stream) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return ls;
}

gvr_status gvr_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                               const int32_t* prev_topk, int32_t k, int32_t* out_idx, cudaStream_t stream,
                               const gvr_options* opt, float* out_val, gvr_row_stats* stats)
{
    return gvr_launch(scores, row_stride, row_lens, num_rows, prev_topk, k, out_idx, stream, opt, out_val, stats,
                      nullptr);
}

gvr_status gvr_topk_batched_events(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                   int32_t num_rows, const int32_t* prev_topk, int32_t k, int32_t* out_idx,
                                   cudaStream_t stream, cudaEvent_t guess_start, cudaEvent_t stream_start,
                                   cudaEvent_t stream_end, cudaEvent_t call_end, const gvr_options* opt)
{
    const cudaEvent_t ev[4] = {guess_start, stream_start, stream_end, call_end};
    return gvr_launch(scores, row_stride, row_lens, num_rows, prev_topk, k, out_idx, stream, opt, nullptr, nullptr,
                      nullptr, ev);
}

gvr_status gvr_topk_phase_timing(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                                 const int32_t* prev_topk, int32_t k, int32_t* out_idx, cudaStream_t stream,
                                 long long* phase_ts)
{
    if (!phase_ts && num_rows > 0) return GVR_ERR_INVALID_ARGUMENT;
    return gvr_launch(scores, row_stride, row_lens, num_rows, prev_topk, k, out_idx, stream, nullptr, nullptr,
                      nullptr, phase_ts);
}

gvr_status gvr_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                            const int32_t* prev_topk, int32_t k, int32_t* out_idx, cudaStream_t stream)
{
    return gvr_topk_batched_ex(scores, row_stride, row_lens, num_rows, prev_topk, k, out_idx, stream, nullptr,
                               nullptr, nullptr);
}

gvr_status radix_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                 int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream,
                                 float* out_val, gvr_row_stats* stats)
{
    gvr_status st = validate(scores, row_stride, num_rows, k, out_idx);
    if (st != GVR_OK) return st;
    if (num_rows == 0) return GVR_OK;
    if ((st = set_smem(radix_topk_kernel, RADIX_SMEM_BYTES)) != GVR_OK) return st;
    radix_topk_kernel<<<num_rows, RADIX_NT, RADIX_SMEM_BYTES, stream>>>(scores, row_stride, row_lens, k, out_idx, out_val,
                                                            stats);
    return launch_status();
}

gvr_status gvr_indexer_scores(const void* keys, int64_t n_max, const int32_t* row_set, const int32_t* row_lens,
                              const void* q, const float* w, int32_t num_rows, float* out, int64_t out_stride,
                              cudaStream_t stream)
{
    if (num_rows < 0 || n_max < 1 || out_stride < n_max) return GVR_ERR_INVALID_ARGUMENT;
    if (num_rows == 0) return GVR_OK;
    if (!keys || !row_set || !q || !w || !out) return GVR_ERR_INVALID_ARGUMENT;
    if (n_max > 0x7fffffffLL) return GVR_ERR_UNSUPPORTED;
    gvr_status st;
    if ((st = set_smem(indexer_scores_kernel, IX_SMEM_BYTES)) != GVR_OK) return st;
    const IndexerArgs ia{static_cast<const __nv_bfloat16*>(keys), n_max, row_set, static_cast<const __nv_bfloat16*>(q), w};
    const int tiles = (int)((n_max + IX_TILE - 1) / IX_TILE);
    const dim3 grid((unsigned)min(tiles, 64), (unsigned)num_rows);
    indexer_scores_kernel<<<grid, IX_NT, IX_SMEM_BYTES, stream>>>(ia, row_lens, out, out_stride);
    return launch_status();
}

gvr_status gvr_indexer_topk_batched(const void* keys, int64_t n_max, const int32_t* row_set, const int32_t* row_lens,
                                    const void* q, const float* w, int32_t num_rows, const int32_t* prev_topk, int32_t k,
                                    int32_t* out_idx, float* score_scratch, cudaStream_t stream)
{
    gvr_status st = validate(score_scratch, n_max, num_rows, k, out_idx);
    if (st != GVR_OK) return st;
    if (num_rows == 0) return GVR_OK;
    if (!keys || !row_set || !q || !w) return GVR_ERR_INVALID_ARGUMENT;
    if (n_max % 4 != 0 || (reinterpret_cast<uintptr_t>(score_scratch) & 15u) != 0) return GVR_ERR_UNSUPPORTED;
    const size_t bytes = (size_t)num_rows * (size_t)k * sizeof(int32_t);
    if (prev_topk && prev_topk != out_idx && ranges_overlap(prev_topk, bytes, out_idx, bytes))
        return GVR_ERR_INVALID_ARGUMENT;
    GvrParams prm;
    prm.window_z = P2_Z_DEFAULT;
    prm.max_secant = 8;
    prm.guess_stride = GVR_DEFAULT_GUESS_STRIDE;
    int sms = 0, dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                   cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    if ((st = set_smem(indexer_guess_kernel, IXG_SMEM_BYTES)) != GVR_OK ||
        (st = set_smem(indexer_filter_kernel, IXF_SMEM_BYTES)) != GVR_OK ||
        (st = set_refine_smem()) != GVR_OK ||
        (st = set_smem(indexer_fixup_kernel, GVR_SMEM_BYTES)) != GVR_OK)
        return st;
    // the candidate lists of the batch filter path, one filter CTA per SM
    CandLists cl{};
    const int tpr = (int)((n_max + STAGE_FLOATS - 1) / STAGE_FLOATS);
    const long long V = (long long)num_rows * tpr;
    const int min_tiles = (tpr + 2) / 3;
    long long G = sms;
    if (G > V / min_tiles) G = V / min_tiles;
    if (G < 1) G = 1;
    const long long per = (V + G - 1) / G;
    long long reg = per * STAGE_FLOATS / 8;
    if (reg < F_REG_MIN) reg = F_REG_MIN;
    if (G * reg > 0x7fffffffLL) return GVR_ERR_UNSUPPORTED;
    cl.V = V;
    cl.G = (int)G;
    cl.tpr = tpr;
    cl.reg = (int)reg;
    const size_t gp_bytes = (size_t)num_rows * sizeof(GuessOut);
    const size_t fix_off = gp_bytes + (size_t)num_rows * 4;
    const size_t rec_off = (fix_off + (size_t)num_rows * 4 + 255) & ~(size_t)255;
    const size_t region_off = (rec_off + (size_t)num_rows * F_SEGS * sizeof(int4) + 255) & ~(size_t)255;
    const size_t after_bytes = region_off + (size_t)G * (size_t)reg * sizeof(uint2);
    ScratchLease lease;
    if (acquire_scratch(stream, num_rows, [&](int64_t) { return after_bytes; }, lease) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    unsigned char* scratch = lease.ptr;
    unsigned char* per_call = scratch + zero_region_bytes(lease.rows_cap);
    int32_t* ctl = reinterpret_cast<int32_t*>(scratch);
    GuessOut* gp = reinterpret_cast<GuessOut*>(per_call);
    BatchQueue bq{};
    bq.qctl = reinterpret_cast<int32_t*>(scratch + 16);
    bq.queue = bq.qctl + 4;
    bq.segdone = bq.queue + lease.rows_cap;
    bq.fixlist = reinterpret_cast<int32_t*>(per_call + fix_off);
    cl.rec = reinterpret_cast<int4*>(per_call + rec_off);
    cl.region = reinterpret_cast<uint2*>(per_call + region_off);
    cudaError_t e = cudaSuccess;
    if (lease.fresh) e = cudaMemsetAsync(scratch, 0, zero_region_bytes(lease.rows_cap), stream);
    const IndexerArgs ia{static_cast<const __nv_bfloat16*>(keys), n_max, row_set, static_cast<const __nv_bfloat16*>(q), w};
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    auto launch = [&](auto kern, int grid, int threads, int smem_bytes, auto... args) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3((unsigned)threads);
        cfg.dynamicSmemBytes = (size_t)smem_bytes;
        cfg.stream = stream;
        cfg.attrs = pdl;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, args...);
    };
    const float* sc = score_scratch;
    const GuessOut* gpc = gp;
    if (e == cudaSuccess)
        e = launch(indexer_guess_kernel, (int)num_rows, IX_NT, IXG_SMEM_BYTES, ia, sc, row_lens, prev_topk, (int)k, prm,
                   gp, bq);
    if (e == cudaSuccess)
        e = launch(indexer_filter_kernel, cl.G, IX_NT, IXF_SMEM_BYTES, ia, sc, row_lens, (int)k, gpc, cl, bq);
    if (e == cudaSuccess)
        e = launch_refine(num_rows, sms, false, [&](auto kern, int grid, int threads) {
            return launch(kern, grid, threads, RF_SMEM_BYTES, sc, n_max, row_lens, (int)k, (int)num_rows, out_idx,
                          (float*)nullptr, (gvr_row_stats*)nullptr, gpc, cl, bq, (long long*)nullptr, true, ctl);
        });
    if (e == cudaSuccess)
        e = launch(indexer_fixup_kernel, min((int)num_rows, sms), GVR_NT, GVR_SMEM_BYTES, ia, score_scratch, row_lens,
                   (int)k, out_idx, (float*)nullptr, (gvr_row_stats*)nullptr, prm, gpc, prev_topk, ctl, bq);
    if (e != cudaSuccess) {
        g_last_cuda_error = e;
        (void)cudaGetLastError();
        lease.fail();
    }
    const gvr_status ls = e != cudaSuccess ? GVR_ERR_CUDA : launch_status();
    if (lease.temporary && cudaFreeAsync(scratch, stream) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return ls;
}

gvr_status radix2_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                  int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream,
                                  float* out_val, gvr_row_stats* stats)
{
    return gvr_launch(scores, row_stride, row_lens, num_rows, nullptr, k, out_idx, stream, nullptr, out_val, stats,
                      nullptr, nullptr, true);
}

gvr_status radix2_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                               int32_t k, int32_t* out_idx, cudaStream_t stream)
{
    return radix2_topk_batched_ex(scores, row_stride, row_lens, num_rows, k, out_idx, stream, nullptr, nullptr);
}

gvr_status radix_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                              int32_t k, int32_t* out_idx, cudaStream_t stream)
{
    return radix_topk_batched_ex(scores, row_stride, row_lens, num_rows, k, out_idx, stream, nullptr, nullptr);
}

// ------------------------------------------------------------------ host-buffer path
struct gvr_workspace {
    int32_t max_rows;
    int64_t row_stride;
    int32_t k;
    float* d_scores;
    int32_t* d_lens;
    int32_t* d_prev;
    int32_t* d_out;
};

gvr_status gvr_workspace_create(int32_t max_rows, int64_t row_stride, int32_t k, gvr_workspace** ws)
{
    if (!ws || max_rows < 1 || row_stride < 1 || k < 1) return GVR_ERR_INVALID_ARGUMENT;
    if (k > GVR_MAX_K || row_stride > 0x7fffffffLL) return GVR_ERR_UNSUPPORTED;
    *ws = nullptr;
    gvr_workspace* w = new (std::nothrow) gvr_workspace();
    if (!w) return GVR_ERR_CUDA;
    w->max_rows = max_rows;
    w->row_stride = row_stride;
    w->k = k;
    const size_t ns = (size_t)max_rows * (size_t)row_stride * sizeof(float);
    const size_t no = (size_t)max_rows * (size_t)k * sizeof(int32_t);
    bool ok = cudaMalloc(&w->d_scores, ns) == cudaSuccess;
    ok = ok && cudaMalloc(&w->d_lens, (size_t)max_rows * sizeof(int32_t)) == cudaSuccess;
    ok = ok && cudaMalloc(&w->d_prev, no) == cudaSuccess;
    ok = ok && cudaMalloc(&w->d_out, no) == cudaSuccess;
    if (!ok) {
        (void)cudaGetLastError();
        gvr_workspace_destroy(w);
        return GVR_ERR_CUDA;
    }
    *ws = w;
    return GVR_OK;
}

gvr_status gvr_workspace_destroy(gvr_workspace* ws)
{
    if (!ws) return GVR_OK;
    cudaFree(ws->d_scores);
    cudaFree(ws->d_lens);
    cudaFree(ws->d_prev);
    cudaFree(ws->d_out);
    delete ws;
    return GVR_OK;
}

gvr_status gvr_topk_batched_host(const float* h_scores, int64_t row_stride, const int32_t* h_row_lens,
                                 int32_t num_rows, const int32_t* h_prev, int32_t k, int32_t* h_out,
                                 gvr_workspace* ws, cudaStream_t stream)
{
    if (!ws) return GVR_ERR_INVALID_ARGUMENT;
    gvr_status st = validate(h_scores, row_stride, num_rows, k, h_out);
    if (st != GVR_OK) return st;
    if (num_rows > ws->max_rows || row_stride != ws->row_stride || k != ws->k) return GVR_ERR_INVALID_ARGUMENT;
    if (num_rows == 0) return GVR_OK;
    const size_t ns = (size_t)num_rows * (size_t)row_stride * sizeof(float);
    const size_t no = (size_t)num_rows * (size_t)k * sizeof(int32_t);
    bool ok = cudaMemcpyAsync(ws->d_scores, h_scores, ns, cudaMemcpyHostToDevice, stream) == cudaSuccess;
    if (ok && h_row_lens)
        ok = cudaMemcpyAsync(ws->d_lens, h_row_lens, (size_t)num_rows * sizeof(int32_t), cudaMemcpyHostToDevice,
                             stream) == cudaSuccess;
    if (ok && h_prev) ok = cudaMemcpyAsync(ws->d_prev, h_prev, no, cudaMemcpyHostToDevice, stream) == cudaSuccess;
    if (!ok) {
        (void)cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    st = gvr_topk_batched(ws->d_scores, row_stride, h_row_lens ? ws->d_lens : nullptr, num_rows,
                          h_prev ? ws->d_prev : nullptr, k, ws->d_out, stream);
    if (st != GVR_OK) return st;
    if (cudaMemcpyAsync(h_out, ws->d_out, no, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess) {
        (void)cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return GVR_OK;
}

}  // extern "C"
