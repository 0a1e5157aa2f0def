// gvr_topk.cu — C ABI of libgvrtopk.so (declared in include/gvr_topk.h): argument
// validation, launch configuration and the host-buffer workspace entry point.
#include <map>
#include <mutex>
#include <utility>
#include <type_traits>

#include "../../include/gvr_topk.h"
#include "gvr_kernel.cuh"
#include "radix_kernel.cuh"

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

// Per-(device, stream) scratch for the guess-kernel hand-off, grown stream-ordered
// from scratch_pool() and then reused: steady-state calls allocate nothing (CUDA-Graph
// friendly).  Calls on one stream are serialised by the stream, so one buffer per
// stream is race-free.  While the stream is being captured the cache is not modified:
// a too-small cache is bypassed with an allocation / free pair recorded in the graph.
struct ScratchLease {
    unsigned char* ptr = nullptr;
    bool temporary = false;  // free after the launch (capture-time allocation)
    bool fresh = false;      // newly allocated: its control words must be zeroed
};

cudaError_t acquire_scratch(cudaStream_t stream, size_t bytes, ScratchLease& lease)
{
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = scratch_pool();
    if (!pool) return cudaErrorMemoryAllocation;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if ((e = cudaStreamIsCapturing(stream, &cap)) != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = cache[std::make_pair(dev, stream)];
    if (slot.second >= bytes) {
        lease.ptr = static_cast<unsigned char*>(slot.first);
        return cudaSuccess;
    }
    if (cap != cudaStreamCaptureStatusNone) {
        lease.temporary = true;
        lease.fresh = true;
        return cudaMallocFromPoolAsync(reinterpret_cast<void**>(&lease.ptr), bytes, pool, stream);
    }
    const size_t grow = bytes > 2 * slot.second ? bytes : 2 * slot.second;
    void* p = nullptr;
    if ((e = cudaMallocFromPoolAsync(&p, grow, pool, stream)) != cudaSuccess) return e;
    if (slot.first) (void)cudaFreeAsync(slot.first, stream);  // stream-ordered after earlier users
    slot = std::make_pair(p, grow);
    lease.ptr = static_cast<unsigned char*>(p);
    lease.fresh = true;
    return cudaSuccess;
}

// Largest batch handled by the single-launch fused path: one wave of the streaming
// kernel (resident CTAs per SM x SMs), where the guess kernel's row ordering cannot help
// and its extra launch and hand-off only add latency.
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
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    return GVR_OK;
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

static gvr_status gvr_launch(const float* scores, int64_t row_stride, const int32_t* row_lens, int32_t num_rows,
                             const int32_t* prev_topk, int32_t k, int32_t* out_idx, cudaStream_t stream,
                             const gvr_options* opt, float* out_val, gvr_row_stats* stats, long long* phase_ts,
                             cudaEvent_t const* ev = nullptr)
{
    gvr_status st = validate(scores, row_stride, num_rows, k, out_idx);
    if (st != GVR_OK) return st;
    if (num_rows == 0) return GVR_OK;
    const size_t bytes = (size_t)num_rows * (size_t)k * sizeof(int32_t);
    if (prev_topk && prev_topk != out_idx && ranges_overlap(prev_topk, bytes, out_idx, bytes))
        return GVR_ERR_INVALID_ARGUMENT;
    GvrParams prm;
    prm.collect_sigma = 0.3f;  // DESIGN.md R22: measured sweep (cfg2, cfg4)
    prm.max_secant = 8;
#ifndef GVR_DEFAULT_GUESS_STRIDE
#define GVR_DEFAULT_GUESS_STRIDE 4  // DESIGN.md R29
#endif
    prm.guess_stride = GVR_DEFAULT_GUESS_STRIDE;
    if (opt) {
        if (opt->guess_stride > 0) prm.guess_stride = opt->guess_stride;
        if (opt->collect_sigma == opt->collect_sigma) prm.collect_sigma = opt->collect_sigma;
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
    const int wave = fused_max_rows();
    if (opt && opt->force_cluster > 0) {
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
        if (e != cudaSuccess) {
            g_last_cuda_error = e;
            (void)cudaGetLastError();
            return GVR_ERR_CUDA;
        }
        return launch_status();
    }
    if (num_rows <= wave) {
        // one wave: a single launch, Phase 1 inside each row's CTA (no hand-off, no
        // scratch); the gathers overlap the CTA's first tile loads
        mark(0);
        mark(1);
        gvr_topk_kernel<<<num_rows, GVR_NT, GVR_SMEM_BYTES, stream>>>(scores, row_stride, row_lens, k, out_idx, out_val,
                                                                      stats, prm, nullptr, nullptr, prev_topk, phase_ts,
                                                                      nullptr);
        mark(2);
        return launch_status();
    }
    // Phase 1 for every row (one small CTA per row), then the streaming / refine kernel
    // (one CTA per row, two CTAs per SM).  The per-row hand-off lives in the stream's
    // cached scratch (acquire_scratch), so concurrent calls on different streams do not
    // share it and steady-state calls allocate nothing.
    // scratch: ctl[4] | GuessOut[num_rows] | order[num_rows].  ctl = {front cursor, back
    // cursor, finished CTAs, 0} lives at a fixed offset and is zero between calls: the
    // streaming kernel's last CTA resets it, so only a new buffer needs a memset.
    const size_t gp_bytes = (size_t)num_rows * sizeof(GuessOut);
    const size_t scratch_bytes = 16 + gp_bytes + (size_t)num_rows * 4;
    ScratchLease lease;
    if (acquire_scratch(stream, scratch_bytes, lease) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        return GVR_ERR_CUDA;
    }
    unsigned char* scratch = lease.ptr;
    int32_t* ctl = reinterpret_cast<int32_t*>(scratch);
    GuessOut* gp = reinterpret_cast<GuessOut*>(scratch + 16);
    RowSched sched{reinterpret_cast<int32_t*>(scratch + 16 + gp_bytes), ctl};
    if (lease.fresh && cudaMemsetAsync(ctl, 0, 16, stream) != cudaSuccess) {
        g_last_cuda_error = cudaGetLastError();
        if (lease.temporary) (void)cudaFreeAsync(scratch, stream);
        return GVR_ERR_CUDA;
    }
    mark(0);
    gvr_guess_kernel<<<num_rows, GUESS_NT, 0, stream>>>(scores, row_stride, row_lens, prev_topk, k, num_rows, prm, gp,
                                                        sched);
    mark(1);
    {
        // programmatic dependent launch: scheduled while the guess kernel runs, the
        // streaming kernel waits for it (griddepcontrol.wait) before reading the hand-off;
        // serialised when per-kernel events are recorded between the two
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)num_rows);
        cfg.blockDim = dim3(GVR_NT);
        cfg.dynamicSmemBytes = GVR_SMEM_BYTES;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = ev ? 0 : 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, gvr_topk_kernel, scores, row_stride, row_lens, (int)k, out_idx,
                                                 out_val, stats, prm, static_cast<const GuessOut*>(gp),
                                                 static_cast<const int32_t*>(sched.order),
                                                 static_cast<const int32_t*>(nullptr), phase_ts, ctl);
        if (e != cudaSuccess) {
            g_last_cuda_error = e;
            (void)cudaGetLastError();
        }
    }
    mark(2);
    const gvr_status ls = launch_status();
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
                                   cudaEvent_t stream_end)
{
    const cudaEvent_t ev[3] = {guess_start, stream_start, stream_end};
    return gvr_launch(scores, row_stride, row_lens, num_rows, prev_topk, k, out_idx, stream, nullptr, nullptr, nullptr,
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
