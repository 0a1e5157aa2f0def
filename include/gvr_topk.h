/*
 * gvr_topk.h — C ABI of the B200-native GVR exact Top-K library (libgvrtopk.so).
 *
 * Operation (PAPER.md = arXiv 2604.22312 source):
 *   For each row r of a batch of fp32 score rows x (one DSA indexer score vector
 *   I_t per decode query, Eq. 1, lines 78-85), return the indices of its
 *   k largest values (exact Top-K, Sec. 4.1), ORDERED by score
 *   descending and, among equal scores, by index ascending (BASELINE.json
 *   north_star; the paper itself leaves ties non-deterministic).
 *   Scores are compared through the sortable FP32 key: +0 ranks
 *   above -0, +/-Inf are ordinary values, NaNs sort beyond +/-Inf by bit pattern.
 *   gvr_topk_* use the previous decode step's Top-K as a guess (Guess-Verify-Refine,
 *   PAPER.md Sec. 4.2, Phases 1-4); radix_topk_* is the distribution-agnostic
 *   radix-select baseline of PAPER.md Sec. 2.2 (lines 125-148).  Both produce the
 *   same bytes for the same input; the guess never changes the result.
 *
 * Conventions shared by every entry point:
 *   - Device pointers are caller-owned CUDA device pointers; the library keeps no
 *     reference to them after return.  Its only memory is a scratch lease per (device,
 *     stream) — Phase-1 hand-off, ready queue and, on the batch filter path, candidate
 *     lists (8 B per entry, room for 1/8 of the batch's elements; ~60 MB for 488 rows
 *     of 100K) — grown stream-ordered from a private pool on first use and reused, so
 *     steady-state calls allocate nothing (CUDA-Graph capturable; the stable-address
 *     requirement of PAPER.md:1476-1482).
 *   - Calls are stream-ordered on `stream` (0 = legacy default stream) and do not
 *     synchronise the host, except gvr_topk_batched_host (documented below).
 *   - Layout: scores is row-major [num_rows, row_stride] fp32; row r occupies
 *     scores[r*row_stride .. r*row_stride + row_lens[r]).  Rows need not be 16-byte
 *     aligned (row_stride may be any value >= 1).
 *   - Output: out_idx is row-major [num_rows, k] int32.  For j < min(k, len):
 *     out_idx[r*k+j] = j-th index of the row in (score desc, index asc) order; for
 *     j >= len it is -1 (rows shorter than k are padded).
 *   - Errors are reported synchronously before any launch:
 *       GVR_ERR_INVALID_ARGUMENT: num_rows < 0, k < 1, row_stride < 1, a required
 *         pointer is NULL while num_rows > 0, or prev_topk partially overlaps out_idx;
 *       GVR_ERR_UNSUPPORTED: k > GVR_MAX_K, row_stride > INT32_MAX;
 *       GVR_ERR_CUDA: the launch failed (cudaGetLastError() is consumed).
 *     num_rows == 0 is a successful no-op.
 *   - Device-side precondition 0 <= row_lens[r] <= row_stride; out-of-range lengths
 *     are clamped into that range.
 */
#ifndef GVR_TOPK_H
#define GVR_TOPK_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVR_MAX_K 2048           /* K of DSA decode; k is 1..2048 */
#define GVR_WINDOW_C 6144        /* MAX_CANDIDATES C of Lemma 1  */

typedef enum {
    GVR_OK = 0,
    GVR_ERR_INVALID_ARGUMENT = 1,
    GVR_ERR_UNSUPPORTED = 2,
    GVR_ERR_CUDA = 3
} gvr_status;

/* How a row finished (gvr_row_stats.done_kind). */
typedef enum {
    GVR_DONE_TRIVIAL = 0,    /* len <= k: every element emitted, then -1 padding      */
    GVR_DONE_CONVERGED = 1,  /* Phases 1-4 found K <= f(T) <= capacity */
    GVR_DONE_TIEFILL = 2,    /* massive ties at the K-th value: ordered tie fill        */
                             /* (PAPER.md:417-420 caveat; R13)               */
    GVR_DONE_RADIX = 3       /* radix-select entry point (baseline)                     */
} gvr_done_kind;

/* How Phase 2 ended (gvr_row_stats.phase2_exit; R34-R36). */
typedef enum {
    GVR_P2_ALL = 0,        /* len <= 6016: every element is collected, no search        */
    GVR_P2_WINDOW = 1,     /* a probe's sample count fell in the window [L, H]          */
    GVR_P2_TIES = 2,       /* the anchors became adjacent keys (ties): lo anchor taken  */
    GVR_P2_EXHAUSTED = 3   /* 12 probes without a window hit: lo anchor taken           */
} gvr_phase2_exit;

/* Per-row statistics (optional output of the _ex entry point). Reported, not part of
 * the result contract. */
typedef struct {
    int32_t secant_iters;   /* I: threshold probes f(T) of Phase 2,  */
                            /* counted over the row sample (R34)             */
    int32_t snap_iters;     /* S: Phase-4 snap iterations          */
    int32_t cand_count;     /* candidates collected in Phase 3 (|{x >= T}|)           */
    int32_t done_kind;      /* gvr_done_kind                                          */
    int32_t global_passes;  /* full-row reads of the row from global memory           */
    int32_t raises;         /* row kernel: mid-stream collect-threshold raises; filter */
                            /* path refine: Phase-4 histogram narrowings  */
    int32_t buffer_count;   /* f(T_c): size of the streamed candidate buffer          */
    int32_t cluster;        /* CTAs cooperating on the row                            */
    int32_t phase2_exit;    /* gvr_phase2_exit                                        */
    int32_t sample_count;   /* sample hits at T_c (of 4096; R34)            */
    uint32_t tc_key;        /* T_c as a sortable key               */
    int32_t reserved;
} gvr_row_stats;

/* Tuning knobs; NULL selects the defaults.  None of them changes the result. */
typedef struct {
    float window_z;           /* Phase-2 window lower edge mu + z sqrt(mu) sample hits     */
                              /* (R35); 0 or NaN = default 4.5; a negative z    */
                              /* aims below the K-th value (forces the second pass, tests)*/
    int32_t max_secant_iters; /* Phase-2 secant steps before pure bisection; default 8     */
    int32_t force_cluster;    /* 0 = automatic; else CTAs per row (1,2,4,8)                */
    int32_t guess_stride;     /* Phase-1 statistics over every n-th guessed position;      */
                              /* 0 = default 4 (R29); 1 = all of them, as in    */
                              /* PAPER.md:449-457.  Never changes the result.             */
    int32_t batch_path;       /* batches of more than one wave: 0 = filter path            */
                              /* (gvr_filter_kernel streams the whole batch, then one     */
                              /* refine CTA per row); 1 = row path (one CTA streams and   */
                              /* refines each row).  Never changes the result.           */
} gvr_options;

/* GVR exact Top-K.  prev_topk: nullable device int32 [num_rows, k], the previous
 * step's Top-K.  Entries may be any int32: negative,
 * >= len, duplicated or all -1 are tolerated (ignored/used only as hints); NULL means
 * "no guess" and a deterministic stride sample of the row is used instead
 * (SPEC.md:287).  prev_topk may equal out_idx (in-place update of the feedback
 * buffer); any other overlap is an error.  row_lens: nullable device int32
 * [num_rows] (NULL => every row has row_stride elements). */
gvr_status gvr_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens,
                            int32_t num_rows, const int32_t* prev_topk, int32_t k,
                            int32_t* out_idx, cudaStream_t stream);

/* Same as gvr_topk_batched plus: opt (nullable), out_val (nullable device fp32
 * [num_rows, k]: the selected scores x[out_idx], 0 for padding),
 * stats (nullable device gvr_row_stats [num_rows]). */
gvr_status gvr_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens,
                               int32_t num_rows, const int32_t* prev_topk, int32_t k,
                               int32_t* out_idx, cudaStream_t stream, const gvr_options* opt,
                               float* out_val, gvr_row_stats* stats);

/* Same as gvr_topk_batched_ex (opt nullable; no values or stats), and records
 * caller-created CUDA events (cudaEventCreate; any may be NULL) on `stream`: right before
 * the Phase-1 guess kernel (guess_start), before the streaming kernel (stream_start),
 * after it (stream_end) and at the end of the call (call_end).  The streaming kernel is
 * gvr_filter_kernel on the batch filter path (then stream_end .. call_end times the
 * refine kernel), else gvr_topk_kernel (then stream_end == call_end).  For the caller's
 * per-kernel timing (the benchmark's roofline).  Events are not launches: recording them
 * between the kernels serialises the programmatic dependent launches.  Ownership of the
 * events stays with the caller. */
gvr_status gvr_topk_batched_events(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                   int32_t num_rows, const int32_t* prev_topk, int32_t k, int32_t* out_idx,
                                   cudaStream_t stream, cudaEvent_t guess_start, cudaEvent_t stream_start,
                                   cudaEvent_t stream_end, cudaEvent_t call_end, const gvr_options* opt);

/* Per-phase timing of the GVR kernel (the paper's GVR_PHASE_TIMING instrumentation,
 * PAPER.md:1645-1656): phase_ts is a device int64 [num_rows, 9] array receiving clock64()
 * of each row's CTA at: start, end of Phase 1 (the guess hand-off read), end of the
 * streaming pass, end of Phases 2-3, end of Phase 4, end; then %globaltimer (ns) at the
 * CTA's start and end, and the SM id (%smid) the CTA ran on.  Rows that take a fallback
 * or the len <= k path leave the intermediate clock64 stamps 0.  Same result as
 * gvr_topk_batched (prev_topk nullable). */
gvr_status gvr_topk_phase_timing(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                 int32_t num_rows, const int32_t* prev_topk, int32_t k, int32_t* out_idx,
                                 cudaStream_t stream, long long* phase_ts);

/* Radix-select baseline: 2048-bin shared-memory histogram rounds
 * over the sortable key (11/11/10 bits) with global re-reads and an early exit to an
 * in-shared-memory finish once the threshold bucket holds <= 2048 elements.  Same
 * output contract as gvr_topk_batched. */
gvr_status radix_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens,
                              int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream);

gvr_status radix_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                 int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream,
                                 float* out_val, gvr_row_stats* stats);

/* Same-geometry radix baseline: the radix select run on
 * the machinery of the GVR batch path ("identical thread-level
 * resources").  Pass 1 streams the whole batch once (persistent CTAs, TMA ring; long rows
 * split over several CTAs) into a 2048-bin histogram per row of the
 * paper's 16-bit "half" digit (top 11 bits of the fp16-rounded score's sortable key,
 * PAPER.md:138, 143-147); the K-th bin gives a collect threshold T1; pass 2 is the GVR
 * filter kernel at T1 and the GVR refine / fixup kernels finish the remaining digits on
 * the candidate lists.  Same output contract and scratch conventions as gvr_topk_batched
 * (no guess); two HBM passes per row. */
gvr_status radix2_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens,
                               int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream);

gvr_status radix2_topk_batched_ex(const float* scores, int64_t row_stride, const int32_t* row_lens,
                                  int32_t num_rows, int32_t k, int32_t* out_idx, cudaStream_t stream,
                                  float* out_val, gvr_row_stats* stats);

/* ---- DSA indexer (Eq. 1, lines 78-81) -------------------------
 * I_t[i] = sum_{j<64} w[r][j] * ReLU(q[r][j] . keys[set][i]) for i < row_lens[r], with
 * bf16 inputs and fp32 accumulation on tensor cores.  keys: device bf16
 * [num_sets][n_max][128] (RoPE applied, the indexer key cache); row_set: device int32
 * [num_rows], the key set of row r (the draft rows of an MTP request share one); row_lens:
 * device int32 [num_rows] or NULL (= n_max), each <= n_max; q: device bf16
 * [num_rows][64][128]; w: device fp32 [num_rows][64].  The score arithmetic is one fixed
 * order shared by every indexer entry point, so the scores are bit-identical across them.
 *
 * gvr_indexer_scores: the scores themselves, out: device fp32 [num_rows][out_stride]
 * (out_stride >= n_max; entries past row_lens[r] untouched). */
gvr_status gvr_indexer_scores(const void* keys, int64_t n_max, const int32_t* row_set, const int32_t* row_lens,
                              const void* q, const float* w, int32_t num_rows, float* out, int64_t out_stride,
                              cudaStream_t stream);

/* gvr_indexer_topk_batched: the fused indexer -> GVR Top-K: the exact
 * ordered Top-K of the rows' indexer scores (the gvr_indexer_scores values) without
 * writing the score rows: Phases 1-2 score only the guessed and the 4096 sample positions,
 * the one pass over the key cache scores each 256-key step in shared memory and keeps the
 * candidates >= T_c, and the refine kernel selects from the candidate lists.
 * score_scratch: device fp32 [num_rows][n_max], 16-byte aligned, caller-owned — written
 * only for the rows the lists cannot finish (rows of <= k keys, massive ties, a threshold
 * overshoot), which are then finished from their materialised scores.  n_max must be a
 * multiple of 4.  prev_topk, k, out_idx as in gvr_topk_batched.  Same errors as
 * gvr_topk_batched, plus GVR_ERR_UNSUPPORTED for n_max % 4 != 0 or a misaligned scratch. */
gvr_status gvr_indexer_topk_batched(const void* keys, int64_t n_max, const int32_t* row_set,
                                    const int32_t* row_lens, const void* q, const float* w,
                                    int32_t num_rows, const int32_t* prev_topk, int32_t k,
                                    int32_t* out_idx, float* score_scratch, cudaStream_t stream);

/* ---- host-buffer entry point (end-to-end use) ------------------------------------
 * A workspace owns device buffers for up to max_rows rows of row_stride elements and
 * k outputs.  gvr_topk_batched_host copies HOST scores/row_lens/prev (pinned memory
 * recommended) to the device on `stream`, runs gvr_topk_batched, copies the result
 * into HOST out_idx and synchronises `stream` before returning.  h_row_lens and
 * h_prev are nullable.  Returns GVR_ERR_INVALID_ARGUMENT if num_rows > max_rows or
 * the stride/k differ from the workspace's. */
typedef struct gvr_workspace gvr_workspace;
gvr_status gvr_workspace_create(int32_t max_rows, int64_t row_stride, int32_t k,
                                gvr_workspace** ws);
gvr_status gvr_workspace_destroy(gvr_workspace* ws);
gvr_status gvr_topk_batched_host(const float* h_scores, int64_t row_stride,
                                 const int32_t* h_row_lens, int32_t num_rows,
                                 const int32_t* h_prev, int32_t k, int32_t* h_out,
                                 gvr_workspace* ws, cudaStream_t stream);

/* Static string for a status code (never NULL). */
const char* gvr_status_string(gvr_status s);

/* Text of the last CUDA error behind a GVR_ERR_CUDA returned on this host thread. */
const char* gvr_last_cuda_error(void);

/* Library/ABI version: major*10000 + minor*100 + patch. */
int32_t gvr_version(void);

/* CTA timeline of the batch filter path (diagnostics).  kernel = 0: the
 * gvr_filter_kernel CTAs b < 4096 — globaltimer (ns) at entry, after the wait for Phases
 * 1-2, at exit, and the SM id; kernel = 1: the gvr_guess_kernel CTAs (one per row, rows
 * < 4096) — globaltimer at entry, at exit, when its loads have arrived and after Phase 1.  enable = 1 starts recording
 * (both kernels) for the following calls; enable = 0 synchronizes the device, copies
 * min(max_ctas, 4096) records of 4 int64 each of the chosen kernel into host_out (caller-
 * owned, 4 * max_ctas int64), stores the count in *n_out (may be NULL) and stops recording.
 * Records of CTAs that did not run since enabling are stale.  GVR_ERR_INVALID_ARGUMENT for
 * a kernel other than 0/1, or host_out == NULL or max_ctas < 0 when enable == 0;
 * GVR_ERR_CUDA on a CUDA failure. */
gvr_status gvr_cta_timeline(int32_t kernel, int32_t enable, int64_t* host_out, int32_t max_ctas, int32_t* n_out);

/* Launch geometry of the two kernels on the current device (diagnostics): resident CTAs
 * per SM, threads per CTA and dynamic shared memory per CTA.  Any pointer may be NULL.
 * Returns GVR_ERR_CUDA if the occupancy query fails (no device). */
gvr_status gvr_kernel_info(int32_t* gvr_ctas_per_sm, int32_t* gvr_threads, int32_t* gvr_smem_bytes,
                           int32_t* radix_ctas_per_sm, int32_t* radix_threads, int32_t* radix_smem_bytes);

#ifdef __cplusplus
}
#endif
#endif /* GVR_TOPK_H */
