/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU definition of what the GVR hot path
 * computes: the exact Top-K of each row, ordered by (score descending, index
 * ascending).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * header, helper, table or constant with the CUDA path (paper_2604_22312_b200/)
 * and the CUDA path never loads it.
 *
 * Passages followed (PAPER.md = /root/reference/PAPER.md, SPEC.md likewise):
 *   - Problem statement, PAPER.md:385-388 (Sec. 4.1 "Core Idea"): S* = indices
 *     of the K largest values of x.
 *   - Sortable FP32 key, PAPER.md:144-148 (Sec. 2.2) and SPEC.md:335-343:
 *     negative values flip all bits, non-negative values flip the sign bit.
 *   - Tie rule "lowest index wins" and sorted output: BASELINE.json north_star
 *     ("score descending, then index ascending"; "bit-exactly, both as an
 *     index set and in order").  The paper itself is
 *     non-deterministic on ties; reading R1.
 *   - n < k: emit all n in order, then -1 padding (reading R5).
 *
 * Two independent formulations are provided:
 *   oracle_topk_row       : full sort of (key, idx) pairs with qsort.
 *   oracle_topk_rank_row  : O(n^2) rank counting, rank_i = #{j : j precedes i}.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

uint32_t oracle_sortable_key(float x)
{
    uint32_t u;
    memcpy(&u, &x, sizeof u);
    /* negative -> flip all bits; non-negative -> flip sign bit */
    if (u & 0x80000000u) return ~u;
    return u | 0x80000000u;
}

typedef struct {
    uint32_t key;
    int32_t idx;
} oracle_pair;

/* i precedes j  <=>  key_i > key_j, or key_i == key_j and i < j */
static int oracle_cmp(const void* a, const void* b)
{
    const oracle_pair* p = (const oracle_pair*)a;
    const oracle_pair* q = (const oracle_pair*)b;
    if (p->key != q->key) return (p->key > q->key) ? -1 : 1;
    if (p->idx != q->idx) return (p->idx < q->idx) ? -1 : 1;
    return 0;
}

/* Returns 0 on success, -1 on bad arguments / allocation failure. */
int oracle_topk_row(const float* x, int64_t n, int32_t k, int32_t* out)
{
    if (n < 0 || k < 0 || (n > 0 && x == NULL) || (k > 0 && out == NULL)) return -1;
    oracle_pair* pairs = NULL;
    if (n > 0) {
        pairs = (oracle_pair*)malloc((size_t)n * sizeof(oracle_pair));
        if (!pairs) return -1;
    }
    for (int64_t i = 0; i < n; ++i) {
        pairs[i].key = oracle_sortable_key(x[i]);
        pairs[i].idx = (int32_t)i;
    }
    if (n > 1) qsort(pairs, (size_t)n, sizeof(oracle_pair), oracle_cmp);
    for (int32_t r = 0; r < k; ++r) out[r] = (r < n) ? pairs[r].idx : -1;
    free(pairs);
    return 0;
}

/* Second formulation: the rank of i is the number of j that precede it. */
int oracle_topk_rank_row(const float* x, int64_t n, int32_t k, int32_t* out)
{
    if (n < 0 || k < 0 || (n > 0 && x == NULL) || (k > 0 && out == NULL)) return -1;
    for (int32_t r = 0; r < k; ++r) out[r] = -1;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t ki = oracle_sortable_key(x[i]);
        int64_t rank = 0;
        for (int64_t j = 0; j < n; ++j) {
            uint32_t kj = oracle_sortable_key(x[j]);
            if (kj > ki || (kj == ki && j < i)) ++rank;
        }
        if (rank < k) out[rank] = (int32_t)i;
    }
    return 0;
}

typedef struct {
    const float* scores;
    int64_t row_stride;
    const int32_t* row_lens;
    int32_t num_rows;
    int32_t k;
    int32_t* out;
    int32_t next_row;
    int32_t failed;
    pthread_mutex_t lock;
} oracle_job;

static void* oracle_worker(void* arg)
{
    oracle_job* job = (oracle_job*)arg;
    for (;;) {
        pthread_mutex_lock(&job->lock);
        int32_t r = job->next_row++;
        pthread_mutex_unlock(&job->lock);
        if (r >= job->num_rows) break;
        int64_t n = job->row_lens ? (int64_t)job->row_lens[r] : job->row_stride;
        if (oracle_topk_row(job->scores + (int64_t)r * job->row_stride, n, job->k,
                            job->out + (int64_t)r * job->k) != 0) {
            pthread_mutex_lock(&job->lock);
            job->failed = 1;
            pthread_mutex_unlock(&job->lock);
        }
    }
    return NULL;
}

/* Host rows [num_rows, row_stride] fp32; row_lens nullable (=> row_stride).
 * out [num_rows, k] int32.  Rows are independent; one row per task. */
int oracle_topk_batched(const float* scores, int64_t row_stride, const int32_t* row_lens,
                        int32_t num_rows, int32_t k, int32_t* out, int32_t num_threads)
{
    if (num_rows < 0 || k < 0 || row_stride < 0) return -1;
    if (row_lens) {
        for (int32_t r = 0; r < num_rows; ++r)
            if (row_lens[r] < 0 || row_lens[r] > row_stride) return -1;
    }
    oracle_job job;
    job.scores = scores;
    job.row_stride = row_stride;
    job.row_lens = row_lens;
    job.num_rows = num_rows;
    job.k = k;
    job.out = out;
    job.next_row = 0;
    job.failed = 0;
    pthread_mutex_init(&job.lock, NULL);
    if (num_threads < 1) num_threads = 1;
    if (num_threads > 256) num_threads = 256;
    pthread_t tids[256];
    int started = 0;
    for (int t = 0; t < num_threads; ++t) {
        if (pthread_create(&tids[t], NULL, oracle_worker, &job) != 0) break;
        ++started;
    }
    if (started == 0) oracle_worker(&job);
    for (int t = 0; t < started; ++t) pthread_join(tids[t], NULL);
    pthread_mutex_destroy(&job.lock);
    return job.failed ? -1 : 0;
}
