// refine_kernel.cuh — the batch path's refine step: Phase 4 and the ordered output from the
// candidate lists gvr_filter_kernel leaves in L2.
//
// A persistent grid of four small CTAs per SM (37 KB of shared memory, <= 64 registers)
// launched behind the filter with programmatic dependent launch: one wave covers a decode
// batch, and CTAs that find room early start on the rows already complete.  CTAs pop rows
// from the ready queue in the // order their lists complete.  Per row (all of it exact key-space arithmetic):
//   * the row's <= F_SEGS list segments and their largest keys (filter records);
//   * Phase 4 fused with the ordered output (R28), over the
//     list itself, read from L2: a 2048-bin linear histogram of the keys >= T_c over
//     [T_c, kmax] (bin 0 = highest), the bin holding sorted position K-1 from the bin scan,
//     the entries of the bins up to it counting-sorted into shared memory as 64-bit
//     composites (key, ~index), each ranked inside its bin, and position j < K written to
//     out[j] — score descending, index ascending;
//   * rows this cannot finish — no tiles (len <= k or tiny rows), a list that overflowed its
//     region or holds fewer than K keys >= T_c (the guess overshot), a K-th bin crowded by
//     ties — go to the fixup list, worked off by gvr_topk_kernel in fixup mode.
// Phase 2 (the secant search) ran in gvr_guess_kernel over the row
// sample, so the list is {key >= T_c} with K <= f(T_c) ~ 1.3-2 K (R34-R36).
#pragma once
#include "filter_kernel.cuh"

namespace gvr {

constexpr int RF_NT = 256;
constexpr int RF_CSORT = 2560;     // entries up to the K-th bin sorted in shared memory
constexpr int RF_MAXLIST = 1 << 22;  // longest list refined here
constexpr int RF_BIN_FAST = 16;    // largest bin ranked without narrowing first
using RefineGroup = Group<RF_NT, 1>;
constexpr int RF_OFF_HIST = 0;                       // int32 bin counts
constexpr int RF_OFF_CUR = RF_OFF_HIST + NBINS * 4;  // int32 bin cursors
constexpr int RF_OFF_CS = RF_OFF_CUR + NBINS * 4;
constexpr int RF_OFF_ROW = RF_OFF_CS + RF_CSORT * 8;
constexpr int RF_OFF_SCR = RF_OFF_ROW + 16;
constexpr int RF_SMEM_BYTES = RF_OFF_SCR + GROUP_SCRATCH_BYTES;
constexpr int RF_CTAS_PER_SM = 4;  // one wave for a decode batch: the per-row work is latency bound
static_assert(RF_CTAS_PER_SM * (RF_SMEM_BYTES + 1024) <= 233472, "refine CTAs per SM");


// Visit the row's list in batches of UNR entries per thread, segment by segment (segment s:
// n[s] entries from region position gs[s]; a row with len <= k is one segment read from
// the row itself, rowx).  fn(kv, aux, valid) gets the keys, a validity mask and per entry
// either its region position (or row position) or, WITH_IDX, its row index (the entry's
// second word, loaded with the key).
template <int UNR, bool WITH_IDX = false, class Fn>
__device__ __forceinline__ void for_list(const RefineGroup& c, const CandLists& cl, const float* rowx,
                                         const int (&gs)[F_SEGS], const int (&n)[F_SEGS], Fn&& fn)
{
    const uint32_t* rk = reinterpret_cast<const uint32_t*>(cl.region);
#pragma unroll
    for (int s = 0; s < F_SEGS; ++s) {
        const int base = gs[s], ns = n[s];
        for (int j0 = c.tid; j0 < ns; j0 += UNR * RF_NT) {
            uint32_t kv[UNR];
            int aux[UNR];
            uint32_t valid = 0u;
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int j = j0 + u * RF_NT;
                const int pos = base + j;
                kv[u] = 0u;
                aux[u] = pos;
                if (j < ns) {
                    if (rowx) {
                        kv[u] = f2key(__ldg(rowx + pos));
                    } else if (WITH_IDX) {
                        const uint2 e = __ldcg(cl.region + pos);
                        kv[u] = e.x;
                        aux[u] = (int)e.y;
                    } else {
                        kv[u] = __ldcg(rk + 2 * (size_t)pos);
                    }
                    valid |= 1u << u;
                }
            }
            fn(kv, aux, valid);
        }
    }
}

__global__ void __launch_bounds__(RF_NT, RF_CTAS_PER_SM)
gvr_refine_kernel(const float* __restrict__ scores, int64_t stride, const int32_t* __restrict__ row_lens, int k,
                  int num_rows, int32_t* out, float* out_val, gvr_row_stats* stats, const GuessOut* gp, CandLists cl,
                  BatchQueue bq, long long* phase_ts, bool fused = false, int32_t* ctl = nullptr)
{
    // the fixup grid may be scheduled now: it waits for this grid's release flag (ctl)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // fused (the indexer path, indexer_kernel.cuh): the score rows do not exist, so rows
    // that need them — len <= k, the ties fill — go to the fixup list, which materialises them
    // phase_ts (optional, [num_rows][TS_N]): clock64 at the pop, after the segment records,
    // after the histogram pass, after the K-th bin search, after the scatter, at the end;
    // then globaltimer at the pop and the end, and the SM id.
    extern __shared__ __align__(128) unsigned char smem[];
    int32_t* hist = reinterpret_cast<int32_t*>(smem + RF_OFF_HIST);
    int32_t* cur = reinterpret_cast<int32_t*>(smem + RF_OFF_CUR);
    unsigned long long* cs = reinterpret_cast<unsigned long long*>(smem + RF_OFF_CS);
    int* sh_row = reinterpret_cast<int*>(smem + RF_OFF_ROW);
    RefineGroup c;
    c.init(threadIdx.x, smem + RF_OFF_SCR);
    const int K = k;
    constexpr int BPT = NBINS / RF_NT;
    constexpr int UNR = 8;
    // thread 0 claims the next queue slot during the current row's last step (ranking),
    // so the claim's round trip is off the critical path without hoarding rows early
    int next_slot = -1;
    for (;;) {
        if (c.tid == 0) {
            const int slot = next_slot >= 0 ? next_slot : atomicAdd(bq.qctl + Q_HEAD, 1);
            next_slot = -1;
            int r = -1;
            if (slot < num_rows) {
                int v;
                while ((v = ld_acquire(bq.queue + slot)) == 0) __nanosleep(100);
                r = v - 1;
                bq.queue[slot] = 0;
            }
            *sh_row = r;
        }
        c.sync();
        const int r = *sh_row;
        if (r < 0) break;
        long long tsr[TS_N] = {phase_ts ? clock64() : 0ll, 0, 0, 0, 0, 0, phase_ts ? global_ns() : 0ll, 0, 0};
        // the segment records, the row length and T_c are loaded together (the records of
        // slots past the row's segment count are stale and ignored)
        const int4 erec = c.warp == 0 && c.lane < F_SEGS ? __ldcg(cl.rec + (long long)r * F_SEGS + c.lane)
                                                         : make_int4(0, 0, 0, 0);
        const uint4 g0 = __ldcg(reinterpret_cast<const uint4*>(gp + r));      // Tc, tie, tmin, top
        const uint4 g1 = __ldcg(reinterpret_cast<const uint4*>(gp + r) + 1);  // T0, iters | exit, ...
        uint32_t Tc = g0.x;
        const uint32_t tie = g0.y;
        const RowPlan p = plan_row(scores, stride, row_lens, r, k);
        // ---- the row's list segments (filter records)
        int total = -1;
        uint32_t kmax = 0u;
        if (p.ntiles > 0 && c.warp == 0) {
            const long long v0 = (long long)r * cl.tpr;
            const int b0 = cl_cta_of(cl, v0);
            const int ns = cl_cta_of(cl, v0 + p.ntiles - 1) - b0 + 1;
            int gsv = 0, n = 0, bad = ns > F_SEGS ? 1 : 0;
            uint32_t km = 0u;
            if (c.lane < ns && c.lane < F_SEGS) {
                const int4 e = erec;
                bad = (e.x != b0 + c.lane || e.y < 0 || e.z < e.y || e.z > cl.reg) ? 1 : 0;
                gsv = e.x * cl.reg + e.y;
                n = e.z - e.y;
                km = (uint32_t)e.w;
            }
            bad = __any_sync(FULL, bad);
            const int tot = (int)__reduce_add_sync(FULL, (uint32_t)n);
            km = __reduce_max_sync(FULL, km);
            if (c.lane < F_SEGS) {
                c.misc[24 + 2 * c.lane] = gsv;
                c.misc[25 + 2 * c.lane] = n;
            }
            if (c.lane == 0) {
                c.misc[22] = bad ? -1 : tot;
                c.misc[23] = (int)km;
                bq.segdone[r] = 0;  // popped: reset for the next call
            }
        }
        c.sync();
        int gs[F_SEGS], ns[F_SEGS];
#pragma unroll
        for (int s = 0; s < F_SEGS; ++s) gs[s] = ns[s] = 0;
        if (p.ntiles > 0) {
            total = c.misc[22];
            kmax = (uint32_t)c.misc[23];
#pragma unroll
            for (int s = 0; s < F_SEGS; ++s) {
                gs[s] = c.misc[24 + 2 * s];
                ns[s] = c.misc[25 + 2 * s];
            }
        }
        bool ok = p.ntiles > 0 && p.n > k && total >= K && total <= RF_MAXLIST && kmax >= Tc;
        // a Phase-2 ties exit collected the keys strictly above the tied key (R37): when
        // they are fewer than K, all of them lead the output and the tie's lowest indices
        // follow (an ordered scan of the row below)
        const int p2exit = (int)(int16_t)(g1.y >> 16);
        const bool tie_fill = p.ntiles > 0 && p.n > k && p2exit == GVR_P2_TIES && tie < 0xffffffffu &&
                              Tc == tie + 1u && total >= 0 && total < K;
        if (tie_fill) ok = !fused && (total == 0 || kmax >= Tc);
        // a row with len <= k: every element is selected (take = len), binned over its own
        // key range [min, max], then -1 padding (R5)
        const bool trivial = p.n <= k;
        const float* rowx = nullptr;
        int take = tie_fill ? total : K;
        if (trivial && fused) ok = false;
        if (trivial && !fused) {
            uint32_t mn = 0xffffffffu, mx2 = 0u;
            for (int q = c.tid; q < p.n; q += RF_NT) {
                const uint32_t kv = f2key(__ldg(p.x + q));
                mn = min(mn, kv);
                mx2 = max(mx2, kv);
            }
            group_red2<R_MIN, R_MAX>(c, mn, mx2);
            rowx = p.x;
            total = p.n;
            take = p.n;
            gs[0] = 0;  // one segment: the row itself
            ns[0] = p.n;
#pragma unroll
            for (int s = 1; s < F_SEGS; ++s) ns[s] = 0;
            Tc = mn;
            kmax = mx2;
            ok = p.n > 0;
        }
        if (phase_ts) tsr[TS_PHASE1] = clock64();
        int ftc = 0, nsel = 0, levels = 0;
        if (ok && take > 0) {
            // ---- Phase 4: histogram of the keys >= lo over [lo, kmax],
            // the K-th bin from the bin scan.  lo starts at T_c; if the
            // bins up to the K-th one are too crowded to rank (keys spread over a wide key
            // range, e.g. both signs, leave the top K in few linear bins), lo is raised to
            // the K-th bin's lower edge and the histogram redone over the narrower range
            // (every key >= lo still holds the first `take` positions).
            uint32_t lo = Tc, scale = 0u, off0 = 0u;
            const int b0 = c.tid * BPT;
            int h[BPT];
            int bk = -1;
            for (int lvl = 0; lvl < 3; ++lvl) {
                levels = lvl + 1;
                reinterpret_cast<int4*>(hist + b0)[0] = make_int4(0, 0, 0, 0);
                reinterpret_cast<int4*>(hist + b0)[1] = make_int4(0, 0, 0, 0);
                if (c.tid == 0) c.misc[12] = -1;  // K-th bin: set below by the thread that holds it
                c.sync();
                scale = bin_scale((uint64_t)kmax - lo + 1ull);
                uint32_t f = 0;
                for_list<16>(c, cl, rowx, gs, ns, [&](const uint32_t (&kv)[16], const int (&)[16], uint32_t valid) {
#pragma unroll
                    for (int u = 0; u < 16; ++u)
                        if ((valid >> u & 1u) && kv[u] >= lo) {
                            atomicAdd(&hist[(NBINS - 1) - lin_bin(kv[u] - lo, scale)], 1);
                            ++f;
                        }
                });
                f = group_red1<R_ADD>(c, f);  // its barrier also completes the histogram
                if (lvl == 0) {
                    ftc = (int)f;
                    if (phase_ts) tsr[TS_STREAM] = clock64();
                }
                uint32_t loc = 0;
                {
                    const int4 h0 = reinterpret_cast<const int4*>(hist + b0)[0];
                    const int4 h1 = reinterpret_cast<const int4*>(hist + b0)[1];
                    h[0] = h0.x, h[1] = h0.y, h[2] = h0.z, h[3] = h0.w;
                    h[4] = h1.x, h[5] = h1.y, h[6] = h1.z, h[7] = h1.w;
                }
#pragma unroll
                for (int i = 0; i < BPT; ++i) loc += (uint32_t)h[i];
                uint32_t tot;
                off0 = group_excl_scan(c, loc, tot);
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
                bk = ftc >= take ? c.misc[12] : -1;
                nsel = c.misc[13];
                uint32_t mx = 0;
#pragma unroll
                for (int i = 0; i < BPT; ++i)
                    if (b0 + i <= bk) mx = max(mx, (uint32_t)h[i]);
                mx = group_red1<R_MAX>(c, mx);
                ok = bk >= 0 && nsel <= RF_CSORT && mx <= (uint32_t)CSORT_BIN_MAX;  // group-uniform
                // narrow also when the ranking would loop over bins of more than RF_BIN_FAST
                if (bk < 0 || lvl == 2 || (ok && mx <= (uint32_t)RF_BIN_FAST)) break;
                // lower edge of bin bk: the smallest d with lin_bin(d) = NBINS - 1 - bk
                const uint64_t L = (uint64_t)(NBINS - 1 - bk);
                const uint64_t dmin = ((L << 32) + scale - 1ull) / scale;
                if (dmin == 0ull) break;  // the K-th bin is the lowest: narrowing cannot help
                lo += (uint32_t)dmin;
            }
            if (phase_ts) tsr[TS_PHASE23] = clock64();
            if (ok) {
                {
                    // bin starts; they become the bin ends after the scatter
                    int st[BPT];
                    int off = (int)off0;
#pragma unroll
                    for (int i = 0; i < BPT; ++i) {
                        st[i] = off;
                        off += h[i];
                    }
                    reinterpret_cast<int4*>(cur + b0)[0] = make_int4(st[0], st[1], st[2], st[3]);
                    reinterpret_cast<int4*>(cur + b0)[1] = make_int4(st[4], st[5], st[6], st[7]);
                }
                c.sync();
                // ---- counting sort of the bins up to the K-th bin (composites)
                for_list<UNR, true>(c, cl, rowx, gs, ns, [&](const uint32_t (&kv)[UNR], const int (&ix)[UNR], uint32_t valid) {
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const int b = (valid >> u & 1u) && kv[u] >= lo ? (NBINS - 1) - lin_bin(kv[u] - lo, scale) : NBINS;
                        if (b <= bk) cs[atomicAdd(&cur[b], 1)] = make_comp(kv[u], ix[u]);
                    }
                });
                c.sync();
                if (phase_ts) tsr[TS_PHASE4] = clock64();
                if (c.tid == 0) next_slot = atomicAdd(bq.qctl + Q_HEAD, 1);
                // ---- rank inside the bin; positions < K are the ordered output
                int32_t* o = out + (int64_t)r * k;
                float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
                for (int j = c.tid; j < nsel; j += RF_NT) {
                    const unsigned long long v = cs[j];
                    const int b = (NBINS - 1) - lin_bin(comp_key(v) - lo, scale);
                    const int cnt = hist[b];
                    const int st = cur[b] - cnt;
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
                        o[pos] = comp_idx(v);
                        if (ov) ov[pos] = key2f(comp_key(v));
                    }
                }
                if (!tie_fill)
                    for (int j = take + c.tid; j < k; j += RF_NT) {  // len < k: -1 padding
                        o[j] = -1;
                        if (ov) ov[j] = 0.f;
                    }
            }
        }
        if (ok && tie_fill) {
            // positions [take, K): the first K - take elements of the row equal to the tied
            // key, in index order — thread t scans 8 consecutive elements per step, an
            // exclusive scan orders the matches; fewer than needed: the tie is not the K-th
            // key after all and the row goes to the fixup list
            int32_t* o = out + (int64_t)r * k;
            float* ov = out_val ? out_val + (int64_t)r * k : nullptr;
            const int need = K - take;
            int found = 0;
            for (int base = 0; base < p.n && found < need; base += 8 * RF_NT) {
                const int i0 = base + 8 * c.tid;
                uint32_t hit = 0u;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (i0 + j < p.n && f2key(__ldg(p.x + i0 + j)) == tie) hit |= 1u << j;
                uint32_t tot;
                uint32_t pos = (uint32_t)(take + found) + group_excl_scan(c, (uint32_t)__popc(hit), tot);
                for (; hit; hit &= hit - 1u, ++pos)
                    if (pos < (uint32_t)K) {
                        o[pos] = i0 + __ffs(hit) - 1;
                        if (ov) ov[pos] = key2f(tie);
                    }
                found += (int)tot;
            }
            ok = found >= need;
            levels = 0;
            ftc = total;
        }
        if (trivial && p.n == 0 && !fused) {
            int32_t* o = out + (int64_t)r * k;
            for (int j = c.tid; j < k; j += RF_NT) {
                o[j] = -1;
                if (out_val) out_val[(int64_t)r * k + j] = 0.f;
            }
            ok = true;
        }
        if (c.tid == 0) {
            if (!ok) {
                // a complete list with fewer than K keys >= T_c: the fixup streams the row at
                // the second-pass threshold directly (flag bit 31)
                const bool short_list = p.ntiles > 0 && p.n > k && total >= 0 && total < K;
                bq.fixlist[atomicAdd(bq.qctl + Q_NFIX, 1)] = (int32_t)((uint32_t)r | (short_list ? 0x80000000u : 0u));
            } else if (stats) {
                const GuessOut g = trivial ? GuessOut{} : gp[r];
                gvr_row_stats s;
                s.secant_iters = g.iters;  // Phase-2 probes (gvr_guess_kernel)
                s.snap_iters = 0;
                s.cand_count = trivial ? p.n : ftc;
                s.done_kind = trivial ? GVR_DONE_TRIVIAL : tie_fill ? GVR_DONE_TIEFILL : GVR_DONE_CONVERGED;
                s.global_passes = tie_fill ? 2 : 1;  // the tie scan reads (part of) the row again
                s.raises = levels > 1 ? levels - 1 : 0;  // Phase-4 histogram narrowings (R32)
                s.buffer_count = trivial ? 0 : ftc;
                s.cluster = 1;
                s.phase2_exit = g.exit;
                s.sample_count = g.scount;
                s.tc_key = g.Tc;
                s.reserved = 0;
                stats[r] = s;
            }
            if (phase_ts && ok) {
                tsr[TS_END] = clock64();
                tsr[TS_GEND] = global_ns();
                tsr[TS_SMID] = sm_id();
                for (int i = 0; i < TS_N; ++i) phase_ts[(int64_t)r * TS_N + i] = tsr[i];
            }
        }
        c.sync();  // smem (row slot, histogram, sort buffer) is reused for the next row
    }
    // the last CTA to finish releases the fixup grid (its list is complete)
    if (c.tid == 0 && ctl) {
        __threadfence();
        if (atomicAdd(bq.qctl + Q_RDONE, 1) == (int)gridDim.x - 1) {
            __threadfence();
            st_release(ctl + CTL_RDONE, 1);
        }
    }
}

}  // namespace gvr
