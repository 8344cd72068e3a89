/*
 * memcolor_b200.h -- C ABI of the B200-native batched local-search engine.
 *
 * Drop-in boundary for the data-parallel hot path of the reference package
 * `memcolor` (arxiv 2109.05948; paths below are relative to
 * /root/reference/pkg/src/memcolor/).  Each entry point replaces one numba
 * kernel and takes exactly that kernel's arrays, as pointer + sizes, with
 * the same in/out roles:
 *
 *   mcb_tabucol_batch  <- _tabucol_batch   localsearch.py:266-286 (body :287-410)
 *   mcb_wvcp_batch     <- _wvcp_batch      localsearch.py:89-119  (body :120-263)
 *   mcb_gpx_batch      <- _gpx_batch       crossover.py:60-66     (+ _gpx_into :14-57)
 *   mcb_pairwise       <- _pairwise_kernel distance.py:90-119     (+ _greedy_match_total :40-72)
 *   mcb_stream_values  <- stream_value     rng.py:56-59 (known-answer tests)
 *
 * Conventions
 *  - Plain `mcb_*` functions take DEVICE pointers and enqueue on `stream`
 *    (a cudaStream_t, NULL = legacy default stream); they do not synchronise
 *    unless stated.  `mcb_*_host` variants take HOST pointers, perform the
 *    host<->device copies themselves and return after the results are back
 *    (the ctypes binding a reference maintainer adds).
 *  - Array layouts are row-major and exactly the reference's dtypes:
 *    assigns int32[p,n], adj_indptr int64[n+1], adj_indices int32[2m],
 *    edges_u/edges_v int32[m], keys uint64[p], scalar outputs int64[p].
 *  - Ownership follows `_run_tabucol_batch` (localsearch.py:556-598):
 *    `assigns` is overwritten with the end state; every output is
 *    preallocated by the caller.
 *  - Errors: nonzero status; `mcb_last_error()` gives the message.  The
 *    Python shim maps MCB_ERR_VALUE/UNSUPPORTED/RANGE to ValueError and
 *    MCB_ERR_CUDA to RuntimeError; a nonzero `diag[i]` (incremental state
 *    diverged from scratch recomputation, localsearch.py:398-405) is mapped to
 *    AssertionError exactly like localsearch.py:589-590.
 */
#ifndef MEMCOLOR_B200_H
#define MEMCOLOR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCB_OK 0
#define MCB_ERR_VALUE 1
#define MCB_ERR_CUDA 2
#define MCB_ERR_UNSUPPORTED 3
#define MCB_ERR_RANGE 4

/* flags */
#define MCB_FLAG_DIAG 0x1u         /* scratch re-evaluation every 1024 iterations (reference behaviour) */
#define MCB_FLAG_PRODUCTION 0x2u   /* Philox4x32 tie-break + tenure draws instead of SplitMix64 streams */
#define MCB_FLAG_FORCE_WIDE 0x4u   /* int16 gamma / 32-bit tabu stamps from the start (tests) */
#define MCB_FLAG_FORCE_GLOBAL 0x8u /* gamma/tabu tables in global memory (L2-resident path, tests) */
#define MCB_FLAG_PROFILE 0x100u    /* accumulate per-phase clock64 cycles (mcb_debug_phase_cycles) */
#define MCB_FLAG_WSTATS 0x200u     /* warp kernel: event counters + phase cycles (mcb_debug_warp_stats) */
#define MCB_FLAG_FORCE_CLUSTER 0x800u /* TabuCol on the 2-CTA cluster kernel whatever the shape (tests) */
#define MCB_FLAG_ASYNC 0x400u      /* mcb_tabucol_batch: no host synchronisation (per-stream scratch, every
                                      fallback pass enqueued with device-side counts; CUDA-graph capturable
                                      after one warm-up call); errors via mcb_tabucol_async_status */

const char *mcb_version(void);
const char *mcb_last_error(void);
int mcb_device_count(void);

/* Diagnostics: aggregate shared-memory read bandwidth of the current device
 * (GB/s), measured with a conflict-free LDS.128 stream; the roofline
 * denominator of the shared-memory-bound kernels. */
int mcb_probe_smem_bandwidth(double *gbs, double *ms);
/* L2 read bandwidth (16-byte loads, L1 bypassed, 48 MB resident buffer): the
 * roofline denominator of the out-of-shared-memory TabuCol shapes. */
int mcb_probe_l2_bandwidth(double *gbs, double *ms);
/* Diagnostics: per-phase cycle totals of the TabuCol iteration accumulated
 * by runs with MCB_FLAG_PROFILE (out: 16 counters; [10] = iterations; the
 * CTA kernel's and the cluster kernel's counters, see tabucol_cluster.cu). */
int mcb_debug_phase_cycles(unsigned long long *out, int reset);
/* Diagnostics: counters of the last warp-kernel TabuCol launch made with
 * MCB_FLAG_WSTATS (out: 40 counters, see tabucol_warp.cu WS_*). */
int mcb_debug_warp_stats(unsigned long long *out);
/* Cluster TabuCol kernel under MCB_FLAG_PROFILE, rank-0 CTAs: per warp w,
 * out[w] pass-1 cycles, out[32+w] start delays, out[64+w] warp scans (96). */
int mcb_debug_cluster_warps(unsigned long long *out, int reset);
/* Group-of-warps TabuCol kernel run with MCB_GSTATS=1 in the environment:
 * thread 0's cycles per phase (out: 32 counters; [15] = iterations). */
int mcb_debug_group_stats(unsigned long long *out);
/* WVCP kernel under MCB_FLAG_WSTATS: out[0] iterations, out[1..8] thread 0's
 * cycles per phase (pass 1, chunk minima, prefix + walks, warp-0 section,
 * gamma update, class refresh, best copy, tail); reset != 0 clears them. */
int mcb_debug_wvcp_stats(unsigned long long *out, int reset);
/* Diagnostics: the exact fp64 divisibility test of the reservoir draws against
 * the 64-bit integer %, on `count` pseudo-random pairs; out: #mismatches. */
int mcb_debug_modcheck(int64_t count, unsigned long long *mismatches);
/* Diagnostics: which TabuCol kernel variant a call with (n, k, p) launches on
 * the current device, as text (no launch). */
int mcb_tabucol_describe(int64_t n, int64_t k, int64_t p, char *buf, int len);

/* out[i] = stream_value(keys[i], ctrs[i]) (rng.py:56-59); device pointers. */
int mcb_stream_values(const uint64_t *keys, const uint64_t *ctrs, uint64_t *out, int64_t count,
                      void *stream);

/*
 * Batched TabuCol (localsearch.py:266-410).  One individual per CTA.
 * log_* may be NULL when log_cap == 0.  counters (nullable) receives int64[p,2]:
 * sum over iterations of the conflicting-vertex count and of deg(v*) (the
 * algorithmic-bytes counters of SURVEY.md 8(d)).
 */
int mcb_tabucol_batch(int32_t *assigns, int64_t p, int64_t n, int64_t k,
                      const int64_t *adj_indptr, const int32_t *adj_indices,
                      const int32_t *edges_u, const int32_t *edges_v, int64_t m,
                      int64_t depth, const uint64_t *keys,
                      int32_t *best_assigns, int64_t *best_conflicts, int64_t *end_conflicts,
                      int64_t *iters_used, int64_t *diag,
                      int64_t log_cap, int32_t *log_v, int64_t *log_iter, int64_t *log_tt,
                      int64_t *log_cnt, int64_t *counters, uint32_t flags, void *stream);
/* Status of the last MCB_FLAG_ASYNC mcb_tabucol_batch on `stream`
 * (synchronises the stream; MCB_ERR_RANGE for colours outside [0, k)). */
int mcb_tabucol_async_status(void *stream);
int mcb_tabucol_batch_host(int32_t *assigns, int64_t p, int64_t n, int64_t k,
                           const int64_t *adj_indptr, const int32_t *adj_indices,
                           const int32_t *edges_u, const int32_t *edges_v, int64_t m,
                           int64_t depth, const uint64_t *keys,
                           int32_t *best_assigns, int64_t *best_conflicts, int64_t *end_conflicts,
                           int64_t *iters_used, int64_t *diag,
                           int64_t log_cap, int32_t *log_v, int64_t *log_iter, int64_t *log_tt,
                           int64_t *log_cnt, int64_t *counters, uint32_t flags, void *stream);

/*
 * Batched weighted-colouring tabu search (localsearch.py:89-263).
 * phi_used is double[p, rounds+1]; log_asp int8[p, log_cap].
 */
int mcb_wvcp_batch(int32_t *assigns, int64_t p, int64_t n, int64_t k,
                   const int64_t *adj_indptr, const int32_t *adj_indices,
                   const int32_t *edges_u, const int32_t *edges_v, int64_t m,
                   const int32_t *wranks, const int64_t *wvals, int64_t nranks,
                   const int64_t *weights, int64_t depth, int64_t rounds, int32_t schedule_on,
                   const double *phi0s, double forced_phi, int64_t tt_base, const uint64_t *keys,
                   int32_t *best_assigns, int64_t *best_scores, int64_t *end_scores,
                   int64_t *end_conflicts, double *phi_used, int64_t *diag,
                   int64_t log_cap, int32_t *log_v, int64_t *log_iter, int64_t *log_tt,
                   int8_t *log_asp, int64_t *log_cnt, uint32_t flags, void *stream);
int mcb_wvcp_batch_host(int32_t *assigns, int64_t p, int64_t n, int64_t k,
                        const int64_t *adj_indptr, const int32_t *adj_indices,
                        const int32_t *edges_u, const int32_t *edges_v, int64_t m,
                        const int32_t *wranks, const int64_t *wvals, int64_t nranks,
                        const int64_t *weights, int64_t depth, int64_t rounds, int32_t schedule_on,
                        const double *phi0s, double forced_phi, int64_t tt_base,
                        const uint64_t *keys, int32_t *best_assigns, int64_t *best_scores,
                        int64_t *end_scores, int64_t *end_conflicts, double *phi_used,
                        int64_t *diag, int64_t log_cap, int32_t *log_v, int64_t *log_iter,
                        int64_t *log_tt, int8_t *log_asp, int64_t *log_cnt, uint32_t flags,
                        void *stream);

/*
 * Batched GPX crossover (crossover.py:14-66): out[i,j,:] = GPX(pop[i],
 * pop[matches[i,j]]) with stream keys[i*K+j].  out is int32[p,K,n].
 */
int mcb_gpx_batch(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t K,
                  int64_t k, const uint64_t *keys, int32_t *out, uint32_t flags, void *stream);
int mcb_gpx_batch_host(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches,
                       int64_t K, int64_t k, const uint64_t *keys, int32_t *out, uint32_t flags,
                       void *stream);
/*
 * Sharded GPX: the offspring of rows [row_off, row_off + rows) only; matches,
 * keys and out hold just those rows (matches[r,j] index the full population).
 * mcb_gpx_batch == mcb_gpx_rows with rows = p, row_off = 0.
 */
int mcb_gpx_rows(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t rows,
                 int64_t row_off, int64_t K, int64_t k, const uint64_t *keys, int32_t *out,
                 uint32_t flags, void *stream);

/*
 * Approximate partition distances over the reference's linear job space
 * (distance.py:90-119): jobs [0, p*q) -> cross[i,j] = d(pop_i, off_j);
 * jobs [p*q, p*q + q(q-1)/2) -> within[i,j] = within[j,i] = d(off_i, off_j).
 * Only jobs in [job_begin, job_end) are computed (job_end < 0: all), which is
 * how ranks shard the pass.  cross int32[p,q], within int32[q,q].
 */
int mcb_pairwise(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                 int64_t k, int32_t *cross, int32_t *within, int64_t job_begin, int64_t job_end,
                 uint32_t flags, void *stream);
int mcb_pairwise_host(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                      int64_t k, int32_t *cross, int32_t *within, int64_t job_begin,
                      int64_t job_end, uint32_t flags, void *stream);
/*
 * Sharded distances: a rank computes the job range
 * [job_begin, job_end) of the same job space and writes the distances
 * compactly, jobs16[j - job_begin] (int16: distances are <= n <= 32767);
 * the ranks all-gather those vectors and mcb_pairwise_scatter expands the
 * whole job space's vector into cross (p x q) and within (q x q, symmetric,
 * zero diagonal).  Device pointers, asynchronous on `stream` except
 * mcb_pairwise_jobs' range check of the colours (one flag read).
 */
int mcb_pairwise_jobs(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                      int64_t k, int16_t *jobs16, int64_t job_begin, int64_t job_end, uint32_t flags,
                      void *stream);
int mcb_pairwise_scatter(const int16_t *jobs16, int64_t p, int64_t q, int32_t *cross, int32_t *within,
                         void *stream);

/*
 * Population update (mc/population.py:59-127): merge p incumbents (pdist
 * p x p, fitness fit_pop) and q newcomers (cross p x q, within q x q,
 * fitness fit_new); admit candidates in (fitness, origin, index) order when
 * their distance to every admitted candidate exceeds ms; fill with the best
 * rejected ones.  out_adm int32[p] = admitted candidate ids in slot order
 * (0..p-1 incumbents, p.. newcomers), out_rule uint8[p] = admitted by the
 * spacing rule.  Optional (NULL to skip): out_dist int32[p,p] (the new
 * population's distance matrix), out_assigns int32[p,n] + out_fit int64[p]
 * (gathered from pop_assigns int32[p,n] / new_assigns int32[q,n]).  Device
 * pointers, asynchronous on `stream`.
 */
int mcb_update_population(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                          const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q, int64_t ms,
                          const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                          int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                          int64_t *out_fit, void *stream);
int mcb_update_population_host(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                               const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q,
                               int64_t ms, const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                               int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                               int64_t *out_fit, void *stream);
/*
 * K nearest neighbours of every individual by (distance, index), excluding
 * itself (mc/population.py:130-141): dist int32[p,p] with values in
 * [0, max_dist]; matches int64[p,K] in (distance, index) order.
 */
int mcb_match_parents(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                      void *stream);
int mcb_match_parents_host(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                           void *stream);
/*
 * Randomized greedy colourings for weighted runs, p at once
 * (mc/init.py:30-46 greedy_wvcp_init, :57-64 init_wvcp_population): every
 * individual i walks `order` int32[n] (the reference's greedy_order, :23-27)
 * with stream key keys[i] (= stream_key(seed, TAG_INIT, i)); CSR adjacency
 * indptr int64[n+1] / indices int32[2m].  Out: assigns int32[p,n] (legal
 * colourings) and used int32[p] (colours each opened; the run's palette is
 * their maximum).  MCB_ERR_UNSUPPORTED beyond 1024 colours or n > 32767.
 */
int mcb_greedy_wvcp_init(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                         const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, void *stream);
int mcb_greedy_wvcp_init_host(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                              const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, void *stream);
/*
 * First layer of the surrogate network on colour ids (mc/surrogate.py:146
 * with the one-hot encoding of :123-133 folded in).  Forward (backward = 0):
 * src = Lam [n, L], dst = z [B, k, L], z[b,i,:] = sum_{v: assigns[b,v]=i} Lam[v,:].
 * Backward (backward = 1): src = dz [B, k, L], dst = dLam [n, L],
 * dLam[v,:] = sum_b dz[b, assigns[b,v], :] (:209).  dtype_bytes 4 (float32)
 * or 8 (float64); device pointers; deterministic summation order.
 */
int mcb_segsum(int dtype_bytes, int backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
               int64_t k, int64_t L, void *dst, void *stream);
/* Same, without the colour-range check and its synchronising readback
 * (CUDA-graph capturable); ids must already be in [0, k). */
int mcb_segsum_async(int dtype_bytes, int backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
                     int64_t k, int64_t L, void *dst, void *stream);
/*
 * Inference path of the surrogate (eval mode, :137-178 with the one-hot
 * folded in).  mcb_colour_order: stable counting sort of each coloring's
 * vertices by colour -> order int32[B,n], offs int32[B,k+1].
 * mcb_segsum_sorted: z[b,i,:] = sum over colour-i vertices of Lam[v,:] in that
 * order; with A, C non-NULL the eval epilogue y = leaky(s A[col] + C[col],
 * slope) is applied (A, C: the folded batch norm + biases).
 * mcb_rowbias_affine_leaky: in place z[b,i,:] = leaky((z[b,i,:] + r[b,:]) A + C).
 * dtype_bytes 4 or 8; device pointers.
 */
int mcb_colour_order(const int32_t *assigns, int64_t B, int64_t n, int64_t k, int32_t *order, int32_t *offs,
                     void *stream);
int mcb_segsum_sorted(int dtype_bytes, const void *lam, const int32_t *order, const int32_t *offs, int64_t B,
                      int64_t n, int64_t k, int64_t L, const void *A, const void *C, double slope, void *z,
                      void *stream);
int mcb_rowbias_affine_leaky(int dtype_bytes, void *z, const void *r, const void *A, const void *C, double slope,
                             int64_t B, int64_t k, int64_t L, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MEMCOLOR_B200_H */
