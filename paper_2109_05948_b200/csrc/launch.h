// launch.h -- internal host-side interface between the C ABI (capi.cu) and
// the kernel launchers.  Not part of the public ABI (include/memcolor_b200.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace mcb {

int set_error(int code, const char *fmt, ...);
int num_sms();
int max_smem_optin();
// Grow-only per-device scratch buffer (stream-ordered users must be done with
// the previous contents; every entry point synchronises before returning).
void *workspace(size_t bytes);
void *workspace2(size_t bytes);
void *workspace3(size_t bytes);
void *workspace4(size_t bytes);
// scope in which workspace / workspace2 / workspace4 are per-stream buffers
struct WsStreamKey {
    explicit WsStreamKey(cudaStream_t s);
    ~WsStreamKey();
    bool prev_keyed;
    void *prev_stream;
};
// device-side error word of the last MCB_FLAG_ASYNC TabuCol call on a stream
int tabucol_async_status(cudaStream_t st);

struct TabucolArgs {
    int32_t *assigns;
    int64_t p, n, k;
    const int64_t *indptr;
    const int32_t *indices;
    const int32_t *eu, *ev;
    int64_t m, depth;
    const uint64_t *keys;
    int32_t *best_assigns;
    int64_t *best_conflicts, *end_conflicts, *iters_used, *diag;
    int64_t log_cap;
    int32_t *log_v;
    int64_t *log_iter, *log_tt, *log_cnt, *counters;
    uint32_t flags;
};
int tabucol_run(const TabucolArgs &a, cudaStream_t st);
// warp-per-individual kernel (tabucol_warp.cu); -1 = shape outside its envelope
// work_list/nwork: a subset of individuals (nullptr/-1: all); spill: the
// variant whose tabu ring continues in global memory (no 1024-entry limit)
int tabucol_warp_launch(const TabucolArgs &A, cudaStream_t st, int32_t *work_counter, int32_t *ovf_list,
                        int32_t *ovf_count, int32_t *err_flag, const int32_t *work_list = nullptr,
                        int64_t nwork = -1, bool spill = false, const int32_t *nwork_dev = nullptr);
// group-of-warps kernel (tabucol_group.cu); -1 = shape outside its envelope
int tabucol_group_launch(const TabucolArgs &A, cudaStream_t st, int32_t *work_counter, int32_t *ovf_list,
                         int32_t *ovf_count, int32_t *err_flag);
int tabucol_group_describe(int64_t n, int64_t k, int64_t p, char *buf, int len);
int tabucol_group_stats(unsigned long long *out);
int tabucol_phase_cycles(unsigned long long *out, int reset);
struct TabuParams;  // tc_shared.cuh
int tabucol_cta_describe(int64_t n, int64_t k, int64_t p, char *buf, int len);
size_t tabucol_cluster_smem(int n, int k);
int tabucol_cluster_phase_cycles(unsigned long long *out, int reset);
int tabucol_cluster_warp_stats(unsigned long long *out, int reset);
size_t tabucol_cluster_stamp_stride(int n, int k);
int tabucol_cluster_launch(const TabuParams &P, int max_clusters, cudaStream_t st, int *grid_out, bool query_only);
int tabucol_warp_stats(unsigned long long *out);

struct WvcpArgs {
    int32_t *assigns;
    int64_t p, n, k;
    const int64_t *indptr;
    const int32_t *indices;
    const int32_t *eu, *ev;
    int64_t m;
    const int32_t *wranks;
    const int64_t *wvals;
    int64_t nranks;
    const int64_t *weights;
    int64_t depth, rounds;
    int32_t schedule_on;
    const double *phi0s;
    double forced_phi;
    int64_t tt_base;
    const uint64_t *keys;
    int32_t *best_assigns;
    int64_t *best_scores, *end_scores, *end_conflicts;
    double *phi_used;
    int64_t *diag;
    int64_t log_cap;
    int32_t *log_v;
    int64_t *log_iter, *log_tt;
    int8_t *log_asp;
    int64_t *log_cnt;
    uint32_t flags;
};
int wvcp_run(const WvcpArgs &a, cudaStream_t st);

int gpx_run(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t K, int64_t k,
            const uint64_t *keys, int32_t *out, uint32_t flags, cudaStream_t st);
int gpx_rows_run(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t rows,
                 int64_t row_off, int64_t K, int64_t k, const uint64_t *keys, int32_t *out,
                 uint32_t flags, cudaStream_t st);
int pairwise_run(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n, int64_t k,
                 int32_t *cross, int32_t *within, int64_t job_begin, int64_t job_end,
                 uint32_t flags, cudaStream_t st, int16_t *jobs16 = nullptr);
int pairwise_scatter_run(const int16_t *jobs, int64_t p, int64_t q, int32_t *cross, int32_t *within,
                         cudaStream_t st);
int update_population_run(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                          const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q, int64_t ms,
                          const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                          int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                          int64_t *out_fit, cudaStream_t st);
int match_parents_run(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                      cudaStream_t st);
int greedy_init_run(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                    const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, cudaStream_t st);
int segsum_run(int dtype, bool backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
               int64_t k, int64_t L, void *dst, cudaStream_t st, bool checked = true);
int colour_order_run(const int32_t *assigns, int64_t B, int64_t n, int64_t k, int32_t *order, int32_t *offs,
                     cudaStream_t st);
int segsum_sorted_run(int dtype, const void *lam, const int32_t *order, const int32_t *offs, int64_t B, int64_t n,
                      int64_t k, int64_t L, const void *A, const void *C, double slope, void *z, cudaStream_t st);
int rowbias_affine_leaky_run(int dtype, void *z, const void *r, const void *A, const void *C, double slope,
                             int64_t B, int64_t k, int64_t L, cudaStream_t st);
int wvcp_stats(unsigned long long *out, int reset);
int stream_values_run(const uint64_t *keys, const uint64_t *ctrs, uint64_t *out, int64_t count,
                      cudaStream_t st);

}  // namespace mcb
