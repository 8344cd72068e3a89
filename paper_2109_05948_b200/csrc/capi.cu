// capi.cu -- extern "C" entry points (include/memcolor_b200.h) and the
// host-side runtime shared by the kernel launchers: error state, device
// properties, grow-only scratch, and the host-pointer (`*_host`) variants
// that own the host<->device copies.
#include <chrono>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace mcb {

static thread_local char g_err[512] = "";
static std::mutex g_mu;  // serialises entry points (shared per-device scratch)

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

int num_sms() {
    static int cache[64] = {0};
    const int d = cur_dev();
    if (!cache[d]) cudaDeviceGetAttribute(&cache[d], cudaDevAttrMultiProcessorCount, d);
    return cache[d] > 0 ? cache[d] : 1;
}

int max_smem_optin() {
    static int cache[64] = {0};
    const int d = cur_dev();
    if (!cache[d]) cudaDeviceGetAttribute(&cache[d], cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return cache[d];
}

static void *grow_buffer(void **buf, size_t *cap, size_t bytes);

// MCB_FLAG_ASYNC calls key their scratch by stream (WsStreamKey), so calls
// on different streams may overlap on the device and a stream's calls can be
// captured into a CUDA graph (after one warm-up call has sized the buffers)
static thread_local bool t_ws_keyed = false;
static thread_local cudaStream_t t_ws_stream = nullptr;
WsStreamKey::WsStreamKey(cudaStream_t s) : prev_keyed(t_ws_keyed), prev_stream(t_ws_stream) {
    t_ws_keyed = true;
    t_ws_stream = s;
}
WsStreamKey::~WsStreamKey() {
    t_ws_keyed = prev_keyed;
    t_ws_stream = (cudaStream_t)prev_stream;
}
static void *keyed_workspace(int slot, size_t bytes) {
    static std::map<std::tuple<int, int, void *>, std::pair<void *, size_t>> bufs;
    auto &e = bufs[std::make_tuple(cur_dev(), slot, (void *)t_ws_stream)];
    return grow_buffer(&e.first, &e.second, bytes);
}

void *workspace(size_t bytes) {
    if (t_ws_keyed) return keyed_workspace(1, bytes);
    static void *buf[64] = {nullptr};
    static size_t cap[64] = {0};
    const int d = cur_dev();
    return grow_buffer(&buf[d], &cap[d], bytes);
}

// third: the device arena of the host-pointer entry points
void *workspace3(size_t bytes) {
    static void *buf[64] = {nullptr};
    static size_t cap[64] = {0};
    const int d = cur_dev();
    return grow_buffer(&buf[d], &cap[d], bytes);
}

// fourth: the group TabuCol kernel's adjacency bitset (alive while the
// warp/CTA fallbacks of the same call use workspace / workspace2)
void *workspace4(size_t bytes) {
    if (t_ws_keyed) return keyed_workspace(4, bytes);
    static void *buf[64] = {nullptr};
    static size_t cap[64] = {0};
    const int d = cur_dev();
    return grow_buffer(&buf[d], &cap[d], bytes);
}

// second independent scratch (kernels that need their own tables while the
// first holds control words of the same call)
void *workspace2(size_t bytes) {
    if (t_ws_keyed) return keyed_workspace(2, bytes);
    static void *buf[64] = {nullptr};
    static size_t cap[64] = {0};
    const int d = cur_dev();
    return grow_buffer(&buf[d], &cap[d], bytes);
}

static void *grow_buffer(void **bufp, size_t *capp, size_t bytes) {
    void *&b = *bufp;
    size_t &c = *capp;
    if (bytes <= c) return b;
    if (b) {
        cudaDeviceSynchronize();
        cudaFree(b);
        b = nullptr;
        c = 0;
    }
    size_t want = bytes + bytes / 4;
    if (cudaMalloc(&b, want) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    c = want;
    return b;
}

__global__ void stream_values_kernel(const uint64_t *keys, const uint64_t *ctrs, uint64_t *out,
                                     int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = stream_value(keys[i], ctrs[i]);
}

int stream_values_run(const uint64_t *keys, const uint64_t *ctrs, uint64_t *out, int64_t count,
                      cudaStream_t st) {
    if (count < 0) return set_error(MCB_ERR_VALUE, "count < 0");
    if (count == 0) return MCB_OK;
    int grid = (int)std::min<int64_t>((count + 255) / 256, 4 * num_sms());
    stream_values_kernel<<<grid, 256, 0, st>>>(keys, ctrs, out, count);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "stream_values kernel failed");
    return MCB_OK;
}

// Device arena for the host-pointer variants: one stream-ordered allocation.
struct Arena {
    struct Item {
        void *host;
        void **dev;
        size_t bytes;
        bool in, out;
    };
    std::vector<Item> items;
    uint8_t *base = nullptr;
    cudaStream_t st;
    explicit Arena(cudaStream_t s) : st(s) {}
    template <typename T>
    void add(T *host, T **dev, size_t count, bool in, bool out) {
        if (!host || count == 0) {
            *dev = nullptr;
            return;
        }
        items.push_back({(void *)host, (void **)dev, count * sizeof(T), in, out});
    }
    template <typename T>
    void add(const T *host, const T **dev, size_t count) {
        add(const_cast<T *>(host), const_cast<T **>(dev), count, true, false);
    }
    int upload() {
        size_t total = 0;
        for (auto &it : items) total += (it.bytes + 255) & ~(size_t)255;
        if (total == 0) return MCB_OK;
        // persistent grow-only buffer (entry points are serialised by g_mu): no
        // per-call pool allocation / release on the host path
        base = (uint8_t *)workspace3(total);
        if (!base) return set_error(MCB_ERR_CUDA, "host-path arena allocation (%zu) failed", total);
        size_t off = 0;
        for (auto &it : items) {
            *it.dev = base + off;
            if (it.in && cudaMemcpyAsync(*it.dev, it.host, it.bytes, cudaMemcpyHostToDevice, st) !=
                             cudaSuccess)
                return set_error(MCB_ERR_CUDA, "H2D copy failed");
            off += (it.bytes + 255) & ~(size_t)255;
        }
        return MCB_OK;
    }
    int download() {
        for (auto &it : items)
            if (it.out && cudaMemcpyAsync(it.host, *it.dev, it.bytes, cudaMemcpyDeviceToHost, st) !=
                              cudaSuccess)
                return set_error(MCB_ERR_CUDA, "D2H copy failed");
        if (cudaStreamSynchronize(st) != cudaSuccess) return set_error(MCB_ERR_CUDA, "sync failed");
        return MCB_OK;
    }
    ~Arena() {}
};

}  // namespace mcb

using namespace mcb;

extern "C" {

const char *mcb_version(void) { return "memcolor-b200 0.1.0 (sm_100a)"; }
const char *mcb_last_error(void) { return g_err; }

int mcb_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

int mcb_stream_values(const uint64_t *keys, const uint64_t *ctrs, uint64_t *out, int64_t count,
                      void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return stream_values_run(keys, ctrs, out, count, (cudaStream_t)stream);
}

int mcb_tabucol_batch(int32_t *assigns, int64_t p, int64_t n, int64_t k, const int64_t *adj_indptr,
                      const int32_t *adj_indices, const int32_t *edges_u, const int32_t *edges_v,
                      int64_t m, int64_t depth, const uint64_t *keys, int32_t *best_assigns,
                      int64_t *best_conflicts, int64_t *end_conflicts, int64_t *iters_used,
                      int64_t *diag, int64_t log_cap, int32_t *log_v, int64_t *log_iter,
                      int64_t *log_tt, int64_t *log_cnt, int64_t *counters, uint32_t flags,
                      void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (log_cap > 0 && (!log_v || !log_iter || !log_tt))
        return set_error(MCB_ERR_VALUE, "log_cap > 0 requires log arrays");
    TabucolArgs a{assigns, p, n, k, adj_indptr, adj_indices, edges_u, edges_v, m, depth, keys,
                  best_assigns, best_conflicts, end_conflicts, iters_used, diag,
                  log_cap > 0 ? log_cap : 0, log_v, log_iter, log_tt, log_cnt, counters, flags};
    return tabucol_run(a, (cudaStream_t)stream);
}

int mcb_tabucol_batch_host(int32_t *assigns, int64_t p, int64_t n, int64_t k,
                           const int64_t *adj_indptr, const int32_t *adj_indices,
                           const int32_t *edges_u, const int32_t *edges_v, int64_t m, int64_t depth,
                           const uint64_t *keys, int32_t *best_assigns, int64_t *best_conflicts,
                           int64_t *end_conflicts, int64_t *iters_used, int64_t *diag,
                           int64_t log_cap, int32_t *log_v, int64_t *log_iter, int64_t *log_tt,
                           int64_t *log_cnt, int64_t *counters, uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 0 || n < 1) return set_error(MCB_ERR_VALUE, "bad shape");
    const size_t pn = (size_t)p * n, pc = (size_t)p * (log_cap > 0 ? log_cap : 0);
    Arena ar(st);
    TabucolArgs a{};
    ar.add(assigns, &a.assigns, pn, true, true);
    ar.add(adj_indptr, &a.indptr, (size_t)n + 1);
    ar.add(adj_indices, &a.indices, (size_t)adj_indptr[n]);
    ar.add(edges_u, &a.eu, (size_t)m);
    ar.add(edges_v, &a.ev, (size_t)m);
    ar.add(keys, &a.keys, (size_t)p);
    ar.add(best_assigns, &a.best_assigns, pn, false, true);
    ar.add(best_conflicts, &a.best_conflicts, (size_t)p, false, true);
    ar.add(end_conflicts, &a.end_conflicts, (size_t)p, false, true);
    ar.add(iters_used, &a.iters_used, (size_t)p, false, true);
    ar.add(diag, &a.diag, (size_t)p, true, true);
    // the kernels write only the first log_cnt[i] entries of a row: the rest
    // keeps the caller's content (as the numba kernel leaves it), so upload too
    ar.add(log_v, &a.log_v, pc, true, true);
    ar.add(log_iter, &a.log_iter, pc, true, true);
    ar.add(log_tt, &a.log_tt, pc, true, true);
    ar.add(log_cnt, &a.log_cnt, (size_t)p, false, true);
    ar.add(counters, &a.counters, 2 * (size_t)p, false, true);
    const bool timing = getenv("MCB_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    int rc = ar.upload();
    if (rc) return rc;
    a.p = p;
    a.n = n;
    a.k = k;
    a.m = m;
    a.depth = depth;
    a.log_cap = (log_cap > 0 && a.log_v) ? log_cap : 0;
    a.flags = flags;
    if (timing) cudaStreamSynchronize(st);
    const auto t1 = now();
    rc = tabucol_run(a, st);
    if (rc) return rc;
    const auto t2 = now();
    rc = ar.download();
    if (timing) {
        const auto t3 = now();
        auto ms = [](auto x, auto y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
        fprintf(stderr, "[mcb] tabucol_host: upload %.1f ms, run %.1f ms, download %.1f ms\n", ms(t0, t1),
                ms(t1, t2), ms(t2, t3));
    }
    return rc;
}

int mcb_wvcp_batch(int32_t *assigns, int64_t p, int64_t n, int64_t k, const int64_t *adj_indptr,
                   const int32_t *adj_indices, const int32_t *edges_u, const int32_t *edges_v,
                   int64_t m, const int32_t *wranks, const int64_t *wvals, int64_t nranks,
                   const int64_t *weights, int64_t depth, int64_t rounds, int32_t schedule_on,
                   const double *phi0s, double forced_phi, int64_t tt_base, const uint64_t *keys,
                   int32_t *best_assigns, int64_t *best_scores, int64_t *end_scores,
                   int64_t *end_conflicts, double *phi_used, int64_t *diag, int64_t log_cap,
                   int32_t *log_v, int64_t *log_iter, int64_t *log_tt, int8_t *log_asp,
                   int64_t *log_cnt, uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (log_cap > 0 && (!log_v || !log_iter || !log_tt || !log_asp))
        return set_error(MCB_ERR_VALUE, "log_cap > 0 requires log arrays");
    WvcpArgs a{assigns, p, n, k, adj_indptr, adj_indices, edges_u, edges_v, m, wranks, wvals,
               nranks, weights, depth, rounds, schedule_on, phi0s, forced_phi, tt_base, keys,
               best_assigns, best_scores, end_scores, end_conflicts, phi_used, diag,
               log_cap > 0 ? log_cap : 0, log_v, log_iter, log_tt, log_asp, log_cnt, flags};
    return wvcp_run(a, (cudaStream_t)stream);
}

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
                        void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 0 || n < 1 || rounds < 0) return set_error(MCB_ERR_VALUE, "bad shape");
    const size_t pn = (size_t)p * n, pc = (size_t)p * (log_cap > 0 ? log_cap : 0);
    Arena ar(st);
    WvcpArgs a{};
    ar.add(assigns, &a.assigns, pn, true, true);
    ar.add(adj_indptr, &a.indptr, (size_t)n + 1);
    ar.add(adj_indices, &a.indices, (size_t)adj_indptr[n]);
    ar.add(edges_u, &a.eu, (size_t)m);
    ar.add(edges_v, &a.ev, (size_t)m);
    ar.add(wranks, &a.wranks, (size_t)n);
    ar.add(wvals, &a.wvals, (size_t)nranks);
    ar.add(weights, &a.weights, (size_t)n);
    ar.add(phi0s, &a.phi0s, (size_t)p);
    ar.add(keys, &a.keys, (size_t)p);
    ar.add(best_assigns, &a.best_assigns, pn, true, true);
    ar.add(best_scores, &a.best_scores, (size_t)p, false, true);
    ar.add(end_scores, &a.end_scores, (size_t)p, false, true);
    ar.add(end_conflicts, &a.end_conflicts, (size_t)p, false, true);
    ar.add(phi_used, &a.phi_used, (size_t)p * (rounds + 1), true, true);
    ar.add(diag, &a.diag, (size_t)p, true, true);
    // the kernels write only the first log_cnt[i] entries of a row: the rest
    // keeps the caller's content (as the numba kernel leaves it), so upload too
    ar.add(log_v, &a.log_v, pc, true, true);
    ar.add(log_iter, &a.log_iter, pc, true, true);
    ar.add(log_tt, &a.log_tt, pc, true, true);
    ar.add(log_asp, &a.log_asp, pc, true, true);
    ar.add(log_cnt, &a.log_cnt, (size_t)p, false, true);
    int rc = ar.upload();
    if (rc) return rc;
    a.p = p;
    a.n = n;
    a.k = k;
    a.m = m;
    a.nranks = nranks;
    a.depth = depth;
    a.rounds = rounds;
    a.schedule_on = schedule_on;
    a.forced_phi = forced_phi;
    a.tt_base = tt_base;
    a.log_cap = (log_cap > 0 && a.log_v) ? log_cap : 0;
    a.flags = flags;
    rc = wvcp_run(a, st);
    if (rc) return rc;
    return ar.download();
}

int mcb_gpx_batch(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t K,
                  int64_t k, const uint64_t *keys, int32_t *out, uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return gpx_run(pop, p, n, matches, K, k, keys, out, flags, (cudaStream_t)stream);
}

int mcb_gpx_batch_host(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches,
                       int64_t K, int64_t k, const uint64_t *keys, int32_t *out, uint32_t flags,
                       void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 0 || n < 0 || K < 0) return set_error(MCB_ERR_VALUE, "bad shape");
    Arena ar(st);
    const int32_t *dpop;
    const int64_t *dmatch;
    const uint64_t *dkeys;
    int32_t *dout;
    ar.add(pop, &dpop, (size_t)p * n);
    ar.add(matches, &dmatch, (size_t)p * K);
    ar.add(keys, &dkeys, (size_t)p * K);
    ar.add(out, &dout, (size_t)p * K * n, false, true);
    int rc = ar.upload();
    if (rc) return rc;
    rc = gpx_run(dpop, p, n, dmatch, K, k, dkeys, dout, flags, st);
    if (rc) return rc;
    return ar.download();
}

int mcb_gpx_rows(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t rows,
                 int64_t row_off, int64_t K, int64_t k, const uint64_t *keys, int32_t *out,
                 uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return gpx_rows_run(pop, p, n, matches, rows, row_off, K, k, keys, out, flags, (cudaStream_t)stream);
}

int mcb_pairwise(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                 int64_t k, int32_t *cross, int32_t *within, int64_t job_begin, int64_t job_end,
                 uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return pairwise_run(pop, p, off, q, n, k, cross, within, job_begin, job_end, flags,
                        (cudaStream_t)stream);
}

int mcb_tabucol_async_status(void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return tabucol_async_status((cudaStream_t)stream);
}

int mcb_pairwise_jobs(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                      int64_t k, int16_t *jobs16, int64_t job_begin, int64_t job_end, uint32_t flags,
                      void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!jobs16) return set_error(MCB_ERR_VALUE, "pairwise_jobs: jobs16 is null");
    return pairwise_run(pop, p, off, q, n, k, nullptr, nullptr, job_begin, job_end, flags, (cudaStream_t)stream,
                        jobs16);
}

int mcb_pairwise_scatter(const int16_t *jobs16, int64_t p, int64_t q, int32_t *cross, int32_t *within,
                         void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return pairwise_scatter_run(jobs16, p, q, cross, within, (cudaStream_t)stream);
}

int mcb_pairwise_host(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n,
                      int64_t k, int32_t *cross, int32_t *within, int64_t job_begin,
                      int64_t job_end, uint32_t flags, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 0 || q < 0 || n < 0) return set_error(MCB_ERR_VALUE, "bad shape");
    Arena ar(st);
    const int32_t *dpop, *doff;
    int32_t *dcross, *dwithin;
    ar.add(pop, &dpop, (size_t)p * n);
    ar.add(off, &doff, (size_t)q * n);
    ar.add(cross, &dcross, (size_t)p * q, true, true);
    ar.add(within, &dwithin, (size_t)q * q, true, true);
    int rc = ar.upload();
    if (rc) return rc;
    rc = pairwise_run(dpop, p, doff, q, n, k, dcross, dwithin, job_begin, job_end, flags, st);
    if (rc) return rc;
    return ar.download();
}

}  // extern "C"

extern "C" {

int mcb_update_population(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                          const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q, int64_t ms,
                          const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                          int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                          int64_t *out_fit, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    const int rc = update_population_run(pdist, cross, within, fit_pop, fit_new, p, q, ms, pop_assigns,
                                         new_assigns, n, out_adm, out_rule, out_dist, out_assigns, out_fit,
                                         (cudaStream_t)stream);
    if (rc) return rc;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "update_population failed: %s", cudaGetErrorString(cudaGetLastError()));
    return MCB_OK;
}

int mcb_update_population_host(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                               const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q,
                               int64_t ms, const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                               int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                               int64_t *out_fit, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 1 || q < 0) return set_error(MCB_ERR_VALUE, "bad shape");
    Arena ar(st);
    const int32_t *dpd, *dcr, *dwi, *dpa, *dna;
    const int64_t *dfp, *dfn;
    int32_t *dadm, *ddist, *das;
    uint8_t *drule;
    int64_t *dfit;
    ar.add(pdist, &dpd, (size_t)p * p);
    ar.add(cross, &dcr, (size_t)p * q);
    ar.add(within, &dwi, (size_t)q * q);
    ar.add(fit_pop, &dfp, (size_t)p);
    ar.add(fit_new, &dfn, (size_t)q);
    ar.add(pop_assigns, &dpa, out_assigns ? (size_t)p * n : 0);
    ar.add(new_assigns, &dna, out_assigns ? (size_t)q * n : 0);
    ar.add(out_adm, &dadm, (size_t)p, false, true);
    ar.add(out_rule, &drule, (size_t)p, false, true);
    ar.add(out_dist, &ddist, (size_t)p * p, false, true);
    ar.add(out_assigns, &das, (size_t)p * n, false, true);
    ar.add(out_fit, &dfit, (size_t)p, false, true);
    int rc = ar.upload();
    if (rc) return rc;
    rc = update_population_run(dpd, dcr, dwi, dfp, dfn, p, q, ms, dpa, dna, n, dadm, drule, ddist,
                               out_assigns ? das : nullptr, out_assigns ? dfit : nullptr, st);
    if (rc) return rc;
    return ar.download();
}

int mcb_match_parents(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                      void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return match_parents_run(dist, p, K, max_dist, matches, (cudaStream_t)stream);
}

int mcb_match_parents_host(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                           void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (p < 1) return set_error(MCB_ERR_VALUE, "bad shape");
    Arena ar(st);
    const int32_t *dd;
    int64_t *dm;
    ar.add(dist, &dd, (size_t)p * p);
    ar.add(matches, &dm, (size_t)p * (K > 0 ? K : 0), false, true);
    int rc = ar.upload();
    if (rc) return rc;
    rc = match_parents_run(dd, p, K, max_dist, dm, st);
    if (rc) return rc;
    return ar.download();
}

int mcb_greedy_wvcp_init(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                         const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return greedy_init_run(order, indptr, indices, n, keys, p, assigns, used, (cudaStream_t)stream);
}

int mcb_greedy_wvcp_init_host(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                              const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 1 || p < 0) return set_error(MCB_ERR_VALUE, "bad shape");
    Arena ar(st);
    const int32_t *dord, *dind;
    const int64_t *dptr;
    const uint64_t *dkeys;
    int32_t *dasg, *dused;
    ar.add(order, &dord, (size_t)n);
    ar.add(indptr, &dptr, (size_t)n + 1);
    ar.add(indices, &dind, (size_t)std::max<int64_t>(indptr[n], 1));
    ar.add(keys, &dkeys, (size_t)p);
    ar.add(assigns, &dasg, (size_t)p * n, false, true);
    ar.add(used, &dused, (size_t)p, false, true);
    int rc = ar.upload();
    if (rc) return rc;
    rc = greedy_init_run(dord, dptr, dind, n, dkeys, p, dasg, dused, st);
    if (rc) return rc;
    return ar.download();
}

int mcb_segsum(int dtype_bytes, int backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
               int64_t k, int64_t L, void *dst, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return segsum_run(dtype_bytes, backward != 0, src, assigns, B, n, k, L, dst, (cudaStream_t)stream);
}

int mcb_segsum_async(int dtype_bytes, int backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
                     int64_t k, int64_t L, void *dst, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return segsum_run(dtype_bytes, backward != 0, src, assigns, B, n, k, L, dst, (cudaStream_t)stream, false);
}

int mcb_colour_order(const int32_t *assigns, int64_t B, int64_t n, int64_t k, int32_t *order, int32_t *offs,
                     void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return colour_order_run(assigns, B, n, k, order, offs, (cudaStream_t)stream);
}

int mcb_segsum_sorted(int dtype_bytes, const void *lam, const int32_t *order, const int32_t *offs, int64_t B,
                      int64_t n, int64_t k, int64_t L, const void *A, const void *C, double slope, void *z,
                      void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return segsum_sorted_run(dtype_bytes, lam, order, offs, B, n, k, L, A, C, slope, z, (cudaStream_t)stream);
}

int mcb_rowbias_affine_leaky(int dtype_bytes, void *z, const void *r, const void *A, const void *C, double slope,
                             int64_t B, int64_t k, int64_t L, void *stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    return rowbias_affine_leaky_run(dtype_bytes, z, r, A, C, slope, B, k, L, (cudaStream_t)stream);
}

}  // extern "C"
