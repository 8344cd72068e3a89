// distance.cu -- approximate partition distance over the pairwise job space,
// one warp per pair (sm_100a).
//
// Replaces `_pairwise_kernel` + `_greedy_match_total` (reference
// pkg/src/memcolor/distance.py:40-72, 90-119).  The reference builds the k x k
// class-overlap matrix M, stable-argsorts -M (value desc, flat index r*k+c asc)
// and greedily takes entries whose row and column are still free, stopping at k
// matches; distance = n - total.
//
// Here the same greedy is evaluated without sorting k^2 cells:
//   * M lives in shared memory as u16 counters (one warp-private tile);
//   * entries >= 32 (at most n/32 of them, since they sum to <= n) are sorted
//     explicitly and taken first, in the reference order;
//   * every smaller value x = 31..1 is one "level": within a level the
//     reference visits cells in flat order, i.e. rows ascending and, inside a
//     row, columns ascending -- so a free row takes its lowest free column
//     holding x.  Per-row bitmasks of the values present let a level skip
//     rows without x, and a ballot over a row's columns finds that column.
// Zero cells add nothing to the total, so they are never visited.
// The job space and the cross/within unranking are the reference's own
// (:94-113), so ranks shard it by contiguous [job_begin, job_end) ranges.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int PD_WARPS = 4;

struct PdLayout {
    size_t hist_words, rowlev, used, big, per;
};

__host__ __device__ inline PdLayout pd_layout(int n, int k) {
    PdLayout L;
    L.hist_words = ((size_t)k * k + 1) / 2;
    L.rowlev = (size_t)k;
    L.used = 16;  // 8 row words + 8 column words (k <= 255)
    L.big = (size_t)n / 32 + 2;
    L.per = (L.hist_words + L.rowlev + L.used + L.big + 4) * 4;
    L.per = (L.per + 15) & ~(size_t)15;
    return L;
}

__global__ void __launch_bounds__(PD_WARPS * 32)
    pairwise_kernel(const int32_t *__restrict__ pop, int64_t p, const int32_t *__restrict__ off,
                    int64_t q, int n, int k, int32_t *__restrict__ cross,
                    int32_t *__restrict__ within, int64_t job_begin, int64_t job_end,
                    int32_t *err) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const PdLayout L = pd_layout(n, k);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem + warp * L.per);
    uint32_t *rowlev = hist + L.hist_words;
    uint32_t *rowused = rowlev + L.rowlev;
    uint32_t *colused = rowused + 8;
    uint32_t *big = colused + 8;
    uint32_t *bigcnt = big + L.big;
    const int kk = k * k;

    for (size_t i = lane; i < L.hist_words; i += 32) hist[i] = 0u;
    for (int r = lane; r < k; r += 32) rowlev[r] = 0u;
    if (lane < 16) rowused[lane] = 0u;
    if (lane == 0) *bigcnt = 0u;
    __syncwarp();

    const int64_t pq = p * q;
    for (int64_t job = job_begin + (int64_t)blockIdx.x * PD_WARPS + warp; job < job_end;
         job += (int64_t)gridDim.x * PD_WARPS) {
        const int32_t *x, *y;
        int64_t oi, oj;
        bool is_cross = job < pq;
        if (is_cross) {
            oi = job / q;
            oj = job % q;
            x = pop + (size_t)oi * n;
            y = off + (size_t)oj * n;
        } else {
            // unrank r into (i < j) with row i holding q-1-i pairs (:106-112)
            const int64_t r = job - pq;
            const double b = 2.0 * (double)q - 1.0;
            int64_t i = (int64_t)floor((b - sqrt(fmax(b * b - 8.0 * (double)r, 0.0))) / 2.0);
            i = max((int64_t)0, min(i, q - 2));
            auto S = [&](int64_t t) { return t * (2 * q - t - 1) / 2; };
            while (i > 0 && S(i) > r) i--;
            while (i + 1 <= q - 2 && S(i + 1) <= r) i++;
            oi = i;
            oj = i + 1 + (r - S(i));
            x = off + (size_t)oi * n;
            y = off + (size_t)oj * n;
        }
        // overlap histogram
        int bad = 0;
        for (int v = lane; v < n; v += 32) {
            const int a = x[v], b = y[v];
            if (a < 0 || a >= k || b < 0 || b >= k) {
                bad = 1;
                continue;
            }
            const int code = a * k + b;
            atomicAdd(&hist[code >> 1], 1u << (16 * (code & 1)));
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) atomicExch(err, 1);
            // clear and skip
            for (size_t i = lane; i < L.hist_words; i += 32) hist[i] = 0u;
            __syncwarp();
            continue;
        }
        __syncwarp();
        // per-row value-presence masks; entries >= 32 go to the explicit list
        uint32_t levels = 0;
        for (int r = 0; r < k; r++) {
            uint32_t m = 0;
            for (int c0 = 0; c0 < k; c0 += 32) {
                const int c = c0 + lane;
                if (c < k) {
                    const int flat = r * k + c;
                    const uint32_t val = (hist[flat >> 1] >> (16 * (flat & 1))) & 0xFFFFu;
                    if (val >= 32) {
                        m |= 1u;
                        const uint32_t slot = atomicAdd(bigcnt, 1u);
                        big[slot] = (val << 16) | (uint32_t)(0xFFFF - flat);
                    } else if (val) {
                        m |= 1u << val;
                    }
                }
            }
            m = __reduce_or_sync(0xffffffffu, m);
            if (lane == 0) rowlev[r] = m;
            levels |= m;
        }
        __syncwarp();
        long long total = 0;
        int matched = 0;
        // big entries first: sort keys descending (value desc, flat asc)
        if (levels & 1u) {
            const int nb = (int)*bigcnt;
            if (lane == 0) {
                for (int a = 1; a < nb; a++) {
                    const uint32_t t = big[a];
                    int b = a - 1;
                    while (b >= 0 && big[b] < t) {
                        big[b + 1] = big[b];
                        b--;
                    }
                    big[b + 1] = t;
                }
                for (int a = 0; a < nb && matched < k; a++) {
                    const uint32_t t = big[a];
                    const int flat = 0xFFFF - (int)(t & 0xFFFFu);
                    const int r = flat / k, c = flat % k;
                    if (((rowused[r >> 5] >> (r & 31)) & 1u) || ((colused[c >> 5] >> (c & 31)) & 1u))
                        continue;
                    rowused[r >> 5] |= 1u << (r & 31);
                    colused[c >> 5] |= 1u << (c & 31);
                    total += t >> 16;
                    matched++;
                }
            }
            total = __shfl_sync(0xffffffffu, total, 0);
            matched = __shfl_sync(0xffffffffu, matched, 0);
            __syncwarp();
        }
        // levels 31..1, rows ascending, lowest free column
        uint32_t lv = levels & ~1u;
        while (lv && matched < k) {
            const int xval = 31 - __clz(lv);
            lv &= ~(1u << xval);
            for (int r0 = 0; r0 < k && matched < k; r0 += 32) {
                const int r = r0 + lane;
                const bool has = r < k && ((rowlev[r] >> xval) & 1u) &&
                                 !((rowused[r >> 5] >> (r & 31)) & 1u);
                uint32_t rows = __ballot_sync(0xffffffffu, has);
                while (rows) {
                    const int rr = r0 + __ffs(rows) - 1;
                    rows &= rows - 1u;
                    int found = -1;
                    for (int c0 = 0; c0 < k && found < 0; c0 += 32) {
                        const int c = c0 + lane;
                        bool ok = false;
                        if (c < k) {
                            const int flat = rr * k + c;
                            const uint32_t val = (hist[flat >> 1] >> (16 * (flat & 1))) & 0xFFFFu;
                            ok = val == (uint32_t)xval && !((colused[c >> 5] >> (c & 31)) & 1u);
                        }
                        const uint32_t bm = __ballot_sync(0xffffffffu, ok);
                        if (bm) found = c0 + __ffs(bm) - 1;
                    }
                    if (found >= 0) {
                        if (lane == 0) {
                            rowused[rr >> 5] |= 1u << (rr & 31);
                            colused[found >> 5] |= 1u << (found & 31);
                        }
                        __syncwarp();
                        total += xval;
                        matched++;
                        if (matched >= k) break;
                    }
                }
            }
        }
        const int d = n - (int)total;
        if (lane == 0) {
            if (is_cross) {
                cross[oi * q + oj] = d;
            } else {
                within[oi * q + oj] = d;
                within[oj * q + oi] = d;
            }
        }
        // reset the warp's tile for the next pair
        __syncwarp();
        for (int v = lane; v < n; v += 32) {
            const int code = x[v] * k + y[v];
            hist[code >> 1] = 0u;
        }
        for (int r = lane; r < k; r += 32) rowlev[r] = 0u;
        if (lane < 16) rowused[lane] = 0u;
        if (lane == 0) *bigcnt = 0u;
        __syncwarp();
    }
}

int pairwise_run(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n, int64_t k,
                 int32_t *cross, int32_t *within, int64_t job_begin, int64_t job_end,
                 uint32_t flags, cudaStream_t st) {
    if (p < 0 || q < 0 || n < 0 || k < 0) return set_error(MCB_ERR_VALUE, "pairwise: bad shape");
    const int64_t total = p * q + q * (q - 1) / 2;
    if (job_end < 0 || job_end > total) job_end = total;
    if (job_begin < 0) job_begin = 0;
    if (job_begin >= job_end || n == 0) return MCB_OK;
    if (k < 1) return set_error(MCB_ERR_VALUE, "pairwise: k must be >= 1");
    if (k > 255 || n > 65535) return set_error(MCB_ERR_UNSUPPORTED, "pairwise: k<=255, n<=65535");
    const PdLayout L = pd_layout((int)n, (int)k);
    const size_t smem = PD_WARPS * L.per;
    if (smem > (size_t)max_smem_optin())
        return set_error(MCB_ERR_UNSUPPORTED, "pairwise: k too large for shared memory");
    if (cudaFuncSetAttribute(pairwise_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "pairwise: smem attribute failed");
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pairwise_kernel, PD_WARPS * 32, smem);
    nb = std::max(nb, 1);
    const int64_t jobs = job_end - job_begin;
    const int grid = (int)std::min<int64_t>((jobs + PD_WARPS - 1) / PD_WARPS, (int64_t)nb * num_sms());
    int32_t *err = (int32_t *)workspace(256);
    if (!err) return set_error(MCB_ERR_CUDA, "pairwise: workspace");
    cudaMemsetAsync(err, 0, 4, st);
    pairwise_kernel<<<grid, PD_WARPS * 32, smem, st>>>(pop, p, off, q, (int)n, (int)k, cross, within,
                                                       job_begin, job_end, err);
    int32_t herr = 0;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "pairwise kernel failed: %s",
                         cudaGetErrorString(cudaGetLastError()));
    if (herr) return set_error(MCB_ERR_RANGE, "pairwise: color id out of range [0, k)");
    (void)flags;
    return MCB_OK;
}

}  // namespace mcb
