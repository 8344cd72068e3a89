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
//   * M lives in shared memory as u16 counters (one warp-private tile); the
//     first increment of a cell appends it to a compact list of the (<= n)
//     nonzero cells, so no pass ever scans the k^2 tile;
//   * entries >= 32 (at most n/32 of them, since they sum to <= n) are sorted
//     explicitly and taken first, in the reference order;
//   * every smaller value x = 31..1 is one "level": within a level the
//     reference visits cells in flat order, i.e. rows ascending and, inside a
//     row, columns ascending -- so a free row takes its lowest free column
//     holding x.  The level's cells are scattered into row -> column bitmasks
//     and one lane walks the free rows holding x with bit operations.
// Zero cells add nothing to the total, so they are never visited.
// The job space and the cross/within unranking are the reference's own
// (:94-113), so ranks shard it by contiguous [job_begin, job_end) ranges.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int PD_WARPS = 4;

// Per-warp shared tile: the k x k overlap histogram (u8 counters, or u16 when
// WIDE), the nonzero cells in first-touch order and bucketed by value, the
// per-level row -> column and column -> row bitmasks, the explicit list of
// entries >= 32 and the level counters.
struct PdLayout {
    size_t hist_words, list_words, big, cmask, uni, per;
};

__host__ __device__ inline PdLayout pd_layout(int n, int k, bool wide) {
    PdLayout L;
    const size_t kk = (size_t)k * k;
    L.hist_words = wide ? (kk + 1) / 2 : (kk + 3) / 4;
    L.list_words = ((size_t)n + 1) / 2;        // u16 (r << 8 | c) per cell
    L.big = (size_t)n / 32 + 2;
    L.cmask = (size_t)k * ((k + 31) / 32);
    // the first-touch list is dead once the cells are bucketed; the level
    // masks are live only after that: one region for both
    L.uni = L.list_words > 2 * L.cmask ? L.list_words : 2 * L.cmask;
    // hist + (list | cmask + rmask) + bucket + big + lvbeg[32] + lvcur[32] + rowused/colused[16] + bigcnt
    L.per = (L.hist_words + L.uni + L.list_words + L.big + 32 + 32 + 16 + 4) * 4;
    L.per = (L.per + 15) & ~(size_t)15;
    return L;
}

template <bool WIDE>
__device__ __forceinline__ uint32_t hist_get(const uint32_t *hist, int flat) {
    if (WIDE) return (hist[flat >> 1] >> (16 * (flat & 1))) & 0xFFFFu;
    return (hist[flat >> 2] >> (8 * (flat & 3))) & 0xFFu;
}

// colour ids -> u8 rows of NB (multiple of 16) bytes, range-checked once per
// colouring instead of once per pair
__global__ void pd_to_u8_kernel(const int32_t *__restrict__ src, int64_t rows, int n, int nb, int k,
                                uint8_t *__restrict__ dst, int32_t *err) {
    const int64_t words = rows * (nb / 4);
    int bad = 0;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = w / (nb / 4);
        const int v0 = (int)(w - row * (nb / 4)) * 4;
        uint32_t out = 0;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            if (v0 + b < n) {
                const int a = src[row * n + v0 + b];
                if (a < 0 || a >= k) bad = 1;
                out |= (uint32_t)(a & 0xFF) << (8 * b);
            }
        }
        reinterpret_cast<uint32_t *>(dst)[w] = out;
    }
    if (bad) atomicOr(err, 1);
}

template <int KWD, bool WIDE>
__global__ void __launch_bounds__(PD_WARPS * 32)
    pairwise_kernel(const uint8_t *__restrict__ pop, int64_t p, const uint8_t *__restrict__ off,
                    int64_t q, int n, int nb, int k, int32_t *__restrict__ cross,
                    int32_t *__restrict__ within, int64_t job_begin, int64_t job_end,
                    int16_t *__restrict__ jobs16, int32_t *err) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const PdLayout L = pd_layout(n, k, WIDE);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smem + warp * L.per);
    uint16_t *list = reinterpret_cast<uint16_t *>(hist + L.hist_words);  // shares with cmask / rmask
    uint32_t *cmask = hist + L.hist_words;  // [k][KWD]: row r -> columns holding the level
    uint32_t *rmask = cmask + L.cmask;      // [k][KWD]: column c -> rows holding the level
    uint16_t *bucket = reinterpret_cast<uint16_t *>(hist + L.hist_words + L.uni);
    uint32_t *big = reinterpret_cast<uint32_t *>(bucket + 2 * L.list_words);
    uint32_t *lvbeg = big + L.big;
    uint32_t *lvcur = lvbeg + 32;
    uint32_t *s_used = lvcur + 32;   // rowused[8], colused[8] (entries >= 32 only)
    uint32_t *bigcnt = s_used + 16;
    const uint32_t lt_mask = (1u << lane) - 1u;

    for (size_t i = lane; i < L.hist_words; i += 32) hist[i] = 0u;
    __syncwarp();

    const int64_t pq = p * q;
    for (int64_t job = job_begin + (int64_t)blockIdx.x * nwarps + warp; job < job_end;
         job += (int64_t)gridDim.x * nwarps) {
        const uint8_t *x, *y;
        int64_t oi, oj;
        bool is_cross = job < pq;
        if (is_cross) {
            oi = job / q;
            oj = job % q;
            x = pop + (size_t)oi * nb;
            y = off + (size_t)oj * nb;
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
            x = off + (size_t)oi * nb;
            y = off + (size_t)oj * nb;
        }
        lvbeg[lane] = 0u;
        if (lane == 0) *bigcnt = 0u;
        // overlap histogram (4 vertices per 32-bit load); the first touch of
        // a cell appends it to the list
        int bad = 0, m = 0;
        const int nw = (n + 3) >> 2;
        for (int w0 = 0; w0 < nw; w0 += 32) {
            const int w = w0 + lane;
            uint32_t xa = 0, yb = 0;
            if (w < nw) {
                xa = __ldg(reinterpret_cast<const uint32_t *>(x) + w);
                yb = __ldg(reinterpret_cast<const uint32_t *>(y) + w);
            }
#pragma unroll
            for (int b = 0; b < 4; b++) {
                bool first = false;
                const uint32_t a = (xa >> (8 * b)) & 0xFFu, c = (yb >> (8 * b)) & 0xFFu;
                if (4 * w + b < n) {
                    const int code = (int)a * k + (int)c;
                    const uint32_t sh = WIDE ? 16 * (code & 1) : 8 * (code & 3);
                    const uint32_t old = atomicAdd(&hist[WIDE ? code >> 1 : code >> 2], 1u << sh);
                    const uint32_t was = (old >> sh) & (WIDE ? 0xFFFFu : 0xFFu);
                    first = was == 0u;
                    if (!WIDE && was == 0xFFu) bad |= 2;  // u8 counter overflow
                }
                const uint32_t bm = __ballot_sync(0xffffffffu, first);
                if (first) list[m + __popc(bm & lt_mask)] = (uint16_t)((a << 8) | c);
                m += __popc(bm);
            }
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (bad) {
            if (lane == 0) atomicOr(err, bad);
            __syncwarp();
            for (size_t i = lane; i < L.hist_words; i += 32) hist[i] = 0u;
            __syncwarp();
            continue;
        }
        __syncwarp();
        // values: count each level; entries >= 32 go to the explicit list
        uint32_t levels = 0;
        for (int i = lane; i < m; i += 32) {
            const uint32_t e = list[i];
            const int flat = (int)(e >> 8) * k + (int)(e & 0xFFu);
            const uint32_t val = hist_get<WIDE>(hist, flat);
            if (val >= 32) {
                levels |= 1u;
                const uint32_t slot = atomicAdd(bigcnt, 1u);
                big[slot] = (val << 16) | (uint32_t)(0xFFFF - flat);
            } else {
                levels |= 1u << val;
                atomicAdd(&lvbeg[val], 1u);
            }
        }
        levels = __reduce_or_sync(0xffffffffu, levels);
        __syncwarp();
        {   // bucket offsets: exclusive prefix over the 32 level counts
            const uint32_t c = lvbeg[lane];
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            lvbeg[lane] = inc - c;
            lvcur[lane] = inc - c;
        }
        __syncwarp();
        for (int i = lane; i < m; i += 32) {
            const uint32_t e = list[i];
            const uint32_t val = hist_get<WIDE>(hist, (int)(e >> 8) * k + (int)(e & 0xFFu));
            if (val < 32) bucket[atomicAdd(&lvcur[val], 1u)] = (uint16_t)e;
        }
        // the list is dead: its region becomes the (zeroed) level masks
        __syncwarp();
        for (size_t i = lane; i < 2 * L.cmask; i += 32) cmask[i] = 0u;
        __syncwarp();
        uint32_t rowused[KWD], colused[KWD];
#pragma unroll
        for (int w = 0; w < KWD; w++) rowused[w] = colused[w] = 0u;
        long long total = 0;
        int matched = 0;
        // big entries first: sort keys descending (value desc, flat asc)
        if (levels & 1u) {
            if (lane < 16) s_used[lane] = 0u;
            __syncwarp();
            if (lane == 0) {
                const int nb = (int)*bigcnt;
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
                    if (((s_used[r >> 5] >> (r & 31)) & 1u) || ((s_used[8 + (c >> 5)] >> (c & 31)) & 1u))
                        continue;
                    s_used[r >> 5] |= 1u << (r & 31);
                    s_used[8 + (c >> 5)] |= 1u << (c & 31);
                    total += t >> 16;
                    matched++;
                }
            }
            total = __shfl_sync(0xffffffffu, total, 0);
            matched = __shfl_sync(0xffffffffu, matched, 0);
            __syncwarp();
#pragma unroll
            for (int w = 0; w < KWD; w++) {
                rowused[w] = s_used[w];
                colused[w] = s_used[8 + w];
            }
        }
        __syncwarp();
        // levels 31..1.  Within a level the reference visits cells in flat
        // order (rows ascending, then columns ascending).  That greedy equals
        // repeated rounds in which every free row r whose lowest free column c
        // (at this level) has r as its lowest free row takes (r, c): such a
        // cell precedes every other live cell in its row and column, so the
        // ordered greedy takes it too, and removing it leaves the rest of the
        // greedy unchanged.  Rows are lanes (r = lane + 32 j).
        uint32_t lv = levels & ~1u;
        while (lv && matched < k) {
            const int xval = 31 - __clz(lv);
            lv &= ~(1u << xval);
            const int beg = (int)lvbeg[xval], end = (int)lvcur[xval];
            for (int i = beg + lane; i < end; i += 32) {
                const uint32_t e = bucket[i];
                const int r = (int)(e >> 8), c = (int)(e & 0xFFu);
                atomicOr(&cmask[r * KWD + (c >> 5)], 1u << (c & 31));
                atomicOr(&rmask[c * KWD + (r >> 5)], 1u << (r & 31));
            }
            __syncwarp();
            while (true) {
                bool act = false;
                int col[KWD];
#pragma unroll
                for (int j = 0; j < KWD; j++) {
                    col[j] = -1;
                    const int r = lane + 32 * j;
                    if (r < k && !((rowused[j] >> lane) & 1u)) {
                        int c = -1;
#pragma unroll
                        for (int w = KWD - 1; w >= 0; w--) {
                            const uint32_t av = cmask[r * KWD + w] & ~colused[w];
                            if (av) c = 32 * w + __ffs(av) - 1;
                        }
                        if (c >= 0) {
                            act = true;
                            int r2 = -1;
#pragma unroll
                            for (int w = KWD - 1; w >= 0; w--) {
                                const uint32_t fr = rmask[c * KWD + w] & ~rowused[w];
                                if (fr) r2 = 32 * w + __ffs(fr) - 1;
                            }
                            if (r2 == r) col[j] = c;
                        }
                    }
                }
                if (!__any_sync(0xffffffffu, act)) break;
                int took = 0;
#pragma unroll
                for (int j = 0; j < KWD; j++) {
                    const uint32_t tb = __ballot_sync(0xffffffffu, col[j] >= 0);
                    rowused[j] |= tb;
                    took += __popc(tb);
                }
#pragma unroll
                for (int w = 0; w < KWD; w++) {
                    uint32_t mine = 0;
#pragma unroll
                    for (int j = 0; j < KWD; j++)
                        if (col[j] >= 0 && (col[j] >> 5) == w) mine |= 1u << (col[j] & 31);
                    colused[w] |= __reduce_or_sync(0xffffffffu, mine);
                }
                total += (long long)xval * took;
                matched += took;
                if (matched >= k) break;
            }
            for (int i = beg + lane; i < end; i += 32) {
                const uint32_t e = bucket[i];
                const int r = (int)(e >> 8), c = (int)(e & 0xFFu);
                cmask[r * KWD + (c >> 5)] = 0u;
                rmask[c * KWD + (r >> 5)] = 0u;
            }
            __syncwarp();
        }
        const int d = n - (int)total;
        if (lane == 0) {
            if (jobs16) {
                jobs16[job - job_begin] = (int16_t)d;  // compact job-range output (sharding)
            } else if (is_cross) {
                cross[oi * q + oj] = d;
            } else {
                within[oi * q + oj] = d;
                within[oj * q + oi] = d;
            }
        }
        // reset the warp's histogram for the next pair: only its nonzero cells,
        // i.e. the level buckets and the entries >= 32
        const int nbk = (int)lvcur[31], nbig = (int)*bigcnt;
        for (int i = lane; i < nbk; i += 32) {
            const uint32_t e = bucket[i];
            const int flat = (int)(e >> 8) * k + (int)(e & 0xFFu);
            hist[WIDE ? flat >> 1 : flat >> 2] = 0u;
        }
        for (int i = lane; i < nbig; i += 32) {
            const int flat = 0xFFFF - (int)(big[i] & 0xFFFFu);
            hist[WIDE ? flat >> 1 : flat >> 2] = 0u;
        }
        __syncwarp();
    }
}

namespace {

using PdKernel = void (*)(const uint8_t *, int64_t, const uint8_t *, int64_t, int, int, int, int32_t *,
                          int32_t *, int64_t, int64_t, int16_t *, int32_t *);

template <bool WIDE>
PdKernel pd_pick(int kwd) {
    switch (kwd) {
        case 1: return pairwise_kernel<1, WIDE>;
        case 2: return pairwise_kernel<2, WIDE>;
        case 3: return pairwise_kernel<3, WIDE>;
        case 4: return pairwise_kernel<4, WIDE>;
        case 5: return pairwise_kernel<5, WIDE>;
        case 6: return pairwise_kernel<6, WIDE>;
        case 7: return pairwise_kernel<7, WIDE>;
        default: return pairwise_kernel<8, WIDE>;
    }
}

}  // namespace

int pairwise_run(const int32_t *pop, int64_t p, const int32_t *off, int64_t q, int64_t n, int64_t k,
                 int32_t *cross, int32_t *within, int64_t job_begin, int64_t job_end,
                 uint32_t flags, cudaStream_t st, int16_t *jobs16) {
    if (p < 0 || q < 0 || n < 0 || k < 0) return set_error(MCB_ERR_VALUE, "pairwise: bad shape");
    const int64_t total = p * q + q * (q - 1) / 2;
    if (job_end < 0 || job_end > total) job_end = total;
    if (job_begin < 0) job_begin = 0;
    if (job_begin >= job_end || n == 0) return MCB_OK;
    if (k < 1) return set_error(MCB_ERR_VALUE, "pairwise: k must be >= 1");
    if (k > 255 || n > 65535) return set_error(MCB_ERR_UNSUPPORTED, "pairwise: k<=255, n<=65535");
    // u8 copies of both populations (rows padded to 16 bytes) after the flag word
    const int nb = (int)((n + 15) & ~(int64_t)15);
    uint8_t *ws = (uint8_t *)workspace(256 + (size_t)(p + q) * nb);
    if (!ws) return set_error(MCB_ERR_CUDA, "pairwise: workspace");
    int32_t *err = (int32_t *)ws;
    uint8_t *pop8 = ws + 256, *off8 = pop8 + (size_t)p * nb;
    cudaMemsetAsync(err, 0, 4, st);
    for (int side = 0; side < 2; side++) {
        const int64_t rows = side ? q : p;
        if (rows == 0) continue;
        const int64_t words = rows * (nb / 4);
        const int g = (int)std::min<int64_t>((words + 255) / 256, (int64_t)num_sms() * 8);
        pd_to_u8_kernel<<<g, 256, 0, st>>>(side ? off : pop, rows, (int)n, nb, (int)k, side ? off8 : pop8, err);
    }
    // u8 counters first; a launch in which some class overlap reached 256
    // (possible only when n >= 256) is re-run with u16 counters
    for (int wide = 0; wide < 2; wide++) {
        const PdLayout L = pd_layout((int)n, (int)k, wide);
        // warps per block: as many of PD_WARPS as shared memory holds
        int warps = PD_WARPS;
        while (warps > 1 && (size_t)warps * L.per > (size_t)max_smem_optin()) warps >>= 1;
        const size_t smem = warps * L.per;
        if (smem > (size_t)max_smem_optin())
            return set_error(MCB_ERR_UNSUPPORTED, "pairwise: k too large for shared memory");
        const PdKernel kern = wide ? pd_pick<true>((int)(k + 31) / 32) : pd_pick<false>((int)(k + 31) / 32);
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "pairwise: smem attribute failed");
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
        per_sm = std::max(per_sm, 1);
        const int64_t jobs = job_end - job_begin;
        const int grid = (int)std::min<int64_t>((jobs + warps - 1) / warps, (int64_t)per_sm * num_sms());
        kern<<<grid, warps * 32, smem, st>>>(pop8, p, off8, q, (int)n, nb, (int)k, cross, within, job_begin,
                                             job_end, jobs16, err);
        int32_t herr = 0;
        if (cudaGetLastError() != cudaSuccess ||
            cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "pairwise kernel failed: %s",
                             cudaGetErrorString(cudaGetLastError()));
        if (herr & 1) return set_error(MCB_ERR_RANGE, "pairwise: color id out of range [0, k)");
        if (!(herr & 2)) break;
        cudaMemsetAsync(err, 0, 4, st);
    }
    (void)flags;
    return MCB_OK;
}

// the whole job space's results (int16, job order: cross row-major, then the
// within pairs i < j) -> the cross matrix and the symmetric within matrix
__global__ void pd_scatter_kernel(const int16_t *__restrict__ jobs, int64_t p, int64_t q, int32_t *__restrict__ cross,
                                  int32_t *__restrict__ within) {
    const int64_t pq = p * q;
    const int64_t total = pq + q * (q - 1) / 2;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
        const int d = jobs[j];
        if (j < pq) {
            cross[j] = d;
        } else {
            // row i of the upper triangle holds q-1-i pairs (distance.py:106-112)
            const int64_t r = j - pq;
            const double b = 2.0 * (double)q - 1.0;
            int64_t i = (int64_t)floor((b - sqrt(fmax(b * b - 8.0 * (double)r, 0.0))) / 2.0);
            i = max((int64_t)0, min(i, q - 2));
            auto S = [&](int64_t t) { return t * (2 * q - t - 1) / 2; };
            while (i > 0 && S(i) > r) i--;
            while (i + 1 <= q - 2 && S(i + 1) <= r) i++;
            const int64_t jj = i + 1 + (r - S(i));
            within[i * q + jj] = d;
            within[jj * q + i] = d;
        }
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q; i += (int64_t)gridDim.x * blockDim.x)
        within[i * q + i] = 0;
}

int pairwise_scatter_run(const int16_t *jobs, int64_t p, int64_t q, int32_t *cross, int32_t *within,
                         cudaStream_t st) {
    if (p < 0 || q < 0) return set_error(MCB_ERR_VALUE, "pairwise_scatter: bad shape");
    const int64_t total = p * q + q * (q - 1) / 2;
    if (total == 0 && q == 0) return MCB_OK;
    const int grid = (int)std::min<int64_t>((std::max<int64_t>(total, q) + 255) / 256, 8 * (int64_t)num_sms());
    pd_scatter_kernel<<<std::max(grid, 1), 256, 0, st>>>(jobs, p, q, cross, within);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "pairwise_scatter launch failed");
    return MCB_OK;
}

}  // namespace mcb
