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
//     holding x.  A level's cells are row -> column / column -> row bitmasks,
//     resolved by parallel rounds (pd_level_rounds).  Level 1 -- most nonzero
//     cells of unrelated colourings -- needs no list or bucket: only the
//     cells reaching 2 (<= n / 2) are listed and bucketed into levels 2..31,
//     and level 1, when the matching reaches it, takes its masks from one pass
//     over the pair's vertices (the vertex of a cell holding exactly 1).
// Zero cells add nothing to the total, so they are never visited.
// The job space and the cross/within unranking are the reference's own
// (:94-113), so ranks shard it by contiguous [job_begin, job_end) ranges.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int PD_WARPS = 8;
#ifndef PD_FAST
#define PD_FAST 1  // levels of <= 32 cells with distinct free rows / columns taken in one step
#endif

// Per-warp shared tile: the k x k overlap histogram (u8 counters, or u16 when
// WIDE); the cells reaching 2 in a compact list, later bucketed by value; the
// row -> column / column -> row masks of one level at a time; the explicit
// list of entries >= 32 and the level counters.
struct PdLayout {
    size_t hist_words, mlist_words, big, cmask, uni, per;
};

__host__ __device__ inline PdLayout pd_layout(int n, int k, bool wide) {
    PdLayout L;
    const size_t kk = (size_t)k * k;
    L.hist_words = ((wide ? (kk + 1) / 2 : (kk + 3) / 4) + 3) & ~(size_t)3;  // uint4-clearable
    L.cmask = (size_t)k * ((k + 31) / 32);
    L.mlist_words = ((size_t)n / 2 + 2) / 2;  // u16 (r << 8 | c) per cell >= 2 (<= n / 2 cells)
    L.big = (size_t)n / 32 + 2;
    // the multi-cell list is dead once its cells are bucketed; the level masks
    // are live only after that: one region for both
    L.uni = L.mlist_words > 2 * L.cmask ? L.mlist_words : 2 * L.cmask;
    // hist + (mlist | cmask + rmask) + bucket + big + lvbeg[32] + lvcur[32] + rowused/colused[16] + counters
    L.per = (L.hist_words + L.uni + L.mlist_words + L.big + 32 + 32 + 16 + 4) * 4;
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

// One level of the greedy over its row -> column (cm) and column -> row (rm)
// masks.  The reference visits a level's cells in flat order (rows ascending,
// then columns ascending): a free row takes its lowest free column.  That
// greedy equals repeated rounds in which every free row r whose lowest free
// column c has r as its lowest free row takes (r, c): such a cell precedes
// every other live cell in its row and column, so the ordered greedy takes it
// too, and removing it leaves the rest unchanged.  Rows are lanes
// (r = lane + 32 j).
template <int KWD>
__device__ __forceinline__ void pd_level_rounds(const uint32_t *cm, const uint32_t *rm, int k, int lane, int xval,
                                                uint32_t (&rowused)[KWD], uint32_t (&colused)[KWD],
                                                long long &total, int &matched, int &bad) {
    // every round takes the smallest live cell at least, so <= k rounds; more
    // means inconsistent masks (reported, never an endless loop).  A row's
    // column words do not change during the level: in registers for k <= 128
    constexpr bool CACHE = KWD <= 4;
    uint32_t cmr[CACHE ? KWD : 1][CACHE ? KWD : 1];
    if constexpr (CACHE) {
#pragma unroll
        for (int j = 0; j < KWD; j++) {
            const int r = lane + 32 * j;
#pragma unroll
            for (int w = 0; w < KWD; w++) cmr[j][w] = r < k ? cm[r * KWD + w] : 0u;
        }
    }
    for (int round = 0;; round++) {
        if (round > k) {
            bad |= 4;
            break;
        }
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
                    const uint32_t av = (CACHE ? cmr[CACHE ? j : 0][CACHE ? w : 0] : cm[r * KWD + w]) & ~colused[w];
                    if (av) c = 32 * w + __ffs(av) - 1;
                }
                if (c >= 0) {
                    act = true;
                    int r2 = -1;
#pragma unroll
                    for (int w = KWD - 1; w >= 0; w--) {
                        const uint32_t fr = rm[c * KWD + w] & ~rowused[w];
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
    uint16_t *mlist = reinterpret_cast<uint16_t *>(hist + L.hist_words);  // shares with cmask / rmask
    uint32_t *cmask = hist + L.hist_words;  // [k][KWD]: row r -> columns holding the level
    uint32_t *rmask = cmask + L.cmask;      // [k][KWD]: column c -> rows holding the level
    uint16_t *bucket = reinterpret_cast<uint16_t *>(hist + L.hist_words + L.uni);
    uint32_t *big = reinterpret_cast<uint32_t *>(bucket + 2 * L.mlist_words);
    uint32_t *lvbeg = big + L.big;
    uint32_t *lvcur = lvbeg + 32;
    uint32_t *s_used = lvcur + 32;   // rowused[8], colused[8] (entries >= 32 only)
    uint32_t *bigcnt = s_used + 16;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // clearing the histogram: whole tile (uint4) when it is small, else the
    // words the pair's vertices touched
    const bool bulk_clear = L.hist_words <= 4 * (size_t)n;

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
        // overlap histogram (4 vertices per 32-bit load): the second increment
        // of a cell appends it to the multi-vertex list
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
                bool second = false;
                const uint32_t a = (xa >> (8 * b)) & 0xFFu, c = (yb >> (8 * b)) & 0xFFu;
                if (4 * w + b < n) {
                    const int code = (int)a * k + (int)c;
                    const uint32_t sh = WIDE ? 16 * (code & 1) : 8 * (code & 3);
                    const uint32_t old = atomicAdd(&hist[WIDE ? code >> 1 : code >> 2], 1u << sh);
                    const uint32_t was = (old >> sh) & (WIDE ? 0xFFFFu : 0xFFu);
                    second = was == 1u;
                    if (!WIDE && was == 0xFFu) bad |= 2;  // u8 counter overflow
                }
                const uint32_t bm = __ballot_sync(0xffffffffu, second);
                if (second) mlist[m + __popc(bm & lt_mask)] = (uint16_t)((a << 8) | c);
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
        // multi-vertex cells: count each level; entries >= 32 go to the
        // explicit list
        uint32_t levels = 0;
        for (int i = lane; i < m; i += 32) {
            const uint32_t e = mlist[i];
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
        if (levels & ~3u) {
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
                const uint32_t e = mlist[i];
                const uint32_t val = hist_get<WIDE>(hist, (int)(e >> 8) * k + (int)(e & 0xFFu));
                if (val < 32) bucket[atomicAdd(&lvcur[val], 1u)] = (uint16_t)e;
            }
            // the multi list is dead: its region becomes the (zeroed) level masks
            __syncwarp();
            for (size_t i = lane; i < 2 * L.cmask; i += 32) cmask[i] = 0u;
        }
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
                const int nbg = (int)*bigcnt;
                for (int a = 1; a < nbg; a++) {
                    const uint32_t t = big[a];
                    int b = a - 1;
                    while (b >= 0 && big[b] < t) {
                        big[b + 1] = big[b];
                        b--;
                    }
                    big[b + 1] = t;
                }
                for (int a = 0; a < nbg && matched < k; a++) {
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
        // levels 31..2 from their buckets (each level's masks cleared after
        // it, so the region stays zero), then level 1
        uint32_t lv = levels & ~3u;
        while (lv && matched < k) {
            const int xval = 31 - __clz(lv);
            lv &= ~(1u << xval);
            const int beg = (int)lvbeg[xval], end = (int)lvcur[xval];
            bool fast = false;
            if (PD_FAST && end - beg <= 32) {
                // few cells (related colourings: the level's large cells):
                // when its free cells have pairwise distinct rows and columns,
                // the ordered greedy takes every one of them
                int r = -1, c = -1;
                if (beg + lane < end) {
                    const uint32_t e = bucket[beg + lane];
                    const int rr = (int)(e >> 8), cc = (int)(e & 0xFFu);
                    bool fr = false, fc = false;
#pragma unroll
                    for (int w = 0; w < KWD; w++) {
                        if ((rr >> 5) == w) fr = !((rowused[w] >> (rr & 31)) & 1u);
                        if ((cc >> 5) == w) fc = !((colused[w] >> (cc & 31)) & 1u);
                    }
                    if (fr && fc) {
                        r = rr;
                        c = cc;
                    }
                }
                const int nlive = __popc(__ballot_sync(0xffffffffu, r >= 0));
                uint32_t rb[KWD], cb[KWD];
                int nr = 0, nc = 0;
#pragma unroll
                for (int w = 0; w < KWD; w++) {
                    rb[w] = __reduce_or_sync(0xffffffffu, (r >= 0 && (r >> 5) == w) ? 1u << (r & 31) : 0u);
                    cb[w] = __reduce_or_sync(0xffffffffu, (c >= 0 && (c >> 5) == w) ? 1u << (c & 31) : 0u);
                    nr += __popc(rb[w]);
                    nc += __popc(cb[w]);
                }
                if (nr == nlive && nc == nlive) {
#pragma unroll
                    for (int w = 0; w < KWD; w++) {
                        rowused[w] |= rb[w];
                        colused[w] |= cb[w];
                    }
                    total += (long long)xval * nlive;
                    matched += nlive;
                    fast = true;
                }
            }
            if (!fast) {
                for (int i = beg + lane; i < end; i += 32) {
                    const uint32_t e = bucket[i];
                    const int r = (int)(e >> 8), c = (int)(e & 0xFFu);
                    atomicOr(&cmask[r * KWD + (c >> 5)], 1u << (c & 31));
                    atomicOr(&rmask[c * KWD + (r >> 5)], 1u << (r & 31));
                }
                __syncwarp();
                pd_level_rounds<KWD>(cmask, rmask, k, lane, xval, rowused, colused, total, matched, bad);
                for (int i = beg + lane; i < end; i += 32) {
                    const uint32_t e = bucket[i];
                    const int r = (int)(e >> 8), c = (int)(e & 0xFFu);
                    cmask[r * KWD + (c >> 5)] = 0u;
                    rmask[c * KWD + (r >> 5)] = 0u;
                }
            }
            __syncwarp();
        }
        if (matched < k) {
            // level 1, only when reached (pairs of related colourings are
            // matched by their large cells): a vertex whose cell holds exactly
            // 1 is that cell's only vertex, so one pass over the pair's
            // vertices sets the level's masks
            if (!(levels & ~3u)) {
                for (size_t i = lane; i < 2 * L.cmask; i += 32) cmask[i] = 0u;  // still holds the multi list
                __syncwarp();
            }
            for (int w = lane; w < nw; w += 32) {
                const uint32_t xa = __ldg(reinterpret_cast<const uint32_t *>(x) + w);
                const uint32_t yb = __ldg(reinterpret_cast<const uint32_t *>(y) + w);
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int r = (int)((xa >> (8 * b)) & 0xFFu), c = (int)((yb >> (8 * b)) & 0xFFu);
                    if (4 * w + b < n && hist_get<WIDE>(hist, r * k + c) == 1u) {
                        atomicOr(&cmask[r * KWD + (c >> 5)], 1u << (c & 31));
                        atomicOr(&rmask[c * KWD + (r >> 5)], 1u << (r & 31));
                    }
                }
            }
            __syncwarp();
            pd_level_rounds<KWD>(cmask, rmask, k, lane, 1, rowused, colused, total, matched, bad);
        }
        if (bad && lane == 0) atomicOr(err, bad);
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
        // reset the histogram for the next pair: whole, or through the pair's
        // vertices (the mask region is zeroed before its next use)
        __syncwarp();
        if (bulk_clear) {
            uint4 *h4 = reinterpret_cast<uint4 *>(hist);
            for (size_t i = lane; i < L.hist_words / 4; i += 32) h4[i] = make_uint4(0u, 0u, 0u, 0u);
        } else {
            for (int w = lane; w < nw; w += 32) {
                const uint32_t xa = __ldg(reinterpret_cast<const uint32_t *>(x) + w);
                const uint32_t yb = __ldg(reinterpret_cast<const uint32_t *>(y) + w);
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    if (4 * w + b < n) {
                        const int code = (int)((xa >> (8 * b)) & 0xFFu) * k + (int)((yb >> (8 * b)) & 0xFFu);
                        hist[WIDE ? code >> 1 : code >> 2] = 0u;
                    }
                }
            }
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
        const PdKernel kern = wide ? pd_pick<true>((int)(k + 31) / 32) : pd_pick<false>((int)(k + 31) / 32);
        // warps per block: the count (<= PD_WARPS) with the most warps resident
        // per SM (the per-block shared-memory reservation makes the best count
        // depend on the tile size)
        int warps = 0, per_sm = 0, dev = 0;
        cudaGetDevice(&dev);
        static thread_local struct { PdKernel kern; size_t per; int dev, warps, per_sm; } memo = {nullptr, 0, -1, 0, 0};
        if (memo.kern == kern && memo.per == L.per && memo.dev == dev) {
            warps = memo.warps;
            per_sm = memo.per_sm;
        }
        for (int w = warps ? PD_WARPS + 1 : 1; w <= PD_WARPS; w++) {
            const size_t sm_w = w * L.per;
            if (sm_w > (size_t)max_smem_optin()) break;
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_w) != cudaSuccess)
                return set_error(MCB_ERR_CUDA, "pairwise: smem attribute failed");
            int b = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, w * 32, sm_w);
            if (w * b >= warps * per_sm) {
                warps = w;
                per_sm = b;
            }
        }
        if (warps == 0) return set_error(MCB_ERR_UNSUPPORTED, "pairwise: k too large for shared memory");
        memo = {kern, L.per, dev, warps, per_sm};
        const size_t smem = warps * L.per;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "pairwise: smem attribute failed");
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
        if (herr & 4) return set_error(MCB_ERR_CUDA, "pairwise: internal error (greedy rounds did not converge)");
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
