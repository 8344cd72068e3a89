// population.cu -- the population update and parent matching of the memetic
// loop on the GPU.
//
//   update_population  <- mc/population.py:59-127
//   match_parents      <- mc/population.py:130-141
//
// update_population merges p incumbents and q newcomers (candidate ids
// 0..p-1, p..p+q-1), ranks them by (fitness, origin, index) -- a stable sort
// of the fitness in candidate-id order (:72-75) -- and admits candidates in
// that order when their distance to every admitted one exceeds ms (:93-98);
// if fewer than p pass, the rejected ones fill the remaining slots in rank
// order (:99-103).  The reference loop is sequential in the rank; here one
// persistent CTA keeps a "blocked" bit per candidate: admitting candidate c
// blocks, in one parallel pass over c's distance row, every candidate within
// ms of it, and the next admitted candidate is simply the next unblocked one
// in rank order.  Same admissions, same order; O(p) steps of O(p) parallel
// work instead of O(p^2) serial distance checks per step.
//
// match_parents: K nearest neighbours of every individual by (distance,
// index) (:137-140).  One warp per row: a distance histogram gives the K-th
// smallest distance d*; one pass in index order then keeps the rows below d*
// and the first rows at d*, and places each at its (distance, index) rank
// (counting-sort offsets from the histogram + match_any ranks), i.e. exactly
// np.lexsort((idx, dist)) order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "launch.h"

namespace mcb {

namespace {

// distance between candidates i, j (ids: 0..p-1 incumbents, p.. newcomers),
// mc/population.py:77-85
struct CandDist {
    const int32_t *pdist;   // p x p
    const int32_t *cross;   // p x q
    const int32_t *crossT;  // q x p
    const int32_t *within;  // q x q
    int64_t p, q;
    __device__ __forceinline__ int32_t operator()(int64_t i, int64_t j) const {
        if (i < p && j < p) return pdist[i * p + j];
        if (i < p) return cross[i * q + (j - p)];
        if (j < p) return crossT[(i - p) * p + j];
        return within[(i - p) * q + (j - p)];
    }
};

__global__ void transpose_i32(const int32_t *in, int64_t rows, int64_t cols, int32_t *out) {
    __shared__ int32_t tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t r = r0 + dy, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        const int64_t c = c0 + dy, r = r0 + threadIdx.x;  // out[c][r]
        if (c < cols && r < rows) out[c * rows + r] = tile[threadIdx.x][dy];
    }
}

__global__ void iota_i32(int32_t *x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = (int32_t)i;
}

// One CTA: the greedy admission in rank order (mc/population.py:90-103).
// out_adm[slot] = candidate id, out_rule[slot] = admitted by the spacing rule.
constexpr int UP_NT = 1024;
__global__ void __launch_bounds__(UP_NT, 1)
    greedy_admit_kernel(CandDist D, const int32_t *order, int64_t ms, int32_t *out_adm, uint8_t *out_rule,
                        uint32_t *gblocked, int use_smem_bits) {
    extern __shared__ uint32_t sbits[];
    __shared__ int s_found;
    const int64_t p = D.p, tot = D.p + D.q;
    const int nw = (int)((tot + 31) / 32);
    uint32_t *blocked = use_smem_bits ? sbits : gblocked;
    for (int i = threadIdx.x; i < nw; i += UP_NT) blocked[i] = 0u;
    __syncthreads();
    int64_t pos = 0, cnt = 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int s_wmin[UP_NT / 32];
    while (cnt < p && pos < tot) {
        // next unblocked candidate in rank order, from pos
        int64_t f = -1;
        for (int64_t base = pos; base < tot && f < 0; base += UP_NT) {
            const int64_t i = base + threadIdx.x;
            bool ok = false;
            if (i < tot) {
                const int c = order[i];
                ok = ((blocked[c >> 5] >> (c & 31)) & 1u) == 0u;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            if (lane == 0) s_wmin[wid] = bal ? (wid * 32 + __ffs(bal) - 1) : INT_MAX;
            __syncthreads();
            if (threadIdx.x < 32) {
                int m = s_wmin[threadIdx.x];
                for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
                if (threadIdx.x == 0) s_found = m;
            }
            __syncthreads();
            if (s_found != INT_MAX) f = base + s_found;
            __syncthreads();
        }
        if (f < 0) {  // every remaining candidate is within ms of an admitted one
            pos = tot;
            break;
        }
        const int c = order[f];
        if (threadIdx.x == 0) {
            out_adm[cnt] = c;
            out_rule[cnt] = 1;
        }
        cnt++;
        pos = f + 1;
        if (cnt == p) break;
        // block every candidate within ms of c (its own bit included)
        for (int64_t j = threadIdx.x; j < tot; j += UP_NT) {
            if (j == c || D(c, j) <= ms) atomicOr(&blocked[j >> 5], 1u << (j & 31));
        }
        __syncthreads();
    }
    // fallback fill: the rejected candidates (examined, not admitted) in rank order
    if (cnt < p) {
        // candidates examined = rank positions [0, pos); admitted ones are those with
        // no blocked bit when examined -- recover them from out_adm (few) by a mark
        __syncthreads();
        // mark admitted ids in a fresh bitmap region after the blocked bits
        uint32_t *adm_bits = blocked + nw;
        for (int i = threadIdx.x; i < nw; i += UP_NT) adm_bits[i] = 0u;
        __syncthreads();
        for (int64_t s = threadIdx.x; s < cnt; s += UP_NT) {
            const int c = out_adm[s];
            atomicOr(&adm_bits[c >> 5], 1u << (c & 31));
        }
        __syncthreads();
        int64_t fill = cnt;
        for (int64_t base = 0; base < pos && fill < p; base += UP_NT) {
            const int64_t i = base + threadIdx.x;
            bool rej = false;
            int c = 0;
            if (i < pos) {
                c = order[i];
                rej = ((adm_bits[c >> 5] >> (c & 31)) & 1u) == 0u;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, rej);
            if (lane == 0) s_wmin[wid] = __popc(bal);
            __syncthreads();
            int off = 0, total = 0;
            for (int w = 0; w < UP_NT / 32; w++) {
                const int x = s_wmin[w];
                off += (w < wid) ? x : 0;
                total += x;
            }
            if (rej) {
                const int64_t slot = fill + off + __popc(bal & ((1u << lane) - 1u));
                if (slot < p) {
                    out_adm[slot] = c;
                    out_rule[slot] = 0;
                }
            }
            fill += total;
            __syncthreads();
        }
    }
}

// new_dist[a][b] = dist(adm[a], adm[b]) (mc/population.py:113-118)
__global__ void gather_dist_kernel(CandDist D, const int32_t *adm, int64_t p, int32_t *out) {
    const int64_t a = blockIdx.y;
    const int ia = adm[a];
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < p; b += (int64_t)gridDim.x * blockDim.x)
        out[a * p + b] = (a == b) ? 0 : D(ia, adm[b]);
}

// new assigns / fitness (mc/population.py:106-112)
__global__ void gather_rows_kernel(const int32_t *adm, int64_t p, int64_t n, const int32_t *pop_assigns,
                                   const int32_t *new_assigns, const int64_t *fit_pop, const int64_t *fit_new,
                                   int32_t *out_assigns, int64_t *out_fit) {
    const int64_t s = blockIdx.x;
    const int64_t c = adm[s];
    const int32_t *src = c < p ? pop_assigns + c * n : new_assigns + (c - p) * n;
    for (int64_t v = threadIdx.x; v < n; v += blockDim.x) out_assigns[s * n + v] = src[v];
    if (threadIdx.x == 0) out_fit[s] = c < p ? fit_pop[c] : fit_new[c - p];
}

// ---------------------------------------------------------------------------
// match_parents: one warp per row, distance histogram in shared memory
// ---------------------------------------------------------------------------
constexpr int MP_WARPS = 4;
__global__ void __launch_bounds__(32 * MP_WARPS)
    match_parents_kernel(const int32_t *dist, int64_t p, int K, int nb, int64_t *matches, int *err) {
    extern __shared__ int32_t sh[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t *hist = sh + (size_t)wid * 2 * nb;  // [0, nb): counts, [nb, 2nb): running ranks
    int32_t *run = hist + nb;
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t i = blockIdx.x * (int64_t)MP_WARPS + wid; i < p; i += (int64_t)gridDim.x * MP_WARPS) {
        const int32_t *row = dist + i * p;
        for (int b = lane; b < nb; b += 32) {
            hist[b] = 0;
            run[b] = 0;
        }
        __syncwarp();
        for (int64_t j = lane; j < p; j += 32) {
            if (j == i) continue;
            const int d = row[j];
            if (d < 0 || d >= nb) {
                atomicExch(err, 1);
                continue;
            }
            atomicAdd(&hist[d], 1);
        }
        __syncwarp();
        // d* = smallest d with #(dist <= d) >= K; lanes own contiguous bin chunks
        const int per = (nb + 31) / 32, b0 = lane * per, b1 = min(nb, b0 + per);
        int mine = 0;
        for (int b = b0; b < b1; b++) mine += hist[b];
        int incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned hb = __ballot_sync(0xffffffffu, incl >= K);
        const int src = __ffs(hb) - 1;
        int dstar = 0, below = 0;
        if (lane == src) {
            int cum = incl - mine;
            int b = b0;
            while (cum + hist[b] < K) cum += hist[b++];
            dstar = b;
            below = cum;
        }
        dstar = __shfl_sync(0xffffffffu, dstar, src);
        below = __shfl_sync(0xffffffffu, below, src);  // #(dist < d*)
        const int need_eq = K - below;
        // counting-sort offsets: rank of distance d among the kept = #(kept < d)
        // = prefix of hist below d (d <= d*); hist[] becomes the offsets in place
        {
            int run_off = 0;
            for (int c0 = 0; c0 <= dstar; c0 += 32) {
                const int b = c0 + lane;
                const int h = (b <= dstar) ? hist[b] : 0;
                int inc = h;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                if (b <= dstar) hist[b] = run_off + inc - h;
                run_off += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
        __syncwarp();
        // one pass in index order: keep d < d* and the first need_eq rows at d*
        int eq_seen = 0;
        for (int64_t j0 = 0; j0 < p; j0 += 32) {
            const int64_t j = j0 + lane;
            int d = INT_MAX;
            if (j < p && j != i) d = row[j];
            bool keep = d < dstar;
            const bool at = d == dstar;
            const unsigned ab = __ballot_sync(0xffffffffu, at);
            if (at) keep = eq_seen + __popc(ab & lt) < need_eq;
            eq_seen += __popc(ab);
            const unsigned grp = __match_any_sync(0xffffffffu, keep ? d : -1);
            if (keep) {
                const int r = __popc(grp & lt);
                const int slot = hist[d] + run[d] + r;
                matches[i * (int64_t)K + slot] = j;
            }
            __syncwarp();
            if (keep && (grp & lt) == 0u) run[d] += __popc(grp);  // group leader
            __syncwarp();
        }
        __syncwarp();
    }
}

}  // namespace

int update_population_run(const int32_t *pdist, const int32_t *cross, const int32_t *within,
                          const int64_t *fit_pop, const int64_t *fit_new, int64_t p, int64_t q, int64_t ms,
                          const int32_t *pop_assigns, const int32_t *new_assigns, int64_t n,
                          int32_t *out_adm, uint8_t *out_rule, int32_t *out_dist, int32_t *out_assigns,
                          int64_t *out_fit, cudaStream_t st) {
    if (p < 1 || q < 0 || (int64_t)(p + q) >= (int64_t)INT32_MAX)
        return set_error(MCB_ERR_VALUE, "update_population: bad sizes p=%lld q=%lld", (long long)p, (long long)q);
    const int64_t tot = p + q;
    // scratch: fitness keys + ids (in, out), sort temp, crossT, blocked bits
    size_t sort_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)tot, 0, 64, st);
    auto a256 = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t o_kin = 0, o_kout = o_kin + a256(8 * tot), o_vin = o_kout + a256(8 * tot),
                 o_vout = o_vin + a256(4 * tot), o_tmp = o_vout + a256(4 * tot), o_ct = o_tmp + a256(sort_tmp),
                 o_bits = o_ct + a256(4 * (size_t)p * q), o_end = o_bits + a256(8 * ((tot + 31) / 32) + 16);
    uint8_t *ws = (uint8_t *)workspace2(o_end);
    if (!ws) return set_error(MCB_ERR_CUDA, "update_population: workspace allocation failed");
    int64_t *kin = (int64_t *)(ws + o_kin), *kout = (int64_t *)(ws + o_kout);
    int32_t *vin = (int32_t *)(ws + o_vin), *vout = (int32_t *)(ws + o_vout);
    int32_t *crossT = (int32_t *)(ws + o_ct);
    uint32_t *gbits = (uint32_t *)(ws + o_bits);
    if (cudaMemcpyAsync(kin, fit_pop, 8 * p, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        (q && cudaMemcpyAsync(kin + p, fit_new, 8 * q, cudaMemcpyDeviceToDevice, st) != cudaSuccess))
        return set_error(MCB_ERR_CUDA, "update_population: copy failed");
    iota_i32<<<std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, 4 * num_sms())), 256, 0, st>>>(vin, tot);
    // rank order: stable by fitness; ties keep candidate-id order = (origin, index)
    if (cub::DeviceRadixSort::SortPairs(ws + o_tmp, sort_tmp, kin, kout, vin, vout, (int)tot, 0, 64, st) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "update_population: sort failed");
    if (q) {
        dim3 tb(32, 8), tg((unsigned)((q + 31) / 32), (unsigned)((p + 31) / 32));
        transpose_i32<<<tg, tb, 0, st>>>(cross, p, q, crossT);
    }
    CandDist D{pdist, cross, crossT, within, p, q};
    const size_t bits_bytes = 8 * (size_t)((tot + 31) / 32);  // blocked + admitted marks
    const int use_smem = bits_bytes <= (size_t)max_smem_optin() - 2048;
    const size_t smem = use_smem ? bits_bytes : 0;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(greedy_admit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return set_error(MCB_ERR_CUDA, "update_population: smem attribute failed");
    greedy_admit_kernel<<<1, UP_NT, smem, st>>>(D, vout, ms, out_adm, out_rule, gbits, use_smem);
    if (out_dist) {
        dim3 g2((unsigned)std::min<int64_t>((p + 255) / 256, 64), (unsigned)p);
        gather_dist_kernel<<<g2, 256, 0, st>>>(D, out_adm, p, out_dist);
    }
    if (out_assigns && out_fit)
        gather_rows_kernel<<<(unsigned)p, 256, 0, st>>>(out_adm, p, n, pop_assigns, new_assigns, fit_pop, fit_new,
                                                        out_assigns, out_fit);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "update_population: launch failed");
    return MCB_OK;
}

int match_parents_run(const int32_t *dist, int64_t p, int64_t K, int64_t max_dist, int64_t *matches,
                      cudaStream_t st) {
    if (!(0 < K && K < p)) return set_error(MCB_ERR_VALUE, "need 0 < K < p");
    if (max_dist < 0 || max_dist > 65535) return set_error(MCB_ERR_UNSUPPORTED, "match_parents: distances <= 65535");
    const int nb = (int)max_dist + 1;
    const size_t smem = (size_t)MP_WARPS * 2 * nb * sizeof(int32_t);
    if (smem > (size_t)max_smem_optin()) return set_error(MCB_ERR_UNSUPPORTED, "match_parents: histogram too large");
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(match_parents_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return set_error(MCB_ERR_CUDA, "match_parents: smem attribute failed");
    int *err = (int *)workspace2(256);
    if (!err || cudaMemsetAsync(err, 0, sizeof(int), st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "match_parents: scratch failed");
    const int grid = (int)std::min<int64_t>((p + MP_WARPS - 1) / MP_WARPS, 8 * num_sms());
    match_parents_kernel<<<grid, 32 * MP_WARPS, smem, st>>>(dist, p, (int)K, nb, matches, err);
    int h = 0;
    if (cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "match_parents: kernel failed");
    if (h) return set_error(MCB_ERR_RANGE, "match_parents: distance outside [0, max_dist]");
    return MCB_OK;
}

}  // namespace mcb
