// tabucol.cu -- batched TabuCol for sm_100a, one individual per CTA.
//
// Replaces the numba kernel `_tabucol_batch` (reference
// pkg/src/memcolor/localsearch.py:266-410).  Semantics reproduced exactly
// (validation mode, the default):
//   * scan order = conflict-list order x colours ascending (:328-334), the list
//     maintained by append / swap-remove over (CSR neighbours asc, then v)
//     (:368-385);
//   * tabu test `it < tabu[v,c]` with aspiration `conflicts + d < best` (:336-339);
//   * reservoir tie-break: the SplitMix64 counter advances once per candidate
//     that ties the running minimum (:340-350); tenure draw
//     `U{0..9} + (6*conflicts_after)//10` (:363-366), last-write-wins stamp;
//   * early exit at zero conflicts (:322), `it` counts no-move iterations (:398),
//     O(m) scratch check every 1024 iterations -> diag (:398-405).
//
// The sequential reservoir is evaluated in parallel and exactly:
//   pass 1  every row-group (RG lanes) evaluates one conflicting vertex's k-1
//           candidates from shared memory -> (row min, #candidates at the min);
//   pass 2  warp 0 runs an exclusive prefix-min over the row minima.  Each tie
//           event of the sequential scan is a candidate equal to the running
//           minimum; rows whose minimum is above the running minimum have none,
//           rows whose minimum equals it have exactly #min of them, and the few
//           rows that LOWER the running minimum are re-evaluated with an in-row
//           prefix-min scan.  That gives the total number of tie events, hence
//           the counter offset E of the final minimum group.
//   pass 3  the T-1 reservoir draws of the final group are independent
//           (counter ctr+E+s-2 for rank s); the winner is the LAST rank whose
//           draw is zero (warp max).
//   pass 4  locate the winning (v, c), apply tenure.
//   pass 5  all threads update gamma over N(v) and flag conflict-set events;
//   pass 6  one thread applies the (few) events in neighbour order.
//
// Data layout per individual (shared memory when it fits, else a per-CTA
// global slice that stays L2-resident):
//   gamma  int8 [n][kp]  (kp = k rounded up to 4)   -- int16 fallback on overflow
//   tabu   u16  [n][kp]  wrap-around stamps, swept every 16384 iterations
//                        -- u32 fallback when a tenure exceeds 16383
//   assign u8 [n], conflict list / positions u16 [n], per-row (min, count) [n].
// Individuals whose int8/u16 tables would overflow are re-run from their
// original start by the wide (int16 / u32) instantiation; results are
// identical by construction (same arithmetic, wider storage).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int TC_NT = 256;
constexpr int TC_EVCAP = 64;
constexpr int TC_BIG = 1 << 20;

struct TabuParams {
    int32_t *assigns;
    int32_t *best_assigns;
    const int64_t *indptr;
    const int32_t *indices;
    const int32_t *eu;
    const int32_t *ev;
    int64_t m;
    int n, k, kp;
    int64_t depth;
    const uint64_t *keys;
    int64_t *best_conflicts, *end_conflicts, *iters_used, *diag;
    int64_t log_cap;
    int32_t *log_v;
    int64_t *log_iter, *log_tt, *log_cnt;
    int64_t *counters;
    const int32_t *work;       // optional list of individual ids
    const int32_t *nwork_dev;  // optional device-side work count
    int nwork;
    int32_t *work_counter;
    int32_t *ovf_list, *ovf_count;  // individuals to redo wide
    int32_t *err_flag;
    uint8_t *ws_gamma, *ws_stamp;  // per-CTA global slices (global variants)
    size_t ws_g_stride, ws_s_stride;
    uint32_t flags;
    int rg, wpl, words;
};

struct TabuCtrl {
    long long it, conflicts, best, nlog, sum_c, sum_deg, diag;
    unsigned long long ctr;
    int C, work, mv_v, mv_a, mv_b, mv_gvb, has_move, nev, copy, ovf;
    long long red[TC_NT / 32];
    int wcnt[TC_NT / 32];
};

template <typename G>
struct RowInfoT;
template <>
struct RowInfoT<int8_t> {
    using T = uint16_t;
    static constexpr int NONE = 127;
    __device__ static T pack(int rm, int nq) {
        return (T)((uint8_t)(int8_t)(rm >= TC_BIG ? NONE : rm) | ((uint32_t)nq << 8));
    }
    __device__ static void unpack(T x, int &rm, int &nq) {
        rm = (int)(int8_t)(x & 0xFF);
        if (rm == NONE) rm = TC_BIG;
        nq = x >> 8;
    }
};
template <>
struct RowInfoT<int16_t> {
    using T = uint32_t;
    static constexpr int NONE = 32767;
    __device__ static T pack(int rm, int nq) {
        return (T)((uint16_t)(int16_t)(rm >= TC_BIG ? NONE : rm) | ((uint32_t)nq << 16));
    }
    __device__ static void unpack(T x, int &rm, int &nq) {
        rm = (int)(int16_t)(x & 0xFFFF);
        if (rm == NONE) rm = TC_BIG;
        nq = (int)(x >> 16);
    }
};

template <typename S>
__device__ __forceinline__ bool stamp_active(S st, uint32_t it) {
    if constexpr (sizeof(S) == 2)
        return (int16_t)(uint16_t)((uint16_t)st - (uint16_t)it) > 0;
    else
        return (int32_t)((uint32_t)st - it) > 0;
}

// Load the EPW stamps of gamma word w of a row.
template <typename S, int EPW>
__device__ __forceinline__ void load_stamps(const S *srow, int w, S (&st)[EPW]) {
    if constexpr (sizeof(S) * EPW == 8) {
        uint2 x = *reinterpret_cast<const uint2 *>(srow + w * EPW);
        uint32_t wd[2] = {x.x, x.y};
#pragma unroll
        for (int e = 0; e < EPW; e++) {
            if constexpr (sizeof(S) == 2)
                st[e] = (S)(wd[e >> 1] >> (16 * (e & 1)));
            else
                st[e] = (S)wd[e];
        }
    } else if constexpr (sizeof(S) * EPW == 16) {
        uint4 x = *reinterpret_cast<const uint4 *>(srow + w * EPW);
        uint32_t wd[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < EPW; e++) st[e] = (S)wd[e];
    } else {
        uint32_t x = *reinterpret_cast<const uint32_t *>(srow + w * EPW);
#pragma unroll
        for (int e = 0; e < EPW; e++) st[e] = (S)(x >> (16 * e));
    }
}

// Evaluate one lane's share of a row: dv[j*EPW+e] = delta of colour
// (lig + j*RG)*EPW + e if the move is admissible, else TC_BIG.
template <typename G, typename S, int MAXV>
__device__ __forceinline__ void eval_row(const G *gamma, const S *stamp, const uint8_t *assign, int v,
                                         int kp, int k, int lig, int RG, int WPL, int W,
                                         uint32_t it, int thr, int (&dv)[MAXV]) {
    constexpr int EPW = 4 / (int)sizeof(G);
    const int a = assign[v];
    const G *grow = gamma + (size_t)v * kp;
    const S *srow = stamp + (size_t)v * kp;
    const int gva = grow[a];
#pragma unroll
    for (int j = 0; j < MAXV / EPW; j++) {
        const int w = lig + j * RG;
        if (j < WPL && w < W) {
            const uint32_t gw = reinterpret_cast<const uint32_t *>(grow)[w];
            S st[EPW];
            load_stamps<S, EPW>(srow, w, st);
#pragma unroll
            for (int e = 0; e < EPW; e++) {
                const int c = w * EPW + e;
                int gv;
                if constexpr (sizeof(G) == 1)
                    gv = (int)(int8_t)(gw >> (8 * e));
                else
                    gv = (int)(int16_t)(gw >> (16 * e));
                const int d = gv - gva;
                const bool tabu = stamp_active<S>(st[e], it);
                const bool adm = (c < k) && (c != a) && (!tabu || d < thr);
                dv[j * EPW + e] = adm ? d : TC_BIG;
            }
        } else {
#pragma unroll
            for (int e = 0; e < EPW; e++) dv[j * EPW + e] = TC_BIG;
        }
    }
}

// Number of sequential tie events inside a row when the scan enters it with
// running minimum R (group-cooperative, RG lanes, colour order (j, lig, e)).
template <int EPW, int MAXV>
__device__ __forceinline__ int row_ties(const int (&dv)[MAXV], int R, int lig, int RG, int WPL) {
    int running = R, ties = 0;
#pragma unroll
    for (int j = 0; j < MAXV / EPW; j++) {
        if (j < WPL) {
            int lmin = TC_BIG;
#pragma unroll
            for (int e = 0; e < EPW; e++) lmin = min(lmin, dv[j * EPW + e]);
            const int incl = warp_incl_min(lmin, lig, RG);
            int excl = __shfl_up_sync(0xffffffffu, incl, 1, RG);
            if (lig == 0) excl = TC_BIG;
            int cur = min(running, excl);
            int cnt = 0;
#pragma unroll
            for (int e = 0; e < EPW; e++) {
                const int x = dv[j * EPW + e];
                if (x != TC_BIG) {
                    if (x < cur) cur = x;
                    else if (x == cur) cnt++;
                }
            }
            ties += warp_sum(cnt, RG);
            running = min(running, __shfl_sync(0xffffffffu, incl, RG - 1, RG));
        }
    }
    return ties;
}

template <typename G, typename S, bool GSM, bool SSM>
__global__ void __launch_bounds__(TC_NT) tabucol_kernel(TabuParams P) {
    constexpr int NT = TC_NT;
    constexpr int NW = NT / 32;
    constexpr int EPW = 4 / (int)sizeof(G);
    constexpr int MAXV = 8;
    constexpr int GMAX = sizeof(G) == 1 ? 127 : 32767;
    constexpr uint32_t SWEEP = sizeof(S) == 2 ? 16384u : (1u << 30);
    using RI = RowInfoT<G>;
    using RowT = typename RI::T;

    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ TabuCtrl ctl;

    const int n = P.n, k = P.k, kp = P.kp;
    size_t off = 0;
    G *gamma;
    S *stamp;
    if constexpr (GSM) {
        gamma = reinterpret_cast<G *>(smem + off);
        off += ((size_t)n * kp * sizeof(G) + 15) & ~(size_t)15;
    } else {
        gamma = reinterpret_cast<G *>(P.ws_gamma + blockIdx.x * P.ws_g_stride);
    }
    if constexpr (SSM) {
        stamp = reinterpret_cast<S *>(smem + off);
        off += ((size_t)n * kp * sizeof(S) + 15) & ~(size_t)15;
    } else {
        stamp = reinterpret_cast<S *>(P.ws_stamp + blockIdx.x * P.ws_s_stride);
    }
    uint8_t *assign = smem + off;
    off += (n + 15) & ~15;
    uint16_t *clist = reinterpret_cast<uint16_t *>(smem + off);
    off += (2 * n + 15) & ~15;
    uint16_t *cpos = reinterpret_cast<uint16_t *>(smem + off);
    off += (2 * n + 15) & ~15;
    RowT *rinfo = reinterpret_cast<RowT *>(smem + off);
    off += (sizeof(RowT) * n + 15) & ~15;
    uint32_t *evl = reinterpret_cast<uint32_t *>(smem + off);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int RG = P.rg, WPL = P.wpl, W = P.words;
    const int lig = lane & (RG - 1);
    const int gpw = 32 / RG;  // groups per warp
    const int gig = lane / RG;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const size_t tab_elems = (size_t)n * kp;

    for (;;) {
        if (tid == 0) ctl.work = atomicAdd(P.work_counter, 1);
        __syncthreads();
        const int wi = ctl.work;
        const int nwork = P.nwork_dev ? *P.nwork_dev : P.nwork;
        if (wi >= nwork) break;
        const int ind = P.work ? P.work[wi] : wi;
        const uint64_t key = P.keys[ind];
        int32_t *a_io = P.assigns + (size_t)ind * n;
        int32_t *b_out = P.best_assigns + (size_t)ind * n;

        // ---------------- init (localsearch.py:289-318) ----------------
        for (int v = tid; v < n; v += NT) {
            int c = a_io[v];
            if (c < 0 || c >= k) {
                atomicExch(P.err_flag, 1);
                c = 0;
            }
            assign[v] = (uint8_t)c;
        }
        {
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gamma);
            const size_t gw = tab_elems * sizeof(G) / 4;
            for (size_t i = tid; i < gw; i += NT) g32[i] = 0u;
            uint32_t *s32 = reinterpret_cast<uint32_t *>(stamp);
            const size_t sw = tab_elems * sizeof(S) / 4;
            for (size_t i = tid; i < sw; i += NT) s32[i] = 0u;
        }
        if (tid == 0) {
            ctl.ovf = 0;
            ctl.diag = 0;
        }
        __syncthreads();
        // gamma[u][c] = #neighbours of u coloured c; each thread owns its rows
        {
            int bad = 0;
            for (int u = tid; u < n; u += NT) {
                G *row = gamma + (size_t)u * kp;
                const int64_t s0 = P.indptr[u], s1 = P.indptr[u + 1];
                for (int64_t idx = s0; idx < s1; idx++) {
                    const int c = assign[P.indices[idx]];
                    const int x = (int)row[c] + 1;
                    if (x > GMAX) bad = 1;
                    else row[c] = (G)x;
                }
            }
            if (bad) ctl.ovf = 1;
        }
        __syncthreads();
        // conflicts and the ascending conflict list (:298-310)
        {
            long long c2 = 0;
            int base = 0;
            for (int ch = 0; ch < n; ch += NT) {
                const int v = ch + tid;
                bool f = false;
                if (v < n) {
                    const int g = gamma[(size_t)v * kp + assign[v]];
                    f = g > 0;
                    c2 += g;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, f);
                if (lane == 0) ctl.wcnt[warp] = __popc(bal);
                __syncthreads();
                int woff = 0, tot = 0;
#pragma unroll
                for (int j = 0; j < NW; j++) {
                    const int cj = ctl.wcnt[j];
                    woff += (j < warp) ? cj : 0;
                    tot += cj;
                }
                if (v < n) {
                    if (f) {
                        const int pos = base + woff + __popc(bal & ((1u << lane) - 1u));
                        clist[pos] = (uint16_t)v;
                        cpos[v] = (uint16_t)pos;
                    } else {
                        cpos[v] = 0xFFFF;
                    }
                }
                base += tot;
                __syncthreads();
            }
            c2 = warp_sum64(c2);
            if (lane == 0) ctl.red[warp] = c2;
            __syncthreads();
            if (tid == 0) {
                long long s = 0;
                for (int j = 0; j < NW; j++) s += ctl.red[j];
                ctl.conflicts = s / 2;
                ctl.best = s / 2;
                ctl.C = base;
                ctl.it = 0;
                ctl.ctr = 0;
                ctl.nlog = 0;
                ctl.sum_c = 0;
                ctl.sum_deg = 0;
            }
        }
        for (int v = tid; v < n; v += NT) b_out[v] = assign[v];
        __syncthreads();

        // ---------------- iterations (:320-405) ----------------
        if (k >= 2 && !ctl.ovf) {
            for (long long step = 0; step < P.depth; step++) {
                const long long conflicts = ctl.conflicts;
                if (conflicts == 0 || ctl.ovf) break;
                const long long it = ctl.it;
                const int C = ctl.C;
                const long long best = ctl.best;
                const int thr = (int)max(best - conflicts, (long long)-TC_BIG);
                const uint32_t it32 = (uint32_t)it;

                // pass 1: per-row (min, count) over admissible candidates
                for (int r0 = warp * gpw; r0 < C; r0 += NW * gpw) {
                    const int li = r0 + gig;
                    const bool act = li < C;
                    int dv[MAXV];
                    eval_row<G, S, MAXV>(gamma, stamp, assign, act ? clist[li] : clist[0], kp, k,
                                         lig, RG, WPL, W, it32, thr, dv);
                    int lmin = TC_BIG;
#pragma unroll
                    for (int i = 0; i < MAXV; i++) lmin = min(lmin, dv[i]);
                    const int rmin = warp_min(lmin, RG);
                    int cnt = 0;
#pragma unroll
                    for (int i = 0; i < MAXV; i++) cnt += (dv[i] == rmin && rmin != TC_BIG);
                    const int nq = warp_sum(cnt, RG);
                    if (act && lig == 0) rinfo[li] = RI::pack(rmin, nq);
                }
                __syncthreads();

                // passes 2-4: warp 0
                if (warp == 0) {
                    int carry = TC_BIG, tsum = 0;
                    for (int base = 0; base < C; base += 32) {
                        const int li = base + lane;
                        int rm = TC_BIG, nq = 0;
                        if (li < C) RI::unpack(rinfo[li], rm, nq);
                        const int incl = warp_incl_min(rm, lane);
                        int excl = __shfl_up_sync(0xffffffffu, incl, 1);
                        if (lane == 0) excl = TC_BIG;
                        const int RM = min(carry, excl);
                        if (!prod) {
                            if (rm == RM && rm != TC_BIG) tsum += nq;
                            unsigned lm = __ballot_sync(0xffffffffu, rm < RM);
                            while (lm) {
                                unsigned mm = lm;
                                for (int t = 0; t < gig && mm; t++) mm &= mm - 1u;
                                const int src = mm ? (__ffs(mm) - 1) : -1;
                                for (int t = 0; t < gpw && lm; t++) lm &= lm - 1u;
                                const int R2 = __shfl_sync(0xffffffffu, RM, src < 0 ? 0 : src);
                                const int li2 = base + (src < 0 ? 0 : src);
                                int dv[MAXV];
                                eval_row<G, S, MAXV>(gamma, stamp, assign, clist[li2], kp, k, lig, RG,
                                                     WPL, W, it32, thr, dv);
                                const int ties = row_ties<EPW, MAXV>(dv, R2, lig, RG, WPL);
                                if (lig == 0 && src >= 0) tsum += ties;
                            }
                        }
                        carry = min(carry, __shfl_sync(0xffffffffu, incl, 31));
                    }
                    const int D = carry;
                    int T = 0;
                    if (D != TC_BIG) {
                        for (int base = 0; base < C; base += 32) {
                            const int li = base + lane;
                            int rm = TC_BIG, nq = 0;
                            if (li < C) RI::unpack(rinfo[li], rm, nq);
                            if (rm == D) T += nq;
                        }
                    }
                    T = warp_sum(T);
                    const int total = warp_sum(tsum);
                    unsigned long long ctr = ctl.ctr;
                    int sstar = 1;
                    if (D != TC_BIG && T > 1) {
                        if (!prod) {
                            const unsigned long long c0 = ctr + (unsigned long long)(total - (T - 1));
                            int smax = 1;
                            for (int s = 2 + lane; s <= T; s += 32)
                                if (below_is_zero(key, c0 + (unsigned long long)(s - 2), (uint32_t)s))
                                    smax = s;
                            sstar = warp_max(smax);
                        } else {
                            sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                        }
                    }
                    if (D != TC_BIG) {
                        // locate the sstar-th candidate with delta D in scan order
                        int cum = 0, row_li = 0, need = 1;
                        for (int base = 0; base < C; base += 32) {
                            const int li = base + lane;
                            int rm = TC_BIG, nq = 0;
                            if (li < C) RI::unpack(rinfo[li], rm, nq);
                            const int c = (rm == D) ? nq : 0;
                            const int incl = warp_incl_sum(c, lane);
                            const int tot = __shfl_sync(0xffffffffu, incl, 31);
                            if (cum + tot >= sstar) {
                                const unsigned bm = __ballot_sync(0xffffffffu, cum + incl >= sstar);
                                const int src = __ffs(bm) - 1;
                                row_li = base + src;
                                need = sstar - cum - __shfl_sync(0xffffffffu, incl - c, src);
                                break;
                            }
                            cum += tot;
                        }
                        const int v = clist[row_li];
                        int dv[MAXV];
                        eval_row<G, S, MAXV>(gamma, stamp, assign, v, kp, k, lig, RG, WPL, W, it32,
                                             thr, dv);
                        int b = -1;
#pragma unroll
                        for (int j = 0; j < MAXV / EPW; j++) {
                            if (j < WPL && need > 0) {
                                int cnt = 0;
#pragma unroll
                                for (int e = 0; e < EPW; e++) cnt += dv[j * EPW + e] == D;
                                const int incl = warp_incl_sum(cnt, lig, RG);
                                const int tot = __shfl_sync(0xffffffffu, incl, RG - 1, RG);
                                if (need <= tot) {
                                    if (incl >= need && incl - cnt < need) {
                                        int r = need - (incl - cnt);
#pragma unroll
                                        for (int e = 0; e < EPW; e++) {
                                            if (dv[j * EPW + e] == D) {
                                                if (--r == 0) b = (j * RG + lig) * EPW + e;
                                            }
                                        }
                                    }
                                    need = 0;
                                } else {
                                    need -= tot;
                                }
                            }
                        }
                        b = warp_max(b, 32);
                        if (lane == 0) {
                            const int a = assign[v];
                            const long long nconf = conflicts + D;
                            unsigned long long c = ctr;
                            uint32_t ll;
                            if (!prod) {
                                c += (unsigned long long)total;
                                ll = u64_below32(key, c, 10u);
                                c += 1;
                            } else {
                                ll = philox_below(key, c + 1, 10u);
                                c += 2;
                            }
                            const long long tt = (long long)ll + (6LL * nconf) / 10LL;
                            if (tt >= (long long)SWEEP) ctl.ovf = 1;
                            stamp[(size_t)v * kp + a] = (S)(uint32_t)(it + tt + 1);
                            ctl.mv_v = v;
                            ctl.mv_a = a;
                            ctl.mv_b = b;
                            ctl.mv_gvb = gamma[(size_t)v * kp + b];
                            ctl.conflicts = nconf;
                            ctl.ctr = c;
                            ctl.has_move = 1;
                            assign[v] = (uint8_t)b;
                            const long long nl = ctl.nlog;
                            if (nl < P.log_cap) {
                                const size_t o = (size_t)ind * P.log_cap + nl;
                                P.log_v[o] = v;
                                P.log_iter[o] = it;
                                P.log_tt[o] = tt;
                                ctl.nlog = nl + 1;
                            }
                            ctl.sum_deg += P.indptr[v + 1] - P.indptr[v];
                        }
                    } else if (lane == 0) {
                        ctl.has_move = 0;
                    }
                    if (lane == 0) {
                        ctl.sum_c += C;
                        ctl.nev = 0;
                    }
                }
                __syncthreads();

                // pass 5: gamma update over N(v) + conflict-set events (:356-359)
                const bool mv = ctl.has_move != 0;
                if (mv) {
                    const int v = ctl.mv_v, a = ctl.mv_a, b = ctl.mv_b;
                    const int64_t s0 = P.indptr[v], s1 = P.indptr[v + 1];
                    for (int64_t idx = s0 + tid; idx < s1; idx += NT) {
                        const int u = P.indices[idx];
                        G *row = gamma + (size_t)u * kp;
                        const int ga = (int)row[a] - 1;
                        row[a] = (G)ga;
                        const int gb = row[b];
                        if (gb >= GMAX) ctl.ovf = 1;
                        else row[b] = (G)(gb + 1);
                        const int au = assign[u];
                        if ((au == a && ga == 0) || (au == b && gb == 0)) {
                            const int slot = atomicAdd(&ctl.nev, 1);
                            if (slot < TC_EVCAP) evl[slot] = ((uint32_t)(idx - s0) << 16) | (uint32_t)u;
                        }
                    }
                }
                __syncthreads();

                // pass 6: conflict-list maintenance in neighbour order, then v (:368-390)
                if (tid == 0) {
                    if (mv) {
                        const int v = ctl.mv_v;
                        int Cn = ctl.C;
                        const int nev = ctl.nev;
                        auto apply = [&](int u, bool in_conf) {
                            const int pu = cpos[u];
                            if (in_conf && pu == 0xFFFF) {
                                cpos[u] = (uint16_t)Cn;
                                clist[Cn] = (uint16_t)u;
                                Cn++;
                            } else if (!in_conf && pu != 0xFFFF) {
                                const int last = clist[Cn - 1];
                                clist[pu] = (uint16_t)last;
                                cpos[last] = (uint16_t)pu;
                                Cn--;
                                cpos[u] = 0xFFFF;
                            }
                        };
                        if (nev <= TC_EVCAP) {
                            for (int i = 1; i < nev; i++) {  // insertion sort by position
                                const uint32_t x = evl[i];
                                int j = i - 1;
                                while (j >= 0 && evl[j] > x) {
                                    evl[j + 1] = evl[j];
                                    j--;
                                }
                                evl[j + 1] = x;
                            }
                            for (int i = 0; i < nev; i++) {
                                const int u = evl[i] & 0xFFFF;
                                apply(u, cpos[u] == 0xFFFF);  // enter iff outside, leave iff inside
                            }
                        } else {
                            const int64_t s0 = P.indptr[v], s1 = P.indptr[v + 1];
                            for (int64_t idx = s0; idx < s1; idx++) {
                                const int u = P.indices[idx];
                                apply(u, gamma[(size_t)u * kp + assign[u]] > 0);
                            }
                        }
                        apply(v, ctl.mv_gvb > 0);
                        ctl.C = Cn;
                        if (ctl.conflicts < ctl.best) {
                            ctl.best = ctl.conflicts;
                            ctl.copy = 1;
                        } else {
                            ctl.copy = 0;
                        }
                    } else {
                        ctl.copy = 0;
                    }
                    ctl.it = it + 1;
                }
                __syncthreads();
                const long long itn = it + 1;
                const bool chk = diagf && (itn % 1024 == 0);
                const bool swp = (itn % SWEEP) == 0;
                if (ctl.copy)
                    for (int v = tid; v < n; v += NT) b_out[v] = assign[v];
                if (chk) {  // scratch conflicts over the edge list (:398-405)
                    long long c2 = 0;
                    for (int64_t e = tid; e < P.m; e += NT) c2 += assign[P.eu[e]] == assign[P.ev[e]];
                    c2 = warp_sum64(c2);
                    if (lane == 0) ctl.red[warp] = c2;
                }
                if (swp) {
                    const uint32_t itw = (uint32_t)itn;
                    for (size_t i = tid; i < tab_elems; i += NT)
                        if (!stamp_active<S>(stamp[i], itw)) stamp[i] = (S)itw;
                }
                if (chk || swp) __syncthreads();
                if (chk && tid == 0) {
                    long long s = 0;
                    for (int j = 0; j < NW; j++) s += ctl.red[j];
                    if (s != ctl.conflicts) ctl.diag += 1;
                }
            }
        }
        __syncthreads();

        // ---------------- outputs (:407-410) ----------------
        if (!ctl.ovf) {
            for (int v = tid; v < n; v += NT) a_io[v] = assign[v];
            if (tid == 0) {
                P.end_conflicts[ind] = ctl.conflicts;
                P.best_conflicts[ind] = ctl.best;
                P.iters_used[ind] = ctl.it;
                P.diag[ind] = ctl.diag;
                if (P.log_cnt) P.log_cnt[ind] = ctl.nlog;
                if (P.counters) {
                    P.counters[2 * (size_t)ind] = ctl.sum_c;
                    P.counters[2 * (size_t)ind + 1] = ctl.sum_deg;
                }
            }
        } else if (tid == 0) {
            if (P.ovf_list) {
                const int slot = atomicAdd(P.ovf_count, 1);
                P.ovf_list[slot] = ind;
            } else {
                atomicExch(P.err_flag, 2);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t misc_bytes(int n, size_t rowinfo_bytes) {
    return (size_t)((n + 15) & ~15) + 2 * (size_t)((2 * n + 15) & ~15) +
           ((rowinfo_bytes * n + 15) & ~(size_t)15) + TC_EVCAP * 4;
}

template <typename G, typename S, bool GSM, bool SSM>
static int launch_variant(TabuParams P, int max_grid, int p_hint, cudaStream_t st, int *grid_out,
                          size_t *smem_out, bool query_only) {
    using RowT = typename RowInfoT<G>::T;
    const size_t tab = (size_t)P.n * P.kp;
    size_t smem = misc_bytes(P.n, sizeof(RowT));
    if (GSM) smem += (tab * sizeof(G) + 15) & ~(size_t)15;
    if (SSM) smem += (tab * sizeof(S) + 15) & ~(size_t)15;
    auto kern = tabucol_kernel<G, S, GSM, SSM>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "cudaFuncSetAttribute(smem=%zu) failed", smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, TC_NT, smem) != cudaSuccess || nb < 1)
        return set_error(MCB_ERR_CUDA, "tabucol: no occupancy for smem=%zu", smem);
    int grid = std::min(p_hint, nb * num_sms());
    if (max_grid > 0) grid = std::min(grid, max_grid);
    grid = std::max(grid, 1);
    *grid_out = grid;
    *smem_out = smem;
    if (query_only) return MCB_OK;
    kern<<<grid, TC_NT, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol launch failed");
    return MCB_OK;
}

static bool fits_smem(size_t bytes) { return bytes <= (size_t)max_smem_optin(); }

int tabucol_run(const TabucolArgs &A, cudaStream_t st) {
    if (A.p < 0 || A.n < 1 || A.k < 1 || A.depth < 0 || A.m < 0)
        return set_error(MCB_ERR_VALUE, "tabucol: bad shape p=%lld n=%lld k=%lld depth=%lld",
                         (long long)A.p, (long long)A.n, (long long)A.k, (long long)A.depth);
    if (A.n > 32767 || A.k > 255)
        return set_error(MCB_ERR_UNSUPPORTED, "tabucol: n<=32767 and k<=255 required");
    if (A.p == 0) return MCB_OK;
    const int n = (int)A.n, k = (int)A.k, kp = (k + 3) & ~3;

    TabuParams P{};
    P.assigns = A.assigns;
    P.best_assigns = A.best_assigns;
    P.indptr = A.indptr;
    P.indices = A.indices;
    P.eu = A.eu;
    P.ev = A.ev;
    P.m = A.m;
    P.n = n;
    P.k = k;
    P.kp = kp;
    P.depth = A.depth;
    P.keys = A.keys;
    P.best_conflicts = A.best_conflicts;
    P.end_conflicts = A.end_conflicts;
    P.iters_used = A.iters_used;
    P.diag = A.diag;
    P.log_cap = A.log_cap;
    P.log_v = A.log_v;
    P.log_iter = A.log_iter;
    P.log_tt = A.log_tt;
    P.log_cnt = A.log_cnt;
    P.counters = A.counters;
    P.flags = A.flags;
    P.nwork = (int)A.p;

    const bool force_wide = (A.flags & MCB_FLAG_FORCE_WIDE) != 0;
    const bool force_glob = (A.flags & MCB_FLAG_FORCE_GLOBAL) != 0;
    const size_t tab = (size_t)n * kp;
    const size_t misc8 = misc_bytes(n, 2);
    const size_t g8 = (tab + 15) & ~(size_t)15, s16 = (tab * 2 + 15) & ~(size_t)15;
    int variant;  // 0: all smem, 1: gamma smem + stamps global, 2: all global (narrow), 3: wide global
    if (force_wide) variant = 3;
    else if (!force_glob && fits_smem(g8 + s16 + misc8)) variant = 0;
    else if (!force_glob && fits_smem(g8 + misc8)) variant = 1;
    else variant = 2;

    // work counters, overflow list, error flag
    const int grid_cap = 8 * num_sms();
    const size_t ctl_bytes = 256 + sizeof(int32_t) * (size_t)A.p;
    // global tables: narrow variant (per CTA) and wide fallback (per CTA)
    const size_t ng_stride = (tab * 1 + 255) & ~(size_t)255, ns_stride = (tab * 2 + 255) & ~(size_t)255;
    const size_t wg_stride = (tab * 2 + 255) & ~(size_t)255, ws_stride = (tab * 4 + 255) & ~(size_t)255;
    const int wide_grid = std::min<int>((int)A.p, 2 * num_sms());

    int grid = 1;
    size_t smem = 0;
    int rc;
    // query grid for the narrow variant first (to size its workspace)
    auto set_rows = [&](TabuParams &Q, int gbytes) {
        const int words = kp * gbytes / 4;
        int rg = 1;
        while (rg < words && rg < 32) rg <<= 1;
        Q.rg = rg;
        Q.words = words;
        Q.wpl = (words + rg - 1) / rg;
    };
    size_t narrow_ws = 0;
    if (variant != 3) {
        set_rows(P, 1);
        switch (variant) {
            case 0: rc = launch_variant<int8_t, uint16_t, true, true>(P, grid_cap, (int)A.p, st, &grid, &smem, true); break;
            case 1: rc = launch_variant<int8_t, uint16_t, true, false>(P, grid_cap, (int)A.p, st, &grid, &smem, true); break;
            default: rc = launch_variant<int8_t, uint16_t, false, false>(P, grid_cap, (int)A.p, st, &grid, &smem, true); break;
        }
        if (rc) return rc;
        if (variant == 1) narrow_ws = (size_t)grid * ns_stride;
        if (variant == 2) narrow_ws = (size_t)grid * (ng_stride + ns_stride);
    }
    const size_t wide_ws = (size_t)wide_grid * (wg_stride + ws_stride);
    uint8_t *ws = (uint8_t *)workspace(ctl_bytes + narrow_ws + wide_ws + 512);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol: workspace allocation failed");
    int32_t *ctl32 = reinterpret_cast<int32_t *>(ws);  // [0]=work(narrow) [1]=work(wide) [2]=ovf_count [3]=err
    if (cudaMemsetAsync(ws, 0, 256, st) != cudaSuccess) return set_error(MCB_ERR_CUDA, "memset failed");
    P.err_flag = ctl32 + 3;
    uint8_t *tables = ws + ((ctl_bytes + 255) & ~(size_t)255);

    if (variant != 3) {
        P.work_counter = ctl32 + 0;
        P.ovf_count = ctl32 + 2;
        P.ovf_list = ctl32 + 64;
        if (variant == 1) {
            P.ws_stamp = tables;
            P.ws_s_stride = ns_stride;
        } else if (variant == 2) {
            P.ws_gamma = tables;
            P.ws_g_stride = ng_stride;
            P.ws_stamp = tables + (size_t)grid * ng_stride;
            P.ws_s_stride = ns_stride;
        }
        switch (variant) {
            case 0: rc = launch_variant<int8_t, uint16_t, true, true>(P, grid_cap, (int)A.p, st, &grid, &smem, false); break;
            case 1: rc = launch_variant<int8_t, uint16_t, true, false>(P, grid_cap, (int)A.p, st, &grid, &smem, false); break;
            default: rc = launch_variant<int8_t, uint16_t, false, false>(P, grid_cap, (int)A.p, st, &grid, &smem, false); break;
        }
        if (rc) return rc;
    }
    // wide pass: either everything (forced) or the overflowed individuals
    TabuParams Q = P;
    set_rows(Q, 2);
    Q.work_counter = ctl32 + 1;
    Q.ovf_list = nullptr;
    Q.ovf_count = nullptr;
    if (variant != 3) {
        Q.work = ctl32 + 64;
        Q.nwork_dev = ctl32 + 2;
    }
    Q.ws_gamma = tables + narrow_ws;
    Q.ws_g_stride = wg_stride;
    Q.ws_stamp = tables + narrow_ws + (size_t)wide_grid * wg_stride;
    Q.ws_s_stride = ws_stride;
    int g2 = 1;
    rc = launch_variant<int16_t, uint32_t, false, false>(Q, wide_grid, (int)A.p, st, &g2, &smem, false);
    if (rc) return rc;

    int32_t err = 0;
    if (cudaMemcpyAsync(&err, ctl32 + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol: kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (err == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
    if (err == 2) return set_error(MCB_ERR_UNSUPPORTED, "tabucol: wide tables overflowed");
    return MCB_OK;
}

}  // namespace mcb
