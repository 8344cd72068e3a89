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
// One iteration = two block barriers:
//   pass 1 (all threads)  thread-per-row: each conflicting vertex's k-1
//          candidates are evaluated 4 at a time with byte-SIMD (int8 deltas,
//          u16 wrap-around tabu stamps, aspiration) -> (row min, #at min).
//   pass 2 (warp 0)       exclusive prefix-min over the row minima.  A tie
//          event of the sequential reservoir is a candidate equal to the
//          running minimum: rows above the running minimum contribute none,
//          rows equal to it contribute #min, and the few rows that LOWER it are
//          re-walked lane-locally.  That yields the global minimum D, its
//          multiplicity T and the counter offset E of D's group, so the T-1
//          reservoir draws (counter ctr+E+s-2 for rank s) are independent: the
//          winner is the last rank whose draw is zero (warp max).
//          Then the winner is located, the tenure drawn, gamma updated over
//          N(v) by the warp (32 neighbours per step) and conflict-set events
//          applied in neighbour order (ballot order), then v itself.
//
// Data layout per individual (shared memory when it fits, else a per-CTA
// global slice that stays L2-resident):
//   gamma  int8 [n][kp]  (kp = k rounded up to 4)   -- int16 fallback on overflow
//   tabu   u16  [n][kp]  wrap-around stamps, swept every 16384 iterations
//                        -- u32 fallback when a tenure exceeds 16383
//   assign u8 [n], conflict list / positions u16 [n], per-row (min, count) [n].
//   CSR row offsets in __constant__ memory (u32) when n < 12288.
// Individuals whose int8/u16 tables would overflow are re-run from their
// original start by the wide (int16 / u32) instantiation; results are
// identical by construction (same arithmetic, wider storage).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int TC_BIG = 1 << 20;
constexpr int TC_CONST_INDPTR = 12288;

__constant__ uint32_t c_indptr[TC_CONST_INDPTR];

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
    int const_indptr;
};

__device__ unsigned long long g_phase_cycles[16];
#define PH(i)                                          \
    if (profile && tid == 0) {                         \
        const long long _t = clock64();                \
        ctl.ph[i] += _t - ph_t;                        \
        ph_t = _t;                                     \
    }

struct TabuCtrl {
    long long it, conflicts, best, nlog, sum_c, sum_deg, diag;
    unsigned long long ctr;
    int C, work, ovf;
    long long ph[12];
    long long red[32];
    int wcnt[32];
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

// signed byte-min of the 4 bytes of x; *bc = that byte broadcast to 4 lanes
__device__ __forceinline__ int bmin4(uint32_t x, uint32_t &bc) {
    uint32_t y = __vmins4(x, __byte_perm(x, 0, 0x3232));
    y = __vmins4(y, __byte_perm(y, 0, 0x1111));
    bc = __byte_perm(y, 0, 0x0000);
    return (int)(int8_t)(y & 0xFFu);
}

// One conflicting vertex's candidate row: delta = gamma[v][c] - gamma[v][a],
// admissible = c != a && (not tabu || conflicts + delta < best).
template <typename G, typename S>
struct Row {
    const G *g;
    const S *s;
    int a, gva, k, W;
    uint32_t it, gva4, thr4, it2, amask, kmask;
    int thr, aw;

    __device__ __forceinline__ Row(const G *gamma, const S *stamp, const uint8_t *assign, int v, int kp,
                                   int k_, uint32_t it_, int thr_) {
        a = assign[v];
        g = gamma + (size_t)v * kp;
        s = stamp + (size_t)v * kp;
        gva = g[a];
        k = k_;
        it = it_;
        thr = thr_;
        W = kp / 4;
        if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
            gva4 = (uint32_t)gva * 0x01010101u;
            const int t8 = max(thr, -128);
            thr4 = (uint32_t)(uint8_t)(int8_t)t8 * 0x01010101u;
            it2 = ((it & 0xFFFFu) << 16) | (it & 0xFFFFu);
            aw = a >> 2;
            amask = 0xFFu << (8 * (a & 3));
            const int rem = k & 3;
            kmask = rem ? (0xFFFFFFFFu >> (8 * (4 - rem))) : 0xFFFFFFFFu;
        }
    }
    // narrow path: 4 candidates (colours 4w..4w+3) as signed bytes, 127 = inadmissible
    __device__ __forceinline__ uint32_t word(int w) const {
        const uint32_t gw = reinterpret_cast<const uint32_t *>(g)[w];
        const uint2 st = reinterpret_cast<const uint2 *>(s)[w];
        const uint32_t d = __vsub4(gw, gva4);
        const uint32_t m0 = __vcmpgts2(__vsub2(st.x, it2), 0u);
        const uint32_t m1 = __vcmpgts2(__vsub2(st.y, it2), 0u);
        const uint32_t tabu = __byte_perm(m0, m1, 0x6420);
        uint32_t ok = ~tabu | __vcmplts4(d, thr4);
        if (w == aw) ok &= ~amask;
        if (w == W - 1) ok &= kmask;
        return (d & ok) | (0x7F7F7F7Fu & ~ok);
    }
    // wide path: one candidate, TC_BIG if inadmissible
    __device__ __forceinline__ int cand(int c) const {
        if (c == a) return TC_BIG;
        const int d = (int)g[c] - gva;
        if (stamp_active<S>(s[c], it) && !(d < thr)) return TC_BIG;
        return d;
    }

    // (row min, #candidates at the min); min = TC_BIG if none admissible
    __device__ __forceinline__ void scan(int &rmin, int &nq) const {
        if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
            int m = 127, cnt = 0;
#pragma unroll 4
            for (int w = 0; w < W; w++) {
                const uint32_t dv = word(w);
                uint32_t bc;
                const int wm = bmin4(dv, bc);
                const int c = __popc(__vcmpeq4(dv, bc)) >> 3;
                cnt = (wm < m) ? c : (wm == m ? cnt + c : cnt);
                m = min(m, wm);
            }
            rmin = (m == 127) ? TC_BIG : m;
            nq = (m == 127) ? 0 : cnt;
        } else {
            int m = TC_BIG, cnt = 0;
            for (int c = 0; c < k; c++) {
                const int x = cand(c);
                if (x < m) {
                    m = x;
                    cnt = 1;
                } else if (x == m && x != TC_BIG) {
                    cnt++;
                }
            }
            rmin = m;
            nq = cnt;
        }
    }
    // (min, count) over words sub, sub+tpr, ... (narrow path only)
    __device__ __forceinline__ void scan_part(int sub, int tpr, int &rmin, int &nq) const {
        int m = 127, cnt = 0;
#pragma unroll 2
        for (int w = sub; w < W; w += tpr) {
            const uint32_t dv = word(w);
            uint32_t bc;
            const int wm = bmin4(dv, bc);
            const int c = __popc(__vcmpeq4(dv, bc)) >> 3;
            cnt = (wm < m) ? c : (wm == m ? cnt + c : cnt);
            m = min(m, wm);
        }
        rmin = (m == 127) ? TC_BIG : m;
        nq = (m == 127) ? 0 : cnt;
    }
    // sequential tie events inside the row when entered with running minimum R
    __device__ __forceinline__ int ties(int R) const {
        int cur = R, t = 0;
        if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
            for (int w = 0; w < W; w++) {
                const uint32_t dv = word(w);
                uint32_t bc;
                const int wm = bmin4(dv, bc);
                if (wm == 127 || wm > cur) continue;
                if (wm == cur) {
                    t += __popc(__vcmpeq4(dv, bc)) >> 3;
                    continue;
                }
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int x = (int)(int8_t)(dv >> (8 * e));
                    if (x == 127) continue;
                    if (x < cur) cur = x;
                    else if (x == cur) t++;
                }
            }
        } else {
            for (int c = 0; c < k; c++) {
                const int x = cand(c);
                if (x == TC_BIG) continue;
                if (x < cur) cur = x;
                else if (x == cur) t++;
            }
        }
        return t;
    }
    // colour of the j-th (1-based) admissible candidate with delta D
    __device__ __forceinline__ int find(int D, int j) const {
        if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
            const uint32_t d4 = (uint32_t)(uint8_t)(int8_t)D * 0x01010101u;
            for (int w = 0; w < W; w++) {
                const uint32_t eq = __vcmpeq4(word(w), d4);
                const int c = __popc(eq) >> 3;
                if (j <= c) {
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if ((eq >> (8 * e)) & 1u)
                            if (--j == 0) return 4 * w + e;
                }
                j -= c;
            }
        } else {
            for (int c = 0; c < k; c++)
                if (cand(c) == D && --j == 0) return c;
        }
        return -1;
    }
};

template <typename G, typename S, bool GSM, bool SSM, int NT>
__global__ void __launch_bounds__(NT) tabucol_kernel(TabuParams P) {
    constexpr int NW = NT / 32;
    constexpr int GMAX = sizeof(G) == 1 ? 127 : 32767;
    constexpr uint32_t SWEEP = sizeof(S) == 2 ? 16384u : (1u << 30);
    constexpr unsigned FULL = 0xffffffffu;
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

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool profile = (P.flags & MCB_FLAG_PROFILE) != 0;
    const size_t tab_elems = (size_t)n * kp;
    const bool cidx = P.const_indptr != 0;
    auto row_begin = [&](int v) -> int64_t { return cidx ? (int64_t)c_indptr[v] : P.indptr[v]; };

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
            for (int q = 0; q < 12; q++) ctl.ph[q] = 0;
        }
        __syncthreads();
        // gamma[u][c] = #neighbours of u coloured c; each thread owns its rows
        {
            int bad = 0;
            for (int u = tid; u < n; u += NT) {
                G *row = gamma + (size_t)u * kp;
                const int64_t s0 = row_begin(u), s1 = row_begin(u + 1);
                for (int64_t idx = s0; idx < s1; idx++) {
                    const int c = assign[__ldg(P.indices + idx)];
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
                const unsigned bal = __ballot_sync(FULL, f);
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
                long long ph_t = clock64();
                const long long conflicts = ctl.conflicts;
                if (conflicts == 0 || ctl.ovf) break;
                const long long it = ctl.it;
                const int C = ctl.C;
                const long long best = ctl.best;
                const int thr = (int)max(best - conflicts, (long long)-TC_BIG);
                const uint32_t it32 = (uint32_t)it;

                // pass 1: (min, count) over admissible candidates of every row;
                // tpr threads per row (power of two) when rows are few
                {
                    int tpr = 1;
                    if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
                        const int W = kp / 4;
                        while (tpr < 16 && tpr * 2 * C <= NT && tpr * 2 <= W) tpr *= 2;
                    }
                    const int sub = tid & (tpr - 1);
                    const int rows_per_pass = NT / tpr;
                    for (int r0 = 0; r0 < C; r0 += rows_per_pass) {
                        const int li = r0 + tid / tpr;
                        int rm = TC_BIG, nq = 0;
                        if (li < C) {
                            const Row<G, S> row(gamma, stamp, assign, clist[li], kp, k, it32, thr);
                            if constexpr (sizeof(G) == 1 && sizeof(S) == 2) {
                                if (tpr == 1) row.scan(rm, nq);
                                else row.scan_part(sub, tpr, rm, nq);
                            } else {
                                row.scan(rm, nq);
                            }
                        }
                        if (tpr > 1) {  // combine the tpr partial (min, count)
                            for (int o = 1; o < tpr; o <<= 1) {
                                const int om = __shfl_xor_sync(0xffffffffu, rm, o);
                                const int oq = __shfl_xor_sync(0xffffffffu, nq, o);
                                nq = (om < rm) ? oq : (om == rm ? nq + oq : nq);
                                rm = min(rm, om);
                            }
                        }
                        if (li < C && sub == 0) rinfo[li] = RI::pack(rm, rm == TC_BIG ? 0 : nq);
                    }
                }
                __syncthreads();

                PH(1);
                // pass 2: warp 0 -- reservoir, move, gamma update, conflict list
                if (warp == 0) {
                    // -- exclusive prefix-min over the row minima, R rows per lane
                    const int R = C <= 32 ? 1 : (C <= 64 ? 2 : 4);
                    int carry = TC_BIG, lmin = TC_BIG, lT = 0, lfirst = INT_MAX, tsum = 0;
                    for (int base = 0; base < C; base += 32 * R) {
                        const int l0 = base + lane * R;
                        int rm[4], nq[4];
                        int lmn = TC_BIG;
#pragma unroll
                        for (int r = 0; r < 4; r++) {
                            rm[r] = TC_BIG;
                            nq[r] = 0;
                            if (r < R && l0 + r < C) RI::unpack(rinfo[l0 + r], rm[r], nq[r]);
                            lmn = min(lmn, rm[r]);
                        }
                        const int incl = warp_incl_min(lmn, lane);
                        int excl = __shfl_up_sync(FULL, incl, 1);
                        if (lane == 0) excl = TC_BIG;
                        int RM = min(carry, excl);
#pragma unroll
                        for (int r = 0; r < 4; r++) {
                            if (r >= R) break;
                            const int x = rm[r];
                            if (x < lmin) {
                                lmin = x;
                                lT = nq[r];
                                lfirst = l0 + r;
                            } else if (x == lmin && x != TC_BIG) {
                                lT += nq[r];
                            }
                            if (!prod && x != TC_BIG) {
                                if (x == RM) {
                                    tsum += nq[r];
                                } else if (x < RM) {  // lowers the running minimum: walk it
                                    const Row<G, S> row(gamma, stamp, assign, clist[l0 + r], kp, k, it32, thr);
                                    tsum += row.ties(RM);
                                }
                            }
                            RM = min(RM, x);
                        }
                        carry = min(carry, __shfl_sync(FULL, incl, 31));
                    }
                    const int D = carry;
                    PH(2);
                    int mv_v = -1, mv_a = 0, mv_b = 0, gvb = 0;
                    int64_t s0 = 0, s1 = 0;
                    constexpr int NB = 8;  // neighbour chunks of 32 held in registers
                    int uu[NB];
                    int v_guess = -1;
                    if (D != TC_BIG) {
                        const int T = __reduce_add_sync(FULL, lmin == D ? lT : 0);
                        const int L = (int)__reduce_min_sync(FULL, (unsigned)(lmin == D ? lfirst : INT_MAX));
                        // speculative prefetch: adjacency of the first D-row's vertex (the
                        // winner whenever the reservoir keeps rank 1 or stays in that row)
                        v_guess = clist[L];
                        {
                            const int64_t g0 = row_begin(v_guess), g1 = row_begin(v_guess + 1);
#pragma unroll
                            for (int j = 0; j < NB; j++) {
                                const int64_t idx = g0 + j * 32 + lane;
                                uu[j] = idx < g1 ? __ldg(P.indices + idx) : 0;
                            }
                        }
                        const int total = __reduce_add_sync(FULL, tsum);
                        const unsigned long long ctr = ctl.ctr;
                        int sstar = 1;
                        if (T > 1) {
                            if (!prod) {
                                const unsigned long long c0 = ctr + (unsigned long long)(total - (T - 1));
                                int smax = 1;
                                for (int s = 2 + lane; s <= T; s += 32)
                                    if (below_is_zero(key, c0 + (unsigned long long)(s - 2), (uint32_t)s))
                                        smax = s;
                                sstar = __reduce_max_sync(FULL, smax);
                            } else {
                                sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                            }
                        }
                        PH(3);
                        int row_li = L, need = 1;
                        if (sstar > 1) {  // rank sstar among the D-candidates in scan order
                            int cum = 0;
                            for (int base = 0; base < C; base += 32) {
                                const int li = base + lane;
                                int rm = TC_BIG, nq = 0;
                                if (li < C) RI::unpack(rinfo[li], rm, nq);
                                const int c = (rm == D) ? nq : 0;
                                const int incl = warp_incl_sum(c, lane);
                                const int tot = __shfl_sync(FULL, incl, 31);
                                if (cum + tot >= sstar) {
                                    const unsigned bm = __ballot_sync(FULL, cum + incl >= sstar);
                                    const int src = __ffs(bm) - 1;
                                    row_li = base + src;
                                    need = sstar - cum - __shfl_sync(FULL, incl - c, src);
                                    break;
                                }
                                cum += tot;
                            }
                        }
                        PH(4);
                        if (lane == 0) {
                            const int v = clist[row_li];
                            const Row<G, S> row(gamma, stamp, assign, v, kp, k, it32, thr);
                            const int b = row.find(D, need);
                            const int a = row.a;
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
                            if (tt >= (long long)SWEEP || b < 0) ctl.ovf = 1;
                            stamp[(size_t)v * kp + a] = (S)(uint32_t)(it + tt + 1);
                            gvb = gamma[(size_t)v * kp + b];
                            assign[v] = (uint8_t)b;
                            ctl.conflicts = nconf;
                            ctl.ctr = c;
                            const long long nl = ctl.nlog;
                            if (nl < P.log_cap) {
                                const size_t o = (size_t)ind * P.log_cap + nl;
                                P.log_v[o] = v;
                                P.log_iter[o] = it;
                                P.log_tt[o] = tt;
                                ctl.nlog = nl + 1;
                            }
                            s0 = row_begin(v);
                            s1 = row_begin(v + 1);
                            ctl.sum_deg += s1 - s0;
                            mv_v = v;
                            mv_a = a;
                            mv_b = b;
                        }
                        mv_v = __shfl_sync(FULL, mv_v, 0);
                        mv_a = __shfl_sync(FULL, mv_a, 0);
                        mv_b = __shfl_sync(FULL, mv_b, 0);
                        s0 = __shfl_sync(FULL, s0, 0);
                        s1 = __shfl_sync(FULL, s1, 0);
                    }
                    PH(5);
                    if (mv_v >= 0) {
                        // gamma update over N(v) (:356-359) and conflict-list events in
                        // neighbour order (:368-385): NB*32 neighbours per batch, all
                        // loads in flight together, events applied in ballot order
                        int Cn = C;
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
                        bool bad = false;
                        bool have = (mv_v == v_guess);
                        for (int64_t b0 = s0; b0 < s1; b0 += 32 * NB) {
                            if (!have) {
#pragma unroll
                                for (int j = 0; j < NB; j++) {
                                    const int64_t idx = b0 + j * 32 + lane;
                                    uu[j] = idx < s1 ? __ldg(P.indices + idx) : 0;
                                }
                            }
                            have = false;
                            unsigned em[NB];
#pragma unroll
                            for (int j = 0; j < NB; j++) {
                                const int64_t idx = b0 + j * 32 + lane;
                                bool evt = false;
                                if (idx < s1) {
                                    const int u = uu[j];
                                    G *row = gamma + (size_t)u * kp;
                                    const int ga = (int)row[mv_a] - 1;
                                    row[mv_a] = (G)ga;
                                    const int gb = row[mv_b];
                                    if (gb >= GMAX) bad = true;
                                    else row[mv_b] = (G)(gb + 1);
                                    const int au = assign[u];
                                    evt = (au == mv_a && ga == 0) || (au == mv_b && gb == 0);
                                }
                                em[j] = __ballot_sync(FULL, evt);
                            }
#pragma unroll
                            for (int j = 0; j < NB; j++) {
                                unsigned e = em[j];
                                while (e) {
                                    const int src = __ffs(e) - 1;
                                    e &= e - 1u;
                                    const int u = __shfl_sync(FULL, uu[j], src);
                                    if (lane == 0) apply(u, cpos[u] == 0xFFFF);  // enter iff outside
                                }
                            }
                        }
                        PH(6);
                        if (__any_sync(FULL, bad) && lane == 0) ctl.ovf = 1;
                        bool improved = false;
                        if (lane == 0) {
                            apply(mv_v, gvb > 0);
                            ctl.C = Cn;
                            if (ctl.conflicts < ctl.best) {
                                ctl.best = ctl.conflicts;
                                improved = true;
                            }
                        }
                        if (__shfl_sync(FULL, improved, 0)) {
                            __syncwarp();
                            for (int v = lane; v < n; v += 32) b_out[v] = assign[v];
                        }
                    }
                    if (lane == 0) {
                        ctl.sum_c += C;
                        ctl.it = it + 1;
                    }
                    PH(7);
                }
                __syncthreads();
                PH(8);
                const long long itn = it + 1;
                const bool chk = diagf && (itn % 1024 == 0);
                const bool swp = (itn % SWEEP) == 0;
                if (chk) {  // scratch conflicts over the edge list (:398-405)
                    long long c2 = 0;
                    for (int64_t e = tid; e < P.m; e += NT)
                        c2 += assign[__ldg(P.eu + e)] == assign[__ldg(P.ev + e)];
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
                PH(9);
            }
        }
        __syncthreads();

        // ---------------- outputs (:407-410) ----------------
        if (profile && tid == 0) {
            for (int q = 1; q < 10; q++) atomicAdd(&g_phase_cycles[q], (unsigned long long)ctl.ph[q]);
            atomicAdd(&g_phase_cycles[10], (unsigned long long)ctl.it);
        }
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

__global__ void indptr_to_u32(const int64_t *in, uint32_t *out, int count) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t misc_bytes(int n, size_t rowinfo_bytes) {
    return (size_t)((n + 15) & ~15) + 2 * (size_t)((2 * n + 15) & ~15) +
           ((rowinfo_bytes * n + 15) & ~(size_t)15);
}

template <typename G, typename S, bool GSM, bool SSM, int NT>
static int launch_variant(TabuParams P, int max_grid, int p_hint, cudaStream_t st, int *grid_out,
                          size_t *smem_out, bool query_only) {
    using RowT = typename RowInfoT<G>::T;
    const size_t tab = (size_t)P.n * P.kp;
    size_t smem = misc_bytes(P.n, sizeof(RowT));
    if (GSM) smem += (tab * sizeof(G) + 15) & ~(size_t)15;
    if (SSM) smem += (tab * sizeof(S) + 15) & ~(size_t)15;
    auto kern = tabucol_kernel<G, S, GSM, SSM, NT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "cudaFuncSetAttribute(smem=%zu) failed", smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NT, smem) != cudaSuccess || nb < 1)
        return set_error(MCB_ERR_CUDA, "tabucol: no occupancy for smem=%zu", smem);
    int grid = std::min(p_hint, nb * num_sms());
    if (max_grid > 0) grid = std::min(grid, max_grid);
    grid = std::max(grid, 1);
    *grid_out = grid;
    *smem_out = smem;
    if (query_only) return MCB_OK;
    kern<<<grid, NT, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol launch failed");
    return MCB_OK;
}

static bool fits_smem(size_t bytes) { return bytes <= (size_t)max_smem_optin(); }

static int env_nt() {
    const char *e = getenv("MCB_TABU_NT");
    return e ? atoi(e) : 0;
}

template <int NT>
static int launch_narrow(int variant, TabuParams &P, int grid_cap, int p, cudaStream_t st, int *grid,
                         size_t *smem, bool q) {
    switch (variant) {
        case 0: return launch_variant<int8_t, uint16_t, true, true, NT>(P, grid_cap, p, st, grid, smem, q);
        case 1: return launch_variant<int8_t, uint16_t, true, false, NT>(P, grid_cap, p, st, grid, smem, q);
        default: return launch_variant<int8_t, uint16_t, false, false, NT>(P, grid_cap, p, st, grid, smem, q);
    }
}

int tabucol_phase_cycles(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "phase counters unavailable");
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return MCB_OK;
}

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
    const int nt = env_nt() == 128 ? 128 : 256;

    const int grid_cap = 8 * num_sms();
    const size_t ctl_bytes = 256 + sizeof(int32_t) * (size_t)A.p;
    const size_t ng_stride = (tab * 1 + 255) & ~(size_t)255, ns_stride = (tab * 2 + 255) & ~(size_t)255;
    const size_t wg_stride = (tab * 2 + 255) & ~(size_t)255, ws_stride = (tab * 4 + 255) & ~(size_t)255;
    const int wide_grid = std::min<int>((int)A.p, 2 * num_sms());
    const size_t indptr_bytes = 4 * (size_t)(n + 1);

    int grid = 1;
    size_t smem = 0;
    int rc;
    size_t narrow_ws = 0;
    if (variant != 3) {
        rc = nt == 128 ? launch_narrow<128>(variant, P, grid_cap, (int)A.p, st, &grid, &smem, true)
                       : launch_narrow<256>(variant, P, grid_cap, (int)A.p, st, &grid, &smem, true);
        if (rc) return rc;
        if (variant == 1) narrow_ws = (size_t)grid * ns_stride;
        if (variant == 2) narrow_ws = (size_t)grid * (ng_stride + ns_stride);
    }
    const size_t wide_ws = (size_t)wide_grid * (wg_stride + ws_stride);
    const size_t tables_off = (ctl_bytes + 255) & ~(size_t)255;
    const size_t indptr_off = tables_off + ((narrow_ws + wide_ws + 255) & ~(size_t)255);
    uint8_t *ws = (uint8_t *)workspace(indptr_off + indptr_bytes + 256);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol: workspace allocation failed");
    int32_t *ctl32 = reinterpret_cast<int32_t *>(ws);  // [0]=work(narrow) [1]=work(wide) [2]=ovf_count [3]=err
    if (cudaMemsetAsync(ws, 0, 256, st) != cudaSuccess) return set_error(MCB_ERR_CUDA, "memset failed");
    P.err_flag = ctl32 + 3;
    uint8_t *tables = ws + tables_off;

    // CSR row offsets -> __constant__ (u32) when they fit
    P.const_indptr = 0;
    if (n + 1 <= TC_CONST_INDPTR && 2 * A.m < (int64_t)UINT32_MAX) {
        uint32_t *tmp = reinterpret_cast<uint32_t *>(ws + indptr_off);
        indptr_to_u32<<<(n + 256) / 256, 256, 0, st>>>(A.indptr, tmp, n + 1);
        if (cudaMemcpyToSymbolAsync(c_indptr, tmp, indptr_bytes, 0, cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
            return set_error(MCB_ERR_CUDA, "tabucol: constant upload failed");
        P.const_indptr = 1;
    }

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
        rc = nt == 128 ? launch_narrow<128>(variant, P, grid_cap, (int)A.p, st, &grid, &smem, false)
                       : launch_narrow<256>(variant, P, grid_cap, (int)A.p, st, &grid, &smem, false);
        if (rc) return rc;
    }
    // wide pass: either everything (forced) or the overflowed individuals
    TabuParams Q = P;
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
    rc = launch_variant<int16_t, uint32_t, false, false, 256>(Q, wide_grid, (int)A.p, st, &g2, &smem,
                                                               false);
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
