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
//     `U{0..9} + (6*conflicts_after)//10` (:363-366), last-write-wins expiry;
//   * early exit at zero conflicts (:322), `it` counts no-move iterations (:398),
//     O(m) scratch check every 1024 iterations -> diag (:398-405).
//
// Iteration structure (NT threads):
//   pass 1 (all threads, one conflicting vertex per thread): the row's
//     candidates are scanned 4 colours per 32-bit word (u8 gamma; native
//     VIMNMX.U16x2 byte minima and LOP3/IADD zero-byte counts, branch-free --
//     no emulated video-SIMD), tabu/aspiration exclusions applied as byte
//     masks -> (row minimum, #candidates at the minimum).
//   pass 2a (all warps, per-warp contiguous blocks of rows): block minima,
//     then each block's exclusive prefix-min from its entering running
//     minimum.  A tie event of the sequential reservoir is a candidate equal to
//     the running minimum, so rows above the running minimum hold none, rows
//     equal to it hold #min of them, and only the few rows that LOWER it need
//     an in-row walk (warp-cooperative, by the block's warp).  That gives the
//     minimum D, its multiplicity T and the counter offset of D's group.
//   pass 2b (warp 0): the T-1 reservoir draws are independent (rank s uses
//     counter ctr + E + s - 2) and the winner is the last rank whose draw is
//     zero; its block from the per-warp D-counts, its row in the block, then
//     locate (parallel over the row's words), tenure, gamma update over N(v)
//     (adjacency prefetched speculatively), conflict-list events in
//     neighbour order, best copy.
//
// Tabu state: the reference's dense `tabu_pair[n][k]` int64 table is replaced
// by 4 (colour, expiry) slots per vertex in shared memory; a vertex needing a
// 5th live entry spills to a dense per-CTA table in global memory (L2
// resident), flagged per vertex.  Expiries are 16-bit wrap-around stamps,
// swept every 16384 iterations (32-bit in the wide variant).
//
// Shared memory per individual at G(500,.5) k=48: gamma 24 KB + slots 6 KB +
// lists 5.5 KB = 37 KB -> 6 CTAs per SM.  Individuals whose u8 gamma (max 254)
// or 16-bit tenure would overflow are re-run from their start by the wide
// (u16 gamma / u32 expiry) instantiation; results are identical by
// construction (same arithmetic, wider storage).
#include <algorithm>
#include <map>
#include <memory>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tc_shared.cuh"

namespace mcb {

constexpr int TC_CONST_INDPTR = 12288;
constexpr int TC_NT = 128;

__constant__ uint32_t c_indptr[TC_CONST_INDPTR];
__device__ unsigned long long g_phase_cycles[16];

#define PH(i)                                   \
    if (profile && warp == 0 && lane == 0) {    \
        const long long _t = clock64(); \
        ctl.ph[i] += _t - ph_t;         \
        ph_t = _t;                      \
    }

template <int NW>
struct TabuCtrl {
    long long it, conflicts, best, nlog, sum_c, sum_deg, diag;
    unsigned long long ctr;
    long long s0, s1;
    int C, work, ovf, mv_v, mv_a, mv_b, gvb;
    long long red[NW];
    int wcnt[NW];
    int bmin[NW], bD[NW], bsum[NW], bfirst[NW];  // pass 2a per-warp block results
    long long ph[10];
};

// Candidate row of one conflicting vertex v.  Candidates are gamma values g
// (delta = g - gva); excluded: c == a, and live tabu colours without
// aspiration (g - gva < thr  <=>  g < A).  KQ = 64-colour words of the
// exclusion mask (1 when k <= 64).
template <typename G, typename S, int KQ>
struct RowEval {
    static constexpr bool NARROW = sizeof(G) == 1;
    const G *g;
    const uint32_t *lut;  // nibble -> byte mask (shared)
    int a, gva, k, kp, rot;
    uint64_t ex[KQ];

    // physical word of logical word w (rows are rotated by `rot` words so that
    // rows sharing a bank offset land on different banks)
    __device__ __forceinline__ int wp(int w) const {
        const int p = w + rot, W = kp >> 2;
        return p >= W ? p - W : p;
    }
    // gamma value of colour c
    __device__ __forceinline__ int gv(int c) const {
        if constexpr (NARROW)
            return reinterpret_cast<const uint8_t *>(g)[4 * wp(c >> 2) + (c & 3)];
        else
            return g[c];
    }

    __device__ __forceinline__ void setbit(int c) {
        const uint64_t b = 1ull << (c & 63);
        if constexpr (KQ == 1) {
            ex[0] |= b;
        } else {
#pragma unroll
            for (int q = 0; q < KQ; q++)
                if ((c >> 6) == q) ex[q] |= b;
        }
    }
    __device__ __forceinline__ uint64_t exq(int q) const {
        if constexpr (KQ == 1) {
            return ex[0];
        } else {
            uint64_t r = ex[0];
#pragma unroll
            for (int j = 1; j < KQ; j++)
                if (q == j) r = ex[j];
            return r;
        }
    }
    __device__ __forceinline__ bool excluded(int c) const { return (exq(c >> 6) >> (c & 63)) & 1ull; }
    // word w of the row with excluded colours forced to 0xFF (narrow path)
    __device__ __forceinline__ uint32_t word(int w) const {
        return reinterpret_cast<const uint32_t *>(g)[wp(w)] |
               lut[(uint32_t)(exq(w >> 4) >> (4 * (w & 15))) & 0xFu];
    }

    __device__ __forceinline__ void init(const G *gamma, const S *texp, const uint8_t *tcol,
                                         const S *tovf, const S *gstamp, const uint8_t *assign, int v,
                                         int kp_, int k_, uint32_t it, int thr, const uint32_t *lut_,
                                         int swz_rs, int swz_rm) {
        lut = lut_;
        kp = kp_;
        k = k_;
        rot = (v >> swz_rs) & swz_rm;
        a = assign[v];
        g = gamma + (size_t)v * kp;
        gva = gv(a);
        const int A = thr + gva;
#pragma unroll
        for (int q = 0; q < KQ; q++) ex[q] = 0;
        setbit(a);
        const uint32_t cols = reinterpret_cast<const uint32_t *>(tcol)[v];
        if (cols != 0xFFFFFFFFu) {
            S e[4];
            if constexpr (sizeof(S) == 2) {
                const uint2 x = reinterpret_cast<const uint2 *>(texp)[v];
                e[0] = (S)x.x;
                e[1] = (S)(x.x >> 16);
                e[2] = (S)x.y;
                e[3] = (S)(x.y >> 16);
            } else {
                const uint4 x = reinterpret_cast<const uint4 *>(texp)[v];
                e[0] = x.x;
                e[1] = x.y;
                e[2] = x.z;
                e[3] = x.w;
            }
#pragma unroll
            for (int s = 0; s < 4; s++) {
                const int c = (cols >> (8 * s)) & 0xFF;
                if (c != 0xFF && active<S>(e[s], it) && !(gv(c) < A)) setbit(c);
            }
        }
        if (active<S>(tovf[v], it)) spill_scan(gstamp + (size_t)v * kp, it, A);
    }
    // spilled expiries: dense global row (rare; kept out of the hot code)
    __device__ __forceinline__ void spill_scan(const S *gs, uint32_t it, int A) {
        for (int c = 0; c < k; c++)
            if (active<S>(gs[c], it) && !(gv(c) < A)) setbit(c);
    }

    // (row minimum delta or TC_BIG, #admissible candidates at the minimum)
    __device__ __forceinline__ void min_count(int &rmin, int &cnt) const {
        if constexpr (NARROW && KQ == 1) {
            // k <= 64: one pass, byte minima as 16x2 lanes (even bytes, odd bytes
            // via PRMT) and the count of bytes at the running minimum
            const int W = kp >> 2;
            const uint32_t *g32 = reinterpret_cast<const uint32_t *>(g);
            uint64_t exm = ex[0];
            int m = 0xFF, c = 0, p = rot;
#pragma unroll 2
            for (int w = 0; w < W; w++) {
                const uint32_t x = g32[p] | lut[(uint32_t)exm & 0xFu];
                exm >>= 4;
                p = (p + 1 == W) ? 0 : p + 1;
                const uint32_t m2 = __vminu2(x & 0x00FF00FFu, __byte_perm(x, 0, 0x4341));
                const int wm = (int)min(m2 & 0xFFFFu, m2 >> 16);
                const int wc = count_eq_bytes(x, (uint32_t)wm);
                c = (wm < m) ? wc : (wm == m ? c + wc : c);
                m = min(m, wm);
            }
            rmin = (m == 0xFF) ? TC_BIG : m - gva;
            cnt = (m == 0xFF) ? 0 : c;
        } else if constexpr (NARROW) {
            const int W = kp >> 2;
            int m = 0xFF, c = 0;
            // 16 words in flight: with gamma in L2 a row is a few round trips,
            // not one per 4 words
#pragma unroll 16
            for (int w = 0; w < W; w++) {
                const uint32_t x = word(w);
                const int wm = (int)min_bytes(x);
                const int wc = count_eq_bytes(x, (uint32_t)wm);
                c = (wm < m) ? wc : (wm == m ? c + wc : c);
                m = min(m, wm);
            }
            rmin = (m == 0xFF) ? TC_BIG : m - gva;
            cnt = (m == 0xFF) ? 0 : c;
        } else {
            int m = INT_MAX, c = 0;
            for (int cc = 0; cc < k; cc++) {
                if (excluded(cc)) continue;
                const int b = gv(cc);
                if (b < m) {
                    m = b;
                    c = 1;
                } else if (b == m) {
                    c++;
                }
            }
            rmin = (m == INT_MAX) ? TC_BIG : m - gva;
            cnt = (m == INT_MAX) ? 0 : c;
        }
    }

    // Exact sequential tie count of the row entered with running minimum R,
    // warp-cooperative (all 32 lanes, same row): lane = word (narrow) or
    // colour (wide); an exclusive prefix-min over the units gives each lane the
    // running minimum entering its unit, then each lane walks its <= 4 bytes.
    __device__ __forceinline__ int warp_walk_ties(int R, int lane) const {
        constexpr unsigned FULL = 0xffffffffu;
        constexpr int NONE = NARROW ? 0xFF : INT_MAX - 1;
        const int units = NARROW ? (kp >> 2) : k;
        int carry = (R >= TC_BIG) ? INT_MAX : R + gva;  // g-space
        int t = 0;
        for (int u0 = 0; u0 < units; u0 += 32) {
            const int u = u0 + lane;
            uint32_t x = 0xFFFFFFFFu;
            int um = NONE;
            if (u < units) {
                if constexpr (NARROW) {
                    x = word(u);
                    um = (int)min_bytes(x);
                } else {
                    um = excluded(u) ? NONE : gv(u);
                }
            }
            const int incl = warp_incl_min(um, lane);
            int excl = __shfl_up_sync(FULL, incl, 1);
            if (lane == 0) excl = INT_MAX;
            int cur = min(carry, excl);
            if constexpr (NARROW) {
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const int b = (x >> (8 * e)) & 0xFF;
                    if (b == 0xFF) continue;
                    if (b < cur) cur = b;
                    else if (b == cur) t++;
                }
            } else {
                if (um != NONE && um == cur) t++;
            }
            carry = min(carry, __shfl_sync(FULL, incl, 31));
        }
        return __reduce_add_sync(FULL, t);
    }
};

template <typename G, typename S, bool GSM, int KQ, int NT>
__global__ void __launch_bounds__(NT, (GSM && sizeof(G) == 1) ? 6 : 1) tabucol_kernel(TabuParams P) {
    constexpr int NW = NT / 32;
    constexpr bool NARROW = sizeof(G) == 1;
    constexpr int GMAX = NARROW ? 254 : 65534;
    constexpr uint32_t SWEEP = sizeof(S) == 2 ? 16384u : (1u << 30);
    constexpr unsigned FULL = 0xffffffffu;
    using RE = RowEval<G, S, KQ>;

    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ TabuCtrl<NW> ctl;
    __shared__ uint32_t s_nib[16];
    if (threadIdx.x < 16) s_nib[threadIdx.x] = expand_nibble(threadIdx.x);

    const int n = P.n, k = P.k, kp = P.kp;
    size_t off = 0;
    G *gamma;
    if constexpr (GSM) {
        gamma = reinterpret_cast<G *>(smem + off);
        off += ((size_t)n * kp * sizeof(G) + 15) & ~(size_t)15;
    } else {
        gamma = reinterpret_cast<G *>(P.ws_gamma + blockIdx.x * P.ws_g_stride);
    }
    S *texp = reinterpret_cast<S *>(smem + off);
    off += ((size_t)n * 4 * sizeof(S) + 15) & ~(size_t)15;
    uint8_t *tcol = smem + off;
    off += ((size_t)n * 4 + 15) & ~(size_t)15;
    S *tovf = reinterpret_cast<S *>(smem + off);
    off += ((size_t)n * sizeof(S) + 15) & ~(size_t)15;
    uint8_t *assign = smem + off;
    off += (n + 15) & ~15;
    uint16_t *clist = reinterpret_cast<uint16_t *>(smem + off);
    off += (2 * n + 15) & ~15;
    uint16_t *cpos = reinterpret_cast<uint16_t *>(smem + off);
    off += (2 * n + 15) & ~15;
    using Rec = typename RecT<NARROW>::T;
    Rec *rmc = reinterpret_cast<Rec *>(smem + off);  // per row: (min delta, count)
    off += (sizeof(Rec) * n + 15) & ~(size_t)15;
    uint16_t *nbs = reinterpret_cast<uint16_t *>(smem + off);  // staged N(v)
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint32_t *evm = reinterpret_cast<uint32_t *>(smem + off);  // event ballots per 32 neighbours
    S *gstamp = reinterpret_cast<S *>(P.ws_stamp + blockIdx.x * P.ws_s_stride);

    const int tid = threadIdx.x, lane = tid & 31, hw_warp = tid >> 5;
    // The serial part of every iteration runs on one "master" warp.  Warp slot
    // w of an SM issues from sub-partition w % 4, so CTAs resident on the same
    // SM take their master round-robin from a per-SM ticket: the serial chains
    // spread over the 4 schedulers instead of all landing on one.
    if (tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        ctl.work = P.sm_ticket ? atomicAdd(P.sm_ticket + (smid & 255), 1) : 0;
    }
    __syncthreads();
    const int master = ctl.work % NW;
    const int warp = ((tid >> 5) - master + NW) % NW;  // warp 0 = this CTA's master
    __syncthreads();
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool profile = (P.flags & MCB_FLAG_PROFILE) != 0;
    const bool cidx = P.const_indptr != 0;
    const int Wq = kp >> 2, swz_rs = P.swz_rs, swz_rm = P.swz_rm;
    // element offset of (vertex, colour) in gamma, rows rotated by rot(v) words
    auto goff = [=](int v, int c) -> size_t {
        if constexpr (NARROW) {
            int p = (c >> 2) + ((v >> swz_rs) & swz_rm);
            if (p >= Wq) p -= Wq;
            return (size_t)v * kp + 4 * p + (c & 3);
        } else {
            return (size_t)v * kp + c;
        }
    };
    const int64_t *indptr_g = P.indptr;
    auto row_begin = [=](int v) -> int64_t { return cidx ? (int64_t)c_indptr[v] : indptr_g[v]; };

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
            reinterpret_cast<uint32_t *>(tcol)[v] = 0xFFFFFFFFu;
            tovf[v] = (S)0;
        }
        {
            // gamma rows: real colours 0, padding colours all-ones (never a candidate)
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gamma);
            const int wpr = kp * (int)sizeof(G) / 4;  // words per row
            const uint32_t padw = NARROW ? ((k & 3) ? (0xFFFFFFFFu << (8 * (k & 3))) : 0u)
                                         : ((k & 1) ? 0xFFFF0000u : 0u);
            for (int i = tid; i < n * wpr; i += NT) {
                const int v = i / wpr, w = i - v * wpr;  // physical word w of row v
                int lw = w - (NARROW ? ((v >> P.swz_rs) & P.swz_rm) : 0);
                if (lw < 0) lw += wpr;
                g32[i] = (lw == wpr - 1) ? padw : 0u;
            }
        }
        if (tid == 0) {
            ctl.ovf = 0;
            ctl.diag = 0;
            for (int q = 0; q < 10; q++) ctl.ph[q] = 0;
        }
        __syncthreads();
        // gamma[u][c] = #neighbours of u coloured c; each thread owns its rows
        {
            int bad = 0;
            for (int u = tid; u < n; u += NT) {
                const int64_t s0 = row_begin(u), s1 = row_begin(u + 1);
                for (int64_t idx = s0; idx < s1; idx++) {
                    const int c = assign[__ldg(P.indices + idx)];
                    G *e = gamma + goff(u, c);
                    const int x = (int)*e + 1;
                    if (x > GMAX) bad = 1;
                    else *e = (G)x;
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
                    const int gv = gamma[goff(v, assign[v])];
                    f = gv > 0;
                    c2 += gv;
                }
                const unsigned bal = __ballot_sync(FULL, f);
                if (lane == 0) ctl.wcnt[hw_warp] = __popc(bal);
                __syncthreads();
                int woff = 0, tot = 0;
#pragma unroll
                for (int j = 0; j < NW; j++) {
                    const int cj = ctl.wcnt[j];
                    woff += (j < hw_warp) ? cj : 0;
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
            if (lane == 0) ctl.red[hw_warp] = c2;
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

                // pass 1: (min, count) of every conflicting row, one row per thread
                for (int li = tid; li < C; li += NT) {
                    RE re;
                    re.init(gamma, texp, tcol, tovf, gstamp, assign, clist[li], kp, k, it32, thr, s_nib, swz_rs, swz_rm);
                    int rm, cnt;
                    re.min_count(rm, cnt);
                    rmc[li] = rec_pack(rm, cnt, (Rec *)nullptr);
                }
                __syncthreads();
                PH(1);
                // pass 2a (all warps): exclusive prefix-min over per-warp contiguous
                // blocks of rows -- block minima first, then every block scanned
                // from its entering running minimum.  Rows above it hold no tie
                // event, rows equal to it hold #min of them, rows below it (few)
                // are walked by the block's warp.
                const int BS = (C + NW - 1) / NW;
                const int b0 = min(C, warp * BS), b1 = min(C, b0 + BS);
                {
                    int bm = TC_BIG;
                    for (int q = b0 + lane; q < b1; q += 32) bm = min(bm, rec_unpack(rmc[q]).x);
                    bm = __reduce_min_sync(FULL, bm);
                    if (lane == 0) ctl.bmin[warp] = bm;
                }
                __syncthreads();
                {
                    const int binc = warp_incl_min(lane < NW ? ctl.bmin[lane] : TC_BIG, lane);
                    const int Dg = __shfl_sync(FULL, binc, 31);
                    int carry = warp == 0 ? TC_BIG : __shfl_sync(FULL, binc, warp - 1);
                    int tsum = 0, dc = 0, first = INT_MAX;
                    for (int q0 = b0; q0 < b1; q0 += 32) {
                        const int q = q0 + lane;
                        const int2 mc = q < b1 ? rec_unpack(rmc[q]) : make_int2(TC_BIG, 0);
                        const int x = mc.x;
                        const int incl = warp_incl_min(x, lane);
                        int excl = __shfl_up_sync(FULL, incl, 1);
                        if (lane == 0) excl = TC_BIG;
                        const int RM = min(carry, excl);
                        bool low = false;
                        if (!prod && x != TC_BIG) {
                            if (x == RM) tsum += mc.y;
                            else if (x < RM) low = true;
                        }
                        if (x == Dg && x != TC_BIG) {
                            dc += mc.y;
                            first = min(first, q);
                        }
                        for (unsigned wm = __ballot_sync(FULL, low); wm; wm &= wm - 1) {
                            const int src = __ffs(wm) - 1;
                            const int Rs = __shfl_sync(FULL, RM, src);
                            RE re;
                            re.init(gamma, texp, tcol, tovf, gstamp, assign, clist[q0 + src], kp, k, it32, thr, s_nib,
                                    swz_rs, swz_rm);
                            const int t = re.warp_walk_ties(Rs, lane);
                            if (lane == 0) tsum += t;
                        }
                        carry = min(carry, __shfl_sync(FULL, incl, 31));
                    }
                    tsum = __reduce_add_sync(FULL, tsum);
                    dc = __reduce_add_sync(FULL, dc);
                    first = (int)__reduce_min_sync(FULL, (unsigned)first);
                    if (lane == 0) {
                        ctl.bsum[warp] = tsum;
                        ctl.bD[warp] = dc;
                        ctl.bfirst[warp] = first;
                    }
                }
                __syncthreads();
                PH(2);

                // pass 2b (warp 0): reservoir, move, gamma update, conflict list
                if (warp == 0) {
                    const int D = __reduce_min_sync(FULL, lane < NW ? ctl.bmin[lane] : TC_BIG);
                    int mv_v = -1, mv_a = 0, mv_b = 0, gvb = 0;
                    int64_t s0 = 0, s1 = 0;
                    constexpr int NB = 8;  // neighbour chunks of 32 held in registers
                    int uu[NB];
                    if (D != TC_BIG) {
                        const int T = __reduce_add_sync(FULL, lane < NW ? ctl.bD[lane] : 0);
                        const int L = (int)__reduce_min_sync(FULL, (unsigned)(lane < NW ? ctl.bfirst[lane] : INT_MAX));
                        const int total = __reduce_add_sync(FULL, lane < NW ? ctl.bsum[lane] : 0);
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
                        if (sstar > 1) {  // rank sstar among the D-candidates in scan order:
                            // its block from the per-warp counts, then the row in the block
                            const int cj = lane < NW ? ctl.bD[lane] : 0;
                            const int cin = warp_incl_sum(cj, lane);
                            const int wb = __ffs(__ballot_sync(FULL, cin >= sstar)) - 1;
                            int nd = sstar - __shfl_sync(FULL, cin - cj, wb);
                            const int r0 = min(C, wb * BS), r1 = min(C, r0 + BS);
                            for (int base = r0; base < r1; base += 32) {
                                const int li = base + lane;
                                int c = 0;
                                if (li < r1) {
                                    const int2 mc = rec_unpack(rmc[li]);
                                    c = (mc.x == D) ? mc.y : 0;
                                }
                                const int incl = warp_incl_sum(c, lane);
                                const int tot = __shfl_sync(FULL, incl, 31);
                                if (tot >= nd) {
                                    const unsigned bm = __ballot_sync(FULL, incl >= nd);
                                    const int src = __ffs(bm) - 1;
                                    row_li = base + src;
                                    need = nd - __shfl_sync(FULL, incl - c, src);
                                    break;
                                }
                                nd -= tot;
                            }
                        }
                        // the winner's vertex is known: start its adjacency loads now so
                        // they overlap the in-row locate and the tenure/slot bookkeeping
                        const int v = clist[row_li];
                        {
                            const int64_t g0 = row_begin(v), g1 = row_begin(v + 1);
#pragma unroll
                            for (int j = 0; j < NB; j++) {
                                const int64_t idx = g0 + j * 32 + lane;
                                uu[j] = idx < g1 ? __ldg(P.indices + idx) : 0;
                            }
                        }
                        // locate the need-th D-candidate of the row (lanes over words)
                        RE re;
                        re.init(gamma, texp, tcol, tovf, gstamp, assign, v, kp, k, it32, thr, s_nib, swz_rs, swz_rm);
                        int b = -1;
                        {
                            const int Dg = D + re.gva;
                            const int units = NARROW ? (kp >> 2) : k;
                            int cum = 0;
                            for (int u0 = 0; u0 < units && b < 0; u0 += 32) {
                                const int u = u0 + lane;
                                int c = 0;
                                uint32_t x = 0;
                                if (u < units) {
                                    if constexpr (NARROW) {
                                        const uint64_t m64 = re.exq(u >> 4);
                                        x = reinterpret_cast<const uint32_t *>(re.g)[re.wp(u)] |
                                            expand_nibble((uint32_t)(m64 >> (4 * (u & 15))) & 0xFu);
                                        c = count_eq_bytes(x, (uint32_t)Dg);
                                    } else {
                                        c = (!re.excluded(u) && re.gv(u) == Dg) ? 1 : 0;
                                    }
                                }
                                const int incl = warp_incl_sum(c, lane);
                                const int tot = __shfl_sync(FULL, incl, 31);
                                if (cum + tot >= need) {
                                    const unsigned bm = __ballot_sync(FULL, cum + incl >= need);
                                    const int src = __ffs(bm) - 1;
                                    int r = need - cum - (incl - c);  // rank inside the unit
                                    int col = -1;
                                    if (lane == src) {
                                        if constexpr (NARROW) {
#pragma unroll
                                            for (int e = 0; e < 4; e++)
                                                if ((int)((x >> (8 * e)) & 0xFF) == Dg && --r == 0 && col < 0)
                                                    col = 4 * u + e;
                                        } else {
                                            col = u;
                                        }
                                    }
                                    b = __shfl_sync(FULL, col, src);
                                }
                                cum += tot;
                            }
                        }
                        PH(4);
                        if (lane == 0) {
                            const int a = re.a;
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
                            // tabu (v, a) until it + tt + 1: slot hit, free slot, or spill
                            const S e_new = (S)(uint32_t)(it + tt + 1);
                            const uint32_t cols = reinterpret_cast<const uint32_t *>(tcol)[v];
                            int s_hit = -1, s_free = -1;
#pragma unroll
                            for (int s = 0; s < 4; s++) {
                                const int cs = (cols >> (8 * s)) & 0xFF;
                                if (cs == a) s_hit = s;
                                else if (s_free < 0 && (cs == 0xFF || !active<S>(texp[4 * v + s], it32)))
                                    s_free = s;
                            }
                            const int s = s_hit >= 0 ? s_hit : s_free;
                            const bool ovf_live = active<S>(tovf[v], it32);
                            if (s >= 0) {
                                tcol[4 * v + s] = (uint8_t)a;
                                texp[4 * v + s] = e_new;
                                if (ovf_live) gstamp[(size_t)v * kp + a] = (S)it32;  // supersede
                            } else {
                                spill_set(gstamp + (size_t)v * kp, tovf + v, ovf_live, k, a, e_new, it32);
                            }
                            gvb = re.gv(b < 0 ? 0 : b);
                            assign[v] = (uint8_t)(b < 0 ? a : b);
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
                            mv_b = b < 0 ? a : b;
                        }
                        mv_v = __shfl_sync(FULL, mv_v, 0);
                        mv_a = __shfl_sync(FULL, mv_a, 0);
                        mv_b = __shfl_sync(FULL, mv_b, 0);
                        s0 = __shfl_sync(FULL, s0, 0);
                        s1 = __shfl_sync(FULL, s1, 0);
                    }
                    PH(5);
                    // publish the move and stage the (prefetched) adjacency of v
                    if (lane == 0) {
                        ctl.mv_v = mv_v;
                        ctl.mv_a = mv_a;
                        ctl.mv_b = mv_b;
                        ctl.gvb = gvb;
                        ctl.s0 = s0;
                        ctl.s1 = s1;
                    }
                    if (mv_v >= 0) {
#pragma unroll
                        for (int j = 0; j < NB; j++)
                            if (s0 + j * 32 + lane < s1) nbs[j * 32 + lane] = (uint16_t)uu[j];
                    }
                }
                __syncthreads();
                // all warps: gamma update over N(v) (:356-359), one neighbour per
                // thread; each warp publishes the ballot of conflict-set events of
                // its 32 consecutive neighbours
                const int mvv = ctl.mv_v;
                if (mvv >= 0) {
                    const int ma = ctl.mv_a, mb = ctl.mv_b;
                    const int64_t s0 = ctl.s0;
                    const int deg = (int)(ctl.s1 - s0);
                    bool bad = false;
                    for (int j0 = 0; j0 < deg; j0 += NT) {
                        const int j = j0 + tid;
                        bool evt = false;
                        if (j < deg) {
                            int u;
                            if (j < 32 * 8) {
                                u = nbs[j];
                            } else {
                                u = __ldg(P.indices + s0 + j);
                                nbs[j] = (uint16_t)u;
                            }
                            G *pa = gamma + goff(u, ma);
                            G *pb = gamma + goff(u, mb);
                            const int ga = (int)*pa - 1;
                            *pa = (G)ga;
                            const int gb = *pb;
                            if (gb >= GMAX) bad = true;
                            else *pb = (G)(gb + 1);
                            const int au = assign[u];
                            evt = (au == ma && ga == 0) || (au == mb && gb == 0);
                        }
                        const unsigned em = __ballot_sync(FULL, evt);
                        if (lane == 0) evm[(j0 >> 5) + hw_warp] = em;
                    }
                    if (bad) ctl.ovf = 1;
                }
                __syncthreads();
                PH(6);
                // master: conflict-list events in neighbour order (:368-385), then v
                if (warp == 0) {
                    if (mvv >= 0) {
                        bool improved = false;
                        if (lane == 0) {
                            int Cn = C;
                            const int deg = (int)(ctl.s1 - ctl.s0);
                            for (int c = 0; c * 32 < deg; c++) {
                                unsigned e = evm[c];
                                while (e) {
                                    const int bit = __ffs(e) - 1;
                                    e &= e - 1u;
                                    const int u = nbs[c * 32 + bit];
                                    cl_apply(clist, cpos, Cn, u, cpos[u] == 0xFFFF);  // enter iff outside
                                }
                            }
                            cl_apply(clist, cpos, Cn, mvv, ctl.gvb > 0);
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
                    if (lane == 0) ctl.red[hw_warp] = c2;
                }
                if (swp) {  // keep 16-bit expiries unambiguous
                    const uint32_t itw = (uint32_t)itn;
                    for (int v = tid; v < n; v += NT) {
                        for (int s = 0; s < 4; s++)
                            if (!active<S>(texp[4 * v + s], itw)) tcol[4 * v + s] = 0xFF;
                        if (active<S>(tovf[v], itw)) {
                            S *gs = gstamp + (size_t)v * kp;
                            for (int c = 0; c < k; c++)
                                if (!active<S>(gs[c], itw)) gs[c] = (S)itw;
                        } else {
                            tovf[v] = (S)itw;
                        }
                    }
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
        if (profile && warp == 0 && lane == 0) {
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
template <typename S>
static size_t misc_bytes(int n, int nt) {
    auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    const size_t rec = sizeof(S) == 2 ? 4 : 8;
    return a16((size_t)n * 4 * sizeof(S)) + a16((size_t)n * 4) + a16((size_t)n * sizeof(S)) +
           a16(n) + 2 * a16(2 * (size_t)n) + a16(rec * (size_t)n) +
           a16(2 * (size_t)n) + a16(4 * (size_t)((n + 31) / 32));
}

template <typename G, typename S, bool GSM>
static size_t smem_bytes(int n, int kp) {
    size_t s = misc_bytes<S>(n, TC_NT);
    if (GSM) s += ((size_t)n * kp * sizeof(G) + 15) & ~(size_t)15;
    return s;
}

// threads per individual (gamma-in-L2 shapes): 256 when every individual is
// resident at 256 threads (pass 1's conflicting rows, read from L2, spread
// over twice the lanes; config 4 at its 256 individuals per GPU: 3.6e6 -> 5.7e6
// moves/s), else 128 so that more individuals are resident.  With gamma in
// shared memory 128 measured slightly better (C3 shape).  MCB_TC_NT overrides.
static int pick_nt(int slots256, int p_hint) {
    if (const char *e = getenv("MCB_TC_NT")) {
        const int v = atoi(e);
        if (v == 128 || v == 256) return v;
    }
    return p_hint <= slots256 ? 256 : TC_NT;
}

template <typename G, typename S, bool GSM, int NT>
static auto kernel_for(int kp) {
    return (GSM && kp <= 64) ? tabucol_kernel<G, S, GSM, 1, NT> : tabucol_kernel<G, S, GSM, 4, NT>;
}

template <typename G, typename S, bool GSM>
static int launch_variant(TabuParams P, int max_grid, int p_hint, cudaStream_t st, int *grid_out,
                          bool query_only) {
    const size_t smem = smem_bytes<G, S, GSM>(P.n, P.kp);
    int nt = TC_NT;
    auto kern = kernel_for<G, S, GSM, TC_NT>(P.kp);
    if constexpr (sizeof(S) == 2 && !GSM) {  // narrow pass, gamma in L2 (the L2 latency is what more lanes hide)
        auto k256 = kernel_for<G, S, GSM, 256>(P.kp);
        int nb256 = 0;
        if (cudaFuncSetAttribute(k256, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb256, k256, 256, smem) == cudaSuccess && nb256 > 0 &&
            pick_nt(nb256 * num_sms(), p_hint) == 256) {
            nt = 256;
            kern = k256;
        }
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "cudaFuncSetAttribute(smem=%zu) failed", smem);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, nt, smem) != cudaSuccess || nb < 1)
        return set_error(MCB_ERR_CUDA, "tabucol: no occupancy for smem=%zu", smem);
    int grid = std::min(p_hint, nb * num_sms());
    if (max_grid > 0) grid = std::min(grid, max_grid);
    grid = std::max(grid, 1);
    *grid_out = grid;
    if (query_only) return MCB_OK;
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] tabucol<%s,%s,gsm=%d,kq=%d,nt=%d> grid=%d (%d/SM) smem=%zu\n",
                sizeof(G) == 1 ? "u8" : "u16", sizeof(S) == 2 ? "u16" : "u32", (int)GSM,
                (GSM && P.kp <= 64) ? 1 : 4, nt, grid, nb, smem);
    kern<<<grid, nt, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol launch failed");
    return MCB_OK;
}

static bool fits_smem(size_t bytes) { return bytes <= (size_t)max_smem_optin(); }

int tabucol_phase_cycles(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "phase counters unavailable");
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
    }
    return tabucol_cluster_phase_cycles(out, reset);  // added in: a run uses one of the two kernels
}

static const int32_t *&async_err_slot(cudaStream_t st) {
    static std::map<std::pair<int, void *>, const int32_t *> slots;
    int d = 0;
    cudaGetDevice(&d);
    return slots[std::make_pair(d, (void *)st)];
}

int tabucol_async_status(cudaStream_t st) {
    const int32_t *e = async_err_slot(st);
    if (!e) return MCB_OK;
    int32_t h = 0;
    if (cudaMemcpyAsync(&h, e, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol: kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (h == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
    if (h == 2) return set_error(MCB_ERR_UNSUPPORTED, "tabucol: wide tables overflowed");
    return MCB_OK;
}

// 0: narrow, gamma in smem (warp / group kernels first); 1: narrow, gamma in
// global (L2) slices; 2: wide only; 3: narrow, gamma split over a 2-CTA
// cluster's shared memory (tabucol_cluster.cu) -- the default where one
// SM's shared memory cannot hold the table (MCB_NO_CLUSTER=1: variant 1)
static int tabucol_variant(int n, int k, uint32_t flags) {
    const int kp = (k + 3) & ~3;
    if (flags & MCB_FLAG_FORCE_WIDE) return 2;
    if (flags & MCB_FLAG_FORCE_CLUSTER) return 3;
    if (flags & MCB_FLAG_FORCE_GLOBAL) return 1;
    if (fits_smem(smem_bytes<uint8_t, uint16_t, true>(n, kp))) return 0;
    if (!getenv("MCB_NO_CLUSTER") && fits_smem(tabucol_cluster_smem(n, k))) return 3;
    return 1;
}

int tabucol_cta_describe(int64_t n, int64_t k, int64_t p, char *buf, int len) {
    const int v = tabucol_variant((int)n, (int)k, 0);
    if (v == 3)
        snprintf(buf, len, "tabucol_cluster_kernel (2-CTA cluster per individual, %zu B smem per CTA)",
                 tabucol_cluster_smem((int)n, (int)k));
    else
        snprintf(buf, len, "tabucol_kernel (CTA per individual; gamma in %s)", v == 0 ? "shared memory" : "L2");
    (void)p;
    return MCB_OK;
}

int tabucol_run(const TabucolArgs &A, cudaStream_t st) {
    if (A.p < 0 || A.n < 1 || A.k < 1 || A.depth < 0 || A.m < 0)
        return set_error(MCB_ERR_VALUE, "tabucol: bad shape p=%lld n=%lld k=%lld depth=%lld",
                         (long long)A.p, (long long)A.n, (long long)A.k, (long long)A.depth);
    if (A.n > 32767 || A.k > 255)
        return set_error(MCB_ERR_UNSUPPORTED, "tabucol: n<=32767 and k<=255 required");
    if (A.p == 0) return MCB_OK;
    // MCB_FLAG_ASYNC: no host synchronisation at all -- per-stream scratch, the
    // fallback passes always enqueued with device-side work counts, errors left
    // in the device word mcb_tabucol_async_status reads (graph-capturable)
    const bool async = (A.flags & MCB_FLAG_ASYNC) != 0;
    std::unique_ptr<WsStreamKey> wskey(async ? new WsStreamKey(st) : nullptr);
    const int n = (int)A.n, k = (int)A.k, kp = (k + 3) & ~3;
    // every shape must be able to fall back to the wide CTA pass, whose
    // per-vertex state (u32 expiries, scan records, lists) lives in shared
    // memory: ~39 B per vertex -> n <= ~5900 on B200
    if (smem_bytes<uint16_t, uint32_t, false>(n, kp) > (size_t)max_smem_optin())
        return set_error(MCB_ERR_UNSUPPORTED, "tabucol: n=%d needs %zu B of per-vertex shared state (max %d B)", n,
                         smem_bytes<uint16_t, uint32_t, false>(n, kp), max_smem_optin());

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
    {
        // rows of W words: bank base (v*W) mod 32 repeats every Pd = 32/g rows
        // with g = gcd(W, 32); rotating row v by (v / Pd) mod g words fills the gaps
        const int W = kp / 4;
        int g = 1;
        while (g < 32 && W % (2 * g) == 0) g *= 2;
        int pd = 32 / g, rs = 0;
        while ((1 << rs) < pd) rs++;
        P.swz_rs = rs;
        P.swz_rm = g - 1;
        if (!getenv("MCB_SWIZZLE")) P.swz_rm = 0;  // measured: no gain at k=48 (latency-bound)
    }

    const int variant = tabucol_variant(n, k, A.flags);

    const size_t tab = (size_t)n * kp;
    const int grid_cap = 16 * num_sms();
    // control words, per-SM tickets, overflow list of the warp pass, overflow
    // list of its spill pass
    const size_t ctl_bytes = 256 + 1024 + 2 * sizeof(int32_t) * (size_t)A.p;
    const size_t ng_stride = (tab + 255) & ~(size_t)255, ns_stride = (tab * 2 + 255) & ~(size_t)255;
    const size_t wg_stride = (tab * 2 + 255) & ~(size_t)255, ws_stride = (tab * 4 + 255) & ~(size_t)255;
    const int wide_grid = std::min<int>((int)A.p, 2 * num_sms());
    const size_t indptr_bytes = 4 * (size_t)(n + 1);

    int grid = 1, rc;
    size_t narrow_ws = 0;
    const size_t cl_stride = tabucol_cluster_stamp_stride(n, k);
    if (variant == 3) {
        rc = tabucol_cluster_launch(P, (int)A.p, st, &grid, true);
        if (rc) return rc;
        narrow_ws = (size_t)grid * cl_stride;
    } else if (variant != 2) {
        rc = variant == 0
                 ? launch_variant<uint8_t, uint16_t, true>(P, grid_cap, (int)A.p, st, &grid, true)
                 : launch_variant<uint8_t, uint16_t, false>(P, grid_cap, (int)A.p, st, &grid, true);
        if (rc) return rc;
        narrow_ws = (size_t)grid * (ns_stride + (variant == 1 ? ng_stride : 0));
    }
    const size_t wide_ws = (size_t)wide_grid * (wg_stride + ws_stride);
    const size_t tables_off = (ctl_bytes + 255) & ~(size_t)255;
    const size_t indptr_off = tables_off + ((narrow_ws + wide_ws + 255) & ~(size_t)255);
    uint8_t *ws = (uint8_t *)workspace(indptr_off + indptr_bytes + 256);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol: workspace allocation failed");
    int32_t *ctl32 = reinterpret_cast<int32_t *>(ws);  // [0]=work(narrow) [1]=work(wide) [2]=ovf_count [3]=err
    if (cudaMemsetAsync(ws, 0, 256 + 1024, st) != cudaSuccess) return set_error(MCB_ERR_CUDA, "memset failed");
    P.err_flag = ctl32 + 3;
    P.sm_ticket = ctl32 + 64;  // 256 per-SM counters
    uint8_t *tables = ws + tables_off;

    // fast path: one individual per warp (tabucol_warp.cu).  Individuals whose
    // tabu list outgrows the 1024-entry register ring re-run on the SPILL
    // variant (ring continued in global memory); what still overflows (gamma
    // > 63, tenure >= 8190) lands on the list the wide pass below consumes,
    // which is launched only when that list is not empty
    bool warp_done = false;
    int32_t *ovf_warp = ctl32 + 64 + 256, *ovf_spill = ovf_warp + A.p;
    int32_t *ovf_final = ovf_warp, *ovf_final_count = ctl32 + 2;
    if (variant == 0) {
        // group of warps per individual first (tabucol_group.cu), else one warp
        rc = tabucol_group_launch(A, st, ctl32 + 0, ovf_warp, ctl32 + 2, ctl32 + 3);
        if (rc < 0) rc = tabucol_warp_launch(A, st, ctl32 + 0, ovf_warp, ctl32 + 2, ctl32 + 3);
        if (rc > 0) return rc;
        warp_done = rc == MCB_OK;
    }
    if (warp_done && async) {
        // the SPILL pass over the warp pass's overflow list, then the wide pass
        // over the SPILL pass's list, both sized for the worst case
        rc = tabucol_warp_launch(A, st, ctl32 + 4, ovf_spill, ctl32 + 5, ctl32 + 3, ovf_warp, A.p, true,
                                 ctl32 + 2);
        if (rc > 0) return rc;
        ovf_final = rc == MCB_OK ? ovf_spill : ovf_warp;
        ovf_final_count = rc == MCB_OK ? ctl32 + 5 : ctl32 + 2;
    } else if (warp_done) {
        int32_t h[2] = {0, 0};  // [0] = overflowed individuals, [1] = error flag
        if (cudaMemcpyAsync(h, ctl32 + 2, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "tabucol: kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
        if (h[1] == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
        if (h[0] == 0) return MCB_OK;
        if (!getenv("MCB_NO_SPILL")) {
            rc = tabucol_warp_launch(A, st, ctl32 + 4, ovf_spill, ctl32 + 5, ctl32 + 3, ovf_warp, h[0], true);
            if (rc > 0) return rc;
            if (rc == MCB_OK) {
                int32_t h2 = 0;
                if (cudaMemcpyAsync(&h2, ctl32 + 5, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                    cudaStreamSynchronize(st) != cudaSuccess)
                    return set_error(MCB_ERR_CUDA, "tabucol: spill pass failed: %s",
                                     cudaGetErrorString(cudaGetLastError()));
                if (h2 == 0) return MCB_OK;
                ovf_final = ovf_spill;
                ovf_final_count = ctl32 + 5;
            }
        }
    }

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

    if (variant != 2 && !warp_done) {
        P.work_counter = ctl32 + 0;
        P.ovf_count = ctl32 + 2;
        P.ovf_list = ctl32 + 64 + 256;
        P.ws_stamp = tables;
        P.ws_s_stride = variant == 3 ? cl_stride : ns_stride;
        if (variant == 1) {
            P.ws_gamma = tables + (size_t)grid * ns_stride;
            P.ws_g_stride = ng_stride;
        }
        rc = variant == 3   ? tabucol_cluster_launch(P, (int)A.p, st, &grid, false)
             : variant == 0 ? launch_variant<uint8_t, uint16_t, true>(P, grid_cap, (int)A.p, st, &grid, false)
                            : launch_variant<uint8_t, uint16_t, false>(P, grid_cap, (int)A.p, st, &grid, false);
        if (rc) return rc;
    }
    // wide pass: either everything (forced) or the overflowed individuals
    TabuParams Q = P;
    Q.work_counter = ctl32 + 1;
    Q.ovf_list = nullptr;
    Q.ovf_count = nullptr;
    if (variant != 2) {
        Q.work = ovf_final;
        Q.nwork_dev = ovf_final_count;
    }
    Q.ws_gamma = tables + narrow_ws;
    Q.ws_g_stride = wg_stride;
    Q.ws_stamp = tables + narrow_ws + (size_t)wide_grid * wg_stride;
    Q.ws_s_stride = ws_stride;
    int g2 = 1;
    rc = launch_variant<uint16_t, uint32_t, false>(Q, wide_grid, (int)A.p, st, &g2, false);
    if (rc) return rc;
    if (async) {
        async_err_slot(st) = ctl32 + 3;
        return MCB_OK;
    }

    int32_t err = 0;
    if (cudaMemcpyAsync(&err, ctl32 + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol: kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (err == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
    if (err == 2) return set_error(MCB_ERR_UNSUPPORTED, "tabucol: wide tables overflowed");
    return MCB_OK;
}

}  // namespace mcb
