// tabucol_cluster.cu -- batched TabuCol for shapes whose u8 gamma table does
// not fit one SM's shared memory (config 4, G(2000,.5) k=150: 300 KB per
// individual): one individual per 2-CTA thread-block cluster.
//
// Same semantics as tabucol.cu / the numba kernel `_tabucol_batch` (reference
// pkg/src/memcolor/localsearch.py:266-410), bit for bit in validation mode:
// scan order = conflict-list order x colours ascending (:328-334), tabu test
// with aspiration (:336-339), the sequential reservoir's counter advancing
// once per candidate that ties the running minimum (:340-350), tenure draw
// (:363-366), conflict-list append / swap-remove in (neighbours asc, then v)
// order (:368-385), best copy (:387-390), scratch check every 1024 (:398-405).
//
// Split.  CTA r of the pair owns the colours [r KH, r KH + KH) (KH = ceil(k/2)
// rounded to 4) of EVERY row: its half of gamma (u8, n x KH: 152 KB at
// config 4) and the tabu entries of its colours live in its own shared
// memory.  Replicated in both CTAs: the colouring, gva[v] = gamma[v][a_v]
// (maintained from the move alone: neighbours with colour a lose one, with
// colour b gain one, gva[v*] += D), the conflict list and every counter --
// so list maintenance, the tenure draw and the reservoir draws need no
// exchange.  Per iteration the CTAs meet at three cluster barriers:
//   #1 after pass 1: each CTA has evaluated its half of every conflicting
//      row ((min delta, #candidates at it) per half, from its row cache plus
//      the admissible tabu-slot colours) and the per-warp block minima; each
//      warp then pulls its block of the partner's records (DSMEM loads);
//   #2 after the prefix-min pass: rows equal to the running minimum carry
//      their combined count of tie events, rows that lower it are walked --
//      each CTA walks its own half, half 1 entered with min(R, half-0
//      minimum) -- and the walk events are exchanged;
//   #3 after the draw (spread over all warps): every warp derives the same
//      winner row and half, the owner of that half locates the column b and
//      publishes it, all threads prefetch their slice of N(v*).
// The prefix-min pass is spread over all warps (per-warp contiguous blocks of
// rows, block minima from pass 1, each block scanned from its entering
// minimum).  After #3 warp 0 does the tenure / tabu / log bookkeeping while
// the other warps update gamma, gva and the row caches over N(v*).
//
// Overflow (a gamma count reaching 255, tenure >= 16384) stops the individual
// in both CTAs at the same barrier; the host re-runs it on the wide CTA pass.
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "launch.h"
#include "tc_shared.cuh"

namespace cg = cooperative_groups;

namespace mcb {

namespace {

constexpr int CL_GMAX = 254;
// MCB_FLAG_PROFILE: rank 0 thread 0's cycles per phase ([1] pass 1 + barrier
// #1, [2] prefix/walk pass + #2, [3] draw/locate + #3, [4] move + update,
// [6] list events, [7] tail, [8] / [9] slowest warp's pass 1 in rank 0 / 1),
// [10] iterations, [11] pass-1 rows with spilled tabu expiries, [12] walked
// half-rows, [13] stale cache rescans, [14] masked scans, [15] init cycles
__device__ unsigned long long g_cl_cycles[16];
// MCB_FLAG_PROFILE, rank 0: per warp w, [w] summed pass-1 durations (clock
// from the warp's own start), [32 + w] summed start delays after thread 0's
// iteration start, [64 + w] masked + stale scans done by the warp
__device__ unsigned long long g_cl_warp[96];
constexpr uint32_t CL_SWEEP = 16384u;

template <int NW>
struct ClCtrl {
    long long it, conflicts, best, nlog, sum_c, sum_deg, diag;
    unsigned long long ctr;
    long long s0, s1;
    int C, wi, ovf, D, mylow, mv_b, gvb, plow;
    int smax[NW];
    int bmin[2][NW];  // per-warp block minima of the half-0 / half-1 records
    int beq[NW], blow[NW], bD[NW];
    long long red[NW];
    int wcnt[NW];
    unsigned long long ph[10];
    long long ph_t, t_top;
    unsigned p1max;
};

// segment offsets of the dynamic shared memory, computed on the host
enum ClSeg { CS_GAMMA, CS_TEXP, CS_TCOL, CS_TOVF, CS_ASSIGN, CS_GVA, CS_CLIST, CS_CPOS, CS_RLO, CS_RHI, CS_NBS,
             CS_EVM, CS_HC, CS_IP, CS_NSEG };
struct ClLayout {
    uint32_t off[CS_NSEG + 1];
    int kh;
};

// Word `lane` of row v's local half with its excluded colours forced to 0xFF:
// the own colour (aloc >= 0) and live tabu colours without aspiration (their
// g >= A = thr + gva, :336-339) -- from the 4 slots (cols / expiries tx) and,
// when spl, the dense spilled row, each lane checking its own 4 colours.
// A == INT_MIN: every slot colour excluded whatever its state (the row cache).
// Padding colours are 0xFF already.  Warp-cooperative: lanes >= KW get ~0.
__device__ __forceinline__ uint32_t cl_word(const uint8_t *gamma, const uint16_t *gstamp, int KH, int v, int aloc,
                                            uint32_t cols, uint2 tx, bool spl, int A, uint32_t it, int lane) {
    const int KW = KH >> 2;
    const uint8_t *gr = gamma + (size_t)v * KH;
    const uint32_t x0 = lane < KW ? reinterpret_cast<const uint32_t *>(gr)[lane] : 0xFFFFFFFFu;
    uint32_t x = x0;
    if (aloc >= 0 && (aloc >> 2) == lane) x |= 0xFFu << (8 * (aloc & 3));
    if (cols != 0xFFFFFFFFu) {
        const uint16_t e[4] = {(uint16_t)tx.x, (uint16_t)(tx.x >> 16), (uint16_t)tx.y, (uint16_t)(tx.y >> 16)};
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int t = (cols >> (8 * q)) & 0xFF;
            if (t != 0xFF && (t >> 2) == lane &&
                (A == INT_MIN || (active<uint16_t>(e[q], it) && !((int)((x0 >> (8 * (t & 3))) & 0xFF) < A))))
                x |= 0xFFu << (8 * (t & 3));
        }
    }
    if (spl && lane < KW) {
        const uint16_t *gs = gstamp + (size_t)v * KH + 4 * lane;
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (active<uint16_t>(gs[e], it) && !((int)((x0 >> (8 * e)) & 0xFF) < A)) x |= 0xFFu << (8 * e);
    }
    return x;
}
// (minimum byte or 0xFF, #bytes at it) over the warp's words
__device__ __forceinline__ void warp_min_count(uint32_t x, int &m, int &c) {
    constexpr unsigned FULL = 0xffffffffu;
    m = (int)__reduce_min_sync(FULL, min_bytes(x));
    c = m == 0xFF ? 0 : (int)__reduce_add_sync(FULL, (unsigned)count_eq_bytes(x, (uint32_t)m));
}
// Tie events of the sequential scan over a half row (words x, lane = word)
// entered with running minimum E (delta space): an exclusive prefix-min over
// the words gives each lane the running minimum entering its word, then each
// lane walks its 4 bytes (:340-350).
__device__ __forceinline__ int walk_ties(uint32_t x, int E, int gva, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const int incl = warp_incl_min((int)min_bytes(x), lane);
    int excl = __shfl_up_sync(FULL, incl, 1);
    if (lane == 0) excl = INT_MAX;
    int cur = min(E >= TC_BIG ? INT_MAX : E + gva, excl);
    int t = 0;
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const int b = (x >> (8 * e)) & 0xFF;
        if (b == 0xFF) continue;
        if (b < cur) cur = b;
        else if (b == cur) t++;
    }
    return __reduce_add_sync(FULL, t);
}
// local column of the need-th byte equal to Dg in word order, or -1
__device__ __forceinline__ int locate_col(uint32_t x, int Dg, int need, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    const int c = count_eq_bytes(x, (uint32_t)Dg);
    const int incl = warp_incl_sum(c, lane);
    const unsigned bm = __ballot_sync(FULL, incl >= need);
    if (!bm) return -1;
    const int src = __ffs(bm) - 1;
    int col = -1;
    if (lane == src) {
        int r = need - (incl - c);
#pragma unroll
        for (int e = 0; e < 4; e++)
            if ((int)((x >> (8 * e)) & 0xFF) == Dg && --r == 0 && col < 0) col = 4 * lane + e;
    }
    return __shfl_sync(FULL, col, src);
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) tabucol_cluster_kernel(TabuParams P, ClLayout L) {
    constexpr int NW = NT / 32;
    constexpr unsigned FULL = 0xffffffffu;

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ ClCtrl<NW> ctl;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) ctl.ovf = 0;

    const int n = P.n, k = P.k, KH = L.kh;
    const int cb = rank * KH;  // first colour of this CTA
    uint8_t *gamma = smem + L.off[CS_GAMMA];
    uint16_t *texp = reinterpret_cast<uint16_t *>(smem + L.off[CS_TEXP]);
    uint8_t *tcol = smem + L.off[CS_TCOL];
    uint16_t *tovf = reinterpret_cast<uint16_t *>(smem + L.off[CS_TOVF]);
    uint8_t *assign = smem + L.off[CS_ASSIGN];
    uint8_t *gva = smem + L.off[CS_GVA];
    uint16_t *clist = reinterpret_cast<uint16_t *>(smem + L.off[CS_CLIST]);
    uint16_t *cpos = reinterpret_cast<uint16_t *>(smem + L.off[CS_CPOS]);
    uint32_t *rlo = reinterpret_cast<uint32_t *>(smem + L.off[CS_RLO]);  // half-0 records per list slot
    uint32_t *rhi = reinterpret_cast<uint32_t *>(smem + L.off[CS_RHI]);  // half-1 records
    uint16_t *nbs = reinterpret_cast<uint16_t *>(smem + L.off[CS_NBS]);
    uint32_t *evm = reinterpret_cast<uint32_t *>(smem + L.off[CS_EVM]);
    // Row cache (this CTA's colours): minimum of gamma over the row's local
    // colours except its own colour and its tabu-slot colours (low byte, 0xFF
    // = none) and how many reach it (high byte; 0 = stale).  A move v*: a -> b
    // changes two columns of the neighbours' rows, so the update loop keeps it
    // in O(1) per neighbour; a row whose minimum group empties, v*'s own row
    // (own colour and slots change) and, at the expiry sweep, every row go
    // stale and are rescanned when next needed.  Pass 1 merges in the slot
    // colours that are admissible at the time (expired, or aspiration).
    uint16_t *hc = reinterpret_cast<uint16_t *>(smem + L.off[CS_HC]);
    // CSR row offsets (2m < 2^32 for n <= 32767): the move needs indptr[v*]
    // before barrier #3, and every cluster barrier invalidates L1
    uint32_t *ip = reinterpret_cast<uint32_t *>(smem + L.off[CS_IP]);
    for (int v = tid; v <= n; v += NT) ip[v] = (uint32_t)P.indptr[v];
    uint16_t *gstamp = reinterpret_cast<uint16_t *>(P.ws_stamp + blockIdx.x * P.ws_s_stride);
    uint32_t *rown = rank ? rhi : rlo, *rpeer = rank ? rlo : rhi;
    // the partner CTA's records and control block (distributed shared memory).
    // Records are pulled (coalesced DSMEM loads of each warp's block after
    // barrier #1): pushing them with per-lane remote stores measured ~7k
    // cycles per iteration at config 4, the pull a few hundred.
    const uint32_t *rpeer_src = cluster.map_shared_rank(rpeer, rank ^ 1);  // the peer's own half
    ClCtrl<NW> *ctl_peer = cluster.map_shared_rank(&ctl, rank ^ 1);

    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool prof = (P.flags & MCB_FLAG_PROFILE) != 0;
    const bool prof0 = prof && rank == 0 && tid == 0;
    unsigned n_spill = 0, n_walk = 0, n_stale = 0, n_mask = 0;
    if (tid == 0)
        for (int q = 0; q < 10; q++) ctl.ph[q] = 0;
#define CLPH(i)                             \
    if (prof0) {                            \
        const long long _t = clock64();     \
        ctl.ph[i] += _t - ctl.ph_t;         \
        ctl.ph_t = _t;                      \
    }
    auto local_col = [=](int c) { return (c >= cb && c < cb + KH) ? c - cb : -1; };
    auto both = [&](int ClCtrl<NW>::*f, int val) {  // a control word in both CTAs
        ctl.*f = val;
        ctl_peer->*f = val;
    };
    cluster.sync();

    for (;;) {
        if (rank == 0 && tid == 0) both(&ClCtrl<NW>::wi, atomicAdd(P.work_counter, 1));
        cluster.sync();
        const int wi = ctl.wi;
        const int nwork = P.nwork_dev ? *P.nwork_dev : P.nwork;
        if (wi >= nwork) break;
        const int ind = P.work ? P.work[wi] : wi;
        const uint64_t key = P.keys[ind];
        int32_t *a_io = P.assigns + (size_t)ind * n;
        int32_t *b_out = P.best_assigns + (size_t)ind * n;

        // ---------------- init (localsearch.py:289-318) ----------------
        const long long t_init = prof0 ? clock64() : 0;
        for (int v = tid; v < n; v += NT) {
            int c = a_io[v];
            if (c < 0 || c >= k) {
                atomicExch(P.err_flag, 1);
                c = 0;
            }
            assign[v] = (uint8_t)c;
            reinterpret_cast<uint32_t *>(tcol)[v] = 0xFFFFFFFFu;
            tovf[v] = 0;
            hc[v] = 0;
        }
        {
            // real colours 0, colours >= k (padding) all-ones: never a candidate
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gamma);
            const int KW = KH >> 2;
            for (int i = tid; i < n * KW; i += NT) {
                const int w = i % KW;
                uint32_t x = 0;
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (cb + 4 * w + e >= k) x |= 0xFFu << (8 * e);
                g32[i] = x;
            }
        }
        if (tid == 0) ctl.diag = 0;
        __syncthreads();
        {
            // this CTA's half of gamma[u] and (both CTAs) gva[u]: a warp per row,
            // lanes over the CSR neighbours (coalesced), byte counts added to
            // their 32-bit words by shared atomics; a count passing 254 shows
            // as a 0xFF byte or, once it carried, as a row sum short of the
            // number of local-coloured neighbours
            bool bad = false;
            const int KW = KH >> 2;
            for (int u = warp; u < n; u += NW) {
                const int au = assign[u];
                int gu = 0, nl = 0;
                uint32_t *row32 = reinterpret_cast<uint32_t *>(gamma + (size_t)u * KH);
                const int64_t s0 = ip[u], s1 = ip[u + 1];
#pragma unroll 4
                for (int64_t idx = s0 + lane; idx < s1; idx += 32) {
                    const int c = assign[__ldg(P.indices + idx)];
                    gu += c == au;
                    const int lc = local_col(c);
                    if (lc >= 0) {
                        atomicAdd(row32 + (lc >> 2), 1u << (8 * (lc & 3)));
                        nl++;
                    }
                }
                gu = __reduce_add_sync(FULL, gu);
                nl = __reduce_add_sync(FULL, nl);
                __syncwarp();
                int sum = 0;
                bool ff = false;
                if (lane < KW) {
                    const uint32_t x = row32[lane];
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        if (cb + 4 * lane + e >= k) continue;  // padding byte
                        const int b = (x >> (8 * e)) & 0xFF;
                        sum += b;
                        ff |= b == 0xFF;
                    }
                }
                sum = __reduce_add_sync(FULL, sum);
                if (__any_sync(FULL, ff) || sum != nl || gu > CL_GMAX) bad = true;
                if (lane == 0) gva[u] = (uint8_t)min(gu, CL_GMAX);
            }
            if (bad && lane == 0) both(&ClCtrl<NW>::ovf, 1);
        }
        __syncthreads();
        // conflicts and the ascending conflict list (:298-310), identical in both CTAs
        {
            long long c2 = 0;
            int base = 0;
            for (int ch = 0; ch < n; ch += NT) {
                const int v = ch + tid;
                bool f = false;
                if (v < n) {
                    f = gva[v] > 0;
                    c2 += gva[v];
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
        if (rank == 0)
            for (int v = tid; v < n; v += NT) b_out[v] = assign[v];
        cluster.sync();  // both halves built; an init overflow is visible to both
        if (prof0) atomicAdd(&g_cl_cycles[15], (unsigned long long)(clock64() - t_init));

        // ---------------- iterations (:320-405) ----------------
        if (k >= 2 && !ctl.ovf) {
            for (long long step = 0; step < P.depth; step++) {
                const long long conflicts = ctl.conflicts;
                if (conflicts == 0) break;  // (:322-323) identical in both CTAs
                if (prof && tid == 0) {
                    ctl.ph_t = ctl.t_top = clock64();
                    ctl.ph[0]++;
                    ctl.p1max = 0;
                }
                const long long it = ctl.it;
                const int C = ctl.C;
                const long long best = ctl.best;
                const int thr = (int)max(best - conflicts, (long long)-TC_BIG);
                const uint32_t it32 = (uint32_t)it;

                // pass 1: this CTA's half of every conflicting row (per-warp
                // contiguous blocks), records and block minima to both CTAs
                const int BS = (C + NW - 1) / NW;
                const int b0 = min(C, warp * BS), b1 = min(C, b0 + BS);
                const long long t_p1 = prof ? clock64() : 0;
                unsigned n_scans = 0;
                {
                    int bm = TC_BIG;
                    // up to 4 rows per lane in flight: their dependent shared-memory
                    // chains (list -> vertex -> cache / slots -> slot columns) overlap
                    constexpr int R = 4;
                    for (int c0 = b0; c0 < b1; c0 += 32 * R) {
                        int v[R], aloc[R], gv[R], m[R], c[R];
                        uint32_t h[R], cols[R];
                        uint2 tx[R];
                        bool on[R], spl[R], masked[R];
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            const int li = c0 + 32 * r + lane;
                            on[r] = li < b1;
                            v[r] = on[r] ? clist[li] : 0;
                        }
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            aloc[r] = local_col(assign[v[r]]);
                            gv[r] = gva[v[r]];
                            h[r] = on[r] ? hc[v[r]] : 0x1FFu;
                            cols[r] = reinterpret_cast<const uint32_t *>(tcol)[v[r]];
                            tx[r] = reinterpret_cast<const uint2 *>(texp)[v[r]];
                            spl[r] = active<uint16_t>(tovf[v[r]], it32);
                        }
                        // stale cache rows: rescanned by the whole warp (own and slot colours excluded)
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            for (unsigned sm = __ballot_sync(FULL, (h[r] >> 8) == 0); sm; sm &= sm - 1) {
                                const int src = __ffs(sm) - 1;
                                const uint32_t x = cl_word(gamma, gstamp, KH, __shfl_sync(FULL, v[r], src),
                                                           __shfl_sync(FULL, aloc[r], src), __shfl_sync(FULL, cols[r], src),
                                                           make_uint2(0, 0), false, INT_MIN, it32, lane);
                                int wm, wc;
                                warp_min_count(x, wm, wc);
                                if (lane == src) {
                                    h[r] = (uint32_t)wm | (uint32_t)(wm == 0xFF ? 1 : wc) << 8;
                                    hc[v[r]] = (uint16_t)h[r];
                                }
                                n_stale += prof && lane == 0;
                                n_scans++;
                            }
                        }
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            m[r] = (int)(h[r] & 0xFFu);
                            c[r] = (int)(h[r] >> 8);
                            masked[r] = false;
                            if (on[r]) {
                                // the cache holds the minimum over the colours that are
                                // neither the own colour nor in a tabu slot; a slot colour
                                // joins when its entry expired or aspiration admits it
                                // (g < thr + gva, :336-339)
                                const int A = thr + gv[r];
                                const uint8_t *gr = gamma + (size_t)v[r] * KH;
                                if (cols[r] != 0xFFFFFFFFu) {
                                    const uint16_t e[4] = {(uint16_t)tx[r].x, (uint16_t)(tx[r].x >> 16),
                                                           (uint16_t)tx[r].y, (uint16_t)(tx[r].y >> 16)};
#pragma unroll
                                    for (int q = 0; q < 4; q++) {
                                        const int t = (cols[r] >> (8 * q)) & 0xFF;
                                        if (t == 0xFF || t == aloc[r]) continue;
                                        const int g = gr[t];
                                        if (!active<uint16_t>(e[q], it32) || g < A) {
                                            c[r] = g < m[r] ? 1 : c[r] + (g == m[r]);
                                            m[r] = min(m[r], g);
                                        }
                                    }
                                }
                                if (prof) n_spill += spl[r];
                                masked[r] = spl[r];  // live spilled entries: full masked scan
                                if (m[r] == 0xFF) {
                                    m[r] = TC_BIG;
                                    c[r] = 0;
                                } else {
                                    m[r] -= gv[r];
                                }
                            } else {
                                m[r] = TC_BIG;
                                c[r] = 0;
                            }
                        }
                        // rows with live spilled tabu entries: masked scan by the warp
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            for (unsigned mm = __ballot_sync(FULL, masked[r]); mm; mm &= mm - 1) {
                                const int src = __ffs(mm) - 1;
                                const int gs = __shfl_sync(FULL, gv[r], src);
                                const uint32_t x = cl_word(
                                    gamma, gstamp, KH, __shfl_sync(FULL, v[r], src), __shfl_sync(FULL, aloc[r], src),
                                    __shfl_sync(FULL, cols[r], src),
                                    make_uint2(__shfl_sync(FULL, tx[r].x, src), __shfl_sync(FULL, tx[r].y, src)),
                                    __shfl_sync(FULL, spl[r], src), thr + gs, it32, lane);
                                int wm, wc;
                                warp_min_count(x, wm, wc);
                                if (lane == src) {
                                    m[r] = wm == 0xFF ? TC_BIG : wm - gs;
                                    c[r] = wc;
                                }
                                n_mask += prof && lane == 0;
                                n_scans++;
                            }
                        }
#pragma unroll
                        for (int r = 0; r < R; r++) {
                            if (on[r]) {
                                rown[c0 + 32 * r + lane] = rec_pack(m[r], c[r], (uint32_t *)nullptr);
                                bm = min(bm, m[r]);
                            }
                        }
                    }
                    bm = __reduce_min_sync(FULL, bm);
                    if (lane == 0) {
                        ctl.bmin[rank][warp] = bm;
                        ctl_peer->bmin[rank][warp] = bm;
                        if (prof) {
                            const long long t1 = clock64();
                            atomicMax(&ctl.p1max, (unsigned)(t1 - ctl.t_top));
                            if (rank == 0) {
                                atomicAdd(&g_cl_warp[warp], (unsigned long long)(t1 - t_p1));
                                atomicAdd(&g_cl_warp[32 + warp], (unsigned long long)(t_p1 - ctl.t_top));
                                atomicAdd(&g_cl_warp[64 + warp], (unsigned long long)n_scans);
                            }
                        }
                    }
                }
                cluster.sync();  // #1
                if (prof && tid == 0) ctl.ph[8] += ctl.p1max;  // this CTA's slowest warp, pass 1 alone
                if (ctl.ovf) break;  // set before #1 by either CTA: both stop here
                for (int q = b0 + lane; q < b1; q += 32) rpeer[q] = rpeer_src[q];  // this warp's block
                __syncwarp();
                CLPH(1);

                // pass 2: each block scanned from its entering running minimum
                auto rows = [&](int q, int2 &h0, int2 &h1, int &x, int &y) {
                    h0 = q < b1 ? rec_unpack(rlo[q]) : make_int2(TC_BIG, 0);
                    h1 = q < b1 ? rec_unpack(rhi[q]) : make_int2(TC_BIG, 0);
                    x = min(h0.x, h1.x);
                    y = (x >= TC_BIG) ? 0 : (h0.x == x ? h0.y : 0) + (h1.x == x ? h1.y : 0);
                };
                {
                    const int bmv = lane < NW ? min(ctl.bmin[0][lane], ctl.bmin[1][lane]) : TC_BIG;
                    const int binc = warp_incl_min(bmv, lane);
                    const int D = __shfl_sync(FULL, binc, 31);
                    int carry = warp == 0 ? TC_BIG : __shfl_sync(FULL, binc, warp - 1);
                    int eq = 0, low = 0, dc = 0;
                    for (int q0 = b0; q0 < b1; q0 += 32) {
                        const int q = q0 + lane;
                        int2 h0, h1;
                        int x, y;
                        rows(q, h0, h1, x, y);
                        const int incl = warp_incl_min(x, lane);
                        int excl = __shfl_up_sync(FULL, incl, 1);
                        if (lane == 0) excl = TC_BIG;
                        const int RM = min(carry, excl);
                        int E = 0;
                        bool wlk = false;
                        if (!prod && x < TC_BIG) {
                            if (x == RM) {
                                eq += y;
                            } else if (x < RM) {
                                // this CTA's half entered with RM (half 0) or min(RM, half-0 min)
                                const int2 hm = rank ? h1 : h0;
                                E = rank ? min(RM, h0.x) : RM;
                                if (hm.x < TC_BIG) {
                                    if (hm.x == E) low += hm.y;
                                    else if (hm.x < E) wlk = true;
                                }
                            }
                        }
                        if (x == D && x < TC_BIG) dc += y;
                        for (unsigned wm = __ballot_sync(FULL, wlk); wm; wm &= wm - 1) {
                            const int src = __ffs(wm) - 1;
                            const int Es = __shfl_sync(FULL, E, src);
                            const int v = clist[q0 + src];
                            const int gvv = gva[v];
                            const uint32_t x = cl_word(gamma, gstamp, KH, v, local_col(assign[v]),
                                                       reinterpret_cast<const uint32_t *>(tcol)[v],
                                                       reinterpret_cast<const uint2 *>(texp)[v],
                                                       active<uint16_t>(tovf[v], it32), thr + gvv, it32, lane);
                            const int t = walk_ties(x, Es, gvv, lane);
                            if (lane == 0) {
                                low += t;
                                n_walk += prof;
                            }
                        }
                        carry = min(carry, __shfl_sync(FULL, incl, 31));
                    }
                    eq = __reduce_add_sync(FULL, eq);
                    low = __reduce_add_sync(FULL, low);
                    dc = __reduce_add_sync(FULL, dc);
                    if (lane == 0) {
                        ctl.beq[warp] = eq;
                        ctl.blow[warp] = low;
                        ctl.bD[warp] = dc;
                    }
                    if (tid == 0) ctl.D = D;
                }
                __syncthreads();
                if (warp == 0) {
                    const int lw = __reduce_add_sync(FULL, lane < NW ? ctl.blow[lane] : 0);
                    if (lane == 0) ctl_peer->plow = lw;
                    if (lane == 0) ctl.mylow = lw;
                }
                cluster.sync();  // #2: the partner's walk events
                CLPH(2);

                // the reservoir draw (:340-350) spread over all warps, then every warp
                // derives the same winner row; the CTA owning the winner's half
                // locates its column while all threads prefetch N(v*)
                const int D = ctl.D;
                const unsigned long long ctr = ctl.ctr;
                int T = 0, total = 0, mv_v = -1, need = 0, c0d = 0;
                if (D < TC_BIG) {
                    T = __reduce_add_sync(FULL, lane < NW ? ctl.bD[lane] : 0);
                    total = __reduce_add_sync(FULL, lane < NW ? ctl.beq[lane] : 0) + ctl.mylow + ctl.plow;
                    int smax = 1;
                    if (T > 1 && !prod) {
                        const unsigned long long c0 = ctr + (unsigned long long)(total - (T - 1));
                        for (int s = 2 + tid; s <= T; s += NT)
                            if (below_is_zero(key, c0 + (unsigned long long)(s - 2), (uint32_t)s)) smax = s;
                    }
                    smax = __reduce_max_sync(FULL, smax);
                    if (lane == 0) ctl.smax[warp] = smax;
                }
                __syncthreads();
                if (D < TC_BIG) {
                    int sstar = 1;
                    if (T > 1)
                        sstar = prod ? 1 + (int)philox_below(key, ctr, (uint32_t)T)
                                     : (int)__reduce_max_sync(FULL, lane < NW ? ctl.smax[lane] : 1);
                    // block, then row, then half holding the sstar-th D-candidate
                    const int cj = lane < NW ? ctl.bD[lane] : 0;
                    const int cin = warp_incl_sum(cj, lane);
                    const int wb = __ffs(__ballot_sync(FULL, cin >= sstar)) - 1;
                    need = sstar - __shfl_sync(FULL, cin - cj, wb);
                    const int r0 = min(C, wb * BS), r1 = min(C, r0 + BS);
                    for (int q0 = r0; q0 < r1 && mv_v < 0; q0 += 32) {
                        const int q = q0 + lane;
                        int2 h0 = make_int2(TC_BIG, 0), h1 = make_int2(TC_BIG, 0);
                        if (q < r1) {
                            h0 = rec_unpack(rlo[q]);
                            h1 = rec_unpack(rhi[q]);
                        }
                        const int x = min(h0.x, h1.x);
                        const int y = (x == D) ? (h0.x == x ? h0.y : 0) + (h1.x == x ? h1.y : 0) : 0;
                        const int inc = warp_incl_sum(y, lane);
                        const unsigned bm = __ballot_sync(FULL, inc >= need);
                        if (bm) {
                            const int src = __ffs(bm) - 1;
                            mv_v = clist[q0 + src];
                            need -= __shfl_sync(FULL, inc - y, src);
                            const int h0x = __shfl_sync(FULL, h0.x, src), h0y = __shfl_sync(FULL, h0.y, src);
                            c0d = h0x == D ? h0y : 0;
                        } else {
                            need -= __shfl_sync(FULL, inc, 31);
                        }
                    }
                }
                // N(v*): update threads (warps 1..) hold their neighbours in registers
                constexpr int NBR = 4;
                int64_t g0 = 0, g1 = 0;
                int nb[NBR];
                if (mv_v >= 0) {
                    g0 = ip[mv_v];
                    g1 = ip[mv_v + 1];
                }
#pragma unroll
                for (int q = 0; q < NBR; q++) {
                    const int64_t j = g0 + (tid - 32) + (int64_t)q * (NT - 32);
                    nb[q] = (warp > 0 && j < g1) ? __ldg(P.indices + j) : 0;
                }
                if (warp == 0 && mv_v >= 0) {
                    const int owner = need <= c0d ? 0 : 1;
                    if (owner == rank) {
                        const int gvv = gva[mv_v];
                        const uint32_t x = cl_word(gamma, gstamp, KH, mv_v, local_col(assign[mv_v]),
                                                   reinterpret_cast<const uint32_t *>(tcol)[mv_v],
                                                   reinterpret_cast<const uint2 *>(texp)[mv_v],
                                                   active<uint16_t>(tovf[mv_v], it32), thr + gvv, it32, lane);
                        const int col = locate_col(x, D + gvv, owner ? need - c0d : need, lane);
                        if (lane == 0) both(&ClCtrl<NW>::mv_b, col < 0 ? -1 : cb + col);
                    }
                }
                cluster.sync();  // #3: the column from its owner
                CLPH(3);

                // the move (:352-396).  Warp 0: tenure, tabu entry (owner of colour a),
                // counters, log; warps 1..: gamma (this CTA's colours), gva and the row
                // cache over N(v) (:356-359) with ballots of conflict-set events per 32
                // neighbours, and the best copy (:387-390).  assign[v] changes after the
                // next barrier (the update reads the old colours).
                const int mvv = mv_v;
                bool improved = false;
                if (mvv >= 0) {
                    const int ma = assign[mvv];
                    int mb = ctl.mv_b;
                    const long long nconf = conflicts + D;
                    improved = nconf < best;
                    const int deg = (int)(g1 - g0);
                    if (warp == 0) {
                        if (lane == 0) {
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
                            if (tt >= (long long)CL_SWEEP || mb < 0) ctl.ovf = 1;
                            const int v = mvv, al = local_col(ma);
                            if (al >= 0) {  // tabu (v, a) until it + tt + 1: slot hit, free slot, or spill
                                const uint16_t e_new = (uint16_t)(uint32_t)(it + tt + 1);
                                const uint32_t cols = reinterpret_cast<const uint32_t *>(tcol)[v];
                                int s_hit = -1, s_free = -1;
#pragma unroll
                                for (int s = 0; s < 4; s++) {
                                    const int cs = (cols >> (8 * s)) & 0xFF;
                                    if (cs == al) s_hit = s;
                                    else if (s_free < 0 && (cs == 0xFF || !active<uint16_t>(texp[4 * v + s], it32)))
                                        s_free = s;
                                }
                                const int s = s_hit >= 0 ? s_hit : s_free;
                                const bool ovf_live = active<uint16_t>(tovf[v], it32);
                                if (s >= 0) {
                                    tcol[4 * v + s] = (uint8_t)al;
                                    texp[4 * v + s] = e_new;
                                    if (ovf_live) gstamp[(size_t)v * KH + al] = (uint16_t)it32;  // supersede
                                } else {
                                    spill_set<uint16_t>(gstamp + (size_t)v * KH, tovf + v, ovf_live, KH, al, e_new,
                                                        it32);
                                }
                            }
                            ctl.gvb = gva[v] + D;  // gamma[v][b] (row v is not changed by its own move)
                            hc[v] = 0;             // its own colour changes
                            ctl.conflicts = nconf;
                            ctl.ctr = c;
                            const long long nl = ctl.nlog;
                            if (nl < P.log_cap) {
                                if (rank == 0) {
                                    const size_t o = (size_t)ind * P.log_cap + nl;
                                    P.log_v[o] = v;
                                    P.log_iter[o] = it;
                                    P.log_tt[o] = tt;
                                }
                                ctl.nlog = nl + 1;
                            }
                            ctl.sum_deg += deg;
                        }
                    } else {
                        if (mb < 0) mb = ma;  // (overflow path: the individual is re-run)
                        const int al = local_col(ma), bl = local_col(mb);
                        bool bad = false;
                        for (int q = 0; q * (NT - 32) < deg; q++) {
                            const int j = (tid - 32) + q * (NT - 32);
                            bool evt = false;
                            if (j < deg) {
                                int u = 0;
#pragma unroll
                                for (int r = 0; r < NBR; r++)
                                    if (q == r) u = nb[r];
                                if (q >= NBR) u = __ldg(P.indices + g0 + j);
                                nbs[j] = (uint16_t)u;
                                uint8_t *gr = gamma + (size_t)u * KH;
                                const int au = assign[u];
                                const uint32_t cu = reinterpret_cast<const uint32_t *>(tcol)[u];
                                uint32_t h = hc[u];
                                int hm = (int)(h & 0xFFu), hn = (int)(h >> 8);
                                // colours in u's tabu slots are outside its cache
                                auto in_slots = [cu](int x) {
                                    return ((cu & 0xFFu) == (uint32_t)x) | (((cu >> 8) & 0xFFu) == (uint32_t)x) |
                                           (((cu >> 16) & 0xFFu) == (uint32_t)x) | ((cu >> 24) == (uint32_t)x);
                                };
                                if (al >= 0) {
                                    const int ga = gr[al] - 1;
                                    gr[al] = (uint8_t)ga;
                                    if (au != ma && hn != 0 && !in_slots(al)) {
                                        hn = ga < hm ? 1 : hn + (ga == hm);
                                        hm = min(hm, ga);
                                    }
                                }
                                if (bl >= 0) {
                                    const int gb = gr[bl];
                                    if (gb >= CL_GMAX) bad = true;
                                    else gr[bl] = (uint8_t)(gb + 1);
                                    if (au != mb && hn != 0 && gb == hm && !in_slots(bl)) hn--;  // 0: stale
                                }
                                hc[u] = (uint16_t)(hm | hn << 8);
                                if (au == ma) {
                                    const int g = gva[u] - 1;
                                    gva[u] = (uint8_t)g;
                                    evt = g == 0;
                                } else if (au == mb) {
                                    const int g = gva[u];
                                    if (g >= CL_GMAX) bad = true;
                                    else gva[u] = (uint8_t)(g + 1);
                                    evt = g == 0;
                                }
                            }
                            const unsigned em = __ballot_sync(FULL, evt);
                            if (lane == 0) evm[q * (NW - 1) + warp - 1] = em;
                        }
                        if (bad) both(&ClCtrl<NW>::ovf, 1);
                        if (rank == 0 && improved)
                            for (int u = tid - 32; u < n; u += NT - 32) b_out[u] = u == mvv ? mb : assign[u];
                    }
                }
                __syncthreads();
                CLPH(4);
                // conflict-list events in neighbour order, then v (:368-385): warp 0
                // loads the event words in parallel, lane 0 applies the non-zero ones
                if (warp == 0) {
                    int Cn = C;
                    if (mvv >= 0) {
                        const int nwd = (int)((g1 - g0 + 31) >> 5);
                        for (int w0 = 0; w0 < nwd; w0 += 32) {
                            const unsigned el = w0 + lane < nwd ? evm[w0 + lane] : 0u;
                            for (unsigned nz = __ballot_sync(FULL, el != 0u); nz; nz &= nz - 1) {
                                const int src = __ffs(nz) - 1;
                                unsigned e = __shfl_sync(FULL, el, src);
                                if (lane == 0) {
                                    while (e) {
                                        const int bit = __ffs(e) - 1;
                                        e &= e - 1u;
                                        const int u = nbs[(w0 + src) * 32 + bit];
                                        cl_apply(clist, cpos, Cn, u, cpos[u] == 0xFFFF);  // enter iff outside
                                    }
                                }
                            }
                        }
                    }
                    if (lane == 0) {
                        if (mvv >= 0) {
                            const int mb = ctl.mv_b;
                            assign[mvv] = (uint8_t)(mb < 0 ? assign[mvv] : mb);
                            gva[mvv] = (uint8_t)ctl.gvb;
                            cl_apply(clist, cpos, Cn, mvv, ctl.gvb > 0);
                            ctl.C = Cn;
                            if (improved) ctl.best = ctl.conflicts;
                        }
                        ctl.sum_c += C;
                        ctl.it = it + 1;
                    }
                }
                __syncthreads();
                CLPH(6);
                const long long itn = it + 1;
                const bool chk = diagf && rank == 0 && (itn % 1024 == 0);
                const bool swp = (itn % CL_SWEEP) == 0;
                if (chk) {  // scratch conflicts over the edge list (:398-405)
                    long long c2 = 0;
                    for (int64_t e = tid; e < P.m; e += NT)
                        c2 += assign[__ldg(P.eu + e)] == assign[__ldg(P.ev + e)];
                    c2 = warp_sum64(c2);
                    if (lane == 0) ctl.red[warp] = c2;
                }
                if (swp) {  // keep 16-bit expiries unambiguous
                    const uint32_t itw = (uint32_t)itn;
                    for (int v = tid; v < n; v += NT) {
                        for (int s = 0; s < 4; s++)
                            if (!active<uint16_t>(texp[4 * v + s], itw)) tcol[4 * v + s] = 0xFF;
                        hc[v] = 0;  // its slot set (outside the cache) may have changed
                        if (active<uint16_t>(tovf[v], itw)) {
                            uint16_t *gs = gstamp + (size_t)v * KH;
                            for (int c = 0; c < KH; c++)
                                if (!active<uint16_t>(gs[c], itw)) gs[c] = (uint16_t)itw;
                        } else {
                            tovf[v] = (uint16_t)itw;
                        }
                    }
                }
                if (chk || swp) __syncthreads();
                if (chk && tid == 0) {
                    long long s = 0;
                    for (int j = 0; j < NW; j++) s += ctl.red[j];
                    if (s != ctl.conflicts) ctl.diag += 1;
                }
                CLPH(7);
            }
        }
        if (prof) {
            if (prof0) {
                for (int q = 1; q < 9; q++) atomicAdd(&g_cl_cycles[q], ctl.ph[q]);
                atomicAdd(&g_cl_cycles[10], ctl.ph[0]);
            }
            if (prof && rank == 1 && tid == 0) atomicAdd(&g_cl_cycles[9], ctl.ph[8]);
            if (tid == 0)
                for (int q = 0; q < 10; q++) ctl.ph[q] = 0;
            if (rank == 0) {
                atomicAdd(&g_cl_cycles[11], (unsigned long long)n_spill);
                atomicAdd(&g_cl_cycles[12], (unsigned long long)n_walk);
                atomicAdd(&g_cl_cycles[13], (unsigned long long)n_stale);
                atomicAdd(&g_cl_cycles[14], (unsigned long long)n_mask);
            }
            n_spill = n_walk = n_stale = n_mask = 0;
        }
        cluster.sync();  // every overflow flag is visible to both

        // ---------------- outputs (:407-410) ----------------
        if (rank == 0) {
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
        }
        __syncthreads();
        if (tid == 0) ctl.ovf = 0;  // before the next work barrier: no remote write can race it
    }
    cluster.sync();  // neither CTA leaves while the other may still address its shared memory
}

ClLayout cl_layout(int n, int k) {
    ClLayout L{};
    L.kh = (((k + 1) / 2) + 3) & ~3;
    const size_t N = (size_t)n;
    const size_t bytes[CS_NSEG] = {N * L.kh, N * 8, N * 4, N * 2, N,     N,
                                   N * 2,    N * 2, N * 4, N * 4, N * 2, 4 * ((N + 31) / 32 + 32), N * 2, (N + 1) * 4};  // evm: + one word per warp
    size_t off = 0;
    for (int i = 0; i < CS_NSEG; i++) {
        L.off[i] = (uint32_t)off;
        off += (bytes[i] + 15) & ~(size_t)15;
    }
    L.off[CS_NSEG] = (uint32_t)off;
    return L;
}

int cl_threads() {
    if (const char *e = getenv("MCB_CL_NT")) {
        const int v = atoi(e);
        if (v == 256 || v == 512 || v == 1024) return v;
    }
    return 512;
}

template <int NT>
int cl_launch_t(const TabuParams &P, const ClLayout &L, int max_clusters, cudaStream_t st, int *grid_out,
                bool query_only) {
    auto kern = tabucol_cluster_kernel<NT>;
    const size_t smem = L.off[CS_NSEG];
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol cluster: smem attribute (%zu B) failed", smem);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(2 * num_sms());
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess || nc < 1)
        return set_error(MCB_ERR_CUDA, "tabucol cluster: no resident 2-CTA cluster at %zu B", smem);
    const int clusters = std::max(1, std::min(nc, max_clusters));
    *grid_out = 2 * clusters;
    if (query_only) return MCB_OK;
    cfg.gridDim = dim3(2 * clusters);
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] tabucol_cluster<nt=%d> clusters=%d (max %d) smem=%zu kh=%d\n", NT, clusters,
                nc, smem, L.kh);
    if (cudaLaunchKernelEx(&cfg, kern, P, L) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol cluster launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return MCB_OK;
}

int cl_launch_nt(const TabuParams &P, const ClLayout &L, int max_clusters, cudaStream_t st, int *grid_out,
                 bool query_only) {
    switch (cl_threads()) {
        case 256: return cl_launch_t<256>(P, L, max_clusters, st, grid_out, query_only);
        case 1024: return cl_launch_t<1024>(P, L, max_clusters, st, grid_out, query_only);
        default: return cl_launch_t<512>(P, L, max_clusters, st, grid_out, query_only);
    }
}

}  // namespace

int tabucol_cluster_warp_stats(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_cl_warp, sizeof(unsigned long long) * 96) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "cluster warp counters unavailable");
    if (reset) {
        const unsigned long long z[96] = {0};
        cudaMemcpyToSymbol(g_cl_warp, z, sizeof(z));
    }
    return MCB_OK;
}

int tabucol_cluster_phase_cycles(unsigned long long *out, int reset) {
    unsigned long long h[16];
    if (cudaMemcpyFromSymbol(h, g_cl_cycles, sizeof(h)) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "cluster phase counters unavailable");
    for (int i = 0; i < 16; i++) out[i] += h[i];
    if (reset) {
        const unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_cl_cycles, z, sizeof(z));
    }
    return MCB_OK;
}

size_t tabucol_cluster_smem(int n, int k) { return cl_layout(n, k).off[CS_NSEG]; }

size_t tabucol_cluster_stamp_stride(int n, int k) {
    return ((size_t)n * cl_layout(n, k).kh * 2 + 255) & ~(size_t)255;
}

int tabucol_cluster_launch(const TabuParams &P, int max_clusters, cudaStream_t st, int *grid_out, bool query_only) {
    const ClLayout L = cl_layout(P.n, P.k);
    if (L.off[CS_NSEG] > (size_t)max_smem_optin())
        return set_error(MCB_ERR_UNSUPPORTED, "tabucol cluster: n=%d k=%d needs %u B per CTA", P.n, P.k,
                         L.off[CS_NSEG]);
    return cl_launch_nt(P, L, max_clusters, st, grid_out, query_only);
}

}  // namespace mcb
