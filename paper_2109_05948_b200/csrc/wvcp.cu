// wvcp.cu -- batched weighted-colouring tabu search for sm_100a, one
// individual per CTA.
//
// Replaces the numba kernel `_wvcp_batch` (reference
// pkg/src/memcolor/localsearch.py:89-263, with _refresh_class :46-67 and
// _wvcp_scratch :70-86).  Reproduced exactly:
//   * objective g = fp64(d_score) + phi * fp64(d_conf), a separate fp64 multiply
//     and add (__dmul_rn / __dadd_rn: the reference's numba code has no FMA,
//     :193); candidates compared with fp64 < and == (:194-210);
//   * full scan v = 0..n-1, c = 0..k-1 (c != a) with
//       rem = uniq_drop[a] if rank(v) == max_rank[a] else 0,
//       d_add = max(0, w_v - max_val[c]), d_score = d_add - rem (:172-186);
//   * frozen vertex (it < tabu_until[v]) admissible only if the move is legal
//     and strictly improves the best legal score (:187-192);
//   * reservoir tie-break on the SplitMix64 stream (:202-210), tenure
//     U{0..9} + tt_base on the same stream (:228-231), tabu_until reset at every
//     round start (:160-161), phi halved/doubled after each round and forced on
//     the last (:157-159, :251-258), scratch check every 1024 iterations (:245-249).
//
// Parallel evaluation of the sequential reservoir, as in tabucol.cu: pass 1
// computes every row's (min g, #candidates at the min) -- one vertex per thread,
// all n rows, in exact 32/64-bit integers when phi = t 2^-s (gv_mode); the
// prefix minimum over the rows in vertex order runs on all 8 warps (chunks of
// 32 rows entered with the minimum of the chunks before), counting the tie
// events of rows equal to the running minimum and walking the rows that lower
// it (lanes over colours); warp 0 combines the partials, draws the final
// group's T - 1 independent reservoir draws, locates the move and applies it.
//
// State per individual: gamma u8[n][k] (u16 in the re-run of individuals whose
// counts reach 256) and the per-vertex arrays in shared memory -- 4 CTAs per SM
// at config 3; the per-class weight-rank counts wc[k][nranks] in a per-CTA
// global slice (touched for two classes per move).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cuda_pipeline.h>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int WV_NT = 256;
constexpr int WV_INF_SCORE_SHIFT = 62;
// shared-memory segments, in layout order
enum WvSeg { S_GAMMA, S_TABU, S_WGT, S_WRK, S_ASSIGN, S_RMIN, S_RCNT, S_MAXRANK, S_MAXVAL, S_UNIQ, S_CMAX, S_MX32,
             S_LOWQ, S_IP32, S_NBUF, S_LOWR, WV_NSEG };

struct WvParams {
    int32_t *assigns;
    int32_t *best_assigns;
    const int64_t *indptr;
    const int32_t *indices;
    const int32_t *eu, *ev;
    int64_t m;
    const int32_t *wranks;
    const int64_t *wvals;
    int nranks;
    const int64_t *weights;
    int n, k;
    int64_t depth, rounds;
    int schedule_on;
    const double *phi0s;
    double forced_phi;
    int64_t tt_base;
    const uint64_t *keys;
    int64_t *best_scores, *end_scores, *end_conflicts;
    double *phi_used;
    int64_t *diag;
    int64_t log_cap;
    int32_t *log_v;
    int64_t *log_iter, *log_tt;
    int8_t *log_asp;
    int64_t *log_cnt;
    uint32_t flags;
    int nwork;
    const int32_t *work_list;  // individual ids (nullptr: 0 .. nwork-1)
    int32_t *ovf_list, *ovf_count;  // u8 gamma: individuals whose gamma reached 256
    int32_t *work_counter;
    int32_t *err_flag;
    uint16_t *ws_wc;  // per-CTA [k][nranks]
    size_t ws_wc_stride;
    // dynamic shared-memory layout, computed on the host (wv_layout): offsets
    // read from the parameter bank are free operands, whereas offsets carved
    // in the kernel are rematerialised inside the loop under the register cap
    uint32_t so[WV_NSEG + 1];
};

struct WvCtrl {
    long long it, score, conflicts, best, nlog, diag;
    unsigned long long ctr;
    double phi;
    int work, mv_v, mv_a, mv_b, has_move, ovf, copy, deg;
    // 32-bit path's row caches: 0 = none valid, 1 = valid before the move
    // (mv_v, mv_a, mv_b; class maxima of mv_a / mv_b before it: ma_old, mb_old),
    // 2 = valid, no move since
    int inc, ma_old, mb_old;
    long long red[WV_NT / 32];
    long long red2[WV_NT / 32];
};

// x % s == 0 for the reservoir draws: s < 64 by a table (inverse of the odd
// part mod 2^64 and floor((2^64 - 1) / odd)), larger s by the fp64 test
__device__ ulonglong2 g_divtab_wv[32];
__device__ __forceinline__ bool divisible_wv(uint64_t x, uint32_t s) {
    if (s < 64u) {
        const int t = __ffs(s) - 1;
        const ulonglong2 e = g_divtab_wv[(s >> t) >> 1];
        return (x & ((1ull << t) - 1ull)) == 0ull && (x >> t) * e.x <= e.y;
    }
    return mod_is_zero(x, s);
}

__device__ __forceinline__ double gval_of(long long ds, long long dc, double phi) {
    return __dadd_rn((double)ds, __dmul_rn(phi, (double)dc));  // no FMA (:193)
}

// Exact integer evaluation of the objective.  When phi = t * 2^-s with small
// t and s (the reference's schedule phi0 * 2^j, e.g. 6 * 2^j at config 4), and
// |ds| < 2^31, |dc| < 2^16, every fp64 operation of gval_of is exact, so the
// fp64 values are the rationals (ds * 2^s + t * dc) * 2^-s: comparing the
// integer numerators G gives exactly the same order and the same ties.  The
// scan then keeps G (as an exact double where a double is stored).
struct GvMode {
    int fast, s;
    long long t;
    double phi;
};
__device__ __forceinline__ GvMode gv_mode(double phi, int n) {
    GvMode m{0, 0, 0, phi};
    if (n < (1 << 16)) {
        double f = phi;
        for (int s = 0; s <= 16; s++, f *= 2.0) {  // f = phi * 2^s exactly
            if (f == trunc(f) && fabs(f) < 1048576.0) {
                m.fast = 1;
                m.s = s;
                m.t = (long long)f;
                break;
            }
        }
    }
    return m;
}
__device__ __forceinline__ long long gnum(const GvMode &m, long long ds, long long dc) {
    return (ds << m.s) + m.t * dc;
}
__device__ __forceinline__ double gval(const GvMode &m, long long ds, long long dc) {
    return m.fast ? (double)gnum(m, ds, dc) : gval_of(ds, dc, m.phi);
}

__device__ __forceinline__ double shfl_up_d(double x, int o) {
    return __longlong_as_double(__shfl_up_sync(0xffffffffu, __double_as_longlong(x), o));
}
__device__ __forceinline__ double shfl_d(double x, int src) {
    return __longlong_as_double(__shfl_sync(0xffffffffu, __double_as_longlong(x), src));
}

// GT: gamma element type.  uint8_t halves the dominant shared-memory table
// (2 -> 4 individuals per SM at config 4); a count that would reach 256 stops
// the individual, which the host re-runs with uint16_t.
// MCB_FLAG_WSTATS: thread 0's cycles per phase, summed over all iterations
// ([0] iterations, [1..8] phases: pass 1, chunk minima, prefix + walks, warp-0
// section, gamma update, class refresh, best copy, tail)
__device__ unsigned long long g_wvstats[16];

template <typename GT, bool STATS>
__global__ void __launch_bounds__(WV_NT, 4) wvcp_kernel(WvParams P) {
    constexpr bool NARROW = sizeof(GT) == 1;
    constexpr int NT = WV_NT, NW = NT / 32;
    constexpr unsigned FULL = 0xffffffffu;
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const long long INF_SCORE = 1LL << WV_INF_SCORE_SHIFT;

    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ WvCtrl ctl;
    const int n = P.n, k = P.k, nranks = P.nranks;
    GT *gamma = reinterpret_cast<GT *>(smem + P.so[S_GAMMA]);
    uint32_t *tabu_until = reinterpret_cast<uint32_t *>(smem + P.so[S_TABU]);
    int32_t *wgt = reinterpret_cast<int32_t *>(smem + P.so[S_WGT]);
    uint16_t *wrk = reinterpret_cast<uint16_t *>(smem + P.so[S_WRK]);
    uint8_t *assign = smem + P.so[S_ASSIGN];
    double *rmin = reinterpret_cast<double *>(smem + P.so[S_RMIN]);
    uint16_t *rcnt = reinterpret_cast<uint16_t *>(smem + P.so[S_RCNT]);
    int32_t *max_rank = reinterpret_cast<int32_t *>(smem + P.so[S_MAXRANK]);
    int64_t *max_val = reinterpret_cast<int64_t *>(smem + P.so[S_MAXVAL]);
    int64_t *uniq_drop = reinterpret_cast<int64_t *>(smem + P.so[S_UNIQ]);
    int32_t *cmax = reinterpret_cast<int32_t *>(smem + P.so[S_CMAX]);  // scratch
    int32_t *mx32 = reinterpret_cast<int32_t *>(smem + P.so[S_MX32]);  // max_val as int32 (the scan's copy)
    int32_t *lowq = reinterpret_cast<int32_t *>(smem + P.so[S_LOWQ]);  // 32-bit path: chunk minima / counts, walk queue
    int32_t *ip32 = reinterpret_cast<int32_t *>(smem + P.so[S_IP32]);  // CSR row offsets
    int32_t *nbuf = reinterpret_cast<int32_t *>(smem + P.so[S_NBUF]);  // the moved vertex's neighbours
    double *lowR = reinterpret_cast<double *>(smem + P.so[S_LOWR]);
    uint16_t *wc = P.ws_wc + blockIdx.x * P.ws_wc_stride;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;

    __shared__ int s_maxw;
    __shared__ int s_nlow, s_wts[NW], s_wts2[NW];  // 32-bit path: walk queue length, warp event sums
    if (tid == 0) s_maxw = 0;
    __syncthreads();
    {
        int mw = 0;
        for (int v = tid; v <= n; v += NT) ip32[v] = (int32_t)P.indptr[v];  // 2m < 2^31 (host-checked)
        for (int v = tid; v < n; v += NT) {
            wgt[v] = (int32_t)P.weights[v];
            wrk[v] = (uint16_t)P.wranks[v];
            mw = max(mw, abs((int)P.weights[v]));
        }
        atomicMax(&s_maxw, mw);
    }

    // refresh_class (:46-67) by one warp: highest rank with a member, and the
    // drop of the class max if that member were the only one at its rank
    auto refresh_class = [&](int c) {
        const uint16_t *row = wc + (size_t)c * nranks;
        int mr = -1, sr = -1;
        unsigned cnt_mr = 0;
        if (nranks <= 128) {
            // all of the class's rank counts in flight at once (one L2 round trip):
            // lane L holds ranks nranks-1-L-32j, j < 4, top rank first
            uint32_t h[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int r = nranks - 1 - lane - 32 * j;
                h[j] = r >= 0 ? row[r] : 0u;
            }
            int found = 0;  // ranks with a member, highest first: mr, then sr
#pragma unroll
            for (int j = 0; j < 4; j++) {
                unsigned b = __ballot_sync(FULL, h[j] > 0);
                while (b && found < 2) {
                    const int L = __ffs(b) - 1;
                    b &= b - 1;
                    const int r = nranks - 1 - L - 32 * j;
                    if (found == 0) {
                        mr = r;
                        cnt_mr = __shfl_sync(FULL, h[j], L);
                    } else {
                        sr = r;
                    }
                    found++;
                    if (found == 1 && cnt_mr > 1) found = 2;  // the drop is 0: no second rank needed
                }
            }
        } else {
            for (int r0 = nranks - 1; r0 >= 0 && mr < 0; r0 -= 32) {
                const int r = r0 - lane;
                const bool has = r >= 0 && row[r] > 0;
                const unsigned b = __ballot_sync(FULL, has);
                if (b) mr = r0 - (__ffs(b) - 1);
            }
            if (mr >= 0) cnt_mr = row[mr];
            if (mr >= 0 && cnt_mr == 1) {
                for (int r0 = mr - 1; r0 >= 0 && sr < 0; r0 -= 32) {
                    const int r = r0 - lane;
                    const bool has = r >= 0 && row[r] > 0;
                    const unsigned b = __ballot_sync(FULL, has);
                    if (b) sr = r0 - (__ffs(b) - 1);
                }
            }
        }
        long long mv = 0, ud = 0;
        if (mr >= 0) {
            mv = P.wvals[mr];
            ud = cnt_mr > 1 ? 0 : mv - (sr >= 0 ? P.wvals[sr] : 0);
        }
        if (lane == 0) {
            max_rank[c] = mr;
            max_val[c] = mv;
            mx32[c] = (int32_t)mv;  // class maxima are vertex weights (< 2^31)
            uniq_drop[c] = ud;
        }
    };

    for (;;) {
        if (tid == 0) {
            ctl.work = atomicAdd(P.work_counter, 1);
            ctl.ovf = 0;
        }
        __syncthreads();
        if (ctl.work >= P.nwork) break;
        const int ind = P.work_list ? P.work_list[ctl.work] : ctl.work;
        const uint64_t key = P.keys[ind];
        int32_t *a_io = P.assigns + (size_t)ind * n;
        int32_t *b_out = P.best_assigns + (size_t)ind * n;
        double *phis = P.phi_used + (size_t)ind * (P.rounds + 1);

        // ---------------- init (:120-154) ----------------
        for (int v = tid; v < n; v += NT) {
            int c = a_io[v];
            if (c < 0 || c >= k) {
                atomicExch(P.err_flag, 1);
                c = 0;
            }
            assign[v] = (uint8_t)c;
        }
        // (the table's region is padded to 16 bytes: whole words are zeroed)
        for (size_t i = tid; i < ((size_t)n * k * sizeof(GT) + 3) / 4; i += NT)
            reinterpret_cast<uint32_t *>(gamma)[i] = 0u;
        for (size_t i = tid; i < (size_t)k * nranks; i += NT) wc[i] = 0;
        __syncthreads();
        for (int u = tid; u < n; u += NT) {  // gamma rows owned per thread
            GT *row = gamma + (size_t)u * k;
            bool o = false;
            for (int64_t idx = P.indptr[u]; idx < P.indptr[u + 1]; idx++) {
                GT &x = row[assign[__ldg(P.indices + idx)]];
                if (NARROW && x == (GT)0xFF) o = true;
                else x++;
            }
            if (o) ctl.ovf = 1;
        }
        __syncthreads();
        {  // wc[c][rank] member counts (u16 pairs updated with 32-bit atomics)
            for (int v = tid; v < n; v += NT) {
                const size_t e = (size_t)assign[v] * nranks + wrk[v];
                unsigned int *w32 = reinterpret_cast<unsigned int *>(wc) + (e >> 1);
                atomicAdd(w32, 1u << (16 * (e & 1)));
            }
        }
        __syncthreads();
        for (int c = warp; c < k; c += NW) refresh_class(c);
        __syncthreads();
        // scratch score / conflicts (:70-86)
        {
            long long sc = 0, cf = 0;
            for (int c = tid; c < k; c += NT) sc += max_rank[c] >= 0 ? P.wvals[max_rank[c]] : 0;
            for (int64_t e = tid; e < P.m; e += NT) cf += assign[__ldg(P.eu + e)] == assign[__ldg(P.ev + e)];
            __syncthreads();
            sc = warp_sum64(sc);
            cf = warp_sum64(cf);
            if (lane == 0) {
                ctl.red[warp] = sc;
                ctl.red2[warp] = cf;
            }
            __syncthreads();
            if (tid == 0) {
                long long s = 0, f = 0;
                for (int j = 0; j < NW; j++) {
                    s += ctl.red[j];
                    f += ctl.red2[j];
                }
                ctl.score = s;
                ctl.conflicts = f;
                ctl.best = (f == 0) ? s : INF_SCORE;
                ctl.it = 0;
                ctl.ctr = 0;
                ctl.nlog = 0;
                ctl.diag = 0;
                ctl.phi = P.phi0s[ind];
                phis[0] = ctl.phi;
            }
            __syncthreads();
        }
        if (ctl.conflicts == 0)
            for (int v = tid; v < n; v += NT) b_out[v] = assign[v];

        // the move's bookkeeping (:212-231), one thread: tenure draw on the
        // stream after the scan's `total` tie events, tabu stamp, score /
        // conflicts, log
        auto wv_apply_move = [&](int v, int a, int b, long long mv_ds, long long mv_dc, bool mv_tabu, long long it,
                                 int total, long long score, long long conflicts) {
            unsigned long long c = ctl.ctr;
            uint32_t ll;
            if (!prod) {
                c += (unsigned long long)total;
                ll = u64_below32(key, c, 10u);
                c += 1;
            } else {
                ll = philox_below(key, c + 1, 10u);
                c += 2;
            }
            const long long tt = (long long)ll + P.tt_base;
            tabu_until[v] = (uint32_t)(it + tt + 1);
            ctl.ctr = c;
            ctl.mv_v = v;
            ctl.mv_a = a;
            ctl.mv_b = b;
            ctl.ma_old = mx32[a];  // class maxima before the move (refreshed in the update phase)
            ctl.mb_old = mx32[b];
            ctl.score = score + mv_ds;
            ctl.conflicts = conflicts + mv_dc;
            // best legal score (:233-236); the colouring is copied after the move
            ctl.copy = (ctl.conflicts == 0 && ctl.score < ctl.best);
            if (ctl.copy) ctl.best = ctl.score;
            const long long nl = ctl.nlog;
            if (nl < P.log_cap) {
                const size_t o = (size_t)ind * P.log_cap + nl;
                P.log_v[o] = v;
                P.log_iter[o] = it;
                P.log_tt[o] = tt;
                P.log_asp[o] = mv_tabu ? 1 : 0;
                ctl.nlog = nl + 1;
            }
            if (b < 0) atomicExch(P.err_flag, 3);
        };

        // warp 0, as soon as the moving vertex is known: its neighbour list into
        // shared memory (the L2 round trip overlaps the colour locate)
        // N(v*) into nbuf by asynchronous global -> shared copies: the L2 round
        // trip overlaps the colour locate and the move bookkeeping; warp 0 waits
        // for them (__pipeline_wait_prior) just before the barrier that
        // publishes the move
        auto fetch_nbrs = [&](int v) {
            const int e0 = ip32[v], d = ip32[v + 1] - e0;
            for (int i = lane; i < d; i += 32) __pipeline_memcpy_async(nbuf + i, P.indices + e0 + i, 4);
            __pipeline_commit();
            if (lane == 0) ctl.deg = d;
        };

        // ---------------- rounds (:156-258) ----------------
        for (int64_t rnd = 0; rnd < P.rounds; rnd++) {
            if (NARROW && ctl.ovf) break;  // read after a barrier: uniform
            if (tid == 0 && P.schedule_on && rnd == P.rounds - 1) {
                ctl.phi = P.forced_phi;
                phis[P.rounds] = ctl.phi;
            }
            for (int v = tid; v < n; v += NT) tabu_until[v] = 0;
            {
                uint32_t *nbits = reinterpret_cast<uint32_t *>(lowR) + ((size_t)n + 1) / 2;  // after the u16 counts
                for (int i = tid; i < 2 * ((n + 31) / 32); i += NT) nbits[i] = 0u;
                if (tid == 0) ctl.inc = 0;
            }
            // the objective's exact-integer mode depends on phi only: once per round
            __shared__ GvMode s_gm;
            __shared__ int s_fast32;
            if (tid == 0) {
                const GvMode g0 = gv_mode(ctl.phi, n);
                s_gm = g0;
                // 32-bit numerators when |t| n + maxw 2^s < 2^30 (|dc| <= n, |ds| <= maxw)
                s_fast32 = g0.fast && (long long)(g0.t < 0 ? -g0.t : g0.t) * n + ((long long)s_maxw << g0.s) < (1ll << 30);
            }
            __syncthreads();
            // phase counters live in shared memory (thread 0 only): no registers
            // held across the iteration when the flag is off
            __shared__ unsigned long long s_wsa[9];
            __shared__ long long s_wt0;
            constexpr bool wst = STATS;
            if (wst && tid == 0)
                for (int i = 0; i < 9; i++) s_wsa[i] = 0;
#define WVPH(i)                                              \
    if (wst && tid == 0) {                                   \
        const long long t1 = clock64();                      \
        s_wsa[i] += (unsigned long long)(t1 - s_wt0);        \
        s_wt0 = t1;                                          \
    }
            for (int64_t step = 0; step < P.depth; step++) {
                if (wst && tid == 0) {
                    s_wsa[0]++;
                    s_wt0 = clock64();
                }
                const long long it = ctl.it, score = ctl.score, conflicts = ctl.conflicts,
                                best = ctl.best;
                const GvMode gm = s_gm;
                const bool fast32 = s_fast32 != 0;
                // pass 1: (min g, count) per vertex row over admissible candidates
                const int nch = (n + 31) >> 5;
                if (fast32 && nch <= 32) {
                    // ================= exact 32-bit path (all arrays int) =================
                    const int S = gm.s, Tt = (int)gm.t;
                    // 32-bit forms of the iteration scalars (it < 2^32 as the u32 expiries
                    // assume, conflicts <= m < 2^31; score + ds >= best <=> ds >= room,
                    // clamping best - score keeps that exact): fewer live registers
                    const uint32_t it32 = (uint32_t)it;
                    const int conf32 = (int)min(conflicts, (long long)INT_MAX);
                    const int room32 = (int)max(min(best - score, (long long)INT_MAX), (long long)INT_MIN);
                    int32_t *r32 = reinterpret_cast<int32_t *>(rmin);  // row minima (numerators)
                    int32_t *c_min = lowq;                           // [32] chunk minima
                    int32_t *c_cnt = lowq + 32;                      // [32] multiplicity at the chunk minimum
                    int32_t *q = lowq + 64;                          // walk queue (row, entering minimum)
                    int32_t *hc_min = r32 + n;                       // row caches (rmin's second half)
                    uint16_t *hc_cnt = reinterpret_cast<uint16_t *>(lowR);
                    const uint32_t *nbr_bits = reinterpret_cast<const uint32_t *>(lowR) + ((size_t)n + 1) / 2 +
                                               (size_t)((it32 - 1u) & 1u) * ((n + 31) / 32);
                    const int inc = ctl.inc, mvv = ctl.mv_v, mva = ctl.mv_a, mvb = ctl.mv_b;
                    const int mao = ctl.ma_old, mbo = ctl.mb_old;
                    // class maxima moved by the last move (rows not adjacent to v* see
                    // columns a* / b* change only through them)
                    const bool a_moved = inc == 1 && mao != mx32[mva], b_moved = inc == 1 && mbo != mx32[mvb];
                    // pass 1, rows warp-uniform (chunk = warp + NW j): every row's
                    // (min G, #candidates at it), then the chunk's minimum and multiplicity
                    for (int v0 = warp * 32; v0 < n; v0 += NT) {
                        const int v = v0 + lane;
                        int m = INT_MAX, cnt = 0, mh = INT_MAX;
                        int a = 0, rem = 0, gva = 0, wv = 0;
                        bool full = false;
                        if (v < n) {
                            a = assign[v];
                            rem = (wrk[v] == max_rank[a]) ? (int)uniq_drop[a] : 0;
                            const GT *row = gamma + (size_t)v * k;
                            gva = row[a];
                            const bool frozen = it32 < tabu_until[v];
                            wv = wgt[v];
                            if (!frozen) {
                                // G = (ds << S) + t dc = H_c + K with the row constant
                                // K = -(rem << S) - t gva and H_c = (max(0, w_v - M_c) << S)
                                // + t gamma_c; the (min, multiplicity) over H (own colour
                                // excluded) is cached per row: after a move v*: a* -> b*
                                // only columns a* and b* change for any row (gamma of v*'s
                                // neighbours, the two class maxima), so a valid cache is
                                // updated with those two columns -- old contributions out,
                                // new ones in -- and the row is rescanned (below, by the
                                // whole warp) when its minimum group empties, after it was
                                // frozen, for v* itself and at round start (ctl.inc == 0)
                                full = true;
                                if (inc != 0 && hc_cnt[v] != 0xFFFFu && !(inc == 1 && v == mvv)) {
                                    mh = hc_min[v];
                                    cnt = hc_cnt[v];
                                    full = false;
                                    if (inc == 1) {
                                        const int nb = (int)((nbr_bits[v >> 5] >> (v & 31)) & 1u);
                                        int hn[2], nx = 0;
#pragma unroll
                                        for (int side = 0; side < 2; side++) {
                                            const int x = side ? mvb : mva;
                                            if (x == a) continue;  // the own colour is not a candidate
                                            // unchanged column: out and in again is a no-op (and
                                            // would empty a unique minimum group for nothing)
                                            if (!nb && !(side ? b_moved : a_moved)) continue;
                                            const int gnew = (int)row[x];
                                            const int gold = gnew + (side ? -nb : nb);  // a*: -1, b*: +1 on N(v*)
                                            const int hold = (max(0, wv - (side ? mbo : mao)) << S) + Tt * gold;
                                            if (hold == mh) cnt--;
                                            hn[nx++] = (max(0, wv - mx32[x]) << S) + Tt * gnew;
                                        }
                                        if (cnt == 0) {
                                            full = true;  // the minimum group emptied
                                        } else {
                                            for (int i2 = 0; i2 < nx; i2++) {
                                                cnt = (hn[i2] < mh) ? 1 : cnt + (hn[i2] == mh);
                                                mh = min(mh, hn[i2]);
                                            }
                                        }
                                    }
                                }
                            } else {
                                hc_cnt[v] = 0xFFFFu;
                                if (conf32 <= gva && (long long)rem + room32 > 0) {
                                    // (a frozen row needs ds = max(0, w - M_c) - rem < best - score:
                                    // impossible when rem + best - score <= 0, e.g. every row
                                    // whose move cannot lower a class maximum at a legal state)
                                    // frozen vertex: only legal moves (dc == -conflicts, reachable
                                    // only if conflicts <= gva) that beat the best legal score
                                    const int need_dc = -conf32;
                                    const int dsmax = room32;  // ds < best - score
                                    auto cand = [&](int c) {
                                        const int ds = max(0, wv - mx32[c]) - rem;
                                        if (c != a && ds < dsmax) {
                                            const int G = (ds << S) + Tt * need_dc;
                                            cnt = (G < m) ? 1 : cnt + (G == m);
                                            m = min(m, G);
                                        }
                                    };
                                    if (NARROW && (k & 3) == 0) {
                                        // only colours with gamma == gva - conflicts qualify:
                                        // found 4 at a time by a byte-equality mask
                                        const uint32_t *r32w = reinterpret_cast<const uint32_t *>(row);
                                        const uint32_t t4 = (uint32_t)(gva + need_dc) * 0x01010101u;
                                        for (int w = 0; w < (k >> 2); w++) {
                                            const uint32_t z = r32w[w] ^ t4;
                                            uint32_t eq = ~(((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & 0x80808080u;
                                            while (eq) {
                                                cand(4 * w + ((__ffs(eq) - 1) >> 3));
                                                eq &= eq - 1u;
                                            }
                                        }
                                    } else {
                                        for (int c = 0; c < k; c++)
                                            if ((int)row[c] - gva == need_dc) cand(c);
                                    }
                                }
                            }
                        }
                        // full rescans of this chunk's rows by the whole warp: lanes over
                        // colours, minimum by REDUX, multiplicity by ballots
                        for (unsigned rs = __ballot_sync(FULL, full); rs; rs &= rs - 1) {
                            const int src = __ffs(rs) - 1;
                            const int au = __shfl_sync(FULL, a, src), wu = __shfl_sync(FULL, wv, src);
                            const GT *ru = gamma + (size_t)(v0 + src) * k;
                            int hm, hcn = 0;
                            if (k <= 64) {  // each lane's two colours evaluated once
                                const int c0 = lane, c1 = lane + 32;
                                const int h0 = (c0 < k && c0 != au) ? (max(0, wu - mx32[c0]) << S) + Tt * (int)ru[c0] : INT_MAX;
                                const int h1 = (c1 < k && c1 != au) ? (max(0, wu - mx32[c1]) << S) + Tt * (int)ru[c1] : INT_MAX;
                                hm = __reduce_min_sync(FULL, min(h0, h1));
                                hcn = __popc(__ballot_sync(FULL, h0 == hm)) + __popc(__ballot_sync(FULL, h1 == hm));
                            } else {
                                int lmin = INT_MAX;
                                for (int cb = 0; cb < k; cb += 32) {
                                    const int c = cb + lane;
                                    if (c < k && c != au) lmin = min(lmin, (max(0, wu - mx32[c]) << S) + Tt * (int)ru[c]);
                                }
                                hm = __reduce_min_sync(FULL, lmin);
                                for (int cb = 0; cb < k; cb += 32) {
                                    const int c = cb + lane;
                                    const bool eq = c < k && c != au && (max(0, wu - mx32[c]) << S) + Tt * (int)ru[c] == hm;
                                    hcn += __popc(__ballot_sync(FULL, eq));
                                }
                            }
                            if (lane == src) {
                                mh = hm;
                                cnt = hm == INT_MAX ? 0 : hcn;
                            }
                        }
                        if (v < n) {
                            if (it32 >= tabu_until[v]) {  // not frozen: the cache and the row minimum
                                hc_min[v] = mh;
                                hc_cnt[v] = (uint16_t)cnt;
                                m = (mh == INT_MAX) ? INT_MAX : mh - (rem << S) - Tt * gva;
                            }
                            r32[v] = m;
                            rcnt[v] = (uint16_t)(m == INT_MAX ? 0 : cnt);
                        }
                        const int cm = __reduce_min_sync(FULL, m);
                        const int cc = __reduce_add_sync(FULL, (m == cm && m != INT_MAX) ? cnt : 0);
                        if (lane == 0) {
                            c_min[v0 >> 5] = cm;
                            c_cnt[v0 >> 5] = cc;
                        }
                    }
                    if (tid == 0) s_nlow = 0;
                    __syncthreads();
                    WVPH(1);
                    // prefix minimum over the rows in vertex order: every chunk's entering
                    // minimum from one scan over the chunk minima; only chunks reaching
                    // the running minimum hold tie events or rows that lower it
                    const int cmv = lane < nch ? c_min[lane] : INT_MAX;
                    int cin_all = cmv;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t2 = __shfl_up_sync(FULL, cin_all, o);
                        if (lane >= o) cin_all = min(cin_all, t2);
                    }
                    const int D = __shfl_sync(FULL, cin_all, 31);
                    int cex = __shfl_up_sync(FULL, cin_all, 1);
                    if (lane == 0) cex = INT_MAX;
                    int tsum = 0;
                    if (!prod && D != INT_MAX) {
                        for (int cb = warp; cb < nch; cb += NW) {
                            const int cin = __shfl_sync(FULL, cex, cb);
                            if (__shfl_sync(FULL, cmv, cb) > cin) continue;  // no row at or below it
                            const int v = cb * 32 + lane;
                            const int x = v < n ? r32[v] : INT_MAX;
                            const int nq = v < n ? rcnt[v] : 0;
                            int incl = x;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const int t2 = __shfl_up_sync(FULL, incl, o);
                                if (lane >= o) incl = min(incl, t2);
                            }
                            int excl = __shfl_up_sync(FULL, incl, 1);
                            if (lane == 0) excl = INT_MAX;
                            const int RM = min(cin, excl);
                            if (x != INT_MAX) {
                                if (x == RM) {
                                    tsum += nq;
                                } else if (x < RM) {
                                    const int pos = atomicAdd(&s_nlow, 1);
                                    q[2 * pos] = v;
                                    q[2 * pos + 1] = RM;
                                }
                            }
                        }
                    }
                    {
                        const int wts = __reduce_add_sync(FULL, tsum);
                        if (lane == 0) s_wts[warp] = wts;
                    }
                    __syncthreads();
                    WVPH(2);
                    // walks of the rows that lower the running minimum (their tie
                    // events in colour order, :194-210), spread over the warps
                    {   // the neighbour flags pass 1 read are dead: clear them for the move after next
                        uint32_t *nb_clear = reinterpret_cast<uint32_t *>(lowR) + ((size_t)n + 1) / 2 +
                                             (size_t)((it32 - 1u) & 1u) * ((n + 31) / 32);
                        for (int i = tid; i < (n + 31) / 32; i += NT) nb_clear[i] = 0u;
                    }
                    {
                        int tw = 0;
                        const int nlow = s_nlow;
                        for (int i = warp; i < nlow; i += NW) {
                            const int wvx = q[2 * i], R = q[2 * i + 1];
                            const int a = assign[wvx];
                            const int rem = (wrk[wvx] == max_rank[a]) ? (int)uniq_drop[a] : 0;
                            const GT *row = gamma + (size_t)wvx * k;
                            const int gva = row[a];
                            const bool frozen = it32 < tabu_until[wvx];
                            const int wv = wgt[wvx];
                            int cr = R;
                            for (int c0 = 0; c0 < k; c0 += 32) {
                                const int c = c0 + lane;
                                int G = INT_MAX;
                                if (c < k && c != a) {
                                    const int dc = (int)row[c] - gva;
                                    const int ds = max(0, wv - mx32[c]) - rem;
                                    if (!(frozen && (dc != -conf32 || ds >= room32))) G = (ds << S) + Tt * dc;
                                }
                                int inc2 = G;
#pragma unroll
                                for (int o = 1; o < 32; o <<= 1) {
                                    const int t2 = __shfl_up_sync(FULL, inc2, o);
                                    if (lane >= o) inc2 = min(inc2, t2);
                                }
                                int ex2 = __shfl_up_sync(FULL, inc2, 1);
                                if (lane == 0) ex2 = INT_MAX;
                                if (G != INT_MAX && G == min(cr, ex2)) tw++;
                                cr = min(cr, __shfl_sync(FULL, inc2, 31));
                            }
                        }
                        const int wtw = __reduce_add_sync(FULL, tw);
                        if (lane == 0) s_wts2[warp] = wtw;
                    }
                    __syncthreads();
                    WVPH(3);
                    if (warp == 0) {
                        long long t_sp = (wst && lane == 0) ? clock64() : 0;
#define WVSP(i)                                                             \
    if (wst && lane == 0) {                                                 \
        const long long _t = clock64();                                     \
        atomicAdd(&g_wvstats[9 + (i)], (unsigned long long)(_t - t_sp));    \
        t_sp = _t;                                                          \
    }
                        const int total = __reduce_add_sync(FULL, lane < NW ? s_wts[lane] + s_wts2[lane] : 0);
                        int mv_v = -1;
                        if (D != INT_MAX) {
                            const int cc = (lane < nch && cmv == D) ? c_cnt[lane] : 0;
                            const int T = __reduce_add_sync(FULL, cc);
                            const unsigned long long ctr = ctl.ctr;
                            int sstar = 1;
                            if (T > 1) {
                                if (!prod) {
                                    const unsigned long long c0 = ctr + (unsigned long long)(total - (T - 1));
                                    int smax = 1;
                                    for (int s2 = 2 + lane; s2 <= T; s2 += 32)
                                        if (divisible_wv(stream_value(key, c0 + (unsigned long long)(s2 - 2)), (uint32_t)s2))
                                            smax = s2;
                                    sstar = __reduce_max_sync(FULL, smax);
                                } else {
                                    sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                                }
                            }
                            WVSP(0);
                            // the chunk, then the row holding the sstar-th D-candidate
                            const int ci = warp_incl_sum(cc, lane);
                            const int ch = __ffs(__ballot_sync(FULL, ci >= sstar)) - 1;
                            const int before = __shfl_sync(FULL, ci - cc, ch);
                            const int vv = ch * 32 + lane;
                            const int c1 = (vv < n && r32[vv] == D) ? rcnt[vv] : 0;
                            const int incl = warp_incl_sum(c1, lane);
                            const int src = __ffs(__ballot_sync(FULL, before + incl >= sstar)) - 1;
                            const int v = ch * 32 + src;
                            WVSP(1);
                            fetch_nbrs(v);
                            const int need = sstar - before - __shfl_sync(FULL, incl - c1, src);
                            // within the row: the need-th colour with G == D
                            const int a = assign[v];
                            const int rem = (wrk[v] == max_rank[a]) ? (int)uniq_drop[a] : 0;
                            const GT *rw = gamma + (size_t)v * k;
                            const int gva = rw[a];
                            const bool frozen = it32 < tabu_until[v];
                            const int wv = wgt[v];
                            int cum = 0, b = -1, bds = 0, bdc = 0;
                            for (int c0 = 0; c0 < k && b < 0; c0 += 32) {
                                const int c = c0 + lane;
                                bool hit = false;
                                int ds = 0, dc = 0;
                                if (c < k && c != a) {
                                    dc = (int)rw[c] - gva;
                                    ds = max(0, wv - mx32[c]) - rem;
                                    if (!(frozen && (dc != -conf32 || ds >= room32)))
                                        hit = (ds << S) + Tt * dc == D;
                                }
                                const unsigned hm = __ballot_sync(FULL, hit);
                                const int hc = __popc(hm);
                                if (cum + hc >= need) {
                                    unsigned mm = hm;
                                    for (int q2 = 1; q2 < need - cum; q2++) mm &= mm - 1u;
                                    const int sl = __ffs(mm) - 1;
                                    b = c0 + sl;
                                    bds = __shfl_sync(FULL, ds, sl);
                                    bdc = __shfl_sync(FULL, dc, sl);
                                }
                                cum += hc;
                            }
                            mv_v = v;
                            WVSP(2);
                            if (lane == 0) wv_apply_move(v, a, b, bds, bdc, frozen, ctl.it, total, ctl.score, ctl.conflicts);
                            WVSP(3);
                        }
                        if (lane == 0) ctl.has_move = (mv_v >= 0);
                        __pipeline_wait_prior(0);
                        WVSP(4);
#undef WVSP
                    }
                } else {
                // pass 1: (min g, count) per vertex row over admissible candidates
                if (gm.fast) {
                    // exact integer numerators (see gv_mode)
                    for (int v = tid; v < n; v += NT) {
                        const int a = assign[v];
                        const long long rem = (wrk[v] == max_rank[a]) ? uniq_drop[a] : 0;
                        const GT *row = gamma + (size_t)v * k;
                        const int gva = row[a];
                        const bool frozen = (uint64_t)it < tabu_until[v];
                        const long long wv = wgt[v];
                        long long m = LLONG_MAX;
                        int cnt = 0;
                        for (int c = 0; c < k; c++) {
                            const long long dc = (long long)row[c] - gva;
                            long long dadd = wv - max_val[c];
                            if (dadd < 0) dadd = 0;
                            const long long ds = dadd - rem;
                            const bool skip = (c == a) || (frozen && (conflicts + dc != 0 || score + ds >= best));
                            const long long G = skip ? LLONG_MAX : gnum(gm, ds, dc);
                            cnt = (G < m) ? 1 : cnt + (G == m && G != LLONG_MAX);
                            m = min(m, G);
                        }
                        rmin[v] = (m == LLONG_MAX) ? INF : (double)m;
                        rcnt[v] = (uint16_t)cnt;
                    }
                } else
                for (int v = tid; v < n; v += NT) {
                    const int a = assign[v];
                    const long long rem = (wrk[v] == max_rank[a]) ? uniq_drop[a] : 0;
                    const GT *row = gamma + (size_t)v * k;
                    const int gva = row[a];
                    const bool frozen = (uint64_t)it < tabu_until[v];
                    const long long wv = wgt[v];
                    double m = INF;
                    int cnt = 0;
                    for (int c = 0; c < k; c++) {
                        if (c == a) continue;
                        const long long dc = (long long)row[c] - gva;
                        long long dadd = wv - max_val[c];
                        if (dadd < 0) dadd = 0;
                        const long long ds = dadd - rem;
                        if (frozen && (conflicts + dc != 0 || score + ds >= best)) continue;
                        const double gv = gval_of(ds, dc, gm.phi);
                        if (gv < m) {
                            m = gv;
                            cnt = 1;
                        } else if (gv == m) {
                            cnt++;
                        }
                    }
                    rmin[v] = m;
                    rcnt[v] = (uint16_t)cnt;
                }
                __syncthreads();
                WVPH(1);
                // prefix-min over the rows in vertex order, parallel over the warps:
                // chunks of 32 rows (warp w: chunks w, w + NW, ...); (1) chunk
                // minima; (2) each warp enters its chunks with the minimum of the
                // chunks before, counts the tie events of rows equal to the running
                // minimum and walks the rows that lower it; (3) warp 0 combines.
                double *s_cmin = lowR;  // chunk minima (n >= #chunks)
                __shared__ double s_wmin[NW];
                __shared__ int s_wT[NW], s_wfirst[NW], s_wtsum[NW];
                const int nch = (n + 31) >> 5;
                for (int cb = warp; cb < nch; cb += NW) {
                    const int v = cb * 32 + lane;
                    double x = v < n ? rmin[v] : INF;
                    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __longlong_as_double(__shfl_xor_sync(
                                                                     FULL, __double_as_longlong(x), o)));
                    if (lane == 0) s_cmin[cb] = x;
                }
                __syncthreads();
                WVPH(2);
                {
                    double lmin = INF;
                    int lT = 0, lfirst = INT_MAX, tsum = 0;
                    for (int cb = warp; cb < nch; cb += NW) {
                        // running minimum entering this chunk
                        double cin = INF;
                        for (int j = lane; j < cb; j += 32) cin = fmin(cin, s_cmin[j]);
                        for (int o = 16; o > 0; o >>= 1) cin = fmin(cin, __longlong_as_double(__shfl_xor_sync(
                                                                           FULL, __double_as_longlong(cin), o)));
                        const int v = cb * 32 + lane;
                        const double x = v < n ? rmin[v] : INF;
                        const int nq = v < n ? rcnt[v] : 0;
                        double incl = x;
                        for (int o = 1; o < 32; o <<= 1) {
                            const double t = shfl_up_d(incl, o);
                            if (lane >= o) incl = fmin(incl, t);
                        }
                        double excl = shfl_up_d(incl, 1);
                        if (lane == 0) excl = INF;
                        const double RM = fmin(cin, excl);
                        if (x < lmin) {
                            lmin = x;
                            lT = nq;
                            lfirst = v;
                        } else if (x == lmin && x != INF) {
                            lT += nq;
                        }
                        bool low = false;
                        if (!prod && x != INF) {
                            if (x == RM) tsum += nq;
                            else if (x < RM) low = true;
                        }
                        // walk the rows that lower the running minimum (lanes over colours)
                        unsigned lb = __ballot_sync(FULL, low);
                        while (lb) {
                            const int src = __ffs(lb) - 1;
                            lb &= lb - 1;
                            const int wvx = cb * 32 + src;
                            const double R = shfl_d(RM, src);
                            const int a = assign[wvx];
                            const long long rem = (wrk[wvx] == max_rank[a]) ? uniq_drop[a] : 0;
                            const GT *row = gamma + (size_t)wvx * k;
                            const int gva = row[a];
                            const bool frozen = (uint64_t)it < tabu_until[wvx];
                            const long long wv = wgt[wvx];
                            double cr = R;
                            int t = 0;
                            for (int c0 = 0; c0 < k; c0 += 32) {
                                const int c = c0 + lane;
                                double gv = INF;
                                if (c < k && c != a) {
                                    const long long dc = (long long)row[c] - gva;
                                    long long dadd = wv - max_val[c];
                                    if (dadd < 0) dadd = 0;
                                    const long long ds = dadd - rem;
                                    if (!(frozen && (conflicts + dc != 0 || score + ds >= best)))
                                        gv = gval(gm, ds, dc);
                                }
                                double inc2 = gv;
                                for (int o = 1; o < 32; o <<= 1) {
                                    const double tt = shfl_up_d(inc2, o);
                                    if (lane >= o) inc2 = fmin(inc2, tt);
                                }
                                double ex2 = shfl_up_d(inc2, 1);
                                if (lane == 0) ex2 = INF;
                                const double cur = fmin(cr, ex2);
                                if (gv != INF && gv == cur) t++;
                                cr = fmin(cr, shfl_d(inc2, 31));
                            }
                            tsum += (lane == 0) ? __reduce_add_sync(FULL, t) : (__reduce_add_sync(FULL, t), 0);
                        }
                    }
                    // warp partials: minimum, its multiplicity, first row, tie events
                    double wm = lmin;
                    for (int o = 16; o > 0; o >>= 1)
                        wm = fmin(wm, __longlong_as_double(__shfl_xor_sync(FULL, __double_as_longlong(wm), o)));
                    const int wT = __reduce_add_sync(FULL, lmin == wm ? lT : 0);
                    const int wf = (int)__reduce_min_sync(FULL, (unsigned)(lmin == wm ? lfirst : INT_MAX));
                    const int wts = __reduce_add_sync(FULL, tsum);
                    if (lane == 0) {
                        s_wmin[warp] = wm;
                        s_wT[warp] = wT;
                        s_wfirst[warp] = wf;
                        s_wtsum[warp] = wts;
                    }
                }
                __syncthreads();
                WVPH(3);
                if (warp == 0) {
                    // lane w carries warp w's partials into the combination below
                    double lmin = lane < NW ? s_wmin[lane] : INF;
                    const int lT = lane < NW ? s_wT[lane] : 0;
                    const int lfirst = lane < NW ? s_wfirst[lane] : INT_MAX;
                    const int tsum = lane < NW ? s_wtsum[lane] : 0;
                    double carry = lmin;
                    for (int o = 16; o > 0; o >>= 1)
                        carry = fmin(carry, __longlong_as_double(__shfl_xor_sync(FULL, __double_as_longlong(carry), o)));
                    const double D = carry;
                    int mv_v = -1;
                    long long mv_ds = 0, mv_dc = 0;
                    bool mv_tabu = false;
                    if (D != INF) {
                        // all lanes agree on D; T, first row, total ties
                        const int T = __reduce_add_sync(FULL, lmin == D ? lT : 0);
                        const int L = (int)__reduce_min_sync(FULL, (unsigned)(lmin == D ? lfirst : INT_MAX));
                        const int total = __reduce_add_sync(FULL, tsum);
                        const unsigned long long ctr = ctl.ctr;
                        int sstar = 1;
                        if (T > 1) {
                            if (!prod) {
                                const unsigned long long c0 = ctr + (unsigned long long)(total - (T - 1));
                                int smax = 1;
                                for (int s = 2 + lane; s <= T; s += 32)
                                    if (divisible_wv(stream_value(key, c0 + (unsigned long long)(s - 2)), (uint32_t)s))
                                        smax = s;
                                sstar = __reduce_max_sync(FULL, smax);
                            } else {
                                sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                            }
                        }
                        int row = L, need = 1;
                        const int nchk = (n + 31) >> 5;
                        if (sstar > 1 && nchk <= 32) {
                            // lane = chunk of 32 rows: D-candidate counts per chunk, one scan
                            // over the chunks, one within the chosen chunk
                            int cs = 0;
                            if (lane < nchk)
                                for (int r = 0; r < 32; r++) {
                                    const int vv = lane * 32 + r;
                                    if (vv < n && rmin[vv] == D) cs += rcnt[vv];
                                }
                            const int ci = warp_incl_sum(cs, lane);
                            const unsigned cb = __ballot_sync(FULL, ci >= sstar);
                            const int ch = __ffs(cb) - 1;
                            const int before = __shfl_sync(FULL, ci - cs, ch);
                            const int vv = ch * 32 + lane;
                            const int c = (vv < n && rmin[vv] == D) ? rcnt[vv] : 0;
                            const int incl = warp_incl_sum(c, lane);
                            const unsigned bm = __ballot_sync(FULL, before + incl >= sstar);
                            const int src = __ffs(bm) - 1;
                            row = ch * 32 + src;
                            need = sstar - before - __shfl_sync(FULL, incl - c, src);
                        } else if (sstar > 1) {
                            int cum = 0;
                            for (int base = 0; base < n; base += 32) {
                                const int v = base + lane;
                                const int c = (v < n && rmin[v] == D) ? rcnt[v] : 0;
                                const int incl = warp_incl_sum(c, lane);
                                const int tot = __shfl_sync(FULL, incl, 31);
                                if (cum + tot >= sstar) {
                                    const unsigned bm = __ballot_sync(FULL, cum + incl >= sstar);
                                    const int src = __ffs(bm) - 1;
                                    row = base + src;
                                    need = sstar - cum - __shfl_sync(FULL, incl - c, src);
                                    break;
                                }
                                cum += tot;
                            }
                        }
                        // within the row: the need-th colour with g == D
                        const int v = row;
                        fetch_nbrs(v);
                        const int a = assign[v];
                        const long long rem = (wrk[v] == max_rank[a]) ? uniq_drop[a] : 0;
                        const GT *rw = gamma + (size_t)v * k;
                        const int gva = rw[a];
                        const bool frozen = (uint64_t)it < tabu_until[v];
                        const long long wv = wgt[v];
                        int cum = 0, b = -1;
                        long long bds = 0, bdc = 0;
                        for (int c0 = 0; c0 < k && b < 0; c0 += 32) {
                            const int c = c0 + lane;
                            bool hit = false;
                            long long ds = 0, dc = 0;
                            if (c < k && c != a) {
                                dc = (long long)rw[c] - gva;
                                long long dadd = wv - max_val[c];
                                if (dadd < 0) dadd = 0;
                                ds = dadd - rem;
                                if (!(frozen && (conflicts + dc != 0 || score + ds >= best)))
                                    hit = gval(gm, ds, dc) == D;
                            }
                            const unsigned hm = __ballot_sync(FULL, hit);
                            const int hc = __popc(hm);
                            if (cum + hc >= need) {
                                unsigned mm = hm;
                                for (int q = 1; q < need - cum; q++) mm &= mm - 1u;
                                const int src = __ffs(mm) - 1;
                                b = c0 + src;
                                bds = __shfl_sync(FULL, ds, src);
                                bdc = __shfl_sync(FULL, dc, src);
                            }
                            cum += hc;
                        }
                        mv_v = v;
                        mv_ds = bds;
                        mv_dc = bdc;
                        mv_tabu = frozen;
                        if (lane == 0) wv_apply_move(v, a, b, mv_ds, mv_dc, mv_tabu, it, total, score, conflicts);
                    }
                    if (lane == 0) ctl.has_move = (mv_v >= 0);
                    __pipeline_wait_prior(0);
                }
                }
                __syncthreads();
                WVPH(4);
                const bool moved = ctl.has_move;
                if (moved) {
                    // gamma over N(v) (:218-221) by all threads; warp 0 / warp 1 move v
                    // between the weight-rank counts of classes a / b and refresh them
                    const int v = ctl.mv_v, a = ctl.mv_a, b = ctl.mv_b, deg = ctl.deg;
                    uint32_t *nbw = reinterpret_cast<uint32_t *>(lowR) + ((size_t)n + 1) / 2 +
                                    (size_t)(it & 1) * ((n + 31) / 32);
                    for (int i = tid; i < deg; i += NT) {
                        const int u = nbuf[i];
                        atomicOr(&nbw[u >> 5], 1u << (u & 31));  // the 32-bit path's row caches read this
                        gamma[(size_t)u * k + a]--;
                        const GT old = gamma[(size_t)u * k + b];
                        if (NARROW && old == (GT)0xFF) ctl.ovf = 1;
                        gamma[(size_t)u * k + b] = (GT)(old + 1);
                    }
                    if (warp <= 1) {
                        const int c = warp == 0 ? a : b;
                        if (lane == 0) wc[(size_t)c * nranks + wrk[v]] += (warp == 0) ? (uint16_t)0xFFFF : (uint16_t)1;
                        __syncwarp();
                        refresh_class(c);
                        if (warp == 1 && lane == 0) assign[v] = (uint8_t)b;
                    }
                }
                if (tid == 0) {
                    ctl.it = it + 1;
                    ctl.inc = (fast32 && nch <= 32) ? (moved ? 1 : 2) : 0;  // row caches valid after a 32-bit pass 1
                }
                __syncthreads();
                WVPH(5);
                if (moved && ctl.copy)
                    for (int u = tid; u < n; u += NT) b_out[u] = assign[u];
                const long long itn = it + 1;
                if (diagf && itn % 1024 == 0) {  // scratch check (:245-249)
                    for (int c = tid; c < k; c += NT) cmax[c] = -1;
                    __syncthreads();
                    for (int u = tid; u < n; u += NT) atomicMax(&cmax[assign[u]], (int)wrk[u]);
                    long long cf = 0;
                    for (int64_t e = tid; e < P.m; e += NT) cf += assign[__ldg(P.eu + e)] == assign[__ldg(P.ev + e)];
                    __syncthreads();
                    long long sc = 0;
                    for (int c = tid; c < k; c += NT) sc += cmax[c] >= 0 ? P.wvals[cmax[c]] : 0;
                    sc = warp_sum64(sc);
                    cf = warp_sum64(cf);
                    if (lane == 0) {
                        ctl.red[warp] = sc;
                        ctl.red2[warp] = cf;
                    }
                    __syncthreads();
                    if (tid == 0) {
                        long long s = 0, f = 0;
                        for (int j = 0; j < NW; j++) {
                            s += ctl.red[j];
                            f += ctl.red2[j];
                        }
                        if (s != ctl.score || f != ctl.conflicts) ctl.diag += 1;
                    }
                }
                // (no barrier here: the next iteration's first writes are ordered
                // behind its pass-1 barrier, every read of this one's results is done)
                WVPH(8);
                if (NARROW && ctl.ovf) break;
            }
            if (wst && tid == 0)
                for (int i = 0; i < 9; i++) atomicAdd(&g_wvstats[i], s_wsa[i]);
#undef WVPH
            if (tid == 0) {  // phi schedule (:251-258)
                if (P.schedule_on && rnd < P.rounds - 1) {
                    ctl.phi = (ctl.conflicts == 0) ? ctl.phi / 2.0 : ctl.phi * 2.0;
                    phis[rnd + 1] = ctl.phi;
                } else if (!P.schedule_on) {
                    phis[rnd + 1] = ctl.phi;
                }
            }
            __syncthreads();
        }
        if (NARROW && ctl.ovf) {
            if (tid == 0) P.ovf_list[atomicAdd(P.ovf_count, 1)] = ind;
            __syncthreads();
            continue;
        }
        for (int v = tid; v < n; v += NT) a_io[v] = assign[v];
        if (tid == 0) {
            P.end_scores[ind] = ctl.score;
            P.end_conflicts[ind] = ctl.conflicts;
            P.best_scores[ind] = ctl.best;
            P.diag[ind] = ctl.diag;
            if (P.log_cnt) P.log_cnt[ind] = ctl.nlog;
        }
        __syncthreads();
    }
}

// segment sizes in WvSeg order, each 16-byte aligned; so[WV_NSEG] = total
static size_t wv_layout(int n, int k, int gbytes, uint32_t *so) {
    const size_t N = (size_t)n, K = (size_t)k;
    const size_t bytes[WV_NSEG] = {N * K * gbytes, N * 4, N * 4, N * 2, N, N * 8, N * 2, K * 4,
                                   K * 8,          K * 8, K * 4, K * 4, (2 * N + 64) * 4, (N + 1) * 4,
                                   N * 4,          N * 8};
    size_t off = 0;
    for (int i = 0; i < WV_NSEG; i++) {
        if (so) so[i] = (uint32_t)off;
        off += (bytes[i] + 15) & ~(size_t)15;
    }
    if (so) so[WV_NSEG] = (uint32_t)off;
    return off;
}
static size_t wv_smem(int n, int k, int gbytes) { return wv_layout(n, k, gbytes, nullptr); }

static int upload_divtab_wv(cudaStream_t st) {
    static bool done[64] = {false};
    int d = 0;
    cudaGetDevice(&d);
    if (done[d & 63]) return MCB_OK;
    ulonglong2 tab[32];
    for (int i = 0; i < 32; i++) {
        const uint64_t o = 2 * (uint64_t)i + 1;
        uint64_t x = o;  // Newton: inverse of o modulo 2^64
        for (int r = 0; r < 6; r++) x *= 2 - o * x;
        tab[i] = make_ulonglong2(x, ~0ull / o);
    }
    if (cudaMemcpyToSymbolAsync(g_divtab_wv, tab, sizeof(tab), 0, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "wvcp: divisor table upload failed");
    done[d & 63] = true;
    return MCB_OK;
}

template <typename GT, bool STATS>
static int wvcp_launch_t(WvParams P, int64_t nwork, cudaStream_t st, uint8_t *ws_base, size_t ws_cap_ctas,
                         size_t wc_stride) {
    if (int rc = upload_divtab_wv(st)) return rc;
    const size_t smem = wv_layout(P.n, P.k, sizeof(GT), P.so);
    if (smem > (size_t)max_smem_optin())
        return set_error(MCB_ERR_UNSUPPORTED, "wvcp: n*k too large for shared memory (%zu B)", smem);
    if (cudaFuncSetAttribute(wvcp_kernel<GT, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "wvcp: smem attribute failed");
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wvcp_kernel<GT, STATS>, WV_NT, smem);
    nb = std::max(nb, 1);
    const int grid = (int)std::min<int64_t>(std::min<int64_t>(nwork, (int64_t)nb * num_sms()), ws_cap_ctas);
    P.nwork = (int)nwork;
    P.ws_wc = reinterpret_cast<uint16_t *>(ws_base);
    P.ws_wc_stride = wc_stride;
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] wvcp<gamma u%d> grid=%d (%d/SM) smem=%zu work=%lld\n", (int)(8 * sizeof(GT)), grid,
                nb, smem, (long long)nwork);
    wvcp_kernel<GT, STATS><<<grid, WV_NT, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "wvcp launch failed");
    return MCB_OK;
}

// the phase counters are a separate instantiation: zero cost when off
template <typename GT>
static int wvcp_launch(WvParams P, int64_t nwork, cudaStream_t st, uint8_t *ws_base, size_t ws_cap_ctas,
                       size_t wc_stride) {
    return (P.flags & MCB_FLAG_WSTATS) ? wvcp_launch_t<GT, true>(P, nwork, st, ws_base, ws_cap_ctas, wc_stride)
                                       : wvcp_launch_t<GT, false>(P, nwork, st, ws_base, ws_cap_ctas, wc_stride);
}

int wvcp_stats(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_wvstats, sizeof(unsigned long long) * 16) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "wvcp stats unavailable");
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_wvstats, z, sizeof(z));
    }
    return MCB_OK;
}

int wvcp_run(const WvcpArgs &A, cudaStream_t st) {
    if (A.p < 0 || A.n < 1 || A.k < 1 || A.depth < 0 || A.rounds < 0 || A.nranks < 1)
        return set_error(MCB_ERR_VALUE, "wvcp: bad shape");
    if (A.k > 255 || A.n > 65535)
        return set_error(MCB_ERR_UNSUPPORTED, "wvcp: k<=255 and n<=65535 required");
    if (A.rounds * A.depth >= (int64_t)1 << 31)
        return set_error(MCB_ERR_UNSUPPORTED, "wvcp: rounds*depth must be < 2^31");
    if (A.p == 0) return MCB_OK;
    // gamma u8 first (twice the individuals per SM); individuals whose gamma
    // would reach 256 re-run with u16 (MCB_WVCP_WIDE=1: u16 throughout)
    const bool wide_only = getenv("MCB_WVCP_WIDE") != nullptr ||
                           wv_smem((int)A.n, (int)A.k, 1) > (size_t)max_smem_optin();
    const size_t max_ctas = (size_t)16 * num_sms();
    const size_t wc_stride = (((size_t)A.k * A.nranks + 1) / 2 * 2 + 127) & ~(size_t)127;  // u16 elements
    const size_t ctl_bytes = (256 + 4 * (size_t)A.p + 255) & ~(size_t)255;
    uint8_t *ws = (uint8_t *)workspace(ctl_bytes + max_ctas * wc_stride * 2);
    if (!ws) return set_error(MCB_ERR_CUDA, "wvcp: workspace");
    cudaMemsetAsync(ws, 0, 256, st);
    WvParams P{};
    P.assigns = A.assigns;
    P.best_assigns = A.best_assigns;
    P.indptr = A.indptr;
    P.indices = A.indices;
    P.eu = A.eu;
    P.ev = A.ev;
    P.m = A.m;
    P.wranks = A.wranks;
    P.wvals = A.wvals;
    P.nranks = (int)A.nranks;
    P.weights = A.weights;
    P.n = (int)A.n;
    P.k = (int)A.k;
    P.depth = A.depth;
    P.rounds = A.rounds;
    P.schedule_on = A.schedule_on;
    P.phi0s = A.phi0s;
    P.forced_phi = A.forced_phi;
    P.tt_base = A.tt_base;
    P.keys = A.keys;
    P.best_scores = A.best_scores;
    P.end_scores = A.end_scores;
    P.end_conflicts = A.end_conflicts;
    P.phi_used = A.phi_used;
    P.diag = A.diag;
    P.log_cap = A.log_cap;
    P.log_v = A.log_v;
    P.log_iter = A.log_iter;
    P.log_tt = A.log_tt;
    P.log_asp = A.log_asp;
    P.log_cnt = A.log_cnt;
    P.flags = A.flags;
    int32_t *ctl32 = reinterpret_cast<int32_t *>(ws);  // [0], [2] work counters, [1] err, [3] ovf count
    P.err_flag = ctl32 + 1;
    int32_t *ovf = reinterpret_cast<int32_t *>(ws + 256);
    int rc;
    int32_t h[3] = {0, 0, 0};
    if (!wide_only) {
        P.work_counter = ctl32;
        P.work_list = nullptr;
        P.ovf_list = ovf;
        P.ovf_count = ctl32 + 3;
        rc = wvcp_launch<uint8_t>(P, A.p, st, ws + ctl_bytes, max_ctas, wc_stride);
        if (rc) return rc;
        if (cudaMemcpyAsync(h, ctl32 + 1, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "wvcp kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
        if (h[0] == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
        if (h[0]) return set_error(MCB_ERR_CUDA, "wvcp: internal error %d", h[0]);
    }
    if (wide_only || h[2] > 0) {
        P.work_counter = ctl32 + 2;
        P.work_list = wide_only ? nullptr : ovf;
        P.ovf_list = nullptr;
        P.ovf_count = nullptr;
        rc = wvcp_launch<uint16_t>(P, wide_only ? A.p : h[2], st, ws + ctl_bytes, max_ctas, wc_stride);
        if (rc) return rc;
        int32_t err = 0;
        if (cudaMemcpyAsync(&err, P.err_flag, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "wvcp kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
        if (err == 1) return set_error(MCB_ERR_RANGE, "color id out of range [0, k)");
        if (err) return set_error(MCB_ERR_CUDA, "wvcp: internal error %d", err);
    }
    return MCB_OK;
}

}  // namespace mcb
