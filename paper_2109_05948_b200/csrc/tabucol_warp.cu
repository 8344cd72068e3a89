// tabucol_warp.cu -- batched TabuCol, one individual per WARP (sm_100a).
//
// Same semantics as tabucol.cu / the reference `_tabucol_batch`
// (pkg/src/memcolor/localsearch.py:266-410), bit-exact in validation mode:
//   * scan order = conflict list x colours ascending (:328-334); the list is
//     maintained by append / swap-remove over (N(v) ascending, then v) (:368-385);
//   * tabu test `it < tabu[v,c]` with aspiration `conflicts + d < best` (:336-339);
//   * reservoir tie-break: the SplitMix64 counter advances once per candidate
//     equal to the running minimum (:340-350); tenure U{0..9}+(6*conf)//10 after
//     the move (:363-366), last write wins;
//   * early exit at zero conflicts (:322); `it` counts every step (:398).
//
// Why a warp and not a CTA per individual: the reference iteration is a short
// serial chain (scan -> reservoir -> move -> neighbour update -> list update).
// With a CTA per individual every phase boundary is a block barrier and three
// of four warps idle in the serial phases.  Here every phase is warp-synchronous
// (shuffles / ballots, no __syncthreads in the loop), all per-individual
// scalars live in registers (uniform across lanes), and an SM runs as many
// independent individuals as shared memory holds (8 at G(500,.5) k=48).
//
// Gamma byte per (vertex, colour), shared memory, rows of KP = 16 KV bytes:
//     bit 7  OWN   the vertex's own colour (never a candidate)
//     bit 6  TABU  (vertex, colour) is tabu this iteration
//     bits 0-5     gamma = #neighbours of that colour (<= 63, else the
//                  individual is re-run by the wide CTA kernel, tabucol.cu)
//     padding colours 0x7F.
// So a row's candidate moves are exactly its bytes < 0x40, and the row minimum
// is a branch-free SIMD byte minimum.  Aspiration (a tabu move reaching a new
// best: gamma < gva + best - conflicts) is only possible when gva + best -
// conflicts > 0; then the row's tabu bytes are folded in (bytes ^ 0x40).
//
// Tabu expiry is exact and eager: every tabu entry (v, c, expiry) lives in a
// register ring ordered by age -- register row 0 holds the newest 32 entries
// (lane = insertion % 32), the rows shift down once per 32 insertions -- so
// every access uses a static register index; each iteration checks the rows
// that still hold live entries (2 in steady state) and clears the TABU bit of
// entries expiring now.  Re-tabu of a tabu pair invalidates the older entry
// (last write wins, :366).  The registers hold 1024 entries; the SPILL
// instantiation continues the ring, in age order, in a per-warp global buffer
// (individuals that need it are re-run on it from their start).
//
// Adjacency: a lane-interleaved bitset, row v = 32 chunks of CH bits, bit q of
// chunk L <-> vertex L + 32 q (the rows lane L owns in the gamma table), read
// from L2 as soon as the moving vertex is known; the neighbour update is one
// chunk per lane, all CH slots unrolled.  A CSR (u16 indices) variant remains
// for A/B (MCB_WARP_MODE=csr).
#include <algorithm>
#include <climits>
#include <utility>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "launch.h"
#include "tw_helpers.cuh"

#ifndef TW_DIVREG
#define TW_DIVREG 1  // first-round reservoir divisor entries in registers
#endif

#ifndef TW_STATS_TU
#define TW_STATS_TU 0  // 1: the instrumented instantiations (tabucol_warp_stats.cu)
#endif

namespace mcb {

using namespace tw;

struct WarpTabuParams {
    int32_t *assigns;
    int32_t *best_assigns;
    const uint8_t *bitset;     // BITSET variant: n rows of 4*CH bytes
    const uint16_t *nbr16;     // CSR variant: neighbour ids (u16)
    const uint32_t *indptr32;  // CSR offsets (u32, n+1)
    const int32_t *eu, *ev;
    int64_t m;
    int n, k;
    int64_t depth;
    const uint64_t *keys;
    int64_t *best_conflicts, *end_conflicts, *iters_used, *diag;
    int64_t log_cap;
    int32_t *log_v;
    int64_t *log_iter, *log_tt, *log_cnt;
    int64_t *counters;
    int nwork;
    const int32_t *nwork_dev;  // device-side count (overrides nwork when set)
    const int32_t *work_list;  // individual ids (nullptr: 0 .. nwork-1)
    uint32_t *spill;           // SPILL variant: per-warp ring rows in global memory
    int spill_rows;            // rows per warp (power of two)
    int32_t *work_counter;
    int32_t *ovf_list, *ovf_count, *err_flag;
    uint32_t flags;
    int warp_smem;     // bytes per warp region
    int bitset_bytes;  // bytes of the CTA-shared bitset copy (0: rows read from L2)
};

namespace {

__device__ unsigned long long g_wstats[40];
// divisibility by s = o * 2^t, odd o < 64: x % s == 0  <=>  low t bits of x are
// zero and (x >> t) * inv(o) <= floor((2^64 - 1) / o)  (inv = inverse mod 2^64)
__device__ ulonglong2 g_divtab[32];
__device__ __forceinline__ bool divisible(uint64_t x, uint32_t s) {
    if (s < 64u) {
        const int t = __ffs(s) - 1;
        const uint32_t o = s >> t;
        const ulonglong2 e = __ldg(&g_divtab[o >> 1]);
        return (x & ((1ull << t) - 1ull)) == 0ull && (x >> t) * e.x <= e.y;
    }
    return mod_is_zero(x, s);
}
// stats slots (MCB_FLAG_WSTATS): event counters, then per-phase cycles
enum {
    WS_IT,
    WS_ROUNDS,
    WS_ASP_ROUNDS,
    WS_EXPIRE_ROWS,
    WS_SUPERSEDE,
    WS_WALK_PASSES,
    WS_DRAW_ROUNDS,
    WS_EVENTS,
    WS_REMOVES,
    WS_BEST,
    WS_SPILL_ROWS,
    WS_CY_SCAN = 16,
    WS_CY_SELECT,
    WS_CY_MOVE,
    WS_CY_UPDATE,
    WS_CY_EVENTS,
    WS_CY_TAIL,
    WS_CY_EXPIRE,
    WS_CY_ROWMIN,
    WS_CY_PREFIX,
    WS_CY_LIST,
    WS_CY_WALK,
    WS_CY_P2,
    WS_CY_DRAW,
    WS_CY_LOCROW,
    WS_NCL_SUM,
    WS_NCL_GT32,
    WS_NCL_GT144,
    WS_N = 40
};
#define WST(i, x) \
    if constexpr (stats) st[i] += (x)
#define WPH(i)                          \
    if constexpr (stats) {              \
        const long long _t = clock64(); \
        st[i] += _t - ph_t;             \
        ph_t = _t;                      \
    }

}  // namespace

// ---------------------------------------------------------------------------
// the kernel
//   KV     = 16-byte vectors per gamma row (KP = 16 KV >= k)
//   CH     = bitset chunk bits per lane (BITSET): lane L owns vertices
//            L + 32 q, q < CH  (n <= 32 CH)
// Row u is stored rotated by g(u) words (g depends on u mod 32 only), so that
// the 32 lanes of the neighbour update -- rows L + 32 q for one q -- hit
// distinct banks.  Scans read whole rows (order-free); walks / locate / single
// bytes translate colours with phys().
// ---------------------------------------------------------------------------

template <int KV, int CH, bool BITSET, bool SPILL, bool STATS>
__global__ void __launch_bounds__(32 * TW_MAX_WARPS, 1) tabucol_warp_kernel(WarpTabuParams P) {
    constexpr int KP = 16 * KV, KW = 4 * KV;
    constexpr int CBITS = KP <= 16 ? 4 : KP <= 32 ? 5 : KP <= 64 ? 6 : 7;  // a row's tie count < KP
    constexpr int RW = 2;  // conflicting rows per lane per scan round
    constexpr int SW = KW <= 4 ? 4 : KW <= 8 ? 8 : KW <= 16 ? 16 : 32;  // walk segment width
    static_assert(KW <= 32, "k <= 128");
    using S = Swz<KW>;
    using CT = typename ChunkT<BITSET ? CH : 32>::T;

    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n = P.n, k = P.k;
    const unsigned lt_mask = (1u << lane) - 1u;

    // CTA-shared adjacency bitset (read-only afterwards; warps never sync again)
    // bitset rows: a CTA-shared copy, or straight from L2 (the update's row is
    // loaded as soon as the moving vertex is known, ~600 cycles before use)
    const uint8_t *brows = P.bitset_bytes ? smem : P.bitset;
    if (BITSET && P.bitset_bytes) {
        const uint4 *src = reinterpret_cast<const uint4 *>(P.bitset);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < P.bitset_bytes / 16; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    uint8_t *base = smem + P.bitset_bytes + (size_t)wid * P.warp_smem;
    uint8_t *gam = base;
    size_t off = (size_t)n * KP;
    uint32_t *rmc = reinterpret_cast<uint32_t *>(base + off);  // compact list of scanned rows
    off += 4 * (size_t)n;
    uint16_t *clist = reinterpret_cast<uint16_t *>(base + off);
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint16_t *cpos = reinterpret_cast<uint16_t *>(base + off);  // position in clist (members only)
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint8_t *asg = base + off;

    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool cnt_on = P.counters != nullptr;
    constexpr bool stats = STATS;  // MCB_FLAG_WSTATS selects the instrumented instantiation
    long long st[STATS ? WS_N : 1];
    if constexpr (stats)
        for (int i = 0; i < WS_N; i++) st[i] = 0;
    const int g_lane = S::g(lane);  // rotation of every row this lane owns (u = lane + 32q)
    // this lane's first-round reservoir divisor s = 2 + lane (< 64): its table
    // entry in registers, off the draw chain (the table sits in L2 otherwise)
    const int dv_t = __ffs(2 + lane) - 1;
    const ulonglong2 dv_e = g_divtab[((2 + lane) >> dv_t) >> 1];
    constexpr int s_first = TW_DIVREG ? 34 : 2;

    for (;;) {
        int wi = 0;
        if (lane == 0) wi = atomicAdd(P.work_counter, 1);
        wi = __shfl_sync(FULLM, wi, 0);
        if (wi >= (P.nwork_dev ? *P.nwork_dev : P.nwork)) break;
        const int ind = P.work_list ? P.work_list[wi] : wi;
        const uint64_t key = P.keys[ind];
        int32_t *a_io = P.assigns + (size_t)ind * n;
        int32_t *b_out = P.best_assigns + (size_t)ind * n;

        // ---------------- init (localsearch.py:289-318) ----------------
        bool bad = false, rangeerr = false;
        for (int v = lane; v < n; v += 32) {
            int c = a_io[v];
            if (c < 0 || c >= k) {
                rangeerr = true;
                c = 0;
            }
            asg[v] = (uint8_t)c;
            b_out[v] = c;
        }
        {
            // logical padding colours >= k are 0xFF; rows rotated by g(u)
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gam);
            // padding colours 0x7F: never a candidate (gamma 63 >= any A), and the
            // own colour is the only byte of a row with bit 7 set
            const uint32_t padw = (k & 3) ? (0x7F7F7F7Fu << (8 * (k & 3))) : 0u;
            for (int i = lane; i < n * KW; i += 32) {
                const int u = i / KW, p = i - u * KW;
                int w = p - S::g(u);
                if (w < 0) w += KW;
                g32[i] = (4 * w + 4 <= k) ? 0u : (4 * w >= k ? 0x7F7F7F7Fu : padw);
            }
        }
        __syncwarp();
        // gamma[u][c] = #neighbours of u coloured c; lane-private rows u = lane + 32j
        for (int u = lane; u < n; u += 32) {
            uint8_t *row = gam + (size_t)u * KP;
            const int gu = S::g(u);
            if constexpr (BITSET) {
                const CT *br = reinterpret_cast<const CT *>(brows + (size_t)u * 4 * CH);
                for (int L = 0; L < 32; L++) {
                    uint32_t ch = br[L];
                    while (ch) {
                        const int q = __ffs(ch) - 1;
                        ch &= ch - 1;
                        const int c = asg[L + 32 * q];
                        uint8_t *e = row + S::phys(c, gu);
                        const int x = *e + 1;
                        if (x > (int)GM) bad = true;
                        else *e = (uint8_t)x;
                    }
                }
            } else {
                const uint32_t s0 = P.indptr32[u], s1 = P.indptr32[u + 1];
                for (uint32_t idx = s0; idx < s1; idx++) {
                    const int c = asg[P.nbr16[idx]];
                    uint8_t *e = row + S::phys(c, gu);
                    const int x = *e + 1;
                    if (x > (int)GM) bad = true;
                    else *e = (uint8_t)x;
                }
            }
        }
        __syncwarp();
        int conflicts, best;  // <= n (n - 1) / 2 < 2^19 (n <= 1024): 32-bit on the chain
        int C = 0;
        {
            long long c2 = 0;
            for (int v0 = 0; v0 < n; v0 += 32) {
                const int v = v0 + lane;
                bool f = false;
                if (v < n) {
                    uint8_t *p = gam + (size_t)v * KP + S::phys(asg[v], S::g(v));
                    const int g = *p;
                    *p = (uint8_t)(g | OWN);
                    f = g > 0;
                    c2 += g;
                }
                const unsigned bal = __ballot_sync(FULLM, f);
                if (f) {
                    const int pos = C + __popc(bal & lt_mask);
                    clist[pos] = (uint16_t)v;
                    cpos[v] = (uint16_t)pos;
                }
                C += __popc(bal);
            }
            c2 = warp_sum64(c2);
            conflicts = (int)(c2 / 2);
            best = conflicts;
        }
        if (__any_sync(FULLM, rangeerr) && lane == 0) atomicExch(P.err_flag, 1);
        bad = __any_sync(FULLM, bad);
        if constexpr (!SPILL) {
            // tenures of U{0..9} + 0.6 conflicts beyond the register ring's 1024
            // entries from the start (e.g. C3 from random colourings: ~1800):
            // straight to the SPILL pass instead of overflowing after ~1000 moves
            if (9 + (6 * conflicts) / 10 > 32 * KE) bad = true;
        }
        __syncwarp();

        long long it = 0, nlog = 0, sum_c = 0, sum_deg = 0, diag = 0;
        unsigned long long ctr = 0;
        // tabu ring (see header): rows [0, nrows) may hold live entries
        uint32_t ring[KE];
#pragma unroll
        for (int j = 0; j < KE; j++) ring[j] = 0u;
        int nrows = 0;
        uint32_t ins = 0;
        uint32_t next_exp = 0;  // lower bound of the earliest live expiry (valid if nrows)
        // SPILL: rows pushed out of the register ring (older than all register
        // rows) continue, in age order, in this warp's global ring [sp_head,
        // sp_tail); sp_next bounds their earliest live expiry from below
        uint32_t *spw = nullptr;
        uint32_t sp_head = 0, sp_tail = 0, sp_next = 0;
        const uint32_t sp_mask = (uint32_t)P.spill_rows - 1u;
        if constexpr (SPILL) spw = P.spill + ((size_t)blockIdx.x * (blockDim.x >> 5) + wid) * P.spill_rows * 32;

        // ---------------- iterations (:320-405) ----------------
        if (k >= 2 && !bad) {
            for (long long step = 0; step < P.depth; step++) {
                if (conflicts == 0) break;
                long long ph_t = 0;
                if constexpr (stats) ph_t = clock64();
                WST(WS_IT, 1);
                const uint32_t it32 = (uint32_t)it;
                const int thr = max(best - conflicts, -TW_BIG);

                // ---- tabu expiry: it < tabu[v,c] fails from it == expiry on
                if (nrows > 0 && (int)(next_exp - it32) <= 0) {
                    // some entry may expire now (next_exp is a lower bound)
                    int last = -1;  // this lane's last live row; one reduction after the rows
                    uint32_t dmin = 0x4000u;
#pragma unroll
                    for (int j = 0; j < KE; j++) {
                        if (j >= nrows) break;
                        const uint32_t e = ring[j];
                        const uint32_t dist = ent_dist(e, it32);
                        const bool hit = (e >> 31) != 0u && dist == 0u;
                        if (hit) {
                            const int v = (e >> 21) & 0x3FF, c = (e >> 14) & 0x7F;
                            gam[(size_t)v * KP + S::phys(c, S::g(v))] &= (uint8_t)~TABU;
                        }
                        ring[j] = hit ? 0u : e;
                        const bool live = (ring[j] >> 31) != 0u;
                        if (live) {
                            dmin = min(dmin, dist);
                            last = j;
                        }
                    }
                    WST(WS_EXPIRE_ROWS, nrows);
                    nrows = __reduce_max_sync(FULLM, last) + 1;
                    next_exp = it32 + __reduce_min_sync(FULLM, dmin);
                    __syncwarp();
                }
                if constexpr (SPILL) {
                    if (sp_head != sp_tail && (int)(sp_next - it32) <= 0) {
                        // spilled rows, 8 loads in flight; fully dead rows at
                        // the old end are released
                        uint32_t dmin = 0x4000u, newhead = sp_head;
                        bool lead = true;
                        for (uint32_t r0 = sp_head; r0 != sp_tail; r0 += 8) {
                            uint32_t e8[8];
#pragma unroll
                            for (int q = 0; q < 8; q++)
                                e8[q] = (r0 + q != sp_tail && (int)(sp_tail - (r0 + q)) > 0)
                                            ? spw[((r0 + q) & sp_mask) * 32 + lane]
                                            : 0u;
#pragma unroll
                            for (int q = 0; q < 8; q++) {
                                if ((int)(sp_tail - (r0 + q)) <= 0) break;
                                const uint32_t e = e8[q];
                                const uint32_t dist = ent_dist(e, it32);
                                const bool hit = (e >> 31) != 0u && dist == 0u;
                                if (hit) {
                                    const int v = (e >> 21) & 0x3FF, c = (e >> 14) & 0x7F;
                                    gam[(size_t)v * KP + S::phys(c, S::g(v))] &= (uint8_t)~TABU;
                                    spw[((r0 + q) & sp_mask) * 32 + lane] = 0u;
                                }
                                const bool live = (e >> 31) != 0u && !hit;
                                if (live) dmin = min(dmin, dist);
                                if (__any_sync(FULLM, live)) lead = false;
                                else if (lead) newhead = r0 + q + 1;
                            }
                            if ((int)(sp_tail - (r0 + 8)) <= 0) break;
                        }
                        sp_head = newhead;
                        sp_next = it32 + __reduce_min_sync(FULLM, dmin);
                        __syncwarp();
                    }
                }
                WPH(WS_CY_EXPIRE);

                // ---- scan, phase 1 (localsearch.py:328-350): row minima of the
                // conflicting rows, RW rows per lane per round (rows b0 + 32 h +
                // lane, independent chains); running prefix-min over the rows in
                // list order; in-lane walks of the rows that lower it.  Rows at or
                // below the running minimum -- the only ones holding reservoir
                // events -- are appended to a compact list (rmc) for phase 2.
                int carry = TW_BIG, total = 0, ncl = 0;
                const int nr = (C + 31) >> 5;
#pragma unroll 1
                for (int b0 = 0; b0 < C; b0 += 32 * RW) {
                    int rm[RW], v[RW], gva[RW], A[RW];
#pragma unroll
                    for (int h = 0; h < RW; h++) {
                        const int li = b0 + 32 * h + lane;
                        rm[h] = TW_BIG;
                        v[h] = 0;
                        gva[h] = 0;
                        A[h] = 0;
                        if (li < C) {
                            v[h] = clist[li];
                            uint32_t x[KW];
                            load_row<KV>(gam + (size_t)v[h] * KP, x);
                            gva[h] = gam[(size_t)v[h] * KP + S::phys(asg[v[h]], S::g(v[h]))] & GM;
                            A[h] = gva[h] + thr;
                            int m = row_min<KW>(x, 0u);  // non-own, non-tabu (bytes < 0x40)
                            if (A[h] > 0) {
                                // aspiration: tabu colours with gamma < A are admissible
                                const int mt = row_min<KW>(x, TABU * 0x01010101u);
                                if (mt < A[h]) m = min(m, mt);
                            }
                            if (m < (int)TABU) rm[h] = m - gva[h];
                        }
                    }
                    WST(WS_ASP_ROUNDS, __any_sync(FULLM, A[0] > 0));
                    WPH(WS_CY_ROWMIN);
                    // running minimum entering each row (RW interleaved scans)
                    int in[RW];
#pragma unroll
                    for (int h = 0; h < RW; h++) in[h] = rm[h];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        int t[RW];
#pragma unroll
                        for (int h = 0; h < RW; h++) t[h] = __shfl_up_sync(FULLM, in[h], o);
                        if (lane >= o) {
#pragma unroll
                            for (int h = 0; h < RW; h++) in[h] = min(in[h], t[h]);
                        }
                    }
                    int Pl[RW];
                    {
                        int cc = carry;
#pragma unroll
                        for (int h = 0; h < RW; h++) {
                            int ex = __shfl_up_sync(FULLM, in[h], 1);
                            const int tot = __shfl_sync(FULLM, in[h], 31);
                            if (lane == 0) ex = TW_BIG;
                            Pl[h] = min(cc, ex);
                            cc = min(cc, tot);
                        }
                        carry = cc;
                    }
                    WPH(WS_CY_PREFIX);
                    // list entry: v | (rm + 64) << 10 | (entering minimum + 64, 127 =
                    // none) << 17 | gva << 24; rm == entering minimum marks a tie row,
                    // rm below it a row that lowers it (walked in phase 2)
#pragma unroll
                    for (int h = 0; h < RW; h++) {
                        const bool lst = rm[h] < TW_BIG && rm[h] <= Pl[h];
                        const unsigned nb = __ballot_sync(FULLM, lst);
                        if (lst)
                            rmc[ncl + __popc(nb & lt_mask)] = (uint32_t)v[h] | ((uint32_t)(rm[h] + 64) << 10) |
                                                              ((uint32_t)(Pl[h] >= TW_BIG ? 127 : Pl[h] + 64) << 17) |
                                                              ((uint32_t)gva[h] << 24);
                        ncl += __popc(nb);
                    }
                    WPH(WS_CY_LIST);
                }
                __syncwarp();
                const int D = carry;
                WST(WS_ROUNDS, nr);
                WST(WS_NCL_SUM, ncl);
                WST(WS_NCL_GT32, ncl > 32);
                WST(WS_NCL_GT144, ncl > 144);
                WPH(WS_CY_SCAN);
                if (cnt_on) sum_c += C;

                int mv_v = -1, mv_a = 0, mv_b = 0, Dg = 0;
                uint32_t ch_pref = 0;
                if (D < TW_BIG) {
                    // ---- phase 2a: tie counts of the listed rows (one lane per entry).
                    // Rows equal to the running minimum contribute all their minimum
                    // candidates as tie events; rows at D contribute T, the final
                    // group.  The first 32 entries keep (row, exclusive D-count
                    // prefix) in registers for the locate.
                    int T = 0, e_v = 0, e_gv = 0, e_cD = 0, e_ex = 0;
                    // one walk pass over up to 32/SW lowering rows (bit mask `low` of
                    // list lanes); returns this lane's share of the tie events
                    auto walk_pass = [&](unsigned low, int v, int gv, int pe) -> int {
                        const int g = lane / SW, wl = lane % SW;
                        unsigned tmp = low;
#pragma unroll
                        for (int q = 0; q < 32 / SW - 1; q++)
                            if (q < g) tmp &= tmp - 1;
                        const int src = tmp ? __ffs(tmp) - 1 : -1;
                        const int s = max(src, 0);
                        const int wv = __shfl_sync(FULLM, v, s);
                        const int wg = __shfl_sync(FULLM, gv, s);
                        const int wp = __shfl_sync(FULLM, pe, s);
                        uint32_t y = 0xFFFFFFFFu;
                        if (src >= 0 && wl < KW)
                            y = cand_word(reinterpret_cast<const uint32_t *>(gam + (size_t)wv * KP)[S::pw(wl, S::g(wv))],
                                          wg + thr);
                        const uint32_t m2 = __vminu2(y & 0x00FF00FFu, __byte_perm(y, 0, 0x4341));
                        const int um = (int)min(m2 & 0xFFFFu, m2 >> 16);
                        const int ex = seg_excl_min<SW>(um, wl);
                        // running minimum entering this word (clamped: never tied or
                        // lowered by a non-candidate 0xFF), then the exclusive prefix
                        // minima of its 4 bytes, packed; events = equal bytes
                        const int c0 = min(min(wp == 127 ? INT_MAX : wp - 64 + wg, ex), 0xFE);
                        const int c1 = min(c0, (int)(y & 0xFFu));
                        const int c2 = min(c1, (int)__byte_perm(y, 0, 0x4441));
                        const int c3 = min(c2, (int)__byte_perm(y, 0, 0x4442));
                        const uint32_t Cp = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
                        const unsigned segm = (SW == 32 ? 0xffffffffu : ((1u << SW) - 1u)) << (lane & ~(SW - 1));
                        const int t = masked_sum_small<3>(count_eq(y, Cp), segm);
                        return (wl == 0 && src >= 0) ? t : 0;
                    };
                    if (ncl <= 32) {
                        // common case, straight-line: the tie counts (lane = entry) and
                        // the first walk pass are independent and interleave
                        const bool val = lane < ncl;
                        const uint32_t e = rmc[val ? lane : 0];
                        const int v = (int)(e & 0x3FFu);
                        const int rmi = (int)((e >> 10) & 0x7Fu) - 64;
                        const int pe = (int)((e >> 17) & 0x7Fu);
                        const int gv = (int)(e >> 24);
                        const bool tie = val && rmi == pe - 64, lower = val && rmi < pe - 64;
                        const bool atD = val && rmi == D;
                        uint32_t x[KW];
                        load_row<KV>(gam + (size_t)v * KP, x);
                        const int m = rmi + gv;
                        int cnt = row_count<KW>(x, (uint32_t)m);
                        if (m < gv + thr) cnt += row_count<KW>(x, (uint32_t)m | TABU);
                        unsigned low = prod ? 0u : __ballot_sync(FULLM, lower);
                        if (low) {
                            WST(WS_WALK_PASSES, 1);
                            total += walk_pass(low, v, gv, pe);
#pragma unroll
                            for (int q = 0; q < 32 / SW; q++) low &= low - 1;
                        }
                        if (tie) total += cnt;
                        const int cD = atD ? cnt : 0;
                        e_v = v;
                        e_gv = gv;
                        e_cD = cD;
                        e_ex = excl_sum_small<CBITS>(cD, lt_mask);
                        T = __reduce_add_sync(FULLM, cD);
                        while (low) {
                            WST(WS_WALK_PASSES, 1);
                            total += walk_pass(low, v, gv, pe);
#pragma unroll
                            for (int q = 0; q < 32 / SW; q++) low &= low - 1;
                        }
                    } else {
                        for (int i0 = 0; i0 < ncl; i0 += 32) {
                            const int i = i0 + lane;
                            int cD = 0, v = 0, gv = 0, pe = 127;
                            bool lower = false;
                            if (i < ncl) {
                                const uint32_t e = rmc[i];
                                v = (int)(e & 0x3FFu);
                                const int rmi = (int)((e >> 10) & 0x7Fu) - 64;
                                pe = (int)((e >> 17) & 0x7Fu);
                                gv = (int)(e >> 24);
                                const bool tie = rmi == pe - 64;
                                lower = rmi < pe - 64;
                                int cnt = 0;
                                if (tie || rmi == D) {
                                    uint32_t x[KW];
                                    load_row<KV>(gam + (size_t)v * KP, x);
                                    const int m = rmi + gv;
                                    cnt = row_count<KW>(x, (uint32_t)m);
                                    if (m < gv + thr) cnt += row_count<KW>(x, (uint32_t)m | TABU);
                                }
                                if (tie) total += cnt;
                                if (rmi == D) cD = cnt;
                                rmc[i] = (uint32_t)v | ((uint32_t)gv << 10) | ((uint32_t)cD << 16);
                            }
                            if (i0 == 0) {
                                int incl = cD;
#pragma unroll
                                for (int o = 1; o < 32; o <<= 1) {
                                    const int t = __shfl_up_sync(FULLM, incl, o);
                                    if (lane >= o) incl += t;
                                }
                                e_v = v;
                                e_gv = gv;
                                e_cD = cD;
                                e_ex = incl - cD;
                                T = __shfl_sync(FULLM, incl, 31);
                            } else {
                                T += __reduce_add_sync(FULLM, cD);
                            }
                            unsigned low = prod ? 0u : __ballot_sync(FULLM, lower);
                            while (low) {
                                WST(WS_WALK_PASSES, 1);
                                total += walk_pass(low, v, gv, pe);
#pragma unroll
                                for (int q = 0; q < 32 / SW; q++) low &= low - 1;
                            }
                        }
                    }
                    const int tot = prod ? 0 : __reduce_add_sync(FULLM, total);
                    WPH(WS_CY_P2);
                    // tenure draw (:363-365), issued early so it overlaps the reservoir
                    const int nconf = conflicts + D;
                    uint32_t ll;
                    if (!prod) ll = u64_below32(key, ctr + (unsigned long long)tot, 10u);
                    else ll = philox_below(key, ctr + 1, 10u);
                    // ---- reservoir: the T-1 draws of the final group
                    int sstar = 1;
                    if (T > 1) {
                        if (!prod) {
                            const unsigned long long c0 = ctr + (unsigned long long)(tot - (T - 1));
                            int smax = 1;
                            WST(WS_DRAW_ROUNDS, (T + 30) / 32);
                            if (TW_DIVREG && 2 + lane <= T) {
                                const uint64_t x = stream_value(key, c0 + (unsigned long long)lane);
                                if ((x & ((1ull << dv_t) - 1ull)) == 0ull && (x >> dv_t) * dv_e.x <= dv_e.y)
                                    smax = 2 + lane;
                            }
                            for (int s = s_first + lane; s <= T; s += 32)
                                if (divisible(stream_value(key, c0 + (unsigned long long)(s - 2)), (uint32_t)s))
                                    smax = s;
                            sstar = __reduce_max_sync(FULLM, smax);
                        } else {
                            sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                        }
                    }
                    WPH(WS_CY_DRAW);
                    // ---- locate the sstar-th D-candidate in scan order: the row ...
                    int v, gva, need;
                    {
                        const unsigned bm = __ballot_sync(FULLM, e_cD > 0 && e_ex < sstar && sstar <= e_ex + e_cD);
                        if (bm) {
                            const int src = __ffs(bm) - 1;
                            v = __shfl_sync(FULLM, e_v, src);
                            gva = __shfl_sync(FULLM, e_gv, src);
                            need = sstar - __shfl_sync(FULLM, e_ex, src);
                        } else {
                            // beyond the first 32 list entries (rare)
                            int cum = 0;
                            v = 0;
                            gva = 0;
                            need = 1;
                            for (int i0 = 0; i0 < ncl; i0 += 32) {
                                const int i = i0 + lane;
                                int cc = 0;
                                uint32_t e = 0;
                                if (i < ncl) {
                                    e = rmc[i];
                                    cc = (int)(e >> 16);
                                }
                                int incl = cc;
#pragma unroll
                                for (int o = 1; o < 32; o <<= 1) {
                                    const int t = __shfl_up_sync(FULLM, incl, o);
                                    if (lane >= o) incl += t;
                                }
                                const int rt = __shfl_sync(FULLM, incl, 31);
                                if (cum + rt >= sstar) {
                                    const unsigned b2 = __ballot_sync(FULLM, cum + incl >= sstar);
                                    const int src = __ffs(b2) - 1;
                                    const uint32_t es = __shfl_sync(FULLM, e, src);
                                    v = (int)(es & 0x3FFu);
                                    gva = (int)((es >> 10) & 0x3Fu);
                                    need = sstar - cum - __shfl_sync(FULLM, incl - cc, src);
                                    break;
                                }
                                cum += rt;
                            }
                        }
                    }
                    WPH(WS_CY_LOCROW);
                    // the moving vertex is known: fetch its adjacency chunk now
                    if constexpr (BITSET) {
                        const CT *br = reinterpret_cast<const CT *>(brows + (size_t)v * 4 * CH) + lane;
                        ch_pref = P.bitset_bytes ? (uint32_t)*br : (uint32_t)__ldg(br);
                    }
                    // ... then the colour: lanes over the row's words in colour order
                    uint8_t *grow = gam + (size_t)v * KP;
                    const int gvv = S::g(v);
                    Dg = D + gva;
                    int b = -1;
                    {
                        uint32_t xw = 0xFFFFFFFFu;
                        int cc = 0;
                        if (lane < KW) {
                            xw = cand_word(reinterpret_cast<const uint32_t *>(grow)[S::pw(lane, gvv)], gva + thr);
                            cc = count_eq(xw, (uint32_t)Dg * 0x01010101u);
                        }
                        const int incl = excl_sum_small<3>(cc, lt_mask) + cc;
                        const unsigned bm = __ballot_sync(FULLM, incl >= need);
                        const int src = bm ? __ffs(bm) - 1 : 0;
                        int col = -1;
                        if (lane == src && bm) {
                            uint32_t z = zero_flags(xw ^ ((uint32_t)Dg * 0x01010101u));
                            for (int r = need - (incl - cc); r > 1; r--) z &= z - 1;
                            col = 4 * lane + ((__ffs(z) - 1) >> 3);
                        }
                        b = __shfl_sync(FULLM, col, src);
                    }
                    if (b < 0) {
                        bad = true;  // cannot happen; route to the wide kernel
                        break;
                    }
                    const int a = asg[v];
                    const int pa = S::phys(a, gvv);
                    const uint32_t ba = grow[pa];
                    WPH(WS_CY_SELECT);
                    // ---- move, tenure, tabu entry (:352-366)
                    conflicts = nconf;
                    ctr += prod ? 2ull : (unsigned long long)tot + 1ull;
                    const int tt = (int)ll + (6 * conflicts) / 10;
                    if (tt >= 8190) {
                        bad = true;
                        break;
                    }
                    const uint32_t e_new = it32 + (uint32_t)tt + 1u;
                    if (ba & TABU) {
                        // (v, a) is re-tabu'd while tabu: the older entry is void
                        WST(WS_SUPERSEDE, 1);
                        const uint32_t key_vc = ent_pack(v, a, 0) & 0xFFFFC000u;
                        bool found = false;
#pragma unroll
                        for (int j = 0; j < KE; j++) {
                            if (j >= nrows) break;
                            const bool hit = (ring[j] & 0xFFFFC000u) == key_vc;
                            if (hit) ring[j] = 0u;
                            if (__any_sync(FULLM, hit)) {
                                found = true;
                                break;
                            }
                        }
                        if constexpr (SPILL) {
                            if (!found) {
                                for (uint32_t r = sp_head; r != sp_tail; r++) {
                                    uint32_t *slot = spw + (r & sp_mask) * 32 + lane;
                                    const bool hit = (*slot & 0xFFFFC000u) == key_vc;
                                    if (hit) *slot = 0u;
                                    if (__any_sync(FULLM, hit)) break;
                                }
                            }
                        }
                        (void)found;
                    }
                    {
                        // insert at (row 0, lane ins % 32); a full row 0 shifts the rows
                        const int L = (int)(ins & 31u);
                        if (L == 0 && ins != 0u) {
                            if (__any_sync(FULLM, (ring[KE - 1] >> 31) != 0u)) {
                                if constexpr (SPILL) {
                                    if (sp_tail - sp_head > sp_mask) {
                                        bad = true;  // cannot happen: tenure < 8190
                                        break;
                                    }
                                    const uint32_t e = ring[KE - 1];
                                    spw[(sp_tail & sp_mask) * 32 + lane] = e;
                                    WST(WS_SPILL_ROWS, 1);
                                    const uint32_t dm =
                                        __reduce_min_sync(FULLM, (e >> 31) ? ent_dist(e, it32) : 0x4000u);
                                    if (sp_head == sp_tail || (int)(it32 + dm - sp_next) < 0) sp_next = it32 + dm;
                                    sp_tail++;
                                } else {
                                    bad = true;  // > 1024 live tabu entries: the SPILL variant
                                    break;
                                }
                            }
#pragma unroll
                            for (int j = KE - 1; j > 0; j--) ring[j] = ring[j - 1];
                            ring[0] = 0u;
                            nrows = min(nrows + 1, KE);
                        }
                        if (lane == L) ring[0] = ent_pack(v, a, e_new);
                        if (nrows == 0 || (int)(e_new - next_exp) < 0) next_exp = e_new;
                        nrows = max(nrows, 1);
                        ins++;
                    }
                    if (lane == 0) {
                        asg[v] = (uint8_t)b;
                        grow[pa] = (uint8_t)((ba & GM) | TABU);
                        const int pb = S::phys(b, gvv);
                        grow[pb] = (uint8_t)(grow[pb] | OWN);
                        if (nlog < P.log_cap) {
                            const size_t o = (size_t)ind * P.log_cap + nlog;
                            P.log_v[o] = v;
                            P.log_iter[o] = it;
                            P.log_tt[o] = tt;
                        }
                    }
                    if (nlog < P.log_cap) nlog++;
                    mv_v = v;
                    mv_a = a;
                    mv_b = b;
                }
                __syncwarp();
                WPH(WS_CY_MOVE);

                if (mv_v >= 0) {
                    // ---- gamma update over N(v) (:356-359) and conflict-list
                    // events in neighbour order, then v (:368-385)
                    const int v = mv_v, a = mv_a, b = mv_b;
                    int Cn = C;
                    bool ovf = false;
                    // swap-with-last removal / append (:374-385), on lane 0
                    auto cl_remove = [&](int u) {
                        WST(WS_REMOVES, 1);
                        if (lane == 0) {
                            const int pos = cpos[u], last = clist[Cn - 1];
                            clist[pos] = (uint16_t)last;
                            cpos[last] = (uint16_t)pos;
                        }
                        Cn--;
                    };
                    auto cl_append = [&](int u) {
                        if (lane == 0) {
                            clist[Cn] = (uint16_t)u;
                            cpos[u] = (uint16_t)Cn;
                        }
                        Cn++;
                    };
                    if constexpr (BITSET) {
                        // lane L: neighbours L + 32 q, all CH positions unrolled and
                        // predicated; loads first, then stores (distinct rows)
                        const uint32_t ch = ch_pref;
                        if (cnt_on) sum_deg += __reduce_add_sync(FULLM, __popc(ch));
                        // rows u = lane + 32 q for every q < CH: rows >= n lie inside
                        // this warp's region (host-checked) and are written back
                        // unchanged (never neighbours)
                        const uint32_t ra = smem_addr(gam) + (uint32_t)(lane * KP + S::phys(a, g_lane));
                        const uint32_t rb = smem_addr(gam) + (uint32_t)(lane * KP + S::phys(b, g_lane));
                        constexpr int QS = 32 * KP;
                        uint32_t oa[CH], ob[CH];
                        static_for<CH>([&](auto qc) {
                            constexpr int q = decltype(qc)::value;
                            oa[q] = lds8<q * QS>(ra);
                            ob[q] = lds8<q * QS>(rb);
                        });
                        // 4 slots per 32-bit word: SIMD +-1 and SIMD event / overflow
                        // tests (bytes never borrow: a neighbour's gamma[u,a] >= 1)
                        uint32_t evE = 0, evL = 0, ovm = 0;
                        static_for<CH / 4>([&](auto gc) {
                            constexpr int g0 = 4 * decltype(gc)::value;
                            const uint32_t nbm = (((ch >> g0) & 0xFu) * 0x00204081u) & 0x01010101u;
                            const uint32_t pa4 = __byte_perm(__byte_perm(oa[g0], oa[g0 + 1], 0x0040),
                                                             __byte_perm(oa[g0 + 2], oa[g0 + 3], 0x0040), 0x5410);
                            const uint32_t pb4 = __byte_perm(__byte_perm(ob[g0], ob[g0 + 1], 0x0040),
                                                             __byte_perm(ob[g0 + 2], ob[g0 + 3], 0x0040), 0x5410);
                            const uint32_t na4 = pa4 - nbm, nb4 = pb4 + nbm;
                            sts8<(g0 + 0) * QS>(ra, na4);
                            sts8<(g0 + 1) * QS>(ra, na4 >> 8);
                            sts8<(g0 + 2) * QS>(ra, na4 >> 16);
                            sts8<(g0 + 3) * QS>(ra, na4 >> 24);
                            sts8<(g0 + 0) * QS>(rb, nb4);
                            sts8<(g0 + 1) * QS>(rb, nb4 >> 8);
                            sts8<(g0 + 2) * QS>(rb, nb4 >> 16);
                            sts8<(g0 + 3) * QS>(rb, nb4 >> 24);
                            const uint32_t nbh = nbm << 7;
                            // leave: own colour a, gamma 1 -> 0; enter: own b, 0 -> 1;
                            // overflow: gamma 63 -> 64 wrapped to 0
                            const uint32_t zl = zero_flags((na4 & 0xBFBFBFBFu) ^ 0x80808080u) & nbh;
                            const uint32_t ze = zero_flags((nb4 & 0xBFBFBFBFu) ^ 0x81818181u) & nbh;
                            ovm |= zero_flags(nb4 & 0x3F3F3F3Fu) & nbh;
                            evL |= ((((zl >> 7) * 0x00204081u) >> 21) & 0xFu) << g0;
                            evE |= ((((ze >> 7) * 0x00204081u) >> 21) & 0xFu) << g0;
                        });
                        ovf = ovm != 0u;
                        __syncwarp();
                        WPH(WS_CY_UPDATE);
                        // events in ascending vertex order u = L + 32 q: q-major
                        uint32_t qs = __reduce_or_sync(FULLM, evE | evL);
                        while (qs) {
                            const int q = __ffs(qs) - 1;
                            qs &= qs - 1;
                            unsigned lm = __ballot_sync(FULLM, ((evE | evL) >> q) & 1u);
                            const unsigned lE = __ballot_sync(FULLM, (evE >> q) & 1u);
                            while (lm) {
                                const int L = __ffs(lm) - 1;
                                lm &= lm - 1;
                                WST(WS_EVENTS, 1);
                                if ((lE >> L) & 1u) cl_append(L + 32 * q);
                                else cl_remove(L + 32 * q);
                            }
                        }
                    } else {
                        const uint32_t s0 = P.indptr32[v], s1 = P.indptr32[v + 1];
                        if (cnt_on) sum_deg += s1 - s0;
                        for (uint32_t j0 = s0; j0 < s1; j0 += 32) {
                            const uint32_t j = j0 + lane;
                            bool eE = false, eL = false;
                            int u = 0;
                            if (j < s1) {
                                u = P.nbr16[j];
                                const int gu = S::g(u);
                                uint8_t *pa = gam + (size_t)u * KP + S::phys(a, gu);
                                uint8_t *pb = gam + (size_t)u * KP + S::phys(b, gu);
                                const uint32_t oa = *pa, ob = *pb;
                                *pa = (uint8_t)(oa - 1);
                                *pb = (uint8_t)(ob + 1);
                                ovf |= (ob & GM) == GM;
                                eL = (oa & 0xBFu) == 0x81u;
                                eE = (ob & 0xBFu) == 0x80u;
                            }
                            __syncwarp();
                            const unsigned bE = __ballot_sync(FULLM, eE);
                            unsigned ball = bE | __ballot_sync(FULLM, eL);
                            while (ball) {
                                const int q = __ffs(ball) - 1;
                                ball &= ball - 1;
                                const int uq = __shfl_sync(FULLM, u, q);
                                WST(WS_EVENTS, 1);
                                if ((bE >> q) & 1u) cl_append(uq);
                                else cl_remove(uq);
                            }
                        }
                    }
                    if (Dg == 0) cl_remove(v);
                    __syncwarp();
                    WPH(WS_CY_EVENTS);
                    C = Cn;
                    if (__any_sync(FULLM, ovf)) {
                        bad = true;
                        break;
                    }
                    // ---- best (:387-390)
                    if (conflicts < best) {
                        best = conflicts;
                        WST(WS_BEST, 1);
                        __syncwarp();
                        const bool al16 = ((reinterpret_cast<uintptr_t>(b_out) & 15u) == 0);
                        for (int q = lane; 4 * q < n; q += 32) {
                            const uint32_t w4 = reinterpret_cast<const uint32_t *>(asg)[q];
                            if (al16 && 4 * q + 3 < n) {
                                reinterpret_cast<int4 *>(b_out)[q] =
                                    make_int4(w4 & 0xFF, (w4 >> 8) & 0xFF, (w4 >> 16) & 0xFF, w4 >> 24);
                            } else {
                                for (int e = 0; e < 4 && 4 * q + e < n; e++) b_out[4 * q + e] = (w4 >> (8 * e)) & 0xFF;
                            }
                        }
                    }
                }
                WPH(WS_CY_TAIL);
                it++;
                // ---- scratch check every 1024 iterations (:398-405)
                if (diagf && (it & 1023) == 0) {
                    __syncwarp();
                    long long c2 = 0;
                    for (int64_t e = lane; e < P.m; e += 32) c2 += asg[__ldg(P.eu + e)] == asg[__ldg(P.ev + e)];
                    c2 = warp_sum64(c2);
                    if (c2 != conflicts) diag++;
                }
            }
        }
        __syncwarp();

        if constexpr (stats) {
            if (lane == 0)
                for (int i = 0; i < WS_N; i++)
                    if (st[i]) atomicAdd(&g_wstats[i], (unsigned long long)st[i]);
        }
        if constexpr (stats)
            for (int i = 0; i < WS_N; i++) st[i] = 0;
        // ---------------- outputs (:407-410) ----------------
        if (!bad) {
            for (int v = lane; v < n; v += 32) a_io[v] = asg[v];
            if (lane == 0) {
                P.end_conflicts[ind] = conflicts;
                P.best_conflicts[ind] = best;
                P.iters_used[ind] = it;
                P.diag[ind] = diag;
                if (P.log_cnt) P.log_cnt[ind] = nlog;
                if (P.counters) {
                    P.counters[2 * (size_t)ind] = sum_c;
                    P.counters[2 * (size_t)ind + 1] = sum_deg;
                }
            }
        } else if (lane == 0) {
            const int s = atomicAdd(P.ovf_count, 1);
            P.ovf_list[s] = ind;
        }
        __syncwarp();
    }
}

#if !TW_STATS_TU
// lane-interleaved bitset: row v = 32 chunks of CH bits, bit q of chunk L <->
// vertex L + 32 q (bit index L*CH + q of the row)
__global__ void tw_bitset_kernel(const int64_t *indptr, const int32_t *indices, int n, int ch,
                                 uint32_t *bits) {
    const int row_words = ch;  // 32 * ch bits
    for (int v = blockIdx.x; v < n; v += gridDim.x) {
        uint32_t *row = bits + (size_t)v * row_words;
        for (int64_t i = indptr[v] + threadIdx.x; i < indptr[v + 1]; i += blockDim.x) {
            const int u = indices[i];
            const int bit = (u & 31) * ch + (u >> 5);
            atomicOr(row + (bit >> 5), 1u << (bit & 31));
        }
    }
}
__global__ void tw_csr16_kernel(const int64_t *indptr, const int32_t *indices, int n, int64_t nnz,
                                uint32_t *ip32, uint16_t *nb16) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i <= n; i += st) ip32[i] = (uint32_t)indptr[i];
    for (int64_t i = t0; i < nnz; i += st) nb16[i] = (uint16_t)indices[i];
}

#endif  // !TW_STATS_TU

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using KernT = void (*)(WarpTabuParams);

template <int KV, bool SPILL, bool STATS>
static KernT pick_mode(int ch) {
    switch (ch) {
        case 8: return tabucol_warp_kernel<KV, 8, true, SPILL, STATS>;
        case 16: return tabucol_warp_kernel<KV, 16, true, SPILL, STATS>;
        case 32: return tabucol_warp_kernel<KV, 32, true, SPILL, STATS>;
        default: return tabucol_warp_kernel<KV, 32, false, SPILL, STATS>;  // CSR, n <= 1024
    }
}
template <bool SPILL, bool STATS>
static KernT pick_kernel(int kv, int ch) {
    switch (kv) {
        case 1: return pick_mode<1, SPILL, STATS>(ch);
        case 2: return pick_mode<2, SPILL, STATS>(ch);
        case 3: return pick_mode<3, SPILL, STATS>(ch);
        case 4: return pick_mode<4, SPILL, STATS>(ch);
        case 6: return pick_mode<6, SPILL, STATS>(ch);
        case 8: return pick_mode<8, SPILL, STATS>(ch);
        default: return nullptr;
    }
}

static int upload_divtab(cudaStream_t st) {
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
    if (cudaMemcpyToSymbolAsync(g_divtab, tab, sizeof(tab), 0, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_warp: divisor table upload failed");
    done[d & 63] = true;
    return MCB_OK;
}

#if TW_STATS_TU
// the instrumented instantiations and the counters they write (this TU's
// g_wstats / g_divtab)
KernT tw_stats_kernel(int kv, int ch, bool spill) {
    return spill ? pick_kernel<true, true>(kv, ch) : pick_kernel<false, true>(kv, ch);
}
int tw_stats_prepare(cudaStream_t st) {
    unsigned long long z[40] = {0};
    cudaMemcpyToSymbolAsync(g_wstats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    return upload_divtab(st);
}
int tabucol_warp_stats(unsigned long long *out) {
    if (cudaMemcpyFromSymbol(out, g_wstats, sizeof(unsigned long long) * 40) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "warp stats unavailable");
    return MCB_OK;
}
#else
KernT tw_stats_kernel(int kv, int ch, bool spill);
int tw_stats_prepare(cudaStream_t st);
#endif

#if !TW_STATS_TU
struct WarpPlan {
    int kv, ch;  // ch = 0: CSR
    int warps, grid;
    size_t warp_smem, bitset_bytes, bitset_global;
};

static size_t tw_warp_bytes(int n, int kp) {
    auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    // gamma rows, scan records (u32), conflict list + positions (u16), colours (u8)
    return a16((size_t)n * kp + 4 * (size_t)n + 2 * a16(2 * (size_t)n) + a16((size_t)n));
}

// Returns false when the shape is outside the warp kernel's envelope.
static bool tw_plan(int n, int k, int64_t p, WarpPlan *pl) {
    if (getenv("MCB_NO_WARP_KERNEL")) return false;
    if (k < 1 || k > 128 || n < 1 || n > 1024 || p < 1) return false;
    static const int kvs[] = {1, 2, 3, 4, 6, 8};
    int kv = 0;
    for (int x : kvs)
        if (16 * x >= k) {
            kv = x;
            break;
        }
    if (!kv) return false;
    const int kp = 16 * kv;
    const size_t wb = tw_warp_bytes(n, kp);
    const size_t cap = (size_t)max_smem_optin();
    const int sms = num_sms();
    const int ch_need = (n + 31) / 32;
    const int ch = ch_need <= 8 ? 8 : ch_need <= 16 ? 16 : 32;
    const size_t bb = ((size_t)n * 4 * ch + 15) & ~(size_t)15;
    // warps wanted per SM: enough to cover p, at most TW_MAX_WARPS
    const int want = (int)std::min<int64_t>(TW_MAX_WARPS, (p + sms - 1) / sms);
    // bitset rows from L2 by default (all of shared memory for individuals);
    // MCB_WARP_BITSET_SMEM=1 keeps a CTA-shared copy (A/B)
    const bool bsm = getenv("MCB_WARP_BITSET_SMEM") != nullptr;
    const size_t bb_smem = bsm ? bb : 0;
    int w_bits = cap > bb_smem ? (int)std::min<size_t>((cap - bb_smem) / wb, TW_MAX_WARPS) : 0;
    int w_csr = (int)std::min<size_t>(cap / wb, TW_MAX_WARPS);
    if (getenv("MCB_WARP_CSR")) w_bits = 0;
    const char *mode = getenv("MCB_WARP_MODE");  // A/B: force "bits" or "csr"
    if (mode && !strcmp(mode, "csr")) w_bits = 0;
    if (mode && !strcmp(mode, "bits") && w_bits > 0) w_csr = 0;
    int use_ch;
    int w;
    // the bitset variant (neighbours from shared memory, no L2 round trip in the
    // update) beats CSR even with fewer resident individuals: measured 2.44e8
    // (7 warps/SM) vs 2.02e8 (8 warps/SM, CSR) at G(500,.5) k=48 D=8192
    if (w_bits >= 1 && (w_bits >= std::min(want, w_csr) || 4 * w_bits >= 3 * std::min(want, w_csr))) {
        use_ch = ch;
        w = std::min(w_bits, want);
    } else {
        use_ch = 0;
        w = std::min(w_csr, want);
    }
    if (const char *e = getenv("MCB_WARPS")) w = std::max(1, std::min(w, atoi(e)));
    if (w < 1) return false;
    if (use_ch) {
        // the unrolled update touches rows lane + 32 q for all q < CH
        const size_t need = (size_t)32 * use_ch * kp;
        if (need > wb) {
            const size_t wb2 = (need + 15) & ~(size_t)15;
            const int w2 = (int)std::min<size_t>((cap - bb_smem) / wb2, TW_MAX_WARPS);
            if (w2 < 1) return false;
            w = std::min(w, w2);
            pl->warp_smem = wb2;
        } else {
            pl->warp_smem = wb;
        }
    } else {
        pl->warp_smem = wb;
    }
    pl->kv = kv;
    pl->ch = use_ch;
    pl->warps = w;
    pl->bitset_bytes = use_ch ? bb_smem : 0;
    pl->bitset_global = use_ch ? bb : 0;
    const int64_t ctas = (p + w - 1) / w;
    pl->grid = (int)std::min<int64_t>(ctas, sms);
    return true;
}

// Launches the warp kernel; individuals it cannot finish (table overflow) are
// appended to ovf_list for the wide CTA kernel.  Returns MCB_OK, or -1 when
// the shape is outside the envelope (caller uses the CTA kernels).
int tabucol_warp_launch(const TabucolArgs &A, cudaStream_t st, int32_t *ctl32, int32_t *ovf_list,
                        int32_t *ovf_count, int32_t *err_flag, const int32_t *work_list, int64_t nwork,
                        bool spill, const int32_t *nwork_dev) {
    if (A.flags & (MCB_FLAG_FORCE_WIDE | MCB_FLAG_FORCE_GLOBAL | MCB_FLAG_PROFILE)) return -1;
    WarpPlan pl;
    if (nwork < 0) nwork = A.p;
    if (!tw_plan((int)A.n, (int)A.k, nwork, &pl)) return -1;
    const bool stats = (A.flags & MCB_FLAG_WSTATS) != 0;
    KernT kern = stats ? tw_stats_kernel(pl.kv, pl.ch, spill)
                       : (spill ? pick_kernel<true, false>(pl.kv, pl.ch) : pick_kernel<false, false>(pl.kv, pl.ch));
    if (!kern) return -1;
    if (int rc = upload_divtab(st)) return rc;
    if (stats)
        if (int rc = tw_stats_prepare(st)) return rc;  // resets this launch's counters
    const int n = (int)A.n, kp = 16 * pl.kv;
    const size_t smem = pl.bitset_bytes + (size_t)pl.warps * pl.warp_smem;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_warp: smem attribute (%zu) failed", smem);
    // SPILL: 256 rows x 32 entries per resident warp (tenure < 8190 keeps the
    // live rows of register ring + spill under 32 + 256)
    constexpr int SPILL_ROWS = 256;
    const size_t spill_bytes = spill ? (size_t)pl.grid * pl.warps * SPILL_ROWS * 32 * 4 : 0;
    (void)kp;
    const int64_t nnz_h = 2 * A.m;  // CSR of an undirected graph (no host read of indptr[n])
    const size_t graph_bytes = pl.ch ? pl.bitset_global : (4 * (size_t)(n + 1) + 2 * (size_t)nnz_h + 256);
    uint8_t *ws = (uint8_t *)workspace2(spill_bytes + graph_bytes + 512);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol_warp: workspace allocation failed");
    WarpTabuParams P{};
    P.assigns = A.assigns;
    P.best_assigns = A.best_assigns;
    P.spill = spill ? reinterpret_cast<uint32_t *>(ws) : nullptr;
    P.spill_rows = SPILL_ROWS;
    P.work_list = work_list;
    uint8_t *gbase = ws + ((spill_bytes + 255) & ~(size_t)255);
    if (pl.ch) {
        if (cudaMemsetAsync(gbase, 0, pl.bitset_global, st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "memset failed");
        tw_bitset_kernel<<<std::min(n, 4 * num_sms()), 128, 0, st>>>(A.indptr, A.indices, n, pl.ch,
                                                                    reinterpret_cast<uint32_t *>(gbase));
        P.bitset = gbase;
    } else {
        uint32_t *ip = reinterpret_cast<uint32_t *>(gbase);
        uint16_t *nb = reinterpret_cast<uint16_t *>(gbase + ((4 * (size_t)(n + 1) + 255) & ~(size_t)255));
        tw_csr16_kernel<<<4 * num_sms(), 256, 0, st>>>(A.indptr, A.indices, n, nnz_h, ip, nb);
        P.indptr32 = ip;
        P.nbr16 = nb;
    }
    P.eu = A.eu;
    P.ev = A.ev;
    P.m = A.m;
    P.n = n;
    P.k = (int)A.k;
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
    P.nwork = (int)nwork;
    P.nwork_dev = nwork_dev;
    P.work_counter = ctl32;
    P.ovf_list = ovf_list;
    P.ovf_count = ovf_count;
    P.err_flag = err_flag;
    P.flags = A.flags;
    P.warp_smem = (int)pl.warp_smem;
    P.bitset_bytes = (int)pl.bitset_bytes;
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] tabucol_warp<kv=%d,%s%d%s> grid=%d warps/CTA=%d smem=%zu work=%lld\n", pl.kv,
                pl.ch ? "bitset ch=" : "csr", pl.ch, spill ? ",spill" : "", pl.grid, pl.warps, smem,
                (long long)nwork);
    kern<<<pl.grid, 32 * pl.warps, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol_warp launch failed");
    return MCB_OK;
}

}  // namespace mcb


namespace mcb {
// Diagnostics: the table divisibility test against the 64-bit %, s in [1, 63]
__global__ void divcheck_kernel(int64_t count, unsigned long long *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x0 = stream_value(0x5151ull, (uint64_t)i);
        const uint32_t s = 1 + (uint32_t)(stream_value(0x7777ull, (uint64_t)i) % 63);
        const uint64_t x = (i & 1) ? x0 : (x0 / s) * s;
        if (divisible(x, s) != (x % s == 0)) atomicAdd(bad, 1ull);
    }
}
int tabucol_warp_divcheck(int64_t count, unsigned long long *mismatches) {
    if (int rc = upload_divtab(0)) return rc;
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return MCB_ERR_CUDA;
    cudaMemset(d, 0, sizeof(*d));
    divcheck_kernel<<<1184, 256>>>(count, d);
    const cudaError_t e = cudaMemcpy(mismatches, d, sizeof(*d), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? MCB_OK : MCB_ERR_CUDA;
}
}  // namespace mcb

namespace mcb {
// The kernel variant tabucol_run would launch for (n, k, p), as text.
int tabucol_warp_describe(int64_t n, int64_t k, int64_t p, char *buf, int len) {
    WarpPlan pl;
    if (!tw_plan((int)n, (int)k, p, &pl)) {
        return tabucol_cta_describe(n, k, p, buf, len);  // shape outside the warp kernel
    }
    snprintf(buf, len, "tabucol_warp_kernel<KV=%d,%s> %d warps/CTA x %d CTAs, %zu B smem/individual", pl.kv,
             pl.ch ? (pl.ch == 8 ? "bitset CH=8" : pl.ch == 16 ? "bitset CH=16" : "bitset CH=32") : "csr",
             pl.warps, pl.grid, pl.warp_smem);
    return MCB_OK;
}
}  // namespace mcb

#endif  // !TW_STATS_TU

#if TW_STATS_TU
}  // namespace mcb
#endif
