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
// independent individuals as shared memory holds (7 at G(500,.5) k=48).
//
// Gamma byte per (vertex, colour), shared memory, rows of KP = 16 KV bytes:
//     bit 7  OWN   the vertex's own colour (never a candidate)
//     bit 6  TABU  (vertex, colour) is tabu this iteration
//     bits 0-5     gamma = #neighbours of that colour (<= 63, else the
//                  individual is re-run by the wide CTA kernel, tabucol.cu)
//     padding colours 0xFF.
// So a row's candidate moves are exactly its bytes < 0x40, and the row minimum
// is a branch-free SIMD byte minimum.  Aspiration (a tabu move reaching a new
// best: gamma < gva + best - conflicts) is only possible when gva + best -
// conflicts > 0; then the row's tabu bytes are folded in (bytes ^ 0x40).
//
// Tabu expiry is exact and eager: every tabu entry (v, c, expiry) lives in a
// register ring (lane = insertion % 32, register = insertion / 32 mod 32,
// 1024 live entries); each ring row tracks its earliest expiry (lane-
// distributed), and only rows whose earliest expiry has come are touched --
// expired entries clear their TABU bit.  Re-tabu of a tabu pair invalidates
// the older entry (last write wins, :366).
//
// Per CTA: the adjacency as a bitset, row v = 32 lane chunks of CH bits (lane
// L owns vertices [L*CH, L*CH+CH)), so the neighbour update of a move is one
// chunk load per lane and neighbours come out in ascending order.  Graphs whose
// bitset does not fit use the CSR (u16 indices, L2) variant.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace mcb {

namespace {

constexpr int TW_BIG = 1 << 20;
constexpr unsigned FULLM = 0xffffffffu;
constexpr int TW_MAX_WARPS = 8;
constexpr int KE = 32;  // ring registers per lane -> 1024 live tabu entries
constexpr uint32_t OWN = 0x80u, TABU = 0x40u, GM = 0x3Fu;

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
    int32_t *work_counter;
    int32_t *ovf_list, *ovf_count, *err_flag;
    uint32_t flags;
    int warp_smem;     // bytes per warp region
    int bitset_bytes;  // bytes of the CTA-shared bitset (0 for CSR)
};

__device__ unsigned long long g_wstats[32];
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
    WS_CY_SCAN = 16,
    WS_CY_SELECT,
    WS_CY_MOVE,
    WS_CY_UPDATE,
    WS_CY_EVENTS,
    WS_CY_TAIL,
    WS_CY_EXPIRE,
    WS_N = 32
};
#define WST(i, x) \
    if (stats) st[i] += (x)
#define WPH(i)                          \
    if (stats) {                        \
        const long long _t = clock64(); \
        st[i] += _t - ph_t;             \
        ph_t = _t;                      \
    }

template <int CH>
struct ChunkT;
template <>
struct ChunkT<8> {
    using T = uint8_t;
};
template <>
struct ChunkT<16> {
    using T = uint16_t;
};
template <>
struct ChunkT<32> {
    using T = uint32_t;
};

// 0x80 in every byte of x that is zero
__device__ __forceinline__ uint32_t zero_flags(uint32_t z) {
    return ~(((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & 0x80808080u;
}
__device__ __forceinline__ int count_eq(uint32_t x, uint32_t M) { return __popc(zero_flags(x ^ M)); }
__device__ __forceinline__ uint32_t min_bytes(uint32_t x) {
    const uint32_t m2 = __vminu2(x & 0x00FF00FFu, __byte_perm(x, 0, 0x4341));
    return min(m2 & 0xFFFFu, m2 >> 16);
}
// (minimum byte, #bytes at it) of a row held as KW words
template <int KW>
__device__ __forceinline__ void row_min_count(const uint32_t (&x)[KW], uint32_t xorv, int &m, int &c) {
    uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu, m3 = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < KW; w += 2) {
        const uint32_t y0 = x[w] ^ xorv;
        m0 = __vminu2(m0, y0 & 0x00FF00FFu);
        m1 = __vminu2(m1, __byte_perm(y0, 0, 0x4341));
        if (w + 1 < KW) {
            const uint32_t y1 = x[w + 1] ^ xorv;
            m2 = __vminu2(m2, y1 & 0x00FF00FFu);
            m3 = __vminu2(m3, __byte_perm(y1, 0, 0x4341));
        }
    }
    const uint32_t mm = __vminu2(__vminu2(m0, m1), __vminu2(m2, m3));
    m = (int)min(mm & 0xFFFFu, mm >> 16);
    const uint32_t M = ((uint32_t)m * 0x01010101u) ^ xorv;
    c = 0;
#pragma unroll
    for (int w = 0; w < KW; w++) c += count_eq(x[w], M);
}
template <int KV>
__device__ __forceinline__ void load_row(const uint8_t *grow, uint32_t (&x)[4 * KV]) {
    const uint4 *r4 = reinterpret_cast<const uint4 *>(grow);
#pragma unroll
    for (int q = 0; q < KV; q++) {
        const uint4 t4 = r4[q];
        x[4 * q] = t4.x;
        x[4 * q + 1] = t4.y;
        x[4 * q + 2] = t4.z;
        x[4 * q + 3] = t4.w;
    }
}
// minimum byte of (row ^ xorv)
template <int KW>
__device__ __forceinline__ int row_min(const uint32_t (&x)[KW], uint32_t xorv) {
    uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu, m3 = 0xFFFFFFFFu;
#pragma unroll
    for (int w = 0; w < KW; w += 2) {
        const uint32_t y0 = x[w] ^ xorv;
        m0 = __vminu2(m0, y0 & 0x00FF00FFu);
        m1 = __vminu2(m1, __byte_perm(y0, 0, 0x4341));
        if (w + 1 < KW) {
            const uint32_t y1 = x[w + 1] ^ xorv;
            m2 = __vminu2(m2, y1 & 0x00FF00FFu);
            m3 = __vminu2(m3, __byte_perm(y1, 0, 0x4341));
        }
    }
    const uint32_t mm = __vminu2(__vminu2(m0, m1), __vminu2(m2, m3));
    return (int)min(mm & 0xFFFFu, mm >> 16);
}
// #bytes of the row equal to byte value b
template <int KW>
__device__ __forceinline__ int row_count(const uint32_t (&x)[KW], uint32_t b) {
    const uint32_t M = b * 0x01010101u;
    int c = 0;
#pragma unroll
    for (int w = 0; w < KW; w++) c += count_eq(x[w], M);
    return c;
}
// candidate bytes of word x (gamma value), every non-candidate 0xFF: plain
// bytes < 0x40, plus (A > 0) tabu bytes of gamma < A (aspiration)
__device__ __forceinline__ uint32_t cand_word(uint32_t x, int A) {
    uint32_t y = x | ((((x | (x << 1)) & 0x80808080u) >> 7) * 0xFFu);
    if (A > 0) {
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint32_t b = (x >> (8 * e)) & 0xFFu;
            if ((b & 0xC0u) == TABU && (int)(b & GM) < A) y = (y & ~(0xFFu << (8 * e))) | ((b & GM) << (8 * e));
        }
    }
    return y;
}

template <int W>
__device__ __forceinline__ int seg_excl_min(int v, int li) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < W; o <<= 1) {
        const int t = __shfl_up_sync(FULLM, incl, o, W);
        if (li >= o) incl = min(incl, t);
    }
    int ex = __shfl_up_sync(FULLM, incl, 1, W);
    return li == 0 ? INT_MAX : ex;
}
template <int W>
__device__ __forceinline__ int seg_sum(int v) {
#pragma unroll
    for (int o = W >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(FULLM, v, o, W);
    return v;
}

// ring register access with a uniform row index (jump table; keeps the ring
// in registers)
#define TW_C4(b) TW_C(b) TW_C(b + 1) TW_C(b + 2) TW_C(b + 3)
__device__ __forceinline__ uint32_t ring_get(const uint32_t (&r)[KE], int j) {
    uint32_t x = 0;
    switch (j) {
#define TW_C(J) \
    case J: x = r[J]; break;
        TW_C4(0) TW_C4(4) TW_C4(8) TW_C4(12) TW_C4(16) TW_C4(20) TW_C4(24) TW_C4(28)
#undef TW_C
    }
    return x;
}
__device__ __forceinline__ void ring_set(uint32_t (&r)[KE], int j, uint32_t x) {
    switch (j) {
#define TW_C(J) \
    case J: r[J] = x; break;
        TW_C4(0) TW_C4(4) TW_C4(8) TW_C4(12) TW_C4(16) TW_C4(20) TW_C4(24) TW_C4(28)
#undef TW_C
    }
}
// entry: [valid:1][v:10][c:7][expiry mod 2^14:14]
__device__ __forceinline__ uint32_t ent_pack(int v, int c, uint32_t e) {
    return 0x80000000u | ((uint32_t)v << 21) | ((uint32_t)c << 14) | (e & 0x3FFFu);
}
__device__ __forceinline__ uint32_t ent_dist(uint32_t ent, uint32_t it) { return (ent - it) & 0x3FFFu; }

}  // namespace

// ---------------------------------------------------------------------------
// the kernel
//   KV     = 16-byte vectors per gamma row (KP = 16 KV >= k)
//   CH     = bitset chunk bits per lane (BITSET) -- n <= 32 CH
// ---------------------------------------------------------------------------
template <int KV, int CH, bool BITSET>
__global__ void __launch_bounds__(32 * TW_MAX_WARPS, 1) tabucol_warp_kernel(WarpTabuParams P) {
    constexpr int KP = 16 * KV, KW = 4 * KV;
    constexpr int SW = KW <= 4 ? 4 : KW <= 8 ? 8 : KW <= 16 ? 16 : 32;  // walk segment width
    constexpr int RPP = 32 / SW;                                          // rows per walk pass
    static_assert(KW <= 32, "k <= 128");
    using CT = typename ChunkT<BITSET ? CH : 32>::T;

    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n = P.n, k = P.k;

    // CTA-shared adjacency bitset (read-only afterwards; warps never sync again)
    if constexpr (BITSET) {
        const uint4 *src = reinterpret_cast<const uint4 *>(P.bitset);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < P.bitset_bytes / 16; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    uint8_t *base = smem + P.bitset_bytes + (size_t)wid * P.warp_smem;
    uint8_t *gam = base;
    size_t off = (size_t)n * KP;
    uint32_t *rmc = reinterpret_cast<uint32_t *>(base + off);  // per scanned row: (int16 delta) | count << 16
    off += 4 * (size_t)n;
    uint16_t *clist = reinterpret_cast<uint16_t *>(base + off);
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint16_t *cpos = reinterpret_cast<uint16_t *>(base + off);  // position in clist (members only)
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint8_t *asg = base + off;

    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool cnt_on = P.counters != nullptr;
    const bool stats = (P.flags & MCB_FLAG_WSTATS) != 0;
    long long st[WS_N];
    if (stats)
        for (int i = 0; i < WS_N; i++) st[i] = 0;

    for (;;) {
        int wi = 0;
        if (lane == 0) wi = atomicAdd(P.work_counter, 1);
        wi = __shfl_sync(FULLM, wi, 0);
        if (wi >= P.nwork) break;
        const int ind = wi;
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
            const uint32_t padw = (k & 3) ? (0xFFFFFFFFu << (8 * (k & 3))) : 0u;
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gam);
            for (int i = lane; i < n * KW; i += 32) {
                const int w = i % KW;
                g32[i] = (4 * w + 4 <= k) ? 0u : (4 * w >= k ? 0xFFFFFFFFu : padw);
            }
        }
        __syncwarp();
        // gamma[u][c] = #neighbours of u coloured c; lane-private rows
        for (int u = lane; u < n; u += 32) {
            uint8_t *row = gam + (size_t)u * KP;
            if constexpr (BITSET) {
                const CT *br = reinterpret_cast<const CT *>(smem + (size_t)u * 4 * CH);
                for (int L = 0; L < 32; L++) {
                    uint32_t ch = br[L];
                    while (ch) {
                        const int j = __ffs(ch) - 1;
                        ch &= ch - 1;
                        const int c = asg[L * CH + j];
                        const int x = row[c] + 1;
                        if (x > (int)GM) bad = true;
                        else row[c] = (uint8_t)x;
                    }
                }
            } else {
                const uint32_t s0 = P.indptr32[u], s1 = P.indptr32[u + 1];
                for (uint32_t idx = s0; idx < s1; idx++) {
                    const int c = asg[P.nbr16[idx]];
                    const int x = row[c] + 1;
                    if (x > (int)GM) bad = true;
                    else row[c] = (uint8_t)x;
                }
            }
        }
        __syncwarp();
        long long conflicts, best;
        int C = 0;
        {
            long long c2 = 0;
            for (int v0 = 0; v0 < n; v0 += 32) {
                const int v = v0 + lane;
                bool f = false;
                if (v < n) {
                    uint8_t *p = gam + (size_t)v * KP + asg[v];
                    const int g = *p;
                    *p = (uint8_t)(g | OWN);
                    f = g > 0;
                    c2 += g;
                }
                const unsigned bal = __ballot_sync(FULLM, f);
                if (f) {
                    const int pos = C + __popc(bal & ((1u << lane) - 1u));
                    clist[pos] = (uint16_t)v;
                    cpos[v] = (uint16_t)pos;
                }
                C += __popc(bal);
            }
            c2 = warp_sum64(c2);
            conflicts = c2 / 2;
            best = conflicts;
        }
        if (__any_sync(FULLM, rangeerr) && lane == 0) atomicExch(P.err_flag, 1);
        bad = __any_sync(FULLM, bad);
        __syncwarp();

        long long it = 0, nlog = 0, sum_c = 0, sum_deg = 0, diag = 0;
        unsigned long long ctr = 0;
        // tabu ring (see header); rlive/rmin: live count and earliest expiry of
        // ring row `lane`
        uint32_t ring[KE];
#pragma unroll
        for (int j = 0; j < KE; j++) ring[j] = 0u;
        int rlive = 0;
        uint32_t rmin = 0;
        uint32_t ins = 0;

        // ---------------- iterations (:320-405) ----------------
        if (k >= 2 && !bad) {
            for (long long step = 0; step < P.depth; step++) {
                if (conflicts == 0) break;
                long long ph_t = stats ? clock64() : 0;
                WST(WS_IT, 1);
                const uint32_t it32 = (uint32_t)it;
                const int thr = (int)max(best - conflicts, (long long)-TW_BIG);

                // ---- tabu expiry: it < tabu[v,c] fails from it == expiry on
                {
                    unsigned due = __ballot_sync(FULLM, rlive > 0 && (int)(rmin - it32) <= 0);
                    while (due) {
                        const int j = __ffs(due) - 1;
                        due &= due - 1;
                        WST(WS_EXPIRE_ROWS, 1);
                        const uint32_t e = ring_get(ring, j);
                        const bool valid = (e >> 31) != 0u;
                        const uint32_t dist = ent_dist(e, it32);
                        const bool hit = valid && dist == 0u;
                        if (hit) {
                            const int v = (e >> 21) & 0x3FF, c = (e >> 14) & 0x7F;
                            gam[(size_t)v * KP + c] &= (uint8_t)~TABU;
                            ring_set(ring, j, 0u);
                        }
                        const bool still = valid && !hit;
                        const int cnt = __popc(__ballot_sync(FULLM, still));
                        const unsigned dmin = __reduce_min_sync(FULLM, still ? dist : 0xFFFFu);
                        if (lane == j) {
                            rlive = cnt;
                            rmin = it32 + dmin;
                        }
                    }
                    __syncwarp();
                }
                WPH(WS_CY_EXPIRE);

                // ---- scan, phase 1 (localsearch.py:328-350): row minima, one
                // conflicting row per lane; running prefix-min over the rows in list
                // order; exact walks of the rows that lower it.  Rows at or below
                // the running minimum -- the only ones holding reservoir events --
                // are appended to a compact list (rmc) for phase 2.
                int carry = TW_BIG, total = 0, ncl = 0;
                const int nr = (C + 31) >> 5;
#pragma unroll 1
                for (int r = 0; r < nr; r++) {
                    const int li = r * 32 + lane;
                    int rm = TW_BIG, v = 0, gva = 0, A = 0;
                    if (li < C) {
                        v = clist[li];
                        const uint8_t *grow = gam + (size_t)v * KP;
                        const int a = asg[v];
                        uint32_t x[KW];
                        load_row<KV>(grow, x);
                        gva = grow[a] & GM;
                        A = gva + thr;
                        int m = row_min<KW>(x, 0u);  // non-own, non-tabu (bytes < 0x40)
                        if (A > 0) {
                            // aspiration: tabu colours with gamma < A are admissible
                            const int mt = row_min<KW>(x, TABU * 0x01010101u);
                            if (mt < A) m = min(m, mt);
                        }
                        if (m < (int)TABU) rm = m - gva;
                    }
                    if (stats) WST(WS_ASP_ROUNDS, __any_sync(FULLM, A > 0));
                    // running minimum entering this row
                    int incl = rm;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(FULLM, incl, o);
                        if (lane >= o) incl = min(incl, t);
                    }
                    int Pl = __shfl_up_sync(FULLM, incl, 1);
                    if (lane == 0) Pl = TW_BIG;
                    Pl = min(Pl, carry);
                    {
                        const bool lst = rm < TW_BIG && rm <= Pl;
                        const unsigned nb = __ballot_sync(FULLM, lst);
                        if (lst)
                            rmc[ncl + __popc(nb & ((1u << lane) - 1u))] =
                                (uint32_t)li | ((uint32_t)(rm + 64) << 16) | (rm == Pl ? 1u << 24 : 0u);
                        ncl += __popc(nb);
                    }
                    if (!prod) {
                        // rows that lower the running minimum: exact in-row walks,
                        // RPP rows per pass (lanes over words)
                        unsigned low = __ballot_sync(FULLM, rm < Pl);
                        while (low) {
                            WST(WS_WALK_PASSES, 1);
                            const int g = lane / SW, wl = lane % SW;
                            unsigned tmp = low;
#pragma unroll
                            for (int q = 0; q < RPP - 1; q++)
                                if (q < g) tmp &= tmp - 1;
                            const int src = tmp ? __ffs(tmp) - 1 : -1;
                            const int s = src < 0 ? 0 : src;
                            const int wv = __shfl_sync(FULLM, v, s);
                            const int wg = __shfl_sync(FULLM, gva, s);
                            const int wA = __shfl_sync(FULLM, A, s);
                            const int wP = __shfl_sync(FULLM, Pl, s);
                            uint32_t x = 0xFFFFFFFFu;
                            if (src >= 0 && wl < KW)
                                x = cand_word(reinterpret_cast<const uint32_t *>(gam + (size_t)wv * KP)[wl], wA);
                            const int um = (int)min_bytes(x);
                            const int ex = seg_excl_min<SW>(um == 0xFF ? INT_MAX : um, wl);
                            int cur = min(wP >= TW_BIG ? INT_MAX : wP + wg, ex);
                            int t = 0;
#pragma unroll
                            for (int e = 0; e < 4; e++) {
                                const int b = (x >> (8 * e)) & 0xFF;
                                if (b == 0xFF) continue;
                                if (b < cur) cur = b;
                                else if (b == cur) t++;
                            }
                            t = seg_sum<SW>(t);
                            if (wl == 0 && src >= 0) total += t;
#pragma unroll
                            for (int q = 0; q < RPP; q++) low &= low - 1;
                        }
                    }
                    carry = min(carry, __shfl_sync(FULLM, incl, 31));
                }
                __syncwarp();
                const int D = carry;
                WST(WS_ROUNDS, nr);
                WPH(WS_CY_SCAN);
                if (cnt_on) sum_c += C;

                int mv_v = -1, mv_a = 0, mv_b = 0, Dg = 0;
                if (D < TW_BIG) {
                    // ---- phase 2: tie counts of the listed rows.  Rows equal to the
                    // running minimum contribute all their minimum candidates as tie
                    // events; rows at D contribute T, the final group.
                    int T = 0;
                    for (int b0 = 0; b0 < ncl; b0 += 32) {
                        const int i = b0 + lane;
                        int cD = 0;
                        if (i < ncl) {
                            const uint32_t e = rmc[i];
                            const int li = (int)(e & 0xFFFFu), rm = (int)((e >> 16) & 0xFFu) - 64;
                            const bool tie = (e >> 24) & 1u;
                            int cnt = 0;
                            if (tie || rm == D) {
                                const int v = clist[li];
                                const uint8_t *grow = gam + (size_t)v * KP;
                                uint32_t x[KW];
                                load_row<KV>(grow, x);
                                const int gva = grow[asg[v]] & GM;
                                const int m = rm + gva;
                                cnt = row_count<KW>(x, (uint32_t)m);
                                if (m < gva + thr) cnt += row_count<KW>(x, (uint32_t)m | TABU);
                            }
                            if (tie) total += cnt;
                            if (rm == D) cD = cnt;
                            rmc[i] = (uint32_t)li | ((uint32_t)cD << 16);
                        }
                        T += __reduce_add_sync(FULLM, cD);
                    }
                    const int tot = prod ? 0 : __reduce_add_sync(FULLM, total);
                    // tenure draw (:363-365), issued early so it overlaps the reservoir
                    const long long nconf = conflicts + D;
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
                            for (int s = 2 + lane; s <= T; s += 32)
                                if (mod_is_zero(stream_value(key, c0 + (unsigned long long)(s - 2)), (uint32_t)s))
                                    smax = s;
                            sstar = __reduce_max_sync(FULLM, smax);
                        } else {
                            sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                        }
                    }
                    // ---- locate the sstar-th D-candidate in scan order
                    int row_li = 0, need = sstar;
                    {
                        int cum = 0;
                        for (int b0 = 0; b0 < ncl; b0 += 32) {
                            const int i = b0 + lane;
                            int cc = 0, li = 0;
                            if (i < ncl) {
                                const uint32_t e = rmc[i];
                                li = (int)(e & 0xFFFFu);
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
                                const unsigned bm = __ballot_sync(FULLM, cum + incl >= sstar);
                                const int src = __ffs(bm) - 1;
                                row_li = __shfl_sync(FULLM, li, src);
                                need = sstar - cum - __shfl_sync(FULLM, incl - cc, src);
                                break;
                            }
                            cum += rt;
                        }
                    }
                    const int v = clist[row_li];
                    uint8_t *grow = gam + (size_t)v * KP;
                    const int a = asg[v];
                    const int gva = grow[a] & GM;
                    const int A = gva + thr;
                    Dg = D + gva;
                    int b = -1;
                    {
                        uint32_t x = 0xFFFFFFFFu;
                        int cc = 0;
                        if (lane < KW) {
                            x = cand_word(reinterpret_cast<const uint32_t *>(grow)[lane], A);
                            cc = count_eq(x, (uint32_t)Dg * 0x01010101u);
                        }
                        int incl = cc;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int t = __shfl_up_sync(FULLM, incl, o);
                            if (lane >= o) incl += t;
                        }
                        const unsigned bm = __ballot_sync(FULLM, incl >= need);
                        const int src = bm ? __ffs(bm) - 1 : 0;
                        int col = -1;
                        if (lane == src && bm) {
                            int rr = need - (incl - cc);
#pragma unroll
                            for (int e = 0; e < 4; e++)
                                if ((int)((x >> (8 * e)) & 0xFF) == Dg && --rr == 0 && col < 0) col = 4 * lane + e;
                        }
                        b = __shfl_sync(FULLM, col, src);
                    }
                    if (b < 0) {
                        bad = true;  // cannot happen; route to the wide kernel
                        break;
                    }
                    WPH(WS_CY_SELECT);
                    // ---- move, tenure, tabu entry (:352-366)
                    conflicts = nconf;
                    ctr += prod ? 2ull : (unsigned long long)tot + 1ull;
                    const long long tt = (long long)ll + (6LL * conflicts) / 10LL;
                    if (tt >= 8190) {
                        bad = true;
                        break;
                    }
                    const uint32_t e_new = it32 + (uint32_t)tt + 1u;
                    const uint32_t ba = grow[a];
                    if (ba & TABU) {
                        // (v, a) is re-tabu'd while tabu: the older entry is void
                        WST(WS_SUPERSEDE, 1);
                        const uint32_t key_vc = ent_pack(v, a, 0) & 0xFFFFC000u;
                        unsigned lv = __ballot_sync(FULLM, rlive > 0);
                        while (lv) {
                            const int j = __ffs(lv) - 1;
                            lv &= lv - 1;
                            const uint32_t e = ring_get(ring, j);
                            const bool hit = (e & 0xFFFFC000u) == key_vc;
                            const unsigned hb = __ballot_sync(FULLM, hit);
                            if (hb) {
                                if (hit) ring_set(ring, j, 0u);
                                if (lane == j) rlive--;
                                break;
                            }
                        }
                    }
                    {
                        const int j = (int)((ins >> 5) % KE), L = (int)(ins & 31u);
                        if (L == 0 && __shfl_sync(FULLM, rlive, j) > 0) {
                            bad = true;  // a tabu entry outlived 1000 insertions
                            break;
                        }
                        if (lane == L) ring_set(ring, j, ent_pack(v, a, e_new));
                        if (lane == j) {
                            rmin = (rlive == 0 || (int)(e_new - rmin) < 0) ? e_new : rmin;
                            rlive++;
                        }
                        ins++;
                    }
                    if (lane == 0) {
                        asg[v] = (uint8_t)b;
                        grow[a] = (uint8_t)((ba & GM) | TABU);
                        grow[b] = (uint8_t)(grow[b] | OWN);
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
                        uint32_t ch = reinterpret_cast<const CT *>(smem + (size_t)v * 4 * CH)[lane];
                        if (cnt_on) sum_deg += __reduce_add_sync(FULLM, __popc(ch));
                        uint32_t evE = 0, evL = 0;
                        uint8_t *ga = gam + a, *gb = gam + b;
                        const int ubase = lane * CH;
                        while (ch) {
                            // up to 4 neighbours per pass: all loads in flight before
                            // the stores (distinct rows, no aliasing)
                            int jj[4];
                            uint8_t *pa[4], *pb[4];
                            uint32_t oa[4], ob[4];
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                jj[q] = __ffs(ch) - 1;
                                ch &= ch - 1;
                                const int u = ubase + max(jj[q], 0);
                                pa[q] = ga + (size_t)u * KP;
                                pb[q] = gb + (size_t)u * KP;
                            }
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (jj[q] >= 0) {
                                    oa[q] = *pa[q];
                                    ob[q] = *pb[q];
                                }
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if (jj[q] >= 0) {
                                    *pa[q] = (uint8_t)(oa[q] - 1);
                                    *pb[q] = (uint8_t)(ob[q] + 1);
                                    ovf |= (ob[q] & GM) == GM;
                                    evL |= ((oa[q] & 0xBFu) == 0x81u) ? 1u << jj[q] : 0u;
                                    evE |= ((ob[q] & 0xBFu) == 0x80u) ? 1u << jj[q] : 0u;
                                }
                        }
                        __syncwarp();
                        WPH(WS_CY_UPDATE);
                        unsigned lw = __ballot_sync(FULLM, (evE | evL) != 0u);
                        while (lw) {
                            const int L = __ffs(lw) - 1;
                            lw &= lw - 1;
                            const uint32_t E = __shfl_sync(FULLM, evE, L);
                            uint32_t all = E | __shfl_sync(FULLM, evL, L);
                            while (all) {
                                const int j = __ffs(all) - 1;
                                all &= all - 1;
                                const int u = L * CH + j;
                                WST(WS_EVENTS, 1);
                                if ((E >> j) & 1u) cl_append(u);
                                else cl_remove(u);
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
                                uint8_t *pa = gam + (size_t)u * KP + a, *pb = gam + (size_t)u * KP + b;
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

        if (stats && lane == 0)
            for (int i = 0; i < WS_N; i++)
                if (st[i]) atomicAdd(&g_wstats[i], (unsigned long long)st[i]);
        if (stats)
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

__global__ void tw_bitset_kernel(const int64_t *indptr, const int32_t *indices, int n, int row_bytes,
                                 uint32_t *bits) {
    for (int v = blockIdx.x; v < n; v += gridDim.x) {
        uint32_t *row = bits + (size_t)v * (row_bytes / 4);
        for (int64_t i = indptr[v] + threadIdx.x; i < indptr[v + 1]; i += blockDim.x) {
            const int u = indices[i];
            atomicOr(row + (u >> 5), 1u << (u & 31));
        }
    }
}
__global__ void tw_csr16_kernel(const int64_t *indptr, const int32_t *indices, int n, int64_t nnz,
                                uint32_t *ip32, uint16_t *nb16) {
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t0; i <= n; i += st) ip32[i] = (uint32_t)indptr[i];
    for (int64_t i = t0; i < nnz; i += st) nb16[i] = (uint16_t)indices[i];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using KernT = void (*)(WarpTabuParams);

template <int KV>
static KernT pick_mode(int ch) {
    switch (ch) {
        case 8: return tabucol_warp_kernel<KV, 8, true>;
        case 16: return tabucol_warp_kernel<KV, 16, true>;
        case 32: return tabucol_warp_kernel<KV, 32, true>;
        default: return tabucol_warp_kernel<KV, 32, false>;  // CSR, n <= 1024
    }
}
static KernT pick_kernel(int kv, int ch) {
    switch (kv) {
        case 1: return pick_mode<1>(ch);
        case 2: return pick_mode<2>(ch);
        case 3: return pick_mode<3>(ch);
        case 4: return pick_mode<4>(ch);
        case 6: return pick_mode<6>(ch);
        case 8: return pick_mode<8>(ch);
        default: return nullptr;
    }
}

struct WarpPlan {
    int kv, ch;  // ch = 0: CSR
    int warps, grid;
    size_t warp_smem, bitset_bytes;
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
    int w_bits = cap > bb ? (int)std::min<size_t>((cap - bb) / wb, TW_MAX_WARPS) : 0;
    int w_csr = (int)std::min<size_t>(cap / wb, TW_MAX_WARPS);
    if (getenv("MCB_WARP_CSR")) w_bits = 0;
    int use_ch;
    int w;
    if (w_bits >= std::min(want, w_csr)) {
        use_ch = ch;
        w = std::min(w_bits, want);
    } else {
        use_ch = 0;
        w = std::min(w_csr, want);
    }
    if (const char *e = getenv("MCB_WARPS")) w = std::max(1, std::min(w, atoi(e)));
    if (w < 1) return false;
    pl->kv = kv;
    pl->ch = use_ch;
    pl->warps = w;
    pl->warp_smem = wb;
    pl->bitset_bytes = use_ch ? bb : 0;
    const int64_t ctas = (p + w - 1) / w;
    pl->grid = (int)std::min<int64_t>(ctas, sms);
    return true;
}

// Launches the warp kernel; individuals it cannot finish (table overflow) are
// appended to ovf_list for the wide CTA kernel.  Returns MCB_OK, or -1 when
// the shape is outside the envelope (caller uses the CTA kernels).
int tabucol_warp_launch(const TabucolArgs &A, cudaStream_t st, int32_t *ctl32, int32_t *ovf_list,
                        int32_t *ovf_count, int32_t *err_flag) {
    if (A.flags & (MCB_FLAG_FORCE_WIDE | MCB_FLAG_FORCE_GLOBAL | MCB_FLAG_PROFILE)) return -1;
    if (A.flags & MCB_FLAG_WSTATS) {
        // reset the counters of this launch
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbolAsync(g_wstats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    }
    WarpPlan pl;
    if (!tw_plan((int)A.n, (int)A.k, A.p, &pl)) return -1;
    KernT kern = pick_kernel(pl.kv, pl.ch);
    if (!kern) return -1;
    const int n = (int)A.n, kp = 16 * pl.kv;
    const size_t smem = pl.bitset_bytes + (size_t)pl.warps * pl.warp_smem;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_warp: smem attribute (%zu) failed", smem);
    const size_t spill_bytes = 0;
    (void)kp;
    int64_t nnz_h = 0;
    if (cudaMemcpyAsync(&nnz_h, A.indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_warp: indptr read failed");
    const size_t graph_bytes = pl.ch ? pl.bitset_bytes : (4 * (size_t)(n + 1) + 2 * (size_t)nnz_h + 256);
    uint8_t *ws = (uint8_t *)workspace2(spill_bytes + graph_bytes + 512);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol_warp: workspace allocation failed");
    WarpTabuParams P{};
    P.assigns = A.assigns;
    P.best_assigns = A.best_assigns;
    uint8_t *gbase = ws + ((spill_bytes + 255) & ~(size_t)255);
    if (pl.ch) {
        if (cudaMemsetAsync(gbase, 0, pl.bitset_bytes, st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "memset failed");
        tw_bitset_kernel<<<std::min(n, 4 * num_sms()), 128, 0, st>>>(A.indptr, A.indices, n, 4 * pl.ch,
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
    P.nwork = (int)A.p;
    P.work_counter = ctl32;
    P.ovf_list = ovf_list;
    P.ovf_count = ovf_count;
    P.err_flag = err_flag;
    P.flags = A.flags;
    P.warp_smem = (int)pl.warp_smem;
    P.bitset_bytes = (int)pl.bitset_bytes;
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] tabucol_warp<kv=%d,%s%d> grid=%d warps/CTA=%d smem=%zu\n", pl.kv,
                pl.ch ? "bitset ch=" : "csr", pl.ch, pl.grid, pl.warps, smem);
    kern<<<pl.grid, 32 * pl.warps, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol_warp launch failed");
    return MCB_OK;
}

}  // namespace mcb

namespace mcb {
int tabucol_warp_stats(unsigned long long *out) {
    if (cudaMemcpyFromSymbol(out, g_wstats, sizeof(unsigned long long) * 32) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "warp stats unavailable");
    return MCB_OK;
}
}  // namespace mcb
