// tabucol_group.cu -- batched TabuCol, one individual per GROUP of NW warps
// (sm_100a).  Same semantics, table format and bit-exact trajectories as
// tabucol_warp.cu / the reference `_tabucol_batch`
// (pkg/src/memcolor/localsearch.py:266-410).
//
// Why a group: measured on B200, one warp running one individual alone on an
// SM takes ~9.7k cycles per move and 8 warps per SM ~11.2k -- the warp kernel
// is a dependent chain (LDS / SHFL / VOTE steps of 25-45 cycles), not an issue
// or bandwidth limit.  Splitting every phase that has parallel work over NW
// warps shortens the chain:
//   * scan: one conflicting row per thread (TG = 32 NW rows per pass instead
//     of 64 per warp); row minimum and its tie count in the same pass; the
//     list-order prefix minimum = warp shuffle scans + the warp totals
//     exchanged through shared memory at one named barrier;
//   * reservoir events: tie rows contribute their counts, rows that lower the
//     running minimum are walked in-lane by their thread, all in parallel;
//   * the draws are evaluated redundantly by every warp (no barrier), the
//     winning row's thread locates the colour;
//   * neighbour update: warp w owns slots q in [w CH/NW, (w+1) CH/NW) of the
//     lane-interleaved bitset row (the moved vertex's own two bytes are
//     rewritten by the thread that owns its slot, so no write races);
//   * tabu ring: warp w holds the entries with insertion index = w mod NW,
//     each warp expires / supersedes its own entries in parallel;
//   * conflict-list events stay serial (one thread, list order), overlapping
//     the other warps' expiry.
// Named barriers (bar.sync 1 + group, 32 NW) separate the phases: B1 per
// scan round, B2 (event / tie-count totals), B4 (the move), B5 (update done;
// bar.red.or carries overflow flags), B6 (list done).
//
// Individuals whose tabu list outgrows the NW x 32 x KEW-entry ring, whose
// gamma exceeds 63 or whose tenure reaches 8190 stop and are appended to the
// overflow list, which the caller hands to the warp kernel's SPILL variant
// and then to the CTA kernel (tabucol.cu), each re-running from the start.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "common.cuh"
#include "launch.h"
#include "tw_helpers.cuh"

namespace mcb {

using namespace tw;

namespace {

struct GroupParams {
    int32_t *assigns;
    int32_t *best_assigns;
    const uint8_t *bitset;  // n rows of 4*CH bytes, lane-interleaved (tw_bitset_kernel)
    const int64_t *indptr;  // degrees for the counters
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
    const int32_t *work_list;
    const int32_t *nwork_dev;  // device-side count (overrides nwork when set)
    int32_t *work_counter;
    int32_t *ovf_list, *ovf_count, *err_flag;
    uint32_t flags;
    int group_smem;    // bytes per group region
    int xch_bytes;     // exchange words at the start of the region
    int bitset_bytes;  // CTA-shared copy of the bitset (0: rows from L2)
    int stats;         // MCB_GSTATS=1: thread 0's per-phase cycles into g_gstats
};

__device__ unsigned long long g_gstats[32];

__device__ ulonglong2 g_divtab_grp[32];
__device__ __forceinline__ bool divisible_g(uint64_t x, uint32_t s) {
    if (s < 64u) {
        const int t = __ffs(s) - 1;
        const uint32_t o = s >> t;
        const ulonglong2 e = __ldg(&g_divtab_grp[o >> 1]);
        return (x & ((1ull << t) - 1ull)) == 0ull && (x >> t) * e.x <= e.y;
    }
    return mod_is_zero(x, s);
}

// exchange-area word offsets
template <int NW, int CH>
struct XO {
    static constexpr int MIN = 0;           // [NW] warp prefix-min totals
    static constexpr int EVS = MIN + NW;    // [NW] warp event sums
    static constexpr int CDW = EVS + NW;    // [NW] warp D-candidate counts
    static constexpr int MV = CDW + NW;     // packed move
    static constexpr int QS = MV + 1;       // [NW] warp event slot masks
    static constexpr int EM = QS + NW;      // [CH][2] lane masks (any event, enter)
    static constexpr int C = EM + 2 * CH;   // conflict list length
    static constexpr int WI = C + 1;        // work item
    static constexpr int CONF = WI + 1;     // initial conflicts
    static constexpr int DIAG = CONF + 1;   // [NW] scratch-check partial sums
    static constexpr int WORDS = DIAG + NW;
};

__device__ __forceinline__ void gbar(int id, int nthr) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthr) : "memory");
}
// barrier with an OR over the group's predicates
__device__ __forceinline__ bool gbar_or(int id, int nthr, bool p) {
    int r;
    asm volatile(
        "{\n\t.reg .pred ip, op;\n\t"
        "setp.ne.u32 ip, %1, 0;\n\t"
        "bar.red.or.pred op, %2, %3, ip;\n\t"
        "selp.u32 %0, 1, 0, op;\n\t}"
        : "=r"(r)
        : "r"((int)p), "r"(id), "r"(nthr)
        : "memory");
    return r != 0;
}

}  // namespace

// ---------------------------------------------------------------------------
// Row summaries.  For every row in the conflict list the group keeps one word
//     gva (6) | rmin (6) << 6 | rcnt (7) << 12 | tmin (6) << 19 | tcnt (7) << 25
// gva = gamma at the own colour; rmin / rcnt = minimum and multiplicity of the
// non-tabu candidate colours; tmin / tcnt = the same over the tabu colours
// (63 = none; gamma is capped at 62 here, larger tables re-run elsewhere).
// The scan then reads one word per conflicting row instead of its KP bytes:
// with aspiration threshold A = gva + best - conflicts the row's minimum is
// m = min(rmin, tmin if tmin < A), its tie count the multiplicities at m --
// exactly row_min / row_count of tabucol_warp.cu.  Summaries are maintained
// by the warp that owns the row (the owner of its update slot): incrementally
// for conflicting neighbours of the moved vertex (column a -1, column b +1),
// by a warp-wide rescan for rows entering the list, the moved vertex, rows
// whose tabu entry expired and the rare increments that empty a minimum group.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t spack(int gva, int rmin, int rcnt, int tmin, int tcnt) {
    return (uint32_t)gva | ((uint32_t)rmin << 6) | ((uint32_t)rcnt << 12) | ((uint32_t)tmin << 19) |
           ((uint32_t)tcnt << 25);
}
template <int KW>
__device__ __forceinline__ uint32_t summary_inlane(const uint32_t (&x)[KW]) {
    const int gva = own_gamma<KW>(x);
    const int rmin = min(row_min<KW>(x, 0u), 63);
    const int tmin = min(row_min<KW>(x, TABU * 0x01010101u), 63);
    const int rcnt = rmin < 63 ? row_count<KW>(x, (uint32_t)rmin) : 0;
    const int tcnt = tmin < 63 ? row_count<KW>(x, (uint32_t)tmin | TABU) : 0;
    return spack(gva, rmin, rcnt, tmin, tcnt);
}
// the whole warp summarises one row: lane L < KW holds physical word L
template <int KW>
__device__ __forceinline__ uint32_t summary_warp(const uint8_t *row, int lane) {
    const uint32_t x = lane < KW ? reinterpret_cast<const uint32_t *>(row)[lane] : 0x7F7F7F7Fu;
    uint32_t og = x & (((x & 0x80808080u) >> 7) * GM);
    og |= og >> 16;
    og |= og >> 8;
    const uint32_t m2 = __vminu2(x & 0x00FF00FFu, __byte_perm(x, 0, 0x4341));
    const uint32_t xt = x ^ 0x40404040u;
    const uint32_t t2 = __vminu2(xt & 0x00FF00FFu, __byte_perm(xt, 0, 0x4341));
    const int gva = (int)__reduce_or_sync(FULLM, og & GM);
    const int rmin = min((int)__reduce_min_sync(FULLM, min(m2 & 0xFFFFu, m2 >> 16)), 63);
    const int tmin = min((int)__reduce_min_sync(FULLM, min(t2 & 0xFFFFu, t2 >> 16)), 63);
    const int rc = rmin < 63 ? count_eq(x, (uint32_t)rmin * 0x01010101u) : 0;
    const int tc = tmin < 63 ? count_eq(x, ((uint32_t)tmin | TABU) * 0x01010101u) : 0;
    const int rcnt = (int)__reduce_add_sync(FULLM, rc);
    const int tcnt = (int)__reduce_add_sync(FULLM, tc);
    return spack(gva, rmin, rcnt, tmin, tcnt);
}
// incremental update of a conflicting neighbour's summary for the move's
// column a (gamma - 1) and column b (gamma + 1); pa / pb are the old bytes.
// `dirty`: column b emptied a minimum group (the new minimum's multiplicity
// is unknown) -- the row needs a rescan.
__device__ __forceinline__ uint32_t summary_move(uint32_t s, uint32_t pa, uint32_t pb, bool &dirty) {
    int gva = s & 63, rmin = (s >> 6) & 63, rcnt = (s >> 12) & 127, tmin = (s >> 19) & 63, tcnt = s >> 25;
    if (pa & OWN) {
        gva--;
    } else {
        const int x = (int)(pa & GM) - 1;
        if (pa & TABU) {
            if (x < tmin) {
                tmin = x;
                tcnt = 1;
            } else if (x == tmin) {
                tcnt++;
            }
        } else {
            if (x < rmin) {
                rmin = x;
                rcnt = 1;
            } else if (x == rmin) {
                rcnt++;
            }
        }
    }
    if (pb & OWN) {
        gva++;
    } else {
        const int x = (int)(pb & GM);
        if (pb & TABU) {
            if (x == tmin && --tcnt == 0) dirty = true;
        } else {
            if (x == rmin && --rcnt == 0) dirty = true;
        }
    }
    return spack(gva, rmin, rcnt, tmin, tcnt);
}
// a conflicting row's scan values from its summary: rm = minimum delta
// (TW_BIG: no admissible move), cnt = candidates at the minimum
__device__ __forceinline__ void summary_eval(uint32_t s, int thr, int &gva, int &rm, int &cnt) {
    gva = s & 63;
    const int rmin = (s >> 6) & 63, rcnt = (s >> 12) & 127, tmin = (s >> 19) & 63, tcnt = s >> 25;
    const bool asp = tmin < gva + thr;  // tabu colours admissible below A (aspiration)
    const int m = asp ? min(rmin, tmin) : rmin;
    cnt = (rmin == m ? rcnt : 0) + (asp && tmin == m ? tcnt : 0);
    rm = m < 63 ? m - gva : TW_BIG;
}

// ---------------------------------------------------------------------------
//   KV  16-byte vectors per gamma row (KP = 16 KV >= k)
//   CH  bitset chunk bits per lane (n <= 32 CH)
//   NW  warps per individual (1, 2 or 4)
// ---------------------------------------------------------------------------
template <int KV, int CH, int NW>
__global__ void __launch_bounds__(256 * NW, 1) tabucol_group_kernel(GroupParams P) {
    constexpr int KP = 16 * KV, KW = 4 * KV, TG = 32 * NW, QW = CH / NW;
    constexpr int KEW = KE / NW;  // ring registers per lane per warp
    constexpr int QS = 32 * KP;   // byte distance between slots q and q + 1
    constexpr int SW = KW <= 4 ? 4 : KW <= 8 ? 8 : KW <= 16 ? 16 : 32;  // walk segment width
    constexpr int NQ = QW / 4;    // packed 4-slot words per thread
    constexpr int CM = 4;         // conflicting rows per thread kept in registers
    static_assert(KW <= 32 && CH % NW == 0 && QW % 4 == 0 && KEW >= 1 && NQ <= 8, "shape");
    using S = Swz<KW>;
    using CT = typename ChunkT<CH>::T;
    using X = XO<NW, CH>;

    extern __shared__ __align__(16) uint8_t smem[];
    const int grp = threadIdx.x / TG, t = threadIdx.x % TG, w = t >> 5, lane = t & 31;
    const int bid = 1 + grp;
    const int n = P.n, k = P.k;
    const unsigned lt_mask = (1u << lane) - 1u;
    auto sync = [&]() {
        if constexpr (NW == 1) __syncwarp();
        else gbar(bid, TG);
    };
    auto sync_or = [&](bool p) -> bool {
        if constexpr (NW == 1) {
            __syncwarp();
            return __any_sync(FULLM, p);
        }
        else return gbar_or(bid, TG, p);
    };

    const uint8_t *brows = P.bitset_bytes ? smem : P.bitset;
    if (P.bitset_bytes) {
        const uint4 *src = reinterpret_cast<const uint4 *>(P.bitset);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < P.bitset_bytes / 16; i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    uint8_t *region = smem + P.bitset_bytes + (size_t)grp * P.group_smem;
    int32_t *xch = reinterpret_cast<int32_t *>(region);
    // exchange words | summaries | gamma rows | list, positions | colours.  The
    // update's unrolled window (rows lane + 32 q < 32 CH, rows >= n written back
    // unchanged) may reach past the gamma rows into the list and colours, which
    // nothing writes during the update -- never into the summaries
    uint32_t *summ = reinterpret_cast<uint32_t *>(region + P.xch_bytes);
    uint8_t *gam = region + P.xch_bytes + ((4 * (size_t)n + 15) & ~(size_t)15);
    size_t off = (size_t)n * KP;
    uint16_t *clist = reinterpret_cast<uint16_t *>(gam + off);
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint16_t *cpos = reinterpret_cast<uint16_t *>(gam + off);
    off += (2 * (size_t)n + 15) & ~(size_t)15;
    uint8_t *asg = gam + off;

    const bool prod = (P.flags & MCB_FLAG_PRODUCTION) != 0;
    const bool diagf = (P.flags & MCB_FLAG_DIAG) != 0;
    const bool cnt_on = P.counters != nullptr;
    const int g_lane = S::g(lane);
    const int nwork = P.nwork_dev ? *P.nwork_dev : P.nwork;
    const bool stats = P.stats && t == 0;
    long long st[16];
#pragma unroll
    for (int i = 0; i < 16; i++) st[i] = 0;
    long long ph_t = 0;
#define GPH(i)                          \
    if (stats) {                        \
        const long long _t = clock64(); \
        st[i] += _t - ph_t;             \
        ph_t = _t;                      \
    }
    // rows this thread owns in the update: u = lane + 32 (w QW + j), j < QW
    const int qbase = w * QW;

    for (;;) {
        if (t == 0) xch[X::WI] = atomicAdd(P.work_counter, 1);
        sync();
        const int wi = xch[X::WI];
        if (wi >= nwork) break;
        const int ind = P.work_list ? P.work_list[wi] : wi;
        const uint64_t key = P.keys[ind];
        int32_t *a_io = P.assigns + (size_t)ind * n;
        int32_t *b_out = P.best_assigns + (size_t)ind * n;

        // ---------------- init (localsearch.py:289-318) ----------------
        bool bad = false, rangeerr = false;
        for (int v = t; v < n; v += TG) {
            int c = a_io[v];
            if (c < 0 || c >= k) {
                rangeerr = true;
                c = 0;
            }
            asg[v] = (uint8_t)c;
            b_out[v] = c;
        }
        {
            uint32_t *g32 = reinterpret_cast<uint32_t *>(gam);
            const uint32_t padw = (k & 3) ? (0x7F7F7F7Fu << (8 * (k & 3))) : 0u;
            for (int i = t; i < n * KW; i += TG) {
                const int u = i / KW, p = i - u * KW;
                int wd = p - S::g(u);
                if (wd < 0) wd += KW;
                g32[i] = (4 * wd + 4 <= k) ? 0u : (4 * wd >= k ? 0x7F7F7F7Fu : padw);
            }
        }
        sync();
        // gamma counts (own colour marked), then the row summaries
        for (int u = t; u < n; u += TG) {
            uint8_t *row = gam + (size_t)u * KP;
            const int gu = S::g(u);
            const CT *br = reinterpret_cast<const CT *>(brows + (size_t)u * 4 * CH);
            for (int L = 0; L < 32; L++) {
                uint32_t ch = br[L];
                while (ch) {
                    const int q = __ffs(ch) - 1;
                    ch &= ch - 1;
                    const int c = asg[L + 32 * q];
                    uint8_t *e = row + S::phys(c, gu);
                    const int x = *e + 1;
                    if (x > (int)GM - 1) bad = true;
                    else *e = (uint8_t)x;
                }
            }
            row[S::phys(asg[u], gu)] |= (uint8_t)OWN;
            uint32_t x[KW];
            load_row<KV>(row, x);
            summ[u] = summary_inlane<KW>(x);
        }
        sync();
        if (w == 0) {
            // conflict list in ascending vertex order (:303-310)
            long long c2 = 0;
            int C0 = 0;
            for (int v0 = 0; v0 < n; v0 += 32) {
                const int v = v0 + lane;
                int g = 0;
                if (v < n) g = summ[v] & 63;
                const bool f = g > 0;
                c2 += g;
                const unsigned bal = __ballot_sync(FULLM, f);
                if (f) {
                    const int pos = C0 + __popc(bal & lt_mask);
                    clist[pos] = (uint16_t)v;
                    cpos[v] = (uint16_t)pos;
                }
                C0 += __popc(bal);
            }
            c2 = warp_sum64(c2);
            if (lane == 0) {
                xch[X::C] = C0;
                xch[X::CONF] = (int)(c2 / 2);
            }
        }
        if (rangeerr) atomicExch(P.err_flag, 1);
        bad = sync_or(bad);
        int C = xch[X::C];
        long long conflicts = xch[X::CONF], best = conflicts;
        // conflicting rows among this thread's update slots
        uint32_t cmask = 0;
#pragma unroll
        for (int j = 0; j < QW; j++) {
            const int u = lane + 32 * (qbase + j);
            if (u < n && (summ[u] & 63) != 0) cmask |= 1u << j;
        }

        long long it = 0, nlog = 0, sum_c = 0, sum_deg = 0, diag = 0;
        unsigned long long ctr = 0;
        // tabu ring of the entries of this warp's rows: register row 0 =
        // newest 32 (lane = insertion % 32), rows shift once per 32 insertions
        uint32_t ring[KEW];
#pragma unroll
        for (int j = 0; j < KEW; j++) ring[j] = 0u;
        int nrows = 0;
        uint32_t ins = 0, next_exp = 0;

        // rescans of this warp's rows listed in `pend` (bit j = slot j of lane)
        auto rescan_pending = [&](uint32_t pend) {
            __syncwarp();
            for (;;) {
                const unsigned bal = __ballot_sync(FULLM, pend != 0u);
                if (!bal) break;
                const int src = __ffs(bal) - 1;
                const int j = __shfl_sync(FULLM, __ffs(pend) - 1, src);
                const int u = src + 32 * (qbase + j);
                const uint32_t sm = summary_warp<KW>(gam + (size_t)u * KP, lane);
                if (lane == 0) summ[u] = sm;
                if (lane == src) pend &= pend - 1;
            }
        };
        // events of one row that lowers the running minimum (entering minimum
        // P, delta space), one pass over up to 32/SW such rows of this warp
        auto walk_pass = [&](unsigned low, int v, int gv, int Pin, int thr) -> int {
            const int g = lane / SW, wl = lane % SW;
            unsigned tmp = low;
#pragma unroll
            for (int q = 0; q < 32 / SW - 1; q++)
                if (q < g) tmp &= tmp - 1;
            const int src = tmp ? __ffs(tmp) - 1 : -1;
            const int s0 = max(src, 0);
            const int wv = __shfl_sync(FULLM, v, s0);
            const int wg = __shfl_sync(FULLM, gv, s0);
            const int wp = __shfl_sync(FULLM, Pin, s0);
            uint32_t y = 0xFFFFFFFFu;
            if (src >= 0 && wl < KW)
                y = cand_word(reinterpret_cast<const uint32_t *>(gam + (size_t)wv * KP)[S::pw(wl, S::g(wv))], wg + thr);
            const uint32_t m2 = __vminu2(y & 0x00FF00FFu, __byte_perm(y, 0, 0x4341));
            const int um = (int)min(m2 & 0xFFFFu, m2 >> 16);
            const int ex = seg_excl_min<SW>(um, wl);
            const int c0 = min(min(wp >= TW_BIG ? INT_MAX : wp + wg, ex), 0xFE);
            const int c1 = min(c0, (int)(y & 0xFFu));
            const int c2 = min(c1, (int)__byte_perm(y, 0, 0x4441));
            const int c3 = min(c2, (int)__byte_perm(y, 0, 0x4442));
            const uint32_t Cp = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
            const unsigned segm = (SW == 32 ? 0xffffffffu : ((1u << SW) - 1u)) << (lane & ~(SW - 1));
            const int tv = masked_sum_small<3>(count_eq(y, Cp), segm);
            return (wl == 0 && src >= 0) ? tv : 0;
        };

        // ---------------- iterations (:320-405) ----------------
        if (k >= 2 && !bad) {
            for (long long step = 0; step < P.depth; step++) {
                if (conflicts == 0) break;
                const uint32_t it32 = (uint32_t)it;
                const int thr = (int)max(best - conflicts, (long long)-TW_BIG);
                if (stats) {
                    ph_t = clock64();
                    st[15] += 1;
                }
                // ---- scan (localsearch.py:328-350).  Thread t owns the list
                // positions [t c, t c + c): minimum over its rows, then the
                // list-order prefix minimum (warp scan + warp totals)
                const int c = (C + TG - 1) / TG;
                const int lo = t * c, hi = min(lo + c, C);
                int rv[CM], rg[CM], rr[CM], rn[CM];  // this thread's rows when c <= CM
                int mch = TW_BIG;
                if (c <= CM) {
#pragma unroll
                    for (int i = 0; i < CM; i++) {
                        rv[i] = (i < c && lo + i < C) ? clist[lo + i] : -1;
                        rr[i] = TW_BIG;
                        rn[i] = 0;
                        rg[i] = 0;
                    }
#pragma unroll
                    for (int i = 0; i < CM; i++)
                        if (rv[i] >= 0) {
                            summary_eval(summ[rv[i]], thr, rg[i], rr[i], rn[i]);
                            mch = min(mch, rr[i]);
                        }
                } else {
                    for (int li = lo; li < hi; li++) {
                        int gv, rm, cn;
                        summary_eval(summ[clist[li]], thr, gv, rm, cn);
                        mch = min(mch, rm);
                    }
                }
                GPH(0);
                int incl = mch;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int tv = __shfl_up_sync(FULLM, incl, o);
                    if (lane >= o) incl = min(incl, tv);
                }
                int ex = __shfl_up_sync(FULLM, incl, 1);
                if (lane == 0) ex = TW_BIG;
                int D = incl, Pin = ex;
                if constexpr (NW > 1) {
                    if (lane == 31) xch[X::MIN + w] = incl;
                    gbar(bid, TG);  // B1
                    int cw = TW_BIG;
                    D = TW_BIG;
#pragma unroll
                    for (int w2 = 0; w2 < NW; w2++) {
                        const int tv = xch[X::MIN + w2];
                        if (w2 < w) cw = min(cw, tv);
                        D = min(D, tv);
                    }
                    Pin = min(cw, ex);
                } else {
                    D = __shfl_sync(FULLM, incl, 31);
                }
                GPH(1);
                if (cnt_on && t == 0) sum_c += C;

                int mv_v = -1, mv_a = 0, mv_b = 0, Dg = 0;
                uint32_t e_new = 0;
                if (D < TW_BIG) {
                    // ---- tie events (rows at the running minimum: their
                    // multiplicity; rows lowering it: walked) and D-counts
                    int ev = 0, cd = 0;
                    // up to two rows per thread that lower the running minimum are
                    // walked by lane groups (walk_pass); more (rare) in-lane
                    int nl = 0, lv0 = 0, lg0 = 0, lp0 = 0, lv1 = 0, lg1 = 0, lp1 = 0;
                    auto row_events = [&](int v, int gv, int rm, int cn, int &Pr) {
                        if (rm >= TW_BIG) return;
                        if (!prod) {
                            if (rm == Pr) {
                                ev += cn;
                            } else if (rm < Pr) {
                                if (nl == 0) {
                                    lv0 = v;
                                    lg0 = gv;
                                    lp0 = Pr;
                                } else if (nl == 1) {
                                    lv1 = v;
                                    lg1 = gv;
                                    lp1 = Pr;
                                } else {
                                    uint32_t wl[KW];
                                    const uint32_t *r32 = reinterpret_cast<const uint32_t *>(gam + (size_t)v * KP);
#pragma unroll
                                    for (int i = 0; i < KW; i++) wl[i] = r32[S::pw(i, S::g(v))];
                                    ev += walk_words<KW>(wl, gv + thr, Pr >= TW_BIG ? 0xFE : Pr + gv);
                                }
                                nl++;
                            }
                        }
                        Pr = min(Pr, rm);
                        if (rm == D) cd += cn;
                    };
                    {
                        int Pr = Pin;
                        if (c <= CM) {
#pragma unroll
                            for (int i = 0; i < CM; i++)
                                if (rv[i] >= 0) row_events(rv[i], rg[i], rr[i], rn[i], Pr);
                        } else {
                            for (int li = lo; li < hi; li++) {
                                const int v = clist[li];
                                int gv, rm, cn;
                                summary_eval(summ[v], thr, gv, rm, cn);
                                row_events(v, gv, rm, cn, Pr);
                            }
                        }
                    }
                    if (!prod) {
                        unsigned low = __ballot_sync(FULLM, nl > 0);
                        while (low) {
                            ev += walk_pass(low, lv0, lg0, lp0, thr);
#pragma unroll
                            for (int q = 0; q < 32 / SW; q++) low &= low - 1;
                        }
                        low = __ballot_sync(FULLM, nl > 1);
                        while (low) {
                            ev += walk_pass(low, lv1, lg1, lp1, thr);
#pragma unroll
                            for (int q = 0; q < 32 / SW; q++) low &= low - 1;
                        }
                    }
                    GPH(2);
                    // exclusive prefix of the D-counts over the list order
                    int cx;
                    if (c == 1) {  // cd <= 127
                        cx = excl_sum_small<7>(cd, lt_mask);
                    } else {
                        int ic = cd;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int tv = __shfl_up_sync(FULLM, ic, o);
                            if (lane >= o) ic += tv;
                        }
                        cx = ic - cd;
                    }
                    const int evw = prod ? 0 : __reduce_add_sync(FULLM, ev);
                    const int cdw = __reduce_add_sync(FULLM, cd);
                    int tot = evw, T = cdw, cdb = 0;  // cdb: D-candidates in warps before this one
                    if constexpr (NW > 1) {
                        if (lane == 0) {
                            xch[X::EVS + w] = evw;
                            xch[X::CDW + w] = cdw;
                        }
                        gbar(bid, TG);  // B2
                        tot = 0;
                        T = 0;
                        int ev_[NW], cd_[NW];
#pragma unroll
                        for (int w2 = 0; w2 < NW; w2++) {
                            ev_[w2] = xch[X::EVS + w2];
                            cd_[w2] = xch[X::CDW + w2];
                        }
#pragma unroll
                        for (int w2 = 0; w2 < NW; w2++) {
                            tot += ev_[w2];
                            if (w2 < w) cdb += cd_[w2];
                            T += cd_[w2];
                        }
                    }
                    GPH(3);
                    // tenure draw (:363-365)
                    uint32_t ll;
                    if (!prod) ll = u64_below32(key, ctr + (unsigned long long)tot, 10u);
                    else ll = philox_below(key, ctr + 1, 10u);
                    // ---- reservoir: the T-1 draws of the final group (every warp)
                    int sstar = 1;
                    if (T > 1) {
                        if (!prod) {
                            const unsigned long long c0 = ctr + (unsigned long long)(tot - (T - 1));
                            int smax = 1;
                            for (int s2 = 2 + lane; s2 <= T; s2 += 32)
                                if (divisible_g(stream_value(key, c0 + (unsigned long long)(s2 - 2)), (uint32_t)s2))
                                    smax = s2;
                            sstar = __reduce_max_sync(FULLM, smax);
                        } else {
                            sstar = 1 + (int)philox_below(key, ctr, (uint32_t)T);
                        }
                    }
                    GPH(4);
                    // ---- the owner of the sstar-th D-candidate (list order):
                    // its row, then the colour with the warp's lanes
                    const int need0 = sstar - cdb;
                    if (need0 >= 1 && need0 <= cdw) {
                        const unsigned bm = __ballot_sync(FULLM, cd > 0 && cx < need0 && need0 <= cx + cd);
                        const int src = __ffs(bm) - 1;
                        int vs = 0, gs = 0, need = need0 - cx;
                        if (lane == src) {
                            // the row inside this thread's chunk
                            int acc = 0;
                            bool found = false;
                            if (c <= CM) {
#pragma unroll
                                for (int i = 0; i < CM; i++)
                                    if (!found && rv[i] >= 0 && rr[i] == D) {
                                        if (acc + rn[i] >= need) {
                                            vs = rv[i];
                                            gs = rg[i];
                                            need -= acc;
                                            found = true;
                                        }
                                        acc += rn[i];
                                    }
                            } else {
                                for (int li = lo; li < hi && !found; li++) {
                                    const int v = clist[li];
                                    int gv, rm, cn;
                                    summary_eval(summ[v], thr, gv, rm, cn);
                                    if (rm == D) {
                                        if (acc + cn >= need) {
                                            vs = v;
                                            gs = gv;
                                            need -= acc;
                                            found = true;
                                        }
                                        acc += cn;
                                    }
                                }
                            }
                        }
                        vs = __shfl_sync(FULLM, vs, src);
                        gs = __shfl_sync(FULLM, gs, src);
                        need = __shfl_sync(FULLM, need, src);
                        const int A = gs + thr, dg = D + gs;
                        const uint32_t DM = (uint32_t)dg * 0x01010101u;
                        uint32_t cw = 0xFFFFFFFFu;
                        int cc = 0;
                        if (lane < KW) {
                            cw = cand_word(reinterpret_cast<const uint32_t *>(gam + (size_t)vs * KP)[S::pw(lane, S::g(vs))], A);
                            cc = count_eq(cw, DM);
                        }
                        const int ic = excl_sum_small<3>(cc, lt_mask) + cc;
                        const unsigned bw = __ballot_sync(FULLM, ic >= need);
                        const int sl = bw ? __ffs(bw) - 1 : 0;
                        if (lane == sl) {
                            int b = -1;
                            if (bw) {
                                uint32_t z = zero_flags(cw ^ DM);
                                for (int r2 = need - (ic - cc); r2 > 1; r2--) z &= z - 1;
                                b = 4 * lane + ((__ffs(z) - 1) >> 3);
                            }
                            const int a = asg[vs];
                            const uint32_t ba = gam[(size_t)vs * KP + S::phys(a, S::g(vs))];
                            // b < 0 cannot happen; it routes the individual to the fallback
                            const int mv = b < 0 ? -1
                                                 : (vs | (a << 10) | (b << 17) | ((ba & TABU) ? (1 << 24) : 0) |
                                                    (dg << 25));
                            if constexpr (NW > 1) xch[X::MV] = mv;
                            else mv_v = mv;
                        }
                        if constexpr (NW == 1) mv_v = __shfl_sync(FULLM, mv_v, sl);
                    }
                    GPH(5);
                    int mv = mv_v;
                    if constexpr (NW > 1) {
                        gbar(bid, TG);  // B4
                        mv = xch[X::MV];
                    }
                    GPH(6);
                    if (mv < 0) {
                        bad = true;
                        break;
                    }
                    mv_v = mv & 0x3FF;
                    mv_a = (mv >> 10) & 0x7F;
                    mv_b = (mv >> 17) & 0x7F;
                    const bool sup = (mv >> 24) & 1;
                    Dg = (mv >> 25) & 0x3F;
                    // ---- move, tenure, tabu entry (:352-366)
                    conflicts += D;
                    ctr += prod ? 2ull : (unsigned long long)tot + 1ull;
                    const long long tt = (long long)ll + (6LL * conflicts) / 10LL;
                    if (tt >= 8190) {
                        bad = true;
                        break;
                    }
                    e_new = it32 + (uint32_t)tt + 1u;
                    if (t == 0) {
                        if (nlog < P.log_cap) {
                            const size_t o = (size_t)ind * P.log_cap + nlog;
                            P.log_v[o] = mv_v;
                            P.log_iter[o] = it;
                            P.log_tt[o] = tt;
                        }
                        if (cnt_on) sum_deg += P.indptr[mv_v + 1] - P.indptr[mv_v];
                    }
                    if (nlog < P.log_cap) nlog++;
                    if (sup && w == ((mv_v >> 5) / QW)) {
                        // (v, a) re-tabu'd while tabu: the older entry is void (:366)
                        const uint32_t key_vc = ent_pack(mv_v, mv_a, 0) & 0xFFFFC000u;
#pragma unroll
                        for (int j = 0; j < KEW; j++) {
                            if (j >= nrows) break;
                            const bool hit = (ring[j] & 0xFFFFC000u) == key_vc;
                            if (hit) ring[j] = 0u;
                            if (__any_sync(FULLM, hit)) break;
                        }
                    }
                }
                GPH(7);

                bool flag = false;
                if (mv_v >= 0) {
                    const int v = mv_v, a = mv_a, b = mv_b;
                    const CT *brp = reinterpret_cast<const CT *>(brows + (size_t)v * 4 * CH) + lane;
                    const uint32_t chv = P.bitset_bytes ? (uint32_t)*brp : (uint32_t)__ldg(brp);
                    const bool vwarp = w == ((v >> 5) / QW);
                    // ring insert: the warp owning row v
                    if (vwarp) {
                        const int L = (int)(ins & 31u);
                        if (L == 0 && ins != 0u) {
                            if (__any_sync(FULLM, (ring[KEW - 1] >> 31) != 0u)) flag = true;  // ring full
#pragma unroll
                            for (int j = KEW - 1; j > 0; j--) ring[j] = ring[j - 1];
                            ring[0] = 0u;
                            nrows = min(nrows + 1, KEW);
                        }
                        if (lane == L) ring[0] = ent_pack(v, a, e_new);
                        if (nrows == 0 || (int)(e_new - next_exp) < 0) next_exp = e_new;
                        nrows = max(nrows, 1);
                        ins++;
                    }
                    // ---- gamma update over N(v) (:356-359); the slot holding v
                    // itself gets the move's own bytes: a -> gamma | TABU, b -> | OWN
                    const uint32_t ch = (chv >> qbase) & ((QW == 32) ? 0xFFFFFFFFu : ((1u << QW) - 1u));
                    const int vq = (v >> 5) - qbase;
                    const bool vmine = (v & 31) == lane && vq >= 0 && vq < QW;
                    const uint32_t ra = smem_addr(gam) + (uint32_t)(lane * KP + S::phys(a, g_lane) + qbase * QS);
                    const uint32_t rb = smem_addr(gam) + (uint32_t)(lane * KP + S::phys(b, g_lane) + qbase * QS);
                    uint32_t oa[QW], ob[QW];
                    static_for<QW>([&](auto qc) {
                        constexpr int q = decltype(qc)::value;
                        oa[q] = lds8<q * QS>(ra);
                        ob[q] = lds8<q * QS>(rb);
                    });
                    uint32_t evE = 0, evL = 0, ovm = 0;
                    uint32_t pa4w[NQ], pb4w[NQ];
                    static_for<NQ>([&](auto gc) {
                        constexpr int gi = decltype(gc)::value, g0 = 4 * gi;
                        const uint32_t nbm = (((ch >> g0) & 0xFu) * 0x00204081u) & 0x01010101u;
                        const uint32_t pa4 = __byte_perm(__byte_perm(oa[g0], oa[g0 + 1], 0x0040),
                                                         __byte_perm(oa[g0 + 2], oa[g0 + 3], 0x0040), 0x5410);
                        const uint32_t pb4 = __byte_perm(__byte_perm(ob[g0], ob[g0 + 1], 0x0040),
                                                         __byte_perm(ob[g0 + 2], ob[g0 + 3], 0x0040), 0x5410);
                        pa4w[gi] = pa4;
                        pb4w[gi] = pb4;
                        uint32_t na4 = pa4 - nbm, nb4 = pb4 + nbm;
                        const uint32_t vmb = (vmine && vq >= g0 && vq < g0 + 4) ? (0xFFu << (8 * (vq - g0))) : 0u;
                        na4 = (na4 & ~vmb) | (((pa4 & 0x3F3F3F3Fu) | 0x40404040u) & vmb);
                        nb4 |= 0x80808080u & vmb;
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
                        // cap: gamma reaches 63
                        const uint32_t zl = zero_flags((na4 & 0xBFBFBFBFu) ^ 0x80808080u) & nbh;
                        const uint32_t ze = zero_flags((nb4 & 0xBFBFBFBFu) ^ 0x81818181u) & nbh;
                        ovm |= zero_flags((nb4 & 0x3F3F3F3Fu) ^ 0x3F3F3F3Fu) & nbh;
                        evL |= ((((zl >> 7) * 0x00204081u) >> 21) & 0xFu) << g0;
                        evE |= ((((ze >> 7) * 0x00204081u) >> 21) & 0xFu) << g0;
                    });
                    flag |= ovm != 0u;
                    // summaries of the conflicting neighbours that stay conflicting
                    uint32_t pend = evE;
                    for (uint32_t upd = ch & cmask & ~evL; upd;) {
                        const int j = __ffs(upd) - 1;
                        upd &= upd - 1;
                        uint32_t pa4 = pa4w[0], pb4 = pb4w[0];
#pragma unroll
                        for (int gi = 1; gi < NQ; gi++)
                            if ((j >> 2) == gi) {
                                pa4 = pa4w[gi];
                                pb4 = pb4w[gi];
                            }
                        const int sh = 8 * (j & 3);
                        const int u = lane + 32 * (qbase + j);
                        bool dirty = false;
                        const uint32_t sm = summary_move(summ[u], (pa4 >> sh) & 0xFFu, (pb4 >> sh) & 0xFFu, dirty);
                        if (dirty) pend |= 1u << j;
                        else summ[u] = sm;
                    }
                    cmask = (cmask | evE) & ~evL;
                    if (vmine && Dg == 0) cmask &= ~(1u << vq);
                    rescan_pending(pend);
                    // this warp's conflict-list events, slot-major (q), lane-minor
                    const uint32_t em = __reduce_or_sync(FULLM, evE | evL);
                    if constexpr (NW > 1) {
                        if (lane == 0) xch[X::QS + w] = (int)em;
                    }
                    for (uint32_t e2 = em; e2;) {
                        const int j = __ffs(e2) - 1;
                        e2 &= e2 - 1;
                        const unsigned lm = __ballot_sync(FULLM, ((evE | evL) >> j) & 1u);
                        const unsigned lE = __ballot_sync(FULLM, (evE >> j) & 1u);
                        if (lane == 0) {
                            xch[X::EM + 2 * (qbase + j)] = (int)lm;
                            xch[X::EM + 2 * (qbase + j) + 1] = (int)lE;
                        }
                    }
                    if constexpr (NW == 1) {
                        if (lane == 0) xch[X::QS] = (int)em;
                    }
                }
                GPH(8);
                if (mv_v >= 0) {
                    if (sync_or(flag)) {  // B5: gamma reached 63 or ring full
                        bad = true;
                        break;
                    }
                    // ---- conflict-list events in ascending vertex order, then v
                    // (:368-385), one thread; asg[v] = b
                    if (t == TG - 32) {
                        int Cn = C;
#pragma unroll 1
                        for (int w2 = 0; w2 < NW; w2++) {
                            uint32_t em = (uint32_t)xch[X::QS + w2];
                            while (em) {
                                const int j = __ffs(em) - 1;
                                em &= em - 1;
                                const int q = w2 * QW + j;
                                uint32_t lm = (uint32_t)xch[X::EM + 2 * q];
                                const uint32_t lE = (uint32_t)xch[X::EM + 2 * q + 1];
                                while (lm) {
                                    const int L = __ffs(lm) - 1;
                                    lm &= lm - 1;
                                    const int u = L + 32 * q;
                                    if ((lE >> L) & 1u) {
                                        clist[Cn] = (uint16_t)u;
                                        cpos[u] = (uint16_t)Cn;
                                        Cn++;
                                    } else {
                                        const int pos = cpos[u], last = clist[Cn - 1];
                                        clist[pos] = (uint16_t)last;
                                        cpos[last] = (uint16_t)pos;
                                        Cn--;
                                    }
                                }
                            }
                        }
                        if (Dg == 0) {
                            const int pos = cpos[mv_v], last = clist[Cn - 1];
                            clist[pos] = (uint16_t)last;
                            cpos[last] = (uint16_t)pos;
                            Cn--;
                        }
                        asg[mv_v] = (uint8_t)mv_b;
                        xch[X::C] = Cn;
                    }
                }
                GPH(9);
                // ---- tabu expiry for iteration it + 1 (this warp's rows), then the
                // summaries of the expired rows and of the moved vertex
                {
                    const uint32_t itn = it32 + 1u;
                    uint32_t pend_u = 0xFFFFFFFFu;  // this lane's expired row (one per lane and ring row)
                    int nexp = 0;
                    if (nrows > 0 && (int)(next_exp - itn) <= 0) {
                        int last = -1;
                        uint32_t dmin = 0x4000u;
#pragma unroll
                        for (int j = 0; j < KEW; j++) {
                            if (j >= nrows) break;
                            const uint32_t e = ring[j];
                            const uint32_t dist = ent_dist(e, itn);
                            const bool hit = (e >> 31) != 0u && dist == 0u;
                            if (hit) {
                                const int vv = (e >> 21) & 0x3FF, cc = (e >> 14) & 0x7F;
                                gam[(size_t)vv * KP + S::phys(cc, S::g(vv))] &= (uint8_t)~TABU;
                                if (pend_u == 0xFFFFFFFFu) pend_u = (uint32_t)vv;
                                else nexp = 1;  // a second expiry in this lane (rare)
                            }
                            ring[j] = hit ? 0u : e;
                            const bool live = (ring[j] >> 31) != 0u;
                            if (live) dmin = min(dmin, dist);
                            if (__any_sync(FULLM, live)) last = j;
                        }
                        nrows = last + 1;
                        next_exp = itn + __reduce_min_sync(FULLM, dmin);
                        __syncwarp();
                        if (__any_sync(FULLM, nexp != 0)) {
                            // several expiries in one lane: rescan every live list row of the warp's entries
                            // by walking the ring once more is not possible (entries are gone), so rescan
                            // all rows this warp owns that are in the list
                            uint32_t all = cmask;
                            rescan_pending(all);
                            pend_u = 0xFFFFFFFFu;
                        }
                        for (;;) {
                            const unsigned bal = __ballot_sync(FULLM, pend_u != 0xFFFFFFFFu);
                            if (!bal) break;
                            const int src = __ffs(bal) - 1;
                            const int u = __shfl_sync(FULLM, (int)pend_u, src);
                            const uint32_t sm = summary_warp<KW>(gam + (size_t)u * KP, lane);
                            if (lane == 0) summ[u] = sm;
                            if (lane == src) pend_u = 0xFFFFFFFFu;
                        }
                    }
                    if (mv_v >= 0 && Dg > 0 && w == ((mv_v >> 5) / QW)) {
                        __syncwarp();
                        const uint32_t sm = summary_warp<KW>(gam + (size_t)mv_v * KP, lane);
                        if (lane == 0) summ[mv_v] = sm;
                    }
                }
                GPH(10);
                sync();  // B6
                GPH(11);
                if (mv_v >= 0) {
                    C = xch[X::C];
                    // ---- best (:387-390)
                    if (conflicts < best) {
                        best = conflicts;
                        const bool al16 = ((reinterpret_cast<uintptr_t>(b_out) & 15u) == 0);
                        for (int q = t; 4 * q < n; q += TG) {
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
                it++;
                GPH(12);
                // ---- scratch check every 1024 iterations (:398-405)
                if (diagf && (it & 1023) == 0) {
                    long long c2 = 0;
                    for (int64_t e = t; e < P.m; e += TG) c2 += asg[__ldg(P.eu + e)] == asg[__ldg(P.ev + e)];
                    c2 = warp_sum64(c2);
                    long long cs = c2;
                    if constexpr (NW > 1) {
                        if (lane == 0) xch[X::DIAG + w] = (int)c2;
                        gbar(bid, TG);
                        cs = 0;
#pragma unroll
                        for (int w2 = 0; w2 < NW; w2++) cs += xch[X::DIAG + w2];
                        gbar(bid, TG);
                    }
                    if (cs != conflicts) diag++;
                }
            }
        }
        sync();
        if (stats) {
            for (int i = 0; i < 16; i++)
                if (st[i]) atomicAdd(&g_gstats[i], (unsigned long long)st[i]);
#pragma unroll
            for (int i = 0; i < 16; i++) st[i] = 0;
        }

        // ---------------- outputs (:407-410) ----------------
        if (!bad) {
            for (int v = t; v < n; v += TG) a_io[v] = asg[v];
            if (t == 0) {
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
        } else if (t == 0) {
            const int s = atomicAdd(P.ovf_count, 1);
            P.ovf_list[s] = ind;
        }
        sync();
    }
#undef GPH
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using GKernT = void (*)(GroupParams);

template <int KV, int NW>
static GKernT pick_ch(int ch) {
    switch (ch) {
        case 8:
            if constexpr (8 / NW >= 4) return tabucol_group_kernel<KV, 8, NW>;
            return nullptr;
        case 16: return tabucol_group_kernel<KV, 16, NW>;
        case 32: return tabucol_group_kernel<KV, 32, NW>;
        default: return nullptr;
    }
}
template <int NW>
static GKernT pick_kv(int kv, int ch) {
    switch (kv) {
        case 1: return pick_ch<1, NW>(ch);
        case 2: return pick_ch<2, NW>(ch);
        case 3: return pick_ch<3, NW>(ch);
        case 4: return pick_ch<4, NW>(ch);
        case 6: return pick_ch<6, NW>(ch);
        case 8: return pick_ch<8, NW>(ch);
        default: return nullptr;
    }
}
static GKernT pick_group_kernel(int nw, int kv, int ch) {
    if (nw == 1) return pick_kv<1>(kv, ch);
    if (nw == 2) return pick_kv<2>(kv, ch);
    if (nw == 4) return pick_kv<4>(kv, ch);
    return nullptr;
}

struct GroupPlan {
    int kv, ch, nw, groups, grid;
    size_t group_smem, xch_bytes;
};

static int upload_divtab_grp(cudaStream_t st) {
    static bool done[64] = {false};
    int d = 0;
    cudaGetDevice(&d);
    if (done[d & 63]) return MCB_OK;
    ulonglong2 tab[32];
    for (int i = 0; i < 32; i++) {
        const uint64_t o = 2 * (uint64_t)i + 1;
        uint64_t x = o;
        for (int r = 0; r < 6; r++) x *= 2 - o * x;
        tab[i] = make_ulonglong2(x, ~0ull / o);
    }
    if (cudaMemcpyToSymbolAsync(g_divtab_grp, tab, sizeof(tab), 0, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_group: divisor table upload failed");
    done[d & 63] = true;
    return MCB_OK;
}

static bool group_plan(int n, int k, int64_t p, GroupPlan *pl) {
    // opt-in (MCB_GROUP_NW=1|2|4): measured slower than the warp kernel at
    // every population so far, so the warp kernel stays default
    const char *e = getenv("MCB_GROUP_NW");
    const int nw = e ? atoi(e) : 0;
    if (nw != 1 && nw != 2 && nw != 4) return false;
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
    const int ch_need = (n + 31) / 32;
    int ch = ch_need <= 8 ? 8 : ch_need <= 16 ? 16 : 32;
    if (ch / nw < 4) ch = 4 * nw;  // slots per thread are processed 4 at a time
    const int xwords = 4 * nw + 1 + nw + 2 * ch + 3 + nw;
    const size_t xb = ((size_t)xwords * 4 + 15) & ~(size_t)15;
    auto a16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
    // exchange words | summaries | gamma rows | conflict list, positions | colours
    const size_t sb = a16(4 * (size_t)n);
    size_t gb = xb + sb + a16((size_t)n * kp) + 2 * a16(2 * (size_t)n) + a16((size_t)n);
    // the unrolled update touches rows lane + 32 q for all q < CH
    gb = std::max(gb, xb + sb + (size_t)32 * ch * kp);
    gb = a16(gb);
    const size_t cap = (size_t)max_smem_optin();
    const int sms = num_sms();
    int g = (int)std::min<size_t>(cap / gb, 8);
    const int want = (int)std::min<int64_t>(8, (p + sms - 1) / sms);
    g = std::min(g, want);
    if (const char *eg = getenv("MCB_GROUPS")) g = std::max(1, std::min(g, atoi(eg)));
    if (g < 1) return false;
    pl->kv = kv;
    pl->ch = ch;
    pl->nw = nw;
    pl->groups = g;
    pl->group_smem = gb;
    pl->xch_bytes = xb;
    pl->grid = (int)std::min<int64_t>((p + g - 1) / g, sms);
    return true;
}

__global__ void tg_bitset_kernel(const int64_t *indptr, const int32_t *indices, int n, int ch, uint32_t *bits) {
    for (int v = blockIdx.x; v < n; v += gridDim.x) {
        uint32_t *row = bits + (size_t)v * ch;
        for (int64_t i = indptr[v] + threadIdx.x; i < indptr[v + 1]; i += blockDim.x) {
            const int u = indices[i];
            const int bit = (u & 31) * ch + (u >> 5);
            atomicOr(row + (bit >> 5), 1u << (bit & 31));
        }
    }
}

// Returns MCB_OK, an error, or -1 when the shape is outside the group kernel's
// envelope (or it is disabled: MCB_GROUP_NW=0).
int tabucol_group_launch(const TabucolArgs &A, cudaStream_t st, int32_t *work_counter, int32_t *ovf_list,
                         int32_t *ovf_count, int32_t *err_flag) {
    if (A.flags & (MCB_FLAG_FORCE_WIDE | MCB_FLAG_FORCE_GLOBAL | MCB_FLAG_PROFILE | MCB_FLAG_WSTATS)) return -1;
    GroupPlan pl;
    if (!group_plan((int)A.n, (int)A.k, A.p, &pl)) return -1;
    GKernT kern = pick_group_kernel(pl.nw, pl.kv, pl.ch);
    if (!kern) return -1;
    if (int rc = upload_divtab_grp(st)) return rc;
    const int n = (int)A.n;
    const size_t smem = (size_t)pl.groups * pl.group_smem;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "tabucol_group: smem attribute (%zu) failed", smem);
    const size_t bb = ((size_t)n * 4 * pl.ch + 255) & ~(size_t)255;
    uint8_t *ws = (uint8_t *)workspace4(bb + 256);
    if (!ws) return set_error(MCB_ERR_CUDA, "tabucol_group: workspace allocation failed");
    if (cudaMemsetAsync(ws, 0, bb, st) != cudaSuccess) return set_error(MCB_ERR_CUDA, "memset failed");
    tg_bitset_kernel<<<std::min(n, 4 * num_sms()), 128, 0, st>>>(A.indptr, A.indices, n, pl.ch,
                                                                 reinterpret_cast<uint32_t *>(ws));
    GroupParams P{};
    P.assigns = A.assigns;
    P.best_assigns = A.best_assigns;
    P.bitset = ws;
    P.indptr = A.indptr;
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
    P.work_list = nullptr;
    P.nwork_dev = nullptr;
    P.work_counter = work_counter;
    P.ovf_list = ovf_list;
    P.ovf_count = ovf_count;
    P.err_flag = err_flag;
    P.flags = A.flags;
    P.group_smem = (int)pl.group_smem;
    P.xch_bytes = (int)pl.xch_bytes;
    P.bitset_bytes = 0;
    P.stats = getenv("MCB_GSTATS") != nullptr;
    if (P.stats) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbolAsync(g_gstats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
    }
    if (getenv("MCB_VERBOSE"))
        fprintf(stderr, "[mcb] tabucol_group<kv=%d,ch=%d,nw=%d> grid=%d groups/CTA=%d smem/group=%zu\n", pl.kv,
                pl.ch, pl.nw, pl.grid, pl.groups, pl.group_smem);
    kern<<<pl.grid, 32 * pl.nw * pl.groups, smem, st>>>(P);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "tabucol_group launch failed");
    return MCB_OK;
}

int tabucol_group_stats(unsigned long long *out) {
    if (cudaMemcpyFromSymbol(out, g_gstats, sizeof(unsigned long long) * 32) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "group stats unavailable");
    return MCB_OK;
}

int tabucol_group_describe(int64_t n, int64_t k, int64_t p, char *buf, int len) {
    GroupPlan pl;
    if (!group_plan((int)n, (int)k, p, &pl)) return -1;
    snprintf(buf, len, "tabucol_group_kernel<KV=%d,CH=%d,NW=%d> %d individuals/CTA x %d CTAs, %zu B smem/individual",
             pl.kv, pl.ch, pl.nw, pl.groups, pl.grid, pl.group_smem);
    return MCB_OK;
}

}  // namespace mcb
