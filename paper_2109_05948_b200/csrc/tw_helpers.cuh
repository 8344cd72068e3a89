// tw_helpers.cuh -- device helpers shared by the warp-per-individual
// (tabucol_warp.cu) and group-of-warps (tabucol_group.cu) TabuCol kernels:
// the byte-packed gamma row operations (OWN | TABU | gamma), SIMD row minima
// and counts, the in-lane reservoir walk, lane-sum helpers, the tabu ring
// entry format and the row rotation.  See tabucol_warp.cu for the layout.
#pragma once
#include <climits>
#include <cstdint>
#include <utility>

#include "common.cuh"

namespace mcb {
namespace tw {

constexpr int TW_BIG = 1 << 20;
constexpr unsigned FULLM = 0xffffffffu;
constexpr int TW_MAX_WARPS = 8;
constexpr int KE = 32;  // ring registers per lane -> 1024 live tabu entries
constexpr uint32_t OWN = 0x80u, TABU = 0x40u, GM = 0x3Fu;

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

// explicit shared-window byte access with compile-time offsets (keeps the
// unrolled neighbour update at one LDS/STS per byte, [reg + imm] addressing)
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int OFF>
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0+%1], %2;" ::"r"(a), "n"(OFF), "r"(v) : "memory");
}
template <typename F, int... I>
__device__ __forceinline__ void static_for_impl(F &&f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// 0x80 in every byte of x that is zero
__device__ __forceinline__ uint32_t zero_flags(uint32_t z) {
    return ~(((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z) & 0x80808080u;
}
__device__ __forceinline__ int count_eq(uint32_t x, uint32_t M) { return __popc(zero_flags(x ^ M)); }
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
// gamma of the row's own colour: the only byte with bit 7 set
template <int KW>
__device__ __forceinline__ int own_gamma(const uint32_t (&x)[KW]) {
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < KW; w++) acc |= x[w] & (((x[w] & 0x80808080u) >> 7) * GM);
    acc |= acc >> 16;
    acc |= acc >> 8;
    return (int)(acc & GM);
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
// bytes < 0x40, plus (A > 0) tabu bytes of gamma < A (aspiration).  SIMD over
// the 4 bytes: low + (64 - A) has bit 6 set iff low >= A (no carry out).
__device__ __forceinline__ uint32_t cand_word(uint32_t x, int A) {
    uint32_t y = x | ((((x | (x << 1)) & 0x80808080u) >> 7) * 0xFFu);
    if (A > 0) {
        const uint32_t low = x & 0x3F3F3F3Fu;
        const uint32_t ge = (low + (uint32_t)(64 - A) * 0x01010101u) & 0x40404040u;
        const uint32_t asp = x & ~(x >> 1) & ~ge & 0x40404040u;  // tabu, not own, gamma < A
        const uint32_t full = (asp >> 6) * 0xFFu;
        y = (y & ~full) | (low & full);
    }
    return y;
}

// tie events of one row entered with running minimum Pg (gamma space): the
// candidates equal to the running minimum when scanned in colour order
// (localsearch.py:340-350).  One lane, logical words read from shared memory.
template <int KW>
__device__ __forceinline__ int walk_words(const uint32_t (&w)[KW], int A, int Pg) {
    uint32_t y[KW];
    int wm[KW];
#pragma unroll
    for (int i = 0; i < KW; i++) {
        y[i] = cand_word(w[i], A);
        const uint32_t m2 = __vminu2(y[i] & 0x00FF00FFu, __byte_perm(y[i], 0, 0x4341));
        wm[i] = (int)min(m2 & 0xFFFFu, m2 >> 16);
    }
    // candidates are <= 63 and non-candidates 0xFF, so a running minimum
    // clamped to 0xFE is never lowered or tied by a non-candidate.  The
    // running minimum entering word i is a short chain over word minima; the
    // 4-byte chains of different words are independent.
    int M = min(Pg, 0xFE), t[KW];
#pragma unroll
    for (int i = 0; i < KW; i++) {
        // exclusive prefix minima of the 4 bytes, packed; events = equal bytes
        const int c0 = M;
        const int c1 = min(c0, (int)(y[i] & 0xFFu));
        const int c2 = min(c1, (int)__byte_perm(y[i], 0, 0x4441));
        const int c3 = min(c2, (int)__byte_perm(y[i], 0, 0x4442));
        const uint32_t Cp = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410);
        t[i] = count_eq(y[i], Cp);
        M = min(M, wm[i]);
    }
#pragma unroll
    for (int d = 1; d < KW; d <<= 1)
#pragma unroll
        for (int i = 0; i + d < KW; i += 2 * d) t[i] += t[i + d];
    return t[0];
}

// exclusive prefix sum over lanes of small values v in [0, 2^BITS): one
// ballot per bit plane, then popcounts (one VOTE + POPC level instead of a
// log-step shuffle scan)
template <int BITS>
__device__ __forceinline__ int excl_sum_small(int v, unsigned lt) {
    int s = 0;
#pragma unroll
    for (int b = 0; b < BITS; b++) s += __popc(__ballot_sync(0xffffffffu, (v >> b) & 1) & lt) << b;
    return s;
}
// sum over the lanes of a mask, values in [0, 2^BITS)
template <int BITS>
__device__ __forceinline__ int masked_sum_small(int v, unsigned m) {
    int s = 0;
#pragma unroll
    for (int b = 0; b < BITS; b++) s += __popc(__ballot_sync(0xffffffffu, (v >> b) & 1) & m) << b;
    return s;
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

// entry: [valid:1][v:10][c:7][expiry mod 2^14:14]
__device__ __forceinline__ uint32_t ent_pack(int v, int c, uint32_t e) {
    return 0x80000000u | ((uint32_t)v << 21) | ((uint32_t)c << 14) | (e & 0x3FFFu);
}
__device__ __forceinline__ uint32_t ent_dist(uint32_t ent, uint32_t it) { return (ent - it) & 0x3FFFu; }


template <int KW>
struct Swz {
    static constexpr int G = (KW % 32 == 0) ? 32 : (KW % 16 == 0) ? 16 : (KW % 8 == 0) ? 8 : (KW % 4 == 0) ? 4 : (KW % 2 == 0) ? 2 : 1;
    static constexpr int SH = G == 32 ? 0 : G == 16 ? 1 : G == 8 ? 2 : G == 4 ? 3 : G == 2 ? 4 : 5;
    __device__ __forceinline__ static int g(int u) { return (u >> SH) & (G - 1); }
    // physical word of logical word w in a row rotated by g
    __device__ __forceinline__ static int pw(int w, int gg) {
        const int p = w + gg;
        return p >= KW ? p - KW : p;
    }
    __device__ __forceinline__ static int phys(int c, int gg) { return 4 * pw(c >> 2, gg) + (c & 3); }
};

}  // namespace tw
}  // namespace mcb
