// tc_shared.cuh -- pieces shared by the CTA TabuCol kernel (tabucol.cu) and
// its cluster variant (tabucol_cluster.cu): launch parameters, packed scan
// records, 16/32-bit wrap-around tabu expiries, SIMD byte helpers and the
// conflict-list update of the reference (pkg/src/memcolor/localsearch.py:368-385).
#pragma once
#include <cstdint>

#include "common.cuh"

namespace mcb {

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
    int32_t *sm_ticket;  // per-SM counters: master-warp assignment
    uint8_t *ws_gamma;  // per-CTA gamma slice (when gamma is not in smem)
    uint8_t *ws_stamp;  // per-CTA dense overflow expiry table
    size_t ws_g_stride, ws_s_stride;
    uint32_t flags;
    int const_indptr;
    int swz_rs, swz_rm;  // gamma row word rotation: rot(v) = (v >> rs) & rm
};

// (int, int) pair records: packed int16 x 2 for the narrow variant (deltas in
// [-254, 254] or TC_BIG), int2 for the wide one
template <bool NARROW>
struct RecT;
template <>
struct RecT<true> {
    using T = uint32_t;
};
template <>
struct RecT<false> {
    using T = int2;
};
__device__ __forceinline__ uint32_t rec_pack(int x, int y, uint32_t *) {
    return (uint32_t)(uint16_t)(int16_t)(x >= TC_BIG ? 0x7FFF : x) | ((uint32_t)y << 16);
}
__device__ __forceinline__ int2 rec_pack(int x, int y, int2 *) { return make_int2(x, y); }
__device__ __forceinline__ int2 rec_unpack(uint32_t r) {
    const int x = (int)(int16_t)(r & 0xFFFFu);
    return make_int2(x == 0x7FFF ? TC_BIG : x, (int)(r >> 16));
}
__device__ __forceinline__ int2 rec_unpack(int2 r) { return r; }

template <typename S>
__device__ __forceinline__ bool active(S e, uint32_t it) {
    if constexpr (sizeof(S) == 2)
        return (int16_t)(uint16_t)((uint16_t)e - (uint16_t)it) > 0;
    else
        return (int32_t)((uint32_t)e - it) > 0;
}

// a 5th live tabu entry of a vertex: spill to its dense global row (rare)
template <typename S>
static __device__ __noinline__ void spill_set(S *gs, S *tovf_v, bool ovf_live, int k, int a, S e_new,
                                       uint32_t it) {
    if (!ovf_live) {  // fresh spill row
        for (int cc = 0; cc < k; cc++) gs[cc] = (S)it;
        *tovf_v = e_new;
    } else if (active<S>(e_new, (uint32_t)*tovf_v)) {
        *tovf_v = e_new;
    }
    gs[a] = e_new;
}

// number of bytes of x equal to byte value c
__device__ __forceinline__ int count_eq_bytes(uint32_t x, uint32_t c) {
    const uint32_t z = x ^ (c * 0x01010101u);
    const uint32_t t = ((z & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z;
    return __popc(~t & 0x80808080u);
}
// unsigned byte minimum (native 16x2 min)
__device__ __forceinline__ uint32_t min_bytes(uint32_t x) {
    const uint32_t m2 = __vminu2(x & 0x00FF00FFu, (x >> 8) & 0x00FF00FFu);
    return min(m2 & 0xFFFFu, m2 >> 16);
}
// 4 bits -> 4 byte masks
__device__ __forceinline__ uint32_t expand_nibble(uint32_t nib) {
    return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// conflict-list membership update (:374-385): append, or swap-with-last remove
__device__ __forceinline__ void cl_apply(uint16_t *clist, uint16_t *cpos, int &Cn, int u, bool in_conf) {
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
}

}  // namespace mcb
