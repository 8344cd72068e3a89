// common.cuh -- shared device helpers for the memcolor B200 kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/memcolor_b200.h"

#define MCB_GOLDEN 0x9E3779B97F4A7C15ULL

namespace mcb {

// SplitMix64 finalizer and counter-based stream (reference rng.py:48-65):
//   out_ctr = mix64(key + (ctr + 1) * GOLDEN)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t stream_value(uint64_t key, uint64_t ctr) {
    return mix64(key + (ctr + 1) * MCB_GOLDEN);
}
// u64_below(key, ctr, n) == 0  <=>  stream_value % n == 0 (rng.py:62-65)
__device__ __forceinline__ bool below_is_zero(uint64_t key, uint64_t ctr, uint32_t n) {
    return (stream_value(key, ctr) % (uint64_t)n) == 0;
}
// x % s == 0 for any 32-bit s >= 1, exactly, without the 64-bit integer
// division helper: two fp64 reciprocal steps.  q1 = x * (1/s) is within
// 2^14/s + 1 of x/s, so r = x - q1 s (mod 2^64, exact as a signed value) has
// |r| < 2^14 + 2s, exact in fp64; one rounded quotient more leaves |r2| <= s.
// (checked against % by mcb_debug_modcheck)
__device__ __forceinline__ bool mod_is_zero(uint64_t x, uint32_t s) {
    const double inv = __drcp_rn((double)s);
    const uint64_t q1 = __double2ull_rz(__dmul_rz(__ull2double_rz(x), inv));
    const long long r = (long long)(x - q1 * (uint64_t)s);
    const long long q2 = __double2ll_rn(__dmul_rn((double)r, inv));
    long long r2 = r - q2 * (long long)s;
    if (r2 < 0) r2 += s;
    else if (r2 >= (long long)s) r2 -= s;
    return r2 == 0;
}
__device__ __forceinline__ uint32_t u64_below32(uint64_t key, uint64_t ctr, uint32_t n) {
    return (uint32_t)(stream_value(key, ctr) % (uint64_t)n);
}

// Production-mode generator: Philox4x32-10 keyed by the individual's stream
// key, counter = (draw index, 0).  Only used when MCB_FLAG_PRODUCTION is set.
__device__ __forceinline__ uint4 philox4x32_10(uint2 key, uint4 ctr) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
        uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += W0;
        key.y += W1;
    }
    return ctr;
}
// uniform draw in [0, n) from the 64-bit key and a 64-bit draw counter
static __device__ __noinline__ uint32_t philox_below(uint64_t key, uint64_t ctr, uint32_t n) {
    uint4 r = philox4x32_10(make_uint2((uint32_t)key, (uint32_t)(key >> 32)),
                            make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), 0x5eed, 0));
    uint64_t x = ((uint64_t)r.x << 32) | r.y;
    return (uint32_t)(__umul64hi(x, (uint64_t)n));  // multiply-shift, no modulo bias
}

__device__ __forceinline__ int warp_min(int v, int width = 32) {
    for (int o = width >> 1; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o, width));
    return v;
}
__device__ __forceinline__ int warp_max(int v, int width = 32) {
    for (int o = width >> 1; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o, width));
    return v;
}
__device__ __forceinline__ int warp_sum(int v, int width = 32) {
    for (int o = width >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, width);
    return v;
}
__device__ __forceinline__ long long warp_sum64(long long v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// inclusive prefix within segments of `width` lanes
__device__ __forceinline__ int warp_incl_min(int v, int lane_in_seg, int width = 32) {
    for (int o = 1; o < width; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o, width);
        if (lane_in_seg >= o) v = min(v, t);
    }
    return v;
}
__device__ __forceinline__ int warp_incl_sum(int v, int lane_in_seg, int width = 32) {
    for (int o = 1; o < width; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o, width);
        if (lane_in_seg >= o) v += t;
    }
    return v;
}

}  // namespace mcb
