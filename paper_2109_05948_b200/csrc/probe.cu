// probe.cu -- shared-memory bandwidth probe (the roofline denominator of the
// shared-memory-bound kernels; MEASURED_PEAKS.json only carries HBM and GEMM).
// Every CTA streams 16-byte, bank-conflict-free LDS.128 reads over a 32 KB
// tile; bytes / elapsed = aggregate shared-memory read bandwidth.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace mcb {

__global__ void __launch_bounds__(1024) smem_probe_kernel(int iters, uint32_t *sink) {
    __shared__ uint4 tile[2048];  // 32 KB
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
        tile[i] = make_uint4(i, i * 3u, i * 5u, i * 7u);
    __syncthreads();
    uint32_t acc = 0;
    int idx = threadIdx.x & 2047;
    for (int it = 0; it < iters; it++) {
#pragma unroll 8
        for (int j = 0; j < 8; j++) {
            const uint4 v = tile[(idx + j * 256) & 2047];
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        idx = (idx + 1) & 2047;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int smem_probe(double *gbs, double *ms) {
    const int iters = 4096;
    const int ctas = 2 * num_sms();
    uint32_t *sink = (uint32_t *)workspace(256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    smem_probe_kernel<<<ctas, 1024>>>(16, sink);  // warm-up
    cudaEventRecord(e0);
    smem_probe_kernel<<<ctas, 1024>>>(iters, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return set_error(MCB_ERR_CUDA, "probe failed");
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double bytes = (double)ctas * 1024.0 * iters * 8 * 16;
    *ms = t;
    *gbs = bytes / (t * 1e-3) / 1e9;
    return MCB_OK;
}

// L2 read bandwidth: every thread streams 16-byte loads (L1 bypassed) over a
// buffer that fits in L2, several passes after one warm-up pass
__global__ void __launch_bounds__(512) l2_probe_kernel(const uint4 *buf, size_t n16, int passes, uint32_t *sink) {
    uint32_t acc = 0;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; p++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += st) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(buf + i));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678u) sink[0] = acc;
}

int l2_probe(double *gbs, double *ms) {
    const size_t bytes = (size_t)48 << 20;  // well inside the 126 MB L2
    uint8_t *buf = (uint8_t *)workspace2(bytes + 256);
    if (!buf) return set_error(MCB_ERR_CUDA, "l2 probe: allocation failed");
    cudaMemset(buf, 1, bytes + 256);
    uint32_t *sink = reinterpret_cast<uint32_t *>(buf + bytes);
    const int grid = 4 * num_sms(), passes = 16;
    const uint4 *b4 = reinterpret_cast<const uint4 *>(buf);
    l2_probe_kernel<<<grid, 512>>>(b4, bytes / 16, 1, sink);  // warm-up: the buffer into L2
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    l2_probe_kernel<<<grid, 512>>>(b4, bytes / 16, passes, sink);
    cudaEventRecord(e1);
    if (cudaEventSynchronize(e1) != cudaSuccess) return set_error(MCB_ERR_CUDA, "l2 probe failed");
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = t;
    *gbs = (double)bytes * passes / (t * 1e-3) / 1e9;
    return MCB_OK;
}

}  // namespace mcb

extern "C" int mcb_probe_l2_bandwidth(double *gbs, double *ms) { return mcb::l2_probe(gbs, ms); }

extern "C" int mcb_probe_smem_bandwidth(double *gbs, double *ms) { return mcb::smem_probe(gbs, ms); }

extern "C" int mcb_debug_phase_cycles(unsigned long long *out, int reset) {
    return mcb::tabucol_phase_cycles(out, reset);
}

extern "C" int mcb_debug_warp_stats(unsigned long long *out) { return mcb::tabucol_warp_stats(out); }
extern "C" int mcb_debug_cluster_warps(unsigned long long *out, int reset) {
    return mcb::tabucol_cluster_warp_stats(out, reset);
}
extern "C" int mcb_debug_group_stats(unsigned long long *out) { return mcb::tabucol_group_stats(out); }
extern "C" int mcb_debug_wvcp_stats(unsigned long long *out, int reset) { return mcb::wvcp_stats(out, reset); }

// Diagnostics: mod_is_zero (common.cuh) against the 64-bit % on `count`
// pseudo-random (x, s) pairs, s drawn log-uniformly from [1, 2^32).
__global__ void modcheck_kernel(int64_t count, unsigned long long *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t x0 = mcb::stream_value(0x1234567ull, (uint64_t)i);
        const uint64_t y = mcb::stream_value(0x89abcdefull, (uint64_t)i);
        const int bits = 1 + (int)(y % 32);
        uint32_t s = (uint32_t)((y >> 8) & ((bits >= 32) ? 0xFFFFFFFFull : ((1ull << bits) - 1)));
        if (s == 0) s = 1;
        // half the samples are exact multiples (the case the draws test for)
        const uint64_t x = (i & 1) ? x0 : (x0 / s) * s;
        if (mcb::mod_is_zero(x, s) != (x % s == 0)) atomicAdd(bad, 1ull);
    }
}
namespace mcb {
int tabucol_warp_divcheck(int64_t count, unsigned long long *mismatches);
}
extern "C" int mcb_debug_modcheck(int64_t count, unsigned long long *mismatches) {
    // fp64 path (any 32-bit s) and the small-divisor table path (s < 64)
    unsigned long long m2 = 0;
    if (int rc = mcb::tabucol_warp_divcheck(count, &m2)) return rc;
    unsigned long long *d = nullptr;
    if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return MCB_ERR_CUDA;
    cudaMemset(d, 0, sizeof(*d));
    modcheck_kernel<<<1184, 256>>>(count, d);
    const cudaError_t e = cudaMemcpy(mismatches, d, sizeof(*d), cudaMemcpyDeviceToHost);
    cudaFree(d);
    *mismatches += m2;
    return e == cudaSuccess ? MCB_OK : MCB_ERR_CUDA;
}

namespace mcb {
int tabucol_warp_describe(int64_t n, int64_t k, int64_t p, char *buf, int len);
}
extern "C" int mcb_tabucol_describe(int64_t n, int64_t k, int64_t p, char *buf, int len) {
    if (mcb::tabucol_group_describe(n, k, p, buf, len) == 0) return 0;
    return mcb::tabucol_warp_describe(n, k, p, buf, len);
}
