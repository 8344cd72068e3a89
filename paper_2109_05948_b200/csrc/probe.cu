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

}  // namespace mcb

extern "C" int mcb_probe_smem_bandwidth(double *gbs, double *ms) { return mcb::smem_probe(gbs, ms); }

extern "C" int mcb_debug_phase_cycles(unsigned long long *out, int reset) {
    return mcb::tabucol_phase_cycles(out, reset);
}
