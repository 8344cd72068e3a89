// segsum.cu -- first layer of the colour-invariant surrogate on colour ids
// (sm_100a).
//
// The reference feeds its deep-set regressor a one-hot (B, k, n) encoding
// (`mc/surrogate.py:123-133`) and multiplies it by Lam (n x L) in the first
// layer (`:146`): z[b, i, :] = sum over v with assign[b, v] = i of Lam[v, :].
// With colour ids that product is a per-colour segment sum of Lam's rows --
// n L adds per coloring instead of k n L multiply-adds, and no (B, k, n)
// tensor (87 GB float32 at C3's p K candidates).  Its gradient w.r.t. Lam
// (`:209`, einsum over the one-hot) is a gather-sum over the batch:
// dLam[v, :] = sum_b dz[b, assign[b, v], :].
//
// Both kernels are deterministic (fixed summation order, no atomics): thread c
// of a block owns column c of an L tile and walks the vertices (forward) or
// the batch (backward) in order.  The forward accumulates the k x TL tile in
// shared memory, one column per thread (bank-conflict-free), and writes it
// out once; Lam's tile rows are read from L2, coalesced across the block.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int SS_TL = 128;  // columns per block (= threads)

template <typename T>
__global__ void __launch_bounds__(SS_TL)
    segsum_fwd_kernel(const T *__restrict__ lam, const int32_t *__restrict__ assigns, int64_t B, int n, int k,
                      int64_t L, T *__restrict__ z, int32_t *err) {
    extern __shared__ __align__(16) uint8_t smem[];
    T *acc = reinterpret_cast<T *>(smem);  // [k][SS_TL]
    const int c = threadIdx.x;
    const int64_t col = (int64_t)blockIdx.y * SS_TL + c;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        for (int i = 0; i < k; i++) acc[i * SS_TL + c] = T(0);
        const int32_t *a = assigns + (size_t)b * n;
        bool bad = false;
        if (col < L) {
            for (int v = 0; v < n; v++) {
                const int i = __ldg(a + v);
                if ((unsigned)i >= (unsigned)k) {
                    bad = true;
                    continue;
                }
                acc[i * SS_TL + c] += __ldg(lam + (size_t)v * L + col);
            }
            T *zb = z + (size_t)b * k * L;
            for (int i = 0; i < k; i++) zb[(size_t)i * L + col] = acc[i * SS_TL + c];
        }
        if (bad) atomicExch(err, 1);
    }
}

template <typename T>
__global__ void __launch_bounds__(SS_TL)
    segsum_bwd_kernel(const T *__restrict__ dz, const int32_t *__restrict__ assigns, int64_t B, int n, int k,
                      int64_t L, T *__restrict__ dlam) {
    const int c = threadIdx.x;
    const int64_t col = (int64_t)blockIdx.y * SS_TL + c;
    if (col >= L) return;
    for (int v = blockIdx.x; v < n; v += gridDim.x) {
        T s = T(0);
        for (int64_t b = 0; b < B; b++) {
            const int i = __ldg(assigns + (size_t)b * n + v);
            if ((unsigned)i < (unsigned)k) s += __ldg(dz + ((size_t)b * k + i) * L + col);
        }
        dlam[(size_t)v * L + col] = s;
    }
}

int segsum_run(int dtype, bool backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
               int64_t k, int64_t L, void *dst, cudaStream_t st) {
    if (B < 0 || n < 1 || k < 1 || L < 1) return set_error(MCB_ERR_VALUE, "segsum: bad shape");
    if (dtype != 4 && dtype != 8) return set_error(MCB_ERR_VALUE, "segsum: dtype must be 4 or 8 bytes");
    if (B == 0) return MCB_OK;
    const int ty = (int)((L + SS_TL - 1) / SS_TL);
    if (!backward) {
        const size_t smem = (size_t)k * SS_TL * dtype;
        if (smem > (size_t)max_smem_optin()) return set_error(MCB_ERR_UNSUPPORTED, "segsum: k too large");
        int32_t *err = (int32_t *)workspace(256);
        if (!err) return set_error(MCB_ERR_CUDA, "segsum: workspace");
        cudaMemsetAsync(err, 0, 4, st);
        const int gx = (int)std::min<int64_t>(B, std::max<int64_t>(1, (int64_t)num_sms() * 16 / ty));
        if (dtype == 4) {
            cudaFuncSetAttribute(segsum_fwd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            segsum_fwd_kernel<float><<<dim3(gx, ty), SS_TL, smem, st>>>((const float *)src, assigns, B, (int)n,
                                                                       (int)k, L, (float *)dst, err);
        } else {
            cudaFuncSetAttribute(segsum_fwd_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            segsum_fwd_kernel<double><<<dim3(gx, ty), SS_TL, smem, st>>>((const double *)src, assigns, B, (int)n,
                                                                        (int)k, L, (double *)dst, err);
        }
        int32_t herr = 0;
        if (cudaGetLastError() != cudaSuccess ||
            cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return set_error(MCB_ERR_CUDA, "segsum kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
        if (herr) return set_error(MCB_ERR_RANGE, "segsum: color id out of range [0, k)");
        return MCB_OK;
    }
    const int gx = (int)std::min<int64_t>(n, std::max<int64_t>(1, (int64_t)num_sms() * 16 / ty));
    if (dtype == 4)
        segsum_bwd_kernel<float><<<dim3(gx, ty), SS_TL, 0, st>>>((const float *)src, assigns, B, (int)n, (int)k, L,
                                                                (float *)dst);
    else
        segsum_bwd_kernel<double><<<dim3(gx, ty), SS_TL, 0, st>>>((const double *)src, assigns, B, (int)n, (int)k,
                                                                 L, (double *)dst);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "segsum backward launch failed");
    return MCB_OK;
}

}  // namespace mcb
