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
        if (bad && err) atomicExch(err, 1);
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

// ---- inference path: colour-sorted segment sums with the eval epilogue ----

// Stable counting sort of each coloring's vertices by colour (one warp per
// coloring, vertices in chunks of 32 in index order): order[b, :] lists the
// vertices of colour 0, then 1, ...; offs[b, i] = start of colour i (k + 1).
__global__ void colour_order_kernel(const int32_t *__restrict__ assigns, int64_t B, int n, int k,
                                    int32_t *__restrict__ order, int32_t *__restrict__ offs, int32_t *err) {
    extern __shared__ int32_t s_base[];  // per warp: k + 1 counters
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t *base = s_base + warp * (k + 1);
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t b = (int64_t)blockIdx.x * nw + warp; b < B; b += (int64_t)gridDim.x * nw) {
        const int32_t *a = assigns + (size_t)b * n;
        for (int i = lane; i <= k; i += 32) base[i] = 0;
        __syncwarp();
        bool bad = false;
        for (int v = lane; v < n; v += 32) {
            const int c = a[v];
            if ((unsigned)c < (unsigned)k) atomicAdd(&base[c + 1], 1);
            else bad = true;
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) atomicExch(err, 1);
            continue;
        }
        __syncwarp();
        if (lane == 0)
            for (int i = 1; i <= k; i++) base[i] += base[i - 1];
        __syncwarp();
        int32_t *ob = offs + (size_t)b * (k + 1);
        for (int i = lane; i <= k; i += 32) ob[i] = base[i];
        __syncwarp();
        int32_t *ord = order + (size_t)b * n;
        for (int v0 = 0; v0 < n; v0 += 32) {
            const int v = v0 + lane;
            const int c = v < n ? a[v] : -1 - lane;  // unique dummy keys past n
            const unsigned same = __match_any_sync(0xffffffffu, c);
            if (v < n) {
                ord[base[c] + __popc(same & lt)] = v;
            }
            __syncwarp();
            if (v < n && (same & lt) == 0u) base[c] += __popc(same);
            __syncwarp();
        }
    }
}

// z[b, i, col] = epi(sum over colour-i vertices of Lam[v, col]) with, when
// A != nullptr, the eval-mode epilogue y = leaky(s A[col] + C[col]); rows are
// summed in colour-sorted vertex order (deterministic), in registers.
template <typename T>
__global__ void __launch_bounds__(SS_TL)
    segsum_sorted_kernel(const T *__restrict__ lam, const int32_t *__restrict__ order,
                         const int32_t *__restrict__ offs, int64_t B, int n, int k, int64_t L,
                         const T *__restrict__ A, const T *__restrict__ C, T slope, T *__restrict__ z) {
    const int64_t col = (int64_t)blockIdx.y * SS_TL + threadIdx.x;
    if (col >= L) return;
    const T a = A ? A[col] : T(1), c = A ? C[col] : T(0);
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const int32_t *ord = order + (size_t)b * n;
        const int32_t *ob = offs + (size_t)b * (k + 1);
        T *zb = z + (size_t)b * k * L + col;
        int j = 0;
        for (int i = 0; i < k; i++) {
            const int e = __ldg(ob + i + 1);
            T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
            for (; j + 3 < e; j += 4) {
                s0 += __ldg(lam + (size_t)__ldg(ord + j) * L + col);
                s1 += __ldg(lam + (size_t)__ldg(ord + j + 1) * L + col);
                s2 += __ldg(lam + (size_t)__ldg(ord + j + 2) * L + col);
                s3 += __ldg(lam + (size_t)__ldg(ord + j + 3) * L + col);
            }
            for (; j < e; j++) s0 += __ldg(lam + (size_t)__ldg(ord + j) * L + col);
            T s = (s0 + s1) + (s2 + s3);
            if (A) {
                s = s * a + c;
                s = s > T(0) ? s : slope * s;
            }
            zb[(size_t)i * L] = s;
        }
    }
}

// Eval-mode epilogue of layers >= 2, in place: z[b,i,:] = leaky((z[b,i,:] +
// r[b,:]) A + C) (r = rho Gam, A/C = the folded batch-norm affine + beta).
template <typename T>
__global__ void rowbias_affine_leaky_kernel(T *__restrict__ z, const T *__restrict__ r, const T *__restrict__ A,
                                            const T *__restrict__ C, T slope, int64_t B, int k, int64_t L) {
    const int64_t total = B * k * L;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = e % L, b = e / (L * k);
        T s = (z[e] + r[b * L + col]) * A[col] + C[col];
        z[e] = s > T(0) ? s : slope * s;
    }
}

int colour_order_run(const int32_t *assigns, int64_t B, int64_t n, int64_t k, int32_t *order, int32_t *offs,
                     cudaStream_t st) {
    if (B < 0 || n < 1 || k < 1) return set_error(MCB_ERR_VALUE, "colour_order: bad shape");
    if (B == 0) return MCB_OK;
    int32_t *err = (int32_t *)workspace(256);
    if (!err) return set_error(MCB_ERR_CUDA, "colour_order: workspace");
    cudaMemsetAsync(err, 0, 4, st);
    const int nw = 8;
    const size_t smem = (size_t)nw * (k + 1) * 4;
    const int grid = (int)std::min<int64_t>((B + nw - 1) / nw, (int64_t)num_sms() * 8);
    colour_order_kernel<<<grid, nw * 32, smem, st>>>(assigns, B, (int)n, (int)k, order, offs, err);
    int32_t herr = 0;
    if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "colour_order failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (herr) return set_error(MCB_ERR_RANGE, "segsum: color id out of range [0, k)");
    return MCB_OK;
}

int segsum_sorted_run(int dtype, const void *lam, const int32_t *order, const int32_t *offs, int64_t B, int64_t n,
                      int64_t k, int64_t L, const void *A, const void *C, double slope, void *z, cudaStream_t st) {
    if (dtype != 4 && dtype != 8) return set_error(MCB_ERR_VALUE, "segsum: dtype must be 4 or 8 bytes");
    if (B == 0) return MCB_OK;
    const int ty = (int)((L + SS_TL - 1) / SS_TL);
    const int gx = (int)std::min<int64_t>(B, std::max<int64_t>(1, (int64_t)num_sms() * 32 / ty));
    if (dtype == 4)
        segsum_sorted_kernel<float><<<dim3(gx, ty), SS_TL, 0, st>>>(
            (const float *)lam, order, offs, B, (int)n, (int)k, L, (const float *)A, (const float *)C, (float)slope,
            (float *)z);
    else
        segsum_sorted_kernel<double><<<dim3(gx, ty), SS_TL, 0, st>>>(
            (const double *)lam, order, offs, B, (int)n, (int)k, L, (const double *)A, (const double *)C, slope,
            (double *)z);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "segsum_sorted launch failed");
    return MCB_OK;
}

int rowbias_affine_leaky_run(int dtype, void *z, const void *r, const void *A, const void *C, double slope,
                             int64_t B, int64_t k, int64_t L, cudaStream_t st) {
    if (dtype != 4 && dtype != 8) return set_error(MCB_ERR_VALUE, "epilogue: dtype must be 4 or 8 bytes");
    const int64_t total = B * k * L;
    if (total == 0) return MCB_OK;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 16);
    if (dtype == 4)
        rowbias_affine_leaky_kernel<float><<<grid, 256, 0, st>>>((float *)z, (const float *)r, (const float *)A,
                                                                 (const float *)C, (float)slope, B, (int)k, L);
    else
        rowbias_affine_leaky_kernel<double><<<grid, 256, 0, st>>>((double *)z, (const double *)r, (const double *)A,
                                                                  (const double *)C, slope, B, (int)k, L);
    if (cudaGetLastError() != cudaSuccess) return set_error(MCB_ERR_CUDA, "epilogue launch failed");
    return MCB_OK;
}

int segsum_run(int dtype, bool backward, const void *src, const int32_t *assigns, int64_t B, int64_t n,
               int64_t k, int64_t L, void *dst, cudaStream_t st, bool checked) {
    if (B < 0 || n < 1 || k < 1 || L < 1) return set_error(MCB_ERR_VALUE, "segsum: bad shape");
    if (dtype != 4 && dtype != 8) return set_error(MCB_ERR_VALUE, "segsum: dtype must be 4 or 8 bytes");
    if (B == 0) return MCB_OK;
    const int ty = (int)((L + SS_TL - 1) / SS_TL);
    if (!backward) {
        const size_t smem = (size_t)k * SS_TL * dtype;
        if (smem > (size_t)max_smem_optin()) return set_error(MCB_ERR_UNSUPPORTED, "segsum: k too large");
        // unchecked (graph-capturable): no flag word, no readback, no sync --
        // the caller has range-checked the colour ids
        int32_t *err = checked ? (int32_t *)workspace(256) : nullptr;
        if (checked && !err) return set_error(MCB_ERR_CUDA, "segsum: workspace");
        if (checked) cudaMemsetAsync(err, 0, 4, st);
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
        if (!checked) return cudaGetLastError() == cudaSuccess ? MCB_OK : set_error(MCB_ERR_CUDA, "segsum launch failed");
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
