// init.cu -- batched randomized greedy colourings for weighted runs (sm_100a).
//
// Replaces `greedy_wvcp_init` + `init_wvcp_population` (reference
// pkg/src/memcolor/init.py:30-46, 57-64): individual i walks the vertices in
// `greedy_order` (weight desc, degree desc, id asc; :23-27) with its own
// stream `Stream.derive(seed, TAG_INIT, i)`; each vertex takes
// `allowed[stream.below(len(allowed))]`, allowed = the open colours
// [0, used) not held by an already-coloured neighbour, ascending; with no
// allowed colour it opens colour `used`.
//
// One warp per individual.  The warp's colouring lives in shared memory as
// int16; per vertex the lanes OR the neighbours' colours into a 1024-bit
// blocked mask (lane L owns colours [32 L, 32 L + 32)), count the allowed
// colours per word, prefix-sum them across lanes and the lane holding the
// drawn rank selects its bit.  One draw per vertex that has an allowed colour,
// in vertex order, exactly like the reference's stream.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int GI_WARPS = 4;
constexpr int GI_MAXC = 1024;  // colours representable in the blocked mask

__global__ void __launch_bounds__(GI_WARPS * 32)
    greedy_init_kernel(const int32_t *__restrict__ order, const int64_t *__restrict__ indptr,
                       const int32_t *__restrict__ indices, int n, const uint64_t *__restrict__ keys,
                       int64_t p, int32_t *__restrict__ assigns, int32_t *__restrict__ used_out,
                       int32_t *err) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const size_t per = (((size_t)n * 2 + 15) & ~(size_t)15) + 32 * 4;
    int16_t *asg = reinterpret_cast<int16_t *>(smem + warp * per);
    uint32_t *blk = reinterpret_cast<uint32_t *>(smem + warp * per + per - 32 * 4);

    for (int64_t ind = (int64_t)blockIdx.x * nw + warp; ind < p; ind += (int64_t)gridDim.x * nw) {
        const uint64_t key = keys[ind];
        for (int v = lane; v < n; v += 32) asg[v] = -1;
        int used = 0;
        unsigned long long ctr = 0;
        bool overflow = false;
        __syncwarp();
        for (int t = 0; t < n; t++) {
            const int v = __ldg(order + t);
            blk[lane] = 0u;
            __syncwarp();
            const int64_t s0 = __ldg(indptr + v), s1 = __ldg(indptr + v + 1);
            for (int64_t j = s0 + lane; j < s1; j += 32) {
                const int c = asg[__ldg(indices + j)];
                if (c >= 0) atomicOr(&blk[c >> 5], 1u << (c & 31));
            }
            __syncwarp();
            const int lo = 32 * lane;
            const uint32_t open = used <= lo ? 0u : (used - lo >= 32 ? 0xFFFFFFFFu : (1u << (used - lo)) - 1u);
            const uint32_t al = ~blk[lane] & open;
            const int cnt = __popc(al);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (total > 0) {
                const int r = (int)(stream_value(key, ctr) % (uint64_t)total);
                ctr++;
                const unsigned bm = __ballot_sync(0xffffffffu, incl > r);
                if (lane == __ffs(bm) - 1) {
                    uint32_t z = al;
                    for (int q = r - (incl - cnt); q > 0; q--) z &= z - 1u;
                    asg[v] = (int16_t)(lo + __ffs(z) - 1);
                }
            } else {
                if (used >= GI_MAXC) overflow = true;
                if (lane == 0) asg[v] = (int16_t)min(used, GI_MAXC - 1);
                used++;
            }
            __syncwarp();
        }
        int32_t *out = assigns + (size_t)ind * n;
        for (int v = lane; v < n; v += 32) out[v] = asg[v];
        if (lane == 0) {
            used_out[ind] = used;
            if (overflow) atomicExch(err, 1);
        }
        __syncwarp();
    }
}

int greedy_init_run(const int32_t *order, const int64_t *indptr, const int32_t *indices, int64_t n,
                    const uint64_t *keys, int64_t p, int32_t *assigns, int32_t *used, cudaStream_t st) {
    if (n < 1 || p < 0) return set_error(MCB_ERR_VALUE, "greedy_init: bad shape");
    if (p == 0) return MCB_OK;
    if (n > 32767) return set_error(MCB_ERR_UNSUPPORTED, "greedy_init: n <= 32767");
    const size_t per = (((size_t)n * 2 + 15) & ~(size_t)15) + 32 * 4;
    int warps = GI_WARPS;  // as many as shared memory holds
    while (warps > 1 && warps * per > (size_t)max_smem_optin()) warps >>= 1;
    const size_t smem = warps * per;
    if (smem > (size_t)max_smem_optin()) return set_error(MCB_ERR_UNSUPPORTED, "greedy_init: n too large");
    if (cudaFuncSetAttribute(greedy_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "greedy_init: smem attribute failed");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, greedy_init_kernel, warps * 32, smem);
    per_sm = std::max(per_sm, 1);
    const int grid = (int)std::min<int64_t>((p + warps - 1) / warps, (int64_t)per_sm * num_sms());
    int32_t *err = (int32_t *)workspace(256);
    if (!err) return set_error(MCB_ERR_CUDA, "greedy_init: workspace");
    cudaMemsetAsync(err, 0, 4, st);
    greedy_init_kernel<<<grid, warps * 32, smem, st>>>(order, indptr, indices, (int)n, keys, p, assigns,
                                                          used, err);
    int32_t herr = 0;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "greedy_init kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (herr) return set_error(MCB_ERR_UNSUPPORTED, "greedy_init: more than %d colours", GI_MAXC);
    return MCB_OK;
}

}  // namespace mcb
