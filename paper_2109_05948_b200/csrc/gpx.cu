// gpx.cu -- batched GPX crossover, one warp per offspring (sm_100a).
//
// Replaces `_gpx_batch` / `_gpx_into` (reference pkg/src/memcolor/crossover.py:14-66).
// Reference semantics, reproduced bit-exactly:
//   round r = 0..k-1 takes parent A on even r, B on odd r; its class with the
//   most still-unassigned vertices (strict '>' scan from class 0, so the lowest
//   id wins ties, :35-43); a zero count skips the round (:38-39, :44-45); every
//   unassigned member gets colour r and is removed from both parents' counts
//   (:46-52); leftovers, in ascending vertex order, draw u64_below(key, ctr++, k)
//   (:53-56).
// The reference rescans all n vertices every round (O(k n)).  Here each parent's
// classes are bucketed once (counting sort in shared memory), so a round only
// touches the members of the chosen class: O(n + k^2/32) per offspring.  The
// leftover draws are independent given their rank among leftovers (a ballot
// prefix), so they are evaluated by all lanes at once.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace mcb {

constexpr int GPX_WARPS = 4;

__global__ void __launch_bounds__(GPX_WARPS * 32)
    gpx_kernel(const int32_t *__restrict__ pop, int64_t p, int n, const int64_t *__restrict__ matches,
               int64_t rows, int64_t row_off, int64_t K, int k, const uint64_t *__restrict__ keys,
               int32_t *__restrict__ out, int32_t *err) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // per-warp layout
    const int kp = (k + 3) & ~3;
    const size_t per = (size_t)4 * kp * 4 + (size_t)2 * n * 2 + (size_t)n * 2 + 64;
    uint8_t *base = smem + warp * ((per + 15) & ~(size_t)15);
    int *cnt_a = reinterpret_cast<int *>(base);
    int *cnt_b = cnt_a + kp;
    int *off_a = cnt_b + kp;  // bucket starts
    int *off_b = off_a + kp;
    uint16_t *mem_a = reinterpret_cast<uint16_t *>(off_b + kp);  // vertices bucketed by class
    uint16_t *mem_b = mem_a + n;
    int16_t *child = reinterpret_cast<int16_t *>(mem_b + n);

    const int64_t njobs = rows * K;
    for (int64_t job = (int64_t)blockIdx.x * GPX_WARPS + warp; job < njobs;
         job += (int64_t)gridDim.x * GPX_WARPS) {
        const int64_t i = job / K, j = job % K;
        const int64_t mi = matches[job];
        if (mi < 0 || mi >= p) {
            if (lane == 0) atomicExch(err, 1);
            continue;
        }
        const int32_t *pa = pop + (size_t)(row_off + i) * n;
        const int32_t *pb = pop + (size_t)mi * n;
        const uint64_t key = keys[job];
        for (int c = lane; c < kp; c += 32) {
            cnt_a[c] = 0;
            cnt_b[c] = 0;
        }
        __syncwarp();
        int bad = 0;
        for (int v = lane; v < n; v += 32) {
            const int a = pa[v], b = pb[v];
            if (a < 0 || a >= k || b < 0 || b >= k) {
                bad = 1;
                continue;
            }
            atomicAdd(&cnt_a[a], 1);
            atomicAdd(&cnt_b[b], 1);
            child[v] = -1;
        }
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) atomicExch(err, 1);
            continue;
        }
        __syncwarp();
        // exclusive scans -> bucket offsets (warp scan over chunks of 32 classes)
        {
            int ca = 0, cb = 0;
            for (int c0 = 0; c0 < k; c0 += 32) {
                const int c = c0 + lane;
                const int xa = c < k ? cnt_a[c] : 0, xb = c < k ? cnt_b[c] : 0;
                const int ia = warp_incl_sum(xa, lane), ib = warp_incl_sum(xb, lane);
                if (c < k) {
                    off_a[c] = ca + ia - xa;
                    off_b[c] = cb + ib - xb;
                }
                ca += __shfl_sync(0xffffffffu, ia, 31);
                cb += __shfl_sync(0xffffffffu, ib, 31);
            }
        }
        __syncwarp();
        for (int v = lane; v < n; v += 32) {
            mem_a[atomicAdd(&off_a[pa[v]], 1)] = (uint16_t)v;
            mem_b[atomicAdd(&off_b[pb[v]], 1)] = (uint16_t)v;
        }
        __syncwarp();
        // off_x[c] now holds the END of bucket c (= start of bucket c+1)
        // rounds (:31-52)
        for (int r = 0; r < k; r++) {
            const bool use_a = (r & 1) == 0;
            int *cnt = use_a ? cnt_a : cnt_b;
            // argmax with lowest index on ties
            int bv = -1, bc = 0;
            for (int c = lane; c < k; c += 32) {
                const int x = cnt[c];
                if (x > bv) {
                    bv = x;
                    bc = c;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const int ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (ov > bv || (ov == bv && oc < bc)) {
                    bv = ov;
                    bc = oc;
                }
            }
            if (bv <= 0) continue;
            // members of class bc of the chosen parent
            const int *offs = use_a ? off_a : off_b;
            const uint16_t *mem = use_a ? mem_a : mem_b;
            const int e = offs[bc];
            const int s = (bc == 0) ? 0 : offs[bc - 1];
            for (int t = s + lane; t < e; t += 32) {
                const int v = mem[t];
                if (child[v] < 0) {
                    child[v] = (int16_t)r;
                    atomicSub(&cnt_a[pa[v]], 1);
                    atomicSub(&cnt_b[pb[v]], 1);
                }
            }
            __syncwarp();
        }
        // leftovers (:53-56): rank among unassigned vertices in ascending order
        int32_t *o = out + (size_t)job * n;
        uint64_t ctr = 0;
        for (int v0 = 0; v0 < n; v0 += 32) {
            const int v = v0 + lane;
            const bool left = v < n && child[v] < 0;
            const unsigned bal = __ballot_sync(0xffffffffu, left);
            int cv = 0;
            if (v < n) {
                cv = child[v];
                if (left) cv = (int)u64_below32(key, ctr + __popc(bal & ((1u << lane) - 1u)), (uint32_t)k);
                o[v] = cv;
            }
            ctr += __popc(bal);
        }
        __syncwarp();
        (void)j;
    }
}

int gpx_run(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t K, int64_t k,
            const uint64_t *keys, int32_t *out, uint32_t flags, cudaStream_t st) {
    return gpx_rows_run(pop, p, n, matches, p, 0, K, k, keys, out, flags, st);
}

int gpx_rows_run(const int32_t *pop, int64_t p, int64_t n, const int64_t *matches, int64_t rows,
                 int64_t row_off, int64_t K, int64_t k, const uint64_t *keys, int32_t *out,
                 uint32_t flags, cudaStream_t st) {
    if (rows < 0 || row_off < 0 || row_off + rows > p)
        return set_error(MCB_ERR_VALUE, "gpx: row range [%lld, %lld) outside the population",
                         (long long)row_off, (long long)(row_off + rows));
    if (p < 0 || n < 0 || K < 0 || k < 1)
        return set_error(MCB_ERR_VALUE, "gpx: bad shape p=%lld n=%lld K=%lld k=%lld", (long long)p,
                         (long long)n, (long long)K, (long long)k);
    if (n > 65535 || k > 32767) return set_error(MCB_ERR_UNSUPPORTED, "gpx: n<=65535, k<=32767");
    if (rows == 0 || K == 0 || n == 0) return MCB_OK;
    const int kp = ((int)k + 3) & ~3;
    const size_t per = (size_t)4 * kp * 4 + (size_t)2 * n * 2 + (size_t)n * 2 + 64;
    const size_t smem = GPX_WARPS * ((per + 15) & ~(size_t)15);
    if (smem > (size_t)max_smem_optin()) return set_error(MCB_ERR_UNSUPPORTED, "gpx: shape too large");
    if (cudaFuncSetAttribute(gpx_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return set_error(MCB_ERR_CUDA, "gpx: smem attribute failed");
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gpx_kernel, GPX_WARPS * 32, smem);
    nb = std::max(nb, 1);
    const int64_t jobs = rows * K;
    const int grid = (int)std::min<int64_t>((jobs + GPX_WARPS - 1) / GPX_WARPS, (int64_t)nb * num_sms());
    int32_t *err = (int32_t *)workspace(256);
    if (!err) return set_error(MCB_ERR_CUDA, "gpx: workspace");
    cudaMemsetAsync(err, 0, 4, st);
    gpx_kernel<<<grid, GPX_WARPS * 32, smem, st>>>(pop, p, (int)n, matches, rows, row_off, K, (int)k,
                                                   keys, out, err);
    int32_t herr = 0;
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return set_error(MCB_ERR_CUDA, "gpx kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
    if (herr) return set_error(MCB_ERR_RANGE, "gpx: color id or parent index out of range");
    (void)flags;
    return MCB_OK;
}

}  // namespace mcb
