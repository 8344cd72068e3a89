// Dependent-chain latency of the primitives the warp TabuCol kernel is built
// from (one warp, clock64 around N dependent ops).  Calibration tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_latency.cu && /tmp/ub
#include <cstdio>
#include <cstdint>

#define N 256

__global__ void k(int *out, long long *cyc, int seed) {
    __shared__ uint32_t sm[1024];
    const int lane = threadIdx.x;
    for (int i = lane; i < 1024; i += 32) sm[i] = (i * 2654435761u) & 1023;
    __syncwarp();
    uint32_t x = seed + lane;
    long long t0, t1;
    int r = 0;
#define BENCH(idx, body)                           \
    t0 = clock64();                                \
    _Pragma("unroll") for (int i = 0; i < N; i++) { body; } \
    t1 = clock64();                                \
    if (lane == 0) cyc[idx] = t1 - t0;             \
    r += x;
    BENCH(0, x = x * 3 + 1)                                   // IMAD
    BENCH(1, x = min(x ^ 5u, x >> 1))                        // LOP/SHF + IMNMX
    BENCH(2, x = __vminu2(x, x >> 3))                         // VIMNMX pair
    BENCH(3, x = __byte_perm(x, x >> 1, 0x4321))             // PRMT
    BENCH(4, x = __shfl_xor_sync(0xffffffffu, x, 1) + 1)      // SHFL
    BENCH(5, x = __shfl_up_sync(0xffffffffu, x, 1) ^ lane)    // SHFL.UP
    BENCH(6, x = sm[x & 1023])                                // LDS chain
    BENCH(7, x = (x == 7u) ? x + 3 : x + 1)                   // ISETP + SEL
    BENCH(8, x = __reduce_add_sync(0xffffffffu, x) & 1023)    // REDUX
    BENCH(9, x = __ballot_sync(0xffffffffu, x & 1) + x)       // VOTE
    BENCH(10, x = __popc(x) + x)                              // POPC
    BENCH(11, x = (uint32_t)__double2int_rn((double)x * 1.5)) // fp64 mul+cvt
    BENCH(12, if (x & 1) x = x * 5; else x = x + 7)           // divergent-free branch
    out[lane] = r + x;
}

int main() {
    int *o;
    long long *c, h[16];
    cudaMalloc(&o, 128);
    cudaMalloc(&c, 16 * 8);
    k<<<1, 32>>>(o, c, 1);
    k<<<1, 32>>>(o, c, 2);
    cudaMemcpy(h, c, 13 * 8, cudaMemcpyDeviceToHost);
    const char *nm[] = {"IMAD", "LOP+IMNMX", "VIMNMX", "PRMT", "SHFL.BFLY+IADD", "SHFL.UP+LOP", "LDS",
                        "ISETP+SEL", "REDUX+LOP", "VOTE+IADD", "POPC+IADD", "DMUL+CVT", "branch"};
    for (int i = 0; i < 13; i++) printf("%-16s %6.1f cyc/op\n", nm[i], (double)h[i] / N);
    return 0;
}
