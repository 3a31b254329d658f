// Microbenchmark: latency / issue cost of REDUX, SHFL, and 5-way independent REDUX on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned *out, long long *cyc, unsigned seed) {
    unsigned a = seed + threadIdx.x, b[5];
    for (int q = 0; q < 5; ++q) b[q] = seed * (q + 3) + threadIdx.x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) a = __reduce_max_sync(0xffffffffu, a) + threadIdx.x;
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int q = 0; q < 5; ++q) b[q] = __reduce_max_sync(0xffffffffu, b[q]) + threadIdx.x;
    }
    long long t2 = clock64();
    float f = seed;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) f = __shfl_xor_sync(0xffffffffu, f, 1) + 1.0f;
    long long t3 = clock64();
    float g[5];
    for (int q = 0; q < 5; ++q) g[q] = seed + q;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int q = 0; q < 5; ++q) g[q] = __shfl_xor_sync(0xffffffffu, g[q], 1) + 1.0f;
    }
    long long t4 = clock64();
    float e = 0.5f;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) e = exp2f(e) * 0.25f;
    long long t5 = clock64();
    out[threadIdx.x + blockIdx.x * 32] = a + b[0] + b[1] + b[2] + b[3] + b[4] + (unsigned)(f + g[0] + g[1] + g[2] + g[3] + g[4] + e);
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
}
int main() {
    unsigned *o; long long *c;
    cudaMalloc(&o, 1 << 20); cudaMallocManaged(&c, 64);
    for (int w : {1, 8}) {
        for (int r = 0; r < 3; ++r) { k<<<1, 32 * w>>>(o, c, 7u); cudaDeviceSynchronize(); }
        printf("warps/CTA %d: REDUX dep chain %.1f cyc; 5 indep REDUX per iter %.1f cyc; SHFL dep %.1f; 5 indep SHFL %.1f; exp2f dep %.1f\n",
               w, c[0] / 256.0, c[1] / 256.0, c[2] / 256.0, c[3] / 256.0, c[4] / 256.0);
    }
    return 0;
}
