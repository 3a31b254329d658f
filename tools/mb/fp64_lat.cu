// Microbenchmark: dependent-chain latency of FP64 ops and the glibc-expf port on one warp.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2502_14856_b200/csrc/frs_device.cuh"
using namespace frs;
__global__ void k(double *out, float *outf, long long *cyc, float seed) {
    __shared__ unsigned long long tab[32];
    if (threadIdx.x < 32) tab[threadIdx.x] = dev::kExp2fTable[threadIdx.x];
    __syncwarp();
    double a = seed, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 512; ++i) a = __fma_rn(a, b, c);
    long long t1 = clock64();
    float f = seed;
#pragma unroll 1
    for (int i = 0; i < 512; ++i) f = (float)((double)f * 1.0000001);
    long long t2 = clock64();
    float e = -seed;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) e = dev::expf_glibc(e - 1.0f, tab) - 0.5f;
    long long t3 = clock64();
    double dv = seed + 3.0;
#pragma unroll 1
    for (int i = 0; i < 64; ++i) dv = 1.0 / dv + 1.0;
    long long t4 = clock64();
    float x = seed;
#pragma unroll 1
    for (int i = 0; i < 512; ++i) x = __fadd_rn(x, 1.0f);
    long long t5 = clock64();
    out[threadIdx.x] = a + dv;
    outf[threadIdx.x] = f + e + x;
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
}
int main() {
    double *o; float *of; long long *c;
    cudaMalloc(&o, 256); cudaMalloc(&of, 256); cudaMallocManaged(&c, 64);
    for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, of, c, 0.5f); cudaDeviceSynchronize(); }
    printf("DFMA chain: %.1f cyc/op; F2F f64<->f32 + DMUL: %.1f cyc/iter; expf_glibc chain: %.1f cyc/call; "
           "DDIV chain: %.1f cyc/div; FADD chain: %.1f cyc/op\n",
           c[0] / 512.0, c[1] / 512.0, c[2] / 256.0, c[3] / 64.0, c[4] / 512.0);
    return 0;
}
