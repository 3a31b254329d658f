// DIAGNOSTIC: FP32 issue rate of the exact dot_f32 step (rounded mul, then add) as scalar
// FMUL+FADD vs FMUL,FMUL+FADD2 (ptxas keeps scalar products and packed adds apart; packed
// mul+add pairs get contracted into FFMA2, which the exact chain cannot use).
#include <cstdio>
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
    unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ unsigned long long pack(float x, float y) {
    unsigned long long d; asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(x), "f"(y)); return d; }
constexpr int CH = 16, IT = 4096;
__global__ void scalar(float *o, float a0, float b0) {
    float s[CH], a[CH];
    for (int c = 0; c < CH; ++c) { s[c] = 0.f; a[c] = a0 + c + threadIdx.x; }
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) s[c] = __fadd_rn(s[c], __fmul_rn(a[c], b0));
        b0 = b0 * 1.0000001f;
    }
    float t = 0; for (int c = 0; c < CH; ++c) t += s[c];
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void packed(float *o, float a0, float b0) {
    unsigned long long s[CH / 2]; float a[CH];
    for (int c = 0; c < CH; ++c) a[c] = a0 + c + threadIdx.x;
    for (int c = 0; c < CH / 2; ++c) s[c] = 0ull;
    for (int i = 0; i < IT; ++i) {
#pragma unroll
        for (int c = 0; c < CH / 2; ++c) s[c] = add2(s[c], pack(__fmul_rn(a[2 * c], b0), __fmul_rn(a[2 * c + 1], b0)));
        b0 = b0 * 1.0000001f;
    }
    float t = 0; for (int c = 0; c < CH / 2; ++c) t += __uint_as_float((unsigned)s[c]) + __uint_as_float((unsigned)(s[c] >> 32));
    o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) scalar<<<148 * 4, 512>>>(o, 1.f, 1.f); else packed<<<148 * 4, 512>>>(o, 1.f, 1.f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double macs = 148.0 * 4 * 512 * CH * IT;
            if (rep == 2) printf("%s: %.3f ms, %.1f T exact-MAC/s\n", v ? "FMUL+FADD2" : "FMUL+FADD ", ms, macs / ms / 1e9);
        }
    }
    return 0;
}
