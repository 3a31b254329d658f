// EXACT mode kernels: CUDA-core fp32 LM head in the reference's dot_f32 order, exact
// softmax (glibc expf port + exact-or-sequential double Σ) and (prob desc, index asc) top-k.
//
// Reference arithmetic reproduced:
//   dot_f32            kernels.cpp:13-32   8 lane chains s_l += a*b (rounded mul, rounded add)
//                                          over indices = l mod 8, then ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)),
//                                          then a scalar rounded tail for d % 8.
//   softmax            kernels.cpp:62-91   mx = max(l/t); e = expf(l/t - mx); total = Σ (double)e in
//                                          index order; inv = (float)(1/total); p = e*inv.
//   topk / argmax      kernels.cpp:93-122  (value desc, index asc); argmax strict '>' => lowest index.
//
// Layout: the LM-head slab is row-major [rows x d] (fp32 or bf16). One persistent CTA per SM
// (1024 threads) keeps the NB hidden rows resident in shared memory as sh[e*NBS + i] =
// h[i][e]; each warp pulls groups of 4 slab rows from an atomic work queue and maps lane =
// 8*q + l to (row q of the group, dot_f32 lane chain l). The chain order is therefore the
// reference's exactly; the final tree is three xor-shuffles (1, 2, 4) whose association is
// the reference's tree. Bound: FP32 issue (2 instructions per MAC, __fmul_rn/__fadd_rn keep
// ptxas from contracting into FFMA), ~72 us at 1965 MHz for n=10, V_sub=32768, d=4096.
#include <cuda_bf16.h>

#include <algorithm>

#include "frs_common.cuh"

namespace frs {
namespace {

__device__ __forceinline__ float load_w(const float *p) { return __ldg(p); }
__device__ __forceinline__ float load_w(const __nv_bfloat16 *p) {
    const unsigned short u = __ldg(reinterpret_cast<const unsigned short *>(p));
    return __uint_as_float(static_cast<uint32_t>(u) << 16);  // bf16 -> fp32 is exact
}

template <int NB, typename WT>
__global__ void __launch_bounds__(1024, 1)
    k_exact_logits(const float *__restrict__ h, int n, int d, const WT *__restrict__ W, int v_rows,
                   float *__restrict__ logits, int ld, unsigned *__restrict__ counter) {
    constexpr int NBS = (NB + 3) & ~3;
    constexpr int U = 16;  // W prefetch depth (loads in flight per thread)
    extern __shared__ float4 smem4[];
    float *sh = reinterpret_cast<float *>(smem4);
    const int T = d >> 3;
    const int E8 = T * 8;
    for (int idx = threadIdx.x; idx < E8 * NBS; idx += blockDim.x) {
        const int e = idx % E8, i = idx / E8;
        sh[e * NBS + i] = (i < n) ? h[(size_t)i * d + e] : 0.0f;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, q = lane >> 3, l = lane & 7;
    const int n_groups = (v_rows + 3) >> 2;
    for (;;) {
        int g = 0;
        if (lane == 0) g = static_cast<int>(atomicAdd(counter, 1u));
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= n_groups) break;
        const int row = g * 4 + q;
        const bool valid = row < v_rows;
        const WT *wr = W + (size_t)(valid ? row : 0) * d + l;
        float s[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) s[i] = 0.0f;

        int t = 0;
        for (; t + U <= T; t += U) {
            float w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) w[u] = load_w(wr + (size_t)(t + u) * 8);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float4 *hp = reinterpret_cast<const float4 *>(sh + ((t + u) * 8 + l) * NBS);
                float hv[NBS];
#pragma unroll
                for (int c = 0; c < NBS / 4; ++c) {
                    const float4 v = hp[c];
                    hv[4 * c] = v.x;
                    hv[4 * c + 1] = v.y;
                    hv[4 * c + 2] = v.z;
                    hv[4 * c + 3] = v.w;
                }
#pragma unroll
                for (int i = 0; i < NB; ++i) s[i] = __fadd_rn(s[i], __fmul_rn(hv[i], w[u]));
            }
        }
        for (; t < T; ++t) {
            const float w = load_w(wr + (size_t)t * 8);
            const float *hp = sh + (t * 8 + l) * NBS;
#pragma unroll
            for (int i = 0; i < NB; ++i) s[i] = __fadd_rn(s[i], __fmul_rn(hp[i], w));
        }
        // ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)) — kernels.cpp:27
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            float a = s[i];
            a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 1));
            a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 2));
            a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 4));
            if (l == 0 && valid && i < n) {
                const WT *wt = W + (size_t)row * d;
                for (int e = E8; e < d; ++e)  // kernels.cpp:28-30 scalar tail
                    a = __fadd_rn(a, __fmul_rn(h[(size_t)i * d + e], load_w(wt + e)));
                logits[(size_t)i * ld + row] = a;
            }
        }
    }
}

// ---- glibc 2.39 expf, FMA ifunc, device port ----
__constant__ unsigned long long kExp2fT[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

__device__ __forceinline__ float expf_glibc(float x, const unsigned long long *tab) {
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = static_cast<double>(x);
    double kd = __fma_rn(0x1.71547652b82fep+5, xd, 0x1.8p+52);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, 0x1.8p+52);
    const double r = __fma_rn(0x1.71547652b82fep+5, xd, -kd);
    const unsigned long long tt = tab[ki & 31ull] + (ki << 47);
    const double s = __longlong_as_double(static_cast<long long>(tt));
    const double z = __fma_rn(0x1.c6af84b912394p-20, r, 0x1.ebfce50fac4f3p-13);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(0x1.62e42ff0c52d6p-6, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// Exponent of the lowest set bit of a positive float (INT_MAX for 0).
__device__ __forceinline__ int lsb_exponent(float v) {
    const uint32_t b = __float_as_uint(v);
    const uint32_t ex = (b >> 23) & 0xffu;
    uint32_t m = b & 0x7fffffu;
    if (ex != 0) m |= 0x800000u;
    if (m == 0) return 0x7fffffff;
    return (ex != 0 ? static_cast<int>(ex) - 150 : -149) + (__ffs(m) - 1);
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < nw ? red[lane] : red[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

struct MaxF { __device__ float operator()(float a, float b) const { return fmaxf(a, b); } };
struct SumD { __device__ double operator()(double a, double b) const { return a + b; } };
struct MinI { __device__ int operator()(int a, int b) const { return min(a, b); } };
struct OrI { __device__ int operator()(int a, int b) const { return a | b; } };
struct MaxU64 {
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        return a > b ? a : b;
    }
};

__device__ __forceinline__ unsigned long long prob_key(float p, int j) {
    return (static_cast<unsigned long long>(__float_as_uint(p)) << 32) | (0xffffffffu - static_cast<uint32_t>(j));
}

// One CTA per row: exact softmax (kernels.cpp:62-91) + top-kk by (prob desc, idx asc)
// (kernels.cpp:93-111) + restricted->full remap (drafting.cpp:151/210).
__global__ void __launch_bounds__(1024)
    k_softmax_topk(const float *__restrict__ logits, int ld, int v, int k, float temperature,
                   const int32_t *__restrict__ ordered, float *__restrict__ ework,
                   int32_t *__restrict__ out_ridx, int32_t *__restrict__ out_full,
                   float *__restrict__ out_prob, float *__restrict__ out_rowmax,
                   double *__restrict__ out_total, uint32_t *__restrict__ out_flags) {
    __shared__ unsigned long long tab[32];
    __shared__ double red_d[32];
    __shared__ float red_f[32];
    __shared__ int red_i[32];
    __shared__ unsigned long long red_k[32];
    const int row = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    if (tid < 32) tab[tid] = kExp2fT[tid];
    const float *L = logits + (size_t)row * ld;
    float *E = ework + (size_t)row * ld;

    float mx = -__int_as_float(0x7f800000);
    int bad = 0;
    for (int j = tid; j < v; j += nt) {
        const float x = L[j];
        if (!isfinite(x)) bad = 1;
        const float y = __fdiv_rn(x, temperature);
        mx = (mx < y) ? y : mx;
    }
    mx = block_reduce(mx, MaxF(), red_f);
    bad = block_reduce(bad, OrI(), red_i);
    uint32_t flags = bad ? FRS_FLAG_NONFINITE : 0u;

    double part = 0.0;
    int lsb = 0x7fffffff;
    for (int j = tid; j < v; j += nt) {
        const float e = expf_glibc(__fsub_rn(__fdiv_rn(L[j], temperature), mx), tab);
        E[j] = e;
        part += static_cast<double>(e);
        lsb = min(lsb, lsb_exponent(e));
    }
    double total = block_reduce(part, SumD(), red_d);
    lsb = block_reduce(lsb, MinI(), red_i);
    // Every partial sum (any order) is exact iff all e_j are multiples of 2^(ilogb(total)-51)
    // (one bit of slack keeps the claim rigorous); then the tree sum equals the reference's
    // index-order sum. Otherwise replay the reference order (kernels.cpp:80-85).
    const bool exact = total > 0.0 && lsb >= ilogb(total) - 51;
    if (!exact) {
        flags |= FRS_FLAG_SEQ_SUM;
        __syncthreads();
        if (tid == 0) {
            double acc = 0.0;
            for (int j = 0; j < v; ++j) acc += static_cast<double>(E[j]);
            red_d[0] = acc;
        }
        __syncthreads();
        total = red_d[0];
    }
    const float inv = __double2float_rn(1.0 / total);

    unsigned long long cand = 0ull;
    for (int j = tid; j < v; j += nt) {
        const unsigned long long key = prob_key(__fmul_rn(E[j], inv), j);
        cand = key > cand ? key : cand;
    }
    const int kk = min(k, v);
    for (int r = 0; r < kk; ++r) {
        const unsigned long long best = block_reduce(cand, MaxU64(), red_k);
        const int j = static_cast<int>(0xffffffffu - static_cast<uint32_t>(best & 0xffffffffull));
        if (tid == 0) {
            out_ridx[(size_t)row * k + r] = j;
            out_full[(size_t)row * k + r] = ordered ? ordered[j] : j;
            out_prob[(size_t)row * k + r] = __uint_as_float(static_cast<uint32_t>(best >> 32));
        }
        if (j % nt == tid) {  // owner rescans for its best key below `best`
            cand = 0ull;
            for (int jj = tid; jj < v; jj += nt) {
                const unsigned long long key = prob_key(__fmul_rn(E[jj], inv), jj);
                if (key < best && key > cand) cand = key;
            }
        }
    }
    if (tid == 0) {
        for (int r = kk; r < k; ++r) {
            out_ridx[(size_t)row * k + r] = -1;
            out_full[(size_t)row * k + r] = -1;
            out_prob[(size_t)row * k + r] = 0.0f;
        }
        if (out_rowmax) out_rowmax[row] = mx;
        if (out_total) out_total[row] = total;
        if (out_flags) out_flags[row] = flags;
    }
}

__device__ __forceinline__ uint32_t ordered_bits(float x) {
    if (x == 0.0f) x = 0.0f;  // -0 == +0 under the reference's '>' (kernels.cpp:119)
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_ordered(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// One CTA per row: argmax with ties to the lowest index (kernels.cpp:113-122).
__global__ void __launch_bounds__(1024)
    k_argmax_rows(const float *__restrict__ logits, int ld, int v, int32_t id_offset,
                  int32_t *__restrict__ out_id, float *__restrict__ out_val,
                  uint32_t *__restrict__ out_flags) {
    __shared__ unsigned long long red_k[32];
    __shared__ int red_i[32];
    const int row = blockIdx.x;
    const float *L = logits + (size_t)row * ld;
    unsigned long long cand = 0ull;
    int bad = 0;
    for (int j = threadIdx.x; j < v; j += blockDim.x) {
        const float x = L[j];
        if (!isfinite(x)) bad = 1;
        const unsigned long long key =
            (static_cast<unsigned long long>(ordered_bits(x)) << 32) | (0xffffffffu - static_cast<uint32_t>(j));
        cand = key > cand ? key : cand;
    }
    cand = block_reduce(cand, MaxU64(), red_k);
    bad = block_reduce(bad, OrI(), red_i);
    if (threadIdx.x == 0) {
        const int j = static_cast<int>(0xffffffffu - static_cast<uint32_t>(cand & 0xffffffffull));
        out_id[row] = id_offset + j;
        if (out_val) out_val[row] = L[j];
        if (out_flags) out_flags[row] = bad ? FRS_FLAG_NONFINITE : 0u;
    }
}

template <int NB, typename WT>
int launch_nb(frs_ctx *ctx, const float *h, int n, int d, const WT *W, int v_rows, float *logits,
              unsigned *counter, cudaStream_t s) {
    constexpr int NBS = (NB + 3) & ~3;
    const size_t smem = (size_t)(d & ~7) * NBS * sizeof(float);
    auto kern = k_exact_logits<NB, WT>;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FRS_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
    kern<<<ctx->sm_count, 1024, smem, s>>>(h, n, d, W, v_rows, logits, v_rows, counter);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

template <typename WT>
int launch_pass(frs_ctx *ctx, const float *h, int n, int d, const WT *W, int v_rows, float *logits,
                unsigned *counter, cudaStream_t s) {
    switch (n) {
#define FRS_NB_CASE(N) \
    case N: return launch_nb<N, WT>(ctx, h, n, d, W, v_rows, logits, counter, s);
        FRS_NB_CASE(1) FRS_NB_CASE(2) FRS_NB_CASE(3) FRS_NB_CASE(4) FRS_NB_CASE(5) FRS_NB_CASE(6)
        FRS_NB_CASE(7) FRS_NB_CASE(8) FRS_NB_CASE(9) FRS_NB_CASE(10) FRS_NB_CASE(11) FRS_NB_CASE(12)
#undef FRS_NB_CASE
        default: return fail(FRS_ENOTSUP, "exact logits: rows per pass must be 1..12");
    }
}

}  // namespace

int launch_exact_logits(frs_ctx *ctx, const float *h, int n, int d, const void *W, int w_dtype,
                        int v_rows, float *logits, cudaStream_t s) {
    // Rows per pass: as many as fit (<= 12) with the hidden rows resident in shared memory.
    const size_t per_row = (size_t)(d & ~7) * sizeof(float);
    int nb_cap = static_cast<int>(std::min<size_t>(12, ctx->smem_optin / std::max<size_t>(per_row, 1)));
    nb_cap &= ~3;
    if (nb_cap < 4) return fail(FRS_ENOTSUP, "exact logits: hidden_dim too large for shared memory");
    int st = ctx->counters.ensure(64 * sizeof(unsigned));
    if (st) return st;
    unsigned *counters = static_cast<unsigned *>(ctx->counters.ptr);
    int pass = 0;
    for (int r0 = 0; r0 < n; r0 += nb_cap, ++pass) {
        const int nb = std::min(nb_cap, n - r0);
        unsigned *counter = counters + (pass % 64);
        st = (w_dtype == FRS_DTYPE_BF16)
                 ? launch_pass(ctx, h + (size_t)r0 * d, nb, d, static_cast<const __nv_bfloat16 *>(W), v_rows,
                               logits + (size_t)r0 * v_rows, counter, s)
                 : launch_pass(ctx, h + (size_t)r0 * d, nb, d, static_cast<const float *>(W), v_rows,
                               logits + (size_t)r0 * v_rows, counter, s);
        if (st) return st;
    }
    return FRS_OK;
}

int launch_softmax_topk(frs_ctx *ctx, const float *logits, int n, int v, int k, float temperature,
                        const int32_t *ordered_ids, int32_t *out_ridx, int32_t *out_full,
                        float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags,
                        cudaStream_t s) {
    int st = ctx->scratch.ensure((size_t)n * v * sizeof(float));
    if (st) return st;
    k_softmax_topk<<<n, 1024, 0, s>>>(logits, v, v, k, temperature, ordered_ids,
                                      static_cast<float *>(ctx->scratch.ptr), out_ridx, out_full,
                                      out_prob, out_rowmax, out_total, out_flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int launch_argmax_rows(frs_ctx *ctx, const float *logits, int m, int v, int32_t id_offset,
                       int32_t *out_id, float *out_val, uint32_t *out_flags, cudaStream_t s) {
    (void)ctx;
    k_argmax_rows<<<m, 1024, 0, s>>>(logits, v, v, id_offset, out_id, out_val, out_flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

}  // namespace frs
