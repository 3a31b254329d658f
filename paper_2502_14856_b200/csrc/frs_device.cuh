// Device helpers shared by the EXACT and FAST kernels: the glibc expf port, order-preserving
// float keys, block reductions and the exact per-row softmax + top-k (kernels.cpp:62-122).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "frspec_cuda.h"

namespace frs {
namespace dev {

// ---- glibc 2.39 expf, FMA ifunc ----
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

// expf_glibc without the special-case branch (bit-identical for every input): the main path
// runs on x clamped into [-104, 89] (glibc's main path is valid on all of [-103.97, 88.72])
// and the special cases are selected afterwards, so several calls interleave freely.
__device__ __forceinline__ float expf_glibc_nb(float x, const unsigned long long *tab) {
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ffu;
    const float xc = fminf(fmaxf(x, -104.0f), 89.0f);
    const double xd = static_cast<double>(xc);
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
    float res = __double2float_rn(y);
    if (abstop >= 0x42bu) {  // selects, not a branch around the main path
        res = x < -0x1.9fe368p6f ? 0.0f : res;
        res = x > 0x1.62e42ep6f ? __int_as_float(0x7f800000) : res;
        res = abstop >= 0x7f8u ? x + x : res;
        res = ux == 0xff800000u ? 0.0f : res;
    }
    return res;
}

static __device__ const unsigned long long kExp2fTable[32] = {
        0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
        0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
        0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
        0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
        0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
        0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
        0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
        0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

__device__ __forceinline__ void load_exp_table(unsigned long long *tab) {
    if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTable[threadIdx.x];
}

// Exponent of the lowest set bit of a non-negative float (INT_MAX for 0).
__device__ __forceinline__ int lsb_exponent(float v) {
    const uint32_t b = __float_as_uint(v);
    const uint32_t ex = (b >> 23) & 0xffu;
    uint32_t m = b & 0x7fffffu;
    if (ex != 0) m |= 0x800000u;
    if (m == 0) return 0x7fffffff;
    return (ex != 0 ? static_cast<int>(ex) - 150 : -149) + (__ffs(m) - 1);
}

// Order-preserving map float -> uint32 (with -0 == +0, as under the reference's '>').
__device__ __forceinline__ uint32_t ordered_bits(float x) {
    if (x == 0.0f) x = 0.0f;
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_ordered(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
// (value desc, index asc) as one descending uint64 key; 0 is below every real key.
__device__ __forceinline__ unsigned long long value_key(float v, int idx) {
    return (static_cast<unsigned long long>(ordered_bits(v)) << 32) | (0xffffffffu - static_cast<uint32_t>(idx));
}
__device__ __forceinline__ int key_index(unsigned long long k) {
    return static_cast<int>(0xffffffffu - static_cast<uint32_t>(k & 0xffffffffull));
}
__device__ __forceinline__ float key_value(unsigned long long k) { return from_ordered(static_cast<uint32_t>(k >> 32)); }
// probabilities are >= +0: their raw bits already order them
__device__ __forceinline__ unsigned long long prob_key(float p, int j) {
    return (static_cast<unsigned long long>(__float_as_uint(p)) << 32) | (0xffffffffu - static_cast<uint32_t>(j));
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {  // serial over the (<= 32) warp partials: no identity element needed
        v = red[0];
        for (int w = 1; w < nw; ++w) v = op(v, red[w]);
        red[0] = v;
    }
    __syncthreads();
    return red[0];
}

struct MaxF { __device__ float operator()(float a, float b) const { return fmaxf(a, b); } };
struct SumD { __device__ double operator()(double a, double b) const { return a + b; } };
struct MinI { __device__ int operator()(int a, int b) const { return min(a, b); } };
struct OrI { __device__ int operator()(int a, int b) const { return a | b; } };
struct MaxU64 {
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a > b ? a : b; }
};

struct ReduceScratch {
    unsigned long long tab[32];
    double d[32];
    float f[32];
    int i[32];
    unsigned long long k[32];
};

// Calls f(j, p[j]) for j in [0, v) split over the block, with U loads in flight per thread:
// float4 loads when p is 16-byte aligned (each thread takes 4 consecutive j), else scalar.
// A one-load-per-iteration loop over an L2-resident row is latency-bound (~30 us per 32K).
template <int U, typename F>
__device__ __forceinline__ void row_pass(const float *p, int v, F &&f) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if ((reinterpret_cast<uintptr_t>(p) & 15u) == 0) {
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        const int v4 = v >> 2;
        for (int base = 0; base < v4; base += U * nt) {
            float4 b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = base + u * nt + tid;
                if (q < v4) b[u] = __ldcg(p4 + q);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = base + u * nt + tid;
                if (q < v4) {
                    f(4 * q, b[u].x);
                    f(4 * q + 1, b[u].y);
                    f(4 * q + 2, b[u].z);
                    f(4 * q + 3, b[u].w);
                }
            }
        }
        for (int j = 4 * v4 + tid; j < v; j += nt) f(j, __ldcg(p + j));
    } else {
        for (int base = 0; base < v; base += 4 * U * nt) {
            float b[4 * U];
#pragma unroll
            for (int u = 0; u < 4 * U; ++u) {
                const int j = base + u * nt + tid;
                if (j < v) b[u] = __ldcg(p + j);
            }
#pragma unroll
            for (int u = 0; u < 4 * U; ++u) {
                const int j = base + u * nt + tid;
                if (j < v) f(j, b[u]);
            }
        }
    }
}

// Exact softmax (kernels.cpp:62-91) + top-kk (kernels.cpp:93-111) + remap for ONE row whose
// exact logits are L[0..v): the whole block cooperates; E is a [v] float scratch. Writes
// out[0..k) (entries past min(k, v) get -1 / 0). Returns flags (thread 0's copy is valid).
// tree_total_ok (FAST fallback rows): ids and probabilities stay bit-exact but *out_total may
// be the tree sum (within v 2^-52 relative) when that pins the reference's 1 / total.
static __device__ __noinline__ uint32_t softmax_topk_row(const float *__restrict__ L, int v, int k,
                                                         float temperature, const int32_t *__restrict__ ordered,
                                                         float *__restrict__ E, int32_t *out_ridx, int32_t *out_full,
                                                         float *out_prob, float *out_rowmax, double *out_total,
                                                         ReduceScratch &rs, bool tree_total_ok = false,
                                                         unsigned long long *stamps = nullptr) {
    const int tid = threadIdx.x, nt = blockDim.x;
#define FRS_STAMP(q)                                                                                  \
    do {                                                                                              \
        if (stamps && tid == 0) {                                                                     \
            unsigned long long t_;                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
            stamps[q] = t_;                                                                           \
        }                                                                                             \
    } while (0)
    load_exp_table(rs.tab);
    float mx = -__int_as_float(0x7f800000);
    int bad = 0;
    const bool unit_t = temperature == 1.0f;  // x / 1 == x: skip the IEEE divisions
    row_pass<8>(L, v, [&](int, float x) {
        if (!isfinite(x)) bad = 1;
        const float y = unit_t ? x : __fdiv_rn(x, temperature);
        mx = (mx < y) ? y : mx;
    });
    mx = block_reduce(mx, MaxF(), rs.f);
    bad = block_reduce(bad, OrI(), rs.i);
    uint32_t flags = bad ? FRS_FLAG_NONFINITE : 0u;
    FRS_STAMP(0);

    double part = 0.0;
    int lsb = 0x7fffffff;
    row_pass<8>(L, v, [&](int j, float x) {
        const float e = expf_glibc(__fsub_rn(unit_t ? x : __fdiv_rn(x, temperature), mx), rs.tab);
        E[j] = e;
        part += static_cast<double>(e);
        lsb = min(lsb, lsb_exponent(e));
    });
    double total = block_reduce(part, SumD(), rs.d);
    lsb = block_reduce(lsb, MinI(), rs.i);
    FRS_STAMP(1);
    // Every partial sum (in any order) is exact iff all e_j are multiples of
    // 2^(ilogb(total)-51) (one bit of slack keeps it rigorous): then the tree sum equals the
    // reference's index-order sum. Otherwise replay the reference order (kernels.cpp:80-85).
    bool exact = total > 0.0 && lsb >= ilogb(total) - 51;
    if (!exact && tree_total_ok && total > 0.0) {
        // FAST fallback rows need the reference's inv = float(1 / total) exactly, not total
        // itself: the tree sum and the index-order sum both lie within gamma_v * S of the
        // exact sum S of v positive terms, so |tree - seq| <= v 2^-52 S (slack: 2 nt more),
        // and inv(x) = float(fl64(1 / x)) is monotone, so equal ends of the interval pin it.
        const double del = static_cast<double>(v + 2 * nt) * 0x1p-52;
        const double lo = __dmul_rd(total, 1.0 - del), hi = __dmul_ru(total, 1.0 + del);
        exact = __double2float_rn(1.0 / lo) == __double2float_rn(1.0 / hi);
    }
    if (!exact) {
        flags |= FRS_FLAG_SEQ_SUM;
        __syncthreads();
        if (tid == 0) {
            double acc = 0.0;
            for (int j = 0; j < v; ++j) acc += static_cast<double>(E[j]);
            rs.d[0] = acc;
        }
        __syncthreads();
        total = rs.d[0];
    }
    const float inv = __double2float_rn(1.0 / total);
    FRS_STAMP(2);

    // top-kk: every thread keeps its KL best keys (descending, 0 = empty); each round the
    // block max is popped from its owner's list, which rescans its slice below the popped key
    // only when the list runs dry while the slice held more than KL keys
    constexpr int KL = 4;
    unsigned long long lst[KL];
#pragma unroll
    for (int q = 0; q < KL; ++q) lst[q] = 0ull;
    int nmine = 0;
    __syncthreads();  // E written by other threads of the block
    row_pass<8>(E, v, [&](int j, float e) {
        unsigned long long key = prob_key(__fmul_rn(e, inv), j);
        ++nmine;
#pragma unroll
        for (int q = 0; q < KL; ++q) {  // insertion into the sorted list
            const unsigned long long o = lst[q];
            const bool gt = key > o;
            lst[q] = gt ? key : o;
            key = gt ? o : key;
        }
    });
    FRS_STAMP(3);
    int left = nmine;  // keys of this slice not yet popped
    const int kk = min(k, v);
    for (int r = 0; r < kk; ++r) {
        const unsigned long long best = block_reduce(lst[0], MaxU64(), rs.k);
        const int j = key_index(best);
        if (tid == 0) {
            out_ridx[r] = j;
            out_full[r] = ordered ? ordered[j] : j;
            out_prob[r] = __uint_as_float(static_cast<uint32_t>(best >> 32));
        }
        if (lst[0] == best) {  // the owner (keys are distinct: the index is part of the key)
#pragma unroll
            for (int q = 0; q + 1 < KL; ++q) lst[q] = lst[q + 1];
            lst[KL - 1] = 0ull;
            --left;
            if (lst[0] == 0ull && left > 0) {  // dry: rebuild from the slice below `best`
                // (this thread's slice only: row_pass's split is a function of tid, v and E's
                // alignment alone, so the scalar walk below visits the same j)
                const bool vec = (reinterpret_cast<uintptr_t>(E) & 15u) == 0;
                const int v4 = vec ? (v >> 2) : 0;
                auto take = [&](int jj) {
                    unsigned long long key = prob_key(__fmul_rn(E[jj], inv), jj);
                    if (key >= best) return;
#pragma unroll
                    for (int q = 0; q < KL; ++q) {
                        const unsigned long long o = lst[q];
                        const bool gt = key > o;
                        lst[q] = gt ? key : o;
                        key = gt ? o : key;
                    }
                };
                for (int q = tid; q < v4; q += nt)
                    for (int c = 0; c < 4; ++c) take(4 * q + c);
                for (int jj = 4 * v4 + tid; jj < v; jj += nt) take(jj);
            }
        }
    }
    FRS_STAMP(4);
#undef FRS_STAMP
    if (tid == 0) {
        for (int r = kk; r < k; ++r) {
            out_ridx[r] = -1;
            out_full[r] = -1;
            out_prob[r] = 0.0f;
        }
        if (out_rowmax) *out_rowmax = mx;
        if (out_total) *out_total = total;
    }
    return flags;
}

// Exact softmax probabilities of ONE row (kernels.cpp:62-91): P[j] = float(e_j) * inv with the
// reference's e_j (glibc expf) and inv = float(1 / total). inv is pinned as in
// softmax_topk_row(tree_total_ok): the tree sum brackets the index-order sum; the sequential
// replay runs only when the bracket straddles a float boundary. Whole block; returns flags.
static __device__ __noinline__ uint32_t softmax_probs_row(const float *__restrict__ L, int v, float temperature,
                                                          float *__restrict__ P, ReduceScratch &rs) {
    const int tid = threadIdx.x, nt = blockDim.x;
    load_exp_table(rs.tab);
    float mx = -__int_as_float(0x7f800000);
    int bad = 0;
    const bool unit_t = temperature == 1.0f;
    row_pass<8>(L, v, [&](int, float x) {
        if (!isfinite(x)) bad = 1;
        const float y = unit_t ? x : __fdiv_rn(x, temperature);
        mx = (mx < y) ? y : mx;
    });
    mx = block_reduce(mx, MaxF(), rs.f);
    bad = block_reduce(bad, OrI(), rs.i);
    uint32_t flags = bad ? FRS_FLAG_NONFINITE : 0u;
    double part = 0.0;
    int lsb = 0x7fffffff;
    row_pass<8>(L, v, [&](int j, float x) {
        const float e = expf_glibc(__fsub_rn(unit_t ? x : __fdiv_rn(x, temperature), mx), rs.tab);
        P[j] = e;
        part += static_cast<double>(e);
        lsb = min(lsb, lsb_exponent(e));
    });
    double total = block_reduce(part, SumD(), rs.d);
    lsb = block_reduce(lsb, MinI(), rs.i);
    bool exact = total > 0.0 && lsb >= ilogb(total) - 51;
    if (!exact && total > 0.0) {
        const double del = static_cast<double>(v + 2 * nt) * 0x1p-52;
        const double lo = __dmul_rd(total, 1.0 - del), hi = __dmul_ru(total, 1.0 + del);
        exact = __double2float_rn(1.0 / lo) == __double2float_rn(1.0 / hi);
    }
    if (!exact) {
        flags |= FRS_FLAG_SEQ_SUM;
        __syncthreads();
        if (tid == 0) {
            double acc = 0.0;
            for (int j = 0; j < v; ++j) acc += static_cast<double>(P[j]);
            rs.d[0] = acc;
        }
        __syncthreads();
        total = rs.d[0];
    }
    const float inv = __double2float_rn(1.0 / total);
    __syncthreads();
    for (int j = tid; j < v; j += nt) P[j] = __fmul_rn(P[j], inv);
    __syncthreads();
    return flags;
}

// Exact dot_f32 (kernels.cpp:13-32) of h (fp32) with a bf16/fp32 row, computed by the 8
// lanes l = threadIdx.x % 8 of an aligned 8-lane group; the result is valid in lane l == 0.
// Requires the 8 lanes of the group to be converged; d % 8 == 0 handled by the lane chains,
// the scalar tail by lane 0.
template <typename WT>
__device__ __forceinline__ float w_at(const WT *w, int i);
template <>
__device__ __forceinline__ float w_at<float>(const float *w, int i) { return w[i]; }
template <>
__device__ __forceinline__ float w_at<unsigned short>(const unsigned short *w, int i) {
    return __uint_as_float(static_cast<uint32_t>(w[i]) << 16);
}

template <typename WT>
__device__ __forceinline__ float dot_f32_lanes8(const float *h, const WT *w, int d) {
    const int l = threadIdx.x & 7;
    const int T = d >> 3;
    float s = 0.0f;
#pragma unroll 8
    for (int t = 0; t < T; ++t) s = __fadd_rn(s, __fmul_rn(h[8 * t + l], w_at(w, 8 * t + l)));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    if (l == 0)
        for (int e = 8 * T; e < d; ++e) s = __fadd_rn(s, __fmul_rn(h[e], w_at(w, e)));
    return s;
}

// Same arithmetic as dot_f32_lanes8 (bf16 row w in shared memory), with the operands of the
// next 16 steps loaded into registers while the current 16 dependent adds run: the chain is
// bound by the FADD latency (d/8 steps) instead of the shared-memory load latency.
__device__ __forceinline__ float dot_f32_lanes8_pf(const float *h, const unsigned short *w, int d) {
    const int l = threadIdx.x & 7;
    const int T = d >> 3;
    constexpr int B = 16;
    float hb[B], wb[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
        hb[u] = u < T ? h[8 * u + l] : 0.0f;
        wb[u] = u < T ? w_at(w, 8 * u + l) : 0.0f;
    }
    float s = 0.0f;
    for (int t0 = 0; t0 < T; t0 += B) {
        float hn[B], wn[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int t = t0 + B + u;
            hn[u] = t < T ? h[8 * t + l] : 0.0f;
            wn[u] = t < T ? w_at(w, 8 * t + l) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (t0 + u < T) s = __fadd_rn(s, __fmul_rn(hb[u], wb[u]));
#pragma unroll
        for (int u = 0; u < B; ++u) {
            hb[u] = hn[u];
            wb[u] = wn[u];
        }
    }
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
    if (l == 0)
        for (int e = 8 * T; e < d; ++e) s = __fadd_rn(s, __fmul_rn(h[e], w_at(w, e)));
    return s;
}

}  // namespace dev
}  // namespace frs
