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
// Exact logits: k_exact_gemv (below; operands staged by bulk copies through an mbarrier ring,
// one dot_f32 chain quad per lane) whenever d % 8 == 0 and the rows are 16-byte aligned, else
// k_exact_logits: one persistent CTA per SM (1024 threads) keeps the NB hidden rows resident in
// shared memory as sh[e*NBS + i] = h[i][e]; each warp pulls groups of 4 slab rows from an
// atomic work queue and maps lane = 8*q + l to (row q of the group, dot_f32 lane chain l). In
// both the chain order is the reference's exactly and the final tree has the reference's
// association. __fmul_rn/__fadd_rn keep ptxas from contracting into FFMA (2 FP32 instructions
// per MAC).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <string>

#include "frs_common.cuh"
#include "frs_device.cuh"

namespace frs {
namespace {

__device__ __forceinline__ float load_w(const float *p) { return __ldg(p); }
__device__ __forceinline__ float load_w(const __nv_bfloat16 *p) {
    const unsigned short u = __ldg(reinterpret_cast<const unsigned short *>(p));
    return __uint_as_float(static_cast<uint32_t>(u) << 16);  // bf16 -> fp32 is exact
}

// masked_attention (kernels.cpp:124-171), every head of a multi-head layer in two grids, K and
// V each read once per (head, query-row block) instead of once per (query row, head):
//  k_attn_scores  grid (heads, key blocks of 64, query-row blocks of 32): the q tile and the k
//                 tile in shared memory (k rows padded by 4 floats: the 16-byte reads of 8
//                 consecutive keys hit distinct banks); one thread per (row, key) dot carries
//                 the 8 dot_f32 lane chains (kernels.cpp:13-32: index order per chain, then
//                 ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)), then the scalar tail), times the
//                 reference's 1/sqrtf(dh); scores of masked pairs are never written.
//  k_attn_pv      grid (heads, 32-column slices of the values, query-row blocks): per row (one
//                 warp) mx over the allowed keys, e_j = expf(s_j - mx) (glibc port), the double
//                 Σ in index order pinned by bracketing a tree sum (replayed sequentially only
//                 when the bracket straddles a float boundary of 1/Σ), p_j = e_j * float(1/Σ);
//                 then one thread per (row, column) adds p_j * v_jc in key order over the allowed
//                 keys (kernels.cpp:162-167) from 64-key value chunks staged in shared memory.
//                 Rows with no allowed key: zeros and FRS_FLAG_EMPTY_ROW (the reference throws).
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
constexpr int kAttnKeyBlk = 64;   // keys per score tile (one mask word)
constexpr int kAttnRowBlk = 32;   // query rows per score tile
constexpr int kAttnCols = 32;     // value columns per PV CTA

__global__ void __launch_bounds__(256)
    k_attn_scores(const float *__restrict__ q, int q_ld, const float *__restrict__ k, int k_ld,
                  const unsigned long long *__restrict__ mask, int n, int m, int dh, float scale,
                  float *__restrict__ S) {
    extern __shared__ float s_att[];
    const int hd = blockIdx.x, j0 = blockIdx.y * kAttnKeyBlk, r0 = blockIdx.z * kAttnRowBlk;
    const int nk = min(kAttnKeyBlk, m - j0), nr = min(kAttnRowBlk, n - r0);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int pitch = ((dh + 3) & ~3) + 4;  // floats; pitch % 8 == 4 for 16-byte reads of 8 rows
    float *sq = s_att, *sk = sq + (size_t)kAttnRowBlk * pitch;
    q += (size_t)hd * dh;
    k += (size_t)hd * dh;
    const bool vec = (dh & 3) == 0 && (q_ld & 3) == 0 && (k_ld & 3) == 0 &&
                     ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k)) & 15) == 0;
    if (vec) {  // every tile word requested at once (cp.async, 16 bytes)
        const int d4 = dh >> 2;
        for (int e = tid; e < nr * d4; e += nt) {
            const int r = e / d4, c = (e - r * d4) * 4;
            cp_async16(sq + r * pitch + c, q + (size_t)(r0 + r) * q_ld + c);
        }
        for (int e = tid; e < nk * d4; e += nt) {
            const int j = e / d4, c = (e - j * d4) * 4;
            cp_async16(sk + j * pitch + c, k + (size_t)(j0 + j) * k_ld + c);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
        for (int e = tid; e < nr * dh; e += nt) {
            const int r = e / dh, c = e - r * dh;
            sq[r * pitch + c] = q[(size_t)(r0 + r) * q_ld + c];
        }
        for (int e = tid; e < nk * dh; e += nt) {
            const int j = e / dh, c = e - j * dh;
            sk[j * pitch + c] = k[(size_t)(j0 + j) * k_ld + c];
        }
    }
    __syncthreads();
    const int stride = (m + 63) >> 6, D8 = dh & ~7;
    for (int p = tid; p < nr * kAttnKeyBlk; p += nt) {
        const int r = p / kAttnKeyBlk, j = p - r * kAttnKeyBlk;  // consecutive threads: consecutive keys
        if (j >= nk) continue;
        const int gr = r0 + r, gj = j0 + j;
        if (!((mask[(size_t)gr * stride + (gj >> 6)] >> (gj & 63)) & 1ull)) continue;
        const float *qa = sq + r * pitch, *ka = sk + j * pitch;
        float c8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int t = 0; t < D8; t += 8) {
            const float4 x0 = *reinterpret_cast<const float4 *>(qa + t), x1 = *reinterpret_cast<const float4 *>(qa + t + 4);
            const float4 y0 = *reinterpret_cast<const float4 *>(ka + t), y1 = *reinterpret_cast<const float4 *>(ka + t + 4);
            c8[0] = __fadd_rn(c8[0], __fmul_rn(x0.x, y0.x));
            c8[1] = __fadd_rn(c8[1], __fmul_rn(x0.y, y0.y));
            c8[2] = __fadd_rn(c8[2], __fmul_rn(x0.z, y0.z));
            c8[3] = __fadd_rn(c8[3], __fmul_rn(x0.w, y0.w));
            c8[4] = __fadd_rn(c8[4], __fmul_rn(x1.x, y1.x));
            c8[5] = __fadd_rn(c8[5], __fmul_rn(x1.y, y1.y));
            c8[6] = __fadd_rn(c8[6], __fmul_rn(x1.z, y1.z));
            c8[7] = __fadd_rn(c8[7], __fmul_rn(x1.w, y1.w));
        }
        float dot = __fadd_rn(__fadd_rn(__fadd_rn(c8[0], c8[1]), __fadd_rn(c8[2], c8[3])),
                              __fadd_rn(__fadd_rn(c8[4], c8[5]), __fadd_rn(c8[6], c8[7])));
        for (int t = D8; t < dh; ++t) dot = __fadd_rn(dot, __fmul_rn(qa[t], ka[t]));  // kernels.cpp:28-30
        S[((size_t)hd * n + gr) * m + gj] = __fmul_rn(dot, scale);
    }
}

__global__ void __launch_bounds__(512)
    k_attn_pv(const float *__restrict__ S, const float *__restrict__ v, int v_ld,
              const unsigned long long *__restrict__ mask, int n, int m, int dv, int rows_per_cta, int whole,
              float *__restrict__ out, int out_ld, uint32_t *__restrict__ flags) {
    extern __shared__ float s_pv[];
    __shared__ unsigned long long s_tab[32];
    const int hd = blockIdx.x, c0 = blockIdx.y * kAttnCols, r0 = blockIdx.z * rows_per_cta;
    const int nr = min(rows_per_cta, n - r0), nc = min(kAttnCols, dv - c0);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    const int stride = (m + 63) >> 6;
    float *P = s_pv;                                  // [rows_per_cta][m] probabilities
    float *sv = P + (((size_t)rows_per_cta * m + 3) & ~size_t(3));  // [whole ? m : 64][kAttnCols] values (16-B aligned)
    __shared__ uint32_t s_rowflag[16];
    if (tid < 32) s_tab[tid] = dev::kExp2fTable[tid];
    // the whole value slice requested before the softmax when it fits (vec_all): its loads
    // overlap the softmax instead of one round trip per 64-key chunk
    const bool vec_all = whole && nc == kAttnCols && (v_ld & 3) == 0 && (dv & 3) == 0 &&
                         (reinterpret_cast<uintptr_t>(v) & 15) == 0;
    // the rows' scores into P (masked entries are stale, never read), all requests in flight
    for (int e = tid; e < nr * m; e += blockDim.x) {
        const int r = e / m, j = e - r * m;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(
                         __cvta_generic_to_shared(P + (size_t)r * m + j))),
                     "l"(S + ((size_t)hd * n + r0 + r) * m + j)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (vec_all) {
        const float *vb = v + (size_t)hd * dv + c0;
        for (int e = tid; e < m * (kAttnCols / 4); e += blockDim.x) {
            const int j = e / (kAttnCols / 4), c = (e - j * (kAttnCols / 4)) * 4;
            cp_async16(sv + (size_t)j * kAttnCols + c, vb + (size_t)j * v_ld + c);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // the scores; the values may still be in flight
    __syncthreads();
    // ---- softmax per row (one warp per row)
    for (int r = warp; r < nr; r += nw) {
        const int gr = r0 + r;
        const unsigned long long *words = mask + (size_t)gr * stride;
        float *Pr = P + (size_t)r * m;
        const float *Sr = Pr;  // the row's scores, staged above (overwritten in place below)
        float mx = -__int_as_float(0x7f800000);
        int any = 0;
        for (int j = lane; j < m; j += 32)
            if ((words[j >> 6] >> (j & 63)) & 1ull) {
                mx = fmaxf(mx, Sr[j]);
                any = 1;
            }
        mx = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(mx)));
        any = __any_sync(0xffffffffu, any);
        uint32_t fl = 0;
        if (!any) {
            fl = FRS_FLAG_EMPTY_ROW;
            for (int j = lane; j < m; j += 32) Pr[j] = 0.0f;
        } else {
            double part = 0.0;
            int lsb = 0x7fffffff;
            for (int j = lane; j < m; j += 32) {
                float e = 0.0f;
                if ((words[j >> 6] >> (j & 63)) & 1ull) {
                    e = dev::expf_glibc(__fsub_rn(Sr[j], mx), s_tab);
                    part += static_cast<double>(e);
                    lsb = min(lsb, dev::lsb_exponent(e));
                }
                Pr[j] = e;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                part += __shfl_xor_sync(0xffffffffu, part, o);
                lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
            }
            double total = part;
            // every partial sum exact (all terms multiples of 2^(ilogb(total) - 51)): the tree sum
            // is the index-order sum; else bracket the index-order sum around it (both within
            // (m + 64) 2^-52 of the exact sum) and pin float(1 / total) from the two ends
            bool exact = total > 0.0 && lsb >= ilogb(total) - 51;
            if (!exact && total > 0.0) {
                const double del = static_cast<double>(m + 64) * 0x1p-52;
                const double lo = __dmul_rd(total, 1.0 - del), hi = __dmul_ru(total, 1.0 + del);
                exact = __double2float_rn(1.0 / lo) == __double2float_rn(1.0 / hi);
            }
            __syncwarp();
            if (!exact) {  // replay the reference's index order (kernels.cpp:155-159)
                fl |= FRS_FLAG_SEQ_SUM;
                double acc = 0.0;
                if (lane == 0)
                    for (int j = 0; j < m; ++j)
                        if ((words[j >> 6] >> (j & 63)) & 1ull) acc += static_cast<double>(Pr[j]);
                total = __shfl_sync(0xffffffffu, acc, 0);
            }
            const float inv = __double2float_rn(1.0 / total);
            for (int j = lane; j < m; j += 32) Pr[j] = __fmul_rn(Pr[j], inv);  // masked e are 0: never added
        }
        if (lane == 0) s_rowflag[r] = fl;
    }
    __syncthreads();
    // ---- key-ordered accumulation, one thread per (row, column)
    const int rr = tid / kAttnCols, cc = tid - rr * kAttnCols;
    float acc = 0.0f;
    const unsigned long long *wr = mask + (size_t)(r0 + min(rr, nr - 1)) * stride;
    if (vec_all) asm volatile("cp.async.wait_all;" ::: "memory");
    for (int j0 = 0; j0 < m; j0 += 64) {
        const int nk = min(64, m - j0);
        const float *svc = vec_all ? sv + (size_t)j0 * kAttnCols : sv;
        if (!vec_all) {
            __syncthreads();  // the previous chunk's readers are done
            for (int e = tid; e < nk * kAttnCols; e += blockDim.x) {
                const int j = e / kAttnCols, c = e - j * kAttnCols;
                sv[e] = c < nc ? __ldg(v + (size_t)(j0 + j) * v_ld + (size_t)hd * dv + c0 + c) : 0.0f;
            }
        }
        __syncthreads();
        if (rr < nr) {
            const unsigned long long bits = wr[j0 >> 6];
            const float *Pr = P + (size_t)rr * m + j0;
            int jj = 0;
            if (nk == 64 && bits == ~0ull) {  // every key of the chunk allowed (the causal context):
                // the reference adds every product, so no per-key mask test (3x fewer instructions)
                for (; jj < 64; jj += 8) {
                    float pr[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) pr[e] = __fmul_rn(Pr[jj + e], svc[(jj + e) * kAttnCols + cc]);
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, pr[e]);
                }
            }
            for (; jj + 8 <= nk; jj += 8) {  // products ahead of the predicated, key-ordered adds
                float pr[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) pr[e] = __fmul_rn(Pr[jj + e], svc[(jj + e) * kAttnCols + cc]);
                // a masked key adds +0.0: an exact no-op (acc starts at +0 and a round-to-nearest
                // sum is never -0 unless both addends are), and the select keeps a non-finite value
                // of a masked key out — the same result as the reference's skip, without branches
#pragma unroll
                for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, ((bits >> (jj + e)) & 1ull) ? pr[e] : 0.0f);
            }
            for (; jj < nk; ++jj)
                acc = __fadd_rn(acc, ((bits >> jj) & 1ull) ? __fmul_rn(Pr[jj], svc[jj * kAttnCols + cc]) : 0.0f);
        }
    }
    if (rr < nr && cc < nc) out[(size_t)(r0 + rr) * out_ld + (size_t)hd * dv + c0 + cc] = acc;
    if (blockIdx.y == 0 && tid < nr && s_rowflag[tid]) atomicOr(flags + r0 + tid, s_rowflag[tid]);
}

// One CTA per row: the exact softmax probabilities (kernels.cpp:62-91) of full-vocabulary
// target logits (verify_stochastic's Residual::init, verification.cpp:80-87); flags per row.
__global__ void __launch_bounds__(1024)
    k_softmax_probs_rows(const float *__restrict__ logits, int v, float temperature, float *__restrict__ probs,
                         uint32_t *__restrict__ out_flags) {
    __shared__ dev::ReduceScratch rs;
    const int row = blockIdx.x;
    const uint32_t flags = dev::softmax_probs_row(logits + (size_t)row * v, v, temperature, probs + (size_t)row * v, rs);
    if (threadIdx.x == 0) out_flags[row] = flags;
}

// Sampled pick_children (drafting.cpp:44-74) for each row: exact probabilities (kernels.cpp:
// 62-91, softmax_probs_row) into probs[row], then w draws without replacement with the caller's
// uniforms (std::uniform_real_distribution<double> of the reference's mt19937_64, in draw
// order). The reference sums work[] sequentially in double each draw and scans for the first
// running sum above u = uni * total; here the prefix is a block scan of per-thread chunk sums,
// and every decision is certified: the tree prefix P_i and the index-order acc_i differ by at
// most eb = (v + 2048 + 64 w) 2^-52 T, so the pick is certain when the first i with
// P_i + eb > u_lo equals the first with P_i - eb > u_hi (u's own bracket from T +- eb). An
// uncertain draw (or the reference's upper-edge guard) stops the row with
// FRS_FLAG_SAMPLE_UNCERTIFIED: the host replays that level from the probabilities.
// The w certified draws of one row (drafting.cpp:44-74) by a block of NT threads over the
// draw weights Wk[0..v) (= the row's probabilities; drawn entries are zeroed), uniforms in
// s_uni (first 64) / uniforms. Returns the flags to OR in and the number of draws made.
template <int NT>
__device__ uint32_t sample_draws(float *Wk, int v, int w, int row, const double *s_uni,
                                 const double *__restrict__ uniforms, const int32_t *__restrict__ ordered,
                                 int32_t *__restrict__ out_ridx, int32_t *__restrict__ out_full,
                                 float *__restrict__ out_prob, int &count) {
    __shared__ double s_cp[NT];
    __shared__ int s_pick, s_pchunk;
    __shared__ float s_pval;
    const int tid = threadIdx.x, lane = tid & 31;
    const int C = (v + NT - 1) / NT, j0 = min(v, tid * C), j1 = min(v, j0 + C);
    // Prefix bookkeeping: a fresh scan (chunk sums of C terms + a log2(NT)-deep block scan, all
    // terms positive) is within errP = (C + log2 NT + 2) 2^-52 T of the exact prefix; each later
    // pick is subtracted in place (one rounding each, errP grows by 2^-52 T). The reference's
    // running sums are within (v + 64) 2^-53 T of the exact ones. Rescan when the remaining mass
    // halves, so the bounds stay relative to it.
    int lg = 0;
    while ((1 << lg) < NT) ++lg;
    double errP = 0.0, t_scan = 0.0;
    bool need_scan = true;
    uint32_t flags = 0u;
    count = 0;
    for (int k = 0; k < w; ++k) {
        if (need_scan) {
            double cs = 0.0;
            // the chunk sum in a lane-rotated order (any order is within errP): chunks are
            // C floats apart, so lane l starting at offset l keeps the 32 lanes on distinct banks
            const int cnt = j1 - j0;
            for (int i = 0; i < cnt; ++i) {
                int o = i + lane;
                o = o >= cnt ? o - cnt : o;
                o = o >= cnt ? o % cnt : o;
                cs += static_cast<double>(Wk[j0 + o]);
            }
            __syncthreads();  // readers of the previous s_cp are done
            s_cp[tid] = cs;
            __syncthreads();
            for (int off = 1; off < NT; off <<= 1) {  // inclusive scan of the chunk sums
                double x = s_cp[tid];
                if (tid >= off) x += s_cp[tid - off];
                __syncthreads();
                s_cp[tid] = x;
                __syncthreads();
            }
            t_scan = s_cp[NT - 1];
            errP = t_scan * static_cast<double>(C + lg + 2) * 0x1p-52;
            need_scan = false;
        }
        const double T = s_cp[NT - 1];
        if (!(T > 0.0)) break;  // all mass drawn: the reference breaks (total <= 0)
        if (tid < 32) {
            const double uni = k < 64 ? s_uni[k] : uniforms[(size_t)row * w + k];
            const double eb = errP + static_cast<double>(v + 64) * 0x1p-53 * T;
            const double u_lo = __dmul_rd(uni, T - eb), u_hi = __dmul_ru(uni, T + eb);
            // first chunk with CP + eb > u_lo, first with CP - eb > u_hi (CP is non-decreasing)
            int c_lo = NT, c_hi = NT;
            for (int c0 = 0; c0 < NT; c0 += 32) {
                const double cp = s_cp[c0 + lane];
                const unsigned bl = __ballot_sync(0xffffffffu, cp + eb > u_lo);
                const unsigned bh = __ballot_sync(0xffffffffu, cp - eb > u_hi);
                if (c_lo == NT && bl) c_lo = c0 + __ffs(bl) - 1;
                if (c_hi == NT && bh) c_hi = c0 + __ffs(bh) - 1;
                if (c_hi != NT) break;
            }
            int pick = -1;
            if (c_lo == c_hi && c_hi < NT) {  // inside chunk c: element prefixes base + warp scan
                const int c = c_lo, e0 = min(v, c * C), e1 = min(v, e0 + C);
                double base = c > 0 ? s_cp[c - 1] : 0.0;
                int i_lo = -1, i_hi = -1;
                for (int p0 = e0; p0 < e1 && i_hi < 0; p0 += 32) {
                    const int j = p0 + lane;
                    double x = j < e1 ? static_cast<double>(Wk[j]) : 0.0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    const double pj = base + x;
                    const unsigned bl = __ballot_sync(0xffffffffu, j < e1 && pj + eb > u_lo);
                    const unsigned bh = __ballot_sync(0xffffffffu, j < e1 && pj - eb > u_hi);
                    if (i_lo < 0 && bl) i_lo = p0 + __ffs(bl) - 1;
                    if (i_hi < 0 && bh) i_hi = p0 + __ffs(bh) - 1;
                    base += __shfl_sync(0xffffffffu, x, 31);
                }
                if (i_lo >= 0 && i_lo == i_hi) pick = i_lo;
            }
            if (lane == 0) {
                s_pick = pick;
                s_pchunk = c_lo;
                if (pick >= 0) {  // Wk[pick] is still P[pick]: only drawn entries are zeroed
                    const float pv = Wk[pick];
                    s_pval = pv;
                    out_ridx[(size_t)row * w + k] = pick;
                    out_full[(size_t)row * w + k] = ordered ? ordered[pick] : pick;
                    out_prob[(size_t)row * w + k] = pv;
                    Wk[pick] = 0.0f;
                }
            }
        }
        __syncthreads();
        if (s_pick < 0) {  // uncertain (or the reference's upper-edge guard): the host replays
            flags |= FRS_FLAG_SAMPLE_UNCERTIFIED;
            break;
        }
        ++count;
        // subtract the drawn mass from the prefixes at and after its chunk
        if (tid >= s_pchunk) s_cp[tid] -= static_cast<double>(s_pval);
        errP += T * 0x1p-52;
        __syncthreads();
        need_scan = s_cp[NT - 1] < 0.5 * t_scan;
    }
    return flags;
}

// Sampled pick_children (drafting.cpp:44-74) for each row: exact probabilities (kernels.cpp:
// 62-91, softmax_probs_row) into probs[row], then w draws without replacement with the caller's
// uniforms (std::uniform_real_distribution<double> of the reference's mt19937_64, in draw
// order). The reference sums work[] sequentially in double each draw and scans for the first
// running sum above u = uni * total; here the prefix is a block scan of per-thread chunk sums,
// and every decision is certified: the tree prefix P_i and the index-order acc_i differ by at
// most eb = errP + (v + 64) 2^-53 T, so the pick is certain when the first i with P_i + eb > u_lo
// equals the first with P_i - eb > u_hi (u's own bracket from T +- eb). An uncertain draw (or
// the reference's upper-edge guard) stops the row with FRS_FLAG_SAMPLE_UNCERTIFIED: the host
// replays that level from the probabilities. One CTA per row (rows longer than the cluster
// kernel takes, or k_softmax_sample_cl unavailable).
__global__ void __launch_bounds__(1024)
    k_softmax_sample(const float *__restrict__ logits, int v, float temperature, const double *__restrict__ uniforms,
                     int w, const int32_t *__restrict__ ordered, float *__restrict__ probs, float *__restrict__ work,
                     int32_t *__restrict__ out_ridx, int32_t *__restrict__ out_full, float *__restrict__ out_prob,
                     int32_t *__restrict__ out_count, uint32_t *__restrict__ out_flags, int wk_in_smem) {
    __shared__ dev::ReduceScratch rs;
    extern __shared__ float s_wk[];  // the draw weights when v floats fit (wk_in_smem)
    const int row = blockIdx.x, tid = threadIdx.x;
    const float *L = logits + (size_t)row * v;
    float *P = probs + (size_t)row * v, *Wk = wk_in_smem ? s_wk : work + (size_t)row * v;
    __shared__ double s_uni[64];  // this row's uniforms, read once
    if (tid < min(w, 64)) s_uni[tid] = uniforms[(size_t)row * w + tid];
    uint32_t flags;
    if (wk_in_smem) {  // probabilities straight into the draw weights, written out alongside
        flags = dev::softmax_probs_row(L, v, temperature, Wk, rs);
        for (int j = tid; j < v; j += 1024) P[j] = Wk[j];
    } else {
        // work = probs (coalesced: the chunk sums and the draws read other threads' chunks)
        flags = dev::softmax_probs_row(L, v, temperature, P, rs);
        for (int j = tid; j < v; j += 1024) Wk[j] = P[j];
        __syncthreads();
    }
    int count = 0;
    flags |= sample_draws<1024>(Wk, v, w, row, s_uni, uniforms, ordered, out_ridx, out_full, out_prob, count);
    if (tid == 0) {
        out_count[row] = count;
        if (out_flags) out_flags[row] = flags;
    }
}

template <int NB, typename WT>
__global__ void __launch_bounds__(1024, 1)
    k_exact_logits(const float *__restrict__ h, int n, int d, const WT *__restrict__ W, int v_rows,
                   float *__restrict__ logits, int ld, unsigned *__restrict__ counter) {
    constexpr int NBS = NB <= 2 ? NB : (NB + 3) & ~3;  // 1-2 rows: unpadded (wide inputs)
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
                float hv[NBS];
                if constexpr (NBS < 4) {
#pragma unroll
                    for (int c = 0; c < NBS; ++c) hv[c] = sh[((t + u) * 8 + l) * NBS + c];
                }
                const float4 *hp = reinterpret_cast<const float4 *>(sh + ((t + u) * 8 + l) * NBS);
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

// One CTA per row: exact softmax + top-k + remap (dev::softmax_topk_row). The probabilities
// and ids are always the reference's; the index-order double Σ itself (kernels.cpp:80-85) is
// replayed sequentially (one thread, ~40 us at V_sub 32768) only when the caller asks for it
// (out_total): otherwise 1 / Σ is pinned by bracketing the tree sum.
__global__ void __launch_bounds__(1024)
    k_softmax_topk(const float *__restrict__ logits, int ld, int v, int k, float temperature,
                   const int32_t *__restrict__ ordered, float *__restrict__ ework, int32_t *__restrict__ out_ridx,
                   int32_t *__restrict__ out_full, float *__restrict__ out_prob, float *__restrict__ out_rowmax,
                   double *__restrict__ out_total, uint32_t *__restrict__ out_flags) {
    __shared__ dev::ReduceScratch rs;
    const int row = blockIdx.x;
    const uint32_t flags = dev::softmax_topk_row(
        logits + (size_t)row * ld, v, k, temperature, ordered, ework + (size_t)row * ld, out_ridx + (size_t)row * k,
        out_full + (size_t)row * k, out_prob + (size_t)row * k, out_rowmax ? out_rowmax + row : nullptr,
        out_total ? out_total + row : nullptr, rs, /*tree_total_ok=*/out_total == nullptr);
    if (threadIdx.x == 0 && out_flags) out_flags[row] = flags;
}

// Same results as k_softmax_topk with out_total == nullptr, each row split over a cluster of
// kSmC CTAs (kSmNT threads, KL logits per thread, all loaded at once): the glibc expf work is
// FP64-throughput bound, so one CTA per row left 138 SMs idle for the 10-row draft levels of a
// tree (64 us per level). The row max and the (p, lsb) partials travel by DSMEM stores into
// every CTA (each CTA folds the kSmC values in rank order, so all agree bit for bit); 1 / Σ is
// pinned exactly as in softmax_topk_row(tree_total_ok); top-k runs as warp pops -> CTA merge
// of the warps' sorted lists -> the leader's merge of the CTAs' lists (pushed into its shared
// memory). The keys (prob desc, index asc) are a total order, so the union's top-k is exact.
constexpr int kSmC = 8, kSmNT = 512, kSmNW = kSmNT / 32, kSmKMax = 16;

__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(const void *p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(a)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(rank));
    return a;
}
__device__ __forceinline__ void cl_st(uint32_t a, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t a, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t a, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}

// Phase A of the cluster kernels: this CTA's slice [lo, hi) of the row (KL logits per thread,
// j = lo + q kSmNT + tid) -> x[q] = e_j = expf(y_j - max) (also written to E, the row's global
// scratch, for the index-order replay), the row max, 1 / Σ pinned as in
// softmax_topk_row(tree_total_ok), and the flags — identical in every CTA of the cluster.
struct ClSoftmax {
    float mx, inv;
    uint32_t flags;
};
template <int KL>
__device__ __forceinline__ ClSoftmax cl_softmax(const float *__restrict__ L, float *__restrict__ E, int v, int lo,
                                                int hi, float temperature, uint32_t r, float (&x)[KL]) {
    __shared__ unsigned long long s_tab[32];
    __shared__ float s_wmx[kSmNW], s_cmx[kSmC];
    __shared__ int s_wi[kSmNW], s_ci[kSmC], s_cbad[kSmC];
    __shared__ double s_wd[kSmNW], s_cd[kSmC], s_seq;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool unit_t = temperature == 1.0f;
    dev::load_exp_table(s_tab);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // logits from the previous kernel (PDL)
#pragma unroll
    for (int q = 0; q < KL; ++q) {
        const int j = lo + q * kSmNT + tid;
        x[q] = j < hi ? __ldcg(L + j) : 0.0f;
    }
    // row max (kernels.cpp:66-75): NaN never wins under either comparison, so any order agrees
    float mx = -__int_as_float(0x7f800000);
    int bad = 0;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
        if (lo + q * kSmNT + tid < hi) {
            if (!isfinite(x[q])) bad = 1;
            x[q] = unit_t ? x[q] : __fdiv_rn(x[q], temperature);
            mx = (mx < x[q]) ? x[q] : mx;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        s_wmx[warp] = mx;
        s_wi[warp] = bad;
    }
    __syncthreads();
    if (tid < kSmC) {  // push this CTA's (max, bad) into CTA tid
        float m = s_wmx[0];
        int b = s_wi[0];
        for (int w = 1; w < kSmNW; ++w) {
            m = fmaxf(m, s_wmx[w]);
            b |= s_wi[w];
        }
        cl_st(cl_map(&s_cmx[r], tid), m);
        cl_st(cl_map(&s_cbad[r], tid), b);
    }
    cl_sync();
    mx = s_cmx[0];
    bad = s_cbad[0];
    for (int c = 1; c < kSmC; ++c) {
        mx = fmaxf(mx, s_cmx[c]);
        bad |= s_cbad[c];
    }
    uint32_t flags = bad ? FRS_FLAG_NONFINITE : 0u;

    // e_j = expf(y_j - max) and the double partial sums (kernels.cpp:76-85)
    double part = 0.0;
    int lsb = 0x7fffffff;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
        const int j = lo + q * kSmNT + tid;
        if (j < hi) {
            const float e = dev::expf_glibc(__fsub_rn(x[q], mx), s_tab);
            x[q] = e;
            E[j] = e;
            part += static_cast<double>(e);
            lsb = min(lsb, dev::lsb_exponent(e));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        part += __shfl_xor_sync(0xffffffffu, part, o);
        lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
    }
    if (lane == 0) {
        s_wd[warp] = part;
        s_wi[warp] = lsb;
    }
    __syncthreads();
    if (tid < kSmC) {
        double p = s_wd[0];
        int l = s_wi[0];
        for (int w = 1; w < kSmNW; ++w) {
            p += s_wd[w];
            l = min(l, s_wi[w]);
        }
        cl_st(cl_map(&s_cd[r], tid), p);
        cl_st(cl_map(&s_ci[r], tid), l);
    }
    cl_sync();
    double total = s_cd[0];
    lsb = s_ci[0];
    for (int c = 1; c < kSmC; ++c) {
        total += s_cd[c];
        lsb = min(lsb, s_ci[c]);
    }
    // 1 / Σ pinned as in softmax_topk_row(tree_total_ok): the same decision in every CTA
    bool exact = total > 0.0 && lsb >= ilogb(total) - 51;
    if (!exact && total > 0.0) {
        const double del = static_cast<double>(v + 2 * kSmC * kSmNT) * 0x1p-52;
        const double lo_ = __dmul_rd(total, 1.0 - del), hi_ = __dmul_ru(total, 1.0 + del);
        exact = __double2float_rn(1.0 / lo_) == __double2float_rn(1.0 / hi_);
    }
    if (!exact) {  // index-order replay by the leader over the row's e_j (global, cluster-visible)
        flags |= FRS_FLAG_SEQ_SUM;
        if (r == 0 && tid == 0) {
            double acc = 0.0;
            for (int j = 0; j < v; ++j) acc += static_cast<double>(__ldcg(E + j));
            for (int c = 0; c < kSmC; ++c) cl_st(cl_map(&s_seq, c), acc);
        }
        cl_sync();
        total = s_seq;
    }
    return ClSoftmax{mx, __double2float_rn(1.0 / total), flags};
}

template <int KL>
__global__ void __launch_bounds__(kSmNT)
    k_softmax_topk_cl(const float *__restrict__ logits, int ld, int v, int k, float temperature,
                      const int32_t *__restrict__ ordered, float *__restrict__ ework, int32_t *__restrict__ out_ridx,
                      int32_t *__restrict__ out_full, float *__restrict__ out_prob, float *__restrict__ out_rowmax,
                      uint32_t *__restrict__ out_flags) {
    __shared__ unsigned long long s_wtop[kSmNW][kSmKMax], s_all[kSmC][kSmKMax];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t r = cl_rank();
    const int row = blockIdx.x / kSmC;
    const int chunk = ((v + kSmC - 1) / kSmC + 3) & ~3;  // host: chunk <= KL * kSmNT
    const int lo = static_cast<int>(r) * chunk, hi = min(v, lo + chunk);
    float x[KL];
    const ClSoftmax sm = cl_softmax<KL>(logits + (size_t)row * ld, ework + (size_t)row * ld, v, lo, hi, temperature,
                                        r, x);
    const float mx = sm.mx, inv = sm.inv;
    const uint32_t flags = sm.flags;

    // top-kk: sorted per-thread lists -> warp pops -> CTA merge -> leader merge
    const int kk = min(k, v);
    unsigned long long lst[KL];
#pragma unroll
    for (int q = 0; q < KL; ++q) lst[q] = 0ull;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
        const int j = lo + q * kSmNT + tid;
        if (j < hi) {
            unsigned long long key = dev::prob_key(__fmul_rn(x[q], inv), j);
#pragma unroll
            for (int u = 0; u < KL; ++u) {
                const unsigned long long o = lst[u];
                const bool gt = key > o;
                lst[u] = gt ? key : o;
                key = gt ? o : key;
            }
        }
    }
    for (int rr = 0; rr < kk; ++rr) {
        unsigned long long best = lst[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        if (lst[0] == best) {  // the owner (keys are distinct; empty lanes shift zeros)
#pragma unroll
            for (int u = 0; u + 1 < KL; ++u) lst[u] = lst[u + 1];
            lst[KL - 1] = 0ull;
        }
        if (lane == 0) s_wtop[warp][rr] = best;
    }
    __syncthreads();
    if (warp == 0) {  // merge the kSmNW sorted warp lists; push the CTA's top-kk to the leader
        int p = 0;
        for (int rr = 0; rr < kk; ++rr) {
            const unsigned long long cur = (lane < kSmNW && p < kk) ? s_wtop[lane][p] : 0ull;
            unsigned long long best = cur;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                best = t > best ? t : best;
            }
            if (lane < kSmNW && cur == best) ++p;
            if (lane == 0) cl_st(cl_map(&s_all[r][rr], 0), best);
        }
    }
    cl_sync();
    if (r != 0 || warp != 0) return;  // no DSMEM access after this point
    int p = 0;
    for (int rr = 0; rr < kk; ++rr) {
        const unsigned long long cur = (lane < kSmC && p < kk) ? s_all[lane][p] : 0ull;
        unsigned long long best = cur;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
            best = t > best ? t : best;
        }
        if (lane < kSmC && cur == best) ++p;
        if (lane == 0) {
            const int j = dev::key_index(best);
            out_ridx[(size_t)row * k + rr] = j;
            out_full[(size_t)row * k + rr] = ordered ? ordered[j] : j;
            out_prob[(size_t)row * k + rr] = __uint_as_float(static_cast<uint32_t>(best >> 32));
        }
    }
    if (lane == 0) {
        for (int rr = kk; rr < k; ++rr) {
            out_ridx[(size_t)row * k + rr] = -1;
            out_full[(size_t)row * k + rr] = -1;
            out_prob[(size_t)row * k + rr] = 0.0f;
        }
        if (out_rowmax) out_rowmax[row] = mx;
        if (out_flags) out_flags[row] = flags;
    }
}

// k_softmax_sample with each row's softmax split over a cluster of kSmC CTAs (cl_softmax: the
// FP64 expf work on 8 SMs instead of 1); every CTA writes its slice's probabilities to probs and
// into the leader's shared draw weights (DSMEM stores), then the leader alone runs the w
// certified draws (sample_draws<kSmNT>). Same outputs as k_softmax_sample.
template <int KL>
__global__ void __launch_bounds__(kSmNT)
    k_softmax_sample_cl(const float *__restrict__ logits, int v, float temperature,
                        const double *__restrict__ uniforms, int w, const int32_t *__restrict__ ordered,
                        float *__restrict__ probs, float *__restrict__ ework, int32_t *__restrict__ out_ridx,
                        int32_t *__restrict__ out_full, float *__restrict__ out_prob, int32_t *__restrict__ out_count,
                        uint32_t *__restrict__ out_flags) {
    extern __shared__ float s_wk[];  // [v]: the leader's draw weights
    __shared__ double s_uni[64];
    const int tid = threadIdx.x;
    const uint32_t r = cl_rank();
    const int row = blockIdx.x / kSmC;
    const int chunk = ((v + kSmC - 1) / kSmC + 3) & ~3;  // host: chunk <= KL * kSmNT
    const int lo = static_cast<int>(r) * chunk, hi = min(v, lo + chunk);
    if (r == 0 && tid < min(w, 64)) s_uni[tid] = uniforms[(size_t)row * w + tid];
    float x[KL];
    const ClSoftmax sm = cl_softmax<KL>(logits + (size_t)row * v, ework + (size_t)row * v, v, lo, hi, temperature,
                                        r, x);
    float *P = probs + (size_t)row * v;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
        const int j = lo + q * kSmNT + tid;
        if (j < hi) {
            const float p = __fmul_rn(x[q], sm.inv);  // kernels.cpp:86-89
            P[j] = p;
            cl_st(cl_map(&s_wk[j], 0), p);
        }
    }
    cl_sync();
    if (r != 0) return;  // no DSMEM access after this point
    int count = 0;
    const uint32_t f =
        sample_draws<kSmNT>(s_wk, v, w, row, s_uni, uniforms, ordered, out_ridx, out_full, out_prob, count);
    if (tid == 0) {
        out_count[row] = count;
        if (out_flags) out_flags[row] = sm.flags | f;
    }
}

// One CTA per row: argmax with ties to the lowest index (kernels.cpp:113-122).
__global__ void __launch_bounds__(1024)
    k_argmax_rows(const float *__restrict__ logits, int ld, int v, int32_t id_offset, int32_t *__restrict__ out_id,
                  float *__restrict__ out_val, uint32_t *__restrict__ out_flags) {
    __shared__ unsigned long long red_k[32];
    __shared__ int red_i[32];
    const int row = blockIdx.x;
    const float *L = logits + (size_t)row * ld;
    unsigned long long cand = 0ull;
    int bad = 0;
    for (int j = threadIdx.x; j < v; j += blockDim.x) {
        const float x = L[j];
        if (!isfinite(x)) bad = 1;
        const unsigned long long key = dev::value_key(x, j);
        cand = key > cand ? key : cand;
    }
    cand = dev::block_reduce(cand, dev::MaxU64(), red_k);
    bad = dev::block_reduce(bad, dev::OrI(), red_i);
    if (threadIdx.x == 0) {
        const int j = dev::key_index(cand);
        out_id[row] = id_offset + j;
        if (out_val) out_val[row] = L[j];
        if (out_flags) out_flags[row] = bad ? FRS_FLAG_NONFINITE : 0u;
    }
}

template <int NB, typename WT>
int launch_nb(frs_ctx *ctx, const float *h, int n, int d, const WT *W, int v_rows, float *logits, unsigned *counter,
              cudaStream_t s) {
    constexpr int NBS = NB <= 2 ? NB : (NB + 3) & ~3;
    const size_t smem = (size_t)(d & ~7) * NBS * sizeof(float);
    auto kern = k_exact_logits<NB, WT>;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FRS_CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
    kern<<<ctx->sm_count, 1024, smem, s>>>(h, n, d, W, v_rows, logits, v_rows, counter);
    ++ctx->launches;
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

template <typename WT>
int launch_pass(frs_ctx *ctx, const float *h, int n, int d, const WT *W, int v_rows, float *logits, unsigned *counter,
                cudaStream_t s) {
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

namespace {
// Wide inputs (fewer than 4 rows fit in shared memory, e.g. the 4d-wide MLP down projection):
// one 8-lane group per (row, output), the hidden row read from global memory (L1 / L2), the
// same dot_f32 arithmetic (dev::dot_f32_lanes8, kernels.cpp:13-32).
template <typename WT>
__global__ void __launch_bounds__(256)
    k_exact_logits_wide(const float *__restrict__ h, int n, int d, const WT *__restrict__ W, int v_rows,
                        float *__restrict__ logits) {
    const long long groups = (long long)n * v_rows;
    const int per_block = blockDim.x >> 3;
    for (long long base = (long long)blockIdx.x * per_block; base < groups; base += (long long)gridDim.x * per_block) {
        const long long g = base + (threadIdx.x >> 3);  // block-uniform trip count: whole warps in the dot
        const long long gg = g < groups ? g : groups - 1;
        const int i = static_cast<int>(gg / v_rows), j = static_cast<int>(gg % v_rows);
        const float v = dev::dot_f32_lanes8(h + (size_t)i * d, W + (size_t)j * d, d);
        if ((threadIdx.x & 7) == 0 && g < groups) logits[(size_t)i * v_rows + j] = v;
    }
}
// ------------------------------------------- staged exact GEMV, short row ranges (round 1 kernel)
// Kept for matrices with fewer than 2 x SMs 32-row groups (the draft layer's 4096-row
// projections): rows split into ceil(V / SMs)-row blocks so every SM has work (4096 x 4096 fp32
// at n = 10: 33.5 us vs 50 us for k_exact_gemv's one 32-row group per CTA).
// The same dot_f32 arithmetic with the operands staged in shared memory by bulk copies
// (cp.async.bulk + mbarrier ring) instead of per-thread loads, so the stream does not depend
// on how many warps have rows to work on: a 4096-row projection at d = 4096 gives the
// per-thread-load kernel 1024 busy warps out of 4736 (~0.8 TB/s); here every SM streams its
// rows through a 4-6 stage ring (~100 KB in flight per SM).
//  * CTA = one producer warp + 2 S consumer warps (S = ceil(n / 2) slices of 2 hidden rows).
//    A block is RB <= 32 consecutive W rows; K is cut into KC-element chunks (rows chunk W[r,
//    c KC .. +KC) and h[i, c KC .. +KC), one bulk copy per row; row pitch KC + 8 elements so
//    the 128-bit (fp32) / 64-bit (bf16) reads of 4 rows x 2 lanes hit distinct banks).
//  * consumer lane = (row rl = 16 (warp & 1) + lane / 2, chain quad cq = lane & 1): it owns
//    the dot_f32 lane chains 4 cq .. 4 cq + 3 (kernels.cpp:19-26: s_l += a*b over indices = l
//    mod 8) of its 2 hidden rows and walks the chunks in index order, so every chain's
//    sequence of rounded mul / add is the reference's; the final tree ((s0+s1)+(s2+s3)) +
//    ((s4+s5)+(s6+s7)) (kernels.cpp:27) is one xor-1 shuffle. Requires d % 8 == 0 (no scalar
//    tail) and 16-byte aligned rows.
// Bound: FP32 issue (2 instructions per MAC) for n >= ~6 at fp32 weights; HBM below.
namespace gv1 {
constexpr int KC = 256;     // k elements per chunk
constexpr int RBMAX = 32;   // W rows per block
constexpr int NMAX = 16;    // hidden rows per launch
constexpr int PAD = 8;      // row pitch padding (elements)
__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GW_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void lds4(const float *p, float (&w)[4]) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
}
__device__ __forceinline__ void lds4(const unsigned short *p, float (&w)[4]) {
    const uint2 v = *reinterpret_cast<const uint2 *>(p);  // bf16 -> fp32 is exact
    w[0] = __uint_as_float(v.x << 16), w[1] = __uint_as_float(v.x & 0xffff0000u);
    w[2] = __uint_as_float(v.y << 16), w[3] = __uint_as_float(v.y & 0xffff0000u);
}
}  // namespace gv1

template <typename WT>
__global__ void __launch_bounds__(32 + 64 * (gv1::NMAX / 2))
    k_exact_gemv_rb(const float *__restrict__ h, int n, int d, const WT *__restrict__ W, int v_rows, int rb, int nblocks,
                 int stages, float *__restrict__ logits, int ld) {
    using namespace gv1;
    extern __shared__ __align__(128) unsigned char g_smem[];
    const int S = (n + 1) >> 1;
    const int pitch = KC + PAD;
    const size_t w_bytes = (size_t)RBMAX * pitch * sizeof(WT);
    const size_t h_bytes = (size_t)(2 * S) * KC * sizeof(float);
    const size_t st_bytes = (w_bytes + h_bytes + 127) & ~size_t(127);
    uint64_t *full = reinterpret_cast<uint64_t *>(g_smem + st_bytes * stages);
    uint64_t *empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nchunks = (d + KC - 1) / KC;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 2 * S * 32);  // every consumer lane releases its own reads
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {  // producer
        uint64_t pol_w, pol_h;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_h));
        int it = 0;
        for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
            const int r0 = blk * rb, nr = min(rb, v_rows - r0);
            for (int c = 0; c < nchunks; ++c, ++it) {
                const int st = it % stages;
                const uint32_t ph = (it / stages) & 1;
                const int k0 = c * KC, kc = min(KC, d - k0);
                bar_wait(&empty[st], ph ^ 1);
                unsigned char *base = g_smem + st_bytes * st;
                if (lane == 0) bar_expect(&full[st], (uint32_t)((nr * sizeof(WT) + n * sizeof(float)) * kc));
                __syncwarp();
                if (lane < nr)
                    g2s(reinterpret_cast<WT *>(base) + (size_t)lane * pitch, W + (size_t)(r0 + lane) * d + k0,
                        (uint32_t)(kc * sizeof(WT)), &full[st], pol_w);
                if (lane < n)
                    g2s(reinterpret_cast<float *>(base + w_bytes) + (size_t)lane * KC, h + (size_t)lane * d + k0,
                        (uint32_t)(kc * sizeof(float)), &full[st], pol_h);
            }
        }
        return;
    }
    const int cw = warp - 1, slice = cw >> 1;
    const int rl = 16 * (cw & 1) + (lane >> 1), cq = lane & 1;
    const int i0 = 2 * slice;
    int it = 0;
    for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
        const int r0 = blk * rb;
        float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
        for (int c = 0; c < nchunks; ++c, ++it) {
            const int st = it % stages;
            const uint32_t ph = (it / stages) & 1;
            const int kc = min(KC, d - c * KC);
            bar_wait(&full[st], ph);
            const unsigned char *base = g_smem + st_bytes * st;
            const WT *wr = reinterpret_cast<const WT *>(base) + (size_t)rl * pitch + 4 * cq;
            const float *h0 = reinterpret_cast<const float *>(base + w_bytes) + (size_t)i0 * KC + 4 * cq;
            const float *h1 = h0 + KC;
            const int T = kc >> 3;
            int t = 0;
            for (; t + 4 <= T; t += 4) {
                float w[4][4], x[4][4], y[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    gv1::lds4(wr + (t + u) * 8, w[u]);
                    gv1::lds4(h0 + (t + u) * 8, x[u]);
                    gv1::lds4(h1 + (t + u) * 8, y[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        a0[j] = __fadd_rn(a0[j], __fmul_rn(x[u][j], w[u][j]));
                        a1[j] = __fadd_rn(a1[j], __fmul_rn(y[u][j], w[u][j]));
                    }
            }
            for (; t < T; ++t) {
                float w[4], x[4], y[4];
                gv1::lds4(wr + t * 8, w);
                gv1::lds4(h0 + t * 8, x);
                gv1::lds4(h1 + t * 8, y);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    a0[j] = __fadd_rn(a0[j], __fmul_rn(x[j], w[j]));
                    a1[j] = __fadd_rn(a1[j], __fmul_rn(y[j], w[j]));
                }
            }
            bar_arrive(&empty[st]);
        }
        // ((s0+s1)+(s2+s3)) + ((s4+s5)+(s6+s7)): cq 0 holds s0..s3, cq 1 holds s4..s7
        float q0 = __fadd_rn(__fadd_rn(a0[0], a0[1]), __fadd_rn(a0[2], a0[3]));
        float q1 = __fadd_rn(__fadd_rn(a1[0], a1[1]), __fadd_rn(a1[2], a1[3]));
        const float p0 = __shfl_xor_sync(0xffffffffu, q0, 1), p1 = __shfl_xor_sync(0xffffffffu, q1, 1);
        const int row = r0 + rl;
        if (cq == 0 && rl < rb && row < v_rows) {
            if (i0 < n) logits[(size_t)i0 * ld + row] = __fadd_rn(q0, p0);
            if (i0 + 1 < n) logits[(size_t)(i0 + 1) * ld + row] = __fadd_rn(q1, p1);
        }
    }
}

template <typename WT>
int launch_gemv_rb(frs_ctx *ctx, const float *h, int n, int d, const WT *W, int v_rows, float *logits, int ld,
                cudaStream_t s) {
    using namespace gv1;
    const int S = (n + 1) / 2;
    const size_t st_bytes = (((size_t)RBMAX * (KC + PAD) * sizeof(WT) + (size_t)(2 * S) * KC * sizeof(float)) + 127) &
                            ~size_t(127);
    const size_t budget = std::min<size_t>(ctx->smem_optin, 220 * 1024) - 2 * 8 * 8;
    const int stages = static_cast<int>(std::min<size_t>(8, budget / st_bytes));
    if (stages < 2) return fail(FRS_ENOTSUP, "exact gemv: shared memory too small");
    const int G = ctx->sm_count;
    const int rounds = (v_rows + G * RBMAX - 1) / (G * RBMAX);
    const int rb = (v_rows + G * rounds - 1) / (G * rounds);
    const int nblocks = (v_rows + rb - 1) / rb;
    const size_t smem = st_bytes * stages + 2 * stages * sizeof(uint64_t);
    auto kern = k_exact_gemv_rb<WT>;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++ctx->launches;
    kern<<<std::min(G, nblocks), 32 + 64 * S, smem, s>>>(h, n, d, W, v_rows, rb, nblocks, stages, logits, ld);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}


// ---------------------------------------------------------------- staged exact GEMV
// The reference's dot_f32 (kernels.cpp:13-32) for every (hidden row, W row) pair on CUDA cores,
// operands staged in shared memory by TMA (cp.async.bulk.tensor) through an mbarrier ring.
//  * Persistent grid, one CTA per SM. W rows come in 32-row groups; CTA c owns the groups
//    [c NG / G, (c+1) NG / G) and walks them in blocks of RW groups (one row warp per group),
//    each block in KC-element chunks (256 B of every W row per chunk): per chunk one TMA box of
//    32 rows x 128 B per (group, 128-byte panel), SWIZZLE_128B (16-byte chunk c of row r lands
//    at c ^ (r & 7), so the 16-byte reads of 8 consecutive rows hit distinct banks), and one
//    box [n rows x KC] of the hidden rows (dense, read as warp-uniform broadcasts). Per-row
//    bulk copies cost ~100 cycles of TMA issue each (measured: 256 B copies ran at 0.55 TB/s);
//    the boxes move 4 KB per request.
//  * Consumer thread = (W row of the block, hidden group hg): it owns ALL 8 lane chains of its
//    W row for the nrg hidden rows of its group (8 nrg accumulators). Per 8-element step it
//    reads its W row's 8 words once and each hidden row's 8 words once, then does 8 nrg
//    rounded multiplies + rounded adds: every chain sees the reference's sequence s_l += a*b
//    over indices = l mod 8 in index order; the final ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7)) is
//    in-thread. __fmul_rn / __fadd_rn keep ptxas from fusing (2 FP32 instructions per MAC).
//  * Warps = RW x HG, hidden groups of nrg <= NRT rows (NRT = template register tile).
// Requires d % 8 == 0 (no scalar tail) and 16-byte aligned rows / row strides; other shapes
// take k_exact_logits.
#ifndef FRS_GEMV_UNROLL
#define FRS_GEMV_UNROLL 4  // steps per unrolled loop body (1 / 2 / 4: 140 / 143 / 135 us at C2)
#endif
constexpr int kGemvUnroll = FRS_GEMV_UNROLL;
namespace gv {
constexpr int NPASS = 32;   // hidden rows per launch
constexpr int GROUP = 32;   // W rows per TMA box (one row warp)
constexpr int PANEL = 128;  // bytes per TMA box row (SWIZZLE_128B)
constexpr int BOX = GROUP * PANEL;
__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "GW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GW_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(b)), "l"(pol)
        : "memory");
}
// 8 consecutive W words (fp32 widening of bf16 is exact) at 16-byte chunks c0, c1 of a row
__device__ __forceinline__ void ldw8(const unsigned char *row, int c, int sw, const float *, float (&w)[8]) {
    const float4 a = *reinterpret_cast<const float4 *>(row + (((2 * c) ^ sw) << 4));
    const float4 b = *reinterpret_cast<const float4 *>(row + (((2 * c + 1) ^ sw) << 4));
    w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w, w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
}
__device__ __forceinline__ void ldw8(const unsigned char *row, int c, int sw, const unsigned short *, float (&w)[8]) {
    const uint4 v = *reinterpret_cast<const uint4 *>(row + ((c ^ sw) << 4));
    w[0] = __uint_as_float(v.x << 16), w[1] = __uint_as_float(v.x & 0xffff0000u);
    w[2] = __uint_as_float(v.y << 16), w[3] = __uint_as_float(v.y & 0xffff0000u);
    w[4] = __uint_as_float(v.z << 16), w[5] = __uint_as_float(v.z & 0xffff0000u);
    w[6] = __uint_as_float(v.w << 16), w[7] = __uint_as_float(v.w & 0xffff0000u);
}
__device__ __forceinline__ void ldh8(const float *p, float (&x)[8]) {
    const float4 a = reinterpret_cast<const float4 *>(p)[0], b = reinterpret_cast<const float4 *>(p)[1];
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
}
constexpr int MAXW = 16;  // consumer warps per CTA
// register estimate (accumulators + one step's W and h words + addressing), for the warp budget
constexpr int regs_of(int nrt, int jt) { return (8 * nrt * jt + 8 * jt + 8 + 64 + 7) & ~7; }
// most consumer warps whose registers fit (warps are allocated per scheduler in fours)
constexpr int maxw_of(int nrt, int jt) {
    for (int w = MAXW; w > 1; --w)
        if (((w + 1 + 3) / 4) * 32 * regs_of(nrt, jt) <= 16384) return w;
    return 1;
}
template <typename WT> constexpr int kc_of() { return 256 / (int)sizeof(WT); }  // 2 panels per row per chunk
}  // namespace gv

template <typename WT, int NRT, int JT>
__global__ void __launch_bounds__(32 + 32 * gv::maxw_of(NRT, JT), 1)
    k_exact_gemv(const __grid_constant__ CUtensorMap w_map, const __grid_constant__ CUtensorMap h_map, int h_row0,
                 int n, int d, int v_rows, int RW, int HG, int stages, float *__restrict__ logits, int ld) {
    using namespace gv;
    constexpr int KC = kc_of<WT>();
    constexpr int P = KC * (int)sizeof(WT) / PANEL;       // panels per chunk
    constexpr int SPP = PANEL / (8 * (int)sizeof(WT));     // 8-element steps per panel
    extern __shared__ __align__(1024) unsigned char g_smem[];
    // 1024-byte aligned for SWIZZLE_128B; pointer arithmetic on g_smem keeps the shared window (LDS)
    unsigned char *smem = g_smem + ((1024u - (su32(g_smem) & 1023u)) & 1023u);
    const int GB = RW * JT;  // 32-row groups per block
    const size_t w_bytes = (size_t)GB * P * BOX;
    const size_t st_bytes = (w_bytes + (size_t)HG * NRT * KC * sizeof(float) + 1023) & ~size_t(1023);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + st_bytes * stages);
    uint64_t *empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cwarps = (blockDim.x >> 5) - 1;
    const int nchunks = (d + KC - 1) / KC;
    const int NG = (v_rows + GROUP - 1) / GROUP;
    const int g_begin = static_cast<int>((long long)blockIdx.x * NG / gridDim.x);
    const int g_end = static_cast<int>((long long)(blockIdx.x + 1) * NG / gridDim.x);
    const int nblk = (g_end - g_begin + GB - 1) / GB;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], cwarps);  // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {  // producer: one elected lane
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&w_map)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&h_map)) : "memory");
            uint64_t pol_w, pol_h;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_h));
            int it = 0;
            for (int b = 0; b < nblk; ++b) {
                const int g0 = g_begin + b * GB, ng = min(GB, g_end - g0);
                for (int c = 0; c < nchunks; ++c, ++it) {
                    const int st = it % stages;
                    const uint32_t ph = (it / stages) & 1;
                    bar_wait(&empty[st], ph ^ 1);
                    unsigned char *base = smem + st_bytes * st;
                    // full boxes always land (OOB rows / columns are zero-filled and counted)
                    bar_expect(&full[st], (uint32_t)(ng * P * BOX + n * KC * sizeof(float)));
                    for (int g = 0; g < ng; ++g)
                        for (int p = 0; p < P; ++p)
                            tma2d(base + (size_t)(g * P + p) * BOX, &w_map, c * KC + p * (PANEL / (int)sizeof(WT)),
                                  (g0 + g) * GROUP, &full[st], pol_w);
                    tma2d(base + w_bytes, &h_map, c * KC, h_row0, &full[st], pol_h);
                }
            }
        }
        return;
    }
    const int cw = warp - 1, hg = cw / RW, rw = cw - hg * RW;
    const int i0 = hg * NRT, nr_t = min(NRT, n - i0);  // this warp's hidden rows
    const int sw = lane & 7;
    int it = 0;
    for (int b = 0; b < nblk; ++b) {
        const int gw = g_begin + b * GB + rw * JT;  // this warp's first group
        float acc[JT][NRT][8];
#pragma unroll
        for (int j = 0; j < JT; ++j)
#pragma unroll
            for (int i = 0; i < NRT; ++i)
#pragma unroll
                for (int l = 0; l < 8; ++l) acc[j][i][l] = 0.0f;
        for (int c = 0; c < nchunks; ++c, ++it) {
            const int st = it % stages;
            const uint32_t ph = (it / stages) & 1;
            const int T = min(KC, d - c * KC) >> 3;
            bar_wait(&full[st], ph);
            const unsigned char *base = smem + st_bytes * st;
            const unsigned char *wb = base + (size_t)rw * JT * P * BOX + lane * PANEL;
            const float *hb = reinterpret_cast<const float *>(base + w_bytes) + (size_t)i0 * KC;
            if (gw < g_end) {  // a second group past g_end computes on stale words, never stored
#pragma unroll kGemvUnroll
                for (int t = 0; t < T; ++t) {
                    const int p = t / SPP, cc = t - p * SPP;
                    float w[JT][8];
#pragma unroll
                    for (int j = 0; j < JT; ++j)
                        ldw8(wb + (size_t)(j * P + p) * BOX, cc, sw, static_cast<const WT *>(nullptr), w[j]);
#pragma unroll
                    for (int i = 0; i < NRT; ++i) {  // rows past n (last group) compute on padding, never stored
                        float x[8];
                        ldh8(hb + (size_t)i * KC + 8 * t, x);
#pragma unroll
                        for (int j = 0; j < JT; ++j)
#pragma unroll
                            for (int l = 0; l < 8; ++l)
                                acc[j][i][l] = __fadd_rn(acc[j][i][l], __fmul_rn(x[l], w[j][l]));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&empty[st]);
        }
#pragma unroll
        for (int j = 0; j < JT; ++j) {
            const int row = (gw + j) * GROUP + lane;
            if (gw + j < g_end && row < v_rows) {
#pragma unroll
                for (int i = 0; i < NRT; ++i)
                    if (i < nr_t) {
                        const float(&a)[8] = acc[j][i];
                        const float s = __fadd_rn(__fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3])),
                                                  __fadd_rn(__fadd_rn(a[4], a[5]), __fadd_rn(a[6], a[7])));
                        logits[(size_t)(i0 + i) * ld + row] = s;
                    }
            }
        }
    }
}

bool gemv_enabled() {
    static const int on = [] {
        const char *e = std::getenv("FRS_EXACT_GEMV");
        return e ? std::atoi(e) : 1;
    }();
    return on != 0;
}

PFN_cuTensorMapEncodeTiled_v12000 gemv_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2D row-major [rows x cols] map, box [box_rows x box_cols]
int gemv_map(CUtensorMap *map, const void *base, bool bf16, long long rows, long long cols, long long row_stride_elems,
             int box_cols, int box_rows, bool swizzle) {
    auto fn = gemv_encode_fn();
    if (!fn) return fail(FRS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const int es = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems) * es};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FRS_ECUDA, "exact gemv: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return FRS_OK;
}

struct GemvCfg {
    int nrt, jt, rw, hg;
};

// (JT W rows x NRT hidden rows) per thread, RW row warps, HG hidden groups: the configuration
// with the least estimated issue time per SM (FP 2 per MAC incl. padding rows / groups, W and h
// shared-memory reads, bf16 widening; x 8 / warps below 8 warps for latency), register budget
// permitting.
GemvCfg gemv_cfg(int n, int d, int v_rows, int G, bool bf16) {
    const int groups = (v_rows + gv::GROUP - 1) / gv::GROUP;
    const int gpc = std::max(1, (groups + G - 1) / G);
    GemvCfg best{1, 1, 1, 1};
    double best_t = 1e300;
    static const int force_jt = [] {  // A/B override (FRS_GEMV_JT=1|2)
        const char *e = std::getenv("FRS_GEMV_JT");
        return e ? std::atoi(e) : 0;
    }();
    // Two W rows per thread halve the h broadcasts per MAC and double the independent work per
    // load: measured faster once a CTA owns >= 6 row groups (C2 slab 143 vs 163 us; verify passes
    // 462 vs 509 us), slower on short ranges (16384 x 4096 fp32: 102 vs 94 us), which the issue
    // model alone does not see (it has no load-latency term).
    const int jt_only = force_jt ? force_jt : (gpc >= 6 ? 2 : 1);
    for (int jt = 1; jt <= 2; ++jt)
        for (int hg = 1; hg <= std::min(n, gv::MAXW); ++hg) {
            if (jt != jt_only) continue;
            const int nrt = (n + hg - 1) / hg;
            if (nrt > (jt == 1 ? 16 : 8)) continue;
            for (int rw = 1; rw <= 8; ++rw) {
                const int warps = rw * hg;
                if (warps > gv::maxw_of(nrt, jt)) continue;
                if (rw > 1 && (rw - 1) * jt >= gpc) continue;  // a whole row warp idle
                {  // two ring stages must fit (launch_gemv_t's budget): wide row groups with few
                   // hidden rows (short d, small n) would otherwise pick an unlaunchable ring
                    const size_t kc = bf16 ? 128 : 64;
                    const size_t stb = ((size_t)rw * jt * 2 * gv::BOX + (size_t)hg * nrt * kc * 4 + 1023) & ~size_t(1023);
                    if (2 * stb > (size_t)227 * 1024 - 1024 - 2 * 8 * 8) continue;  // sm_100 opt-in limit
                }
                const int gb = rw * jt, nblk = (gpc + gb - 1) / gb;
                const double per_step = 16.0 * nrt * jt + jt * (bf16 ? 9 : 2) + 2.0 * nrt + 4;  // instructions
                const double wavefronts = jt * (bf16 ? 4.0 : 8.0) + 4.0 * nrt;  // h: 2 broadcast LDS.128 per row
                double t = (double)nblk * warps * (d / 8) * std::max(per_step / 4.0, wavefronts);
                if (warps < 8) t *= 8.0 / warps;
                if (t < best_t * 0.999) best_t = t, best = GemvCfg{nrt, jt, rw, hg};
            }
        }
    return best;
}

template <typename WT, int NRT, int JT>
int launch_gemv_t(frs_ctx *ctx, const GemvCfg &c, const CUtensorMap &wm, const CUtensorMap &hm, int h_row0, int n,
                  int d, int v_rows, float *logits, int ld, cudaStream_t s) {
    using namespace gv;
    constexpr int KC = kc_of<WT>();
    constexpr int P = KC * (int)sizeof(WT) / PANEL;
    const size_t st_bytes =
        ((size_t)c.rw * JT * P * BOX + (size_t)c.hg * NRT * KC * sizeof(float) + 1023) & ~size_t(1023);
    const size_t budget = std::min<size_t>(ctx->smem_optin, 227 * 1024) - 1024 - 2 * 8 * 8;
    const int stages = static_cast<int>(std::min<size_t>(8, budget / st_bytes));
    if (stages < 2) return fail(FRS_ENOTSUP, "exact gemv: shared memory too small");
    const size_t smem = 1024 + st_bytes * stages + 2 * stages * sizeof(uint64_t);
    auto kern = k_exact_gemv<WT, NRT, JT>;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ++ctx->launches;
    const int groups = (v_rows + GROUP - 1) / GROUP;
    kern<<<std::min(ctx->sm_count, groups), 32 + 32 * c.rw * c.hg, smem, s>>>(wm, hm, h_row0, n, d, v_rows, c.rw,
                                                                             c.hg, stages, logits, ld);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

// One launch per pass of <= NPASS hidden rows; h [n_total x d] fp32, W [v_rows x d].
template <typename WT>
int launch_gemv(frs_ctx *ctx, const float *h, int n_total, int d, const WT *W, int v_rows, float *logits, int ld,
                cudaStream_t s) {
    using namespace gv;
    constexpr int KC = kc_of<WT>();
    CUtensorMap wm, hm;
    int st = gemv_map(&wm, W, sizeof(WT) == 2, v_rows, d, d, PANEL / (int)sizeof(WT), GROUP, true);
    if (st) return st;
    for (int r0 = 0; r0 < n_total && !st; r0 += NPASS) {
        const int n = std::min(NPASS, n_total - r0);
        if ((st = gemv_map(&hm, h, false, n_total, d, d, KC, n, false))) return st;
        const GemvCfg c = gemv_cfg(n, d, v_rows, std::min(ctx->sm_count, (v_rows + GROUP - 1) / GROUP),
                                   sizeof(WT) == 2);
        float *out = logits + (size_t)r0 * ld;
        if (c.jt == 1) {
            switch (c.nrt) {
            case 2: st = launch_gemv_t<WT, 2, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 3: st = launch_gemv_t<WT, 3, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 4: st = launch_gemv_t<WT, 4, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 5: st = launch_gemv_t<WT, 5, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 6: st = launch_gemv_t<WT, 6, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 7: st = launch_gemv_t<WT, 7, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 8: st = launch_gemv_t<WT, 8, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 9: st = launch_gemv_t<WT, 9, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 10: st = launch_gemv_t<WT, 10, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 11: st = launch_gemv_t<WT, 11, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 12: st = launch_gemv_t<WT, 12, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 13: st = launch_gemv_t<WT, 13, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 14: st = launch_gemv_t<WT, 14, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 15: st = launch_gemv_t<WT, 15, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 16: st = launch_gemv_t<WT, 16, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            default: st = launch_gemv_t<WT, 1, 1>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            }
        } else {
            switch (c.nrt) {
            case 2: st = launch_gemv_t<WT, 2, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 3: st = launch_gemv_t<WT, 3, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 4: st = launch_gemv_t<WT, 4, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 5: st = launch_gemv_t<WT, 5, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 6: st = launch_gemv_t<WT, 6, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 7: st = launch_gemv_t<WT, 7, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            case 8: st = launch_gemv_t<WT, 8, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            default: st = launch_gemv_t<WT, 1, 2>(ctx, c, wm, hm, r0, n, d, v_rows, out, ld, s); break;
            }
        }
    }
    return st;
}

}  // namespace

int launch_exact_logits(frs_ctx *ctx, const float *h, int n, int d, const void *W, int w_dtype, int v_rows,
                        float *logits, cudaStream_t s) {
    if (gemv_enabled() && d % 8 == 0 && d >= 8 && (reinterpret_cast<uintptr_t>(W) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(h) & 15) == 0) {
        timing_begin(ctx, s);
        int st = FRS_OK;
        if ((v_rows + gv::GROUP - 1) / gv::GROUP < 2 * ctx->sm_count) {  // short row ranges per SM
            for (int r0 = 0; r0 < n && !st; r0 += gv1::NMAX) {
                const int nb = std::min(gv1::NMAX, n - r0);
                st = (w_dtype == FRS_DTYPE_BF16)
                         ? launch_gemv_rb(ctx, h + (size_t)r0 * d, nb, d, static_cast<const unsigned short *>(W), v_rows,
                                          logits + (size_t)r0 * v_rows, v_rows, s)
                         : launch_gemv_rb(ctx, h + (size_t)r0 * d, nb, d, static_cast<const float *>(W), v_rows,
                                          logits + (size_t)r0 * v_rows, v_rows, s);
            }
        } else {
            st = (w_dtype == FRS_DTYPE_BF16)
                     ? launch_gemv(ctx, h, n, d, static_cast<const unsigned short *>(W), v_rows, logits, v_rows, s)
                     : launch_gemv(ctx, h, n, d, static_cast<const float *>(W), v_rows, logits, v_rows, s);
        }
        timing_end(ctx, s);
        return st;
    }
    // Rows per pass: as many as fit (<= 12) with the hidden rows resident in shared memory.
    const size_t per_row = (size_t)(d & ~7) * sizeof(float);
    int nb_cap = static_cast<int>(std::min<size_t>(12, ctx->smem_optin / std::max<size_t>(per_row, 1)));
    nb_cap = nb_cap >= 4 ? (nb_cap & ~3) : std::min(nb_cap, 2);  // 1-2 unpadded rows for wide inputs
    if (nb_cap < 1) {
        const long long groups = (long long)n * v_rows;
        const int blocks = (int)std::min<long long>((long long)ctx->sm_count * 8, (groups * 8 + 255) / 256);
        ++ctx->launches;
        if (w_dtype == FRS_DTYPE_BF16)  // bf16 words read as raw u16 (w_at widens them exactly)
            k_exact_logits_wide<<<blocks, 256, 0, s>>>(h, n, d, static_cast<const unsigned short *>(W), v_rows, logits);
        else
            k_exact_logits_wide<<<blocks, 256, 0, s>>>(h, n, d, static_cast<const float *>(W), v_rows, logits);
        FRS_CUDA_TRY(cudaGetLastError());
        return FRS_OK;
    }
    int st = ctx->counters.ensure(64 * sizeof(unsigned));
    if (st) return st;
    unsigned *counters = static_cast<unsigned *>(ctx->counters.ptr);
    int pass = 0;
    timing_begin(ctx, s);
    struct EndTiming {
        frs_ctx *c;
        cudaStream_t s;
        ~EndTiming() { timing_end(c, s); }
    } end_timing{ctx, s};
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
                        const int32_t *ordered_ids, int32_t *out_ridx, int32_t *out_full, float *out_prob,
                        float *out_rowmax, double *out_total, uint32_t *out_flags, cudaStream_t s) {
    int st = ctx->scratch.ensure((size_t)n * v * sizeof(float));
    if (st) return st;
    ++ctx->launches;
    float *ework = static_cast<float *>(ctx->scratch.ptr);
    const int chunk = ((v + kSmC - 1) / kSmC + 3) & ~3;
    static const bool one_cta = std::getenv("FRS_SOFTMAX_ONE_CTA") != nullptr;  // DIAGNOSTIC
    if (!out_total && k <= kSmKMax && chunk <= 16 * kSmNT && !one_cta) {  // cluster path (Σ not returned)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(n * kSmC);
        cfg.blockDim = dim3(kSmNT);
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = kSmC;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        if (chunk <= 8 * kSmNT)
            FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_softmax_topk_cl<8>, logits, v, v, k, temperature, ordered_ids,
                                            ework, out_ridx, out_full, out_prob, out_rowmax, out_flags));
        else
            FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_softmax_topk_cl<16>, logits, v, v, k, temperature, ordered_ids,
                                            ework, out_ridx, out_full, out_prob, out_rowmax, out_flags));
        return FRS_OK;
    }
    k_softmax_topk<<<n, 1024, 0, s>>>(logits, v, v, k, temperature, ordered_ids, ework, out_ridx, out_full, out_prob,
                                      out_rowmax, out_total, out_flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int launch_softmax_sample(frs_ctx *ctx, const float *logits, int n, int v, float temperature, const double *uniforms,
                          int w, const int32_t *ordered_ids, float *probs, int32_t *out_ridx, int32_t *out_full,
                          float *out_prob, int32_t *out_count, uint32_t *out_flags, cudaStream_t s) {
    int st = ctx->scratch.ensure((size_t)n * v * sizeof(float));
    if (st) return st;
    ++ctx->launches;
    float *work = static_cast<float *>(ctx->scratch.ptr);
    const size_t wk_bytes = (size_t)v * sizeof(float);
    const bool wk_smem = wk_bytes <= 160 * 1024 && wk_bytes + 16 * 1024 <= (size_t)ctx->smem_optin;
    const int chunk = ((v + kSmC - 1) / kSmC + 3) & ~3;
    static const bool one_cta = std::getenv("FRS_SOFTMAX_ONE_CTA") != nullptr;  // DIAGNOSTIC
    if (wk_smem && chunk <= 16 * kSmNT && !one_cta) {  // cluster softmax, the leader draws
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(n * kSmC);
        cfg.blockDim = dim3(kSmNT);
        cfg.dynamicSmemBytes = wk_bytes;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = kSmC;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        if (chunk <= 8 * kSmNT) {
            FRS_CUDA_TRY(cudaFuncSetAttribute(k_softmax_sample_cl<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)wk_bytes));
            FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_softmax_sample_cl<8>, logits, v, temperature, uniforms, w,
                                            ordered_ids, probs, work, out_ridx, out_full, out_prob, out_count,
                                            out_flags));
        } else {
            FRS_CUDA_TRY(cudaFuncSetAttribute(k_softmax_sample_cl<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)wk_bytes));
            FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_softmax_sample_cl<16>, logits, v, temperature, uniforms, w,
                                            ordered_ids, probs, work, out_ridx, out_full, out_prob, out_count,
                                            out_flags));
        }
        return FRS_OK;
    }
    if (wk_smem)
        FRS_CUDA_TRY(cudaFuncSetAttribute(k_softmax_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wk_bytes));
    k_softmax_sample<<<n, 1024, wk_smem ? wk_bytes : 0, s>>>(logits, v, temperature, uniforms, w, ordered_ids, probs,
                                                             work, out_ridx, out_full, out_prob, out_count, out_flags,
                                                             wk_smem ? 1 : 0);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int launch_masked_attention_strided(frs_ctx *ctx, const float *q, int q_ld, const float *k, int k_ld, const float *v,
                                    int v_ld, const unsigned long long *mask, int n, int m, int dh, int dv, int heads,
                                    float *out, int out_ld, uint32_t *flags, cudaStream_t s) {
    int st = ctx->attn_scratch.ensure((size_t)heads * n * m * sizeof(float));
    if (st) return st;
    // q / k / v / out columns of head h start at h dh (h dv) within rows of stride *_ld
    const int pitch = ((dh + 3) & ~3) + 4;
    const size_t smem_s = (size_t)(kAttnRowBlk + kAttnKeyBlk) * pitch * sizeof(float);
    const size_t budget = std::min<size_t>(ctx->smem_optin, 200 * 1024);
    if (smem_s > budget) return fail(FRS_ENOTSUP, "masked_attention: head width above the shared-memory tile");
    // query rows per PV CTA (rows x 32 threads): all of a short batch (no idle row warps at the
    // barriers), at most 16, fewer for long key ranges
    int rows_pv = std::min(16, n);
    while (rows_pv > 1 && (size_t)rows_pv * m * 4 + 64 * kAttnCols * 4 > budget) rows_pv = (rows_pv + 1) / 2;
    // the whole value slice resident (m x 32 floats) when it fits next to the rows' probabilities
    const size_t p_bytes = (((size_t)rows_pv * m + 3) & ~size_t(3)) * 4;
    const int whole = p_bytes + (size_t)m * kAttnCols * 4 <= budget ? 1 : 0;
    const size_t smem_p = p_bytes + (size_t)(whole ? m : 64) * kAttnCols * 4;
    if (smem_p > budget) return fail(FRS_ENOTSUP, "masked_attention: key range above the shared-memory row buffer");
    const float scale = 1.0f / std::sqrt(static_cast<float>(dh));  // kernels.cpp:135 (float division of 1 by sqrtf)
    FRS_CUDA_TRY(cudaFuncSetAttribute(k_attn_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s));
    FRS_CUDA_TRY(cudaFuncSetAttribute(k_attn_pv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p));
    FRS_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)n * sizeof(uint32_t), s));
    float *S = static_cast<float *>(ctx->attn_scratch.ptr);
    ctx->launches += 2;
    k_attn_scores<<<dim3(heads, (m + kAttnKeyBlk - 1) / kAttnKeyBlk, (n + kAttnRowBlk - 1) / kAttnRowBlk), 256, smem_s,
                    s>>>(q, q_ld, k, k_ld, mask, n, m, dh, scale, S);
    FRS_CUDA_TRY(cudaGetLastError());
    k_attn_pv<<<dim3(heads, (dv + kAttnCols - 1) / kAttnCols, (n + rows_pv - 1) / rows_pv), rows_pv * kAttnCols, smem_p,
                s>>>(S, v, v_ld, mask, n, m, dv, rows_pv, whole, out, out_ld, flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int launch_masked_attention(frs_ctx *ctx, const float *q, const float *k, const float *v,
                            const unsigned long long *mask, int n, int m, int dh, int dv, float *out, uint32_t *flags,
                            cudaStream_t s) {
    return launch_masked_attention_strided(ctx, q, dh, k, dh, v, dv, mask, n, m, dh, dv, 1, out, dv, flags, s);
}

int launch_softmax_probs(frs_ctx *ctx, const float *logits, int n, int v, float temperature, float *probs,
                         uint32_t *flags, cudaStream_t s) {
    ++ctx->launches;
    k_softmax_probs_rows<<<n, 1024, 0, s>>>(logits, v, temperature, probs, flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int launch_argmax_rows(frs_ctx *ctx, const float *logits, int m, int v, int32_t id_offset, int32_t *out_id,
                       float *out_val, uint32_t *out_flags, cudaStream_t s) {
    ++ctx->launches;
    k_argmax_rows<<<m, 1024, 0, s>>>(logits, v, v, id_offset, out_id, out_val, out_flags);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

}  // namespace frs
