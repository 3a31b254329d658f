// K1 slab build, K4 greedy accept, K5 vocab-parallel argmax merge, row gather.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>

#include "frs_common.cuh"
#include "frs_device.cuh"

namespace frs {
namespace {

// K1 — restrict_lm_head (vocab.cpp:152-168) on the device: one CTA per slab row (grid-stride),
// 16-byte vector loads/stores. fp32 -> fp32 is a bitwise copy; fp32 -> bf16 rounds to nearest
// even (exact when W is bf16-representable, which the bf16 parity fixtures guarantee).
template <bool BF16>
__global__ void __launch_bounds__(256)
    k_slab_build(const float *__restrict__ W, long long V, int d, const int32_t *__restrict__ ids,
                 int v_sub, void *__restrict__ slab, int *__restrict__ err) {
    for (int row = blockIdx.x; row < v_sub; row += gridDim.x) {
        const int src = ids[row];
        if (src < 0 || src >= V) {
            if (threadIdx.x == 0) atomicExch(err, 1);
            continue;
        }
        const float *s = W + (size_t)src * d;
        if (!BF16) {
            float *o = static_cast<float *>(slab) + (size_t)row * d;
            if ((d & 3) == 0) {
                const float4 *s4 = reinterpret_cast<const float4 *>(s);
                float4 *o4 = reinterpret_cast<float4 *>(o);
                for (int c = threadIdx.x; c < d / 4; c += blockDim.x) o4[c] = __ldg(s4 + c);
            } else {
                for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = s[c];
            }
        } else {
            __nv_bfloat16 *o = static_cast<__nv_bfloat16 *>(slab) + (size_t)row * d;
            if ((d & 3) == 0) {
                const float4 *s4 = reinterpret_cast<const float4 *>(s);
                for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
                    const float4 v = __ldg(s4 + c);
                    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
                    uint2 packed;
                    packed.x = *reinterpret_cast<uint32_t *>(&a);
                    packed.y = *reinterpret_cast<uint32_t *>(&b);
                    reinterpret_cast<uint2 *>(o)[c] = packed;
                }
            } else {
                for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = __float2bfloat16_rn(s[c]);
            }
        }
    }
}

// K4 — verify_greedy walk (verification.cpp:42-71) in one warp: children of `node` are the
// indices c with parents[c] == node in ascending order (children_by_node, :31-38); the first
// whose token equals the target argmax is accepted, otherwise the argmax is the bonus token.
__global__ void k_accept_greedy(const int32_t *__restrict__ argmax_ids, const int32_t *__restrict__ tokens,
                                const int32_t *__restrict__ parents, int k, int32_t *__restrict__ emitted,
                                int32_t *__restrict__ path, int32_t *__restrict__ counts,
                                const int32_t *__restrict__ k_dev) {
    const int lane = threadIdx.x;
    if (k_dev) k = *k_dev;  // node count produced on the device (fused decode step)
    int node = -1, ne = 0, np = 0;
    for (int step = 0; step <= k; ++step) {  // a path has at most k nodes
        const int32_t best = argmax_ids[node + 1];
        int match = -1;
        for (int base = 0; base < k && match < 0; base += 32) {
            const int c = base + lane;
            const bool hit = c < k && parents[c] == node && tokens[c] == best;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) match = base + __ffs(m) - 1;
        }
        if (lane == 0) emitted[ne] = best;
        ++ne;
        if (match < 0) break;
        if (lane == 0) path[np] = match;
        ++np;
        node = match;
    }
    if (lane == 0) {
        counts[0] = ne;
        counts[1] = np;
    }
}

__device__ __forceinline__ uint32_t ord_bits(float x) {
    if (x == 0.0f) x = 0.0f;
    const uint32_t b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// K5 — merge shard-major (value, id) pairs by (value desc, id asc).
__global__ void k_argmax_merge(const float *__restrict__ vals, const int32_t *__restrict__ ids, int shards,
                               int m, float *__restrict__ out_val, int32_t *__restrict__ out_id) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= m) return;
    unsigned long long best = 0ull;
    int bs = 0;
    for (int g = 0; g < shards; ++g) {
        const unsigned long long key = (static_cast<unsigned long long>(ord_bits(vals[(size_t)g * m + row])) << 32) |
                                       (0xffffffffu - static_cast<uint32_t>(ids[(size_t)g * m + row]));
        if (key > best) {
            best = key;
            bs = g;
        }
    }
    out_val[row] = vals[(size_t)bs * m + row];
    out_id[row] = ids[(size_t)bs * m + row];
}

// grid (n, splits): row i, one slice of it per CTA; float4 when rows are 16-byte aligned (one
// load in flight per thread for d <= 4096: a latency-bound scalar loop took ~10 us per level)
__global__ void __launch_bounds__(256)
    k_gather_rows(const float *__restrict__ table, long long rows, int d, const int32_t *__restrict__ tokens,
                  int n, float *__restrict__ out) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int t = tokens[i];
    const bool ok = t >= 0 && t < rows;
    const int tid = blockIdx.y * blockDim.x + threadIdx.x, nt = gridDim.y * blockDim.x;
    const bool vec = (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(table) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const float4 *src = reinterpret_cast<const float4 *>(table + (size_t)(ok ? t : 0) * d);
        float4 *dst = reinterpret_cast<float4 *>(out + (size_t)i * d);
        for (int c = tid; c < d / 4; c += nt) dst[c] = ok ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
        for (int c = tid; c < d; c += nt) out[(size_t)i * d + c] = ok ? table[(size_t)t * d + c] : 0.0f;
    }
}

// count_frequencies (vocab.cpp:23-38) on the device: counts[t] = occurrences of t. Each CTA
// privatises the ids below kSmemBins in a u32 shared histogram (Zipf-ranked corpora put most
// of the mass there) and sends the rest to the u64 global counters; both with warp-aggregated
// atomics (one per distinct id in the warp); the shared bins are flushed at the end. An id out
// of range records the smallest offending offset (the reference throws at the first one).
constexpr int kSmemBins = 24576;  // 96 KB of u32

__global__ void __launch_bounds__(1024)
    k_count_tokens(const int32_t *__restrict__ tokens, long long count, int vocab, unsigned long long *__restrict__ counts,
                   unsigned long long *__restrict__ bad_offset) {
    extern __shared__ unsigned s_bins[];
    const int nb = min(vocab, kSmemBins);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) s_bins[b] = 0u;
    __syncthreads();
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < count; base += stride) {  // warp-uniform
        const long long i = base + threadIdx.x;
        const bool in = i < count;
        const int t = in ? __ldcs(tokens + i) : 0;
        const bool ok = in && t >= 0 && t < vocab;
        if (in && !ok) atomicMin(bad_offset, static_cast<unsigned long long>(i));
        // one atomic per distinct id in the warp (Zipf corpora repeat the head ids constantly)
        const int key = ok ? t : -1 - lane;  // distinct dummies for the other lanes
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        if (ok && lane == __ffs(peers) - 1) {
            if (t < nb)
                atomicAdd(&s_bins[t], static_cast<unsigned>(__popc(peers)));
            else
                atomicAdd(counts + t, static_cast<unsigned long long>(__popc(peers)));
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (s_bins[b]) atomicAdd(counts + b, static_cast<unsigned long long>(s_bins[b]));
}

}  // namespace

int slab_build(frs_ctx *ctx, const float *W, long long V, int d, const int32_t *ids, int v_sub, int dtype,
               void *slab, cudaStream_t s) {
    int st = ctx->flags.ensure(256);
    if (st) return st;
    int *err = static_cast<int *>(ctx->flags.ptr);
    FRS_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int), s));
    const int grid = ctx->sm_count * 8;
    if (dtype == FRS_DTYPE_BF16)
        k_slab_build<true><<<grid, 256, 0, s>>>(W, V, d, ids, v_sub, slab, err);
    else
        k_slab_build<false><<<grid, 256, 0, s>>>(W, V, d, ids, v_sub, slab, err);
    FRS_CUDA_TRY(cudaGetLastError());
    int host_err = 0;
    FRS_CUDA_TRY(cudaMemcpyAsync(&host_err, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    FRS_CUDA_TRY(cudaStreamSynchronize(s));
    if (host_err) return fail(FRS_EINVAL, "restrict_lm_head: subset id out of range for the LM head");
    return FRS_OK;
}

int accept_greedy(const int32_t *argmax_ids, const int32_t *tokens, const int32_t *parents, int k,
                  int32_t *emitted, int32_t *path, int32_t *counts, cudaStream_t s) {
    k_accept_greedy<<<1, 32, 0, s>>>(argmax_ids, tokens, parents, k, emitted, path, counts, nullptr);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

// Fused decode step (frs_host.cu): the selected tree `out` ([0] count | [1] flags | tokens[64] |
// parents[64] ...) becomes the verify rows [root, tokens..., root padding up to 1 + total] and
// the accept walk's parents / node count, all on the device.
__global__ void k_step_rows(const int32_t *__restrict__ out, int32_t root, int total, int32_t *__restrict__ rt,
                            int32_t *__restrict__ pp, int32_t *__restrict__ kdev) {
    const int i = threadIdx.x, count = out[0];
    if (i == 0) {
        rt[0] = root;
        *kdev = count;
    }
    if (i < total) {
        rt[1 + i] = i < count ? out[2 + i] : root;
        pp[i] = i < count ? out[2 + 64 + i] : -1;
    }
}

int step_rows_accept(const int32_t *tree_out, int32_t root, int total, int32_t *rt, int32_t *pp, int32_t *kdev,
                     cudaStream_t s) {
    k_step_rows<<<1, 64, 0, s>>>(tree_out, root, total, rt, pp, kdev);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int accept_greedy_devk(const int32_t *argmax_ids, const int32_t *tokens, const int32_t *parents,
                       const int32_t *kdev, int32_t *emitted, int32_t *path, int32_t *counts, cudaStream_t s) {
    k_accept_greedy<<<1, 32, 0, s>>>(argmax_ids, tokens, parents, 64, emitted, path, counts, kdev);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int argmax_merge(const float *vals, const int32_t *ids, int shards, int m, float *out_val, int32_t *out_id,
                 cudaStream_t s) {
    k_argmax_merge<<<(m + 127) / 128, 128, 0, s>>>(vals, ids, shards, m, out_val, out_id);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int count_tokens(frs_ctx *ctx, const int32_t *tokens, long long count, int vocab, unsigned long long *counts,
                 unsigned long long *bad_offset, cudaStream_t s) {
    FRS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (size_t)vocab, s));
    FRS_CUDA_TRY(cudaMemsetAsync(bad_offset, 0xff, sizeof(unsigned long long), s));
    if (count == 0) return FRS_OK;
    const size_t smem = sizeof(unsigned) * (size_t)std::min(vocab, kSmemBins);
    FRS_CUDA_TRY(cudaFuncSetAttribute(k_count_tokens, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long blocks = std::min<long long>(ctx->sm_count * 2, (count + 1023) / 1024);
    ++ctx->launches;
    k_count_tokens<<<(int)blocks, 1024, smem, s>>>(tokens, count, vocab, counts, bad_offset);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int gather_rows(const float *table, long long rows, int d, const int32_t *tokens, int n, float *out,
                cudaStream_t s) {
    const int splits = std::max(1, std::min(16, (d / 4 + 255) / 256));
    k_gather_rows<<<dim3(n, splits), 256, 0, s>>>(table, rows, d, tokens, n, out);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

// Known-answer check of the device glibc expf ports: for the
// float bit patterns first_bits + i (i < count) compare expf_glibc and expf_glibc_nb with the
// host libm's expf values `expected`; out[0..1] mismatch counts, out[2..3] first mismatching i
// (atomicMin; preset to ~0 by the caller), variants 0 / 1.
__global__ void k_expf_kat(uint32_t first_bits, long long count, const float *__restrict__ expected,
                           unsigned long long *__restrict__ out) {
    __shared__ unsigned long long tab[32];
    dev::load_exp_table(tab);
    __syncthreads();
    unsigned long long bad0 = 0, bad1 = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        const float x = __uint_as_float(first_bits + static_cast<uint32_t>(i));
        const uint32_t want = __float_as_uint(expected[i]);
        if (__float_as_uint(dev::expf_glibc(x, tab)) != want) {
            ++bad0;
            atomicMin(&out[2], static_cast<unsigned long long>(i));
        }
        if (__float_as_uint(dev::expf_glibc_nb(x, tab)) != want) {
            ++bad1;
            atomicMin(&out[3], static_cast<unsigned long long>(i));
        }
    }
    if (bad0) atomicAdd(&out[0], bad0);
    if (bad1) atomicAdd(&out[1], bad1);
}

int expf_kat(frs_ctx *ctx, uint32_t first_bits, long long count, const float *expected, unsigned long long *out,
             cudaStream_t s) {
    ++ctx->launches;
    k_expf_kat<<<ctx->sm_count * 8, 256, 0, s>>>(first_bits, count, expected, out);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

}  // namespace frs
