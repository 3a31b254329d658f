// C ABI of libfrspec_cuda.so (include/frspec_cuda.h): context, argument validation that
// mirrors the reference's preconditions, and dispatch to the EXACT / FAST kernels.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "frs_common.cuh"

namespace frs {

thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int status, const std::string &msg) {
    g_last_error = msg;
    return status;
}

int DevBuf::ensure(size_t need) {
    if (need <= bytes) return FRS_OK;
    const size_t grow = std::max(need, bytes + bytes / 2);
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, grow);
    if (e != cudaSuccess) {
        ptr = nullptr;
        return fail(FRS_ECUDA, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
    }
    bytes = grow;
    return FRS_OK;
}
DevBuf::~DevBuf() {
    if (ptr) cudaFree(ptr);
}

int slab_build(frs_ctx *ctx, const float *W, long long V, int d, const int32_t *ids, int v_sub, int dtype,
               void *slab, cudaStream_t s);
int accept_greedy(const int32_t *argmax_ids, const int32_t *tokens, const int32_t *parents, int k,
                  int32_t *emitted, int32_t *path, int32_t *counts, cudaStream_t s);
int argmax_merge(const float *vals, const int32_t *ids, int shards, int m, float *out_val, int32_t *out_id,
                 cudaStream_t s);
int gather_rows(const float *table, long long rows, int d, const int32_t *tokens, int n, float *out,
                cudaStream_t s);

static int check_device(frs_ctx *ctx) {
    if (!ctx) return fail(FRS_EINVAL, "null frs_ctx");
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    return FRS_OK;
}

static bool valid_dtype(int dt) { return dt == FRS_DTYPE_F32 || dt == FRS_DTYPE_BF16; }

void timing_begin(frs_ctx *ctx, cudaStream_t s) {
    if (!ctx->timing) return;
    if (ctx->ev_used + 2 > ctx->ev.size()) {
        for (int i = 0; i < 256; ++i) {
            cudaEvent_t e;
            if (cudaEventCreate(&e) != cudaSuccess) return;
            ctx->ev.push_back(e);
        }
    }
    cudaEventRecord(ctx->ev[ctx->ev_used], s);
}

void timing_end(frs_ctx *ctx, cudaStream_t s) {
    if (!ctx->timing || ctx->ev_used + 2 > ctx->ev.size()) return;
    cudaEventRecord(ctx->ev[ctx->ev_used + 1], s);
    ctx->ev_used += 2;
}

}  // namespace frs

using namespace frs;

extern "C" {

int frs_abi_version(void) { return FRS_ABI_VERSION; }
const char *frs_last_error(void) { return g_last_error.c_str(); }

int frs_ctx_create(int device, frs_ctx **out) {
    FRS_REQUIRE(out != nullptr, "frs_ctx_create: null out");
    *out = nullptr;
    int count = 0;
    FRS_CUDA_TRY(cudaGetDeviceCount(&count));
    FRS_REQUIRE(device >= 0 && device < count, "frs_ctx_create: no such CUDA device");
    FRS_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop{};
    FRS_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(FRS_ENOTSUP, "libfrspec_cuda requires an sm_100a (Blackwell) device");
    frs_ctx *c = new frs_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(FRS_ECUDA, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    *out = c;
    return FRS_OK;
}

int frs_ctx_destroy(frs_ctx *ctx) {
    if (!ctx) return FRS_OK;
    cudaSetDevice(ctx->device);
    for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
    for (auto &g : ctx->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    delete ctx;
    return FRS_OK;
}

int frs_ctx_sm_count(const frs_ctx *ctx) { return ctx ? ctx->sm_count : 0; }

int frs_ctx_set_timing(frs_ctx *ctx, int enable) {
    FRS_REQUIRE(ctx, "null frs_ctx");
    ctx->timing = enable != 0;
    ctx->ev_used = 0;
    return FRS_OK;
}

// Latency-bound callers (a dependent draft loop): repeated FAST calls with the same buffers and
// shapes replay a captured CUDA graph of the chain (one launch) instead of eager launches.
int frs_ctx_set_graphs(frs_ctx *ctx, int enable) {
    FRS_REQUIRE(ctx, "null frs_ctx");
    ctx->prefer_graphs = enable != 0;
    return FRS_OK;
}

int frs_ctx_timing_read(frs_ctx *ctx, double *total_ms, int *count) {
    FRS_REQUIRE(ctx && total_ms && count, "frs_ctx_timing_read: null pointer");
    double tot = 0.0;
    for (size_t i = 0; i + 1 < ctx->ev_used; i += 2) {
        FRS_CUDA_TRY(cudaEventSynchronize(ctx->ev[i + 1]));
        float ms = 0.0f;
        FRS_CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev[i], ctx->ev[i + 1]));
        tot += ms;
    }
    *total_ms = tot;
    *count = static_cast<int>(ctx->ev_used / 2);
    ctx->ev_used = 0;
    return FRS_OK;
}

int frs_debug_expf_check(frs_ctx *ctx, uint32_t first_bits, int64_t count, const float *expected, uint64_t *out,
                         void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(expected && out && count >= 0, "expf check: bad arguments");
    return expf_kat(ctx, first_bits, count, expected, reinterpret_cast<unsigned long long *>(out),
                    static_cast<cudaStream_t>(stream));
}

int frs_debug_fast_partials(frs_ctx *ctx, int n, int d, float *pm, float *ps, float *pth, uint64_t *pkey,
                            float *pw2) {
    int st = check_device(ctx);
    if (st) return st;
    return frs::debug_fast_partials(ctx, n, d, pm, ps, pth, reinterpret_cast<unsigned long long *>(pkey), pw2);
}

int frs_ctx_launch_count(const frs_ctx *ctx, uint64_t *out) {
    FRS_REQUIRE(ctx && out, "frs_ctx_launch_count: null pointer");
    *out = ctx->launches;
    return FRS_OK;
}

int frs_ctx_reserve(frs_ctx *ctx, int max_rows, int64_t max_vocab, int d) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(max_rows >= 1 && max_vocab >= 1 && d >= 1, "frs_ctx_reserve: sizes must be positive");
    const size_t cells = (size_t)max_rows * (size_t)max_vocab;
    if ((st = ctx->logits.ensure(cells * sizeof(float)))) return st;
    if ((st = ctx->scratch.ensure(cells * sizeof(float)))) return st;
    if ((st = ctx->counters.ensure(64 * sizeof(unsigned)))) return st;
    if ((st = ctx->flags.ensure(256))) return st;
    if ((st = ctx->hbuf.ensure((size_t)max_rows * d * sizeof(float)))) return st;
    return FRS_OK;
}

size_t frs_slab_bytes(int v_sub, int d, int slab_dtype) {
    return (size_t)v_sub * (size_t)d * (slab_dtype == FRS_DTYPE_BF16 ? 2 : 4);
}

int frs_slab_build(frs_ctx *ctx, const float *W, int64_t V, int d, const int32_t *ordered_ids, int v_sub,
                   int slab_dtype, void *slab, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(W && ordered_ids && slab, "restrict_lm_head: null pointer");
    FRS_REQUIRE(V >= 1 && d >= 1 && v_sub >= 1, "restrict_lm_head: sizes must be positive");
    FRS_REQUIRE(valid_dtype(slab_dtype), "restrict_lm_head: unknown slab dtype");
    ++ctx->launches;
    return slab_build(ctx, W, V, d, ordered_ids, v_sub, slab_dtype, slab, static_cast<cudaStream_t>(stream));
}

int frs_draft_head_topk(frs_ctx *ctx, const float *h, int n, int d, const void *slab, int v_sub,
                        int slab_dtype, const int32_t *ordered_ids, int k, float temperature, int mode,
                        int32_t *out_ridx, int32_t *out_full, float *out_prob, float *out_rowmax,
                        double *out_total, float *out_logits, uint32_t *out_flags, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FRS_REQUIRE(h && slab && out_ridx && out_full && out_prob, "draft head: null pointer");
    FRS_REQUIRE(n >= 1, "forward: empty token batch");                       // model.cpp:217
    FRS_REQUIRE(d >= 1 && v_sub >= 1, "draft head: sizes must be positive");
    FRS_REQUIRE(k >= 1, "draft params: beam_width must be >= 1");           // drafting.cpp:15
    FRS_REQUIRE(std::isfinite(temperature) && temperature > 0.0f,
                "softmax: temperature must be positive and finite");       // kernels.cpp:66-68
    FRS_REQUIRE(valid_dtype(slab_dtype), "draft head: unknown slab dtype");
    FRS_REQUIRE(mode == FRS_MODE_EXACT || mode == FRS_MODE_FAST, "draft head: unknown mode");
    if (mode == FRS_MODE_FAST) {
        FRS_REQUIRE(slab_dtype == FRS_DTYPE_BF16, "FAST draft head needs a bf16 slab");
        FRS_REQUIRE(out_logits == nullptr, "FAST draft head never materialises logits");
        return launch_fast_draft(ctx, h, n, d, slab, nullptr, v_sub, ordered_ids, k, temperature, out_ridx, out_full,
                                 out_prob, out_rowmax, out_total, out_flags, s);
    }
    float *logits = out_logits;
    if (!logits) {
        if ((st = ctx->logits.ensure((size_t)n * v_sub * sizeof(float)))) return st;
        logits = static_cast<float *>(ctx->logits.ptr);
    }
    if ((st = launch_exact_logits(ctx, h, n, d, slab, slab_dtype, v_sub, logits, s))) return st;
    return launch_softmax_topk(ctx, logits, n, v_sub, k, temperature, ordered_ids, out_ridx, out_full, out_prob,
                               out_rowmax, out_total, out_flags, s);
}

size_t frs_slab_tile_bytes(int v_rows, int d) {
    if (v_rows < 1 || d < 1) return 0;
    return slab_tile_bytes(v_rows, d);
}

int frs_slab_tile(frs_ctx *ctx, const void *slab, int v_rows, int d, void *tiled, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(slab && tiled, "slab tile: null pointer");
    FRS_REQUIRE(v_rows >= 1 && d >= 1, "slab tile: sizes must be positive");
    FRS_REQUIRE(d % 8 == 0 && (reinterpret_cast<uintptr_t>(slab) & 15) == 0 && (reinterpret_cast<uintptr_t>(tiled) & 15) == 0,
                "slab tile: d % 8 == 0 and 16-byte aligned buffers");
    return launch_slab_tile(ctx, slab, v_rows, d, tiled, static_cast<cudaStream_t>(stream));
}

int frs_draft_head_topk_tiled(frs_ctx *ctx, const float *h, int n, int d, const void *slab, const void *tiled,
                              int v_sub, const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx,
                              int32_t *out_full, float *out_prob, float *out_rowmax, double *out_total,
                              uint32_t *out_flags, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(h && slab && tiled && out_ridx && out_full && out_prob, "draft head: null pointer");
    FRS_REQUIRE(n >= 1, "forward: empty token batch");                       // model.cpp:217
    FRS_REQUIRE(d >= 1 && v_sub >= 1, "draft head: sizes must be positive");
    FRS_REQUIRE(k >= 1, "draft params: beam_width must be >= 1");           // drafting.cpp:15
    FRS_REQUIRE(std::isfinite(temperature) && temperature > 0.0f,
                "softmax: temperature must be positive and finite");       // kernels.cpp:66-68
    return launch_fast_draft(ctx, h, n, d, slab, tiled, v_sub, ordered_ids, k, temperature, out_ridx, out_full,
                             out_prob, out_rowmax, out_total, out_flags, static_cast<cudaStream_t>(stream));
}

int frs_masked_attention(frs_ctx *ctx, const float *q, const float *k, const float *v, const uint64_t *mask, int n,
                         int m, int dh, int dv, float *out, uint32_t *flags, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(q && k && v && mask && out && flags, "masked_attention: null pointer");
    FRS_REQUIRE(n >= 1 && m >= 1 && dh >= 1 && dv >= 1, "masked_attention: sizes must be positive");
    return launch_masked_attention(ctx, q, k, v, reinterpret_cast<const unsigned long long *>(mask), n, m, dh, dv, out,
                                   flags, static_cast<cudaStream_t>(stream));
}

int frs_draft_head_sample(frs_ctx *ctx, const float *h, int n, int d, const void *slab, int v_sub, int slab_dtype,
                          const int32_t *ordered_ids, int width, float temperature, const double *uniforms,
                          float *probs, int32_t *out_ridx, int32_t *out_full, float *out_prob, int32_t *out_count,
                          uint32_t *out_flags, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FRS_REQUIRE(h && slab && uniforms && probs && out_ridx && out_full && out_prob && out_count,
                "sampled draft head: null pointer");
    FRS_REQUIRE(n >= 1, "forward: empty token batch");                       // model.cpp:217
    FRS_REQUIRE(d >= 1 && v_sub >= 1, "draft head: sizes must be positive");
    FRS_REQUIRE(width >= 1, "draft params: beam_width must be >= 1");       // drafting.cpp:15
    FRS_REQUIRE(std::isfinite(temperature) && temperature > 0.0f,
                "softmax: temperature must be positive and finite");       // kernels.cpp:66-68
    FRS_REQUIRE(valid_dtype(slab_dtype), "draft head: unknown slab dtype");
    const int w = std::min(width, v_sub);                                   // drafting.cpp:40
    if ((st = ctx->logits.ensure((size_t)n * v_sub * sizeof(float)))) return st;
    float *logits = static_cast<float *>(ctx->logits.ptr);
    if ((st = launch_exact_logits(ctx, h, n, d, slab, slab_dtype, v_sub, logits, s))) return st;
    return launch_softmax_sample(ctx, logits, n, v_sub, temperature, uniforms, w, ordered_ids, probs, out_ridx,
                                 out_full, out_prob, out_count, out_flags, s);
}

int frs_verify_head_argmax(frs_ctx *ctx, const float *h, int m, int d, const void *W, int v_rows, int w_dtype,
                           int32_t id_offset, int mode, int32_t *out_id, float *out_val, uint32_t *out_flags,
                           void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FRS_REQUIRE(h && W && out_id, "verify head: null pointer");
    FRS_REQUIRE(m >= 1, "forward: empty token batch");
    FRS_REQUIRE(d >= 1 && v_rows >= 1, "argmax: empty input");               // kernels.cpp:114-116
    FRS_REQUIRE(valid_dtype(w_dtype), "verify head: unknown dtype");
    FRS_REQUIRE(mode == FRS_MODE_EXACT || mode == FRS_MODE_FAST, "verify head: unknown mode");
    if (mode == FRS_MODE_FAST) {
        FRS_REQUIRE(w_dtype == FRS_DTYPE_BF16, "FAST verify head needs a bf16 LM head");
        return launch_fast_verify(ctx, h, m, d, W, nullptr, v_rows, id_offset, out_id, out_val, out_flags, s);
    }
    if ((st = ctx->logits.ensure((size_t)m * v_rows * sizeof(float)))) return st;
    float *logits = static_cast<float *>(ctx->logits.ptr);
    if ((st = launch_exact_logits(ctx, h, m, d, W, w_dtype, v_rows, logits, s))) return st;
    return launch_argmax_rows(ctx, logits, m, v_rows, id_offset, out_id, out_val, out_flags, s);
}

int frs_verify_head_argmax_tiled(frs_ctx *ctx, const float *h, int m, int d, const void *W, const void *W_tiled,
                                 int v_rows, int32_t id_offset, int32_t *out_id, float *out_val, uint32_t *out_flags,
                                 void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(h && W && W_tiled && out_id, "verify head: null pointer");
    FRS_REQUIRE(m >= 1, "forward: empty token batch");
    FRS_REQUIRE(d >= 1 && v_rows >= 1, "argmax: empty input");               // kernels.cpp:114-116
    return launch_fast_verify(ctx, h, m, d, W, W_tiled, v_rows, id_offset, out_id, out_val, out_flags,
                              static_cast<cudaStream_t>(stream));
}

int frs_accept_greedy(frs_ctx *ctx, const int32_t *argmax_ids, const int32_t *tokens, const int32_t *parents,
                      int k, int32_t *out_emitted, int32_t *out_path, int32_t *out_counts, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(argmax_ids && out_emitted && out_path && out_counts, "verify_greedy: null pointer");
    FRS_REQUIRE(k >= 0, "verify_greedy: negative node count");
    if (k > 64) return fail(FRS_ECAPACITY, "build_tree_mask: nodes exceed the 64-bit mask");
    FRS_REQUIRE(k == 0 || (tokens && parents), "verify_greedy: null tree arrays");
    ++ctx->launches;
    return accept_greedy(argmax_ids, tokens, parents, k, out_emitted, out_path, out_counts,
                         static_cast<cudaStream_t>(stream));
}

int frs_argmax_merge(frs_ctx *ctx, const float *vals, const int32_t *ids, int shards, int m, float *out_val,
                     int32_t *out_id, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(vals && ids && out_val && out_id, "argmax merge: null pointer");
    FRS_REQUIRE(shards >= 1 && m >= 1, "argmax merge: sizes must be positive");
    ++ctx->launches;
    return argmax_merge(vals, ids, shards, m, out_val, out_id, static_cast<cudaStream_t>(stream));
}

int frs_gather_rows(frs_ctx *ctx, const float *table, int64_t rows, int d, const int32_t *tokens, int n,
                    float *out, void *stream) {
    int st = check_device(ctx);
    if (st) return st;
    FRS_REQUIRE(table && tokens && out, "gather: null pointer");
    FRS_REQUIRE(rows >= 1 && d >= 1 && n >= 1, "gather: sizes must be positive");
    ++ctx->launches;
    return gather_rows(table, rows, d, tokens, n, out, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
