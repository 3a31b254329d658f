// Shared internals of libfrspec_cuda.so: context, error plumbing, device helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "frspec_cuda.h"

namespace frs {

// ---- error plumbing: status codes + thread-local message (frspec_cuda.h) ----
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
#define FRS_CUDA_TRY(expr)                                                                   \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return ::frs::fail(FRS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define FRS_REQUIRE(cond, msg)                                  \
    do {                                                        \
        if (!(cond)) return ::frs::fail(FRS_EINVAL, (msg));     \
    } while (0)

// Grow-only device scratch buffer.
struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    int ensure(size_t need);
    ~DevBuf();
};

// CUDA-graph cache of repeated FAST calls (frs_fast.cu): the key is every pointer, size and
// parameter the captured chain bakes in.
constexpr int kGraphKeyWords = 21;
struct GraphKey {
    uint64_t w[kGraphKeyWords];
    bool operator==(const GraphKey &o) const {
        for (int i = 0; i < kGraphKeyWords; ++i)
            if (w[i] != o.w[i]) return false;
        return true;
    }
};
struct GraphEntry {
    GraphKey key{};
    cudaGraphExec_t exec = nullptr;
    uint64_t last_use = 0;
};

}  // namespace frs

struct frs_ctx {
    int device = 0;
    int sm_count = 148;
    size_t smem_optin = 0;
    frs::DevBuf logits;    // [rows x vocab] fp32 logits (EXACT)
    frs::DevBuf scratch;   // [rows x vocab] fp32 exp values (EXACT softmax)
    frs::DevBuf counters;  // work-queue counters for persistent kernels
    frs::DevBuf flags;     // uint32 status flags
    frs::DevBuf fast_ws;   // FAST path candidate/partials workspace
    frs::DevBuf fast_ctr;  // FAST counters: fallback queue (zeroed once)
    frs::DevBuf fast_logits;  // FAST batched drafting: approximate logits [n x V_sub] fp32
    frs::DevBuf attn_scratch;  // masked_attention: per (head, query row) scores [heads x n x m] fp32
    frs::DevBuf trace;     // FAST main-kernel globaltimer stamps when FRS_TRACE is set (diagnostics)
    frs::DevBuf hbuf;      // host-API staging of hidden rows
    frs::DevBuf obuf;      // host-API staging of outputs
    frs::DevBuf vp_buf;    // vocab-parallel verify: local + all-gathered (value, id) pairs
    void *pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaStream_t stream = nullptr;  // owned stream for the host-buffer conveniences
    // live timing of the dominant kernel of each call (bench roofline), on its own stream
    bool timing = false;
    std::vector<cudaEvent_t> ev;  // start/stop pairs
    size_t ev_used = 0;
    unsigned long long launches = 0;  // kernels launched by this library on this ctx
    std::vector<frs::GraphEntry> graphs;  // captured FAST chains (LRU)
    uint64_t graph_clock = 0;
    cudaStream_t cap_stream = nullptr;    // private stream for graph capture
    bool prefer_graphs = false;           // set by host loops that wait on every call (frs_draft_tree)
    const float *h_stage_src = nullptr;   // set by frs_head_draft_host around one FAST call: k_hsplit
                                          // reads the hidden rows from this mapped pinned host
                                          // pointer and writes them to the call's h (device)
};

namespace frs {

void timing_begin(frs_ctx *ctx, cudaStream_t s);
void timing_end(frs_ctx *ctx, cudaStream_t s);

constexpr int kMaxK = 64;  // width <= total_draft_tokens <= 64 (drafting.cpp:14-20)

// Launchers (defined in the .cu files); all return frs_status.
int launch_exact_logits(frs_ctx *ctx, const float *h, int n, int d, const void *W, int w_dtype,
                        int v_rows, float *logits, cudaStream_t s);
int launch_masked_attention(frs_ctx *ctx, const float *q, const float *k, const float *v,
                            const unsigned long long *mask, int n, int m, int dh, int dv, float *out, uint32_t *flags,
                            cudaStream_t s);
int count_tokens(frs_ctx *ctx, const int32_t *tokens, long long count, int vocab, unsigned long long *counts,
                 unsigned long long *bad_offset, cudaStream_t s);
int expf_kat(frs_ctx *ctx, uint32_t first_bits, long long count, const float *expected, unsigned long long *out,
             cudaStream_t s);
int launch_softmax_probs(frs_ctx *ctx, const float *logits, int n, int v, float temperature, float *probs,
                         uint32_t *flags, cudaStream_t s);
int launch_softmax_sample(frs_ctx *ctx, const float *logits, int n, int v, float temperature, const double *uniforms,
                          int w, const int32_t *ordered_ids, float *probs, int32_t *out_ridx, int32_t *out_full,
                          float *out_prob, int32_t *out_count, uint32_t *out_flags, cudaStream_t s);
int launch_softmax_topk(frs_ctx *ctx, const float *logits, int n, int v, int k, float temperature,
                        const int32_t *ordered_ids, int32_t *out_ridx, int32_t *out_full,
                        float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags,
                        cudaStream_t s);
int launch_argmax_rows(frs_ctx *ctx, const float *logits, int m, int v, int32_t id_offset,
                       int32_t *out_id, float *out_val, uint32_t *out_flags, cudaStream_t s);
size_t slab_tile_bytes(int v_rows, int d);
int launch_slab_tile(frs_ctx *ctx, const void *slab, int v_rows, int d, void *tiled, cudaStream_t s);
int launch_fast_draft(frs_ctx *ctx, const float *h, int n, int d, const void *slab, const void *tiled, int v_sub,
                      const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx,
                      int32_t *out_full, float *out_prob, float *out_rowmax, double *out_total,
                      uint32_t *out_flags, cudaStream_t s);
int debug_fast_partials(frs_ctx *ctx, int n, int d, float *pm, float *ps, float *pth, unsigned long long *pkey,
                        float *pw2);
int launch_fast_verify(frs_ctx *ctx, const float *h, int m, int d, const void *W, const void *tiled, int v_rows,
                       int32_t id_offset, int32_t *out_id, float *out_val, uint32_t *out_flags,
                       cudaStream_t s);

}  // namespace frs
