// Host side of the boundary (C++20 over the C ABI): the one-time FR vocabulary build
// (vocab.cpp:23-178 semantics), the device-resident RestrictedHead, and the head-path
// build_draft_tree / verify_greedy drivers (drafting.cpp:122-245, verification.cpp:13-71).
// Integer / bookkeeping work stays on the host exactly as in the reference (std::log on the
// same libm, std::sort comparators identical), so the device only runs the HBM-bound heads.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "frs_common.cuh"

// Candidate indices of the rows a hidden-state provider is asked to forward (level >= 1), for
// the library's own model-driven provider (frs_draft_tree_model): the public callback carries
// tokens and parent candidates only.
static thread_local const int *tl_beam_cands = nullptr;

struct frs_rng {
    std::mt19937_64 engine;
};

struct frs_head {
    frs_ctx *ctx = nullptr;
    void *slab = nullptr;
    int32_t *ordered_dev = nullptr;
    std::vector<int32_t> ordered;
    int64_t vocab = 0;
    int v_sub = 0, d = 0, dtype = FRS_DTYPE_F32;
    void *tiled = nullptr;  // bf16 slabs: the FAST head's tiled image (frs_slab_tile)
    // per-level staging (device + pinned host)
    frs::DevBuf lvl_ridx, lvl_full, lvl_prob, lvl_tok, hidden, tree_ws, smp_u, smp_probs;
    // multi-stream decode staging (frs_decode_step_table_multi): row tokens, hidden rows, packed
    // level outputs / verify argmax ids
    frs::DevBuf ms_tok, ms_hidden, ms_out;
    int32_t *h_ridx = nullptr, *h_full = nullptr, *h_tok = nullptr;
    float *h_prob = nullptr;
};

namespace frs {
namespace {

int check_forced(const int32_t *forced, int n_forced, int vocab_size) {
    for (int f = 0; f < n_forced; ++f)
        if (forced[f] < 0 || forced[f] >= vocab_size)
            return fail(FRS_EINVAL, "subset: forced id " + std::to_string(forced[f]) + " out of range");
    return FRS_OK;
}

struct Cand {
    int32_t token, ridx, parent, depth;
    double log_joint;
};

// (log_joint desc, candidate index asc) — drafting.cpp:83-86 / 167-172
struct ByLogJoint {
    const std::vector<Cand> *c;
    bool operator()(int a, int b) const {
        if ((*c)[a].log_joint != (*c)[b].log_joint) return (*c)[a].log_joint > (*c)[b].log_joint;
        return a < b;
    }
};

// pick_children's sampled branch on the host (drafting.cpp:44-74), for levels the device could
// not certify: the same draws from the same engine state, over the exact probabilities.
void pick_sampled_host(const float *probs, int n, int width, std::mt19937_64 &rng, std::vector<int> &idx,
                       std::vector<float> &pr) {
    const int w = std::min(width, n);
    idx.clear();
    pr.clear();
    std::vector<double> work(probs, probs + n);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    for (int draw = 0; draw < w; ++draw) {
        double total = 0.0;
        for (double p : work) total += p;
        if (total <= 0.0) break;
        const double u = uni(rng) * total;
        double acc = 0.0;
        int picked = -1;
        for (int i = 0; i < n; ++i) {
            acc += work[i];
            if (u < acc) {
                picked = i;
                break;
            }
        }
        if (picked < 0) {
            for (int i = n - 1; i >= 0; --i)
                if (work[i] > 0.0) {
                    picked = i;
                    break;
                }
            if (picked < 0) break;
        }
        idx.push_back(picked);
        pr.push_back(probs[picked]);
        work[picked] = 0.0;
    }
}

}  // namespace
}  // namespace frs

using namespace frs;

extern "C" {

// vocab.cpp:23-38
int frs_count_frequencies(const int32_t *stream, int64_t count, int vocab_size, uint64_t *counts) {
    FRS_REQUIRE(vocab_size >= 1, "count_frequencies: vocab_size must be >= 1");
    FRS_REQUIRE(counts && (count == 0 || stream), "count_frequencies: null pointer");
    std::fill(counts, counts + vocab_size, 0ull);
    for (int64_t i = 0; i < count; ++i) {
        const int32_t t = stream[i];
        if (t < 0 || t >= vocab_size)
            return fail(FRS_EINVAL, "count_frequencies: token id " + std::to_string(t) + " out of range at offset " +
                                        std::to_string(i));
        ++counts[t];
    }
    return FRS_OK;
}

// vocab.cpp:70-102 (+ finalize_subset 42-58)
int frs_build_subset(const uint64_t *counts, int vocab_size, int size, const int32_t *forced, int n_forced,
                     int32_t *ordered_out) {
    FRS_REQUIRE(counts && ordered_out, "build_subset: null pointer");
    if (size < 1 || size > vocab_size)
        return fail(FRS_EINVAL, "build_subset: size " + std::to_string(size) + " out of range");
    int st = check_forced(forced, n_forced, vocab_size);
    if (st) return st;
    std::vector<char> is_member(vocab_size, 0);
    std::vector<int32_t> members;
    for (int f = 0; f < n_forced; ++f)
        if (!is_member[forced[f]]) {
            is_member[forced[f]] = 1;
            members.push_back(forced[f]);
        }
    if (static_cast<int>(members.size()) > size)
        return fail(FRS_EINVAL, "build_subset: size smaller than the forced id count");
    auto by_count = [&](int32_t a, int32_t b) {
        if (counts[a] != counts[b]) return counts[a] > counts[b];
        return a < b;
    };
    std::vector<int32_t> order(vocab_size);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), by_count);
    for (int32_t t : order) {
        if (static_cast<int>(members.size()) >= size) break;
        if (!is_member[t]) {
            is_member[t] = 1;
            members.push_back(t);
        }
    }
    std::sort(members.begin(), members.end(), by_count);
    std::copy(members.begin(), members.end(), ordered_out);
    return FRS_OK;
}

// vocab.cpp:104-138
int frs_subset_from_ranking(const int32_t *ranked, int n_ranked, int size, int vocab_size, const int32_t *forced,
                            int n_forced, int32_t *ordered_out) {
    FRS_REQUIRE(ranked && ordered_out, "subset_from_ranking: null pointer");
    if (size < 1 || size > n_ranked) return fail(FRS_EINVAL, "subset_from_ranking: size out of range");
    int st = check_forced(forced, n_forced, vocab_size);
    if (st) return st;
    std::vector<char> seen(vocab_size, 0);
    for (int i = 0; i < n_ranked; ++i) {
        const int32_t t = ranked[i];
        if (t < 0 || t >= vocab_size)
            return fail(FRS_EINVAL, "subset_from_ranking: id " + std::to_string(t) + " out of range");
        if (seen[t]) return fail(FRS_EINVAL, "subset_from_ranking: duplicate id " + std::to_string(t));
        seen[t] = 1;
    }
    std::vector<int32_t> members(ranked, ranked + size);
    std::vector<char> is_member(vocab_size, 0);
    for (int32_t t : members) is_member[t] = 1;
    std::vector<int32_t> missing;
    for (int f = 0; f < n_forced; ++f)
        if (!is_member[forced[f]]) {
            is_member[forced[f]] = 1;
            missing.push_back(forced[f]);
        }
    if (static_cast<int>(missing.size()) > size)
        return fail(FRS_EINVAL, "subset_from_ranking: size smaller than the forced id count");
    for (size_t i = 0; i < missing.size(); ++i) members[members.size() - 1 - i] = missing[missing.size() - 1 - i];
    std::copy(members.begin(), members.end(), ordered_out);
    return FRS_OK;
}

// Vocab-parallel verify: contiguous shard [start, start + count) of rank
// `rank` among `world` (the first V % world ranks hold one extra row).
int frs_vocab_shard(int64_t V, int world, int rank, int64_t *start, int64_t *count) {
    FRS_REQUIRE(start && count, "vocab shard: null pointer");
    FRS_REQUIRE(V >= 1 && world >= 1 && rank >= 0 && rank < world, "vocab shard: bad sizes");
    const int64_t base = V / world, extra = V % world;
    *count = base + (rank < extra ? 1 : 0);
    *start = rank * base + std::min<int64_t>(rank, extra);
    return FRS_OK;
}

// Host twin of K5 (frs_argmax_merge) for host-resident all-gather results: per row, the pair
// with the largest value, ties to the lowest id — argmax's rule (kernels.cpp:117-121) over a
// contiguous vocabulary split. -0 and +0 compare equal, NaN never wins over a number.
int frs_argmax_merge_host(const float *vals, const int32_t *ids, int shards, int m, float *out_val,
                          int32_t *out_id) {
    FRS_REQUIRE(vals && ids && out_val && out_id, "argmax merge: null pointer");
    FRS_REQUIRE(shards >= 1 && m >= 1, "argmax merge: sizes must be positive");
    for (int r = 0; r < m; ++r) {
        int bs = 0;
        for (int g = 1; g < shards; ++g) {
            const float v = vals[(size_t)g * m + r], b = vals[(size_t)bs * m + r];
            const int32_t iv = ids[(size_t)g * m + r], ib = ids[(size_t)bs * m + r];
            if (v > b || (v == b && iv < ib) || (b != b && v == v)) bs = g;
        }
        out_val[r] = vals[(size_t)bs * m + r];
        out_id[r] = ids[(size_t)bs * m + r];
    }
    return FRS_OK;
}

// vocab.cpp:140-150
int frs_coverage(const uint64_t *counts, int vocab_size, const int32_t *ordered, int v_sub, double *out) {
    FRS_REQUIRE(counts && ordered && out, "coverage: null pointer");
    uint64_t total = 0, covered = 0;
    for (int t = 0; t < vocab_size; ++t) total += counts[t];
    if (total == 0) return fail(FRS_ELOGIC, "coverage: undefined for an empty corpus");
    for (int i = 0; i < v_sub; ++i) {
        FRS_REQUIRE(ordered[i] >= 0 && ordered[i] < vocab_size, "coverage: subset does not match the table vocabulary");
        covered += counts[ordered[i]];
    }
    *out = static_cast<double>(covered) / static_cast<double>(total);
    return FRS_OK;
}

// vocab.cpp:170-178
int frs_flops_ratio(int full_size, int restricted_size, double *out) {
    FRS_REQUIRE(out, "flops_ratio: null pointer");
    FRS_REQUIRE(full_size >= 1 && restricted_size >= 1, "flops_ratio: sizes must be positive");
    FRS_REQUIRE(restricted_size <= full_size, "flops_ratio: restricted size exceeds full size");
    *out = static_cast<double>(restricted_size) / static_cast<double>(full_size);
    return FRS_OK;
}

// verification.cpp:13-27
int frs_tree_mask(const int32_t *parents, int k, uint64_t *words) {
    if (k > 64) return fail(FRS_ECAPACITY, "build_tree_mask: " + std::to_string(k) + " nodes exceed the 64-bit mask");
    FRS_REQUIRE(k == 0 || (parents && words), "build_tree_mask: null pointer");
    for (int i = 0; i < k; ++i) {
        if (parents[i] >= i) return fail(FRS_EINVAL, "build_tree_mask: tree is not topological");
        words[i] = (parents[i] >= 0 ? words[parents[i]] : 0ull) | (1ull << i);
    }
    return FRS_OK;
}

int frs_head_create(frs_ctx *ctx, const float *W, int64_t V, int d, int w_on_device, const int32_t *ordered_ids,
                    int v_sub, int slab_dtype, frs_head **out) {
    FRS_REQUIRE(ctx && W && ordered_ids && out, "restrict_lm_head: null pointer");
    FRS_REQUIRE(V >= 1 && d >= 1 && v_sub >= 1 && v_sub <= V, "restrict_lm_head: bad sizes");
    FRS_REQUIRE(slab_dtype == FRS_DTYPE_F32 || slab_dtype == FRS_DTYPE_BF16, "restrict_lm_head: unknown dtype");
    for (int i = 0; i < v_sub; ++i)  // vocab.cpp:154-159
        if (ordered_ids[i] < 0 || ordered_ids[i] >= V)
            return fail(FRS_EINVAL, "restrict_lm_head: id " + std::to_string(ordered_ids[i]) +
                                        " out of range for the LM head");
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    frs_head *h = new frs_head();
    h->ctx = ctx;
    h->vocab = V;
    h->v_sub = v_sub;
    h->d = d;
    h->dtype = slab_dtype;
    h->ordered.assign(ordered_ids, ordered_ids + v_sub);
    auto cleanup = [&](int st) {
        frs_head_destroy(h);
        return st;
    };
    if (cudaMalloc(&h->slab, frs_slab_bytes(v_sub, d, slab_dtype)) != cudaSuccess ||
        cudaMalloc(&h->ordered_dev, sizeof(int32_t) * v_sub) != cudaSuccess)
        return cleanup(fail(FRS_ECUDA, "restrict_lm_head: cudaMalloc failed"));
    cudaStream_t s = ctx->stream;
    if (cudaMemcpyAsync(h->ordered_dev, ordered_ids, sizeof(int32_t) * v_sub, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return cleanup(fail(FRS_ECUDA, "restrict_lm_head: copy of ids failed"));
    const float *Wd = W;
    float *tmp = nullptr;
    if (!w_on_device) {  // stage only the subset rows: the gather happens on the host side of the copy
        if (cudaMalloc(&tmp, sizeof(float) * (size_t)v_sub * d) != cudaSuccess)
            return cleanup(fail(FRS_ECUDA, "restrict_lm_head: cudaMalloc failed"));
        for (int i = 0; i < v_sub; ++i)
            cudaMemcpyAsync(tmp + (size_t)i * d, W + (size_t)ordered_ids[i] * d, sizeof(float) * d,
                            cudaMemcpyHostToDevice, s);
        std::vector<int32_t> iota(v_sub);
        std::iota(iota.begin(), iota.end(), 0);
        int32_t *iota_dev = nullptr;
        cudaMalloc(&iota_dev, sizeof(int32_t) * v_sub);
        cudaMemcpyAsync(iota_dev, iota.data(), sizeof(int32_t) * v_sub, cudaMemcpyHostToDevice, s);
        int st = frs_slab_build(ctx, tmp, v_sub, d, iota_dev, v_sub, slab_dtype, h->slab, s);
        cudaFree(iota_dev);
        cudaFree(tmp);
        if (st) return cleanup(st);
    } else {
        int st = frs_slab_build(ctx, Wd, V, d, h->ordered_dev, v_sub, slab_dtype, h->slab, s);
        if (st) return cleanup(st);
    }
    if (slab_dtype == FRS_DTYPE_BF16 && d % 8 == 0) {  // the FAST head's stream-order image
        if (cudaMalloc(&h->tiled, frs_slab_tile_bytes(v_sub, d)) != cudaSuccess)
            return cleanup(fail(FRS_ECUDA, "restrict_lm_head: cudaMalloc failed"));
        if (int st = frs_slab_tile(ctx, h->slab, v_sub, d, h->tiled, s)) return cleanup(st);
    }
    *out = h;
    return FRS_OK;
}

int frs_head_destroy(frs_head *h) {
    if (!h) return FRS_OK;
    cudaSetDevice(h->ctx->device);
    if (h->slab) cudaFree(h->slab);
    if (h->tiled) cudaFree(h->tiled);
    if (h->ordered_dev) cudaFree(h->ordered_dev);
    if (h->h_ridx) cudaFreeHost(h->h_ridx);
    if (h->h_full) cudaFreeHost(h->h_full);
    if (h->h_prob) cudaFreeHost(h->h_prob);
    if (h->h_tok) cudaFreeHost(h->h_tok);
    delete h;
    return FRS_OK;
}

int frs_head_info(const frs_head *h, const void **slab, const int32_t **ordered_dev, int *v_sub, int *d,
                  int *slab_dtype) {
    FRS_REQUIRE(h, "null frs_head");
    if (slab) *slab = h->slab;
    if (ordered_dev) *ordered_dev = h->ordered_dev;
    if (v_sub) *v_sub = h->v_sub;
    if (d) *d = h->d;
    if (slab_dtype) *slab_dtype = h->dtype;
    return FRS_OK;
}

extern "C++" namespace frs {  // frs_tree.cu (C++ linkage inside this file's extern "C" block)
size_t tree_ws_bytes(int max_cand);
int tree_begin(void *ws, int max_cand, cudaStream_t s);
int tree_level(void *ws, int max_cand, const int32_t *pk, int nb, int w_children, int width, bool prune, int total,
               int32_t *next_tok, cudaStream_t s);
int tree_select(void *ws, int max_cand, int total, int32_t **out_dev, cudaStream_t s);
int step_rows_accept(const int32_t *tree_out, int32_t root, int total, int32_t *rt, int32_t *pp, int32_t *kdev,
                     cudaStream_t s);  // frs_misc.cu
int accept_greedy_devk(const int32_t *argmax_ids, const int32_t *tokens, const int32_t *parents,
                       const int32_t *kdev, int32_t *emitted, int32_t *path, int32_t *counts, cudaStream_t s);
}  // namespace frs

static int head_staging(frs_head *h, int rows, int k) {
    const size_t cells = (size_t)rows * k;
    int st;
    if ((st = h->lvl_ridx.ensure(cells * 12)) || (st = h->lvl_full.ensure(cells * 4)) ||
        (st = h->lvl_prob.ensure(cells * 4)) || (st = h->lvl_tok.ensure(64 * 4)) ||
        (st = h->hidden.ensure((size_t)std::max(rows, 64) * h->d * sizeof(float))))
        return st;
    if (!h->h_ridx) {
        const size_t cap = (size_t)64 * 64 * 4;
        if (cudaMallocHost(&h->h_ridx, 3 * cap) != cudaSuccess || cudaMallocHost(&h->h_full, cap) != cudaSuccess ||
            cudaMallocHost(&h->h_prob, cap) != cudaSuccess || cudaMallocHost(&h->h_tok, 64 * 4) != cudaSuccess)
            return fail(FRS_ECUDA, "pinned staging allocation failed");
    }
    FRS_REQUIRE(cells <= (size_t)64 * 64, "host draft step: at most 64 rows x 64 children");
    return FRS_OK;
}

int frs_head_draft_host(frs_head *h, const float *h_host, int n, int k, int mode, int32_t *ridx, int32_t *full,
                        float *prob) {
    FRS_REQUIRE(h && h_host && ridx && full && prob, "host draft step: null pointer");
    FRS_REQUIRE(n >= 1 && n <= 64 && k >= 1 && k <= 64, "host draft step: 1 <= n, k <= 64");
    FRS_CUDA_TRY(cudaSetDevice(h->ctx->device));
    int st = head_staging(h, n, k);
    if (st) return st;
    cudaStream_t s = h->ctx->stream;
    float *hd = static_cast<float *>(h->hidden.ptr);
    const size_t cells = (size_t)n * k;
    // FAST, one 16-row chain, pinned caller rows: no copy operations at all — k_hsplit reads the
    // rows over the bus from the mapped pinned buffer (writing the device copy the finalize
    // reads) and the finalize writes ids / probabilities straight into the pinned staging.
    // Otherwise: one H2D of the rows, outputs packed [ridx | full | prob] on the device, ONE D2H
    // (the caller's arrays may be pageable, where each async copy degrades to a staged sync copy).
    cudaPointerAttributes pa{};
    static const bool no_zero_copy = std::getenv("FRS_NO_ZERO_COPY") != nullptr;  // A/B switches
    static const bool no_graphs = std::getenv("FRS_NO_HOST_GRAPHS") != nullptr;
    const bool mapped = !no_zero_copy && mode == FRS_MODE_FAST && n <= 16 && h->dtype == FRS_DTYPE_BF16 &&
                        cudaPointerGetAttributes(&pa, h_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
                        pa.devicePointer != nullptr;
    cudaGetLastError();  // cudaPointerGetAttributes leaves no sticky error; clear any non-sticky one
    int32_t *hp = static_cast<int32_t *>(h->h_ridx);
    if (mapped) {
        // a synchronous call is latency-bound: replay the chain from a graph keyed on the buffers
        const bool graphs = h->ctx->prefer_graphs;
        h->ctx->h_stage_src = static_cast<const float *>(pa.devicePointer);
        h->ctx->prefer_graphs = !no_graphs;
        st = h->tiled ? frs_draft_head_topk_tiled(h->ctx, hd, n, h->d, h->slab, h->tiled, h->v_sub, h->ordered_dev, k,
                                                  1.0f, hp, hp + cells, reinterpret_cast<float *>(hp + 2 * cells),
                                                  nullptr, nullptr, nullptr, s)
                      : frs_draft_head_topk(h->ctx, hd, n, h->d, h->slab, h->v_sub, h->dtype, h->ordered_dev, k, 1.0f,
                                            mode, hp, hp + cells, reinterpret_cast<float *>(hp + 2 * cells), nullptr,
                                            nullptr, nullptr, nullptr, s);
        h->ctx->h_stage_src = nullptr;
        h->ctx->prefer_graphs = graphs;
        if (st) return st;
    } else {
        FRS_CUDA_TRY(cudaMemcpyAsync(hd, h_host, sizeof(float) * (size_t)n * h->d, cudaMemcpyHostToDevice, s));
        int32_t *pk = static_cast<int32_t *>(h->lvl_ridx.ptr);
        st = (mode == FRS_MODE_FAST && h->tiled)
                 ? frs_draft_head_topk_tiled(h->ctx, hd, n, h->d, h->slab, h->tiled, h->v_sub, h->ordered_dev, k, 1.0f,
                                             pk, pk + cells, reinterpret_cast<float *>(pk + 2 * cells), nullptr,
                                             nullptr, nullptr, s)
                 : frs_draft_head_topk(h->ctx, hd, n, h->d, h->slab, h->v_sub, h->dtype, h->ordered_dev, k, 1.0f, mode,
                                       pk, pk + cells, reinterpret_cast<float *>(pk + 2 * cells), nullptr, nullptr,
                                       nullptr, nullptr, s);
        if (st) return st;
        FRS_CUDA_TRY(cudaMemcpyAsync(hp, pk, cells * 12, cudaMemcpyDeviceToHost, s));
    }
    FRS_CUDA_TRY(cudaStreamSynchronize(s));
    std::memcpy(ridx, hp, cells * 4);
    std::memcpy(full, hp + cells, cells * 4);
    std::memcpy(prob, hp + 2 * cells, cells * 4);
    return FRS_OK;
}

// Device-resident tree chain (frs_tree.cu): enqueues gather -> K2 -> k_tree_level per level and
// the selection on the context stream, nothing synchronised; *out_dev = the selected tree
// ([0] count | [1] flags | tokens[64] | parents[64] | depths[64] | probs[64]), or nullptr when
// the shape needs the host bookkeeping. Callers ran head_staging(h, width, w).
static int tree_device_enqueue(frs_head *h, int32_t root_token, const float *hidden_table, int width, int depth,
                               int total, int w, int32_t **out_dev) {
    *out_dev = nullptr;
    static const bool no_dev_tree = std::getenv("FRS_HOST_TREE") != nullptr;  // DIAGNOSTIC
    if (!hidden_table || total > 64 || (size_t)w * width > 960 || no_dev_tree) return FRS_OK;
    int max_cand = w, nb = std::min(w, width);
    for (int level = 1; level < depth; ++level) {
        max_cand += nb * w;
        nb = std::min(nb * w, width);
    }
    if (max_cand > 2048) return FRS_OK;
    int st;
    cudaStream_t s = h->ctx->stream;
    float *hd = static_cast<float *>(h->hidden.ptr);
    int32_t *tok_dev = static_cast<int32_t *>(h->lvl_tok.ptr);
    if ((st = h->tree_ws.ensure(frs::tree_ws_bytes(max_cand)))) return st;
    void *ws = h->tree_ws.ptr;
    if ((st = frs::tree_begin(ws, max_cand, s))) return st;
    h->h_tok[0] = root_token;
    FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, h->h_tok, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    int rows = 1;
    int32_t *pk = static_cast<int32_t *>(h->lvl_ridx.ptr);
    for (int level = 0; level < depth && rows > 0; ++level) {
        if ((st = frs_gather_rows(h->ctx, hidden_table, h->vocab, h->d, tok_dev, rows, hd, s))) return st;
        const size_t cells = (size_t)rows * w;
        if ((st = frs_draft_head_topk(h->ctx, hd, rows, h->d, h->slab, h->v_sub, h->dtype, h->ordered_dev, w, 1.0f,
                                      FRS_MODE_EXACT, pk, pk + cells, reinterpret_cast<float *>(pk + 2 * cells),
                                      nullptr, nullptr, nullptr, nullptr, s)))
            return st;
        if ((st = frs::tree_level(ws, max_cand, pk, rows, w, width, level + 1 < depth, total, tok_dev, s))) return st;
        rows = std::min(rows * w, width);
    }
    return frs::tree_select(ws, max_cand, total, out_dev, s);
}

// The selected tree read back from tree_device_enqueue's output; log_joint in the reference's
// accumulation order (parents first). Returns the node count.
static int tree_from_out(const int32_t *ho, int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint) {
    const int K = ho[0];
    const int32_t *tk = ho + 2, *pa = tk + 64, *dp = pa + 64, *pr = dp + 64;
    for (int i = 0; i < K; ++i) {
        float p;
        std::memcpy(&p, pr + i, 4);
        const double lg = std::log(static_cast<double>(p));
        tokens[i] = tk[i];
        parents[i] = pa[i];
        depths[i] = dp[i];
        log_joint[i] = pa[i] < 0 ? lg : log_joint[pa[i]] + lg;
    }
    return K;
}

// drafting.cpp:122-245, greedy, head path: per level the provider supplies the forwarded
// rows' hidden states, the device runs K2, the host keeps the reference's beam bookkeeping.
int frs_draft_tree(frs_head *h, int32_t root_token, frs_hidden_fn fn, void *user, const float *hidden_table,
                   int width, int depth, int total, int mode, int32_t *tokens, int32_t *parents, int32_t *depths,
                   double *log_joint, int *count) {
    FRS_REQUIRE(h && tokens && parents && depths && log_joint && count, "build_draft_tree: null pointer");
    if (width < 1) return fail(FRS_EINVAL, "draft params: beam_width must be >= 1");
    if (depth < 1) return fail(FRS_EINVAL, "draft params: search_depth must be >= 1");
    if (total < width || total > 64)
        return fail(FRS_EINVAL, "draft params: total_draft_tokens must lie in [beam_width, 64]");
    FRS_REQUIRE(fn || hidden_table, "build_draft_tree: need a hidden provider or a hidden table");
    FRS_REQUIRE(mode == FRS_MODE_EXACT || mode == FRS_MODE_FAST, "build_draft_tree: unknown mode");
    // The levels always run EXACT: beam pruning and select_top_k compare log_joints of children
    // of DIFFERENT rows, i.e. log(e_j / Σ_row) across rows, so every row's 1 / Σ must be the
    // reference's (kernels.cpp:86-89). FAST's Σ comes from tensor-core logits whose rigorous
    // error bound (~0.09 in log space at the Llama-3-8B shape) exceeds the typical gap at a
    // beam cut, so no FAST tree could be certified; the exact Σ needs every logit in dot_f32
    // order, which is the EXACT level itself. FAST is accepted for API compatibility.
    mode = FRS_MODE_EXACT;
    FRS_CUDA_TRY(cudaSetDevice(h->ctx->device));
    const int w = std::min(width, h->v_sub);  // drafting.cpp:40
    int st = head_staging(h, width, w);
    if (st) return st;
    cudaStream_t s = h->ctx->stream;
    float *hd = static_cast<float *>(h->hidden.ptr);
    int32_t *tok_dev = static_cast<int32_t *>(h->lvl_tok.ptr);

    // Device-resident beam bookkeeping (frs_tree.cu) when the hidden rows come from a table:
    // every level runs gather -> K2 -> k_tree_level with no host round trip, then one D2H of
    // the selected nodes. An uncertified ordering decision (see frs_tree.cu) falls through to
    // the host bookkeeping below.
    if (!fn) {
        int32_t *out_dev = nullptr;
        if ((st = tree_device_enqueue(h, root_token, hidden_table, width, depth, total, w, &out_dev))) return st;
        if (out_dev) {
            int32_t *ho = h->h_ridx;  // pinned staging
            FRS_CUDA_TRY(cudaMemcpyAsync(ho, out_dev, sizeof(int32_t) * (2 + 4 * 64), cudaMemcpyDeviceToHost, s));
            FRS_CUDA_TRY(cudaStreamSynchronize(s));
            if (ho[1] == 0) {
                *count = tree_from_out(ho, tokens, parents, depths, log_joint);
                return FRS_OK;
            }
        }
    }

    std::vector<Cand> cands;
    std::vector<int> beam;
    std::vector<int32_t> btok, bpar;
    auto run_level = [&](int level, int nb) -> int {
        if (fn) {
            tl_beam_cands = level == 0 ? nullptr : beam.data();
            const int rc = fn(user, level, nb, btok.data(), bpar.data(), hd, s);
            if (rc) return fail(FRS_ELOGIC, "hidden provider failed with code " + std::to_string(rc));
        } else {
            std::memcpy(h->h_tok, btok.data(), sizeof(int32_t) * nb);
            FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, h->h_tok, sizeof(int32_t) * nb, cudaMemcpyHostToDevice, s));
            const int rc = frs_gather_rows(h->ctx, hidden_table, h->vocab, h->d, tok_dev, nb, hd, s);
            if (rc) return rc;
        }
        // outputs packed [ridx | full | prob] (cells each) in lvl_ridx: one D2H per level
        const size_t cells = (size_t)nb * w;
        int32_t *pk = static_cast<int32_t *>(h->lvl_ridx.ptr);
        int rc = frs_draft_head_topk(h->ctx, hd, nb, h->d, h->slab, h->v_sub, h->dtype, h->ordered_dev, w, 1.0f, mode,
                                     pk, pk + cells, reinterpret_cast<float *>(pk + 2 * cells), nullptr, nullptr,
                                     nullptr, nullptr, s);
        if (rc) return rc;
        FRS_CUDA_TRY(cudaMemcpyAsync(h->h_ridx, pk, cells * 12, cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaStreamSynchronize(s));
        std::memcpy(h->h_full, h->h_ridx + cells, cells * 4);
        std::memcpy(h->h_prob, h->h_ridx + 2 * cells, cells * 4);
        return FRS_OK;
    };

    // Forward 1 of search_depth: the root row (drafting.cpp:133-160).
    btok.assign(1, root_token);
    bpar.assign(1, -1);
    if ((st = run_level(0, 1))) return st;
    for (int c = 0; c < w; ++c) {
        beam.push_back(static_cast<int>(cands.size()));
        cands.push_back({h->h_full[c], h->h_ridx[c], -1, 1, std::log(static_cast<double>(h->h_prob[c]))});
    }
    for (int level = 1; level < depth && !beam.empty(); ++level) {
        if (static_cast<int>(beam.size()) > width) {  // drafting.cpp:164-176
            std::sort(beam.begin(), beam.end(), ByLogJoint{&cands});
            beam.resize(width);
            std::sort(beam.begin(), beam.end());
        }
        const int nb = static_cast<int>(beam.size());
        btok.resize(nb);
        bpar.resize(nb);
        for (int i = 0; i < nb; ++i) {
            btok[i] = cands[beam[i]].token;
            bpar[i] = cands[beam[i]].parent;
        }
        if ((st = run_level(level, nb))) return st;
        std::vector<int> next;
        for (int i = 0; i < nb; ++i) {  // drafting.cpp:199-220 (parent fields read by value)
            const int pidx = beam[i];
            const int pdepth = cands[pidx].depth;
            const double plj = cands[pidx].log_joint;
            for (int c = 0; c < w; ++c) {
                const size_t o = (size_t)i * w + c;
                next.push_back(static_cast<int>(cands.size()));
                cands.push_back({h->h_full[o], h->h_ridx[o], pidx, pdepth + 1,
                                 plj + std::log(static_cast<double>(h->h_prob[o]))});
            }
        }
        beam = std::move(next);
    }
    // select_top_k (drafting.cpp:93-118, prefix_closed = false) and emit (230-244)
    std::vector<int> order(cands.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), ByLogJoint{&cands});
    std::vector<char> sel(cands.size(), 0);
    int cnt = 0;
    for (int c : order) {
        if (sel[c]) continue;
        if (cands[c].parent >= 0 && !sel[cands[c].parent]) continue;
        if (cnt + 1 > total) continue;
        sel[c] = 1;
        ++cnt;
    }
    std::vector<int> remap(cands.size(), -1);
    int out = 0;
    for (size_t i = 0; i < cands.size(); ++i) {
        if (!sel[i]) continue;
        remap[i] = out;
        tokens[out] = cands[i].token;
        parents[out] = cands[i].parent >= 0 ? remap[cands[i].parent] : -1;
        depths[out] = cands[i].depth;
        log_joint[out] = cands[i].log_joint;
        ++out;
    }
    *count = out;
    return FRS_OK;
}

// Pinned staging shared by the verify entry points (one H2D of the tree, one D2H of the result).
static int ctx_pinned(frs_ctx *ctx, size_t bytes) {
    if (ctx->pinned_bytes >= bytes) return FRS_OK;
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    if (cudaMallocHost(&ctx->pinned, bytes) != cudaSuccess) return fail(FRS_ECUDA, "pinned staging allocation failed");
    ctx->pinned_bytes = bytes;
    return FRS_OK;
}

// The verify head's argmax over m rows: FAST with the head's tiled image when the caller has one.
static int verify_argmax_rows(frs_ctx *ctx, const float *hd, int m, int d, const void *W, const void *W_tiled, int V,
                              int w_dtype, int mode, int32_t *ids, cudaStream_t s) {
    if (W_tiled && mode == FRS_MODE_FAST && w_dtype == FRS_DTYPE_BF16)
        return frs_verify_head_argmax_tiled(ctx, hd, m, d, W, W_tiled, V, 0, ids, nullptr, nullptr, s);
    return frs_verify_head_argmax(ctx, hd, m, d, W, V, w_dtype, 0, mode, ids, nullptr, nullptr, s);
}

// verify_greedy (verification.cpp:42-71) on the device: verify head argmax over the 1 + k rows
// of h_dev (root first), the accept walk, one packed D2H. table != nullptr: h_dev is ignored
// and the rows are gathered from table[V_table x d] by [root_token, tokens...] on the device.
static int verify_greedy_impl(frs_ctx *ctx, const float *h_dev, const float *table, int64_t V_table, int32_t root_token,
                              const void *W, int V, int d, int w_dtype, int mode, const int32_t *tokens,
                              const int32_t *parents, int k, int32_t *emitted, int *n_emitted, int32_t *path,
                              int *n_path, const void *W_tiled = nullptr) {
    if (k > 64) return fail(FRS_ECAPACITY, "build_tree_mask: nodes exceed the 64-bit mask");
    FRS_REQUIRE(k >= 0 && (k == 0 || (tokens && parents)), "verify_greedy: bad tree");
    for (int i = 0; i < k; ++i)
        if (parents[i] >= i || parents[i] < -1) return fail(FRS_EINVAL, "verify_greedy: tree is not topological");
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // device: argmax ids [65] | root+tokens [65] | parents [64] | emitted [65] | path [64] | counts [2]
    int st = ctx->obuf.ensure(sizeof(int32_t) * 336);
    if (st) return st;
    if ((st = ctx_pinned(ctx, sizeof(int32_t) * 336))) return st;
    int32_t *ids = static_cast<int32_t *>(ctx->obuf.ptr);
    int32_t *rt = ids + 65, *pp = rt + 65, *d_em = pp + 64, *d_path = d_em + 65, *d_cnt = d_path + 64;
    int32_t *hp = static_cast<int32_t *>(ctx->pinned);  // same layout from rt on
    hp[0] = root_token;
    std::copy(tokens, tokens + k, hp + 1);
    std::copy(parents, parents + k, hp + 65);
    FRS_CUDA_TRY(cudaMemcpyAsync(rt, hp, sizeof(int32_t) * (65 + 64), cudaMemcpyHostToDevice, s));
    const float *hd = h_dev;
    if (table) {
        if ((st = ctx->hbuf.ensure((size_t)(1 + k) * d * sizeof(float)))) return st;
        if ((st = frs_gather_rows(ctx, table, V_table, d, rt, 1 + k, static_cast<float *>(ctx->hbuf.ptr), s))) return st;
        hd = static_cast<const float *>(ctx->hbuf.ptr);
    }
    st = verify_argmax_rows(ctx, hd, 1 + k, d, W, W_tiled, V, w_dtype, mode, ids, s);
    if (st) return st;
    st = frs_accept_greedy(ctx, ids, rt + 1, pp, k, d_em, d_path, d_cnt, s);
    if (st) return st;
    int32_t *ho = hp + 129;  // emitted [65] | path [64] | counts [2]
    FRS_CUDA_TRY(cudaMemcpyAsync(ho, d_em, sizeof(int32_t) * (65 + 64 + 2), cudaMemcpyDeviceToHost, s));
    FRS_CUDA_TRY(cudaStreamSynchronize(s));
    *n_emitted = ho[129];
    *n_path = ho[130];
    std::copy(ho, ho + *n_emitted, emitted);
    std::copy(ho + 65, ho + 65 + *n_path, path);
    return FRS_OK;
}

int frs_verify_greedy(frs_ctx *ctx, const float *h_dev, const void *W, int V, int d, int w_dtype, int mode,
                      const int32_t *tokens, const int32_t *parents, int k, int32_t *emitted, int *n_emitted,
                      int32_t *path, int *n_path) {
    FRS_REQUIRE(ctx && h_dev && W && emitted && n_emitted && path && n_path, "verify_greedy: null pointer");
    return verify_greedy_impl(ctx, h_dev, nullptr, 0, 0, W, V, d, w_dtype, mode, tokens, parents, k, emitted,
                              n_emitted, path, n_path);
}

int frs_verify_greedy_table(frs_ctx *ctx, const float *table, int64_t V_table, int32_t root_token, const void *W,
                            int V, int d, int w_dtype, int mode, const int32_t *tokens, const int32_t *parents, int k,
                            int32_t *emitted, int *n_emitted, int32_t *path, int *n_path) {
    FRS_REQUIRE(ctx && table && W && emitted && n_emitted && path && n_path, "verify_greedy: null pointer");
    FRS_REQUIRE(root_token >= 0 && root_token < V_table, "verify_greedy: root token outside the hidden table");
    for (int i = 0; i < k; ++i)
        FRS_REQUIRE(tokens[i] >= 0 && tokens[i] < V_table, "verify_greedy: token outside the hidden table");
    return verify_greedy_impl(ctx, nullptr, table, V_table, root_token, W, V, d, w_dtype, mode, tokens, parents, k,
                              emitted, n_emitted, path, n_path);
}

// One head-path decode iteration with no host round trip between drafting and verification:
// the device-resident tree (tree_device_enqueue), the verify rows built from the selected tree
// on the device (k_step_rows: [root, tokens..., root padding to 1 + total]), the verify head
// argmax over them, the accept walk with the device node count, then ONE synchronisation for
// both results. Same results as frs_draft_tree + frs_verify_greedy_table: verify rows are
// independent of each other, padding rows are never read by the walk. Shapes outside the
// device tree, or an uncertified tree ordering, run those two calls instead.
static int decode_step_impl(frs_head *h, const float *table, int32_t root_token, const void *W, const void *W_tiled,
                            int V, int w_dtype, int verify_mode, int width, int depth, int total, int32_t *tokens,
                            int32_t *parents, int32_t *depths, double *log_joint, int *count, int32_t *emitted,
                            int *n_emitted, int32_t *path, int *n_path) {
    FRS_REQUIRE(h && table && W && tokens && parents && depths && log_joint && count && emitted && n_emitted &&
                    path && n_path,
                "decode_step: null pointer");
    if (width < 1) return fail(FRS_EINVAL, "draft params: beam_width must be >= 1");
    if (depth < 1) return fail(FRS_EINVAL, "draft params: search_depth must be >= 1");
    if (total < width || total > 64)
        return fail(FRS_EINVAL, "draft params: total_draft_tokens must lie in [beam_width, 64]");
    FRS_REQUIRE(root_token >= 0 && root_token < h->vocab, "verify_greedy: root token outside the hidden table");
    FRS_REQUIRE(verify_mode == FRS_MODE_EXACT || verify_mode == FRS_MODE_FAST, "decode_step: unknown mode");
    frs_ctx *ctx = h->ctx;
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    const int w = std::min(width, h->v_sub), d = h->d;
    int st = head_staging(h, width, w);
    if (st) return st;
    cudaStream_t s = ctx->stream;
    int32_t *out_dev = nullptr;
    if ((st = tree_device_enqueue(h, root_token, table, width, depth, total, w, &out_dev))) return st;
    if (out_dev) {
        // device: argmax ids [65] | root+tokens [65] | parents [64] | emitted [65] | path [64] | counts [2] | k
        if ((st = ctx->obuf.ensure(sizeof(int32_t) * 337)) || (st = ctx_pinned(ctx, sizeof(int32_t) * 336)) ||
            (st = ctx->hbuf.ensure((size_t)(1 + total) * d * sizeof(float))))
            return st;
        int32_t *ids = static_cast<int32_t *>(ctx->obuf.ptr);
        int32_t *rt = ids + 65, *pp = rt + 65, *d_em = pp + 64, *d_path = d_em + 65, *d_cnt = d_path + 64;
        int32_t *kdev = d_cnt + 2;
        float *hv = static_cast<float *>(ctx->hbuf.ptr);
        ++ctx->launches;
        if ((st = frs::step_rows_accept(out_dev, root_token, total, rt, pp, kdev, s))) return st;
        if ((st = frs_gather_rows(ctx, table, h->vocab, d, rt, 1 + total, hv, s))) return st;
        if ((st = verify_argmax_rows(ctx, hv, 1 + total, d, W, W_tiled, V, w_dtype, verify_mode, ids, s))) return st;
        ++ctx->launches;
        if ((st = frs::accept_greedy_devk(ids, rt + 1, pp, kdev, d_em, d_path, d_cnt, s))) return st;
        int32_t *ht = h->h_ridx, *hv_out = static_cast<int32_t *>(ctx->pinned) + 129;
        FRS_CUDA_TRY(cudaMemcpyAsync(ht, out_dev, sizeof(int32_t) * (2 + 4 * 64), cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaMemcpyAsync(hv_out, d_em, sizeof(int32_t) * (65 + 64 + 2), cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaStreamSynchronize(s));
        if (ht[1] == 0) {
            *count = tree_from_out(ht, tokens, parents, depths, log_joint);
            *n_emitted = hv_out[129];
            *n_path = hv_out[130];
            std::copy(hv_out, hv_out + *n_emitted, emitted);
            std::copy(hv_out + 65, hv_out + 65 + *n_path, path);
            return FRS_OK;
        }
    }
    if ((st = frs_draft_tree(h, root_token, nullptr, nullptr, table, width, depth, total, FRS_MODE_EXACT, tokens,
                             parents, depths, log_joint, count)))
        return st;
    return verify_greedy_impl(ctx, nullptr, table, h->vocab, root_token, W, V, d, w_dtype, verify_mode, tokens,
                              parents, *count, emitted, n_emitted, path, n_path, W_tiled);
}

int frs_decode_step_table(frs_head *h, const float *table, int32_t root_token, const void *W, int V, int w_dtype,
                          int verify_mode, int width, int depth, int total, int32_t *tokens, int32_t *parents,
                          int32_t *depths, double *log_joint, int *count, int32_t *emitted, int *n_emitted,
                          int32_t *path, int *n_path) {
    return decode_step_impl(h, table, root_token, W, nullptr, V, w_dtype, verify_mode, width, depth, total, tokens,
                            parents, depths, log_joint, count, emitted, n_emitted, path, n_path);
}

int frs_decode_step_table_tiled(frs_head *h, const float *table, int32_t root_token, const void *W, const void *W_tiled,
                                int V, int verify_mode, int width, int depth, int total, int32_t *tokens,
                                int32_t *parents, int32_t *depths, double *log_joint, int *count, int32_t *emitted,
                                int *n_emitted, int32_t *path, int *n_path) {
    FRS_REQUIRE(W_tiled, "decode_step: null pointer");
    return decode_step_impl(h, table, root_token, W, W_tiled, V, FRS_DTYPE_BF16, verify_mode, width, depth, total,
                            tokens, parents, depths, log_joint, count, emitted, n_emitted, path, n_path);
}

// S independent decode streams, one head-path iteration each (drafting.cpp:122-245 then
// verification.cpp:42-71 per stream), batched across streams: every draft level is ONE EXACT
// head call over all streams' beam rows (rows are independent: drafting.cpp:189-193), the
// beam / select_top_k bookkeeping runs per stream on the host in the reference's order, and the
// verify head is ONE call over all streams' [root, tokens...] rows followed by each stream's
// accept walk. Per stream the results equal frs_decode_step_table (same arithmetic per row).
// Outputs are [S][total] (tokens, parents, depths, log_joint, path), [S][total + 1] (emitted) and
// [S] (count, n_emitted, n_path).
int frs_decode_step_table_multi(frs_head *h, const float *table, int S, const int32_t *roots, const void *W,
                                const void *W_tiled, int V, int w_dtype, int verify_mode, int width, int depth,
                                int total, int32_t *tokens,
                                int32_t *parents, int32_t *depths, double *log_joint, int *count, int32_t *emitted,
                                int *n_emitted, int32_t *path, int *n_path) {
    FRS_REQUIRE(h && table && roots && W && tokens && parents && depths && log_joint && count && emitted &&
                    n_emitted && path && n_path,
                "decode_step: null pointer");
    FRS_REQUIRE(S >= 1, "decode_step: at least one stream");
    if (width < 1) return fail(FRS_EINVAL, "draft params: beam_width must be >= 1");
    if (depth < 1) return fail(FRS_EINVAL, "draft params: search_depth must be >= 1");
    if (total < width || total > 64)
        return fail(FRS_EINVAL, "draft params: total_draft_tokens must lie in [beam_width, 64]");
    for (int q = 0; q < S; ++q)
        FRS_REQUIRE(roots[q] >= 0 && roots[q] < h->vocab, "verify_greedy: root token outside the hidden table");
    FRS_REQUIRE(verify_mode == FRS_MODE_EXACT || verify_mode == FRS_MODE_FAST, "decode_step: unknown mode");
    frs_ctx *ctx = h->ctx;
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int w = std::min(width, h->v_sub), d = h->d;  // drafting.cpp:40
    const size_t max_rows = (size_t)S * std::max(width, 1 + total);
    int st;
    if ((st = h->ms_tok.ensure(max_rows * 4)) || (st = h->ms_hidden.ensure(max_rows * d * sizeof(float))) ||
        (st = h->ms_out.ensure(std::max((size_t)S * width * w * 12, max_rows * 4))))
        return st;
    int32_t *tok_dev = static_cast<int32_t *>(h->ms_tok.ptr);
    float *hd = static_cast<float *>(h->ms_hidden.ptr);
    int32_t *pk = static_cast<int32_t *>(h->ms_out.ptr);
    std::vector<int32_t> rtok, hout;
    std::vector<std::vector<Cand>> cands(S);
    std::vector<std::vector<int>> beam(S);
    std::vector<int> roff(S + 1);
    // one EXACT level over rtok (all streams' rows): packed [ridx | full | prob] back to the host
    auto run_level = [&](int nrows) -> int {
        FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, rtok.data(), sizeof(int32_t) * nrows, cudaMemcpyHostToDevice, s));
        int rc = frs_gather_rows(ctx, table, h->vocab, d, tok_dev, nrows, hd, s);
        if (rc) return rc;
        const size_t cells = (size_t)nrows * w;
        rc = frs_draft_head_topk(ctx, hd, nrows, d, h->slab, h->v_sub, h->dtype, h->ordered_dev, w, 1.0f,
                                 FRS_MODE_EXACT, pk, pk + cells, reinterpret_cast<float *>(pk + 2 * cells), nullptr,
                                 nullptr, nullptr, nullptr, s);
        if (rc) return rc;
        hout.resize(cells * 3);
        FRS_CUDA_TRY(cudaMemcpyAsync(hout.data(), pk, cells * 12, cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaStreamSynchronize(s));
        return FRS_OK;
    };
    auto child = [&](size_t cells, size_t o, int parent, int pdepth, double plj) {
        float p;
        std::memcpy(&p, &hout[2 * cells + o], 4);
        return Cand{hout[cells + o], hout[o], parent, pdepth + 1, plj + std::log(static_cast<double>(p))};
    };
    // Forward 1 of search_depth: the roots (drafting.cpp:133-160), one row per stream
    rtok.assign(roots, roots + S);
    if ((st = run_level(S))) return st;
    for (int q = 0; q < S; ++q)
        for (int c = 0; c < w; ++c) {
            beam[q].push_back(static_cast<int>(cands[q].size()));
            cands[q].push_back(child((size_t)S * w, (size_t)q * w + c, -1, 0, 0.0));
        }
    for (int level = 1; level < depth; ++level) {
        rtok.clear();
        for (int q = 0; q < S; ++q) {
            std::vector<int> &b = beam[q];
            if (static_cast<int>(b.size()) > width) {  // drafting.cpp:164-176
                std::sort(b.begin(), b.end(), ByLogJoint{&cands[q]});
                b.resize(width);
                std::sort(b.begin(), b.end());
            }
            roff[q] = static_cast<int>(rtok.size());
            for (int i : b) rtok.push_back(cands[q][i].token);
        }
        roff[S] = static_cast<int>(rtok.size());
        if (rtok.empty()) break;
        if ((st = run_level(roff[S]))) return st;
        const size_t cells = (size_t)roff[S] * w;
        for (int q = 0; q < S; ++q) {  // drafting.cpp:199-220 (parent fields read by value)
            std::vector<int> next;
            for (size_t i = 0; i < beam[q].size(); ++i) {
                const int pidx = beam[q][i];
                const int pdepth = cands[q][pidx].depth;
                const double plj = cands[q][pidx].log_joint;
                for (int c = 0; c < w; ++c) {
                    next.push_back(static_cast<int>(cands[q].size()));
                    cands[q].push_back(child(cells, (size_t)(roff[q] + i) * w + c, pidx, pdepth, plj));
                }
            }
            beam[q] = std::move(next);
        }
    }
    // select_top_k (drafting.cpp:93-118, prefix_closed = false) and emit (230-244), per stream;
    // then the verify rows [root, tokens...] of every stream
    rtok.clear();
    for (int q = 0; q < S; ++q) {
        const std::vector<Cand> &cq = cands[q];
        std::vector<int> order(cq.size());
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), ByLogJoint{&cq});
        std::vector<char> sel(cq.size(), 0);
        int cnt = 0;
        for (int c : order) {
            if (sel[c]) continue;
            if (cq[c].parent >= 0 && !sel[cq[c].parent]) continue;
            if (cnt + 1 > total) continue;
            sel[c] = 1;
            ++cnt;
        }
        std::vector<int> remap(cq.size(), -1);
        int out = 0;
        int32_t *tq = tokens + (size_t)q * total, *pq = parents + (size_t)q * total, *dq = depths + (size_t)q * total;
        double *lq = log_joint + (size_t)q * total;
        for (size_t i = 0; i < cq.size(); ++i) {
            if (!sel[i]) continue;
            remap[i] = out;
            tq[out] = cq[i].token;
            pq[out] = cq[i].parent >= 0 ? remap[cq[i].parent] : -1;
            dq[out] = cq[i].depth;
            lq[out] = cq[i].log_joint;
            ++out;
        }
        count[q] = out;
        roff[q] = static_cast<int>(rtok.size());
        rtok.push_back(roots[q]);
        rtok.insert(rtok.end(), tq, tq + out);
    }
    roff[S] = static_cast<int>(rtok.size());
    // verify head argmax over every stream's rows (rows are independent), then each stream's
    // accept walk (verification.cpp:42-71): emit the argmax at the current node, follow the first
    // child (by index) carrying it, stop at the bonus token
    const int R = roff[S];
    FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, rtok.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice, s));
    if ((st = frs_gather_rows(ctx, table, h->vocab, d, tok_dev, R, hd, s))) return st;
    if ((st = verify_argmax_rows(ctx, hd, R, d, W, W_tiled, V, w_dtype, verify_mode, pk, s))) return st;
    std::vector<int32_t> ids(R);
    FRS_CUDA_TRY(cudaMemcpyAsync(ids.data(), pk, sizeof(int32_t) * R, cudaMemcpyDeviceToHost, s));
    FRS_CUDA_TRY(cudaStreamSynchronize(s));
    for (int q = 0; q < S; ++q) {
        const int k = count[q];
        const int32_t *tq = tokens + (size_t)q * total, *pq = parents + (size_t)q * total, *aq = ids.data() + roff[q];
        int32_t *eq = emitted + (size_t)q * (total + 1), *wq = path + (size_t)q * total;
        int node = -1, ne = 0, np = 0;
        for (int step = 0; step <= k; ++step) {
            const int32_t best = aq[node + 1];
            int match = -1;
            for (int c = 0; c < k && match < 0; ++c)
                if (pq[c] == node && tq[c] == best) match = c;
            eq[ne++] = best;
            if (match < 0) break;
            wq[np++] = match;
            node = match;
        }
        n_emitted[q] = ne;
        n_path[q] = np;
    }
    return FRS_OK;
}

int frs_rng_create(uint64_t seed, frs_rng **out) {
    FRS_REQUIRE(out, "rng: null pointer");
    *out = new frs_rng{std::mt19937_64(seed)};
    return FRS_OK;
}

int frs_rng_destroy(frs_rng *rng) {
    delete rng;
    return FRS_OK;
}

int frs_rng_uniforms(frs_rng *rng, int count, double *out) {
    FRS_REQUIRE(rng && out && count >= 0, "rng: bad arguments");
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    for (int i = 0; i < count; ++i) out[i] = uni(rng->engine);
    return FRS_OK;
}

// build_draft_tree with an rng (drafting.cpp:122-245), head path, EXACT arithmetic: per level
// the device samples every row (frs_draft_head_sample) with uniforms drawn here in the
// reference's order (row by row, draw by draw); a level with an uncertified draw or an early
// stop is replayed on the host from the device's exact probabilities with the engine rewound
// to the level's start. select_top_k is prefix-closed (drafting.cpp:93-118).
int frs_draft_tree_sampled(frs_head *h, int32_t root_token, frs_hidden_fn fn, void *user, const float *hidden_table,
                           int width, int depth, int total, frs_rng *rng, int32_t *tokens, int32_t *parents,
                           int32_t *depths, double *log_joint, int *count, float *root_probs, float *node_probs,
                           int32_t *has_probs) {
    FRS_REQUIRE(h && rng && tokens && parents && depths && log_joint && count, "build_draft_tree: null pointer");
    if (width < 1) return fail(FRS_EINVAL, "draft params: beam_width must be >= 1");
    if (depth < 1) return fail(FRS_EINVAL, "draft params: search_depth must be >= 1");
    if (total < width || total > 64)
        return fail(FRS_EINVAL, "draft params: total_draft_tokens must lie in [beam_width, 64]");
    FRS_REQUIRE(fn || hidden_table, "build_draft_tree: need a hidden provider or a hidden table");
    FRS_CUDA_TRY(cudaSetDevice(h->ctx->device));
    const int w = std::min(width, h->v_sub);
    int st = head_staging(h, width, w);
    if (st) return st;
    cudaStream_t s = h->ctx->stream;
    float *hd = static_cast<float *>(h->hidden.ptr);
    int32_t *tok_dev = static_cast<int32_t *>(h->lvl_tok.ptr);
    const int max_rows = std::max(1, width);
    if ((st = h->smp_u.ensure((size_t)max_rows * w * sizeof(double))) ||
        (st = h->smp_probs.ensure((size_t)max_rows * h->v_sub * sizeof(float))))
        return st;
    struct SCand {
        int32_t token, ridx, parent, depth, sibling_rank;
        double log_joint;
    };
    std::vector<SCand> cands;
    std::vector<int> beam;
    std::vector<int32_t> btok, bpar;
    std::vector<double> uh;
    std::vector<int> idx;
    std::vector<float> pr, probs_host;
    // keep_probs (drafting.cpp:140-141, 219, 236-238): the distribution of every expanded node,
    // by candidate index (-1: the root anchor), copied out of the level's exact probabilities
    const bool keep = root_probs || node_probs;
    FRS_REQUIRE(!node_probs || has_probs, "build_draft_tree: node_probs needs has_probs");
    std::vector<std::vector<float>> kept;  // by candidate index
    std::vector<float> root_kept;
    // one level: hidden rows, device sampling (or host replay), children appended in beam order
    auto run_level = [&](int level, int nb, const std::vector<int> &parents_of_rows) -> int {
        if (fn) {
            tl_beam_cands = level == 0 ? nullptr : parents_of_rows.data();
            const int rc = fn(user, level, nb, btok.data(), bpar.data(), hd, s);
            if (rc) return fail(FRS_ELOGIC, "hidden provider failed with code " + std::to_string(rc));
        } else {
            std::memcpy(h->h_tok, btok.data(), sizeof(int32_t) * nb);
            FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, h->h_tok, sizeof(int32_t) * nb, cudaMemcpyHostToDevice, s));
            const int rc = frs_gather_rows(h->ctx, hidden_table, h->vocab, h->d, tok_dev, nb, hd, s);
            if (rc) return rc;
        }
        const std::mt19937_64 saved = rng->engine;  // the level's start, for a host replay
        uh.resize((size_t)nb * w);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        for (auto &u : uh) u = uni(rng->engine);
        FRS_CUDA_TRY(cudaMemcpyAsync(h->smp_u.ptr, uh.data(), uh.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        const size_t cells = (size_t)nb * w;
        int32_t *pk = static_cast<int32_t *>(h->lvl_ridx.ptr);  // [ridx | full | prob | count | flags]
        if ((st = h->lvl_ridx.ensure(cells * 12 + (size_t)nb * 8))) return st;
        pk = static_cast<int32_t *>(h->lvl_ridx.ptr);
        int rc = frs_draft_head_sample(h->ctx, hd, nb, h->d, h->slab, h->v_sub, h->dtype, h->ordered_dev, width, 1.0f,
                                       static_cast<const double *>(h->smp_u.ptr),
                                       static_cast<float *>(h->smp_probs.ptr), pk, pk + cells,
                                       reinterpret_cast<float *>(pk + 2 * cells), pk + 3 * cells,
                                       reinterpret_cast<uint32_t *>(pk + 3 * cells + nb), s);
        if (rc) return rc;
        std::vector<int32_t> hb(cells * 3 + (size_t)nb * 2);
        FRS_CUDA_TRY(cudaMemcpyAsync(hb.data(), pk, hb.size() * 4, cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaStreamSynchronize(s));
        bool replay = false;
        for (int i = 0; i < nb; ++i)
            if (hb[3 * cells + i] != w || (hb[3 * cells + nb + i] & FRS_FLAG_SAMPLE_UNCERTIFIED)) replay = true;
        for (int i = 0; i < nb; ++i)
            if (hb[3 * cells + nb + i] & FRS_FLAG_NONFINITE)
                return fail(FRS_EINVAL, "softmax: non-finite logit");  // kernels.cpp:72-74
        if (replay || keep) {  // rewind and redo the whole level on the host (rows in order) / keep_probs
            if (replay) rng->engine = saved;
            probs_host.resize((size_t)nb * h->v_sub);
            FRS_CUDA_TRY(cudaMemcpy(probs_host.data(), h->smp_probs.ptr, probs_host.size() * sizeof(float),
                                    cudaMemcpyDeviceToHost));
        }
        if (keep) {
            for (int i = 0; i < nb; ++i) {
                const float *row = probs_host.data() + (size_t)i * h->v_sub;
                const int par = parents_of_rows[i];
                if (par < 0) {
                    root_kept.assign(row, row + h->v_sub);
                } else {
                    if ((int)kept.size() <= par) kept.resize(par + 1);
                    kept[par].assign(row, row + h->v_sub);
                }
            }
        }
        for (int i = 0; i < nb; ++i) {
            int m;
            if (replay) {
                pick_sampled_host(probs_host.data() + (size_t)i * h->v_sub, h->v_sub, width, rng->engine, idx, pr);
                m = static_cast<int>(idx.size());
            } else {
                m = w;
                idx.assign(hb.begin() + (size_t)i * w, hb.begin() + (size_t)(i + 1) * w);
                pr.resize(w);
                std::memcpy(pr.data(), hb.data() + 2 * cells + (size_t)i * w, sizeof(float) * w);
            }
            const int par = parents_of_rows[i];
            for (int c = 0; c < m; ++c) {
                const int j = idx[c];
                const int32_t full = h->ordered.empty() ? j : h->ordered[j];
                const double lg = std::log(static_cast<double>(pr[c]));
                if (par < 0) {
                    cands.push_back({full, j, -1, 1, c, lg});
                } else {
                    cands.push_back({full, j, par, cands[par].depth + 1, c, cands[par].log_joint + lg});
                }
            }
        }
        return FRS_OK;
    };
    auto by_lj = [&](int a, int b) {
        if (cands[a].log_joint != cands[b].log_joint) return cands[a].log_joint > cands[b].log_joint;
        return a < b;
    };
    btok.assign(1, root_token);
    bpar.assign(1, -1);
    if ((st = run_level(0, 1, std::vector<int>{-1}))) return st;
    for (int c = 0; c < static_cast<int>(cands.size()); ++c) beam.push_back(c);
    for (int level = 1; level < depth && !beam.empty(); ++level) {
        if (static_cast<int>(beam.size()) > width) {  // drafting.cpp:164-176
            std::sort(beam.begin(), beam.end(), by_lj);
            beam.resize(width);
            std::sort(beam.begin(), beam.end());
        }
        const int nb = static_cast<int>(beam.size());
        btok.resize(nb);
        bpar.resize(nb);
        for (int i = 0; i < nb; ++i) {
            btok[i] = cands[beam[i]].token;
            bpar[i] = cands[beam[i]].parent;
        }
        const int first = static_cast<int>(cands.size());
        if ((st = run_level(level, nb, beam))) return st;
        beam.clear();
        for (int c = first; c < static_cast<int>(cands.size()); ++c) beam.push_back(c);
    }
    // select_top_k, prefix_closed = true (drafting.cpp:93-118)
    std::vector<int> order(cands.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), by_lj);
    std::vector<char> sel(cands.size(), 0);
    int cnt = 0;
    for (int c : order) {
        if (sel[c]) continue;
        if (cands[c].parent >= 0 && !sel[cands[c].parent]) continue;
        std::vector<int> group;
        for (size_t s2 = 0; s2 < cands.size(); ++s2)
            if (!sel[s2] && cands[s2].parent == cands[c].parent && cands[s2].sibling_rank <= cands[c].sibling_rank)
                group.push_back(static_cast<int>(s2));
        if (cnt + static_cast<int>(group.size()) > total) continue;
        for (int g : group) sel[g] = 1;
        cnt += static_cast<int>(group.size());
    }
    std::vector<int> remap(cands.size(), -1);
    int out = 0;
    for (size_t i = 0; i < cands.size(); ++i) {
        if (!sel[i]) continue;
        remap[i] = out;
        tokens[out] = cands[i].token;
        parents[out] = cands[i].parent >= 0 ? remap[cands[i].parent] : -1;
        depths[out] = cands[i].depth;
        log_joint[out] = cands[i].log_joint;
        if (node_probs) {  // recorded only for expanded nodes; others stay empty (drafting.h:31-33)
            const bool ex = i < kept.size() && !kept[i].empty();
            has_probs[out] = ex ? 1 : 0;
            if (ex) std::memcpy(node_probs + (size_t)out * h->v_sub, kept[i].data(), sizeof(float) * h->v_sub);
        }
        ++out;
    }
    if (root_probs) std::memcpy(root_probs, root_kept.data(), sizeof(float) * h->v_sub);
    *count = out;
    return FRS_OK;
}

int frs_verify_stochastic(frs_ctx *ctx, const float *h_dev, const void *W, int V, int d, int w_dtype,
                          const int32_t *tokens, const int32_t *parents, int k, const float *q_root, int v_sub,
                          const float *q_nodes, const int32_t *has_q, const int32_t *ordered, float temperature,
                          frs_rng *rng, int32_t *emitted, int *n_emitted, int32_t *path, int *n_path) {
    FRS_REQUIRE(ctx && h_dev && W && rng && q_root && emitted && n_emitted && path && n_path,
                "verify_stochastic: null pointer");
    FRS_REQUIRE(k >= 0 && (k == 0 || (tokens && parents && q_nodes && has_q)), "verify_stochastic: bad tree");
    if (k > 64) return fail(FRS_ECAPACITY, "build_tree_mask: nodes exceed the 64-bit mask");
    for (int i = 0; i < k; ++i)
        if (parents[i] >= i || parents[i] < -1) return fail(FRS_EINVAL, "verify_stochastic: tree is not topological");
    FRS_REQUIRE(std::isfinite(temperature) && temperature > 0.0f, "softmax: temperature must be positive and finite");
    FRS_REQUIRE(V >= 1 && d >= 1 && v_sub >= 1, "verify_stochastic: sizes must be positive");
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    int st;
    if ((st = ctx->logits.ensure((size_t)V * sizeof(float))) ||
        (st = ctx->scratch.ensure((size_t)V * sizeof(float) + 256)))
        return st;
    float *logits = static_cast<float *>(ctx->logits.ptr), *probs = static_cast<float *>(ctx->scratch.ptr);
    uint32_t *fl = reinterpret_cast<uint32_t *>(probs + V);
    std::vector<float> prow(V);
    // The walk visits the root row and then only accepted nodes' rows: each row's exact
    // logits + probabilities are computed when the walk reaches it (one head pass per visited
    // row; typically 1-3 of the 1 + k).
    auto fetch = [&](int r) -> int {  // the exact probabilities of target row r (0 = root)
        int rc;
        if ((rc = launch_exact_logits(ctx, h_dev + (size_t)r * d, 1, d, W, w_dtype, V, logits, s))) return rc;
        if ((rc = launch_softmax_probs(ctx, logits, 1, V, temperature, probs, fl, s))) return rc;
        uint32_t hf = 0;
        FRS_CUDA_TRY(cudaMemcpyAsync(prow.data(), probs, sizeof(float) * V, cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaMemcpyAsync(&hf, fl, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        FRS_CUDA_TRY(cudaStreamSynchronize(s));
        if (hf & FRS_FLAG_NONFINITE) return fail(FRS_EINVAL, "softmax: non-finite logit");  // kernels.cpp:72-74
        return FRS_OK;
    };
    // children_by_node (verification.cpp:31-38)
    std::vector<std::vector<int>> kids(k + 1);
    for (int i = 0; i < k; ++i) kids[parents[i] + 1].push_back(i);
    std::vector<int32_t> full_to_r;
    if (ordered) {
        full_to_r.assign(V, -1);
        for (int j = 0; j < v_sub; ++j)
            if (ordered[j] >= 0 && ordered[j] < V) full_to_r[ordered[j]] = j;
    }
    // Residual (verification.cpp:76-128) in the reference's double arithmetic
    std::vector<double> p;
    double total = 1.0;
    auto init = [&](int r) -> int {
        if ((st = fetch(r))) return st;
        p.assign(prow.begin(), prow.end());
        total = 0.0;
        for (double x : p) total += x;
        return FRS_OK;
    };
    auto subtract = [&](const std::vector<double> &q, double q_total) {
        for (int j = 0; j < static_cast<int>(q.size()); ++j) {
            if (q[j] <= 0.0) continue;
            const int t = ordered ? ordered[j] : j;
            p[t] = std::max(0.0, p[t] - (q[j] / q_total) * total);
        }
        double sum = 0.0;
        for (double x : p) sum += x;
        if (sum <= 0.0) {
            p.assign(p.size(), 1.0);
            sum = static_cast<double>(p.size());
        }
        for (double &x : p) x /= sum;
        total = 1.0;
    };
    auto sample = [&]() -> int32_t {
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        const double u = uni(rng->engine) * total;
        double acc = 0.0;
        int32_t last_positive = 0;
        for (size_t t = 0; t < p.size(); ++t) {
            if (p[t] <= 0.0) continue;
            acc += p[t];
            last_positive = static_cast<int32_t>(t);
            if (u < acc) return last_positive;
        }
        return last_positive;
    };
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    std::vector<int32_t> em, pa;
    if ((st = init(0))) return st;
    int node = -1;
    for (;;) {
        const auto &ch = kids[node + 1];
        int accepted = -1;
        if (!ch.empty()) {
            if (node >= 0 && !has_q[node])
                return fail(FRS_ELOGIC, "verify_stochastic: expanded node is missing its draft distribution");
            const float *qs = node < 0 ? q_root : q_nodes + (size_t)node * v_sub;
            std::vector<double> q(qs, qs + v_sub);
            double q_total = 0.0;
            for (double x : q) q_total += x;
            for (int child : ch) {
                const int32_t t = tokens[child];
                const int j = ordered ? (t >= 0 && t < V ? full_to_r[t] : -1) : t;
                if (j < 0 || j >= v_sub || q[j] <= 0.0 || q_total <= 0.0)
                    return fail(FRS_ELOGIC, "verify_stochastic: drafted token has zero draft probability");
                const double q_t = q[j] / q_total;
                const double ratio = (p[t] / total) / q_t;
                if (uni(rng->engine) < std::min(1.0, ratio)) {
                    accepted = child;
                    break;
                }
                subtract(q, q_total);
                q_total -= q[j];
                q[j] = 0.0;
            }
        }
        if (accepted < 0) {
            em.push_back(sample());  // bonus token
            break;
        }
        pa.push_back(accepted);
        em.push_back(tokens[accepted]);
        node = accepted;
        if ((st = init(1 + accepted))) return st;
    }
    *n_emitted = static_cast<int>(em.size());
    *n_path = static_cast<int>(pa.size());
    std::copy(em.begin(), em.end(), emitted);
    std::copy(pa.begin(), pa.end(), path);
    return FRS_OK;
}

int frs_count_frequencies_device(frs_ctx *ctx, const int32_t *tokens, int64_t count, int vocab_size, uint64_t *counts,
                                 void *stream) {
    FRS_REQUIRE(ctx, "count_frequencies: null context");
    FRS_REQUIRE(vocab_size >= 1, "count_frequencies: vocab_size must be >= 1");
    FRS_REQUIRE(counts && (count == 0 || tokens) && count >= 0, "count_frequencies: null pointer");
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int st = ctx->flags.ensure(256);
    if (st) return st;
    auto *bad = reinterpret_cast<unsigned long long *>(static_cast<uint8_t *>(ctx->flags.ptr) + 64);
    if ((st = frs::count_tokens(ctx, tokens, count, vocab_size, reinterpret_cast<unsigned long long *>(counts), bad, s)))
        return st;
    unsigned long long hb = ~0ull;
    FRS_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
    FRS_CUDA_TRY(cudaStreamSynchronize(s));
    if (hb != ~0ull) {
        int32_t t = 0;
        FRS_CUDA_TRY(cudaMemcpy(&t, tokens + hb, sizeof(t), cudaMemcpyDeviceToHost));
        return fail(FRS_EINVAL, "count_frequencies: token id " + std::to_string(t) + " out of range at offset " +
                                    std::to_string(hb));
    }
    return FRS_OK;
}

namespace {
bool read_le(std::ifstream &f, uint64_t &v, int bytes) {
    unsigned char b[8];
    if (!f.read(reinterpret_cast<char *>(b), bytes)) return false;
    v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return true;
}
void write_le(std::ofstream &f, uint64_t v, int bytes) {
    unsigned char b[8];
    for (int i = 0; i < bytes; ++i) b[i] = static_cast<unsigned char>(v >> (8 * i));
    f.write(reinterpret_cast<const char *>(b), bytes);
}
}  // namespace

// vocab.cpp:236-245
int frs_write_token_stream(const char *path, int vocab_size, const int32_t *tokens, int64_t count) {
    FRS_REQUIRE(path && (count == 0 || tokens) && count >= 0, "write_token_stream: bad arguments");
    const std::string p(path);
    std::ofstream f(p, std::ios::binary);
    if (!f) return fail(FRS_EDATA, p + ": cannot open for writing");
    f.write("FRTK", 4);
    write_le(f, 1, 4);
    write_le(f, static_cast<uint32_t>(vocab_size), 4);
    write_le(f, static_cast<uint64_t>(count), 8);
    for (int64_t i = 0; i < count; ++i) write_le(f, static_cast<uint32_t>(tokens[i]), 4);
    if (!f) return fail(FRS_EDATA, p + ": write failed");
    return FRS_OK;
}

// vocab.cpp:247-272
int frs_read_token_stream(const char *path, int32_t *tokens, int64_t capacity, int *vocab_size, int64_t *count) {
    FRS_REQUIRE(path && vocab_size && count, "read_token_stream: null pointer");
    const std::string p(path);
    std::ifstream f(p, std::ios::binary);
    if (!f) return fail(FRS_EDATA, p + ": cannot open");
    char magic[4];
    if (!f.read(magic, 4) || std::memcmp(magic, "FRTK", 4) != 0)
        return fail(FRS_EDATA, p + ": not a token-stream file (bad magic)");
    uint64_t version = 0, vs = 0, n = 0;
    if (!read_le(f, version, 4)) return fail(FRS_EDATA, p + ": truncated header");
    if (version != 1) return fail(FRS_EDATA, p + ": unsupported version " + std::to_string(version));
    if (!read_le(f, vs, 4)) return fail(FRS_EDATA, p + ": truncated header");
    const int v = static_cast<int>(static_cast<uint32_t>(vs));
    if (v < 1) return fail(FRS_EDATA, p + ": bad vocab_size");
    if (!read_le(f, n, 8)) return fail(FRS_EDATA, p + ": truncated header");
    *vocab_size = v;
    *count = static_cast<int64_t>(n);
    if (!tokens) return FRS_OK;  // size query
    if (static_cast<int64_t>(n) > capacity) return fail(FRS_ECAPACITY, "read_token_stream: buffer too small");
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t raw = 0;
        if (!read_le(f, raw, 4)) return fail(FRS_EDATA, p + ": truncated header");
        if (raw >= static_cast<uint64_t>(static_cast<uint32_t>(v)))
            return fail(FRS_EDATA, p + ": token id " + std::to_string(raw) + " out of range at offset " +
                                       std::to_string(i));
        tokens[i] = static_cast<int32_t>(raw);
    }
    return FRS_OK;
}

// vocab.cpp:274-286
int frs_read_token_stream_text(const char *path, int vocab_size, int32_t *tokens, int64_t capacity, int64_t *count) {
    FRS_REQUIRE(path && count, "read_token_stream_text: null pointer");
    const std::string p(path);
    std::ifstream f(p);
    if (!f) return fail(FRS_EDATA, p + ": cannot open");
    long long value = 0;
    int64_t offset = 0;
    while (f >> value) {
        if (value < 0 || value >= vocab_size)
            return fail(FRS_EDATA, p + ": token id " + std::to_string(value) + " out of range at offset " +
                                       std::to_string(offset));
        if (tokens) {
            if (offset >= capacity) return fail(FRS_ECAPACITY, "read_token_stream_text: buffer too small");
            tokens[offset] = static_cast<int32_t>(value);
        }
        ++offset;
    }
    if (!f.eof()) return fail(FRS_EDATA, p + ": unparsable token id at offset " + std::to_string(offset));
    *count = offset;
    return FRS_OK;
}

// vocab.cpp:288-293
int frs_write_ranked_file(const char *path, const int32_t *ids, int64_t n) {
    FRS_REQUIRE(path && (n == 0 || ids) && n >= 0, "write_ranked_file: bad arguments");
    const std::string p(path);
    std::ofstream f(p);
    if (!f) return fail(FRS_EDATA, p + ": cannot open for writing");
    for (int64_t i = 0; i < n; ++i) f << ids[i] << '\n';
    if (!f) return fail(FRS_EDATA, p + ": write failed");
    return FRS_OK;
}

// vocab.cpp:295-306
int frs_read_ranked_file(const char *path, int32_t *ids, int64_t capacity, int64_t *n) {
    FRS_REQUIRE(path && n, "read_ranked_file: null pointer");
    const std::string p(path);
    std::ifstream f(p);
    if (!f) return fail(FRS_EDATA, p + ": cannot open");
    long long value = 0;
    int64_t k = 0;
    while (f >> value) {
        if (value < 0) return fail(FRS_EDATA, p + ": negative token id");
        if (ids) {
            if (k >= capacity) return fail(FRS_ECAPACITY, "read_ranked_file: buffer too small");
            ids[k] = static_cast<int32_t>(value);
        }
        ++k;
    }
    if (!f.eof()) return fail(FRS_EDATA, p + ": unparsable token id at line " + std::to_string(k + 1));
    *n = k;
    return FRS_OK;
}

// build_draft_tree (drafting.cpp:122-245) with the device draft model as the hidden-state
// source: the pending context forward (causal_layout, model.cpp:288-297), then per level the
// beam rows at anchor position + depth seeing the cached prefix, their forwarded ancestors and
// themselves (drafting.cpp:177-196); the cache is truncated back to the prefix afterwards
// (drafting.cpp:225). rng == NULL: greedy; else sampled (EXACT arithmetic).
struct ModelProvider {
    frs_draft_model *dm;
    const int32_t *pending;
    int n_pending;
    int base_len = 0, anchor_pos = 0, d = 0;
    std::vector<int> cand_row, cand_parent;  // by candidate index (-1 unknown)
};

static int model_provider_cb(void *user, int level, int n, const int32_t *tokens, const int32_t *parent_cands,
                             float *hidden_dev, void *stream) {
    auto *mp = static_cast<ModelProvider *>(user);
    frs_draft_model *dm = mp->dm;
    int len0 = 0;
    frs_draft_model_length(dm, &len0);
    if (level == 0) {  // the pending context, causal (the root is its last token)
        const int np = mp->n_pending;
        int start = 0;  // causal_layout (model.cpp:288-297): after the cache's last position
        if (len0 > 0) {
            const int rc = frs_draft_model_position(dm, len0 - 1, &start);
            if (rc) return rc;
            ++start;
        }
        std::vector<int32_t> pos(np);
        const int m = len0 + np, words = (m + 63) / 64;
        std::vector<uint64_t> vis((size_t)np * words, 0);
        for (int i = 0; i < np; ++i) {
            pos[i] = start + i;
            for (int j = 0; j <= len0 + i; ++j) vis[(size_t)i * words + j / 64] |= 1ull << (j & 63);
        }
        float *tmp = nullptr;
        if (cudaMalloc(&tmp, sizeof(float) * (size_t)np * mp->d) != cudaSuccess) return 2;
        int rc = frs_draft_model_forward(dm, mp->pending, pos.data(), np, vis.data(), tmp, stream);
        if (!rc && cudaMemcpyAsync(hidden_dev, tmp + (size_t)(np - 1) * mp->d, sizeof(float) * mp->d,
                                   cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)) != cudaSuccess)
            rc = 2;
        cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
        cudaFree(tmp);
        if (rc) return rc;
        mp->base_len = len0 + np;
        mp->anchor_pos = pos[np - 1];
        return 0;
    }
    if (!tl_beam_cands) return 3;
    const int m = len0 + n, words = (m + 63) / 64;
    std::vector<int32_t> pos(n);
    std::vector<uint64_t> vis((size_t)n * words, 0);
    auto setb = [&](int i, int j) { vis[(size_t)i * words + j / 64] |= 1ull << (j & 63); };
    for (int i = 0; i < n; ++i) {
        const int c = tl_beam_cands[i];
        if (c >= static_cast<int>(mp->cand_row.size())) {
            mp->cand_row.resize(c + 1 + 1024, -1);
            mp->cand_parent.resize(c + 1 + 1024, -1);
        }
        mp->cand_parent[c] = parent_cands[i];
        mp->cand_row[c] = len0 + i;
        pos[i] = mp->anchor_pos + level;  // depth of a level-L beam row is L
        for (int j = 0; j < mp->base_len; ++j) setb(i, j);
        for (int a = parent_cands[i]; a >= 0; a = mp->cand_parent[a]) setb(i, mp->cand_row[a]);
        setb(i, len0 + i);
    }
    const int rc = frs_draft_model_forward(dm, tokens, pos.data(), n, vis.data(), hidden_dev, stream);
    if (rc) return rc;
    return 0;
}

int frs_draft_tree_model(frs_head *h, frs_draft_model *dm, const int32_t *pending, int n_pending, int width,
                         int depth, int total, int mode, frs_rng *rng, int32_t *tokens, int32_t *parents,
                         int32_t *depths, double *log_joint, int *count, float *root_probs, float *node_probs,
                         int32_t *has_probs) {
    FRS_REQUIRE(h && dm && pending, "build_draft_tree: null pointer");
    if (n_pending < 1) return fail(FRS_EINVAL, "build_draft_tree: pending must end with the root token");
    ModelProvider mp{dm, pending, n_pending};
    mp.d = h->d;
    if (!rng && (root_probs || node_probs))
        return fail(FRS_ENOTSUP, "build_draft_tree: keep_probs is provided with an rng (sampled drafting, the "
                                 "distributions verify_stochastic consumes)");
    int st = rng ? frs_draft_tree_sampled(h, pending[n_pending - 1], model_provider_cb, &mp, nullptr, width, depth,
                                          total, rng, tokens, parents, depths, log_joint, count, root_probs,
                                          node_probs, has_probs)
                 : frs_draft_tree(h, pending[n_pending - 1], model_provider_cb, &mp, nullptr, width, depth, total,
                                  mode, tokens, parents, depths, log_joint, count);
    tl_beam_cands = nullptr;
    if (mp.base_len > 0) frs_draft_model_truncate(dm, mp.base_len);  // drafting.cpp:225
    return st;
}

// AcceptanceStats::add / merge / accepted_length_stats (verification.cpp:180-206).
int frs_acceptance_add(frs_acceptance_stats *s, int accepted_length) {
    FRS_REQUIRE(s, "acceptance stats: null pointer");
    if (accepted_length < 0 || accepted_length >= FRS_HIST_MAX)
        return fail(FRS_EINVAL, "acceptance stats: accepted length " + std::to_string(accepted_length) + " out of range");
    s->iterations += 1;
    s->emitted += accepted_length;
    if (s->hist_len <= accepted_length) {  // histogram.resize(accepted_length + 1, 0)
        for (int i = std::max(s->hist_len, 0); i <= accepted_length; ++i) s->histogram[i] = 0;
        s->hist_len = accepted_length + 1;
    }
    s->histogram[accepted_length] += 1;
    s->mean_accepted_length = static_cast<double>(s->emitted) / static_cast<double>(s->iterations);
    return FRS_OK;
}

int frs_acceptance_merge(frs_acceptance_stats *s, const frs_acceptance_stats *o) {
    FRS_REQUIRE(s && o, "acceptance stats: null pointer");
    FRS_REQUIRE(o->hist_len >= 0 && o->hist_len <= FRS_HIST_MAX, "acceptance stats: bad histogram length");
    s->iterations += o->iterations;
    s->emitted += o->emitted;
    if (s->hist_len < o->hist_len) {
        for (int i = std::max(s->hist_len, 0); i < o->hist_len; ++i) s->histogram[i] = 0;
        s->hist_len = o->hist_len;
    }
    for (int i = 0; i < o->hist_len; ++i) s->histogram[i] += o->histogram[i];
    s->mean_accepted_length =
        s->iterations > 0 ? static_cast<double>(s->emitted) / static_cast<double>(s->iterations) : 0.0;
    return FRS_OK;
}

int frs_accepted_length_stats(const int32_t *lengths, int n, frs_acceptance_stats *out) {
    FRS_REQUIRE(out && (lengths || n == 0), "acceptance stats: null pointer");
    if (n <= 0) return fail(FRS_EINVAL, "accepted_length_stats: empty outcome list");
    std::memset(out, 0, sizeof(*out));
    for (int i = 0; i < n; ++i) {
        const int st = frs_acceptance_add(out, lengths[i]);
        if (st) return st;
    }
    return FRS_OK;
}

}  // extern "C"
