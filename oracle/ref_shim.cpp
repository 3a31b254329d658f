// ORACLE / TEST INFRASTRUCTURE ONLY. Never linked into the product library.
//
// extern "C" shim over the *compiled reference* (the frspec sources under
// /root/reference/proj, built from a patched build-dir copy by oracle/Makefile
// into oracle/_ref/). Every entry point forwards to the reference's own public
// API so tests can compare the CUDA path against the real reference behaviour:
//
//   ref_dot_f32 / ref_matmul   -> frspec::dot_f32 / matmul      kernels.cpp:13-60
//   ref_softmax                -> frspec::softmax               kernels.cpp:62-91
//   ref_topk / ref_argmax      -> frspec::topk / argmax         kernels.cpp:93-122
//   ref_count_frequencies      -> frspec::count_frequencies     vocab.cpp:23-38
//   ref_build_subset           -> frspec::build_subset          vocab.cpp:70-102
//   ref_subset_from_ranking    -> frspec::subset_from_ranking   vocab.cpp:104-138
//   ref_restrict_lm_head       -> frspec::restrict_lm_head      vocab.cpp:152-168
//   ref_zipf_tokens            -> frspec::zipf_tokens           vocab.cpp:180-196
//   ref_build_tree_mask        -> frspec::build_tree_mask       verification.cpp:13-27
//   ref_verify_greedy          -> frspec::verify_greedy         verification.cpp:42-71
//   ref_model_draft_tree       -> frspec::build_draft_tree      drafting.cpp:122-245
//   ref_model_draft_capture    -> restated drafting loop calling frspec::forward_raw
//                                 (model.cpp:208-284) to export per-level hidden states
//
// Errors: every function returns 0 on success, 1 for std::invalid_argument,
// 2 CapacityError, 3 DataError, 4 logic/domain error, 5 anything else; the message
// is available from ref_last_error().
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "frspec/drafting.h"
#include "frspec/errors.h"
#include "frspec/kernels.h"
#include "frspec/matrix.h"
#include "frspec/model.h"
#include "frspec/verification.h"
#include "frspec/vocab.h"

using namespace frspec;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F && f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument & e) {
        g_err = e.what();
        return 1;
    } catch (const CapacityError & e) {
        g_err = e.what();
        return 2;
    } catch (const DataError & e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error & e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception & e) {
        g_err = e.what();
        return 5;
    }
}

Matrix to_matrix(const float * p, int rows, int cols) {
    Matrix m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(float) * static_cast<size_t>(rows) * cols);
    return m;
}

DraftTree tree_from(const int32_t * tokens, const int32_t * parents, const int32_t * depths, int k) {
    DraftTree t;
    for (int i = 0; i < k; ++i) t.nodes.push_back({tokens[i], parents[i], depths ? depths[i] : 0, 0.0});
    return t;
}

void export_tree(const DraftTree & t, int32_t * tokens, int32_t * parents, int32_t * depths,
                 double * log_joint, int * count) {
    *count = static_cast<int>(t.nodes.size());
    for (size_t i = 0; i < t.nodes.size(); ++i) {
        tokens[i] = t.nodes[i].token_id;
        parents[i] = t.nodes[i].parent;
        depths[i] = t.nodes[i].depth;
        log_joint[i] = t.nodes[i].log_joint;
    }
}

struct ModelBundle {
    TargetModel target;
    DraftModel draft;
    std::shared_ptr<const RankedSubset> subset;
    RestrictedHead head;
};

ModelBundle make_bundle(int V, int d, int layers, int heads, int max_seq, uint64_t seed,
                        const int32_t * ordered, int v_sub) {
    ModelConfig cfg;
    cfg.vocab_size = V;
    cfg.hidden_dim = d;
    cfg.num_layers = layers;
    cfg.num_heads = heads;
    cfg.max_seq_len = max_seq;
    cfg.seed = seed;
    ModelBundle b;
    b.target = build_target(cfg);
    b.draft = build_draft(b.target, DraftMode::truncated, 0.0f, 0);
    if (ordered != nullptr) {
        std::vector<Token> ids(ordered, ordered + v_sub);
        b.subset = std::make_shared<const RankedSubset>(subset_from_ranking(ids, v_sub, V, {}));
        b.head = restrict_lm_head(b.target.shared->lm_head, b.subset);
    }
    return b;
}
}  // namespace

extern "C" {

const char * ref_last_error(void) { return g_err.c_str(); }

float ref_dot_f32(const float * a, const float * b, int n) { return dot_f32(a, b, n); }

int ref_matmul(const float * a, int m, int k, const float * bt, int n, float * out) {
    return guarded([&] {
        Matrix r = matmul(to_matrix(a, m, k), to_matrix(bt, n, k));
        std::memcpy(out, r.data.data(), sizeof(float) * static_cast<size_t>(m) * n);
    });
}

int ref_softmax(const float * logits, int n, float temperature, float * probs) {
    return guarded([&] {
        ProbVector p = softmax(std::span<const float>(logits, n), temperature);
        std::memcpy(probs, p.probs.data(), sizeof(float) * n);
    });
}

int ref_topk(const float * values, int n, int k, int32_t * idx, float * val) {
    return guarded([&] {
        auto r = topk(std::span<const float>(values, n), k);
        for (int i = 0; i < k; ++i) {
            idx[i] = r[i].first;
            val[i] = r[i].second;
        }
    });
}

int ref_argmax(const float * values, int n, int32_t * out) {
    return guarded([&] { *out = argmax(std::span<const float>(values, n)); });
}

int ref_count_frequencies(const int32_t * stream, int64_t count, int vocab_size, uint64_t * counts,
                          uint64_t * total) {
    return guarded([&] {
        FrequencyTable t = count_frequencies(std::span<const Token>(stream, count), vocab_size);
        std::memcpy(counts, t.counts.data(), sizeof(uint64_t) * vocab_size);
        *total = t.total;
    });
}

int ref_build_subset(const uint64_t * counts, int vocab_size, uint64_t total, int size,
                     const int32_t * forced, int n_forced, int32_t * ordered_out) {
    return guarded([&] {
        FrequencyTable t;
        t.vocab_size = vocab_size;
        t.counts.assign(counts, counts + vocab_size);
        t.total = total;
        RankedSubset s = build_subset(t, size, std::span<const Token>(forced, n_forced));
        std::memcpy(ordered_out, s.ordered_ids.data(), sizeof(int32_t) * s.size());
    });
}

int ref_subset_from_ranking(const int32_t * ranked, int n_ranked, int size, int vocab_size,
                            const int32_t * forced, int n_forced, int32_t * ordered_out) {
    return guarded([&] {
        RankedSubset s = subset_from_ranking(std::span<const Token>(ranked, n_ranked), size, vocab_size,
                                             std::span<const Token>(forced, n_forced));
        std::memcpy(ordered_out, s.ordered_ids.data(), sizeof(int32_t) * s.size());
    });
}

int ref_restrict_lm_head(const float * W, int V, int d, const int32_t * ordered, int v_sub,
                         float * out) {
    return guarded([&] {
        std::vector<Token> ids(ordered, ordered + v_sub);
        auto subset = std::make_shared<const RankedSubset>(subset_from_ranking(ids, v_sub, V, {}));
        RestrictedHead h = restrict_lm_head(to_matrix(W, V, d), subset);
        std::memcpy(out, h.matrix.data.data(), sizeof(float) * static_cast<size_t>(v_sub) * d);
    });
}

int ref_zipf_tokens(int vocab_size, double exponent, int64_t count, uint64_t seed, int32_t * out) {
    return guarded([&] {
        TokenSequence t = zipf_tokens(vocab_size, exponent, static_cast<size_t>(count), seed);
        std::memcpy(out, t.data(), sizeof(int32_t) * t.size());
    });
}

// Seeded Gaussian fill with the reference's generator semantics (model.cpp:24-27):
// std::mt19937_64(seed) + std::normal_distribution<float>(0, std_dev), compiled with
// -ffp-contract=off so the stream is flag-independent.
void ref_fill_gaussian(float * out, int64_t count, uint64_t seed, float std_dev) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> dist(0.0f, std_dev);
    for (int64_t i = 0; i < count; ++i) out[i] = dist(rng);
}

int ref_build_tree_mask(const int32_t * parents, int k, uint64_t * words) {
    return guarded([&] {
        std::vector<int32_t> tok(k, 0);
        TreeMask m = build_tree_mask(tree_from(tok.data(), parents, nullptr, k));
        std::memcpy(words, m.words.data(), sizeof(uint64_t) * k);
    });
}

int ref_verify_greedy(const float * root_logits, int V, const float * node_logits, int k,
                      const int32_t * tokens, const int32_t * parents, int32_t * emitted,
                      int * n_emitted, int32_t * path, int * n_path) {
    return guarded([&] {
        DraftTree t = tree_from(tokens, parents, nullptr, k);
        VerifyOutcome o = verify_greedy(std::span<const float>(root_logits, V), to_matrix(node_logits, k, V), t);
        *n_emitted = static_cast<int>(o.emitted.size());
        *n_path = static_cast<int>(o.accepted_path.size());
        std::copy(o.emitted.begin(), o.emitted.end(), emitted);
        std::copy(o.accepted_path.begin(), o.accepted_path.end(), path);
    });
}

// verify_stochastic (verification.cpp:76-178) of the compiled reference. q_root [v_sub] and
// q_nodes [k][v_sub] are the draft distributions (node rows with has_q[i] == 0 are empty, as
// for unexpanded nodes); ordered (v_sub ids) is the drafting subset (NULL: full vocabulary).
int ref_verify_stochastic(const float * root_logits, int V, const float * node_logits, int k,
                          const int32_t * tokens, const int32_t * parents, const float * q_root, int v_sub,
                          const float * q_nodes, const int32_t * has_q, const int32_t * ordered,
                          float temperature, uint64_t rng_seed, int32_t * emitted, int * n_emitted,
                          int32_t * path, int * n_path) {
    return guarded([&] {
        DraftResult dr;
        dr.tree = tree_from(tokens, parents, nullptr, k);
        dr.root_probs.assign(q_root, q_root + v_sub);
        dr.node_probs.resize(k);
        for (int i = 0; i < k; ++i)
            if (has_q[i]) dr.node_probs[i].assign(q_nodes + static_cast<size_t>(i) * v_sub,
                                                  q_nodes + static_cast<size_t>(i + 1) * v_sub);
        std::shared_ptr<const RankedSubset> sub;
        if (ordered) {
            std::vector<Token> ids(ordered, ordered + v_sub);
            sub = std::make_shared<const RankedSubset>(subset_from_ranking(ids, v_sub, V, {}));
        }
        std::mt19937_64 rng(rng_seed);
        VerifyOutcome o = verify_stochastic(std::span<const float>(root_logits, V), to_matrix(node_logits, k, V), dr,
                                            sub.get(), temperature, rng);
        *n_emitted = static_cast<int>(o.emitted.size());
        *n_path = static_cast<int>(o.accepted_path.size());
        std::copy(o.emitted.begin(), o.emitted.end(), emitted);
        std::copy(o.accepted_path.begin(), o.accepted_path.end(), path);
    });
}

// A reference draft model (build_draft truncated, 1 layer) with its KV cache, for parity of
// the device draft forward: weights export + forward_raw calls on the persistent cache.
struct RefDraftSession {
    ModelBundle b;
    KVCache cache;
};
void * ref_draft_session_new(int V, int d, int heads, int max_seq, uint64_t seed) {
    try {
        ModelBundle b = make_bundle(V, d, 1, heads, max_seq, seed, nullptr, 0);
        KVCache c = make_cache(b.draft);
        return new RefDraftSession{std::move(b), std::move(c)};
    } catch (...) {
        return nullptr;
    }
}
void ref_draft_session_free(void * s) { delete static_cast<RefDraftSession *>(s); }
// embedding [V x d], wq wk wv wo [d x d], w_up [4d x d], w_down [d x 4d] (norm gains are 1)
int ref_draft_session_weights(void * sp, float * emb, float * wq, float * wk, float * wv, float * wo, float * w_up,
                              float * w_down) {
    return guarded([&] {
        auto * s = static_cast<RefDraftSession *>(sp);
        const LayerWeights & L = s->b.draft.layer;
        auto cp = [](const Matrix & m, float * out) { std::memcpy(out, m.data.data(), sizeof(float) * m.data.size()); };
        cp(s->b.draft.shared->embedding, emb);
        cp(L.wq, wq);
        cp(L.wk, wk);
        cp(L.wv, wv);
        cp(L.wo, wo);
        cp(L.w_up, w_up);
        cp(L.w_down, w_down);
    });
}
// forward_raw on the session cache: visible_allow [n x (len + n)] 0/1; hidden_out [n x d]
int ref_draft_session_forward(void * sp, const int32_t * tokens, const int32_t * positions, int n,
                              const uint8_t * allow, float * hidden_out) {
    return guarded([&] {
        auto * s = static_cast<RefDraftSession *>(sp);
        const int m = s->cache.len + n;
        BitMask vis(n, m);
        for (int r = 0; r < n; ++r)
            for (int j = 0; j < m; ++j)
                if (allow[static_cast<size_t>(r) * m + j]) vis.set(r, j);
        std::vector<int> pos(positions, positions + n);
        ForwardResult f = forward_raw(*s->b.draft.shared, {&s->b.draft.layer, 1}, std::span<const Token>(tokens, n), pos,
                                      vis, s->cache, s->b.draft.shared->lm_head);
        std::memcpy(hidden_out, f.hidden.row(0), sizeof(float) * static_cast<size_t>(n) * f.hidden.cols);
    });
}

int ref_draft_session_len(void * sp) { return static_cast<RefDraftSession *>(sp)->cache.len; }
int ref_draft_session_position(void * sp, int row) { return static_cast<RefDraftSession *>(sp)->cache.positions[row]; }
// KVCache::compact (model.cpp:165-196) on the session cache.
int ref_draft_session_compact(void * sp, int keep_from, const int32_t * offs, int n) {
    return guarded([&] {
        auto * s = static_cast<RefDraftSession *>(sp);
        std::vector<int> o(offs, offs + n);
        s->cache.compact(keep_from, o);
    });
}
// build_draft_tree (greedy, restricted head over `ordered` when non-null) on the session's
// persistent cache: a second call drafts after the first call's context, as a decode loop does.
int ref_draft_session_draft_tree(void * sp, const int32_t * ordered, int v_sub, const int32_t * pending, int n_pending,
                                 int width, int depth, int total, int32_t * tokens, int32_t * parents,
                                 int32_t * depths, double * log_joint, int * count) {
    return guarded([&] {
        auto * s = static_cast<RefDraftSession *>(sp);
        const int V = s->b.draft.shared->lm_head.rows;
        std::shared_ptr<const RankedSubset> sub;
        RestrictedHead head;
        if (ordered != nullptr) {
            std::vector<Token> ids(ordered, ordered + v_sub);
            sub = std::make_shared<const RankedSubset>(subset_from_ranking(ids, v_sub, V, {}));
            head = restrict_lm_head(s->b.draft.shared->lm_head, sub);
        }
        DraftParams p{width, depth, total};
        DraftResult r = build_draft_tree(s->b.draft, s->cache, std::span<const Token>(pending, n_pending), p,
                                         ordered ? &head : nullptr, nullptr, false);
        export_tree(r.tree, tokens, parents, depths, log_joint, count);
    });
}

// accepted_length_stats over outcomes with the given accepted lengths (|emitted| = len), then
// (when nb >= 0) .merge() of the stats of a second list (nb == 0: a default AcceptanceStats).
int ref_acceptance_stats(const int32_t * la, int na, const int32_t * lb, int nb, int64_t * iterations,
                         int64_t * emitted, double * mean, int64_t * hist, int hist_cap, int * hist_len) {
    return guarded([&] {
        auto outcomes = [](const int32_t * l, int n) {
            std::vector<VerifyOutcome> v(n);
            for (int i = 0; i < n; ++i) v[i].emitted.assign(l[i], 0);
            return v;
        };
        auto va = outcomes(la, na);
        AcceptanceStats s = accepted_length_stats(va);
        if (nb > 0) {
            auto vb = outcomes(lb, nb);
            s.merge(accepted_length_stats(vb));
        } else if (nb == 0) {
            s.merge(AcceptanceStats{});
        }
        *iterations = s.iterations;
        *emitted = s.emitted;
        *mean = s.mean_accepted_length;
        *hist_len = static_cast<int>(s.histogram.size());
        for (int i = 0; i < *hist_len && i < hist_cap; ++i) hist[i] = s.histogram[i];
    });
}

// masked_attention (kernels.cpp:124-171) with a dense 0/1 mask [n x m].
int ref_masked_attention(const float * q, const float * k, const float * v, const uint8_t * allow, int n, int m,
                         int dh, int dv, float * out) {
    return guarded([&] {
        BitMask bm(n, m);
        for (int r = 0; r < n; ++r)
            for (int j = 0; j < m; ++j)
                if (allow[static_cast<size_t>(r) * m + j]) bm.set(r, j);
        Matrix o = masked_attention(to_matrix(q, n, dh), to_matrix(k, m, dh), to_matrix(v, m, dv), bm);
        std::memcpy(out, o.row(0), sizeof(float) * static_cast<size_t>(n) * dv);
    });
}

// Token-stream / ranked files through the reference (vocab.cpp:198-308), for cross-checks.
int ref_write_token_stream(const char * path, int vocab, const int32_t * tokens, int64_t n) {
    return guarded([&] { write_token_stream(path, vocab, std::span<const Token>(tokens, n)); });
}
int ref_read_token_stream(const char * path, int32_t * out, int64_t cap, int * vocab, int64_t * n) {
    return guarded([&] {
        TokenStreamData d = read_token_stream(path);
        *vocab = d.vocab_size;
        *n = static_cast<int64_t>(d.tokens.size());
        if (out) std::copy(d.tokens.begin(), d.tokens.begin() + std::min<int64_t>(cap, *n), out);
    });
}
int ref_read_token_stream_text(const char * path, int vocab, int32_t * out, int64_t cap, int64_t * n) {
    return guarded([&] {
        TokenStreamData d = read_token_stream_text(path, vocab);
        *n = static_cast<int64_t>(d.tokens.size());
        if (out) std::copy(d.tokens.begin(), d.tokens.begin() + std::min<int64_t>(cap, *n), out);
    });
}
int ref_write_ranked_file(const char * path, const int32_t * ids, int64_t n) {
    return guarded([&] { write_ranked_file(path, std::span<const Token>(ids, n)); });
}
int ref_read_ranked_file(const char * path, int32_t * out, int64_t cap, int64_t * n) {
    return guarded([&] {
        std::vector<Token> ids = read_ranked_file(path);
        *n = static_cast<int64_t>(ids.size());
        if (out) std::copy(ids.begin(), ids.begin() + std::min<int64_t>(cap, *n), out);
    });
}

// A persistent reference Matrix for timing the reference's own draft level without per-call
// copies of the head (the CPU baseline in bench.py).
void * ref_head_new(const float * W, int rows, int d) { return new Matrix(to_matrix(W, rows, d)); }
void ref_head_free(void * head) { delete static_cast<Matrix *>(head); }

// One draft level exactly as the reference runs it: LM-head matmul (model.cpp:278), then per
// row softmax (drafting.cpp:204) and pick_children -> topk(min(width, V_sub)) (drafting.cpp:37-43).
int ref_draft_level(const void * head, const float * h, int n, int d, int k, int32_t * ridx, float * prob) {
    return guarded([&] {
        const Matrix & W = *static_cast<const Matrix *>(head);
        Matrix logits = matmul(to_matrix(h, n, d), W);
        const int w = std::min(k, W.rows);
        for (int i = 0; i < n; ++i) {
            ProbVector p = softmax(logits.row_span(i), 1.0f);
            auto r = topk(p.probs, w);
            for (int c = 0; c < w; ++c) {
                ridx[(size_t)i * k + c] = r[c].first;
                prob[(size_t)i * k + c] = r[c].second;
            }
        }
    });
}

// Verify head as the reference runs it: matmul over the full head, argmax per row.
int ref_verify_argmax(const void * head, const float * h, int m, int d, int32_t * ids) {
    return guarded([&] {
        Matrix logits = matmul(to_matrix(h, m, d), *static_cast<const Matrix *>(head));
        for (int i = 0; i < m; ++i) ids[i] = argmax(logits.row_span(i));
    });
}

// Exports the seeded toy model's LM head [V x d] (model.cpp:93-128).
int ref_model_lm_head(int V, int d, int layers, int heads, uint64_t seed, float * out) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, layers, heads, 8, seed, nullptr, 0);
        std::memcpy(out, b.target.shared->lm_head.data.data(), sizeof(float) * static_cast<size_t>(V) * d);
    });
}

// Runs the reference's build_draft_tree (greedy, restricted head when ordered != null) on
// an empty cache with `pending` as the forwarded context.
int ref_model_draft_tree(int V, int d, int layers, int heads, int max_seq, uint64_t seed,
                         const int32_t * ordered, int v_sub, const int32_t * pending, int n_pending,
                         int width, int depth, int total, int32_t * tokens, int32_t * parents,
                         int32_t * depths, double * log_joint, int * count) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, layers, heads, max_seq, seed, ordered, v_sub);
        KVCache cache = make_cache(b.draft);
        DraftParams p{width, depth, total};
        DraftResult r = build_draft_tree(b.draft, cache, std::span<const Token>(pending, n_pending), p,
                                         ordered ? &b.head : nullptr, nullptr, false);
        export_tree(r.tree, tokens, parents, depths, log_joint, count);
    });
}

// Same drafting run, restated around the reference's public forward_raw so that the
// hidden state of every forwarded draft row can be exported (drafting.cpp:133-221 order).
// hidden_out: [1 + (depth-1)*width] x d rows: row 0 is the root row (last pending row);
// then, level by level, the forwarded beam rows in beam order. beam_tokens/beam_parents
// record, per forwarded row, its token and parent candidate index (-1 for the root row).
// n_rows receives the number of hidden rows written.
int ref_model_draft_capture(int V, int d, int layers, int heads, int max_seq, uint64_t seed,
                            const int32_t * ordered, int v_sub, const int32_t * pending,
                            int n_pending, int width, int depth, int total, float * hidden_out,
                            int32_t * row_token, int32_t * row_level, int * n_rows,
                            int32_t * tokens, int32_t * parents, int32_t * depths,
                            double * log_joint, int * count) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, layers, heads, max_seq, seed, ordered, v_sub);
        KVCache cache = make_cache(b.draft);
        DraftParams params{width, depth, total};
        validate_params(params);
        const RankedSubset * subset = ordered ? b.subset.get() : nullptr;
        const Matrix & head = ordered ? b.head.matrix : b.draft.shared->lm_head;
        struct Cand {
            Token token;
            int parent, depth;
            double log_joint;
            int cache_row;
        };
        int rows = 0;
        auto emit_row = [&](const Matrix & hid, int r, Token tok, int level) {
            std::memcpy(hidden_out + static_cast<size_t>(rows) * d, hid.row(r), sizeof(float) * d);
            row_token[rows] = tok;
            row_level[rows] = level;
            ++rows;
        };
        ForwardResult fwd = draft_forward(b.draft, std::span<const Token>(pending, n_pending), cache,
                                          ordered ? &b.head : nullptr);
        emit_row(fwd.hidden, fwd.hidden.rows - 1, pending[n_pending - 1], 0);
        const int base_len = cache.len;
        const int anchor_pos = cache.positions[base_len - 1];
        std::vector<Cand> cands;
        std::vector<int> beam;
        {
            ProbVector pr = softmax(fwd.logits.row_span(fwd.logits.rows - 1), 1.0f);
            auto kids = topk(pr.probs, std::min(width, static_cast<int>(pr.probs.size())));
            for (auto [idx, prob] : kids) {
                beam.push_back(static_cast<int>(cands.size()));
                cands.push_back({subset ? subset->full_id(idx) : idx, -1, 1, std::log((double)prob), -1});
            }
        }
        for (int level = 1; level < depth && !beam.empty(); ++level) {
            if (static_cast<int>(beam.size()) > width) {
                std::sort(beam.begin(), beam.end(), [&](int a, int c) {
                    if (cands[a].log_joint != cands[c].log_joint) return cands[a].log_joint > cands[c].log_joint;
                    return a < c;
                });
                beam.resize(width);
                std::sort(beam.begin(), beam.end());
            }
            const int batch = static_cast<int>(beam.size());
            TokenSequence bt;
            std::vector<int> bp;
            BitMask visible(batch, cache.len + batch);
            for (int i = 0; i < batch; ++i) {
                Cand & c = cands[beam[i]];
                c.cache_row = cache.len + i;
                bt.push_back(c.token);
                bp.push_back(anchor_pos + c.depth);
                visible.set_range(i, 0, base_len);
                for (int a = c.parent; a >= 0; a = cands[a].parent) visible.set(i, cands[a].cache_row);
                visible.set(i, c.cache_row);
            }
            fwd = forward_raw(*b.draft.shared, {&b.draft.layer, 1}, bt, bp, visible, cache, head);
            std::vector<int> next;
            for (int i = 0; i < batch; ++i) {
                emit_row(fwd.hidden, i, bt[i], level);
                const int pidx = beam[i];
                const int pdepth = cands[pidx].depth;
                const double plj = cands[pidx].log_joint;
                ProbVector pr = softmax(fwd.logits.row_span(i), 1.0f);
                auto kids = topk(pr.probs, std::min(width, static_cast<int>(pr.probs.size())));
                for (auto [idx, prob] : kids) {
                    next.push_back(static_cast<int>(cands.size()));
                    cands.push_back({subset ? subset->full_id(idx) : idx, pidx, pdepth + 1,
                                     plj + std::log((double)prob), -1});
                }
            }
            beam = std::move(next);
        }
        *n_rows = rows;
        // select_top_k, greedy (drafting.cpp:79-118 with prefix_closed=false)
        std::vector<int> order(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) order[i] = static_cast<int>(i);
        std::sort(order.begin(), order.end(), [&](int a, int c) {
            if (cands[a].log_joint != cands[c].log_joint) return cands[a].log_joint > cands[c].log_joint;
            return a < c;
        });
        std::vector<char> sel(cands.size(), 0);
        int cnt = 0;
        for (int c : order) {
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
    });
}

// Sampled drafting (drafting.cpp:44-74 with an rng): the reference's own build_draft_tree
// with std::mt19937_64(rng_seed).
int ref_model_draft_tree_rng(int V, int d, int layers, int heads, int max_seq, uint64_t seed,
                             const int32_t * ordered, int v_sub, const int32_t * pending, int n_pending,
                             int width, int depth, int total, uint64_t rng_seed, int32_t * tokens,
                             int32_t * parents, int32_t * depths, double * log_joint, int * count) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, layers, heads, max_seq, seed, ordered, v_sub);
        KVCache cache = make_cache(b.draft);
        DraftParams p{width, depth, total};
        std::mt19937_64 rng(rng_seed);
        DraftResult r = build_draft_tree(b.draft, cache, std::span<const Token>(pending, n_pending), p,
                                         ordered ? &b.head : nullptr, &rng, false);
        export_tree(r.tree, tokens, parents, depths, log_joint, count);
    });
}

// Sampled drafting with keep_probs, then stochastic verification with the SAME engine (the
// decode loop's order): build_draft_tree(rng, keep_probs = true) on a fresh cache, target logits
// = matmul(h_t[0 .. K], W_t) (h_t: caller rows, root first), verify_stochastic(root, nodes, the
// DraftResult, subset, temperature, rng). Exports the tree, its distributions and the outcome.
int ref_draft_verify_rng(int V, int d, int heads, int max_seq, uint64_t seed, const int32_t * ordered, int v_sub,
                         const int32_t * pending, int n_pending, int width, int depth, int total, uint64_t rng_seed,
                         const float * h_t, const float * W_t, float temperature, int32_t * tokens,
                         int32_t * parents, int32_t * depths, double * log_joint, int * count, float * root_probs,
                         float * node_probs, int32_t * has_probs, int32_t * emitted, int * n_emitted, int32_t * path,
                         int * n_path) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, 1, heads, max_seq, seed, ordered, v_sub);
        KVCache cache = make_cache(b.draft);
        DraftParams p{width, depth, total};
        std::mt19937_64 rng(rng_seed);
        DraftResult r = build_draft_tree(b.draft, cache, std::span<const Token>(pending, n_pending), p,
                                         ordered ? &b.head : nullptr, &rng, true);
        export_tree(r.tree, tokens, parents, depths, log_joint, count);
        const int K = *count;
        const int hv = ordered ? v_sub : V;
        std::copy(r.root_probs.begin(), r.root_probs.end(), root_probs);
        for (int i = 0; i < K; ++i) {
            has_probs[i] = r.node_probs[i].empty() ? 0 : 1;
            if (has_probs[i]) std::copy(r.node_probs[i].begin(), r.node_probs[i].end(), node_probs + (size_t)i * hv);
        }
        Matrix logits = matmul(to_matrix(h_t, 1 + K, d), to_matrix(W_t, V, d));
        Matrix node_logits(K, V);
        if (K > 0) std::memcpy(node_logits.row(0), logits.row(1), sizeof(float) * (size_t)K * V);
        VerifyOutcome o = verify_stochastic(logits.row_span(0), node_logits, r, ordered ? b.subset.get() : nullptr,
                                            temperature, rng);
        *n_emitted = static_cast<int>(o.emitted.size());
        *n_path = static_cast<int>(o.accepted_path.size());
        std::copy(o.emitted.begin(), o.emitted.end(), emitted);
        std::copy(o.accepted_path.begin(), o.accepted_path.end(), path);
    });
}

// Restatement of pick_children's sampled branch (drafting.cpp:44-74; the original sits in an
// anonymous namespace), pinned by the sampled capture test against build_draft_tree above.
static std::vector<std::pair<int, float>> pick_sampled(const std::vector<float> & probs, int width,
                                                       std::mt19937_64 & rng) {
    const int n = static_cast<int>(probs.size());
    const int w = std::min(width, n);
    std::vector<std::pair<int, float>> out;
    std::vector<double> work(probs.begin(), probs.end());
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
        out.emplace_back(picked, probs[picked]);
        work[picked] = 0.0;
    }
    return out;
}

// pick_sampled over given probabilities (unit tests of the device sampler): picks[w], probs[w]
// in draw order; *count = draws made. Consumes draws from a fresh mt19937_64(rng_seed) after
// skipping `skip` uniforms.
int ref_pick_sampled(const float * probs, int n, int width, uint64_t rng_seed, int64_t skip, int32_t * picks,
                     float * out_probs, int * count) {
    return guarded([&] {
        std::mt19937_64 rng(rng_seed);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        for (int64_t i = 0; i < skip; ++i) (void)uni(rng);
        auto kids = pick_sampled(std::vector<float>(probs, probs + n), width, rng);
        for (size_t i = 0; i < kids.size(); ++i) {
            picks[i] = kids[i].first;
            out_probs[i] = kids[i].second;
        }
        *count = static_cast<int>(kids.size());
    });
}

// std::uniform_real_distribution<double>(0, 1) draws of std::mt19937_64(seed) (tests).
int ref_uniforms(uint64_t seed, int64_t skip, int count, double * out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        for (int64_t i = 0; i < skip; ++i) (void)uni(rng);
        for (int i = 0; i < count; ++i) out[i] = uni(rng);
    });
}

// Sampled-mode capture: the drafting loop of ref_model_draft_capture with pick_sampled and the
// prefix-closed select_top_k (drafting.cpp:93-118, prefix_closed = true).
int ref_model_draft_capture_rng(int V, int d, int layers, int heads, int max_seq, uint64_t seed,
                                const int32_t * ordered, int v_sub, const int32_t * pending, int n_pending,
                                int width, int depth, int total, uint64_t rng_seed, float * hidden_out,
                                int32_t * row_token, int32_t * row_level, int * n_rows, int32_t * tokens,
                                int32_t * parents, int32_t * depths, double * log_joint, int * count) {
    return guarded([&] {
        ModelBundle b = make_bundle(V, d, layers, heads, max_seq, seed, ordered, v_sub);
        KVCache cache = make_cache(b.draft);
        DraftParams params{width, depth, total};
        validate_params(params);
        std::mt19937_64 rng(rng_seed);
        const RankedSubset * subset = ordered ? b.subset.get() : nullptr;
        const Matrix & head = ordered ? b.head.matrix : b.draft.shared->lm_head;
        struct Cand {
            Token token;
            int parent, depth, sibling_rank;
            double log_joint;
            int cache_row;
        };
        int rows = 0;
        auto emit_row = [&](const Matrix & hid, int r, Token tok, int level) {
            std::memcpy(hidden_out + static_cast<size_t>(rows) * d, hid.row(r), sizeof(float) * d);
            row_token[rows] = tok;
            row_level[rows] = level;
            ++rows;
        };
        ForwardResult fwd = draft_forward(b.draft, std::span<const Token>(pending, n_pending), cache,
                                          ordered ? &b.head : nullptr);
        emit_row(fwd.hidden, fwd.hidden.rows - 1, pending[n_pending - 1], 0);
        const int base_len = cache.len;
        const int anchor_pos = cache.positions[base_len - 1];
        std::vector<Cand> cands;
        std::vector<int> beam;
        {
            ProbVector pr = softmax(fwd.logits.row_span(fwd.logits.rows - 1), 1.0f);
            int rank = 0;
            for (auto [idx, prob] : pick_sampled(pr.probs, width, rng)) {
                beam.push_back(static_cast<int>(cands.size()));
                cands.push_back({subset ? subset->full_id(idx) : idx, -1, 1, rank++, std::log((double)prob), -1});
            }
        }
        for (int level = 1; level < depth && !beam.empty(); ++level) {
            if (static_cast<int>(beam.size()) > width) {
                std::sort(beam.begin(), beam.end(), [&](int a, int c) {
                    if (cands[a].log_joint != cands[c].log_joint) return cands[a].log_joint > cands[c].log_joint;
                    return a < c;
                });
                beam.resize(width);
                std::sort(beam.begin(), beam.end());
            }
            const int batch = static_cast<int>(beam.size());
            TokenSequence bt;
            std::vector<int> bp;
            BitMask visible(batch, cache.len + batch);
            for (int i = 0; i < batch; ++i) {
                Cand & c = cands[beam[i]];
                c.cache_row = cache.len + i;
                bt.push_back(c.token);
                bp.push_back(anchor_pos + c.depth);
                visible.set_range(i, 0, base_len);
                for (int a = c.parent; a >= 0; a = cands[a].parent) visible.set(i, cands[a].cache_row);
                visible.set(i, c.cache_row);
            }
            fwd = forward_raw(*b.draft.shared, {&b.draft.layer, 1}, bt, bp, visible, cache, head);
            std::vector<int> next;
            for (int i = 0; i < batch; ++i) {
                emit_row(fwd.hidden, i, bt[i], level);
                const int pidx = beam[i];
                const int pdepth = cands[pidx].depth;
                const double plj = cands[pidx].log_joint;
                ProbVector pr = softmax(fwd.logits.row_span(i), 1.0f);
                int rank = 0;
                for (auto [idx, prob] : pick_sampled(pr.probs, width, rng)) {
                    next.push_back(static_cast<int>(cands.size()));
                    cands.push_back({subset ? subset->full_id(idx) : idx, pidx, pdepth + 1, rank++,
                                     plj + std::log((double)prob), -1});
                }
            }
            beam = std::move(next);
        }
        *n_rows = rows;
        std::vector<int> order(cands.size());
        for (size_t i = 0; i < cands.size(); ++i) order[i] = static_cast<int>(i);
        std::sort(order.begin(), order.end(), [&](int a, int c) {
            if (cands[a].log_joint != cands[c].log_joint) return cands[a].log_joint > cands[c].log_joint;
            return a < c;
        });
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
            ++out;
        }
        *count = out;
    });
}

}  // extern "C"
