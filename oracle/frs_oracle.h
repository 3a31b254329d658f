/* ORACLE / TEST INFRASTRUCTURE ONLY — "the checker, never the thing measured or shipped".
 *
 * Plain-C restatement of the FR-Spec reference's drafting hot path
 * (/root/reference/proj, C++20). Each function cites the reference lines it restates.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this.
 *
 * Parity pin: validated against the compiled reference (oracle/_ref/libfrspec_ref.so,
 * built from the reference's own sources by oracle/Makefile) and the SPEC worked
 * examples committed under tests/golden/.
 */
#ifndef FRS_ORACLE_H
#define FRS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* kernels.cpp:13-32 — 8 rounded-mul/rounded-add lane chains, fixed tree, scalar tail. */
float frs_o_dot_f32(const float *a, const float *b, int n);
/* kernels.cpp:34-60 — out[i][j] = dot_f32(h_i, W_j). */
void frs_o_logits(const float *h, int n, const float *W, int V, int d, float *out);
/* glibc 2.39 expf (__expf_fma ifunc) restated — SURVEY.md Appendix A. */
float frs_o_expf_glibc(float x);
/* kernels.cpp:62-91. Returns 0, or 1 on rejected input. mx/total are the internals. */
int frs_o_softmax(const float *logits, int n, float temperature, float *probs, float *out_mx,
                  double *out_total);
/* kernels.cpp:93-111 — k largest by (value desc, index asc). */
int frs_o_topk(const float *values, int n, int k, int32_t *idx, float *val);
/* kernels.cpp:113-122 — strict '>' scan, lowest index on ties. */
int frs_o_argmax(const float *values, int n);

/* One draft level for n hidden rows: model.cpp:276-279 (LM head over the slab), then per
 * row softmax(t) (drafting.cpp:140/204), topk(min(k, V_sub)) (drafting.cpp:37-43) and the
 * restricted->full remap (drafting.cpp:151/210, vocab.h:32). Outputs [n x k]. */
int frs_o_draft_level(const float *h, int n, const float *slab, int v_sub, int d,
                      const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx,
                      int32_t *out_full, float *out_prob, float *out_mx, double *out_total,
                      float *out_logits /* nullable [n x v_sub] */);

/* Verify head: argmax of dot_f32 logits over the full vocabulary, m rows
 * (model.cpp:324-338 -> 276-279, kernels.cpp:113-122). */
void frs_o_verify_argmax(const float *h, int m, const float *W, int V, int d, int32_t *out_id,
                         float *out_val);
/* verification.cpp:42-71 given per-row argmax ids (row 0 = root, row 1+i = node i). */
int frs_o_verify_greedy_ids(const int32_t *argmax_ids, const int32_t *tokens,
                            const int32_t *parents, int k, int32_t *emitted, int *n_emitted,
                            int32_t *path, int *n_path);
/* verification.cpp:13-27. Returns 2 (capacity) beyond 64 nodes, 1 if not topological. */
int frs_o_tree_mask(const int32_t *parents, int k, uint64_t *words);

/* vocab.cpp:23-38 */
int frs_o_count_frequencies(const int32_t *stream, int64_t count, int vocab_size, uint64_t *counts);
/* vocab.cpp:70-102 + finalize_subset 42-58 */
int frs_o_build_subset(const uint64_t *counts, int vocab_size, int size, const int32_t *forced,
                       int n_forced, int32_t *ordered_out);
/* vocab.cpp:104-138 */
int frs_o_subset_from_ranking(const int32_t *ranked, int n_ranked, int size, int vocab_size,
                              const int32_t *forced, int n_forced, int32_t *ordered_out);
/* vocab.cpp:152-168 — bitwise row gather. */
int frs_o_restrict(const float *W, int V, int d, const int32_t *ordered, int v_sub, float *out);

/* Head-path draft tree (drafting.cpp:122-245, greedy) with the transformer replaced by a
 * hidden-state provider: fn(user, level, n, tokens, parent_cand, hidden_out[n x d]).
 * level 0 asks for the single root row (tokens[0] = -1). Returns 0 or the provider's code. */
typedef int (*frs_o_hidden_fn)(void *user, int level, int n, const int32_t *tokens,
                               const int32_t *parent_cand, float *hidden_out);
int frs_o_draft_tree(frs_o_hidden_fn fn, void *user, const float *slab, int v_sub, int d,
                     const int32_t *ordered_ids, int width, int depth, int total,
                     int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint,
                     int *count);

#ifdef __cplusplus
}
#endif
/* host libm expf over bit patterns first_bits + i, i < count (SURVEY.md §4.4 KAT values) */
void frs_o_libm_expf_range(uint32_t first_bits, int64_t count, float *out);

#endif
