/* frspec_cuda.h — C ABI of the B200-native FR-Spec drafting hot path (libfrspec_cuda.so).
 *
 * Drop-in boundary for the reference's C++ hot-path API (/root/reference/proj). The
 * reference has no FFI of its own; these entry points are what a binding of its
 * library API would bind, one per hot-path function:
 *
 *   frs_slab_build          replaces restrict_lm_head            vocab.cpp:152-168, vocab.h:49-52
 *   frs_draft_head_topk     replaces forward_raw's LM-head line + softmax + pick_children/topk
 *                           + RankedSubset::full_id              model.cpp:276-279, kernels.cpp:62-111,
 *                                                                drafting.cpp:37-43,138-156,199-215
 *   frs_verify_head_argmax  replaces the target LM head + argmax model.cpp:324-338, kernels.cpp:113-122
 *   frs_accept_greedy       replaces verify_greedy's walk        verification.cpp:31-71
 *   frs_argmax_merge        (new) vocab-parallel merge of per-shard (value, id) argmax pairs
 *   frs_count_frequencies / frs_build_subset / frs_subset_from_ranking / frs_tree_mask
 *                           host-side restatements of vocab.cpp:23-138 / verification.cpp:13-27
 *   frs_head_* / frs_draft_tree / frs_verify_greedy
 *                           host-buffer conveniences mirroring RestrictedHead, build_draft_tree
 *                           (drafting.cpp:122-245, head path) and verify_greedy.
 *
 * Conventions: plain pointers and sizes; `stream` is a cudaStream_t (NULL = legacy default
 * stream). Device-pointer entry points are asynchronous on `stream` and never allocate
 * after frs_ctx_reserve(); outputs go to caller-owned buffers. Every function returns an
 * frs_status; frs_last_error() gives the thread-local message. Status codes map 1:1 onto
 * the reference's exception types (errors.h:7-17).
 */
#ifndef FRSPEC_CUDA_H
#define FRSPEC_CUDA_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRS_ABI_VERSION 1

#if defined(__GNUC__)
#define FRS_API __attribute__((visibility("default")))
#else
#define FRS_API
#endif

typedef enum {
    FRS_OK = 0,
    FRS_EINVAL = 1,    /* std::invalid_argument (rejected arguments)          errors.h:7     */
    FRS_ECAPACITY = 2, /* frspec::CapacityError (64-node trees, capacities)   errors.h:10-12 */
    FRS_EDATA = 3,     /* frspec::DataError                                   errors.h:15-17 */
    FRS_ELOGIC = 4,    /* std::logic_error / std::domain_error                               */
    FRS_ECUDA = 5,     /* CUDA runtime failure                                               */
    FRS_ENCCL = 6,     /* NCCL failure                                                       */
    FRS_ENOTSUP = 7    /* shape/dtype/mode combination not built for this device            */
} frs_status;

typedef enum { FRS_DTYPE_F32 = 0, FRS_DTYPE_BF16 = 1 } frs_dtype;

/* EXACT: CUDA-core kernels that reproduce the reference arithmetic bit for bit (dot_f32
 *        lane order without FMA, glibc expf, index-order double Σ, (p desc, idx asc) top-k).
 * FAST:  tcgen05 tensor-core head over a bf16 slab; ids/argmax certified against an
 *        exact recompute of the candidates, probabilities within tolerance. */
typedef enum { FRS_MODE_EXACT = 0, FRS_MODE_FAST = 1 } frs_mode;

/* Per-row flag bits written to out_flags (when non-NULL). */
#define FRS_FLAG_NONFINITE 0x1u  /* a logit was NaN/inf: the reference throws (kernels.cpp:72-74) */
#define FRS_FLAG_SEQ_SUM 0x2u    /* Σ exp took the index-order sequential path                  */
#define FRS_FLAG_UNCERTIFIED 0x4u /* FAST: candidate set could not be certified (ids may differ) */
#define FRS_FLAG_RECOMPUTED 0x8u /* FAST: row fell back to the exact kernel                     */
/* FAST: why a row fell back (set together with FRS_FLAG_RECOMPUTED) — "ties at tolerance". */
#define FRS_FLAG_CERT_TIE 0x10u      /* two selected probabilities within 4 ulps: order needs exact Σ  */
#define FRS_FLAG_CERT_BOUND 0x20u    /* the rigorous error bound did not separate the k-th candidate   */
#define FRS_FLAG_CERT_OVERFLOW 0x40u /* more near-boundary candidates than the exact-recompute set     */
/* FAST, certified rows: bits 8..15 hold the size of the exactly recomputed candidate set (info). */
#define FRS_FLAG_EMPTY_ROW 0x100u          /* masked_attention: the row permits no key (reference throws)  */
#define FRS_FLAG_SAMPLE_UNCERTIFIED 0x80u /* sampled draw inside the rounding bound: host replays the level */
#define FRS_FLAG_CAND_SHIFT 8

typedef struct frs_ctx frs_ctx;
typedef struct frs_head frs_head;

FRS_API int frs_abi_version(void);
FRS_API const char *frs_last_error(void);

FRS_API int frs_ctx_create(int device, frs_ctx **out);
FRS_API int frs_ctx_destroy(frs_ctx *ctx);
FRS_API int frs_ctx_sm_count(const frs_ctx *ctx);
/* Live device timing of each call's dominant kernel (CUDA events on the launch stream), for
 * the roofline measurement: enable, run, then read the summed milliseconds and call count. */
FRS_API int frs_ctx_set_timing(frs_ctx *ctx, int enable);
FRS_API int frs_ctx_timing_read(frs_ctx *ctx, double *total_ms, int *count);
/* Latency-bound callers (a dependent draft loop): repeated FAST calls with identical buffers and
 * shapes replay one captured CUDA graph of the chain instead of eager launches (default off:
 * back to back, eager launches keep the PDL overlap with the previous call's tail). */
FRS_API int frs_ctx_set_graphs(frs_ctx *ctx, int enable);
/* Diagnostic: copy the partials of the last FAST call to host buffers: per hidden row one list
 * per (CTA, TMEM lane quarter), L = 4 G lists (G = frs_ctx_sm_count): [n][L] max / sum-exp /
 * bound, [n][L][3] candidate keys, [2 G] max |W_j|^2. With FRS_TRACE set, pkey must have room
 * for the globaltimer trace after the keys (see tools/fast_trace.py). */
FRS_API int frs_debug_fast_partials(frs_ctx *ctx, int n, int d, float *pm, float *ps, float *pth,
                                    uint64_t *pkey, float *pw2);
/* Known-answer check of the device glibc expf ports: for the float bit
 * patterns first_bits + i, i < count, compare both device ports (branchy expf_glibc and
 * branch-free expf_glibc_nb) with expected[i] (the host libm's expf, device buffer). out
 * (device, 4 x u64, out[2..3] preset to ~0): mismatch counts, first mismatching i. */
FRS_API int frs_debug_expf_check(frs_ctx *ctx, uint32_t first_bits, int64_t count, const float *expected,
                                 uint64_t *out, void *stream);
/* Number of kernels this library has launched on ctx (evidence for bench gpu_launches). */
FRS_API int frs_ctx_launch_count(const frs_ctx *ctx, uint64_t *out);
/* Pre-size workspaces for up to max_rows hidden rows against up to max_vocab head rows. */
FRS_API int frs_ctx_reserve(frs_ctx *ctx, int max_rows, int64_t max_vocab, int d);

/* K1 — restrict_lm_head (vocab.cpp:152-168): slab[i,:] = W[ordered_ids[i],:], bitwise for
 * FRS_DTYPE_F32, round-to-nearest-even for FRS_DTYPE_BF16. W, ordered_ids, slab: device.
 * Out-of-range ids -> FRS_EINVAL (this call synchronizes `stream` to report it). */
FRS_API int frs_slab_build(frs_ctx *ctx, const float *W, int64_t V, int d, const int32_t *ordered_ids,
                   int v_sub, int slab_dtype, void *slab, void *stream);
FRS_API size_t frs_slab_bytes(int v_sub, int d, int slab_dtype);

/* K2 — one draft level for n hidden rows h[n x d] (fp32, device) against the slab:
 * logits = h . slab^T; per row softmax(logits / temperature); top-min(k, v_sub) by
 * (prob desc, restricted index asc); full = ordered_ids[ridx] (identity when NULL).
 * Outputs [n x k] (device): out_ridx, out_full, out_prob; optional [n]: out_rowmax (the
 * softmax max), out_total (the double Σ), out_flags; optional [n x v_sub] out_logits. */
FRS_API int frs_draft_head_topk(frs_ctx *ctx, const float *h, int n, int d, const void *slab, int v_sub,
                        int slab_dtype, const int32_t *ordered_ids, int k, float temperature,
                        int mode, int32_t *out_ridx, int32_t *out_full, float *out_prob,
                        float *out_rowmax, double *out_total, float *out_logits,
                        uint32_t *out_flags, void *stream);

/* The bf16 slab in the FAST head's stream order ("tiled image"): for every 64-column K block and
 * 32-row chunk one 4 KB block holding the SWIZZLE_128B shared-memory image of those 32 rows x
 * 128 bytes, blocks ordered [K block][chunk] — so each pipeline stage of the FAST head (a
 * CTA's 1-4 consecutive chunks of one K block) is ONE contiguous 1-D bulk copy instead of a
 * 2-D tensor load (measured: 62.8 -> 58.4 us per Llama-3-8B draft level). Built once per slab
 * (frs_slab_tile; zero fill past v_rows / d), kept next to the row-major slab, which the exact
 * recompute of the certified candidates still reads. Same bytes as the slab (rounded up to
 * whole chunks and K blocks). frs_draft_head_topk_tiled = frs_draft_head_topk in FAST mode
 * (slab_dtype bf16) with the tiled image of that slab. */
FRS_API size_t frs_slab_tile_bytes(int v_rows, int d);
FRS_API int frs_slab_tile(frs_ctx *ctx, const void *slab, int v_rows, int d, void *tiled, void *stream);
FRS_API int frs_draft_head_topk_tiled(frs_ctx *ctx, const float *h, int n, int d, const void *slab,
                                      const void *tiled, int v_sub, const int32_t *ordered_ids, int k,
                                      float temperature, int32_t *out_ridx, int32_t *out_full, float *out_prob,
                                      float *out_rowmax, double *out_total, uint32_t *out_flags, void *stream);

/* K3 — full-vocabulary verify head over rows [id_offset, id_offset + v_rows) of the LM head
 * (W points at that shard): per row i of h[m x d], out_id[i] = id_offset + argmax_j
 * dot_f32(h_i, W_j) with ties to the lowest id, out_val[i] = that logit. Device buffers. */
FRS_API int frs_verify_head_argmax(frs_ctx *ctx, const float *h, int m, int d, const void *W, int v_rows,
                           int w_dtype, int32_t id_offset, int mode, int32_t *out_id,
                           float *out_val, uint32_t *out_flags, void *stream);
/* frs_verify_head_argmax in FAST mode over a bf16 shard W with its tiled image W_tiled
 * (frs_slab_tile(ctx, W, v_rows, d, W_tiled, …)): the shard streams as 1-D bulk copies. */
FRS_API int frs_verify_head_argmax_tiled(frs_ctx *ctx, const float *h, int m, int d, const void *W,
                                         const void *W_tiled, int v_rows, int32_t id_offset, int32_t *out_id,
                                         float *out_val, uint32_t *out_flags, void *stream);

/* K4 — greedy accept walk (verification.cpp:42-71). argmax_ids[0] belongs to the root
 * position, argmax_ids[1+i] to draft node i. Writes out_emitted[<=k+1], out_path[<=k] and
 * out_counts = {n_emitted, n_path}. Device buffers. */
FRS_API int frs_accept_greedy(frs_ctx *ctx, const int32_t *argmax_ids, const int32_t *tokens,
                      const int32_t *parents, int k, int32_t *out_emitted, int32_t *out_path,
                      int32_t *out_counts, void *stream);

/* K5 — merge per-shard argmax pairs vals/ids[shards x m] (shard-major) by (value desc,
 * id asc): reproduces argmax's lowest-id rule over a contiguous vocab split. Device. */
FRS_API int frs_argmax_merge(frs_ctx *ctx, const float *vals, const int32_t *ids, int shards, int m,
                     float *out_val, int32_t *out_id, void *stream);

/* Vocab-parallel verify helpers: the contiguous vocabulary shard of `rank`
 * among `world` ranks, and the host twin of frs_argmax_merge for host-resident all-gathers. */
FRS_API int frs_vocab_shard(int64_t V, int world, int rank, int64_t *start, int64_t *count);
FRS_API int frs_argmax_merge_host(const float *vals, const int32_t *ids, int shards, int m, float *out_val,
                                  int32_t *out_id);

/* Row gather out[i,:] = table[tokens[i],:] (the identity draft layer of the head-path decode
 * loop). Device buffers. */
FRS_API int frs_gather_rows(frs_ctx *ctx, const float *table, int64_t rows, int d, const int32_t *tokens,
                    int n, float *out, void *stream);

/* ---- host-side FR vocabulary (vocab.cpp:23-138) and tree mask (verification.cpp:13-27) ---- */
FRS_API int frs_count_frequencies(const int32_t *stream, int64_t count, int vocab_size, uint64_t *counts);
/* count_frequencies (vocab.cpp:23-38) on the device: tokens and counts [vocab_size] are device
 * buffers; synchronises `stream` to report the first out-of-range id (FRS_EINVAL, the
 * reference's message). */
FRS_API int frs_count_frequencies_device(frs_ctx *ctx, const int32_t *tokens, int64_t count, int vocab_size,
                                         uint64_t *counts, void *stream);
/* Token-stream files (vocab.cpp:198-286): binary "FRTK" v1 (u32 vocab_size, u64 count, u32
 * ids, little endian) and whitespace-separated text; ranked-id files (vocab.cpp:288-308).
 * Readers: pass tokens/ids = NULL to get the count, then a buffer of that capacity.
 * Errors: FRS_EDATA with the reference's DataError messages. */
FRS_API int frs_write_token_stream(const char *path, int vocab_size, const int32_t *tokens, int64_t count);
FRS_API int frs_read_token_stream(const char *path, int32_t *tokens, int64_t capacity, int *vocab_size,
                                  int64_t *count);
FRS_API int frs_read_token_stream_text(const char *path, int vocab_size, int32_t *tokens, int64_t capacity,
                                       int64_t *count);
FRS_API int frs_write_ranked_file(const char *path, const int32_t *ids, int64_t n);
FRS_API int frs_read_ranked_file(const char *path, int32_t *ids, int64_t capacity, int64_t *n);
FRS_API int frs_build_subset(const uint64_t *counts, int vocab_size, int size, const int32_t *forced,
                     int n_forced, int32_t *ordered_out);
FRS_API int frs_subset_from_ranking(const int32_t *ranked, int n_ranked, int size, int vocab_size,
                            const int32_t *forced, int n_forced, int32_t *ordered_out);
FRS_API int frs_coverage(const uint64_t *counts, int vocab_size, const int32_t *ordered, int v_sub,
                 double *out);
FRS_API int frs_flops_ratio(int full_size, int restricted_size, double *out);
FRS_API int frs_tree_mask(const int32_t *parents, int k, uint64_t *words);

/* ---- device-resident RestrictedHead and host-buffer conveniences ---- */
/* W is host memory unless w_on_device; ordered_ids is host memory (validated on the host). */
FRS_API int frs_head_create(frs_ctx *ctx, const float *W, int64_t V, int d, int w_on_device,
                    const int32_t *ordered_ids, int v_sub, int slab_dtype, frs_head **out);
FRS_API int frs_head_destroy(frs_head *head);
FRS_API int frs_head_info(const frs_head *head, const void **slab, const int32_t **ordered_dev,
                  int *v_sub, int *d, int *slab_dtype);
/* One level end to end with HOST buffers: H2D h, K2, D2H outputs, synchronize. */
FRS_API int frs_head_draft_host(frs_head *head, const float *h_host, int n, int k, int mode,
                        int32_t *ridx, int32_t *full, float *prob);

/* Hidden-state provider for the head-path draft tree: fill hidden_dev[n x d] (device) for
 * the n forwarded rows of `level` (level 0: the single root row, tokens[0] = root token;
 * parent_cands[i] = parent candidate index, -1 at the root). Return 0 or an error code. */
typedef int (*frs_hidden_fn)(void *user, int level, int n, const int32_t *tokens,
                             const int32_t *parent_cands, float *hidden_dev, void *stream);
/* build_draft_tree restricted to the head path (drafting.cpp:122-245, greedy): hidden rows
 * come from fn, or from rows of hidden_table[V x d] (device) by token when fn is NULL.
 * Tree outputs are host arrays of capacity `total`. */
FRS_API int frs_draft_tree(frs_head *head, int32_t root_token, frs_hidden_fn fn, void *user,
                   const float *hidden_table, int width, int depth, int total, int mode,
                   int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint,
                   int *count);
/* masked_attention (kernels.cpp:124-171), the tree attention of the draft / target forwards:
 * q [n x dh], k [m x dh], v [m x dv] fp32 and mask [n x ceil(m/64)] u64 (bit j of row r = key j
 * visible to query r, the reference's BitMask words) on the device; out [n x dv]. Bit-exact with
 * the reference (dot_f32 order, glibc expf, pinned 1/Σ, key-ordered accumulation). flags [n]:
 * FRS_FLAG_EMPTY_ROW where a row permits no key (the reference throws; the row is zeros). */
FRS_API int frs_masked_attention(frs_ctx *ctx, const float *q, const float *k, const float *v, const uint64_t *mask,
                                 int n, int m, int dh, int dv, float *out, uint32_t *flags, void *stream);
/* The draft model's transformer layer (model.cpp:208-281 forward_raw, 1-layer draft) on the
 * device, bit-exact with the reference: weights host fp32 (LayerWeights layout, x * W^T; NULL
 * gains = 1), a device KV cache of max_seq rows. forward: tokens / positions host [n], visible
 * host BitMask words [n x ceil((len + n) / 64)] over cache rows [0, len + n), hidden_out device
 * [n x d] (post final norm); appends the rows to the cache. FRS_ECAPACITY past max_seq. */
typedef struct frs_draft_model frs_draft_model;
FRS_API int frs_draft_model_create(frs_ctx *ctx, int V, int d, int heads, int max_seq, const float *embedding,
                                   const float *wq, const float *wk, const float *wv, const float *wo,
                                   const float *w_up, const float *w_down, const float *attn_norm,
                                   const float *mlp_norm, const float *final_norm, frs_draft_model **out);
FRS_API int frs_draft_model_destroy(frs_draft_model *m);
FRS_API int frs_draft_model_truncate(frs_draft_model *m, int new_len);
FRS_API int frs_draft_model_length(const frs_draft_model *m, int *len);
FRS_API int frs_draft_model_forward(frs_draft_model *m, const int32_t *tokens, const int32_t *positions, int n,
                                    const uint64_t *visible, float *hidden_out, void *stream);
/* KVCache::positions[row] (model.cpp:280, 288-297): the position cached row `row` was forwarded
 * at; FRS_EINVAL outside [0, len). */
FRS_API int frs_draft_model_position(const frs_draft_model *m, int row, int *pos);
/* KVCache::compact (model.cpp:165-196): keeps cached rows keep_from + kept_offsets[i] (ascending,
 * < len) at keep_from + i with their positions; len = keep_from + n_kept. FRS_EINVAL for a bad
 * keep_from or offsets (nothing moved); FRS_ELOGIC when the kept positions are not contiguous
 * (raised after the move, as the reference's std::logic_error is). */
FRS_API int frs_draft_model_compact(frs_draft_model *m, int keep_from, const int32_t *kept_offsets, int n_kept,
                                    void *stream);
typedef struct frs_rng frs_rng;
/* build_draft_tree (drafting.cpp:122-245) driven by the device draft model: forwards the
 * pending context (root = its last token) and each level's beam through frs_draft_model with
 * the reference's positions and visibility, then truncates the cache back to the context.
 * rng == NULL: greedy (levels EXACT); else sampled (EXACT). Outputs as frs_draft_tree; keep_probs
 * outputs as frs_draft_tree_sampled (with an rng only, else FRS_ENOTSUP). */
FRS_API int frs_draft_tree_model(frs_head *head, frs_draft_model *draft, const int32_t *pending, int n_pending,
                                 int width, int depth, int total, int mode, frs_rng *rng, int32_t *tokens,
                                 int32_t *parents, int32_t *depths, double *log_joint, int *count, float *root_probs,
                                 float *node_probs, int32_t *has_probs);
/* Sampled drafting (drafting.cpp:44-74): a std::mt19937_64 the caller owns (the reference's
 * `std::mt19937_64 * rng`), advanced by every draw exactly as the reference advances it. */
typedef struct frs_rng frs_rng;
FRS_API int frs_rng_create(uint64_t seed, frs_rng **out);
FRS_API int frs_rng_destroy(frs_rng *rng);
/* Uniforms in [0, 1) the way std::uniform_real_distribution<double>(0, 1) draws them (tests). */
FRS_API int frs_rng_uniforms(frs_rng *rng, int count, double *out);
/* K2 sampled (EXACT arithmetic only): per row, the exact softmax (kernels.cpp:62-91) into
 * probs [n x v_sub] (device) and w = min(width, v_sub) draws without replacement with the
 * given uniforms (device, [n x w], draw order) — pick_children's sampled branch. Outputs
 * ridx/full/prob [n x w] in draw order, count[n] draws made, flags[n] (FRS_FLAG_SAMPLE_
 * UNCERTIFIED: a draw was not certified; the caller replays the row from probs). */
FRS_API int frs_draft_head_sample(frs_ctx *ctx, const float *h, int n, int d, const void *slab, int v_sub,
                                  int slab_dtype, const int32_t *ordered_ids, int width, float temperature,
                                  const double *uniforms, float *probs, int32_t *out_ridx, int32_t *out_full,
                                  float *out_prob, int32_t *out_count, uint32_t *out_flags, void *stream);
/* build_draft_tree with an rng (drafting.cpp:122-245: sampled children, prefix-closed
 * select_top_k), head path, EXACT arithmetic. Same arguments as frs_draft_tree plus rng.
 * keep_probs (drafting.h:31-37, DraftResult): root_probs [v_sub] and node_probs [total x v_sub]
 * with has_probs [total] (0 = node not expanded, its row untouched), host buffers; NULL = off. */
FRS_API int frs_draft_tree_sampled(frs_head *head, int32_t root_token, frs_hidden_fn fn, void *user,
                                   const float *hidden_table, int width, int depth, int total, frs_rng *rng,
                                   int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint,
                                   int *count, float *root_probs, float *node_probs, int32_t *has_probs);
/* verify_stochastic (verification.cpp:76-178): h_dev holds 1 + k target rows (root first),
 * W the full target head [V x d]. The device computes the EXACT target logits and softmax
 * probabilities (kernels.cpp:13-32, 62-91); the residual walk (accept with probability
 * min(1, p/q), p <- norm(max(0, p - q)) on rejection, bonus token from the residual) runs on the
 * host in the reference's double arithmetic over those probabilities, drawing from rng. The
 * draft distributions: q_root [v_sub], q_nodes [k x v_sub] with has_q[i] = 0 for nodes that
 * were not expanded; ordered (host, v_sub ids) maps draft indices to tokens (NULL: identity). */
FRS_API int frs_verify_stochastic(frs_ctx *ctx, const float *h_dev, const void *W, int V, int d, int w_dtype,
                                  const int32_t *tokens, const int32_t *parents, int k, const float *q_root,
                                  int v_sub, const float *q_nodes, const int32_t *has_q, const int32_t *ordered,
                                  float temperature, frs_rng *rng, int32_t *emitted, int *n_emitted, int32_t *path,
                                  int *n_path);
/* verify_greedy (verification.cpp:42-71) with the target head on the device: h_dev holds
 * 1 + k rows (root first), W the full LM head [V x d] (device). Host outputs. */
FRS_API int frs_verify_greedy(frs_ctx *ctx, const float *h_dev, const void *W, int V, int d, int w_dtype,
                      int mode, const int32_t *tokens, const int32_t *parents, int k,
                      int32_t *emitted, int *n_emitted, int32_t *path, int *n_path);

/* verify_greedy with the hidden rows gathered on the device from table[V_table x d] by
 * [root_token, tokens...] (the head-path decode loop's identity layer). Host outputs. */
FRS_API int frs_verify_greedy_table(frs_ctx *ctx, const float *table, int64_t V_table, int32_t root_token,
                                    const void *W, int V, int d, int w_dtype, int mode, const int32_t *tokens,
                                    const int32_t *parents, int k, int32_t *emitted, int *n_emitted, int32_t *path,
                                    int *n_path);

/* One head-path decode iteration (drafting.cpp:122-245 then verification.cpp:42-71): the greedy
 * draft tree from the head h over hidden rows table[h->vocab x d] (device), then verify_greedy of
 * [root_token, tree tokens...] against the full head W [V x d] (device) in verify_mode, with no
 * host round trip between the two (one synchronisation). Results equal frs_draft_tree followed
 * by frs_verify_greedy_table; tokens/parents/depths/log_joint hold >= total entries, emitted
 * total + 1, path total. */
FRS_API int frs_decode_step_table(frs_head *h, const float *table, int32_t root_token, const void *W, int V,
                                  int w_dtype, int verify_mode, int width, int depth, int total, int32_t *tokens,
                                  int32_t *parents, int32_t *depths, double *log_joint, int *count,
                                  int32_t *emitted, int *n_emitted, int32_t *path, int *n_path);

/* S independent decode streams (BASELINE configs[4]), one head-path iteration each: per stream
 * exactly frs_decode_step_table(roots[q]) (drafting.cpp:122-245, verification.cpp:42-71), with the
 * streams batched — every draft level is one EXACT head call over all streams' beam rows (rows
 * are independent, drafting.cpp:189-193) and the verify head one call over all streams'
 * [root, tokens...] rows. Outputs per stream q: tokens/parents/depths/log_joint/path at
 * [q * total], emitted at [q * (total + 1)], count/n_emitted/n_path at [q]. */
FRS_API int frs_decode_step_table_multi(frs_head *h, const float *table, int S, const int32_t *roots, const void *W,
                                        const void *W_tiled, int V, int w_dtype, int verify_mode, int width, int depth,
                                        int total, int32_t *tokens, int32_t *parents, int32_t *depths,
                                        double *log_joint, int *count, int32_t *emitted, int *n_emitted,
                                        int32_t *path, int *n_path);
/* frs_decode_step_table with the bf16 verify head's tiled image W_tiled (frs_slab_tile of W): the
 * FAST verify head streams it; W_tiled may be NULL in frs_decode_step_table_multi. */
FRS_API int frs_decode_step_table_tiled(frs_head *h, const float *table, int32_t root_token, const void *W,
                                        const void *W_tiled, int V, int verify_mode, int width, int depth, int total,
                                        int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint,
                                        int *count, int32_t *emitted, int *n_emitted, int32_t *path, int *n_path);

/* Vocab-parallel verify head (SURVEY.md §8(b) frs_allgather_merge, §8(e)): every rank of an NCCL
 * communicator holds the contiguous LM-head shard [id_offset, id_offset + v_rows) (frs_vocab_shard)
 * and calls this with the same 1 + k hidden rows h [m x d]: K3 over its shard, ncclAllGather of
 * the per-row (value, id) pairs over NVLink / NVSwitch, K5 merge by (value desc, id asc) = the
 * reference argmax's lowest-id rule over contiguous shards (kernels.cpp:113-122). out_id / out_val
 * [m] (device) hold the global argmax on every rank; out_flags [m] this rank's K3 flags.
 * comm is an ncclComm_t (NCCL resolved at run time: FRS_ENCCL when unavailable or failing,
 * ncclCommGetAsyncError checked). frs_nccl_get_unique_id writes an ncclUniqueId (128 bytes) to be
 * broadcast to every rank; frs_nccl_comm_init makes this rank's communicator on ctx's device. */
FRS_API int frs_nccl_get_unique_id(void *id_out);
FRS_API int frs_nccl_comm_init(frs_ctx *ctx, int nranks, const void *id, int rank, void **comm_out);
FRS_API int frs_nccl_comm_destroy(void *comm);
FRS_API int frs_verify_head_argmax_vp(frs_ctx *ctx, void *comm, const float *h, int m, int d, const void *W_shard,
                                      int v_rows, int w_dtype, int32_t id_offset, int mode, int32_t *out_id,
                                      float *out_val, uint32_t *out_flags, void *stream);

/* AcceptanceStats (verification.h:52-62, verification.cpp:180-206): accepted lengths are
 * VerifyOutcome::accepted_length() = |emitted| (accepted tokens + the bonus), at most 65 for a
 * 64-node tree; histogram[len] counts iterations of that length, hist_len = the reference's
 * histogram.size(). add: FRS_EINVAL outside [0, FRS_HIST_MAX). accepted_length_stats: FRS_EINVAL
 * "accepted_length_stats: empty outcome list" for n == 0 (verification.cpp:199-201). */
#define FRS_HIST_MAX 72
typedef struct frs_acceptance_stats {
    int64_t iterations;
    int64_t emitted;
    double mean_accepted_length;
    int32_t hist_len;
    int32_t pad_;
    int64_t histogram[FRS_HIST_MAX];
} frs_acceptance_stats;
FRS_API int frs_acceptance_add(frs_acceptance_stats *s, int accepted_length);
FRS_API int frs_acceptance_merge(frs_acceptance_stats *s, const frs_acceptance_stats *other);
FRS_API int frs_accepted_length_stats(const int32_t *accepted_lengths, int n, frs_acceptance_stats *out);

#ifdef __cplusplus
}
#endif
#endif /* FRSPEC_CUDA_H */
