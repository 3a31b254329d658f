/* ORACLE / TEST INFRASTRUCTURE ONLY — plain-C restatement of the FR-Spec reference hot path.
 * See frs_oracle.h for the contract; every function cites /root/reference/proj lines.
 * Build: oracle/Makefile (-O3 -ffp-contract=off; never -ffast-math).
 */
#define _GNU_SOURCE
#include "frs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdlib.h>
#include <string.h>

/* kernels.cpp:13-32 */
float frs_o_dot_f32(const float *a, const float *b, int n) {
    float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f, s4 = 0.0f, s5 = 0.0f, s6 = 0.0f, s7 = 0.0f;
    int i = 0;
    for (; i + 8 <= n; i += 8) {
        s0 += a[i + 0] * b[i + 0];
        s1 += a[i + 1] * b[i + 1];
        s2 += a[i + 2] * b[i + 2];
        s3 += a[i + 3] * b[i + 3];
        s4 += a[i + 4] * b[i + 4];
        s5 += a[i + 5] * b[i + 5];
        s6 += a[i + 6] * b[i + 6];
        s7 += a[i + 7] * b[i + 7];
    }
    float s = ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7));
    for (; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* out[j - j0] = dot_f32(h, W_j) for j in [j0, j1), split over the host's cores: every element
 * is one dot_f32 call, so the split cannot change a bit (test speed only). */
typedef struct {
    const float *h, *W;
    int n, d, j0, j1, ld;
    float *out;
} dots_job;
static void *dots_worker(void *arg) {  /* W row j read once for all n hidden rows */
    const dots_job *J = (const dots_job *)arg;
    for (int j = J->j0; j < J->j1; ++j)
        for (int i = 0; i < J->n; ++i)
            J->out[(size_t)i * J->ld + j] = frs_o_dot_f32(J->h + (size_t)i * J->d, J->W + (size_t)j * J->d, J->d);
    return NULL;
}
/* out[i * ld + j] = dot_f32(h_i, W_j), i < n, j in [j0, j1) */
static void par_dots_n(const float *h, int n, const float *W, int d, int j0, int j1, float *out, int ld) {
    enum { kMaxT = 64 };
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > kMaxT) nt = kMaxT;
    if ((long)(j1 - j0) * d * n < (1L << 22)) nt = 1;
    pthread_t th[kMaxT];
    dots_job jobs[kMaxT];
    for (long t = 0; t < nt; ++t) {
        jobs[t] = (dots_job){h, W, n, d, j0 + (int)((long)(j1 - j0) * t / nt),
                             j0 + (int)((long)(j1 - j0) * (t + 1) / nt), ld, out};
        th[t] = 0;
        if (t > 0 && pthread_create(&th[t], NULL, dots_worker, &jobs[t]) != 0) {
            th[t] = 0;
            dots_worker(&jobs[t]);
        }
    }
    dots_worker(&jobs[0]);
    for (long t = 1; t < nt; ++t)
        if (th[t]) pthread_join(th[t], NULL);
}

/* kernels.cpp:34-60 (both branches give identical values: per-element order is fixed) */
void frs_o_logits(const float *h, int n, const float *W, int V, int d, float *out) {
    par_dots_n(h, n, W, d, 0, V, out, V);
}

/* glibc 2.39 sysdeps/ieee754/flt-32/e_expf.c as dispatched to the FMA ifunc on x86-64
 * (table __exp2f_data, N=32; verified bit-identical to host expf
 * over every float in [-104, 0]). */
static const uint64_t kExp2fT[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

float frs_o_expf_glibc(float x) {
    const double inv_ln2_n = 0x1.71547652b82fep+5, shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-20, c1 = 0x1.ebfce50fac4f3p-13, c2 = 0x1.62e42ff0c52d6p-6;
    uint32_t ux;
    memcpy(&ux, &x, 4);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42bu) { /* |x| >= 88 or nan */
        if (ux == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8u) return x + x;
        if (x > 0x1.62e42ep6f) return INFINITY;
        if (x < -0x1.9fe368p6f) return 0.0f;
    }
    const double xd = (double)x;
    double kd = fma(inv_ln2_n, xd, shift);
    uint64_t ki;
    memcpy(&ki, &kd, 8);
    kd -= shift;
    const double r = fma(inv_ln2_n, xd, -kd);
    const uint64_t t = kExp2fT[ki % 32] + (ki << 47);
    double s;
    memcpy(&s, &t, 8);
    const double z = fma(c0, r, c1);
    const double r2 = r * r;
    double y = fma(c2, r, 1.0);
    y = fma(z, r2, y);
    y = y * s;
    return (float)y;
}

/* kernels.cpp:62-91 */
int frs_o_softmax(const float *logits, int n, float temperature, float *probs, float *out_mx,
                  double *out_total) {
    if (n < 1 || !isfinite(temperature) || temperature <= 0.0f) return 1;
    float mx = -INFINITY;
    for (int i = 0; i < n; ++i) {
        if (!isfinite(logits[i])) return 1;
        const float v = logits[i] / temperature;
        mx = (mx < v) ? v : mx; /* std::max(mx, v) */
    }
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
        const float e = expf(logits[i] / temperature - mx);
        probs[i] = e;
        total += e;
    }
    const float inv = (float)(1.0 / total);
    for (int i = 0; i < n; ++i) probs[i] *= inv;
    if (out_mx) *out_mx = mx;
    if (out_total) *out_total = total;
    return 0;
}

/* (value desc, index asc) — the comparator of kernels.cpp:101-104 */
static int before(float va, int a, float vb, int b) { return va != vb ? va > vb : a < b; }

/* kernels.cpp:93-111 (partial_sort under a total order = insertion into a k-list) */
int frs_o_topk(const float *values, int n, int k, int32_t *idx, float *val) {
    if (k < 1 || k > n) return 1;
    int cnt = 0;
    for (int j = 0; j < n; ++j) {
        const float v = values[j];
        if (cnt == k && !before(v, j, val[k - 1], idx[k - 1])) continue;
        int p = cnt < k ? cnt++ : k - 1;
        while (p > 0 && before(v, j, val[p - 1], idx[p - 1])) {
            val[p] = val[p - 1];
            idx[p] = idx[p - 1];
            --p;
        }
        val[p] = v;
        idx[p] = j;
    }
    return 0;
}

/* kernels.cpp:113-122 */
int frs_o_argmax(const float *values, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (values[i] > values[best]) best = i;
    return best;
}

int frs_o_draft_level(const float *h, int n, const float *slab, int v_sub, int d,
                      const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx,
                      int32_t *out_full, float *out_prob, float *out_mx, double *out_total,
                      float *out_logits) {
    const int w = k < v_sub ? k : v_sub; /* drafting.cpp:40 */
    float *all = (float *)malloc(sizeof(float) * (size_t)v_sub * n);
    float *probs = (float *)malloc(sizeof(float) * (size_t)v_sub);
    int rc = 0;
    par_dots_n(h, n, slab, d, 0, v_sub, all, v_sub);
    for (int i = 0; i < n && rc == 0; ++i) {
        const float *logits = all + (size_t)i * v_sub;
        if (out_logits) memcpy(out_logits + (size_t)i * v_sub, logits, sizeof(float) * (size_t)v_sub);
        rc = frs_o_softmax(logits, v_sub, temperature, probs, out_mx ? out_mx + i : NULL,
                           out_total ? out_total + i : NULL);
        if (rc) break;
        rc = frs_o_topk(probs, v_sub, w, out_ridx + (size_t)i * k, out_prob + (size_t)i * k);
        for (int c = 0; c < w; ++c) {
            const int32_t r = out_ridx[(size_t)i * k + c];
            out_full[(size_t)i * k + c] = ordered_ids ? ordered_ids[r] : r;
        }
    }
    free(all);
    free(probs);
    return rc;
}

void frs_o_verify_argmax(const float *h, int m, const float *W, int V, int d, int32_t *out_id,
                         float *out_val) {
    float *row = (float *)malloc(sizeof(float) * (size_t)V);
    for (int i = 0; i < m; ++i) {
        par_dots_n(h + (size_t)i * d, 1, W, d, 0, V, row, V);
        float best = row[0];
        int bi = 0;
        for (int j = 1; j < V; ++j)
            if (row[j] > best) { /* kernels.cpp:117-121: strict '>' keeps the lowest id on ties */
                best = row[j];
                bi = j;
            }
        out_id[i] = bi;
        if (out_val) out_val[i] = best;
    }
    free(row);
}

/* verification.cpp:31-71 */
int frs_o_verify_greedy_ids(const int32_t *argmax_ids, const int32_t *tokens,
                            const int32_t *parents, int k, int32_t *emitted, int *n_emitted,
                            int32_t *path, int *n_path) {
    int node = -1, ne = 0, np = 0;
    for (;;) {
        const int32_t best = argmax_ids[node + 1];
        int match = -1;
        for (int c = 0; c < k; ++c) { /* children in node order == children_by_node order */
            if (parents[c] == node && tokens[c] == best) {
                match = c;
                break;
            }
        }
        emitted[ne++] = best;
        if (match < 0) break;
        path[np++] = match;
        node = match;
    }
    *n_emitted = ne;
    *n_path = np;
    return 0;
}

int frs_o_tree_mask(const int32_t *parents, int k, uint64_t *words) {
    if (k > 64) return 2;
    for (int i = 0; i < k; ++i) {
        if (parents[i] >= i) return 1;
        words[i] = (parents[i] >= 0 ? words[parents[i]] : 0) | ((uint64_t)1 << i);
    }
    return 0;
}

int frs_o_count_frequencies(const int32_t *stream, int64_t count, int vocab_size, uint64_t *counts) {
    if (vocab_size < 1) return 1;
    memset(counts, 0, sizeof(uint64_t) * (size_t)vocab_size);
    for (int64_t i = 0; i < count; ++i) {
        if (stream[i] < 0 || stream[i] >= vocab_size) return 1;
        ++counts[stream[i]];
    }
    return 0;
}

static int cmp_count_desc_id_asc(const void *pa, const void *pb, void *ctx) {
    const uint64_t *c = (const uint64_t *)ctx;
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    if (c[a] != c[b]) return c[a] > c[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* vocab.cpp:70-102, finalize_subset vocab.cpp:42-58 */
int frs_o_build_subset(const uint64_t *counts, int vocab_size, int size, const int32_t *forced,
                       int n_forced, int32_t *ordered_out) {
    if (size < 1 || size > vocab_size) return 1;
    for (int f = 0; f < n_forced; ++f)
        if (forced[f] < 0 || forced[f] >= vocab_size) return 1;
    char *is_member = (char *)calloc((size_t)vocab_size, 1);
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)vocab_size);
    int cnt = 0, rc = 0;
    for (int f = 0; f < n_forced; ++f) {
        if (!is_member[forced[f]]) {
            is_member[forced[f]] = 1;
            ordered_out[cnt++] = forced[f];
        }
    }
    if (cnt > size) rc = 1;
    if (!rc) {
        for (int t = 0; t < vocab_size; ++t) order[t] = t;
        qsort_r(order, (size_t)vocab_size, sizeof(int32_t), cmp_count_desc_id_asc, (void *)counts);
        for (int t = 0; t < vocab_size && cnt < size; ++t) {
            if (!is_member[order[t]]) {
                is_member[order[t]] = 1;
                ordered_out[cnt++] = order[t];
            }
        }
        qsort_r(ordered_out, (size_t)cnt, sizeof(int32_t), cmp_count_desc_id_asc, (void *)counts);
    }
    free(is_member);
    free(order);
    return rc;
}

/* vocab.cpp:104-138 */
int frs_o_subset_from_ranking(const int32_t *ranked, int n_ranked, int size, int vocab_size,
                              const int32_t *forced, int n_forced, int32_t *ordered_out) {
    if (size < 1 || size > n_ranked) return 1;
    for (int f = 0; f < n_forced; ++f)
        if (forced[f] < 0 || forced[f] >= vocab_size) return 1;
    char *seen = (char *)calloc((size_t)vocab_size, 1);
    int rc = 0;
    for (int i = 0; i < n_ranked && !rc; ++i) {
        if (ranked[i] < 0 || ranked[i] >= vocab_size || seen[ranked[i]]) rc = 1;
        else seen[ranked[i]] = 1;
    }
    if (!rc) {
        memset(seen, 0, (size_t)vocab_size);
        for (int i = 0; i < size; ++i) {
            ordered_out[i] = ranked[i];
            seen[ranked[i]] = 1;
        }
        int32_t *missing = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_forced + 1));
        int nm = 0;
        for (int f = 0; f < n_forced; ++f) {
            if (!seen[forced[f]]) {
                seen[forced[f]] = 1;
                missing[nm++] = forced[f];
            }
        }
        if (nm > size) rc = 1;
        else
            for (int i = 0; i < nm; ++i) ordered_out[size - 1 - i] = missing[nm - 1 - i];
        free(missing);
    }
    free(seen);
    return rc;
}

int frs_o_restrict(const float *W, int V, int d, const int32_t *ordered, int v_sub, float *out) {
    for (int i = 0; i < v_sub; ++i)
        if (ordered[i] < 0 || ordered[i] >= V) return 1;
    for (int i = 0; i < v_sub; ++i)
        memcpy(out + (size_t)i * d, W + (size_t)ordered[i] * d, sizeof(float) * (size_t)d);
    return 0;
}

/* ---- head-path draft tree: drafting.cpp:122-245 (greedy) ---- */
typedef struct {
    int32_t token, ridx, parent, depth;
    double log_joint;
} cand_t;

static const cand_t *g_cands; /* comparator context (oracle is single-threaded) */
static int cmp_lj_desc_idx_asc(const void *pa, const void *pb) {
    const int a = *(const int *)pa, b = *(const int *)pb;
    if (g_cands[a].log_joint != g_cands[b].log_joint)
        return g_cands[a].log_joint > g_cands[b].log_joint ? -1 : 1;
    return a < b ? -1 : (a > b);
}
static int cmp_int(const void *pa, const void *pb) {
    const int a = *(const int *)pa, b = *(const int *)pb;
    return a < b ? -1 : (a > b);
}

int frs_o_draft_tree(frs_o_hidden_fn fn, void *user, const float *slab, int v_sub, int d,
                     const int32_t *ordered_ids, int width, int depth, int total,
                     int32_t *tokens, int32_t *parents, int32_t *depths, double *log_joint,
                     int *count) {
    /* validate_params drafting.cpp:14-20 */
    if (width < 1 || depth < 1 || total < width || total > 64) return 1;
    const int w = width < v_sub ? width : v_sub;
    const size_t max_c = (size_t)w + (size_t)(depth - 1) * (size_t)width * (size_t)w;
    cand_t *cands = (cand_t *)malloc(sizeof(cand_t) * max_c);
    int *beam = (int *)malloc(sizeof(int) * (max_c + 1));
    int *next = (int *)malloc(sizeof(int) * (max_c + 1));
    float *hid = (float *)malloc(sizeof(float) * (size_t)width * (size_t)d);
    int32_t *btok = (int32_t *)malloc(sizeof(int32_t) * (size_t)width);
    int32_t *bpar = (int32_t *)malloc(sizeof(int32_t) * (size_t)width);
    int32_t *ridx = (int32_t *)malloc(sizeof(int32_t) * (size_t)width * (size_t)w);
    int32_t *full = (int32_t *)malloc(sizeof(int32_t) * (size_t)width * (size_t)w);
    float *prob = (float *)malloc(sizeof(float) * (size_t)width * (size_t)w);
    int nc = 0, nb = 0, rc = 0;

    /* level 0: root row (drafting.cpp:133-160) */
    btok[0] = -1;
    bpar[0] = -1;
    rc = fn(user, 0, 1, btok, bpar, hid);
    if (!rc) rc = frs_o_draft_level(hid, 1, slab, v_sub, d, ordered_ids, w, 1.0f, ridx, full, prob, NULL, NULL, NULL);
    for (int c = 0; c < w && !rc; ++c) {
        cands[nc] = (cand_t){full[c], ridx[c], -1, 1, log((double)prob[c])};
        beam[nb++] = nc++;
    }
    for (int level = 1; level < depth && nb > 0 && !rc; ++level) {
        if (nb > width) { /* drafting.cpp:164-176 */
            g_cands = cands;
            qsort(beam, (size_t)nb, sizeof(int), cmp_lj_desc_idx_asc);
            nb = width;
            qsort(beam, (size_t)nb, sizeof(int), cmp_int);
        }
        for (int i = 0; i < nb; ++i) {
            btok[i] = cands[beam[i]].token;
            bpar[i] = cands[beam[i]].parent;
        }
        rc = fn(user, level, nb, btok, bpar, hid);
        if (!rc) rc = frs_o_draft_level(hid, nb, slab, v_sub, d, ordered_ids, w, 1.0f, ridx, full, prob, NULL, NULL, NULL);
        int nn = 0;
        for (int i = 0; i < nb && !rc; ++i) { /* drafting.cpp:199-220 (UAF-patched semantics) */
            const cand_t p = cands[beam[i]];
            for (int c = 0; c < w; ++c) {
                const size_t o = (size_t)i * w + c;
                cands[nc] = (cand_t){full[o], ridx[o], beam[i], p.depth + 1,
                                     p.log_joint + log((double)prob[o])};
                next[nn++] = nc++;
            }
        }
        memcpy(beam, next, sizeof(int) * (size_t)nn);
        nb = nn;
    }
    if (!rc) { /* select_top_k greedy, drafting.cpp:79-118; emit 230-244 */
        int *order = (int *)malloc(sizeof(int) * (size_t)(nc + 1));
        char *sel = (char *)calloc((size_t)nc + 1, 1);
        int *remap = (int *)malloc(sizeof(int) * (size_t)(nc + 1));
        for (int i = 0; i < nc; ++i) order[i] = i;
        g_cands = cands;
        qsort(order, (size_t)nc, sizeof(int), cmp_lj_desc_idx_asc);
        int cnt = 0;
        for (int o = 0; o < nc; ++o) {
            const int c = order[o];
            if (cands[c].parent >= 0 && !sel[cands[c].parent]) continue;
            if (cnt + 1 > total) continue;
            sel[c] = 1;
            ++cnt;
        }
        int out = 0;
        for (int i = 0; i < nc; ++i) {
            if (!sel[i]) continue;
            remap[i] = out;
            tokens[out] = cands[i].token;
            parents[out] = cands[i].parent >= 0 ? remap[cands[i].parent] : -1;
            depths[out] = cands[i].depth;
            log_joint[out] = cands[i].log_joint;
            ++out;
        }
        *count = out;
        free(order);
        free(sel);
        free(remap);
    }
    free(cands);
    free(beam);
    free(next);
    free(hid);
    free(btok);
    free(bpar);
    free(ridx);
    free(full);
    free(prob);
    return rc;
}

/* The host libm's own expf (NOT the restatement above) over the float bit patterns
 * first_bits + i, i < count: the known-answer values the device ports are checked against
 * (SURVEY.md §4.4). Threads split the range; each value is one libm call. */
typedef struct {
    uint32_t first;
    int64_t i0, i1;
    float *out;
} expf_job;
static void *expf_worker(void *arg) {
    const expf_job *J = (const expf_job *)arg;
    for (int64_t i = J->i0; i < J->i1; ++i) {
        const uint32_t b = J->first + (uint32_t)i;
        float x;
        memcpy(&x, &b, 4);
        J->out[i] = expf(x);
    }
    return NULL;
}
void frs_o_libm_expf_range(uint32_t first_bits, int64_t count, float *out) {
    enum { kMaxT = 64 };
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > kMaxT) nt = kMaxT;
    pthread_t th[kMaxT];
    expf_job jobs[kMaxT];
    for (long t = 0; t < nt; ++t) {
        jobs[t] = (expf_job){first_bits, count * t / nt, count * (t + 1) / nt, out};
        th[t] = 0;
        if (t > 0 && pthread_create(&th[t], NULL, expf_worker, &jobs[t]) != 0) {
            th[t] = 0;
            expf_worker(&jobs[t]);
        }
    }
    expf_worker(&jobs[0]);
    for (long t = 1; t < nt; ++t)
        if (th[t]) pthread_join(th[t], NULL);
}
