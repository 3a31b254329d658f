// The draft model's transformer layer on the device (model.cpp:208-281
// forward_raw for the 1-layer draft): embedding gather -> RMSNorm -> q/k/v projections -> RoPE
// -> KV-cache append -> per-head masked attention -> o projection + residual -> RMSNorm -> 4d
// SiLU MLP + residual -> final RMSNorm (= the hidden state the FR head consumes). Every step
// reproduces the reference's float/double arithmetic bit for bit:
//  * projections: k_exact_logits (dot_f32 lane order, kernels.cpp:13-60) with fp32 weights;
//  * RMSNorm (model.cpp:29-40): the double sum of squares is a tree sum here; the float scale
//    1 / sqrt(ms / d + eps) is pinned by bracketing the reference's index-order sum (both within
//    gamma_d of the exact sum of exact double products), else replayed sequentially;
//  * RoPE (model.cpp:43-62): cos / sin / pow come from the host's glibc (tables per call),
//    the rotation is the reference's fmul / fsub / fadd sequence;
//  * SiLU: z / (1 + expf(-z)) with the glibc expf port; residual adds in float.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "frs_common.cuh"
#include "frs_device.cuh"

namespace frs {
namespace {

constexpr float kRmsEps = 1e-5f;

// One CTA per row: dst = (src * scale) * gain, scale = float(1 / sqrt(ms / d + eps)).
__global__ void __launch_bounds__(256)
    k_rmsnorm_rows(const float *__restrict__ x, int d, const float *__restrict__ gain, float *__restrict__ out) {
    __shared__ double s_red[32];
    __shared__ double s_ms;
    const int r = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    const float *src = x + (size_t)r * d;
    double part = 0.0;
    for (int j = tid; j < d; j += nt) part += static_cast<double>(src[j]) * src[j];
    const double tree = dev::block_reduce(part, dev::SumD(), s_red);
    auto scale_of = [&](double ms) {
        return static_cast<float>(1.0 / ::sqrt(ms / d + static_cast<double>(kRmsEps)));
    };
    const double del = static_cast<double>(d + 2 * nt) * 0x1p-52;
    const double lo = __dmul_rd(tree, 1.0 - del), hi = __dmul_ru(tree, 1.0 + del);
    float scale = scale_of(tree);
    if (scale_of(lo) != scale_of(hi)) {  // replay the index-order sum (model.cpp:33-34)
        if (tid == 0) {
            double ms = 0.0;
            for (int j = 0; j < d; ++j) ms += static_cast<double>(src[j]) * src[j];
            s_ms = ms;
        }
        __syncthreads();
        scale = scale_of(s_ms);
    } else {
        scale = scale_of(lo);
    }
    for (int j = tid; j < d; j += nt)
        out[(size_t)r * d + j] = __fmul_rn(__fmul_rn(src[j], scale), gain ? gain[j] : 1.0f);
}

// RoPE on [n x d] rows, heads of width dh: cs[(r * (dh/2) + i/2) * 2 + {0,1}] = cos, sin.
__global__ void k_rope(float *__restrict__ x, int n, int d, int dh, const float *__restrict__ cs) {
    const int half = dh / 2;
    const long long total = (long long)n * (d / dh) * half;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int ip = static_cast<int>(e % half);
        const long long rh = e / half;
        const int h = static_cast<int>(rh % (d / dh)), r = static_cast<int>(rh / (d / dh));
        float *hr = x + (size_t)r * d + (size_t)h * dh;
        const float c = cs[((size_t)r * half + ip) * 2], s = cs[((size_t)r * half + ip) * 2 + 1];
        const float x0 = hr[2 * ip], x1 = hr[2 * ip + 1];
        hr[2 * ip] = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
        hr[2 * ip + 1] = __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c));
    }
}

__global__ void k_silu(float *__restrict__ z, long long count) {
    __shared__ unsigned long long tab[32];
    dev::load_exp_table(tab);
    __syncthreads();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
        const float v = z[i];
        z[i] = __fdiv_rn(v, __fadd_rn(1.0f, dev::expf_glibc(-v, tab)));
    }
}

__global__ void k_add(float *__restrict__ x, const float *__restrict__ y, long long count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
        x[i] = __fadd_rn(x[i], y[i]);
}

int grid_for(long long count) { return (int)std::max<long long>(1, std::min<long long>(4096, (count + 255) / 256)); }

}  // namespace

int launch_masked_attention_strided(frs_ctx *ctx, const float *q, int q_ld, const float *k, int k_ld, const float *v,
                                    int v_ld, const unsigned long long *mask, int n, int m, int dh, int dv, int heads,
                                    float *out, int out_ld, uint32_t *flags, cudaStream_t s);
int gather_rows(const float *table, long long rows, int d, const int32_t *tokens, int n, float *out, cudaStream_t s);

}  // namespace frs

using namespace frs;

struct frs_draft_model {
    frs_ctx *ctx = nullptr;
    int V = 0, d = 0, heads = 0, max_seq = 0, len = 0;
    frs::DevBuf w;  // embedding | wq | wk | wv | wo | w_up | w_down | attn_norm | mlp_norm | final_norm
    frs::DevBuf kc, vc, work;
    float *emb, *wq, *wk, *wv, *wo, *wup, *wdown, *an, *mn, *fn;
    std::vector<int> positions;
    // RoPE cos / sin per position (model.cpp:50-54 with the host's libm), filled on first use:
    // the values depend only on (position, pair index), so a cache returns the same floats
    std::vector<std::vector<float>> rope;
    const float *rope_row(int pos) {
        const int dh = d / heads;
        auto fill = [&](std::vector<float> &cs) {
            cs.resize((size_t)dh);
            for (int i = 0; i + 1 < dh; i += 2) {
                const float freq = std::pow(10000.0f, -static_cast<float>(i) / dh);
                const float angle = static_cast<float>(pos) * freq;
                cs[(size_t)(i / 2) * 2] = std::cos(angle);
                cs[(size_t)(i / 2) * 2 + 1] = std::sin(angle);
            }
        };
        if (pos < 0 || pos >= 4 * max_seq) {  // outside the cached range: computed each time
            static thread_local std::vector<float> tmp;
            fill(tmp);
            return tmp.data();
        }
        if ((size_t)pos >= rope.size()) rope.resize((size_t)pos + 1);
        if (rope[pos].empty()) fill(rope[pos]);
        return rope[pos].data();
    }
};

extern "C" {

int frs_draft_model_create(frs_ctx *ctx, int V, int d, int heads, int max_seq, const float *embedding,
                           const float *wq, const float *wk, const float *wv, const float *wo, const float *w_up,
                           const float *w_down, const float *attn_norm, const float *mlp_norm,
                           const float *final_norm, frs_draft_model **out) {
    FRS_REQUIRE(ctx && out && embedding && wq && wk && wv && wo && w_up && w_down, "draft model: null pointer");
    if (V < 2 || d < 1 || heads < 1 || d % heads != 0 || max_seq < 1)
        return fail(FRS_EINVAL, "model config: bad vocab/hidden/heads/max_seq");  // model.cpp validate_config
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    auto *m = new frs_draft_model;
    m->ctx = ctx;
    m->V = V, m->d = d, m->heads = heads, m->max_seq = max_seq;
    const size_t dd = (size_t)d * d;
    const size_t total = (size_t)V * d + 4 * dd + 8 * dd + 3 * (size_t)d;
    int st;
    if ((st = m->w.ensure(total * sizeof(float))) || (st = m->kc.ensure((size_t)max_seq * d * sizeof(float))) ||
        (st = m->vc.ensure((size_t)max_seq * d * sizeof(float)))) {
        delete m;
        return st;
    }
    float *p = static_cast<float *>(m->w.ptr);
    m->emb = p, p += (size_t)V * d;
    m->wq = p, p += dd;
    m->wk = p, p += dd;
    m->wv = p, p += dd;
    m->wo = p, p += dd;
    m->wup = p, p += 4 * dd;
    m->wdown = p, p += 4 * dd;
    m->an = p, p += d;
    m->mn = p, p += d;
    m->fn = p;
    std::vector<float> ones(d, 1.0f);  // model.cpp: norm gains initialised to 1
    const std::pair<const float *, float *> parts[] = {
        {embedding, m->emb}, {wq, m->wq}, {wk, m->wk}, {wv, m->wv}, {wo, m->wo}, {w_up, m->wup}, {w_down, m->wdown}};
    const size_t sizes[] = {(size_t)V * d, dd, dd, dd, dd, 4 * dd, 4 * dd};
    for (int i = 0; i < 7; ++i)
        FRS_CUDA_TRY(cudaMemcpy(parts[i].second, parts[i].first, sizes[i] * sizeof(float), cudaMemcpyHostToDevice));
    FRS_CUDA_TRY(cudaMemcpy(m->an, attn_norm ? attn_norm : ones.data(), d * sizeof(float), cudaMemcpyHostToDevice));
    FRS_CUDA_TRY(cudaMemcpy(m->mn, mlp_norm ? mlp_norm : ones.data(), d * sizeof(float), cudaMemcpyHostToDevice));
    FRS_CUDA_TRY(cudaMemcpy(m->fn, final_norm ? final_norm : ones.data(), d * sizeof(float), cudaMemcpyHostToDevice));
    m->positions.assign(max_seq, 0);
    *out = m;
    return FRS_OK;
}

int frs_draft_model_destroy(frs_draft_model *m) {
    delete m;
    return FRS_OK;
}

int frs_draft_model_truncate(frs_draft_model *m, int new_len) {  // KVCache::truncate (model.cpp)
    FRS_REQUIRE(m, "draft model: null pointer");
    FRS_REQUIRE(new_len >= 0 && new_len <= m->len, "truncate: length out of range");
    m->len = new_len;
    return FRS_OK;
}

int frs_draft_model_length(const frs_draft_model *m, int *len) {
    FRS_REQUIRE(m && len, "draft model: null pointer");
    *len = m->len;
    return FRS_OK;
}

// KVCache::positions[row] (model.cpp: the position each cached row was forwarded at).
int frs_draft_model_position(const frs_draft_model *m, int row, int *pos) {
    FRS_REQUIRE(m && pos, "draft model: null pointer");
    FRS_REQUIRE(row >= 0 && row < m->len, "position: row out of range");
    *pos = m->positions[row];
    return FRS_OK;
}

// KVCache::compact (model.cpp:165-196): keep rows keep_from + kept_offsets[i] (ascending, in
// range) at keep_from + i, for K and V, and their positions; the same rejections in the same
// order. As in the reference, the contiguity check runs after the move (the cache is already
// compacted when it throws std::logic_error -> FRS_ELOGIC).
int frs_draft_model_compact(frs_draft_model *m, int keep_from, const int32_t *kept_offsets, int n_kept, void *stream) {
    FRS_REQUIRE(m && (kept_offsets || n_kept == 0), "draft model: null pointer");
    if (keep_from < 0 || keep_from > m->len) return fail(FRS_EINVAL, "KVCache::compact: bad keep_from");
    int prev = -1;
    for (int i = 0; i < n_kept; ++i) {
        const int off = kept_offsets[i];
        if (off <= prev || keep_from + off >= m->len)
            return fail(FRS_EINVAL, "KVCache::compact: offsets must be ascending and in range");
        prev = off;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    FRS_CUDA_TRY(cudaSetDevice(m->ctx->device));
    const int d = m->d;
    // src = keep_from + off_i >= dst = keep_from + i and src_i < src_j for i < j, so a forward
    // sweep of stream-ordered row copies never reads a row it already overwrote
    float *kc = static_cast<float *>(m->kc.ptr), *vc = static_cast<float *>(m->vc.ptr);
    for (int i = 0; i < n_kept; ++i) {
        const size_t src = (size_t)keep_from + kept_offsets[i], dst = (size_t)keep_from + i;
        if (src == dst) continue;
        FRS_CUDA_TRY(cudaMemcpyAsync(kc + dst * d, kc + src * d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
        FRS_CUDA_TRY(cudaMemcpyAsync(vc + dst * d, vc + src * d, sizeof(float) * d, cudaMemcpyDeviceToDevice, s));
    }
    for (int i = 0; i < n_kept; ++i) m->positions[keep_from + i] = m->positions[keep_from + kept_offsets[i]];
    m->len = keep_from + n_kept;
    for (int r = 1; r < m->len; ++r)
        if (m->positions[r] != m->positions[r - 1] + 1)
            return fail(FRS_ELOGIC, "KVCache::compact: kept positions are not contiguous");
    return FRS_OK;
}

// forward_raw (model.cpp:208-281) for the draft layer: tokens / positions host [n]; visible
// host BitMask words [n x ceil((len + n) / 64)] (bit j of row r: cache row j visible to token
// r); hidden_out device [n x d] (post final norm). Appends the n rows to the cache.
int frs_draft_model_forward(frs_draft_model *m, const int32_t *tokens, const int32_t *positions, int n,
                            const uint64_t *visible, float *hidden_out, void *stream) {
    FRS_REQUIRE(m && tokens && positions && visible && hidden_out, "forward: null pointer");
    if (n < 1) return fail(FRS_EINVAL, "forward: empty token batch");                     // model.cpp:217
    if (m->len + n > m->max_seq)
        return fail(FRS_ECAPACITY, "forward: sequence of " + std::to_string(m->len + n) + " exceeds max_seq_len " +
                                       std::to_string(m->max_seq));                       // model.cpp:219-222
    for (int i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= m->V)
            return fail(FRS_EINVAL, "forward: token id " + std::to_string(tokens[i]) + " out of range");
    frs_ctx *ctx = m->ctx;
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int d = m->d, dh = d / m->heads, len0 = m->len, mm = len0 + n, words = (mm + 63) / 64;
    // a query row that permits no key: the reference's masked_attention throws (kernels.cpp);
    // the mask is host data, so this is decided here without a device round trip
    for (int r = 0; r < n; ++r) {
        bool any = false;
        for (int w = 0; w < words && !any; ++w) {
            uint64_t bits = visible[(size_t)r * words + w];
            if (w == words - 1 && (mm & 63)) bits &= (1ull << (mm & 63)) - 1ull;
            any = bits != 0;
        }
        if (!any) return fail(FRS_EINVAL, "masked_attention: query row " + std::to_string(r) + " permits no keys");
    }
    // work: x | normed | q | k | v | attn | tmp | up (4d) | rope cs | mask | tokens
    const size_t nd = (size_t)n * d;
    const size_t need = (7 * nd + 4 * nd + (size_t)n * dh + 64) * sizeof(float) + (size_t)n * words * 8 + (size_t)n * 8 + 256;
    int st = m->work.ensure(need);
    if (st) return st;
    float *x = static_cast<float *>(m->work.ptr), *normed = x + nd, *q = normed + nd, *k = q + nd, *v = k + nd,
          *attn = v + nd, *tmp = attn + nd, *up = tmp + nd, *cs = up + 4 * nd;
    auto *mask = reinterpret_cast<unsigned long long *>(
        (reinterpret_cast<uintptr_t>(cs + (size_t)n * dh) + 15) & ~uintptr_t(15));
    auto *tok_dev = reinterpret_cast<int32_t *>(mask + (size_t)n * words);
    // host: the RoPE cos / sin with the reference's own libm calls (model.cpp:50-54)
    std::vector<float> hcs((size_t)n * dh);
    const size_t rs = (size_t)(dh / 2) * 2;  // k_rope's row stride
    for (int r = 0; r < n; ++r) std::memcpy(hcs.data() + (size_t)r * rs, m->rope_row(positions[r]), sizeof(float) * rs);
    FRS_CUDA_TRY(cudaMemcpyAsync(cs, hcs.data(), hcs.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    FRS_CUDA_TRY(cudaMemcpyAsync(mask, visible, (size_t)n * words * 8, cudaMemcpyHostToDevice, s));
    FRS_CUDA_TRY(cudaMemcpyAsync(tok_dev, tokens, n * 4, cudaMemcpyHostToDevice, s));
    if ((st = frs::gather_rows(m->emb, m->V, d, tok_dev, n, x, s))) return st;  // model.cpp:233-238
    frs::k_rmsnorm_rows<<<n, 256, 0, s>>>(x, d, m->an, normed);
    if ((st = launch_exact_logits(ctx, normed, n, d, m->wq, FRS_DTYPE_F32, d, q, s)) ||
        (st = launch_exact_logits(ctx, normed, n, d, m->wk, FRS_DTYPE_F32, d, k, s)) ||
        (st = launch_exact_logits(ctx, normed, n, d, m->wv, FRS_DTYPE_F32, d, v, s)))
        return st;
    const int rg = frs::grid_for((long long)n * d / 2);
    frs::k_rope<<<rg, 256, 0, s>>>(q, n, d, dh, cs);
    frs::k_rope<<<rg, 256, 0, s>>>(k, n, d, dh, cs);
    float *kc = static_cast<float *>(m->kc.ptr), *vc = static_cast<float *>(m->vc.ptr);
    FRS_CUDA_TRY(cudaMemcpyAsync(kc + (size_t)len0 * d, k, nd * sizeof(float), cudaMemcpyDeviceToDevice, s));
    FRS_CUDA_TRY(cudaMemcpyAsync(vc + (size_t)len0 * d, v, nd * sizeof(float), cudaMemcpyDeviceToDevice, s));
    uint32_t *fl = reinterpret_cast<uint32_t *>(tok_dev + n);
    if ((st = frs::launch_masked_attention_strided(ctx, q, d, kc, d, vc, d, mask, n, mm, dh, dh, m->heads, attn, d, fl, s)))
        return st;
    if ((st = launch_exact_logits(ctx, attn, n, d, m->wo, FRS_DTYPE_F32, d, tmp, s))) return st;
    frs::k_add<<<frs::grid_for((long long)nd), 256, 0, s>>>(x, tmp, (long long)nd);  // model.cpp:264
    frs::k_rmsnorm_rows<<<n, 256, 0, s>>>(x, d, m->mn, normed);
    if ((st = launch_exact_logits(ctx, normed, n, d, m->wup, FRS_DTYPE_F32, 4 * d, up, s))) return st;
    frs::k_silu<<<frs::grid_for(4LL * nd), 256, 0, s>>>(up, 4LL * (long long)nd);     // model.cpp:267
    if ((st = launch_exact_logits(ctx, up, n, 4 * d, m->wdown, FRS_DTYPE_F32, d, tmp, s))) return st;
    frs::k_add<<<frs::grid_for((long long)nd), 256, 0, s>>>(x, tmp, (long long)nd);  // model.cpp:268
    frs::k_rmsnorm_rows<<<n, 256, 0, s>>>(x, d, m->fn, hidden_out);                  // model.cpp:271
    FRS_CUDA_TRY(cudaGetLastError());
    ctx->launches += 8;
    for (int i = 0; i < n; ++i) m->positions[len0 + i] = positions[i];
    m->len = mm;
    return FRS_OK;
}

}  // extern "C"
