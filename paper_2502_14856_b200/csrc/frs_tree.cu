// Device-side beam bookkeeping for the head-path build_draft_tree (drafting.cpp:122-245,
// greedy). One level per call of k_tree_level after the level's gather + K2: the children of
// the forwarded beam become candidates (token, head index, parent, depth, log_joint), the next
// beam is the top-width of the level by (log_joint desc, candidate index asc) re-sorted by
// index (drafting.cpp:164-176), and its tokens feed the next level's row gather — no host round
// trip per level. k_tree_select then keeps the top total_draft_tokens candidates (select_top_k,
// drafting.cpp:93-118, prefix_closed = false) and compacts them in candidate order (230-244).
//
// log_joint uses the device double log(), not glibc's: every ordering decision is certified
// against a rigorous bound on |log_dev - log_glibc| accumulated along the path (both are within
// ~1 ulp of the exact logarithm; each add rounds within 0.5 ulp), and any decision inside the
// bound — unless the two candidates' inputs are identical (same parent, same probability bits),
// so both sides tie exactly — sets the uncertain flag; the host then rebuilds the tree with its
// own std::log (frs_host.cu). The host also recomputes the emitted nodes' log_joint with
// std::log, so the values it returns are the reference's.
#include "frs_common.cuh"

namespace frs {
namespace {

constexpr int kTreeThreads = 1024;

struct TreeState {          // device-resident between the launches of one tree
    int ncand;              // candidates so far
    int nbeam;              // rows of the beam forwarded at the next level
    int flags;              // bit 0: an ordering decision fell inside the error bound
    int level;              // levels done
    int nsel;               // running select_top_k set (sel[], best first)
    int sel[64];
};

__device__ __forceinline__ double lj_err(double lj, int depth) {
    return static_cast<double>(depth) * (fabs(lj) + 1.0) * 0x1p-48;
}

// a before b in (log_joint desc, index asc)
__device__ __forceinline__ bool before(double la, int a, double lb, int b) { return la > lb || (la == lb && a < b); }

// Same inputs on both sides (same parent, same probability): the two log_joints tie exactly
// in the reference too, and the index decides there as well.
__device__ __forceinline__ bool same_inputs(const int32_t *parent, const float *prob, int a, int b) {
    return parent[a] == parent[b] && __float_as_uint(prob[a]) == __float_as_uint(prob[b]);
}

// Inclusive block scan of v (kTreeThreads threads); s: kTreeThreads ints of scratch.
__device__ __forceinline__ int block_scan_incl(int v, int *s) {
    const int tid = threadIdx.x;
    s[tid] = v;
    __syncthreads();
    for (int off = 1; off < kTreeThreads; off <<= 1) {
        int x = s[tid];
        if (tid >= off) x += s[tid - off];
        __syncthreads();
        s[tid] = x;
        __syncthreads();
    }
    return s[tid];
}

// Certify a cut between sorted positions [0, cut) (kept) and [cut, n) (dropped): ord[] holds
// candidate ids in (log_joint desc, index asc) order of the device values. Any kept/dropped
// pair whose device log_joints are within the summed error bounds — unless their inputs are
// identical — could be ordered differently by the reference. Only the window around the cut
// can hold such pairs (one thread; typically one comparison).
__device__ void certify_cut(const int *ord, const double *lj_of, int n, int cut, int maxdepth, const int32_t *c_par,
                            const float *c_prob, const int32_t *c_dep, const double *c_lj, int *flags) {
    if (cut <= 0 || cut >= n) return;
    const double l_last = lj_of[cut - 1], l_first = lj_of[cut];
    // every bound in the window is below this one (depth <= maxdepth, |lj| within 1 of the cut's)
    const double win = 2.0 * lj_err(fmax(fabs(l_last), fabs(l_first)) + 1.0, maxdepth);
    for (int i = cut - 1; i >= 0 && l_last - lj_of[i] >= -win && lj_of[i] - l_first <= win; --i) {
        for (int j = cut; j < n && l_last - lj_of[j] <= win; ++j) {
            const int a = ord[i], bb = ord[j];
            if (fabs(c_lj[a] - c_lj[bb]) <= lj_err(c_lj[a], c_dep[a]) + lj_err(c_lj[bb], c_dep[bb]) &&
                !same_inputs(c_par, c_prob, a, bb)) {
                atomicOr(flags, 1);
                return;
            }
        }
    }
}

__global__ void __launch_bounds__(kTreeThreads)
    k_tree_level(const int32_t *__restrict__ pk, int nb, int w, int width, int prune, int total,
                 int32_t *__restrict__ c_tok,
                 int32_t *__restrict__ c_ridx, int32_t *__restrict__ c_par, int32_t *__restrict__ c_dep,
                 float *__restrict__ c_prob, double *__restrict__ c_lj, int32_t *__restrict__ beam,
                 int32_t *__restrict__ next_tok, TreeState *st) {
    __shared__ double s_lj[kTreeThreads], s_ljo[kTreeThreads];
    __shared__ int s_scan[kTreeThreads], s_ord[kTreeThreads];
    const int tid = threadIdx.x;
    const int cells = nb * w;  // <= 960 (host): cells + the running set fit the shared arrays
    const int c0 = st->ncand;
    const int maxdepth = st->level + 1;  // this level's children; every earlier candidate is shallower
    const int32_t *ridx = pk, *full = pk + cells;
    const float *prob = reinterpret_cast<const float *>(pk + 2 * cells);
    // 1. the children (drafting.cpp:146-158 at the root, 199-220 below it)
    if (tid < cells) {
        const int i = tid / w, c = c0 + tid;
        const int par = c0 == 0 ? -1 : beam[i];
        const double lg = log(static_cast<double>(prob[tid]));
        const double l = par < 0 ? lg : c_lj[par] + lg;
        c_tok[c] = full[tid];
        c_ridx[c] = ridx[tid];
        c_par[c] = par;
        c_dep[c] = par < 0 ? 1 : c_dep[par] + 1;
        c_prob[c] = prob[tid];
        c_lj[c] = l;
        s_lj[tid] = l;
    }
    __syncthreads();  // every beam[] read and child written
    // 2. the next beam: top-width of this level's children, in index order
    const bool cut = prune && cells > width;
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int NW = kTreeThreads / 32;
    __shared__ int s_rank[kTreeThreads];
    if (cut) {  // warp-cooperative ranks: the lanes split the comparisons, one REDUX per child
        for (int e = warp; e < cells; e += NW) {
            const double l = s_lj[e];
            int cnt = 0;
            for (int o = lane; o < cells; o += 32) cnt += before(s_lj[o], o, l, e) ? 1 : 0;
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (lane == 0) {
                s_rank[e] = cnt;
                s_ord[cnt] = c0 + e;
                s_ljo[cnt] = l;
            }
        }
    }
    __syncthreads();
    const int keep = tid < cells ? (cut ? s_rank[tid] < width : 1) : 0;
    if (cut && tid == 0) certify_cut(s_ord, s_ljo, cells, width, maxdepth, c_par, c_prob, c_dep, c_lj, &st->flags);
    const int incl = block_scan_incl(keep, s_scan);
    if (tid < cells && keep) {
        beam[incl - 1] = c0 + tid;
        if (prune) next_tok[incl - 1] = c_tok[c0 + tid];  // <= width <= 64 rows
    }
    __syncthreads();
    // 3. the running select_top_k set: the best `total` of (previous set + this level). A
    //    candidate dropped here never returns (later levels only add competitors), so the
    //    final set is the global top `total` (see k_tree_select).
    const int nbeam = s_scan[kTreeThreads - 1];
    const int ns0 = st->nsel, m = ns0 + cells;  // <= 64 + 960 (host)
    __syncthreads();  // the beam phase's shared arrays are free again
    double *s_mlj = s_lj, *s_mljo = s_ljo;
    int *s_mid = s_scan, *s_mord = s_ord;
    for (int e = tid; e < m; e += kTreeThreads) {
        const int id = e < ns0 ? st->sel[e] : c0 + (e - ns0);
        s_mid[e] = id;
        s_mlj[e] = c_lj[id];
    }
    __syncthreads();
    for (int e = warp; e < m; e += NW) {
        const double l = s_mlj[e];
        const int id = s_mid[e];
        int cnt = 0;
        for (int o = lane; o < m; o += 32) cnt += before(s_mlj[o], s_mid[o], l, id) ? 1 : 0;
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) {
            s_mord[cnt] = id;
            s_mljo[cnt] = l;
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (m > total) certify_cut(s_mord, s_mljo, m, total, maxdepth, c_par, c_prob, c_dep, c_lj, &st->flags);
        st->ncand = c0 + cells;
        st->level = maxdepth;
        st->nbeam = nbeam;
        st->nsel = min(m, total);
    }
    if (tid < min(m, total)) st->sel[tid] = s_mord[tid];
}

// select_top_k (prefix_closed = false): a child's log_joint never exceeds its parent's (log p <=
// 0, monotone rounding; ties fall to the smaller index, the parent's), so the greedy ancestor-
// checked scan keeps exactly the first `total` candidates of the (log_joint desc, index asc)
// order — the running set k_tree_level maintains. Compaction in candidate order with parents
// remapped (drafting.cpp:230-244).
__global__ void __launch_bounds__(kTreeThreads)
    k_tree_select(TreeState *st, const int32_t *__restrict__ c_tok, const int32_t *__restrict__ c_par,
                  const int32_t *__restrict__ c_dep, const float *__restrict__ c_prob, int32_t *__restrict__ out) {
    // out: [0] count | [1] flags | tokens[64] | parents[64] | depths[64] | probs[64] (float bits)
    constexpr int kMax = 2 * kTreeThreads;
    __shared__ int s_idx[kMax], s_scan[kTreeThreads];
    const int tid = threadIdx.x, n = st->ncand, ns = st->nsel;  // n <= kMax (host)
    for (int c = tid; c < n; c += kTreeThreads) s_idx[c] = 0;
    __syncthreads();
    if (tid < ns) s_idx[st->sel[tid]] = 1;
    __syncthreads();
    int sel[2] = {0, 0};
    if (2 * tid < n) sel[0] = s_idx[2 * tid];
    if (2 * tid + 1 < n) sel[1] = s_idx[2 * tid + 1];
    const int incl = block_scan_incl(sel[0] + sel[1], s_scan);  // candidates 2 tid, 2 tid + 1 in order
    const int ex = incl - sel[0] - sel[1];
    __syncthreads();
    if (2 * tid < n) s_idx[2 * tid] = sel[0] ? ex : -1;
    if (2 * tid + 1 < n) s_idx[2 * tid + 1] = sel[1] ? ex + sel[0] : -1;
    __syncthreads();
    int32_t *tok = out + 2, *par = tok + 64, *dep = par + 64, *pr = dep + 64;
    for (int c = tid; c < n; c += kTreeThreads) {
        const int j = s_idx[c];
        if (j < 0) continue;
        tok[j] = c_tok[c];
        par[j] = c_par[c] >= 0 ? s_idx[c_par[c]] : -1;
        dep[j] = c_dep[c];
        pr[j] = __float_as_int(c_prob[c]);
    }
    if (tid == 0) {
        out[0] = ns;
        out[1] = st->flags;
    }
}

}  // namespace

// Host entry points (frs_host.cu): workspace layout in `ws` (DevBuf of the head).
size_t tree_ws_bytes(int max_cand) { return 512 + (size_t)max_cand * (5 * 4 + 8) + 2048 * 4 + (2 + 4 * 64) * 4 + 256; }

struct TreeWs {
    TreeState *st;
    int32_t *c_tok, *c_ridx, *c_par, *c_dep, *beam, *next_tok, *out;
    float *c_prob;
    double *c_lj;
};

static TreeWs carve(void *base, int max_cand) {
    uint8_t *p = static_cast<uint8_t *>(base);
    TreeWs w;
    w.st = reinterpret_cast<TreeState *>(p);
    p += 512;
    w.c_lj = reinterpret_cast<double *>(p);
    p += (size_t)max_cand * 8;
    w.c_tok = reinterpret_cast<int32_t *>(p);
    p += (size_t)max_cand * 4;
    w.c_ridx = reinterpret_cast<int32_t *>(p);
    p += (size_t)max_cand * 4;
    w.c_par = reinterpret_cast<int32_t *>(p);
    p += (size_t)max_cand * 4;
    w.c_dep = reinterpret_cast<int32_t *>(p);
    p += (size_t)max_cand * 4;
    w.c_prob = reinterpret_cast<float *>(p);
    p += (size_t)max_cand * 4;
    w.beam = reinterpret_cast<int32_t *>(p);
    p += 2048 * 4;
    w.out = reinterpret_cast<int32_t *>(p);
    w.next_tok = nullptr;
    return w;
}

int tree_begin(void *ws, int max_cand, cudaStream_t s) {
    TreeWs w = carve(ws, max_cand);
    FRS_CUDA_TRY(cudaMemsetAsync(w.st, 0, sizeof(TreeState), s));
    return FRS_OK;
}

int tree_level(void *ws, int max_cand, const int32_t *pk, int nb, int w_children, int width, bool prune, int total,
               int32_t *next_tok, cudaStream_t s) {
    TreeWs w = carve(ws, max_cand);
    k_tree_level<<<1, kTreeThreads, 0, s>>>(pk, nb, w_children, width, prune ? 1 : 0, total, w.c_tok, w.c_ridx,
                                            w.c_par, w.c_dep, w.c_prob, w.c_lj, w.beam, next_tok, w.st);
    FRS_CUDA_TRY(cudaGetLastError());
    return FRS_OK;
}

int tree_select(void *ws, int max_cand, int total, int32_t **out_dev, cudaStream_t s) {
    TreeWs w = carve(ws, max_cand);
    (void)total;
    k_tree_select<<<1, kTreeThreads, 0, s>>>(w.st, w.c_tok, w.c_par, w.c_dep, w.c_prob, w.out);
    FRS_CUDA_TRY(cudaGetLastError());
    *out_dev = w.out;
    return FRS_OK;
}

}  // namespace frs
