// FAST mode: tcgen05 tensor-core LM head over a bf16 slab, fused with the online-softmax
// statistics and per-CTA top-R candidate tracking, then an exact-recompute finalize that
// certifies the top-k ids against the reference arithmetic.
//
// Per call (one draft level, or one verify head), four kernels on one stream, chained with
// programmatic dependent launch (PDL) so each kernel's prologue overlaps its predecessor's tail:
//
//  k_hsplit         the hi / lo bf16 split of the hidden rows (tiny).
//  k_fast_main      persistent, one CTA per SM; each CTA owns a contiguous run of 32-row slab
//                   chunks (tiles of up to 128 rows), so no CTA streams more than one chunk
//                   beyond the average. Its B operand is hs[2NP x d] bf16 written by k_hsplit
//                   (rows [0,NP) = hi = bf16(h), rows [NP,2NP) = lo = bf16(h - hi):
//                   h = hi + lo + O(2^-16 |h|)); the first ring pass of slab tiles is issued
//                   before waiting for that grid.
//                   Warp 0 streams (slab k-block, hs k-block) stages with TMA (SWIZZLE_128B,
//                   32-row boxes) into a multi-stage mbarrier ring; warp 1 issues tcgen05.mma
//                   (M=128 slab rows, N=2NP, K=16, bf16 -> fp32 in TMEM, double-buffered
//                   accumulator); warps 2-3 accumulate each slab row's squared L2 norm from the
//                   same stages (for the error bound, always fresh); warps 4-11 drain TMEM
//                   (tcgen05.ld 32x32b), form logit = hi + lo per (slab row, hidden row), update
//                   the online (max, sum-exp) statistics and per-thread top-2 keys. Logits never
//                   leave the SM. Each CTA publishes (m, s), its top-R candidate keys per hidden
//                   row, the bound for all its other rows and max |W_j|^2.
//  k_fast_finalize  grid (n, 8) in clusters of 8 (one cluster per hidden row): merge the CTA
//                   partials, find the kk-th largest candidate key (two-level tournament), take
//                   S = {keys >= v_kk - 2 eps - margin}, recompute S EXACTLY (dot_f32 order;
//                   results gathered in the cluster leader through DSMEM), select the top-k by
//                   (prob desc, index asc) with the glibc expf port, and certify that no other
//                   row can enter: every row outside S has exact logit <= bound + eps, eps a
//                   rigorous error bound (reference dot_f32 error + tensor-core accumulation +
//                   hi/lo truncation, Cauchy-Schwarz with |h|_2 |W_j|_2). Rows that cannot be
//                   certified (near-ties within 4 ulps, bound too loose, S overflow) are queued.
//  k_fast_fallback  grid-wide exact recompute of the queued rows (bit-identical to the EXACT
//                   path); exits at once when the queue is empty (the common case).
//
// Memory bound: the slab is read exactly once per call (268,435,456 B for V_sub=32768,
// d=4096); hs (<= 1 MB), partials and candidate rows are L2 traffic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "frs_common.cuh"
#include "frs_device.cuh"

// Diagnostics (globaltimer / clock64 probes, FRS_ABLATE phase skipping) are compiled in only
// with -DFRS_DIAG=1 (FRS_DIAG=1 python -m paper_2502_14856_b200.build -> libfrspec_cuda_diag.so,
// loaded through FRS_LIB_PATH by tools/fast_trace.py, tools/ablate.sh, tools/sm_balance_probe.py);
// release kernels carry no branches for them.
#ifndef FRS_DIAG
#define FRS_DIAG 0
#endif

namespace frs {
namespace {

constexpr bool kDiag = FRS_DIAG != 0;
constexpr int BM = 128;      // slab rows per tile (UMMA M)
constexpr int CH = 32;       // slab rows per TMA box = partition granule: CTAs own contiguous
                             // runs of 32-row chunks (<= 1 chunk of imbalance instead of 1 tile)
constexpr int CPT = BM / CH; // chunks per tile
constexpr int kTrMain = 32;  // globaltimer trace slots per main-kernel CTA (FRS_TRACE diagnostics)
constexpr int BK = 64;       // k elements per stage: 128-byte bf16 rows, SWIZZLE_128B
constexpr int R = 3;         // candidate keys per list (per epilogue warp and hidden row)
constexpr int kListsPerCta = 4;  // one list per TMEM lane quarter (32 slab rows of every tile)
constexpr int kFinThreads = 256;
constexpr int kFbThreads = 256;
constexpr int kFinStage = 8;       // max candidates staged per finalize round (runtime A.fin_stage:
                                   // 8 for drafts (150 KB smem), 4 for verify (83 KB, 2 CTAs/SM))

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_load_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                               uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {  // bytes % 16 == 0
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t *slot, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate (kind::f16).
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B canonical layout: 8-row x 128-byte
// atoms, SBO = 1024 B between atoms, LBO unused (1), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}
// kind::f16 instruction descriptor: fp32 D, bf16 A/B, both K-major, N and M.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// ------------------------------------------------------------------ kernels
// Per hidden row, one "list" per (CTA, TMEM lane quarter): L = 4 G lists.
struct Partials {
    float *pm;                 // [NP][L] max of x = logit / t over the list's slab rows (softmax only)
    float *ps;                 // [NP][L] sum exp(x - pm)
    float *pth;                // [NP][L] bound: every list row not in pkey has approx logit <= pth
    unsigned long long *pkey;  // [NP][L][R] the list's best R (approx value, index) keys, descending
    float *pw2;                // [2G] max squared L2 norm of slab rows (per CTA and norm warp)
    unsigned *rowmax_bits;     // [64] per hidden row: max approximate logit, order-preserving bits
    unsigned *w2_bits;         // [1] max |W_j|^2 (float bits); both reset by k_hsplit, atomicMax here
    float *logits;             // LOGITS mode: approximate logits [n][ld_logits] (batched drafting)
    int late_trigger;          // DIAGNOSTIC (FRS_ABLATE=8): launch_dependents at the end, not the start
    int ablate_main;           // DIAGNOSTIC (FRS_ABLATE=14/15): skip the publish / the epilogue math
    int range_shift;           // DIAGNOSTIC (FRS_RANGE_SHIFT): CTA c streams the row range of CTA c + shift
    int ld_logits;
    int G;
    unsigned long long *trace; // optional [G][16] globaltimer stamps (diagnostics; nullptr = off)
    unsigned *main_done;       // [1] main CTAs whose outputs are published (release; reset by k_hsplit)
    const uint8_t *tiled;      // the slab in stage order ([kb][32-row chunk] blocks of 4 KB, each the
                               // SWIZZLE_128B image of 32 rows x 128 B), or nullptr (2-D tensor loads)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FRS_TRACE(P, slot)                                                       \
    do {                                                                         \
        if (kDiag && (P).trace) (P).trace[(size_t)blockIdx.x * kTrMain + (slot)] = gtimer();   \
    } while (0)

// hs rows [0,NP) = bf16(h), rows [NP,2NP) = bf16(h - bf16(h)); padded rows are zero. Hidden
// rows are interleaved over the two column halves (hs row p = hidden row 2 (p % (NP/2)) +
// p / (NP/2)), so the two epilogue warps of a TMEM lane quarter share the valid rows evenly.
// 128 threads, no shared memory: it co-resides with the main kernel's CTAs, which PDL lets
// launch (and run their prologue and first slab loads) while this grid is still running.
// h_copy != nullptr: h is a mapped pinned HOST pointer (the host-buffer entry point reads the
// rows over the bus here instead of a separate copy) and the fp32 rows are also written to
// h_copy, the device copy the finalize's exact dots read.
__global__ void __launch_bounds__(128) k_hsplit(const float *__restrict__ h, int n, int d, int NP,
                                                __nv_bfloat16 *__restrict__ hs, unsigned *__restrict__ rowmax_bits,
                                                unsigned *__restrict__ w2_bits, unsigned long long *xtrace,
                                                float *__restrict__ h_copy, unsigned *__restrict__ main_done) {
    // launched programmatically after whatever precedes it on the stream: let the main kernel
    // launch at once (its CTAs take the SMs the previous grid leaves and issue their ring fill
    // of slab stages, which needs nothing from this call), then wait for the predecessor (h is
    // final, the previous call's fallback queue is drained) before writing anything
    griddep_launch();  // the main kernel may launch now: it waits for this grid before reading hs
    griddep_wait();
    if (blockIdx.x == 0) {  // this call's atomicMax targets (the previous call is complete)
        if (threadIdx.x < 64) rowmax_bits[threadIdx.x] = 0u;  // below every ordered value
        if (threadIdx.x == 0) {
            *w2_bits = 0u;
            *main_done = 0u;
        }
    }
    if (xtrace && blockIdx.x == 0 && threadIdx.x == 0) xtrace[0] = gtimer();
    const int total4 = NP * d / 4;  // d % 8 == 0 on the FAST path
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total4; idx += gridDim.x * blockDim.x) {
        const int e = idx * 4, p = e / d, c = e - p * d;
        const int i = 2 * (p % (NP / 2)) + p / (NP / 2);  // hs row p holds hidden row i (see k_fast_main)
        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n) {
            if (h_copy) {
                x = *reinterpret_cast<const float4 *>(h + (size_t)i * d + c);
                *reinterpret_cast<float4 *>(h_copy + (size_t)i * d + c) = x;
            } else {
                x = __ldg(reinterpret_cast<const float4 *>(h + (size_t)i * d + c));
            }
        }
        const __nv_bfloat162 h01 = __floats2bfloat162_rn(x.x, x.y), h23 = __floats2bfloat162_rn(x.z, x.w);
        const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
        const __nv_bfloat162 l01 = __floats2bfloat162_rn(x.x - f01.x, x.y - f01.y);
        const __nv_bfloat162 l23 = __floats2bfloat162_rn(x.z - f23.x, x.w - f23.y);
        __nv_bfloat162 *hi = reinterpret_cast<__nv_bfloat162 *>(hs + (size_t)p * d + c);
        __nv_bfloat162 *lo = reinterpret_cast<__nv_bfloat162 *>(hs + (size_t)(NP + p) * d + c);
        hi[0] = h01;
        hi[1] = h23;
        lo[0] = l01;
        lo[1] = l23;
    }
    if (xtrace && blockIdx.x == 0 && threadIdx.x == 0) xtrace[1] = gtimer();
}

// The slab in the main kernel's stage order: block (kb, chunk c) = rows [32 c, 32 c + 32) x
// columns [64 kb, 64 kb + 64) as the SWIZZLE_128B shared-memory image (16-byte group q of row r
// at r 128 + (q ^ (r & 7)) 16), blocks ordered [kb][c] so a tile's chunks of one K block are one
// contiguous bulk copy. Rows past v_rows and columns past d are zero (the TMA's OOB fill).
__global__ void k_slab_tile(const uint16_t *__restrict__ slab, int v_rows, int d, int NCH, uint8_t *__restrict__ out) {
    const int KB = (d + BK - 1) / BK;
    const size_t total = (size_t)KB * NCH * CH * 8;  // 16-byte groups
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int q = static_cast<int>(e & 7), r = static_cast<int>((e >> 3) & (CH - 1));
        const size_t blk = e >> 8;  // (kb NCH + c)
        const int c = static_cast<int>(blk % NCH), kb = static_cast<int>(blk / NCH);
        const int row = c * CH + r, col = kb * BK + q * 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (row < v_rows && col < d) v = *reinterpret_cast<const uint4 *>(slab + (size_t)row * d + col);
        *reinterpret_cast<uint4 *>(out + blk * (CH * BK * 2) + r * 128 + ((q ^ (r & 7)) << 4)) = v;
    }
}

template <int NP, bool SOFTMAX>
struct MainCfg {
    static constexpr int N = 2 * NP;                       // MMA N: hi rows then lo rows
    static constexpr int EPI_WARPS = 8;                    // 4 TMEM lane quarters x 2 column halves
    static constexpr int RPW = NP / (EPI_WARPS / 4);       // hidden rows per epilogue warp
    static constexpr int TOPK = SOFTMAX ? 2 : 1;           // per-thread kept candidates per hidden row
    static constexpr int THREADS = (4 + EPI_WARPS) * 32;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = N * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 12 ? 12 : (200 * 1024) / STAGE_BYTES;
    static constexpr int TMEM_COLS = (2 * N) < 32 ? 32 : 2 * N;
    static_assert(!SOFTMAX || NP == 16, "the fused softmax path handles up to 16 hidden rows per call");
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 4 * NP * 8 + 256;
    // publish scratch per epilogue warp, carved from the A stages once the MMAs are done
    static constexpr int SCRATCH_PER_WARP = (STAGES * A_BYTES) / EPI_WARPS;
    static constexpr int PUB_KSTRIDE = 8 * TOPK + 1, PUB_FSTRIDE = 8 + 1;  // 8 rows per pass, odd strides
    static_assert(32 * PUB_KSTRIDE * 8 + 32 * PUB_FSTRIDE * 4 * (SOFTMAX ? 3 : 1) <= SCRATCH_PER_WARP,
                  "publish scratch");
};

#define FRS_TMEM_LD16(taddr, r)                                                                                 \
    asm volatile(                                                                                               \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
        : "r"(taddr))

#define FRS_TMEM_LD8(taddr, r)                                                                          \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                    \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) \
                 : "r"(taddr))

// Warp max of a (value, index) key with 2 REDUX instead of 10 shuffles: max over the ordered
// value bits, then max over ~index among the lanes holding that value.
// a := top 4 of (a, b), both sorted descending: bitonic half-cleaner, then sort the bitonic 4
__device__ __forceinline__ void top4_merge(unsigned long long (&a)[4], const unsigned long long (&b)[4]) {
    unsigned long long c0 = a[0] > b[3] ? a[0] : b[3], c1 = a[1] > b[2] ? a[1] : b[2];
    unsigned long long c2 = a[2] > b[1] ? a[2] : b[1], c3 = a[3] > b[0] ? a[3] : b[0];
    auto ce = [](unsigned long long &x, unsigned long long &y) {
        const bool sw = y > x;
        const unsigned long long t = sw ? y : x;
        y = sw ? x : y;
        x = t;
    };
    ce(c0, c2);
    ce(c1, c3);
    ce(c0, c1);
    ce(c2, c3);
    a[0] = c0, a[1] = c1, a[2] = c2, a[3] = c3;
}

__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    const unsigned hi = static_cast<unsigned>(k >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? static_cast<unsigned>(k) : 0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

// LOGITS: the epilogue writes the approximate logits of every (hidden row, slab row) to
// P.logits instead of tracking lists (batched drafting with many hidden rows, k_fast_select).
template <int NP, bool SOFTMAX, bool LOGITS = false>
__global__ void __launch_bounds__(MainCfg<NP, SOFTMAX>::THREADS, 1)
    k_fast_main(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapW32,
                const __grid_constant__ CUtensorMap mapH, int n,
                int v_rows, int d, float inv_t, Partials P) {
    using C = MainCfg<NP, SOFTMAX>;
    constexpr int N = C::N, STAGES = C::STAGES, RPW = C::RPW, TOPK = C::TOPK, EPI = C::EPI_WARPS;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (SWIZZLE_128B) by arithmetic on smem_raw itself: the pointer stays in the
    // shared window, so the epilogue's publish scratch is read and written with LDS/STS, not
    // generic accesses (65.9 vs 66.9 us per C2 level)
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = smem;                                   // STAGES x 16 KB
    uint8_t *sB = smem + STAGES * C::A_BYTES;             // STAGES x B_BYTES
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * C::STAGE_BYTES);
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);

    // warp index broadcast from lane 0: provably warp-uniform, so the role branches below
    // keep their shuffles convergent (no WARPSYNC.COLLECTIVE emulation)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int G = gridDim.x, cta = blockIdx.x;
    const int KB = (d + BK - 1) / BK;
    // balanced partition: this CTA owns 32-row chunks [c_begin, c_end); tile t covers chunks
    // c_begin + CPT t .. (at most CPT), so the A tile of a short tile is partly stale (ignored)
    const int NCH = (v_rows + CH - 1) / CH;
    const int pcta = kDiag ? (cta + P.range_shift) % G : cta;  // DIAGNOSTIC: rotate the ranges over the CTAs
    const int c_begin = static_cast<int>((static_cast<long long>(pcta) * NCH) / G);
    const int c_end = static_cast<int>((static_cast<long long>(pcta + 1) * NCH) / G);
    const int t_begin = 0, t_end = (c_end - c_begin + CPT - 1) / CPT;
    auto tile_chunks = [&](int t) { return min(CPT, c_end - (c_begin + t * CPT)); };
    auto tile_row0 = [&](int t) { return (c_begin + t * CPT) * CH; };
    auto tile_rows = [&](int t) { return min(v_rows - tile_row0(t), tile_chunks(t) * CH); };

    // per-CTA maxima, combined in shared memory: ONE global atomic per (CTA, row) and per CTA
    // for |W|^2 (hundreds of same-address atomics per row at the tail cost ~3 us per call)
    __shared__ unsigned s_rmax[64], s_w2max;
    if (threadIdx.x < 64) s_rmax[threadIdx.x] = 0u;
    if (threadIdx.x == 64) s_w2max = 0u;
    if (threadIdx.x == 0) {
        FRS_TRACE(P, 28);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 2);  // MMA commit + the two norm warps
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * (EPI / 4));  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&mapW);
        prefetch_tmap(&mapW32);
        prefetch_tmap(&mapH);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) FRS_TRACE(P, 0);
    // let the finalize grid launch now: its CTAs take SMs as ours retire and run their
    // prologue; griddepcontrol.wait there still waits for this whole grid (and its writes)
    if (!(kDiag && P.late_trigger)) griddep_launch();

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            // Straight-line issue loop: the producer thread's issue rate is on the critical
            // path (a lambda-based version of this loop streamed 15 % slower). A full tile is
            // one 128-row box; a short tile (the CTA's last) is loaded as 32-row boxes.
            const uint64_t pol_w = policy_evict_first(), pol_h = policy_evict_last();
            // Ring fill before the dependency wait: the slab halves of the first STAGES stages
            // (the slab needs nothing from the previous grid); their hs halves after it.
            const int pre = min(STAGES, (t_end - t_begin) * KB);
            for (int g = 0; g < pre; ++g) {
                const int t = t_begin + g / KB, kb = g % KB, nch = tile_chunks(t), r0 = tile_row0(t);
                mbar_expect_tx(&full[g], nch * (CH * BK * 2) + C::B_BYTES);
                if (P.tiled) {  // the tile's nch chunk blocks of this K block are contiguous
                    bulk_load_hint(sA + g * C::A_BYTES, P.tiled + ((size_t)kb * NCH + r0 / CH) * (CH * BK * 2),
                                   nch * (CH * BK * 2), &full[g], pol_w);
                } else if (nch == CPT) {
                    tma_load_2d(sA + g * C::A_BYTES, &mapW, &full[g], kb * BK, r0, pol_w);
                } else {
                    for (int c = 0; c < nch; ++c)
                        tma_load_2d(sA + g * C::A_BYTES + c * (CH * BK * 2), &mapW32, &full[g], kb * BK, r0 + c * CH,
                                    pol_w);
                }
            }
            FRS_TRACE(P, 1);
            griddep_wait();  // hs is written by k_hsplit (programmatic dependency)
            FRS_TRACE(P, 9);
            for (int g = 0; g < pre; ++g)
                tma_load_2d(sB + g * C::B_BYTES, &mapH, &full[g], (g % KB) * BK, 0, pol_h);
            int stage = pre % STAGES;
            uint32_t phase = pre == STAGES ? 1u : 0u;
            for (int t = t_begin + pre / KB, kb0 = pre % KB; t < t_end; ++t, kb0 = 0) {
                const int nch = tile_chunks(t), r0 = tile_row0(t);
                for (int kb = kb0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], nch * (CH * BK * 2) + C::B_BYTES);
                    if (P.tiled) {
                        bulk_load_hint(sA + stage * C::A_BYTES, P.tiled + ((size_t)kb * NCH + r0 / CH) * (CH * BK * 2),
                                       nch * (CH * BK * 2), &full[stage], pol_w);
                    } else if (nch == CPT) {
                        tma_load_2d(sA + stage * C::A_BYTES, &mapW, &full[stage], kb * BK, r0, pol_w);
                    } else {
                        for (int c = 0; c < nch; ++c)
                            tma_load_2d(sA + stage * C::A_BYTES + c * (CH * BK * 2), &mapW32, &full[stage], kb * BK,
                                        r0 + c * CH, pol_w);
                    }
                    tma_load_2d(sB + stage * C::B_BYTES, &mapH, &full[stage], kb * BK, 0, pol_h);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            FRS_TRACE(P, 2);
        }
        __syncwarp();  // reconverge before the CTA-wide (aligned) barriers below
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(BM, N);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin, lt = 0; t < t_end; ++t, ++lt) {
                const int acc = lt & 1;
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * N);
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    if (lt == 0 && kb == 0) FRS_TRACE(P, 3);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)  // +32 bytes per K=16 step inside the swizzle atom
                        umma_bf16(d_tmem, adesc + 2ull * kk, bdesc + 2ull * kk, idesc, (kb | kk) != 0);
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
            }
            FRS_TRACE(P, 4);
        }
        __syncwarp();
    } else if (warp < 4) {  // ---------------- row-norm warps: max_j |W_j|^2 for the error bound
        const int r0 = threadIdx.x - 64;  // 0..63: rows r0 and r0 + 64 of every tile
        float acc0 = 0.0f, acc1 = 0.0f, wmax = 0.0f;
        int stage = 0;
        uint32_t phase = 0;
        for (int t = t_begin; t < t_end; ++t) {
            const int nrows = tile_rows(t);  // rows past it are stale smem: keep them out of the max
            for (int kb = 0; kb < KB; ++kb) {
                mbar_wait(&full[stage], phase);
                const uint4 *a0 = reinterpret_cast<const uint4 *>(sA + stage * C::A_BYTES + r0 * 128);
                const uint4 *a1 = reinterpret_cast<const uint4 *>(sA + stage * C::A_BYTES + (r0 + 64) * 128);
#pragma unroll
                for (int c = 0; c < 8; ++c) {   // order within a row is irrelevant for a sum of squares;
                    const int pc = c ^ (r0 & 7);  // rotate chunks by row so 8 lanes cover all 32 banks
                    const uint4 u = a0[pc], w = a1[pc];
                    const uint32_t uu[4] = {u.x, u.y, u.z, u.w}, ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float x0 = __uint_as_float(uu[e] << 16), x1 = __uint_as_float(uu[e] & 0xffff0000u);
                        const float y0 = __uint_as_float(ww[e] << 16), y1 = __uint_as_float(ww[e] & 0xffff0000u);
                        acc0 = fmaf(x0, x0, fmaf(x1, x1, acc0));
                        acc1 = fmaf(y0, y0, fmaf(y1, y1, acc1));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (r0 < nrows) wmax = fmaxf(wmax, acc0);
            if (r0 + 64 < nrows) wmax = fmaxf(wmax, acc1);
            acc0 = acc1 = 0.0f;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        if (lane == 0) {
            P.pw2[cta * 2 + (warp - 2)] = wmax;
            atomicMax(&s_w2max, __float_as_uint(wmax));  // non-negative: raw bits order
        }
        if (threadIdx.x == 64) FRS_TRACE(P, 8);
        if constexpr (!LOGITS) asm volatile("bar.arrive 1, %0;" ::"r"((2 + EPI) * 32) : "memory");  // sA reads done
    } else {  // ---------------- epilogue warps: TMEM -> (softmax stats, per-thread candidates)
        const int we = warp - 4;         // 0 .. EPI-1
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int half = we >> 2;          // column half: TMEM columns [half RPW, (half + 1) RPW)
        const int cbase = half * RPW;      // = hidden rows 2 r + half, r < RPW (k_hsplit's order)
        const int nv = max(0, min(RPW, (n - half + 1) >> 1));  // valid hidden rows of this warp
        constexpr int NS = SOFTMAX ? RPW : 1;
        const float kNegInf = __int_as_float(0xff800000u);
        float m[NS], s[NS];
        unsigned long long b1[RPW], b2[TOPK == 2 ? RPW : 1];
        float bnd[RPW];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            if constexpr (SOFTMAX) {
                m[r] = kNegInf;
                s[r] = 0.0f;
            }
            b1[r] = 0ull;
            if constexpr (TOPK == 2) b2[r] = 0ull;
            bnd[r] = kNegInf;
        }
        for (int t = t_begin, lt = 0; t < t_end; ++t, ++lt) {
            const int acc = lt & 1;
            if (threadIdx.x == 128 && lt == 0) FRS_TRACE(P, 10);
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            if (threadIdx.x == 128 && lt == 0) FRS_TRACE(P, 11);
            if (threadIdx.x == 128 && t == t_end - 1) FRS_TRACE(P, 14);
            tc_fence_after();
            const int row = tile_row0(t) + q * 32 + lane;
            const bool valid = q * 32 + lane < tile_rows(t);
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * N);
            // hidden rows per TMEM load group (8 for the 32-row argmax warps: 16 spilled registers at NP = 64)
            constexpr int CG = RPW < 16 ? RPW : (TOPK == 1 && RPW > 16 ? 8 : 16);
#pragma unroll
            for (int cg = 0; cg < RPW / CG; ++cg) {
                const int c0 = cbase + cg * CG;
                uint32_t hi[CG], lo[CG];
                if constexpr (CG == 8) {
                    FRS_TMEM_LD8(tbase + c0, hi);
                    FRS_TMEM_LD8(tbase + NP + c0, lo);
                } else {
                    FRS_TMEM_LD16(tbase + c0, hi);
                    FRS_TMEM_LD16(tbase + NP + c0, lo);
                }
                tmem_wait_ld();
                if (cg == RPW / CG - 1) {  // accumulator drained: hand it back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
                if (!LOGITS && (kDiag && P.ablate_main == 15)) continue;
                if constexpr (LOGITS) {  // coalesced: the warp's 32 lanes are 32 consecutive slab rows
#pragma unroll
                    for (int r = 0; r < CG; ++r) {
                        const int i = 2 * (cg * CG + r) + half;
                        if (valid && i < n)
                            P.logits[(size_t)i * P.ld_logits + row] = __uint_as_float(hi[r]) + __uint_as_float(lo[r]);
                    }
                    continue;
                }
#pragma unroll
                for (int r = 0; r < CG; ++r) {
                    const int rr = cg * CG + r, i = 2 * rr + half;
                    if (!valid || i >= n) continue;
                    const float a = __uint_as_float(hi[r]) + __uint_as_float(lo[r]);
                    if constexpr (SOFTMAX) {  // online sum exp(x - m), one MUFU per value
                        const float x = a * inv_t;
                        if (x <= m[rr]) {
                            s[rr] += exp2f((x - m[rr]) * 1.4426950408889634f);
                        } else {
                            s[rr] = s[rr] * exp2f((m[rr] - x) * 1.4426950408889634f) + 1.0f;
                            m[rr] = x;
                        }
                    }
                    // per-thread top-TOPK keys; everything dropped is bounded by bnd
                    const unsigned long long k = dev::value_key(a, row);
                    if constexpr (TOPK == 2) {
                        if (k > b1[rr]) {
                            if (b2[rr]) bnd[rr] = fmaxf(bnd[rr], dev::key_value(b2[rr]));
                            b2[rr] = b1[rr];
                            b1[rr] = k;
                        } else if (k > b2[rr]) {
                            if (b2[rr]) bnd[rr] = fmaxf(bnd[rr], dev::key_value(b2[rr]));
                            b2[rr] = k;
                        } else {
                            bnd[rr] = fmaxf(bnd[rr], a);
                        }
                    } else {
                        if (k > b1[rr]) {
                            if (b1[rr]) bnd[rr] = fmaxf(bnd[rr], dev::key_value(b1[rr]));
                            b1[rr] = k;
                        } else {
                            bnd[rr] = fmaxf(bnd[rr], a);
                        }
                    }
                }
            }
        }
        if (threadIdx.x == 128) FRS_TRACE(P, 13);
        if (lane == 0) FRS_TRACE(P, 20 + we);
        // ---- publish, per hidden row, this warp's list: the softmax partial (m, s) over its
        //      slab rows and their top-R keys + a bound for the rest. Warp-local only: the
        //      max by one REDUX on order-preserving bits, the list by R + 1 tournament rounds
        //      over the lanes' sorted (b1, b2) heads.
        const long long c_pub0 = clock64();
        if constexpr (LOGITS) {
            (void)b1;
            (void)bnd;
        } else if ((kDiag && P.ablate_main >= 14)) {
            asm volatile("bar.sync 1, %0;" ::"r"((2 + EPI) * 32) : "memory");
        } else {
        const int list = cta * kListsPerCta + q, L = G * kListsPerCta;
        // Lanes' states go through shared memory (the A stages: every MMA has completed and
        // the norm warps have signalled barrier 1), then 4 lanes per hidden row merge 8 lanes'
        // entries each and combine over 2 shuffle rounds. (Warp-wide REDUX/shuffle trees per
        // row took ~3 us at the tail of every call.)
        asm volatile("bar.sync 1, %0;" ::"r"((2 + EPI) * 32) : "memory");
        if (kDiag && P.trace && threadIdx.x == 128) P.trace[(size_t)blockIdx.x * kTrMain + 6] = static_cast<unsigned long long>(clock64() - c_pub0);
        constexpr int SLOT = C::SCRATCH_PER_WARP;
        uint8_t *scr = sA + we * SLOT;
        if constexpr (TOPK == 1) {
            // argmax lists (one key per lane and row): ONE pass over every row of the warp —
            // lane r collects row r's 32 lane keys and bounds (rotation-skewed [source lane][row]
            // layout: conflict-free reads) and keeps the top R + 1 by insertion (the 4-lane
            // merges of the pass loop below ran RPW / 8 passes: ~4 us per verify call at NP = 64)
            static_assert(RPW <= 32 && 32 * RPW * 12 <= C::SCRATCH_PER_WARP, "one-pass argmax publish scratch");
            unsigned long long *sk1 = reinterpret_cast<unsigned long long *>(scr);  // [32][RPW]
            float *sb1 = reinterpret_cast<float *>(scr + 32 * RPW * 8);           // [32][RPW]
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const int c = lane * RPW + ((r + lane) & (RPW - 1));
                sk1[c] = b1[r];
                sb1[c] = bnd[r];
            }
            __syncwarp();
            if (lane < nv) {
                const int r = lane, i = 2 * r + half;
                unsigned long long t0 = 0ull, t1 = 0ull, t2 = 0ull, t3 = 0ull;
                float bmx = kNegInf;
#pragma unroll 8
                for (int src = 0; src < 32; ++src) {
                    const int c = src * RPW + ((r + src) & (RPW - 1));
                    const unsigned long long k = sk1[c];
                    bmx = fmaxf(bmx, sb1[c]);
                    // insert k into t0 >= t1 >= t2 >= t3 (keys are distinct or 0)
                    const unsigned long long m0 = k > t0 ? k : t0, r0 = k > t0 ? t0 : k;
                    const unsigned long long m1 = r0 > t1 ? r0 : t1, r1 = r0 > t1 ? t1 : r0;
                    const unsigned long long m2 = r1 > t2 ? r1 : t2, r2 = r1 > t2 ? t2 : r1;
                    t3 = r2 > t3 ? r2 : t3;
                    t0 = m0, t1 = m1, t2 = m2;
                }
                const unsigned long long top[R] = {t0, t1, t2};
#pragma unroll
                for (int z = 0; z < R; ++z) P.pkey[((size_t)i * L + list) * R + z] = top[z];
                P.pth[(size_t)i * L + list] = fmaxf(t3 ? dev::key_value(t3) : kNegInf, bmx);
                if (t0) atomicMax(&s_rmax[i], static_cast<unsigned>(t0 >> 32));
            }
        } else {
        // per pass of 8 rows, lane-major with odd strides: the 8 rows a reader instruction
        // touches sit in distinct banks (row-major [row][lane] made every merge load 8-way
        // bank-conflicted)
        constexpr int KS = C::PUB_KSTRIDE, FS = C::PUB_FSTRIDE;
        unsigned long long *sk = reinterpret_cast<unsigned long long *>(scr);  // [32][KS]: row k's keys at k TOPK
        float *sbn = reinterpret_cast<float *>(scr + 32 * KS * 8);            // [32][FS]
        float *smm = sbn + 32 * FS, *sss = smm + 32 * FS;                     // [32][FS] (SOFTMAX)
        const int g = lane >> 2, u = lane & 3;
        static_assert(R + 1 == 4, "the merge network keeps the top 4 keys");
#pragma unroll
        for (int r0 = 0; r0 < RPW; r0 += 8) {  // warp-uniform passes of 8 rows
            if (r0 >= nv) break;
            if (r0 > 0) __syncwarp();  // the previous pass's reads are done
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (r0 + k >= RPW || r0 + k >= nv) continue;
                sk[lane * KS + k * TOPK] = b1[r0 + k];
                if constexpr (TOPK == 2) sk[lane * KS + k * TOPK + 1] = b2[r0 + k];
                sbn[lane * FS + k] = bnd[r0 + k];
                if constexpr (SOFTMAX) {
                    smm[lane * FS + k] = m[r0 + k];
                    sss[lane * FS + k] = s[r0 + k];
                }
            }
            __syncwarp();
            const int r = r0 + g;
            const bool live = r < nv;
            unsigned long long top[4] = {0ull, 0ull, 0ull, 0ull};
            float bmx = kNegInf, mu = kNegInf, eu = 0.0f;
            if (live) {
                // lanes 8u .. 8u+7: their sorted (b1, b2) pairs -> four sorted 4-lists -> top 4
                // by a bitonic merge tree (short dependent chains, unlike sequential insertion)
                unsigned long long q4[4][4];
#pragma unroll
                for (int pq = 0; pq < 4; ++pq) {
                    const int la = 8 * u + 2 * pq, lb = la + 1;
                    const unsigned long long x0 = sk[la * KS + g * TOPK];
                    const unsigned long long x1 = TOPK == 2 ? sk[la * KS + g * TOPK + (TOPK - 1)] : 0ull;
                    const unsigned long long y0 = sk[lb * KS + g * TOPK];
                    const unsigned long long y1 = TOPK == 2 ? sk[lb * KS + g * TOPK + (TOPK - 1)] : 0ull;
                    const unsigned long long t1 = x0 > y0 ? y0 : x0, t2 = x1 > y1 ? x1 : y1;
                    q4[pq][0] = x0 > y0 ? x0 : y0;
                    q4[pq][1] = t1 > t2 ? t1 : t2;
                    q4[pq][2] = t1 > t2 ? t2 : t1;
                    q4[pq][3] = x1 > y1 ? y1 : x1;
                }
                top4_merge(q4[0], q4[1]);
                top4_merge(q4[2], q4[3]);
                top4_merge(q4[0], q4[2]);
#pragma unroll
                for (int z = 0; z < 4; ++z) top[z] = q4[0][z];
#pragma unroll
                for (int l = 8 * u; l < 8 * u + 8; ++l) {
                    bmx = fmaxf(bmx, sbn[l * FS + g]);
                    if constexpr (SOFTMAX) mu = fmaxf(mu, smm[l * FS + g]);
                }
                if constexpr (SOFTMAX) {
#pragma unroll
                    for (int l = 8 * u; l < 8 * u + 8; ++l) {
                        const float ml = smm[l * FS + g];
                        if (ml != kNegInf) eu += sss[l * FS + g] * exp2f((ml - mu) * 1.4426950408889634f);
                    }
                }
            }
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {  // combine the 4 lanes of the row
                unsigned long long pk[4];
#pragma unroll
                for (int z = 0; z < 4; ++z) pk[z] = __shfl_xor_sync(0xffffffffu, top[z], o);
                top4_merge(top, pk);
                bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, o));
                if constexpr (SOFTMAX) {
                    const float mo = __shfl_xor_sync(0xffffffffu, mu, o), eo = __shfl_xor_sync(0xffffffffu, eu, o);
                    const float mn = fmaxf(mu, mo);
                    const float ea = mu == kNegInf ? 0.0f : eu * exp2f((mu - mn) * 1.4426950408889634f);
                    const float eb = mo == kNegInf ? 0.0f : eo * exp2f((mo - mn) * 1.4426950408889634f);
                    mu = mn;
                    eu = ea + eb;
                }
            }
            if (live && u == 0) {
                const int i = 2 * r + half;
#pragma unroll
                for (int z = 0; z < R; ++z) P.pkey[((size_t)i * L + list) * R + z] = top[z];
                P.pth[(size_t)i * L + list] = fmaxf(top[R] ? dev::key_value(top[R]) : kNegInf, bmx);
                if (top[0]) atomicMax(&s_rmax[i], static_cast<unsigned>(top[0] >> 32));
                if constexpr (SOFTMAX) {
                    P.pm[(size_t)i * L + list] = mu;
                    P.ps[(size_t)i * L + list] = eu;
                }
            }
        }
        }  // TOPK == 2
        if (kDiag && P.trace && threadIdx.x == 128) P.trace[(size_t)blockIdx.x * kTrMain + 31] = static_cast<unsigned long long>(clock64() - c_pub0);
        }  // !LOGITS
        if (threadIdx.x == 128) FRS_TRACE(P, 18);
        if (kDiag && P.trace && lane == 0 && (we == 0 || we == 4))  // DIAGNOSTIC: publish cycles
            P.trace[(size_t)blockIdx.x * kTrMain + (we == 0 ? 29 : 30)] = static_cast<unsigned long long>(clock64() - c_pub0);
    }
    __syncthreads();  // every TMEM read is done; s_rmax / s_w2max complete
    if (threadIdx.x < n && s_rmax[threadIdx.x]) atomicMax(P.rowmax_bits + threadIdx.x, s_rmax[threadIdx.x]);
    if (threadIdx.x == 64) atomicMax(P.w2_bits, s_w2max);
    // this CTA's lists, bounds and maxima are published: one release increment after a barrier
    // (the finalize acquires the count instead of waiting for the whole grid to retire)
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.main_done) : "memory");
    if (kDiag && P.late_trigger) griddep_launch();
    if (threadIdx.x == 0) FRS_TRACE(P, 7);
    if (kDiag && P.trace && threadIdx.x == 0) {  // DIAGNOSTIC: the SM this CTA ran on
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        P.trace[(size_t)blockIdx.x * kTrMain + 17] = smid;
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
}

// Rigorous relative error factor (times |h|_2 |W_j|_2) between the FAST approximate logit and
// the reference dot_f32: reference lane chains (d/8 + 8) u + tensor-core fp32 accumulation
// of the hi and lo products (pessimistic, truncating adds: 2 (d + 64) 2^-23) + the hi/lo
// representation residual 2^-16 + the hi + lo add, with a safety factor.
__device__ __forceinline__ float fast_gamma(int d) {
    const double u = 0x1p-24;
    const double g = (d / 8 + 8) * u + 2.0 * (d + 64) * 0x1p-23 + 0x1p-16 + 0x1p-20;
    return static_cast<float>(g * 1.01);
}

constexpr int kCsMax = 128;   // max exactly-recomputed candidates per row (overflow: fallback)
constexpr int kFinCtas = 8;    // finalize cluster width for draft rows (portable cluster size)

struct FinArgs {
    const float *h;
    int n, d, v_rows, k;
    float temperature;
    const unsigned short *slab;
    const int32_t *ordered;
    Partials P;
    float *fin;                      // [n][kCsMax] exact logits of the selected candidates
    unsigned long long *row_ctr;     // [64] monotonic per-row arrival counters
    float *scratch;                  // [n][2 v_rows] fallback buffer
    int32_t *out_ridx, *out_full;
    float *out_prob, *out_rowmax;
    double *out_total;
    uint32_t *out_flags;
    int argmax;                      // verify mode: out_full = id_offset + argmax id, out_prob = its logit
    int32_t id_offset;
    unsigned *fb_count;              // fallback queue: count, entries row | reasons << 16
    uint32_t *fb_rows;               // [64]
    int ablate;                      // DIAGNOSTIC ONLY (FRS_ABLATE): skip finalize phases for timing
    int fin_ctas;                    // finalize cluster width (power of 2, <= kFinCtas): 8 draft, 2 verify
    int fin_stage;                   // candidates staged per round (<= kFinStage): 8 draft, 4 verify
    int surv_eps;                    // finalize survivor window (units of eps below the row max)
    int flag_sync;                   // acquire the main CTAs' publish count instead of griddepcontrol.wait
    unsigned long long *fb_arrive;   // monotonic CTA arrival counter of k_fast_fallback
};

#define FRS_FTRACE(A, slot)                                                                              \
    do {                                                                                                  \
        if (kDiag && (A).P.trace && threadIdx.x == 0)                                                     \
            (A).P.trace[(size_t)(A).P.G * kTrMain + ((size_t)blockIdx.x * kFinCtas + blockIdx.y) * 16 + (slot)] = gtimer(); \
    } while (0)

// DIAGNOSTIC: clock64 probes of select_certify (FRS_TRACE): [64 rows][16] cycles since entry
#define FRS_CPROBE(A, q)                                                                                 \
    do {                                                                                                  \
        if (kDiag && (A).P.trace && (threadIdx.x & 31) == 0)                                              \
            (A).P.trace[(size_t)(A).P.G * kTrMain + 64 * kFinCtas * 16 + 16 + (size_t)i * 16 + (q)] =    \
                static_cast<unsigned long long>(clock64() - c_entry_);                                    \
    } while (0)

// DIAGNOSTIC: finalize phase cycles (leader CTA, thread 0) since griddepcontrol.wait returned
#define FRS_FPROBE(A, q)                                                                                 \
    do {                                                                                                  \
        if (kDiag && (A).P.trace && threadIdx.x == 0 && cluster_rank() == 0)                              \
            (A).P.trace[(size_t)(A).P.G * kTrMain + 64 * kFinCtas * 16 + 16 + (size_t)blockIdx.x * 16 + (q)] = \
                static_cast<unsigned long long>(clock64() - c_fin0_);                                     \
    } while (0)

// Row pitch (floats) of the transposed per-lane-chain operand tiles of the exact recompute: a
// multiple of 4 (16-byte vector loads) with pitch % 8 == 4, so the 8 lanes of a quarter-warp
// hit 8 distinct 4-bank groups (a 2-way conflict at pitch % 8 == 0 doubled the loop time).
__host__ __device__ inline int fin_pitch(int T) {
    int tp = (T + 3) & ~3;
    if ((tp & 7) != 4) tp += 4;
    return tp;
}

constexpr int kMaxLists = 1024;  // L = 4 G <= 1024 lists of R keys per hidden row
constexpr int kSurvMax = 128;     // finalize fast path: keys within 16 eps of the row max
constexpr int kHistBins = 64;     // threshold histogram of (M - v) / bw: 48 linear bins, then
                                  // 4 bins per octave, the last one a catch-all
__device__ __forceinline__ int hist_bin(float r) {  // r >= 0 (NaN -> the catch-all bin)
    if (r < 48.0f) return static_cast<int>(r);
    // far bins from the float representation of q = r / 48 >= 1: 4 per octave by the top two
    // mantissa bits (no log2f: this runs for every key of every list)
    const uint32_t b = __float_as_uint(r * (1.0f / 48.0f));
    const int e = static_cast<int>((b >> 23) & 0xffu) - 127, m = static_cast<int>((b >> 21) & 3u);
    const int bin = 48 + 4 * e + m;
    return (e < 0 || bin >= kHistBins - 1) ? kHistBins - 1 : bin;
}
// lower edge of bin j (= upper edge of bin j - 1) in units of bw
__device__ __forceinline__ float hist_edge(int j) {
    if (j <= 48) return static_cast<float>(j);
    const int t = j - 48;
    return 48.0f * ldexpf(1.0f + 0.25f * static_cast<float>(t & 3), t >> 2);
}

// Selection + certification of one hidden row (warp 0 only; the other lanes of the CTA are
// gone). fin[0..ns) are the exact logits of the candidate set S (keys sel[], canonical order),
// nsel the untruncated |S|; a_bound bounds every approximate logit outside S, eps the FAST
// error. Writes the row's outputs, or queues it for k_fast_fallback with the reason.
__device__ __forceinline__ uint32_t select_certify(const FinArgs &A, int i, int ns, int nsel, int kk, float a_bound, float eps,
                                            bool any_bad, double tot_approx, float mmax_approx, const float *s_fin,
                                            const unsigned long long *s_sel, unsigned long long *s_sorted,
                                            unsigned long long *s_tab, int32_t *s_spos, const int32_t *s_ord,
                                            bool enqueue = true) {
    const int lane = threadIdx.x & 31;
    const float kNegInf = -__int_as_float(0x7f800000);
    const long long c_entry_ = clock64();
    const double s_tot = tot_approx;
    const float s_mmax = mmax_approx;
    uint32_t why = (nsel > kCsMax || ns < kk) ? FRS_FLAG_CERT_OVERFLOW : 0u;
    if (any_bad) why |= FRS_FLAG_NONFINITE;
    constexpr int CPL = kCsMax / 32;  // candidates per lane
    bool hq[CPL];
    float lq[CPL];
    int jq[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        const int c = lane + 32 * q;
        hq[q] = c < ns;
        lq[q] = hq[q] ? s_fin[c] : kNegInf;
        jq[q] = hq[q] ? dev::key_index(s_sel[c]) : 0;
    }
    if (A.argmax) {
        unsigned long long bv = 0ull;
#pragma unroll
        for (int q = 0; q < CPL; ++q)
            if (hq[q]) {
                const unsigned long long kq = dev::value_key(lq[q], jq[q]);
                bv = kq > bv ? kq : bv;
            }
        const unsigned long long best = warp_max_key(bv);
        const float lb = dev::key_value(best);
        if (!(a_bound + eps < lb || a_bound == kNegInf)) why |= FRS_FLAG_CERT_BOUND;
        if (why) {
            if (enqueue && lane == 0) A.fb_rows[atomicAdd(A.fb_count, 1u)] = static_cast<uint32_t>(i) | (why << 16);
            return why;
        }
        if (lane == 0) {
            A.out_full[i] = A.id_offset + dev::key_index(best);
            if (A.out_prob) A.out_prob[i] = lb;
            if (A.out_flags) A.out_flags[i] = static_cast<uint32_t>(min(ns, 255)) << 8;  // |S| (info)
        }
        FRS_FTRACE(A, 7);
        return 0u;
    }
    const unsigned long long *tab = s_tab;  // glibc exp table, staged by the caller's prologue
    const bool unit_t = A.temperature == 1.0f;  // x = l / 1 is exact: skip the IEEE divisions
    const int nq = (ns + 31) >> 5;              // warp-uniform: candidate slots in use per lane
    float xq[CPL], xm = kNegInf;
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        xq[q] = (q >= nq || unit_t) ? lq[q] : __fdiv_rn(lq[q], A.temperature);
        xm = fmaxf(xm, xq[q]);
    }
    const float mx = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(xm)));
    FRS_CPROBE(A, 0);
    // Three independent latency chains, issued together: the e-keys (branch-free glibc expf),
    // the bound on every non-recomputed row's e, and the denominator 1 / total.
    const bool bnd_live = a_bound != kNegInf;
    const float x_ub = (unit_t ? __fadd_ru(a_bound, eps) : __fdiv_ru(a_bound + eps, A.temperature)) *
                           (1.0f + 0x1p-20f) + 0x1p-20f;
    const float e_ub = dev::expf_glibc_nb(fminf(x_ub - mx, 0.0f), tab) * (1.0f + 0x1p-20f);
    // tot = sum exp(x_j - M) over the approximate logits; rescale to the exact max
    const double total = s_tot * static_cast<double>(exp2f((s_mmax - mx) * 1.4426950408889634f));
    const float inv = __double2float_rn(1.0 / total);
    unsigned long long eq[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
        if (q < nq) {
            const float e = dev::expf_glibc_nb(__fsub_rn(xq[q], mx), tab);
            eq[q] = hq[q] ? dev::prob_key(e, jq[q]) : 0ull;
            if (hq[q]) s_sorted[lane + 32 * q] = eq[q];
        } else {
            eq[q] = 0ull;
        }
    }
    FRS_CPROBE(A, 1);
    // rank of each e-key among the ns (distinct: the index is part of the key): independent
    // broadcast loads from shared memory (no shuffle chain)
    __syncwarp();
    int rq[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) rq[q] = 0;
    if (nq == 1) {
#pragma unroll 8
        for (int c = 0; c < ns; ++c) rq[0] += s_sorted[c] > eq[0];
    } else {
#pragma unroll 4
        for (int c = 0; c < ns; ++c) {
            const unsigned long long o = s_sorted[c];
#pragma unroll
            for (int q = 0; q < CPL; ++q) rq[q] += o > eq[q];
        }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        if (q < nq && hq[q]) {
            s_sorted[rq[q]] = eq[q];
            s_spos[rq[q]] = lane + 32 * q;
        }
    __syncwarp();
    FRS_CPROBE(A, 2);
    const int want = min(ns, kk + 1);
    // near ties (within 4 ulps) among the selected and at the k boundary: the probabilities
    // e * (1 / total) of such a pair may round to one value under the exact denominator, and
    // the reference then orders by index. Rounding is monotone, so only a pair whose e-order
    // disagrees with its index order can change places (a collapsed run that is not index-
    // ascending has such an adjacent pair).
    bool tie = false;
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // want <= kk + 1 <= 65 adjacent pairs
        const int r = lane + 32 * q;
        if (r + 1 < want) {
            const float ea = __uint_as_float(static_cast<uint32_t>(s_sorted[r] >> 32));
            const float eb = __uint_as_float(static_cast<uint32_t>(s_sorted[r + 1] >> 32));
            tie |= ea != eb && ea <= eb * (1.0f + 0x1p-21f) &&
                   dev::key_index(s_sorted[r]) > dev::key_index(s_sorted[r + 1]);
        }
    }
    if (__any_sync(0xffffffffu, tie) || (kDiag && A.ablate == 11)) why |= FRS_FLAG_CERT_TIE;  // 11: DIAGNOSTIC
    FRS_CPROBE(A, 3);
    if (!why && bnd_live) {  // every non-recomputed row stays strictly below the k-th
        if (!(x_ub < mx)) {
            why |= FRS_FLAG_CERT_BOUND;
        } else {
            const float e_k = __uint_as_float(static_cast<uint32_t>(s_sorted[kk - 1] >> 32));
            if (!(e_ub * (1.0f + 0x1p-21f) < e_k)) why |= FRS_FLAG_CERT_BOUND;
        }
    }
    if (why) {
        if (enqueue && lane == 0) A.fb_rows[atomicAdd(A.fb_count, 1u)] = static_cast<uint32_t>(i) | (why << 16);
        return why;
    }
    FRS_CPROBE(A, 4);
    if (lane < A.k) {
        const size_t o = (size_t)i * A.k + lane;
        if (lane < kk) {
            const unsigned long long key = s_sorted[lane];
            const int j = dev::key_index(key);
            A.out_ridx[o] = j;
            A.out_full[o] = A.ordered ? s_ord[s_spos[lane]] : j;
            A.out_prob[o] = __fmul_rn(__uint_as_float(static_cast<uint32_t>(key >> 32)), inv);
        } else {
            A.out_ridx[o] = -1;
            A.out_full[o] = -1;
            A.out_prob[o] = 0.0f;
        }
    }
    if (A.k > 32) {  // k up to 64
        const int r = lane + 32;
        if (r < A.k) {
            const size_t o = (size_t)i * A.k + r;
            if (r < kk) {
                const unsigned long long key = s_sorted[r];
                const int j = dev::key_index(key);
                A.out_ridx[o] = j;
                A.out_full[o] = A.ordered ? s_ord[s_spos[r]] : j;
                A.out_prob[o] = __fmul_rn(__uint_as_float(static_cast<uint32_t>(key >> 32)), inv);
            } else {
                A.out_ridx[o] = -1;
                A.out_full[o] = -1;
                A.out_prob[o] = 0.0f;
            }
        }
    }
    if (lane == 0) {
        if (A.out_rowmax) A.out_rowmax[i] = mx;
        if (A.out_total) A.out_total[i] = total;
        if (A.out_flags) A.out_flags[i] = static_cast<uint32_t>(min(ns, 255)) << 8;  // |S| (info)
    }
    FRS_CPROBE(A, 6);
    FRS_FTRACE(A, 7);
    return 0u;
}

// Finalize: grid (n, kFinCtas) in clusters of kFinCtas (one cluster per hidden row). The work
// per row is tiny, so every step is spread over the CTA and the number of barrier-separated
// phases is kept minimal:
//   0. (before griddepcontrol.wait, overlapping the main kernel's tail) the hidden row,
//      transposed per dot_f32 lane chain, and |h|^2; a cluster barrier orders the DSMEM
//      counters' initialisation before any remote atomic.
//   1. the row max M and max |W_j|^2 arrive as single words (atomics of the main kernel), so
//      eps and the bin width are known at once: every thread bins its union keys (4G lists x
//      R) into a histogram of (M - v) / bw; warps 0-3 merge the softmax partials, 4-5 the bounds.
//   2. every warp scans the histogram (the kk-th key's bin gives t_s = bin edge - 2 eps -
//      margin, so S = {keys >= t_s} holds every row that can reach the top-k); each CTA takes
//      the keys of S with key_index % kFinCtas == its rank (no canonical order needed).
//   3. the CTA recomputes its keys EXACTLY (dot_f32 order) and appends (key, exact logit,
//      full id) to the cluster leader's arrays through DSMEM (remote atomic slot + stores).
//   4. the leader, warp 0: selection + certification (select_certify).
__global__ void __launch_bounds__(kFinThreads) k_fast_finalize(FinArgs A) {
    extern __shared__ __align__(16) uint8_t fsm_raw[];
    const int T = A.d >> 3;           // dot_f32 steps per lane chain (d % 8 == 0 on FAST)
    const int TP = fin_pitch(T);      // padded chain pitch (elements): 16-byte aligned rows
    float *ht = reinterpret_cast<float *>(fsm_raw);  // [8][TP]
    float *wt = ht + 8 * TP;                          // [8 cand][8][TP] fp32 (bf16 widened, exact)
    __shared__ unsigned long long s_mine[kCsMax], s_sel[kCsMax], s_tab[32], s_sorted[kCsMax];
    __shared__ unsigned long long s_surv[kSurvMax], s_vk;
    __shared__ double s_hn2[kFinThreads / 32];
    __shared__ float s_abw[kFinThreads / 32], s_pmw[4], s_thw[2];
    __shared__ float s_psw[4];
    __shared__ unsigned s_hist[kHistBins];
    __shared__ float s_fin[kCsMax];      // leader: exact logits of S, in arrival (slot) order
    __shared__ int32_t s_ord[kCsMax], s_spos[kCsMax];
    __shared__ int s_nsel, s_nmine, s_cnt, s_nsurv, s_badw[kFinThreads / 32];
    __shared__ float s_afar[kFinThreads / 32];
    FRS_FTRACE(A, 0);
    // Draft rows: let the next call's chain launch now (its k_hsplit waits for this grid; its main
    // kernel's CTAs take the SMs no finalize CTA holds and fill their stage rings while this
    // grid runs). Verify rows: no early launch — 148 fallback CTAs parked in griddepcontrol.wait
    // next to this grid slowed it by ~2.7 us per call (measured).
    if (!A.argmax) griddep_launch();

    const int i = blockIdx.x, b = static_cast<int>(cluster_rank()), tid = threadIdx.x;
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = tid & 31;
    const int G = A.P.G, L = G * kListsPerCta, E = L * R;
    const float kNegInf = -__int_as_float(0x7f800000);
    // ---- 0. the hidden row (independent of the main kernel): transposed ht[l][t] = h[8t + l]
    {
        const float4 *hv = reinterpret_cast<const float4 *>(A.h + (size_t)i * A.d);
        double hn2 = 0.0;
        int bad = 0;
        for (int e0 = tid; e0 < 2 * T; e0 += 4 * kFinThreads) {  // float4 e holds h[4e .. 4e + 3]
            float4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // all loads in flight before any use
                const int e = e0 + u * kFinThreads;
                w[u] = e < 2 * T ? __ldg(hv + e) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * kFinThreads;
                if (e >= 2 * T) continue;
                const int t = e >> 1, l0 = (e & 1) * 4;
                ht[(l0 + 0) * TP + t] = w[u].x;
                ht[(l0 + 1) * TP + t] = w[u].y;
                ht[(l0 + 2) * TP + t] = w[u].z;
                ht[(l0 + 3) * TP + t] = w[u].w;
                bad |= !isfinite(w[u].x) | !isfinite(w[u].y) | !isfinite(w[u].z) | !isfinite(w[u].w);
                hn2 += static_cast<double>(w[u].x) * w[u].x + static_cast<double>(w[u].y) * w[u].y +
                       static_cast<double>(w[u].z) * w[u].z + static_cast<double>(w[u].w) * w[u].w;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hn2 += __shfl_xor_sync(0xffffffffu, hn2, o);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            s_hn2[warp] = hn2;
            s_badw[warp] = bad;
        }
        if (tid == 0) {
            s_nsel = 0;
            s_nmine = 0;
            s_cnt = 0;
            s_nsurv = 0;
        }
        if (tid < kHistBins) s_hist[tid] = 0u;
        if (tid < 32) s_tab[tid] = dev::kExp2fTable[tid];
    }
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    FRS_FTRACE(A, 1);
    // The main grid's outputs: every main CTA releases one increment of main_done after
    // publishing, so acquiring main_done == G makes all of them visible — without waiting for
    // the grid's retirement and the dependency flush (~1.3 us). All main CTAs are resident (this
    // grid launches only after each of them has started), so the spin cannot starve them.
    if (A.flag_sync) {
        if (tid == 0) {
            unsigned dn;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(dn) : "l"(A.P.main_done) : "memory");
                if (dn >= static_cast<unsigned>(G)) break;
                __nanosleep(64);
            }
        }
        __syncthreads();
    } else {
        griddep_wait();
    }
    FRS_FTRACE(A, 2);
    const long long c_fin0_ = clock64();
    if (kDiag && A.ablate == 1) return;
    // ---- 1. keys in registers, eps, histogram; softmax / bound partials. Every L2 load of the
    //         phase (keys, row max, max |W|^2, this warp's partials) is issued before any use,
    //         so the phase costs one round trip
    const int kk = min(A.k, A.v_rows);
    constexpr int KPT = kMaxLists * R / kFinThreads;  // union keys per thread
    constexpr int SW = 4;                             // warps merging the softmax partials
    constexpr int PPL = kMaxLists / (32 * SW);        // partials per lane
    constexpr int TPL = kMaxLists / 64;               // bounds per lane (warps SW, SW + 1)
    static_assert(TPL == 2 * PPL, "partials register tile");
    unsigned long long kr[KPT];
    const unsigned long long *src = A.P.pkey + (size_t)i * E;
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int e = tid + u * kFinThreads;
        kr[u] = e < E ? __ldcg(src + e) : 0ull;
    }
    const float M = dev::from_ordered(__ldcg(A.P.rowmax_bits + i));
    const float W2 = __uint_as_float(__ldcg(A.P.w2_bits));
    const bool soft_w = warp < SW && !A.argmax && !(kDiag && A.ablate == 5), bnd_w = warp >= SW && warp < SW + 2;
    float pa[TPL];  // softmax warps: pm[0..PPL) | ps[0..PPL); bound warps: pth
    if (soft_w) {
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
            const int c = warp * 32 + lane + 32 * SW * u;
            pa[u] = c < L ? __ldcg(A.P.pm + (size_t)i * L + c) : kNegInf;
            pa[PPL + u] = c < L ? __ldcg(A.P.ps + (size_t)i * L + c) : 0.0f;
        }
    } else if (bnd_w) {
#pragma unroll
        for (int u = 0; u < TPL; ++u) {
            const int c = (warp - SW) * 32 + lane + 64 * u;
            pa[u] = c < L ? __ldcg(A.P.pth + (size_t)i * L + c) : kNegInf;
        }
    }
    double h2 = 0.0;
#pragma unroll
    for (int q = 0; q < kFinThreads / 32; ++q) h2 += s_hn2[q];
    const float eps = static_cast<float>(sqrt(h2) * sqrt(static_cast<double>(W2) * 1.001)) * fast_gamma(A.d) * 1.01f;
    // coarse filter: the keys within 16 eps of the row max (typically ~30 per row) are the only
    // ones that can matter unless the top-k is spread wider (then the histogram path below)
    const float t0 = M - static_cast<float>(A.surv_eps) * eps - (fabsf(M) * 0x1p-18f + 0x1p-20f);
    {
        float a_far = kNegInf;
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            if (kr[u] == 0ull) continue;
            const float v = dev::key_value(kr[u]);
            if (v >= t0) {
                const int pos = atomicAdd(&s_nsurv, 1);
                if (pos < kSurvMax) s_surv[pos] = kr[u];
                // S is drawn from the survivors (fast path): pull my share's slab rows towards
                // L2 now, so the staging after the selection phases reads L2, not HBM
                if ((dev::key_index(kr[u]) & (A.fin_ctas - 1)) == b)
                    prefetch_l2_bulk(A.slab + (size_t)dev::key_index(kr[u]) * A.d, static_cast<uint32_t>(A.d) * 2u);
            } else {
                a_far = fmaxf(a_far, v);
            }
        }
        a_far = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_far)));
        if (lane == 0) s_afar[warp] = a_far;
    }
    FRS_FPROBE(A, 9);  // filter done (thread 0's share)
    if (soft_w) {  // softmax partials: max m_c, sum s_c exp(m_c - max)
        float mm = kNegInf;
#pragma unroll
        for (int u = 0; u < PPL; ++u) mm = fmaxf(mm, pa[u]);
        mm = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(mm)));
        float t = 0.0f;
#pragma unroll
        for (int u = 0; u < PPL; ++u)  // approximate domain anyway: one MUFU per partial
            if (pa[u] != kNegInf) t += pa[PPL + u] * exp2f((pa[u] - mm) * 1.4426950408889634f);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) {
            s_pmw[warp] = mm;
            s_psw[warp] = t;
        }
    } else if (bnd_w) {  // th = max list bound
        float th = kNegInf;
#pragma unroll
        for (int u = 0; u < TPL; ++u) th = fmaxf(th, pa[u]);
        th = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(th)));
        if (lane == 0) s_thw[warp - SW] = th;
    }
    __syncthreads();
    FRS_FPROBE(A, 10);
    // ---- 2. the kk-th largest key: rank counting among the survivors (fast path), or a
    //         histogram of (M - v) / (eps / 2) over all keys (robust path: the top-k is spread
    //         wider than the filter or there are too many survivors)
    const int nsurv = s_nsurv;
    bool robust = nsurv < kk || nsurv > kSurvMax;
    if (!robust) {
        if (tid < nsurv) {
            const unsigned long long mine = s_surv[tid];
            int rank = 0;
#pragma unroll 8
            for (int c = 0; c < nsurv; ++c) rank += s_surv[c] > mine;
            if (rank == kk - 1) s_vk = mine;
        }
        __syncthreads();
        const float vk = dev::key_value(s_vk);
        const float t_s = vk - 2.0f * eps - (fabsf(vk) * 0x1p-18f + 0x1p-20f);
        robust = t_s < t0;  // S would reach below the filter: uniform across the cluster
        if (!robust) {
            float a_below = kNegInf;
            int in_s = 0;
            if (tid < nsurv) {
                const unsigned long long key = s_surv[tid];
                const float v = dev::key_value(key);
                if (v >= t_s) {
                    in_s = 1;
                    if ((dev::key_index(key) & (A.fin_ctas - 1)) == b) {
                        const int pos = atomicAdd(&s_nmine, 1);
                        if (pos < kCsMax) s_mine[pos] = key;
                    }
                } else {
                    a_below = v;
                }
            }
            in_s = __reduce_add_sync(0xffffffffu, in_s);
            if (lane == 0 && in_s) atomicAdd(&s_nsel, in_s);
            a_below = fmaxf(dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_below))), s_afar[warp]);
            if (lane == 0) s_abw[warp] = a_below;
        }
    }
    if (robust) {
        const float bw = fmaxf(0.5f * eps, fabsf(M) * 0x1p-20f + 0x1p-30f), rbw = 1.0f / bw;
#pragma unroll
        for (int u = 0; u < KPT; ++u) {  // warp-aggregated: one shared atomic per distinct bin
            const int bin = kr[u] != 0ull ? hist_bin((M - dev::key_value(kr[u])) * rbw) : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, bin);
            if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_hist[bin], static_cast<unsigned>(__popc(peers)));
        }
        __syncthreads();
        const unsigned c0 = s_hist[2 * lane], c1 = s_hist[2 * lane + 1];
        unsigned incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const unsigned excl = incl - c0 - c1;
        const bool hit0 = excl < static_cast<unsigned>(kk) && excl + c0 >= static_cast<unsigned>(kk);
        const bool hit1 = !hit0 && excl + c0 < static_cast<unsigned>(kk) && incl >= static_cast<unsigned>(kk);
        const unsigned ball = __ballot_sync(0xffffffffu, hit0 || hit1);
        int bk = kHistBins - 1;
        if (ball) {
            const int srcl = __ffs(ball) - 1;
            bk = 2 * srcl + (__shfl_sync(0xffffffffu, hit0 ? 0 : 1, srcl));
        }
        const float t_s = bk >= kHistBins - 1 ? kNegInf
                                              : M - bw * hist_edge(bk + 1) * (1.0f + 0x1p-20f) - 2.0f * eps -
                                                    (fabsf(M) * 0x1p-18f + 0x1p-20f);
        float a_below = kNegInf;
        int in_s = 0;
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            if (kr[u] == 0ull) continue;
            const float v = dev::key_value(kr[u]);
            if (v >= t_s) {
                ++in_s;
                if ((dev::key_index(kr[u]) & (A.fin_ctas - 1)) == b) {
                    const int pos = atomicAdd(&s_nmine, 1);
                    if (pos < kCsMax) s_mine[pos] = kr[u];
                }
            } else {
                a_below = fmaxf(a_below, v);
            }
        }
        in_s = __reduce_add_sync(0xffffffffu, in_s);
        if (lane == 0 && in_s) atomicAdd(&s_nsel, in_s);
        a_below = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_below)));
        if (lane == 0) s_abw[warp] = a_below;
    }
    __syncthreads();
    FRS_FPROBE(A, 11);
    const int nsel = s_nsel;
    // ---- 3. exact recompute of my share (none if S overflowed: the leader falls back)
    const int nmine = (nsel <= kCsMax && !(kDiag && (kDiag && A.ablate == 2))) ? min(s_nmine, kCsMax) : 0;
    for (int r0 = 0; r0 < nmine; r0 += A.fin_stage) {
        const int nc = min(A.fin_stage, nmine - r0);
        constexpr int TPT = 2;  // uint4 per thread per row and batch: T <= 512 in one batch
        for (int t0 = 0; t0 < T; t0 += TPT * kFinThreads) {
            uint4 v[kFinStage][TPT];
#pragma unroll
            for (int c = 0; c < kFinStage; ++c) {
                const uint4 *row = reinterpret_cast<const uint4 *>(
                    A.slab + (size_t)dev::key_index(s_mine[r0 + (c < nc ? c : 0)]) * A.d);
#pragma unroll
                for (int u = 0; u < TPT; ++u) {
                    const int t = t0 + tid + u * kFinThreads;
                    if (c < nc && t < T) v[c][u] = __ldg(row + t);
                }
            }
#pragma unroll
            for (int c = 0; c < kFinStage; ++c) {
#pragma unroll
                for (int u = 0; u < TPT; ++u) {
                    const int t = t0 + tid + u * kFinThreads;
                    if (!(c < nc && t < T)) continue;
                    float *dst = wt + (size_t)c * 8 * TP + t;
                    const uint32_t w4[4] = {v[c][u].x, v[c][u].y, v[c][u].z, v[c][u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {  // bf16 -> fp32 is exact
                        dst[(2 * q) * TP] = __uint_as_float(w4[q] << 16);
                        dst[(2 * q + 1) * TP] = __uint_as_float(w4[q] & 0xffff0000u);
                    }
                }
            }
        }
        FRS_FPROBE(A, 12);
        __syncthreads();
        if (tid < ((nc * 8 + 31) & ~31)) {  // whole warps: the xor tree below is warp-wide
            const int cl = (tid >> 3) < nc ? tid >> 3 : 0, l = tid & 7;
            const float4 *hp = reinterpret_cast<const float4 *>(ht + l * TP);
            const float4 *wp = reinterpret_cast<const float4 *>(wt + ((size_t)cl * 8 + l) * TP);
            float s = 0.0f;
            const int T8 = T / 8;
            float4 w0 = wp[0], w1 = wp[1], h0 = hp[0], h1 = hp[1];
            for (int t8 = 0; t8 < T8; ++t8) {  // 8 steps per iteration; next operands prefetched
                const int tn = t8 + 1 < T8 ? t8 + 1 : t8;
                const float4 v0 = wp[2 * tn], v1 = wp[2 * tn + 1], g0 = hp[2 * tn], g1 = hp[2 * tn + 1];
                const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int q = 0; q < 8; ++q) s = __fadd_rn(s, __fmul_rn(hv[q], wv[q]));  // kernels.cpp:17-26 lane chain
                w0 = v0;
                w1 = v1;
                h0 = g0;
                h1 = g1;
            }
            for (int t = T8 * 8; t < T; ++t)  // T % 8 steps
                s = __fadd_rn(s, __fmul_rn(ht[l * TP + t], wt[((size_t)cl * 8 + l) * TP + t]));
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));  // ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7))
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
            if (l == 0 && (tid >> 3) < nc) {  // append to the cluster leader's arrays (DSMEM)
                const unsigned long long key = s_mine[r0 + cl];
                const int j = dev::key_index(key);
                const int32_t full = A.ordered ? __ldg(A.ordered + j) : j;
                uint32_t rc, slot;
                asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rc) : "r"(smem_u32(&s_cnt)));
                asm volatile("atom.shared::cluster.add.u32 %0, [%1], 1;" : "=r"(slot) : "r"(rc) : "memory");
                uint32_t rf, rk, ro;
                asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rf) : "r"(smem_u32(&s_fin[slot])));
                asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rk) : "r"(smem_u32(&s_sel[slot])));
                asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(ro) : "r"(smem_u32(&s_ord[slot])));
                asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(rf), "f"(s) : "memory");
                asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(rk), "l"(key) : "memory");
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(ro), "r"(full) : "memory");
            }
        }
        __syncthreads();
    }
    FRS_FPROBE(A, 13);
    // cluster barrier: release our DSMEM stores, acquire everyone's in the leader
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    // draft rows (fin_ctas CTAs, v_rows <= a few 10k) recompute an uncertified row inside the
    // cluster (below), so every CTA waits for the leader's verdict; verify rows use the grid-wide
    // k_fast_fallback queue and the non-leaders leave now
    const bool in_cluster_fb = !A.argmax;
    if (b != 0 && !in_cluster_fb) return;
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    __shared__ uint32_t s_why;
    if (b == 0 && warp == 0) {
        FRS_FPROBE(A, 14);
        // ---- 4. the cluster leader, warp 0: selection + certification
        float a_bound = fmaxf(s_thw[0], s_thw[1]);  // every row not recomputed has approx <= a_bound
        int any_bad = 0;
        for (int w = 0; w < kFinThreads / 32; ++w) {
            a_bound = fmaxf(a_bound, s_abw[w]);
            any_bad |= s_badw[w];
        }
        float mm = kNegInf;
        double tot = 0.0;
        if (!A.argmax) {
            for (int w = 0; w < SW; ++w) mm = fmaxf(mm, s_pmw[w]);
            for (int w = 0; w < SW; ++w)
                if (s_pmw[w] != kNegInf)
                    tot += s_psw[w] * static_cast<double>(exp2f((s_pmw[w] - mm) * 1.4426950408889634f));
        }
        const int ns = nsel <= kCsMax ? s_cnt : 0;  // == nsel when nothing overflowed
        uint32_t why = 0u;
        if (!(kDiag && A.ablate == 3))
            why = select_certify(A, i, ns, nsel, kk, a_bound, eps, any_bad != 0, tot, mm, s_fin, s_sel, s_sorted,
                                 s_tab, s_spos, s_ord, /*enqueue=*/!in_cluster_fb);
        // the verdict into every CTA's own s_why (remote stores before the barrier's release: no
        // CTA reads another's shared memory after it, so the leader may retire right away)
        if (in_cluster_fb && lane < A.fin_ctas) {
            uint32_t ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(&s_why)), "r"(lane));
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(why) : "memory");
        }
    }
    if (!in_cluster_fb) return;
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t why = s_why;
    if (why == 0u) return;
    // ---- 5. (rare: ~1 row in 4000) exact recompute of row i in the cluster, bit-identical to the
    //         EXACT path: each CTA the dot_f32 logits of its contiguous share of slab rows, then
    //         the leader's exact softmax + top-k (the grid-wide k_fast_fallback's arithmetic)
    float *Lr = A.scratch + (size_t)i * 2 * A.v_rows;
    {
        const int C = A.fin_ctas;
        const int r0 = static_cast<int>((long long)b * A.v_rows / C), r1 = static_cast<int>((long long)(b + 1) * A.v_rows / C);
        float *sh = wt;  // the hidden row, natural order (the staging tiles are free now)
        for (int e = tid; e < A.d; e += kFinThreads) sh[e] = A.h[(size_t)i * A.d + e];
        __syncthreads();
        const float4 *sh4 = reinterpret_cast<const float4 *>(sh);
        for (int j = r0 + tid; j < r1; j += kFinThreads) {
            const uint4 *w = reinterpret_cast<const uint4 *>(A.slab + (size_t)j * A.d);
            float c[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int t = 0; t < T; ++t) {
                const uint4 u = __ldcs(w + t);
                const float4 h0 = sh4[2 * t], h1 = sh4[2 * t + 1];
                const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const float wv = __uint_as_float(l & 1 ? (uw[l >> 1] & 0xffff0000u) : (uw[l >> 1] << 16));
                    c[l] = __fadd_rn(c[l], __fmul_rn(hv[l], wv));
                }
            }
            Lr[j] = __fadd_rn(__fadd_rn(__fadd_rn(c[0], c[1]), __fadd_rn(c[2], c[3])),
                             __fadd_rn(__fadd_rn(c[4], c[5]), __fadd_rn(c[6], c[7])));  // kernels.cpp:27
        }
    }
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (b != 0) return;
    __shared__ dev::ReduceScratch rs_fb;
    const uint32_t f2 = dev::softmax_topk_row(Lr, A.v_rows, A.k, A.temperature, A.ordered, Lr + A.v_rows,
                                              A.out_ridx + (size_t)i * A.k, A.out_full + (size_t)i * A.k,
                                              A.out_prob + (size_t)i * A.k, A.out_rowmax ? A.out_rowmax + i : nullptr,
                                              A.out_total ? A.out_total + i : nullptr, rs_fb, true);
    if (tid == 0 && A.out_flags) A.out_flags[i] = FRS_FLAG_RECOMPUTED | why | f2;
}

// Batched drafting (n > 16 hidden rows): per hidden row one CTA over the approximate logits
// row written by k_fast_main<NP,false,true> (L2-resident: n x V_sub x 4 B). Two float4 passes
// over the row (max; Σexp + the survivors above a bound from the threads' maxima), t_s from a
// histogram of the survivors (a third pass over the row only when they cannot hold the top-k),
// exact recompute of S in rounds of A.fin_stage candidates whose slab rows arrive by bulk
// copies (cp.async.bulk, one mbarrier), then the same selection + certification as the
// finalize (select_certify). Every row outside S has approx <= a_below, so a_bound = a_below.
constexpr int kSelThreads = 512;
constexpr int kSelSurv = 512;  // survivor keys kept per row (beyond: the row-scan path)

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Warp 0: the first histogram bin whose cumulative count reaches kk -> the S threshold t_s
// (every key in bins <= bk is >= M - bw * edge(bk + 1), up to the rounding of the bin index).
__device__ __forceinline__ float hist_threshold(const unsigned *s_hist, int kk, float M, float bw, float eps) {
    const int lane = threadIdx.x & 31;
    const unsigned c0 = s_hist[2 * lane], c1 = s_hist[2 * lane + 1];
    unsigned incl = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const unsigned excl = incl - c0 - c1;
    const bool hit0 = excl < static_cast<unsigned>(kk) && excl + c0 >= static_cast<unsigned>(kk);
    const bool hit1 = !hit0 && excl + c0 < static_cast<unsigned>(kk) && incl >= static_cast<unsigned>(kk);
    const unsigned ball = __ballot_sync(0xffffffffu, hit0 || hit1);
    int bk = kHistBins - 1;
    if (ball) {
        const int src = __ffs(ball) - 1;
        bk = 2 * src + (__shfl_sync(0xffffffffu, hit0 ? 0 : 1, src));
    }
    const float kNegInf = -__int_as_float(0x7f800000);
    return bk >= kHistBins - 1 ? kNegInf
                               : M - bw * hist_edge(bk + 1) * (1.0f + 0x1p-20f) - 2.0f * eps -
                                     (fabsf(M) * 0x1p-18f + 0x1p-20f);
}

// Appends for the lanes with pred set (all 32 lanes must call): one shared atomic per warp
// (per-lane atomics on one counter serialise when hundreds of keys survive). Returns the
// lane's slot, or -1.
__device__ __forceinline__ int warp_append(bool pred, int *counter) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (!m) return -1;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    return pred ? base + __popc(m & ((1u << lane) - 1u)) : -1;
}

__global__ void __launch_bounds__(kSelThreads) k_fast_select(FinArgs A) {
    extern __shared__ __align__(16) uint8_t ssm_raw[];
    const int T = A.d >> 3, TP = fin_pitch(T);
    float *ht = reinterpret_cast<float *>(ssm_raw);  // [8][TP]: the hidden row, lane chains
    // [fin_stage][d + 8] bf16: the candidates' slab rows as stored (16-byte pad: the 4 rows a
    // warp reads sit in distinct bank quads)
    unsigned short *wrows = reinterpret_cast<unsigned short *>(ht + 8 * TP);
    const int wpitch = A.d + 8;
    __shared__ unsigned long long s_S[kCsMax], s_sel[kCsMax], s_tab[32], s_sorted[kCsMax];
    __shared__ float s_fin[kCsMax], s_redf[kSelThreads / 32], s_abw[kSelThreads / 32];
    __shared__ double s_redd[kSelThreads / 32], s_hn2[kSelThreads / 32];
    __shared__ unsigned s_hist[kHistBins];
    __shared__ int32_t s_ord[kCsMax], s_spos[kCsMax];
    __shared__ int s_nsel, s_nsurv, s_badw[kSelThreads / 32];
    __shared__ float s_ts, s_afar[kSelThreads / 32];
    __shared__ unsigned long long s_surv[kSelSurv];
    __shared__ __align__(8) uint64_t s_bar;
    FRS_FTRACE(A, 0);
    griddep_launch();

    const int i = blockIdx.x, tid = threadIdx.x;
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = tid & 31;
    constexpr int NW = kSelThreads / 32;
    const float kNegInf = -__int_as_float(0x7f800000);
    {  // the hidden row (independent of the main kernel): ht[l][t] = h[8t + l], |h|^2, finiteness
        const float4 *hv = reinterpret_cast<const float4 *>(A.h + (size_t)i * A.d);
        double hn2 = 0.0;
        int bad = 0;
        for (int e = tid; e < 2 * T; e += kSelThreads) {
            const float4 w = __ldg(hv + e);
            const int t = e >> 1, l0 = (e & 1) * 4;
            ht[(l0 + 0) * TP + t] = w.x;
            ht[(l0 + 1) * TP + t] = w.y;
            ht[(l0 + 2) * TP + t] = w.z;
            ht[(l0 + 3) * TP + t] = w.w;
            bad |= !isfinite(w.x) | !isfinite(w.y) | !isfinite(w.z) | !isfinite(w.w);
            hn2 += static_cast<double>(w.x) * w.x + static_cast<double>(w.y) * w.y +
                   static_cast<double>(w.z) * w.z + static_cast<double>(w.w) * w.w;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) hn2 += __shfl_xor_sync(0xffffffffu, hn2, o);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            s_hn2[warp] = hn2;
            s_badw[warp] = bad;
        }
        if (tid == 0) {
            s_nsel = 0;
            mbar_init(&s_bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (tid < kHistBins) s_hist[tid] = 0u;
        if (tid < 32) s_tab[tid] = dev::kExp2fTable[tid];
    }
    griddep_wait();
    FRS_FTRACE(A, 2);
    const float *Lr = A.P.logits + (size_t)i * A.P.ld_logits;
    const int v = A.v_rows;
    const float inv_t = 1.0f / A.temperature;
    // The row is read with float4 loads, UNR in flight per thread, in CTA-uniform trip counts
    // (a scalar loop paid the L2 latency on every element).
    const float4 *Lr4 = reinterpret_cast<const float4 *>(Lr);
    const int v4 = (v + 3) >> 2;
    constexpr int UNR = 4;
    // ---- pass 1: max approximate logit; max |W_j|^2 (norm warps of the main kernel)
    float mx = kNegInf, w2 = 0.0f;
    for (int base = 0; base < v4; base += UNR * kSelThreads) {
        float4 b4[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int q = base + tid + u * kSelThreads;
            b4[u] = q < v4 ? __ldcg(Lr4 + q) : make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int j = 4 * (base + tid + u * kSelThreads);
            const float e[4] = {b4[u].x, b4[u].y, b4[u].z, b4[u].w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (j + c < v) mx = fmaxf(mx, e[c]);
        }
    }
    for (int c = tid; c < 2 * A.P.G; c += kSelThreads) w2 = fmaxf(w2, __ldcg(A.P.pw2 + c));
    const float mx_own = mx;  // this thread's max over its 4 * UNR * trips keys
    mx = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(mx)));
    w2 = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(w2)));
    if (lane == 0) {
        s_redf[warp] = mx;
        s_abw[warp] = w2;
    }
    if (tid == 0) s_nsurv = 0;
    __syncthreads();
    FRS_FTRACE(A, 3);
    float M = kNegInf, W2 = 0.0f;
    double h2 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        M = fmaxf(M, s_redf[w]);
        W2 = fmaxf(W2, s_abw[w]);
        h2 += s_hn2[w];
    }
    const float eps = static_cast<float>(sqrt(h2) * sqrt(static_cast<double>(W2) * 1.001)) * fast_gamma(A.d) * 1.01f;
    const float bw = fmaxf(0.5f * eps, fabsf(M) * 0x1p-20f + 0x1p-30f), rbw = 1.0f / bw;
    // The survivor threshold t0 from the threads' maxima: they are distinct keys of the row, so
    // the kk-th largest of them bounds the kk-th largest key v_k from below, and t0 =
    // hist_threshold(thread maxima) <= v_k - 2 eps keeps every key S can need.
    {
        const int bin = hist_bin((M - mx_own) * rbw);
        const unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (bin < kHistBins - 1 && lane == __ffs(peers) - 1) atomicAdd(&s_hist[bin], static_cast<unsigned>(__popc(peers)));
    }
    __syncthreads();
    if (warp == 0) {
        const float ts = hist_threshold(s_hist, min(A.k, v), M, bw, eps);
        if (lane == 0) s_ts = ts;
        s_hist[2 * lane] = 0u;  // each lane read only its own two bins
        s_hist[2 * lane + 1] = 0u;
    }
    __syncthreads();
    // ---- pass 2: Σ exp(x - max x) (approximate domain) and the survivors (keys >= t0)
    const float Mx = M * inv_t;
    const float t0 = s_ts;
    double tot = 0.0;
    float a_far = kNegInf;
    for (int base = 0; base < v4; base += UNR * kSelThreads) {
        float4 b4[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int q = base + tid + u * kSelThreads;
            b4[u] = q < v4 ? __ldcg(Lr4 + q) : make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
        }
        float part = 0.0f;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int j = 4 * (base + tid + u * kSelThreads);
            const float e[4] = {b4[u].x, b4[u].y, b4[u].z, b4[u].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // warp-uniform: survivors append warp-aggregated
                const bool in = j + c < v;
                if (in && !A.argmax) part += exp2f((e[c] * inv_t - Mx) * 1.4426950408889634f);
                const bool sv = in && e[c] >= t0;
                const int pos = warp_append(sv, &s_nsurv);
                if (sv && pos < kSelSurv) s_surv[pos] = dev::value_key(e[c], j + c);
                if (in && !sv) a_far = fmaxf(a_far, e[c]);
            }
        }
        tot += static_cast<double>(part);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    a_far = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_far)));
    if (lane == 0) {
        s_redd[warp] = tot;
        s_afar[warp] = a_far;
    }
    __syncthreads();
    FRS_FTRACE(A, 4);
    const int kk = min(A.k, v);
    const int nsurv = s_nsurv;
    bool robust = nsurv < kk || nsurv > kSelSurv || t0 == kNegInf;
    if (!robust) {  // histogram of the survivors -> t_s; S = survivors >= t_s
        for (int c = tid; c < nsurv; c += kSelThreads) {
            const int bin = hist_bin((M - dev::key_value(s_surv[c])) * rbw);
            if (bin < kHistBins - 1) atomicAdd(&s_hist[bin], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            const float ts = hist_threshold(s_hist, kk, M, bw, eps);
            if (lane == 0) s_ts = ts;
        }
        __syncthreads();
        const float t_s = s_ts;
        robust = t_s < t0;  // S would reach below the survivors
        if (!robust) {
            float a_below = kNegInf;
            for (int c = tid; c < nsurv; c += kSelThreads) {
                const unsigned long long key = s_surv[c];
                if (dev::key_value(key) >= t_s) {
                    const int pos = atomicAdd(&s_nsel, 1);
                    if (pos < kCsMax) s_S[pos] = key;
                } else {
                    a_below = fmaxf(a_below, dev::key_value(key));
                }
            }
            a_below = fmaxf(dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_below))), s_afar[warp]);
            if (lane == 0) s_abw[warp] = a_below;
        } else if (tid < kHistBins) {
            s_hist[tid] = 0u;
        }
        __syncthreads();
    }
    if (robust) {  // histogram of (M - a) / bw over the whole row, then S from the row
        for (int base = 0; base < v4; base += UNR * kSelThreads) {
            float4 b4[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int q = base + tid + u * kSelThreads;
                b4[u] = q < v4 ? __ldcg(Lr4 + q) : make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int j = 4 * (base + tid + u * kSelThreads);
                const float e[4] = {b4[u].x, b4[u].y, b4[u].z, b4[u].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int bin = j + c < v ? hist_bin((M - e[c]) * rbw) : kHistBins - 1;
                    const unsigned peers = __match_any_sync(0xffffffffu, bin);
                    if (bin < kHistBins - 1 && lane == __ffs(peers) - 1)
                        atomicAdd(&s_hist[bin], static_cast<unsigned>(__popc(peers)));
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            const float ts = hist_threshold(s_hist, kk, M, bw, eps);
            if (lane == 0) s_ts = ts;
        }
        __syncthreads();
        const float t_s = s_ts;
        float a_below = kNegInf;
        for (int base = 0; base < v4; base += UNR * kSelThreads) {
            float4 b4[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int q = base + tid + u * kSelThreads;
                b4[u] = q < v4 ? __ldcg(Lr4 + q) : make_float4(kNegInf, kNegInf, kNegInf, kNegInf);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int j = 4 * (base + tid + u * kSelThreads);
                const float e[4] = {b4[u].x, b4[u].y, b4[u].z, b4[u].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (j + c >= v) continue;
                    if (e[c] >= t_s) {
                        const int pos = atomicAdd(&s_nsel, 1);
                        if (pos < kCsMax) s_S[pos] = dev::value_key(e[c], j + c);
                    } else {
                        a_below = fmaxf(a_below, e[c]);
                    }
                }
            }
        }
        a_below = dev::from_ordered(__reduce_max_sync(0xffffffffu, dev::ordered_bits(a_below)));
        if (lane == 0) s_abw[warp] = a_below;
        __syncthreads();
    }
    const int nsel = s_nsel, ns = min(nsel, kCsMax);
    if (tid < ns) {  // canonical (descending) order
        const unsigned long long mine = s_S[tid];
        int rank = 0;
        for (int c = 0; c < ns; ++c) rank += s_S[c] > mine;
        s_sel[rank] = mine;
    }
    __syncthreads();
    if (tid < ns && A.ordered) s_ord[tid] = __ldg(A.ordered + dev::key_index(s_sel[tid]));
    FRS_FTRACE(A, 6);
    if (kDiag && A.P.trace && tid == 0)
        A.P.trace[(size_t)A.P.G * kTrMain + (size_t)blockIdx.x * kFinCtas * 16 + 8] =
            static_cast<unsigned long long>(ns) | (robust ? 1ull << 32 : 0ull);
    // ---- exact recompute of S, A.fin_stage candidates per round (dot_f32 order: lane chain l
    //      of candidate c = 8-lane group c of the CTA runs over t = 0..T-1, kernels.cpp:17-26)
    const uint32_t row_bytes = static_cast<uint32_t>(A.d) * 2u;
    for (int c0 = 0, round = 0; c0 < ns; c0 += A.fin_stage, ++round) {
        const int nc = min(A.fin_stage, ns - c0);
        if (warp == 0) {
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the last round's reads
                mbar_expect_tx(&s_bar, row_bytes * static_cast<uint32_t>(nc));
            }
            __syncwarp();
            for (int c = lane; c < nc; c += 32)
                bulk_g2s(wrows + (size_t)c * wpitch, A.slab + (size_t)dev::key_index(s_sel[c0 + c]) * A.d, row_bytes,
                         &s_bar);
        }
        if (tid < ((nc * 8 + 31) & ~31)) {  // whole warps: the xor tree below is warp-wide
            mbar_wait(&s_bar, round & 1);
            if (round == 0) FRS_FTRACE(A, 12);
            if (round == 1) FRS_FTRACE(A, 11);
            const int g = tid >> 3, cl = g < nc ? g : 0, l = tid & 7;
            const float *hp = ht + l * TP;
            const unsigned short *wp = wrows + (size_t)cl * wpitch + l;
            float s = 0.0f;
            int t = 0;
            // 16 steps per half-iteration over ping-pong operand buffers, each half's loads
            // issued before the other half's add chain (4 warps alone on the SM: nothing else
            // hides the shared-memory latency); bf16 words land in 32-bit registers
            constexpr int ST = 16;
            const int TS = T - T % ST;
            float ha[ST], hb[ST];
            uint32_t wa[ST], wb[ST];
            auto load = [&](float(&hv)[ST], uint32_t(&wv)[ST], int t0) {
#pragma unroll
                for (int q = 0; q < ST; q += 4) {
                    const float4 x = *reinterpret_cast<const float4 *>(hp + t0 + q);
                    hv[q] = x.x, hv[q + 1] = x.y, hv[q + 2] = x.z, hv[q + 3] = x.w;
                }
#pragma unroll
                for (int q = 0; q < ST; ++q) wv[q] = wp[8 * (t0 + q)];
            };
            auto chain = [&](const float(&hv)[ST], const uint32_t(&wv)[ST]) {
#pragma unroll
                for (int q = 0; q < ST; ++q) s = __fadd_rn(s, __fmul_rn(hv[q], __uint_as_float(wv[q] << 16)));  // exact
            };
            const long long c_begin = clock64();
            if (TS > 0) load(ha, wa, 0);
            for (; t < TS; t += 2 * ST) {
                const bool second = t + ST < TS;
                if (second) load(hb, wb, t + ST);
                chain(ha, wa);
                if (t + 2 * ST < TS) load(ha, wa, t + 2 * ST);
                if (second) chain(hb, wb);
            }
            t = TS;
            if (kDiag && A.P.trace && tid == 0 && round == 0)  // DIAGNOSTIC: dot cycles (trace row i*8+1)
                A.P.trace[(size_t)A.P.G * kTrMain + ((size_t)blockIdx.x * kFinCtas + 1) * 16 + 15] =
                    static_cast<unsigned long long>(clock64() - c_begin);
            for (; t < T; ++t) s = __fadd_rn(s, __fmul_rn(hp[t], __uint_as_float(static_cast<uint32_t>(wp[8 * t]) << 16)));
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 1));  // ((s0+s1)+(s2+s3))+((s4+s5)+(s6+s7))
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 2));
            s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, 4));
            if (l == 0 && g < nc) s_fin[c0 + cl] = s;
            if (round == 0) FRS_FTRACE(A, 10);
            if (round == 1) FRS_FTRACE(A, 1);
        }
        __syncthreads();
    }
    FRS_FTRACE(A, 5);
    if (warp != 0) return;
    float a_bound = kNegInf, mxx = kNegInf;
    double total = 0.0;
    int any_bad = 0;
    for (int w = 0; w < NW; ++w) {
        a_bound = fmaxf(a_bound, s_abw[w]);
        total += s_redd[w];
        any_bad |= s_badw[w];
    }
    mxx = Mx;
    select_certify(A, i, ns, nsel, kk, a_bound, eps, any_bad != 0, total, mxx, s_fin, s_sel, s_sorted, s_tab, s_spos,
                   s_ord);
}

// Grid-wide exact fallback for the rows the finalize could not certify. Launched after every
// FAST finalize (programmatic dependent launch), it exits at once when the queue is empty.
// Otherwise every CTA computes exact dot_f32 logits for its slice of slab rows of each queued
// hidden row — one thread per slab row carrying the reference's 8 lane chains, 16-byte slab
// loads — and the last CTA to finish runs the exact softmax + top-k (or argmax) of those rows,
// bit-identical to the EXACT path, then empties the queue.
constexpr int kFbBatch = 8;  // 16-byte slab loads per batch of the fallback's exact dots

__global__ void __launch_bounds__(kFbThreads) k_fast_fallback(FinArgs A) {
    extern __shared__ uint8_t fbs_raw[];
    float *sh = reinterpret_cast<float *>(fbs_raw);  // [d]
    __shared__ dev::ReduceScratch rs;
    __shared__ int s_last;
    griddep_wait();
    griddep_launch();  // the next call's main kernel may become resident as we retire
    unsigned long long *xtrace = kDiag && A.P.trace ? A.P.trace + (size_t)A.P.G * kTrMain + 64 * kFinCtas * 16 : nullptr;
    if (xtrace && blockIdx.x == 0 && threadIdx.x == 0) xtrace[2] = gtimer();
    const unsigned nfb = *reinterpret_cast<volatile unsigned *>(A.fb_count);
    if (nfb == 0) {
        if (xtrace && blockIdx.x == 0 && threadIdx.x == 0) xtrace[3] = gtimer();
        return;
    }
    const int tid = threadIdx.x, G = gridDim.x;
    const int T = A.d >> 3;  // d % 8 == 0 on the FAST path
    for (unsigned f = 0; f < nfb; ++f) {
        const int i = static_cast<int>(A.fb_rows[f] & 0xffffu);
        float *L = A.scratch + (size_t)i * 2 * A.v_rows;
        __syncthreads();
        for (int e = tid; e < A.d; e += blockDim.x) sh[e] = A.h[(size_t)i * A.d + e];
        __syncthreads();
        // one thread per slab row carrying the 8 lane chains; the row streams in batches of
        // kFbBatch 16-byte loads, the next batch in flight while the current one is consumed
        // (4 loads in flight per thread left this phase latency-bound at ~1/3 of HBM speed)
        const float4 *sh4 = reinterpret_cast<const float4 *>(sh);
        for (int j = blockIdx.x * blockDim.x + tid; j < A.v_rows; j += G * blockDim.x) {
            const uint4 *w = reinterpret_cast<const uint4 *>(A.slab + (size_t)j * A.d);
            float c[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            auto step = [&](const uint4 &u, int t) {
                const float4 h0 = sh4[2 * t], h1 = sh4[2 * t + 1];
                const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const float wv = __uint_as_float(l & 1 ? (uw[l >> 1] & 0xffff0000u) : (uw[l >> 1] << 16));
                    c[l] = __fadd_rn(c[l], __fmul_rn(hv[l], wv));
                }
            };
            const int TB = T - T % kFbBatch;
            uint4 cur[kFbBatch], nxt[kFbBatch];
            if (TB > 0) {
#pragma unroll
                for (int b = 0; b < kFbBatch; ++b) cur[b] = __ldcs(w + b);
            }
            for (int t0 = 0; t0 < TB; t0 += kFbBatch) {
                const bool more = t0 + kFbBatch < TB;
#pragma unroll
                for (int b = 0; b < kFbBatch; ++b) nxt[b] = more ? __ldcs(w + t0 + kFbBatch + b) : cur[b];
#pragma unroll
                for (int b = 0; b < kFbBatch; ++b) step(cur[b], t0 + b);
#pragma unroll
                for (int b = 0; b < kFbBatch; ++b) cur[b] = nxt[b];
            }
            for (int t = TB; t < T; ++t) step(__ldcs(w + t), t);
            L[j] = __fadd_rn(__fadd_rn(__fadd_rn(c[0], c[1]), __fadd_rn(c[2], c[3])),
                             __fadd_rn(__fadd_rn(c[4], c[5]), __fadd_rn(c[6], c[7])));  // kernels.cpp:27
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned long long old = atomicAdd(A.fb_arrive, 1ull);
        s_last = (old % G) == static_cast<unsigned long long>(G - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (xtrace && threadIdx.x == 0) xtrace[4] = gtimer();
    for (unsigned f = 0; f < nfb; ++f) {
        const uint32_t ent = A.fb_rows[f];
        const int i = static_cast<int>(ent & 0xffffu);
        const uint32_t flags = FRS_FLAG_RECOMPUTED | (ent >> 16);
        float *L = A.scratch + (size_t)i * 2 * A.v_rows;
        __syncthreads();
        if (A.argmax) {
            unsigned long long cand = 0ull;
            int bad = 0;
            for (int j = tid; j < A.v_rows; j += blockDim.x) {
                if (!isfinite(L[j])) bad = 1;
                const unsigned long long kk2 = dev::value_key(L[j], j);
                cand = kk2 > cand ? kk2 : cand;
            }
            const unsigned long long best = dev::block_reduce(cand, dev::MaxU64(), rs.k);
            bad = dev::block_reduce(bad, dev::OrI(), rs.i);
            if (tid == 0) {
                A.out_full[i] = A.id_offset + dev::key_index(best);
                if (A.out_prob) A.out_prob[i] = L[dev::key_index(best)];
                if (A.out_flags) A.out_flags[i] = flags | (bad ? FRS_FLAG_NONFINITE : 0u);
            }
            continue;
        }
        const uint32_t f2 = dev::softmax_topk_row(L, A.v_rows, A.k, A.temperature, A.ordered, L + A.v_rows,
                                                  A.out_ridx + (size_t)i * A.k, A.out_full + (size_t)i * A.k,
                                                  A.out_prob + (size_t)i * A.k,
                                                  A.out_rowmax ? A.out_rowmax + i : nullptr,
                                                  A.out_total ? A.out_total + i : nullptr, rs, true,
                                                  xtrace && f == 0 ? xtrace + 8 : nullptr);
        if (tid == 0 && A.out_flags) A.out_flags[i] = flags | f2;
    }
    __syncthreads();
    if (tid == 0) *A.fb_count = 0u;
    if (xtrace && threadIdx.x == 0) xtrace[5] = gtimer();
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

int make_map(CUtensorMap *map, const void *base, int rows, int cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return fail(FRS_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FRS_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return FRS_OK;
}

// row_ctr[64] u64 | fb_arrive u64 | fb_count u32 | fb_rows[64] u32 | rowmax_bits[64] u32 | w2_bits u32
constexpr size_t kCtrRowmax = 64 * 8 + 8 + 4 + 64 * 4;
constexpr size_t kCtrBytes = kCtrRowmax + 64 * 4 + 4 + 4;  // + main_done

struct FastWs {
    __nv_bfloat16 *hs;
    Partials P;
    float *fin;
    float *scratch;
};

int fast_workspace(frs_ctx *ctx, int NP, int d, int n, int v_rows, FastWs &w) {
    const int CS = kCsMax;
    const int G = ctx->sm_count;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    const size_t o_hs = take((size_t)2 * NP * d * 2);
    const int L = G * kListsPerCta;
    const size_t o_pm = take((size_t)NP * L * 4), o_ps = take((size_t)NP * L * 4), o_pth = take((size_t)NP * L * 4);
    const size_t o_pkey = take((size_t)NP * L * R * 8), o_pw2 = take((size_t)G * 2 * 4);
    const size_t o_fin = take((size_t)NP * CS * 4);
    const size_t o_scr = take((size_t)n * v_rows * 2 * 4);
    int st = ctx->fast_ws.ensure(off);
    if (st) return st;
    uint8_t *base = static_cast<uint8_t *>(ctx->fast_ws.ptr);
    w.hs = reinterpret_cast<__nv_bfloat16 *>(base + o_hs);
    w.P.pm = reinterpret_cast<float *>(base + o_pm);
    w.P.ps = reinterpret_cast<float *>(base + o_ps);
    w.P.pth = reinterpret_cast<float *>(base + o_pth);
    w.P.pkey = reinterpret_cast<unsigned long long *>(base + o_pkey);
    w.P.pw2 = reinterpret_cast<float *>(base + o_pw2);
    w.P.G = G;
    w.fin = reinterpret_cast<float *>(base + o_fin);
    w.scratch = reinterpret_cast<float *>(base + o_scr);
    w.P.trace = nullptr;
    w.P.tiled = nullptr;
    w.P.rowmax_bits = nullptr;
    w.P.w2_bits = nullptr;
    static const bool tracing = std::getenv("FRS_TRACE") != nullptr;
    if (tracing) {
        if ((st = ctx->trace.ensure((size_t)(G * kTrMain + 64 * kFinCtas * 16 + 16 + 64 * 16) * 8))) return st;
        w.P.trace = static_cast<unsigned long long *>(ctx->trace.ptr);
    }
    if (!ctx->fast_ctr.ptr) {  // zeroed once: counters are monotonic or reset in-stream
        if ((st = ctx->fast_ctr.ensure(kCtrBytes))) return st;
        FRS_CUDA_TRY(cudaMemset(ctx->fast_ctr.ptr, 0, kCtrBytes));
    }
    static const int late = std::getenv("FRS_ABLATE") && std::atoi(std::getenv("FRS_ABLATE")) == 8;
    w.P.late_trigger = late;
    static const int abl = std::getenv("FRS_ABLATE") ? std::atoi(std::getenv("FRS_ABLATE")) : 0;
    w.P.ablate_main = abl == 14 || abl == 15 ? abl : 0;
    static const int shift = std::getenv("FRS_RANGE_SHIFT") ? std::atoi(std::getenv("FRS_RANGE_SHIFT")) : 0;
    w.P.range_shift = kDiag ? shift : 0;
    w.P.rowmax_bits = reinterpret_cast<unsigned *>(static_cast<uint8_t *>(ctx->fast_ctr.ptr) + kCtrRowmax);
    w.P.w2_bits = w.P.rowmax_bits + 64;
    w.P.main_done = w.P.w2_bits + 1;
    w.P.tiled = nullptr;
    return FRS_OK;
}

// Per-kernel attributes, set once (and again only when a call needs more dynamic smem):
// every FAST kernel prefers the maximum shared-memory carveout, so consecutive kernels of the
// PDL chain never force an SM to drain for an L1/shared reconfiguration and can co-reside.
template <typename K>
int configure(K *kern, size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<const void *, size_t>> done;
    std::lock_guard<std::mutex> lock(mu);
    for (auto &e : done)
        if (e.first == reinterpret_cast<const void *>(kern) && e.second >= smem) return FRS_OK;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
    for (auto &e : done)
        if (e.first == reinterpret_cast<const void *>(kern)) {
            e.second = smem;
            return FRS_OK;
        }
    done.emplace_back(reinterpret_cast<const void *>(kern), smem);
    return FRS_OK;
}

template <int NP, bool SOFTMAX, bool LOGITS = false>
int launch_main(frs_ctx *ctx, const CUtensorMap &mapW, const CUtensorMap &mapW32, const CUtensorMap &mapH, int n,
                int v_rows, int d,
                float inv_t, const Partials &P, cudaStream_t s) {
    using C = MainCfg<NP, SOFTMAX>;
    auto kern = k_fast_main<NP, SOFTMAX, LOGITS>;
    if (int st = configure(kern, C::SMEM)) return st;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctx->sm_count);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mapW, mapW32, mapH, n, v_rows, d, inv_t, P));
    ++ctx->launches;
    return FRS_OK;
}

// The grid-wide exact fallback: exits at once unless the finalize / select queued a row.
int launch_fallback(frs_ctx *ctx, const FinArgs &A, cudaStream_t s) {
    auto fb = k_fast_fallback;
    const int fsmem = ((A.d + 7) & ~7) * 4;
    if (int st = configure(fb, fsmem)) return st;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ctx->sm_count);
    cfg.blockDim = dim3(kFbThreads);
    cfg.dynamicSmemBytes = fsmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, fb, A));
    ++ctx->launches;
    return FRS_OK;
}

// Candidates per exact-recompute round of k_fast_select: bulk-copied slab rows (2d + 16 B
// each) next to the hidden row's lane-chain tile, up to 16, within the opt-in shared memory
// (the static arrays take ~12 KB). 0 = the batched path does not fit this hidden size.
int sel_stage(const frs_ctx *ctx, int d) {
    const size_t fixed = (size_t)8 * fin_pitch(d / 8) * 4 + 12 * 1024;
    if (fixed >= (size_t)ctx->smem_optin) return 0;
    return (int)std::min<size_t>(16, ((size_t)ctx->smem_optin - fixed) / ((size_t)2 * d + 16));
}

int launch_select(frs_ctx *ctx, const FinArgs &A0, int rows, cudaStream_t s) {
    auto kern = k_fast_select;
    FinArgs A = A0;
    A.fin_stage = sel_stage(ctx, A.d);
    if (A.fin_stage < 1) return fail(FRS_ENOTSUP, "FAST batched draft: hidden_dim too large");
    const size_t smem = (size_t)8 * fin_pitch(A.d / 8) * 4 + (size_t)A.fin_stage * (2 * A.d + 16);
    if (int st = configure(kern, smem)) return st;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows);
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    ++ctx->launches;
    return launch_fallback(ctx, A, s);
}

int launch_fin(frs_ctx *ctx, const FinArgs &A, int rows, cudaStream_t s) {
    if (kDiag && A.ablate >= 13 && A.ablate <= 15) return FRS_OK;  // DIAGNOSTIC: main kernel only (outputs not written)
    auto kern = k_fast_finalize;
    const int TP = fin_pitch(A.d / 8);
    const size_t smem = (size_t)8 * TP * 4 + (size_t)A.fin_stage * 8 * TP * 4 + 64;
    if (smem > ctx->smem_optin) return fail(FRS_ENOTSUP, "FAST finalize: hidden_dim too large");
    if (int st = configure(kern, smem)) return st;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows, A.fin_ctas);
    cfg.blockDim = dim3(kFinThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;  // the row's CTAs meet in one cluster
    at[1].val.clusterDim.x = 1;
    at[1].val.clusterDim.y = A.fin_ctas;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    ++ctx->launches;
    if (kDiag && A.ablate == 7) return FRS_OK;  // DIAGNOSTIC: no fallback kernel
    // draft rows recompute in their finalize cluster; only verify rows (argmax) use the queue
    return A.argmax ? launch_fallback(ctx, A, s) : FRS_OK;
}

int enqueue_fast(frs_ctx *ctx, const float *h, int n, int d, const void *W, const void *tiled, int v_rows,
                 const int32_t *ordered_ids, int k, float temperature, bool argmax, int32_t id_offset,
                 int32_t *out_ridx, int32_t *out_full, float *out_prob, float *out_rowmax, double *out_total,
                 uint32_t *out_flags, int NP, FastWs &w, cudaStream_t s);

inline uint32_t __float_as_uint_host(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

GraphEntry *graph_lookup(frs_ctx *ctx, const GraphKey &key) {
    for (auto &e : ctx->graphs)
        if (e.key == key) {
            e.last_use = ++ctx->graph_clock;
            return &e;
        }
    return nullptr;
}

void graph_insert(frs_ctx *ctx, const GraphKey &key) {
    constexpr size_t kMaxGraphs = 64;
    if (ctx->graphs.size() >= kMaxGraphs) {  // evict the least recently used
        size_t lru = 0;
        for (size_t q = 1; q < ctx->graphs.size(); ++q)
            if (ctx->graphs[q].last_use < ctx->graphs[lru].last_use) lru = q;
        if (ctx->graphs[lru].exec) cudaGraphExecDestroy(ctx->graphs[lru].exec);
        ctx->graphs.erase(ctx->graphs.begin() + lru);
    }
    GraphEntry e;
    e.key = key;
    e.last_use = ++ctx->graph_clock;
    ctx->graphs.push_back(e);
}

// Batched drafting chain (17..64 hidden rows): k_hsplit -> k_fast_main<NP,false,LOGITS> ->
// k_fast_select -> k_fast_fallback. The approximate logits [n x V_sub] fp32 stay in L2.
int enqueue_batched(frs_ctx *ctx, const float *h, int n, int d, const void *W, const void *tiled, int v_rows,
                    const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx, int32_t *out_full,
                    float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags, cudaStream_t s,
                    bool argmax = false, int32_t id_offset = 0) {
    if (k > 64) return fail(FRS_ENOTSUP, "FAST draft head: k <= 64");
    // hidden rows per slab pass: 64 (N = 128) or 128 (N = 256, the widest cta_group::1 UMMA, the
    // whole 512-column TMEM double-buffered); the NP=32 variant measured slower (240 vs 133 us)
    const int NP = n > 64 ? 128 : 64;
    const int G = ctx->sm_count;
    FastWs w;
    int st = fast_workspace(ctx, NP, d, n, v_rows, w);
    if (st) return st;
    const int ld = (v_rows + 3) & ~3;
    if ((st = ctx->fast_logits.ensure((size_t)n * ld * sizeof(float)))) return st;
    w.P.logits = static_cast<float *>(ctx->fast_logits.ptr);
    w.P.ld_logits = ld;
    CUtensorMap mapW, mapW32, mapH;
    if ((st = make_map(&mapW, W, v_rows, d, BM)) || (st = make_map(&mapW32, W, v_rows, d, CH)) ||
        (st = make_map(&mapH, w.hs, 2 * NP, d, 2 * NP)))
        return st;
    timing_begin(ctx, s);
    struct EndTiming {
        frs_ctx *c;
        cudaStream_t s;
        ~EndTiming() { timing_end(c, s); }
    } end_timing{ctx, s};
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(std::min(G, (NP * d / 4 + 127) / 128));
        cfg.blockDim = dim3(128);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if ((st = configure(k_hsplit, 0))) return st;
        FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_hsplit, h, n, d, NP, w.hs, w.P.rowmax_bits, w.P.w2_bits,
                                        static_cast<unsigned long long *>(nullptr), static_cast<float *>(nullptr),
                                        w.P.main_done));
        ++ctx->launches;
    }
    w.P.tiled = static_cast<const uint8_t *>(tiled);
    const float inv_t = 1.0f / temperature;
    st = NP == 128 ? launch_main<128, false, true>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s)
                   : launch_main<64, false, true>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s);
    if (st) return st;
    FinArgs A{};
    A.h = h;
    A.n = n;
    A.d = d;
    A.v_rows = v_rows;
    A.k = k;
    A.temperature = temperature;
    A.slab = static_cast<const unsigned short *>(W);
    A.ordered = ordered_ids;
    A.P = w.P;
    A.fin = w.fin;
    A.row_ctr = static_cast<unsigned long long *>(ctx->fast_ctr.ptr);
    A.fb_arrive = A.row_ctr + 64;
    A.fb_count = reinterpret_cast<unsigned *>(A.row_ctr + 65);
    A.fb_rows = reinterpret_cast<uint32_t *>(A.fb_count + 1);
    A.scratch = w.scratch;
    A.out_ridx = out_ridx;
    A.out_full = out_full;
    A.out_prob = out_prob;
    A.out_rowmax = out_rowmax;
    A.out_total = out_total;
    A.out_flags = out_flags;
    A.argmax = argmax ? 1 : 0;
    A.id_offset = id_offset;
    if (argmax) A.k = 1;
    static const int ablate = std::getenv("FRS_ABLATE") ? std::atoi(std::getenv("FRS_ABLATE")) : 0;
    A.ablate = kDiag && ablate == 11 ? ablate : 0;
    return launch_select(ctx, A, n, s);
}

int launch_fast(frs_ctx *ctx, const float *h, int n, int d, const void *W, const void *tiled, int v_rows,
                const int32_t *ordered_ids, int k, float temperature, bool argmax, int32_t id_offset, int32_t *out_ridx,
                int32_t *out_full, float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags,
                cudaStream_t s) {
    if (d % 8 != 0) return fail(FRS_ENOTSUP, "FAST head: hidden_dim must be a multiple of 8 (TMA row pitch)");
    const bool batched_ok = sel_stage(ctx, d) >= 4;
    static const int batch_env = std::getenv("FRS_BATCH_ROWS") ? std::atoi(std::getenv("FRS_BATCH_ROWS")) : 0;
    const int batch = batch_env == 64 ? 64 : 128;  // rows per slab pass (FRS_BATCH_ROWS=64: A/B)
    if (!argmax && n > 16 && batched_ok) {  // batched drafting: up to `batch` rows per slab pass
        for (int r0 = 0; r0 < n; r0 += batch) {
            const int nr = std::min(batch, n - r0);
            const int st = enqueue_batched(ctx, h + (size_t)r0 * d, nr, d, W, tiled, v_rows, ordered_ids, k, temperature,
                                           out_ridx + (size_t)r0 * k, out_full + (size_t)r0 * k,
                                           out_prob + (size_t)r0 * k, out_rowmax ? out_rowmax + r0 : nullptr,
                                           out_total ? out_total + r0 : nullptr, out_flags ? out_flags + r0 : nullptr, s);
            if (st) return st;
        }
        return FRS_OK;
    }
    if (argmax && n > 64 && batched_ok) {  // verify of many rows: approximate logits + per-row argmax
        // (the list path is faster up to 64 rows: 238 vs 354 us at C2's 61 rows); passes of 128
        // rows (N = 256 UMMA): the pass is HBM / tensor balanced at the Llama-3-8B verify head
        for (int r0 = 0; r0 < n; r0 += 128) {
            const int nr = std::min(128, n - r0);
            const int st = enqueue_batched(ctx, h + (size_t)r0 * d, nr, d, W, tiled, v_rows, nullptr, 1, 1.0f, nullptr,
                                           out_full + r0, out_prob ? out_prob + r0 : nullptr, nullptr, nullptr,
                                           out_flags ? out_flags + r0 : nullptr, s, true, id_offset);
            if (st) return st;
        }
        return FRS_OK;
    }
    if (n > 64 && argmax) return fail(FRS_ENOTSUP, "FAST verify head: at most 64 hidden rows per call");
    if (!argmax && n > 16) {  // the fused softmax path takes 16 hidden rows per pass
        for (int r0 = 0; r0 < n; r0 += 16) {
            const int nr = std::min(16, n - r0);
            const int st = launch_fast(ctx, h + (size_t)r0 * d, nr, d, W, tiled, v_rows, ordered_ids, k, temperature, false, 0,
                                       out_ridx + (size_t)r0 * k, out_full + (size_t)r0 * k, out_prob + (size_t)r0 * k,
                                       out_rowmax ? out_rowmax + r0 : nullptr, out_total ? out_total + r0 : nullptr,
                                       out_flags ? out_flags + r0 : nullptr, s);
            if (st) return st;
        }
        return FRS_OK;
    }
    if (!argmax && k > 64) return fail(FRS_ENOTSUP, "FAST draft head: k <= 64");
    const int NP = n <= 16 ? 16 : (n <= 32 ? 32 : 64);
    const int G = ctx->sm_count;
    if (G * kListsPerCta > kMaxLists) return fail(FRS_ENOTSUP, "FAST head: too many SMs for the candidate merge");
    FastWs w;
    int st = fast_workspace(ctx, NP, d, n, v_rows, w);
    if (st) return st;
    // Optional replay (FRS_GRAPH=1): the 4-kernel chain of a repeated call (same buffers,
    // shapes and parameters) is captured once into a CUDA graph and relaunched with one
    // cudaGraphLaunch, removing the per-call host cost of 3 tensor-map encodes and 4 launches.
    // Off by default: eager launches keep the PDL overlap with the previous call's tail
    // (measured 76.7 vs 78.9 us per C2 level back to back), and the host keeps ahead anyway.
    static const bool env_graphs = std::getenv("FRS_GRAPH") != nullptr;
    const bool use_graphs = env_graphs || ctx->prefer_graphs;  // latency-bound callers (draft tree loop)
    GraphKey key{};
    if (use_graphs) {
        const uint64_t vals[] = {reinterpret_cast<uint64_t>(h), static_cast<uint64_t>(n), static_cast<uint64_t>(d),
                                 reinterpret_cast<uint64_t>(W), static_cast<uint64_t>(v_rows),
                                 reinterpret_cast<uint64_t>(ordered_ids), static_cast<uint64_t>(k),
                                 static_cast<uint64_t>(__float_as_uint_host(temperature)), static_cast<uint64_t>(argmax),
                                 static_cast<uint64_t>(static_cast<uint32_t>(id_offset)),
                                 reinterpret_cast<uint64_t>(out_ridx), reinterpret_cast<uint64_t>(out_full),
                                 reinterpret_cast<uint64_t>(out_prob), reinterpret_cast<uint64_t>(out_rowmax),
                                 reinterpret_cast<uint64_t>(out_total), reinterpret_cast<uint64_t>(out_flags),
                                 reinterpret_cast<uint64_t>(ctx->fast_ws.ptr), reinterpret_cast<uint64_t>(ctx->fast_ctr.ptr),
                                 reinterpret_cast<uint64_t>(ctx->trace.ptr),
                                 reinterpret_cast<uint64_t>(ctx->h_stage_src), reinterpret_cast<uint64_t>(tiled)};
        static_assert(sizeof(vals) / sizeof(vals[0]) == kGraphKeyWords, "graph key size");
        for (int q = 0; q < kGraphKeyWords; ++q) key.w[q] = vals[q];
        GraphEntry *e = graph_lookup(ctx, key);
        if (e && e->exec) {
            timing_begin(ctx, s);
            FRS_CUDA_TRY(cudaGraphLaunch(e->exec, s));
            timing_end(ctx, s);
            ctx->launches += 4;
            return FRS_OK;
        }
        if (e) {  // second use: capture the chain on the ctx's capture stream, then replay
            if (!ctx->cap_stream) FRS_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
            FRS_CUDA_TRY(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
            const unsigned long long l0 = ctx->launches;
            const bool timing = ctx->timing;
            ctx->timing = false;
            st = enqueue_fast(ctx, h, n, d, W, tiled, v_rows, ordered_ids, k, temperature, argmax, id_offset, out_ridx,
                              out_full, out_prob, out_rowmax, out_total, out_flags, NP, w, ctx->cap_stream);
            ctx->timing = timing;
            ctx->launches = l0;
            cudaGraph_t graph = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(ctx->cap_stream, &graph);
            if (st) {
                if (graph) cudaGraphDestroy(graph);
                return st;
            }
            if (ce != cudaSuccess) return fail(FRS_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            const cudaError_t ie = cudaGraphInstantiate(&e->exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ie != cudaSuccess) {
                e->exec = nullptr;
                return fail(FRS_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ie));
            }
            timing_begin(ctx, s);
            FRS_CUDA_TRY(cudaGraphLaunch(e->exec, s));
            timing_end(ctx, s);
            ctx->launches += 4;
            return FRS_OK;
        }
        graph_insert(ctx, key);  // first use: eager below
    }
    timing_begin(ctx, s);
    struct EndTiming {
        frs_ctx *c;
        cudaStream_t s;
        ~EndTiming() { timing_end(c, s); }
    } end_timing{ctx, s};
    return enqueue_fast(ctx, h, n, d, W, tiled, v_rows, ordered_ids, k, temperature, argmax, id_offset, out_ridx,
                        out_full, out_prob, out_rowmax, out_total, out_flags, NP, w, s);
}

// The FAST chain itself: k_hsplit -> k_fast_main -> k_fast_finalize -> k_fast_fallback.
int enqueue_fast(frs_ctx *ctx, const float *h, int n, int d, const void *W, const void *tiled, int v_rows,
                 const int32_t *ordered_ids, int k, float temperature, bool argmax, int32_t id_offset,
                 int32_t *out_ridx, int32_t *out_full, float *out_prob, float *out_rowmax, double *out_total,
                 uint32_t *out_flags, int NP, FastWs &w, cudaStream_t s) {
    const int G = ctx->sm_count;
    int st;
    CUtensorMap mapW, mapH;
    CUtensorMap mapW32;
    if ((st = make_map(&mapW, W, v_rows, d, BM)) || (st = make_map(&mapW32, W, v_rows, d, CH))) return st;
    if ((st = make_map(&mapH, w.hs, 2 * NP, d, 2 * NP))) return st;
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(std::min(ctx->sm_count, (NP * d / 4 + 127) / 128));
        cfg.blockDim = dim3(128);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        unsigned long long *xtrace = w.P.trace ? w.P.trace + (size_t)G * kTrMain + 64 * kFinCtas * 16 : nullptr;
        if ((st = configure(k_hsplit, 0))) return st;
        static const bool skip_hs = std::getenv("FRS_ABLATE") && std::atoi(std::getenv("FRS_ABLATE")) == 10;
        if (!skip_hs)  // DIAGNOSTIC (FRS_ABLATE=10): measure the chain without the split kernel
            FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_hsplit, ctx->h_stage_src ? ctx->h_stage_src : h, n, d, NP, w.hs,
                                            w.P.rowmax_bits, w.P.w2_bits, xtrace,
                                            ctx->h_stage_src ? const_cast<float *>(h) : nullptr, w.P.main_done));
        ++ctx->launches;
    }
    w.P.tiled = static_cast<const uint8_t *>(tiled);
    const float inv_t = 1.0f / temperature;
    if (argmax) {
        st = NP == 16   ? launch_main<16, false>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s)
             : NP == 32 ? launch_main<32, false>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s)
                        : launch_main<64, false>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s);
    } else {
        st = launch_main<16, true>(ctx, mapW, mapW32, mapH, n, v_rows, d, inv_t, w.P, s);
    }
    if (st) return st;
    FinArgs A{};
    A.h = h;
    A.n = n;
    A.d = d;
    A.v_rows = v_rows;
    A.k = argmax ? 1 : k;
    A.temperature = temperature;
    A.slab = static_cast<const unsigned short *>(W);
    A.ordered = ordered_ids;
    A.P = w.P;
    A.fin = w.fin;
    A.row_ctr = static_cast<unsigned long long *>(ctx->fast_ctr.ptr);
    A.fb_arrive = A.row_ctr + 64;
    A.fb_count = reinterpret_cast<unsigned *>(A.row_ctr + 65);
    A.fb_rows = reinterpret_cast<uint32_t *>(A.fb_count + 1);
    A.scratch = w.scratch;
    A.out_ridx = out_ridx;
    A.out_full = out_full;
    A.out_prob = out_prob;
    A.out_rowmax = out_rowmax;
    A.out_total = out_total;
    A.out_flags = out_flags;
    A.argmax = argmax ? 1 : 0;
    A.id_offset = id_offset;
    static const int ablate = std::getenv("FRS_ABLATE") ? std::atoi(std::getenv("FRS_ABLATE")) : 0;
    A.ablate = kDiag ? ablate : 0;
    static const int fin_env = std::getenv("FRS_FIN_CTAS") ? std::atoi(std::getenv("FRS_FIN_CTAS")) : 0;  // DIAGNOSTIC
    A.fin_ctas = argmax ? 2 : (fin_env == 2 || fin_env == 4 ? fin_env : kFinCtas);  // argmax rows: ~1-3 candidates
    A.fin_stage = argmax ? 4 : kFinStage;
    static const int surv_env = std::getenv("FRS_SURV_EPS") ? std::atoi(std::getenv("FRS_SURV_EPS")) : 0;  // DIAGNOSTIC
    // survivor window below the row max, in eps: draft rows 16 (the top-k of a flat row spans a
    // few eps); argmax rows 2: S = {keys >= M - 2 eps - margin} is the top key's own threshold, so
    // the wider window only added survivors to rank and slab rows to prefetch
    A.surv_eps = argmax ? 2 : (surv_env >= 4 ? surv_env : 16);
    static const bool no_flag = std::getenv("FRS_NO_FLAG_SYNC") != nullptr;  // A/B
    A.flag_sync = no_flag ? 0 : 1;
    return launch_fin(ctx, A, n, s);
}

}  // namespace

// Diagnostic: copy the partials of the last FAST call (rows < n) to host buffers.
int debug_fast_partials(frs_ctx *ctx, int n, int d, float *pm, float *ps, float *pth, unsigned long long *pkey,
                        float *pw2) {
    FastWs w;
    const int NP = n <= 16 ? 16 : (n <= 32 ? 32 : 64);
    int st = fast_workspace(ctx, NP, d, n, 1, w);
    if (st) return st;
    const int G = ctx->sm_count;
    FRS_CUDA_TRY(cudaDeviceSynchronize());
    const int L = G * kListsPerCta;
    FRS_CUDA_TRY(cudaMemcpy(pm, w.P.pm, sizeof(float) * n * L, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(ps, w.P.ps, sizeof(float) * n * L, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pth, w.P.pth, sizeof(float) * n * L, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pkey, w.P.pkey, sizeof(unsigned long long) * n * L * R, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pw2, w.P.pw2, sizeof(float) * 2 * G, cudaMemcpyDeviceToHost));
    if (w.P.trace) {  // trailing [G][kTrMain] main stamps, [64][kFinCtas][16] finalize stamps, [8] extra
        FRS_CUDA_TRY(cudaMemcpy(pkey + (size_t)n * L * R, w.P.trace, (size_t)(G * kTrMain + 64 * kFinCtas * 16 + 16 + 64 * 16) * 8,
                                cudaMemcpyDeviceToHost));
    }
    return FRS_OK;
}

int launch_fast_draft(frs_ctx *ctx, const float *h, int n, int d, const void *slab, const void *tiled, int v_sub,
                      const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx, int32_t *out_full,
                      float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags, cudaStream_t s) {
    return launch_fast(ctx, h, n, d, slab, tiled, v_sub, ordered_ids, k, temperature, false, 0, out_ridx, out_full,
                       out_prob, out_rowmax, out_total, out_flags, s);
}

size_t slab_tile_bytes(int v_rows, int d) {
    return (size_t)((d + BK - 1) / BK) * ((v_rows + CH - 1) / CH) * (CH * BK * 2);
}

int launch_slab_tile(frs_ctx *ctx, const void *slab, int v_rows, int d, void *tiled, cudaStream_t s) {
    const int NCH = (v_rows + CH - 1) / CH;
    k_slab_tile<<<4 * ctx->sm_count, 256, 0, s>>>(static_cast<const uint16_t *>(slab), v_rows, d, NCH,
                                                   static_cast<uint8_t *>(tiled));
    FRS_CUDA_TRY(cudaGetLastError());
    ++ctx->launches;
    return FRS_OK;
}

int launch_fast_verify(frs_ctx *ctx, const float *h, int m, int d, const void *W, const void *tiled, int v_rows,
                       int32_t id_offset, int32_t *out_id, float *out_val, uint32_t *out_flags, cudaStream_t s) {
    return launch_fast(ctx, h, m, d, W, tiled, v_rows, nullptr, 1, 1.0f, true, id_offset, nullptr, out_id, out_val,
                       nullptr, nullptr, out_flags, s);
}

namespace {

}  // namespace
}  // namespace frs
