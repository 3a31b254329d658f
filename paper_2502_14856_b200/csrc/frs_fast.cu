// FAST mode: tcgen05 tensor-core LM head over a bf16 slab, fused with the online-softmax
// statistics and per-CTA top-R candidate tracking, then an exact-recompute finalize that
// certifies the top-k ids against the reference arithmetic.
//
// Per call (one draft level, or one verify head), three kernels on one stream, chained with
// programmatic dependent launch so each kernel's prologue overlaps its predecessor's tail:
//
//  k_hsplit      h[n x d] fp32 -> hs[2NP x d] bf16 with rows [0,NP) = hi = bf16(h) and
//                rows [NP,2NP) = lo = bf16(h - hi): h = hi + lo + O(2^-16 |h|).
//  k_fast_main   persistent, one CTA per SM, each CTA owns a contiguous range of 128-row slab
//                tiles. Warp 0 streams (slab tile k-block, hs k-block) pairs with TMA
//                (SWIZZLE_128B, 16 KB + 2NP*128 B per stage) into a multi-stage mbarrier ring;
//                warp 1 issues tcgen05.mma (M=128 slab rows, N=2NP, K=16, bf16 -> fp32 in TMEM,
//                double-buffered accumulator); warps 2-3 read the same smem stages to accumulate
//                each slab row's squared L2 norm (for the error bound, always fresh); warps 4-7
//                drain TMEM (tcgen05.ld 32x32b), form logit = hi + lo per (slab row, hidden row),
//                update the online (max, sum-exp) statistics and a per-warp top-(R+1) list in
//                shared memory. Logits never leave the SM. Each CTA publishes (m, s), its top-R
//                candidate keys, the (R+1)-th value (bound for all its other rows) and max |W_j|^2.
//  k_fast_finalize  per hidden row: merge the CTA partials, take the CS best candidates by
//                approximate logit, recompute them EXACTLY (dot_f32 order, glibc expf), select
//                the top-k by (prob desc, index asc) and certify that no other row can enter:
//                every non-candidate's exact logit is <= bound + eps with eps a rigorous
//                error bound (reference dot_f32 error + tensor-core accumulation + hi/lo
//                truncation, Cauchy-Schwarz with |h|_2 |W_j|_2). Rows that cannot be certified
//                (near-ties within 4 ulps, or a bound too loose) fall back to the exact
//                full-row computation inside the same kernel, so ids are always the reference's.
//
// Memory bound: the slab is read exactly once per call (268,435,456 B for V_sub=32768,
// d=4096); hs (<= 1 MB) and candidate rows are L2 traffic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "frs_common.cuh"
#include "frs_device.cuh"

namespace frs {
namespace {

constexpr int BM = 128;      // slab rows per tile (UMMA M)
constexpr int BK = 64;       // k elements per stage: 128-byte bf16 rows, SWIZZLE_128B
constexpr int R = 8;         // per-CTA candidates per hidden row
constexpr int RL = R + 1;    // tracked per warp / CTA: the (R+1)-th bounds the CTA's other rows
constexpr int kFinThreads = 256;
constexpr int kCandPerFinCta = 8;  // exact recomputes per finalize CTA (8 lanes each)

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
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
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

#define FRS_TMEM_LD32(taddr, r)                                                                                   \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"          \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),       \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),            \
          "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),            \
          "=r"(r[30]), "=r"(r[31])                                                                              \
        : "r"(taddr))

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

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// Warp-wide merge of 32 new keys (one per lane) into a sorted top-RL list held in smem.
// Bitonic sort (descending) of one 64-bit key per lane across the warp, for NR independent
// rows at once so the shuffle chains of different rows interleave (ILP instead of latency).
template <int NR>
__device__ __forceinline__ void warp_sort_desc(unsigned long long (&v)[NR], int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const bool keep_max = ((lane & j) == 0) == ((lane & k) == 0);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const unsigned long long p = __shfl_xor_sync(0xffffffffu, v[r], j);
                v[r] = keep_max ? (v[r] > p ? v[r] : p) : (v[r] < p ? v[r] : p);
            }
        }
    }
}

// ------------------------------------------------------------------ kernels
struct Partials {
    float *pm;                 // [NP][G] running max of x = logit / t (softmax only)
    float *ps;                 // [NP][G] sum exp(x - pm)
    float *pth;                // [NP][G] the CTA's (R+1)-th best approximate logit (-inf if none)
    unsigned long long *pkey;  // [NP][G][R] the CTA's best R (approx value, index) keys, descending
    float *pw2;                // [G] max squared L2 norm of the CTA's slab rows
    int G;
    unsigned long long *trace; // optional [G][16] globaltimer stamps (diagnostics; nullptr = off)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define FRS_TRACE(P, slot)                                                       \
    do {                                                                         \
        if ((P).trace) (P).trace[(size_t)blockIdx.x * 16 + (slot)] = gtimer();   \
    } while (0)

// hs rows [0,NP) = bf16(h), rows [NP,2NP) = bf16(h - bf16(h)); padded rows are zero.
__global__ void __launch_bounds__(256) k_hsplit(const float *__restrict__ h, int n, int d, int NP,
                                                __nv_bfloat16 *__restrict__ hs) {
    const int total = NP * d;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int i = idx / d, c = idx - i * d;
        const float x = i < n ? h[(size_t)i * d + c] : 0.0f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(x);
        const __nv_bfloat16 lo = __float2bfloat16_rn(x - __bfloat162float(hi));
        hs[(size_t)i * d + c] = hi;
        hs[(size_t)(NP + i) * d + c] = lo;
    }
    griddep_launch();
}

template <int NP, bool SOFTMAX>
struct MainCfg {
    static constexpr int N = 2 * NP;                       // MMA N: hi rows then lo rows
    static constexpr int EPI_WARPS = NP <= 32 ? 4 : 8;     // 4 TMEM lane quarters x column halves
    static constexpr int RPW = NP / (EPI_WARPS / 4);       // hidden rows per epilogue warp
    static constexpr int TOPK = SOFTMAX ? 2 : 1;           // per-thread kept candidates per hidden row
    static constexpr int THREADS = (4 + EPI_WARPS) * 32;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = N * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 12 ? 12 : (200 * 1024) / STAGE_BYTES;
    static constexpr int TMEM_COLS = (2 * N) < 32 ? 32 : 2 * N;
    // end-of-kernel candidate scratch, reusing the (then idle) stage ring
    static constexpr int CAND_KEYS = NP * 128 * TOPK;
    static constexpr int CAND_BYTES = CAND_KEYS * 8 + NP * 128 * 4;
    static_assert(CAND_BYTES <= STAGES * STAGE_BYTES, "candidate scratch must fit the stage ring");
    static_assert(!SOFTMAX || NP == 16, "the fused softmax path handles up to 16 hidden rows per call");
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 4 * NP * 8 + 256;
};

#define FRS_TMEM_LD16(taddr, r)                                                                                 \
    asm volatile(                                                                                               \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
        : "r"(taddr))

// Warp max of a (value, index) key with 2 REDUX instead of 10 shuffles: max over the ordered
// value bits, then max over ~index among the lanes holding that value.
__device__ __forceinline__ unsigned long long warp_max_key(unsigned long long k) {
    const unsigned hi = static_cast<unsigned>(k >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? static_cast<unsigned>(k) : 0u);
    return (static_cast<unsigned long long>(mh) << 32) | ml;
}

template <int NP, bool SOFTMAX>
__global__ void __launch_bounds__(MainCfg<NP, SOFTMAX>::THREADS, 1)
    k_fast_main(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapH, int n,
                int v_rows, int d, float inv_t, Partials P) {
    using C = MainCfg<NP, SOFTMAX>;
    constexpr int N = C::N, STAGES = C::STAGES, RPW = C::RPW, TOPK = C::TOPK, EPI = C::EPI_WARPS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;                                   // STAGES x 16 KB
    uint8_t *sB = smem + STAGES * C::A_BYTES;             // STAGES x B_BYTES
    unsigned long long *cand = reinterpret_cast<unsigned long long *>(smem);  // end-of-kernel reuse
    float *cbound = reinterpret_cast<float *>(cand + C::CAND_KEYS);
    float2 *red = reinterpret_cast<float2 *>(smem + STAGES * C::STAGE_BYTES);  // [4][NP] (m, s)
    uint64_t *bars = reinterpret_cast<uint64_t *>(red + 4 * NP);
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    float *wred = reinterpret_cast<float *>(tmem_slot + 1);  // [2] norm-warp maxima

    // warp index broadcast from lane 0: provably warp-uniform, so the role branches below
    // keep their shuffles convergent (no WARPSYNC.COLLECTIVE emulation)
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int G = gridDim.x, cta = blockIdx.x;
    const int T = (v_rows + BM - 1) / BM, KB = (d + BK - 1) / BK;
    const int t_begin = static_cast<int>((static_cast<long long>(cta) * T) / G);
    const int t_end = static_cast<int>((static_cast<long long>(cta + 1) * T) / G);

    if (threadIdx.x == 0) {
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
        prefetch_tmap(&mapH);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) FRS_TRACE(P, 0);

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            const uint64_t pol_w = policy_evict_first(), pol_h = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            bool waited = false;
            for (int t = t_begin; t < t_end; ++t) {
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], C::STAGE_BYTES);
                    tma_load_2d(sA + stage * C::A_BYTES, &mapW, &full[stage], kb * BK, t * BM, pol_w);
                    if (!waited) {  // hs is produced by k_hsplit (programmatic dependency)
                        FRS_TRACE(P, 1);
                        griddep_wait();
                        FRS_TRACE(P, 9);
                        waited = true;
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
    } else if (warp < 4) {  // ---------------- row-norm warps: max_j |W_j|^2 for the error bound
        const int r0 = threadIdx.x - 64;  // 0..63: rows r0 and r0 + 64 of every tile
        float acc0 = 0.0f, acc1 = 0.0f, wmax = 0.0f;
        int stage = 0;
        uint32_t phase = 0;
        for (int t = t_begin; t < t_end; ++t) {
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
            wmax = fmaxf(wmax, fmaxf(acc0, acc1));
            acc0 = acc1 = 0.0f;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
        if (lane == 0) wred[warp - 2] = wmax;
        if (threadIdx.x == 64) FRS_TRACE(P, 8);
        asm volatile("bar.sync 2, %0;" ::"r"((2 + EPI) * 32) : "memory");  // stage ring now idle
    } else {  // ---------------- epilogue warps: TMEM -> (softmax stats, per-thread candidates)
        const int we = warp - 4;         // 0 .. EPI-1
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int cbase = (we / 4) * RPW;  // first hidden row handled by this warp
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
            tc_fence_after();
            const int row = t * BM + q * 32 + lane;
            const bool valid = row < v_rows;
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * N);
#pragma unroll
            for (int cg = 0; cg < RPW / 16; ++cg) {
                const int c0 = cbase + cg * 16;
                uint32_t hi[16], lo[16];
                if constexpr (NP == 16) {
                    uint32_t both[32];
                    FRS_TMEM_LD32(tbase, both);  // cols 0..15 hi, 16..31 lo
                    tmem_wait_ld();
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        hi[r] = both[r];
                        lo[r] = both[16 + r];
                    }
                } else {
                    FRS_TMEM_LD16(tbase + c0, hi);
                    FRS_TMEM_LD16(tbase + NP + c0, lo);
                    tmem_wait_ld();
                }
                if (cg == RPW / 16 - 1) {  // accumulator drained: hand it back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int rr = cg * 16 + r, i = c0 + r;
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
        // ---- publish per-thread state, then the CTA top-R per hidden row
        if constexpr (SOFTMAX) {
#pragma unroll
            for (int r = 0; r < RPW; ++r) {
                const int i = cbase + r;
                if (i >= n) continue;  // uniform
                float mi = m[r], si = s[r];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const float mo = __shfl_xor_sync(0xffffffffu, mi, o), so = __shfl_xor_sync(0xffffffffu, si, o);
                    const float mn = fmaxf(mi, mo);
                    si = (mn == kNegInf) ? 0.0f
                                         : si * exp2f((mi - mn) * 1.4426950408889634f) +
                                               so * exp2f((mo - mn) * 1.4426950408889634f);
                    mi = mn;
                }
                if (lane == 0) red[q * NP + i] = make_float2(mi, si);
            }
        }
        asm volatile("bar.sync 2, %0;" ::"r"((2 + EPI) * 32) : "memory");  // norm warps done with the ring
        const int slot = q * 32 + lane;  // 0..127: the thread's slab-row position within a tile
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int i = cbase + r;
            cand[(size_t)i * 128 * TOPK + slot * TOPK] = b1[r];
            if constexpr (TOPK == 2) cand[(size_t)i * 128 * TOPK + slot * TOPK + 1] = b2[r];
            cbound[i * 128 + slot] = bnd[r];
        }
        if (threadIdx.x == 128) FRS_TRACE(P, 5);
        asm volatile("bar.sync 1, %0;" ::"r"(EPI * 32) : "memory");  // the epilogue warps only
        for (int i = we; i < n; i += EPI) {
            constexpr int PL = 4 * TOPK;  // keys per lane
            unsigned long long kk[PL];
            float bmax = kNegInf;
#pragma unroll
            for (int j = 0; j < PL; ++j) kk[j] = cand[(size_t)i * 128 * TOPK + lane + 32 * j];
#pragma unroll
            for (int j = 0; j < 4; ++j) bmax = fmaxf(bmax, cbound[i * 128 + lane + 32 * j]);
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 16));
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 8));
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 4));
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 2));
            bmax = fmaxf(bmax, __shfl_xor_sync(0xffffffffu, bmax, 1));
            unsigned long long prev = ~0ull, out = 0ull;
#pragma unroll
            for (int rnd = 0; rnd < RL; ++rnd) {  // CTA top-RL by rounds of warp max
                unsigned long long mine = 0ull;
#pragma unroll
                for (int j = 0; j < PL; ++j)
                    if (kk[j] < prev && kk[j] > mine) mine = kk[j];
                const unsigned long long best = warp_max_key(mine);
                if (lane == rnd) out = best;
                prev = best ? best : prev;
                if (!best) break;  // uniform
            }
            if (lane < R) P.pkey[((size_t)i * G + cta) * R + lane] = out;
            if (lane == R) {
                const float th = out ? dev::key_value(out) : kNegInf;
                P.pth[(size_t)i * G + cta] = fmaxf(th, bmax);
            }
            if constexpr (SOFTMAX) {
                if (lane == 0) {
                    float mi = kNegInf, si = 0.0f;
                    for (int w = 0; w < 4; ++w) {
                        const float2 v = red[w * NP + i];
                        const float mn = fmaxf(mi, v.x);
                        if (mn != kNegInf)
                            si = si * exp2f((mi - mn) * 1.4426950408889634f) + v.y * exp2f((v.x - mn) * 1.4426950408889634f);
                        mi = mn;
                    }
                    P.pm[(size_t)i * G + cta] = mi;
                    P.ps[(size_t)i * G + cta] = si;
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        P.pw2[cta] = fmaxf(wred[0], wred[1]);
        FRS_TRACE(P, 7);
    }
    __threadfence();
    griddep_launch();
    __syncthreads();
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

constexpr int kFinKPT = 8;    // union keys held per finalize thread: G * R <= 256 * 8
constexpr int kCsMax = 64;    // max exactly-recomputed candidates per row (kFinCtas x 8)
constexpr int kFinCtas = kCsMax / kCandPerFinCta;

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
};

__device__ void fallback_exact_logits(const float *sh, const unsigned short *slab, int v_rows, int d, float *L) {
    // The whole CTA: 8-lane groups each compute exact dot_f32 for rows g, g + groups, ...
    const int groups = blockDim.x / 8, g = threadIdx.x / 8;
    for (int base = 0; base < v_rows; base += groups) {
        const int j = base + g;
        const int jj = j < v_rows ? j : v_rows - 1;
        const float v = dev::dot_f32_lanes8(sh, slab + (size_t)jj * d, d);
        if ((threadIdx.x & 7) == 0 && j < v_rows) L[j] = v;
    }
}

// Finalize: grid (n, kFinCtas). Every CTA of row i merges the CTA partials (identically),
// selects S = {union keys with approx >= approx_(k) - 2 eps - margin} (typically ~k..2k
// entries), recomputes its slice of S exactly, and the last CTA to arrive selects the top-k
// by (prob desc, index asc) and certifies it (see the file comment).
__global__ void __launch_bounds__(kFinThreads) k_fast_finalize(FinArgs A) {
    extern __shared__ uint8_t fsm_raw[];
    float *sh = reinterpret_cast<float *>(fsm_raw);                                   // [d]
    unsigned short *wrows = reinterpret_cast<unsigned short *>(sh + ((A.d + 7) & ~7));  // [8][d]
    __shared__ dev::ReduceScratch rs;
    __shared__ int s_nsel, s_last, s_cert;
    __shared__ float s_mx;
    __shared__ unsigned long long s_sel[kCsMax];
    __shared__ unsigned long long s_ek[kCsMax];

    const int i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, nt = blockDim.x;
    const int warp_u = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);  // warp-uniform
    const int G = A.P.G, E = G * R;
    // ---- prologue (independent of the main kernel): the hidden row and its norm
    double hn2 = 0.0;
    int bad = 0;
    {  // batch the global loads (all in flight) before the shared stores
        const float4 *hv = reinterpret_cast<const float4 *>(A.h + (size_t)i * A.d);
        const int d4 = A.d / 4;  // d % 8 == 0 on the FAST path
        constexpr int MAXV = 8;  // up to 8 float4 per thread: d <= 8192
        float4 v[MAXV];
#pragma unroll
        for (int u = 0; u < MAXV; ++u) {
            const int e = tid + u * kFinThreads;
            v[u] = e < d4 ? __ldg(hv + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int e = tid + MAXV * kFinThreads; e < d4; e += kFinThreads) {  // d > 8192
            const float4 w = __ldg(hv + e);
            reinterpret_cast<float4 *>(sh)[e] = w;
            const float xs[4] = {w.x, w.y, w.z, w.w};
            for (int q = 0; q < 4; ++q) {
                if (!isfinite(xs[q])) bad = 1;
                hn2 += static_cast<double>(xs[q]) * xs[q];
            }
        }
#pragma unroll
        for (int u = 0; u < MAXV; ++u) {
            const int e = tid + u * kFinThreads;
            if (e < d4) {
                reinterpret_cast<float4 *>(sh)[e] = v[u];
                const float xs[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!isfinite(xs[q])) bad = 1;
                    hn2 += static_cast<double>(xs[q]) * xs[q];
                }
            }
        }
    }
    if (tid == 0) s_nsel = 0;
    hn2 = dev::block_reduce(hn2, dev::SumD(), rs.d);
    bad = dev::block_reduce(bad, dev::OrI(), rs.i);
    griddep_wait();

    // ---- merge the CTA partials (identically in every CTA of this row)
    unsigned long long kr[kFinKPT];
#pragma unroll
    for (int j = 0; j < kFinKPT; ++j) {
        const int e = tid + j * nt;
        kr[j] = e < E ? A.P.pkey[(size_t)i * E + e] : 0ull;
    }
    float th = -__int_as_float(0x7f800000), w2 = 0.0f, mmax = -__int_as_float(0x7f800000);
    for (int c = tid; c < G; c += nt) {
        th = fmaxf(th, A.P.pth[(size_t)i * G + c]);
        w2 = fmaxf(w2, A.P.pw2[c]);
        if (!A.argmax) mmax = fmaxf(mmax, A.P.pm[(size_t)i * G + c]);
    }
    th = dev::block_reduce(th, dev::MaxF(), rs.f);
    w2 = dev::block_reduce(w2, dev::MaxF(), rs.f);
    double tot = 0.0;
    if (!A.argmax) {
        mmax = dev::block_reduce(mmax, dev::MaxF(), rs.f);
        for (int c = tid; c < G; c += nt) {
            const float pm = A.P.pm[(size_t)i * G + c];
            if (pm != -__int_as_float(0x7f800000))
                tot += static_cast<double>(A.P.ps[(size_t)i * G + c]) * exp(static_cast<double>(pm) - mmax);
        }
        tot = dev::block_reduce(tot, dev::SumD(), rs.d);
    }
    const float eps = static_cast<float>(sqrt(hn2) * sqrt(static_cast<double>(w2) * 1.001)) * fast_gamma(A.d) * 1.01f;

    // approx_(kk): the kk-th largest union key, by kk rounds of block max
    const int kk = min(A.k, A.v_rows);
    unsigned long long prev = ~0ull, kth = 0ull;
    for (int r = 0; r < kk; ++r) {
        unsigned long long mine = 0ull;
#pragma unroll
        for (int j = 0; j < kFinKPT; ++j)
            if (kr[j] < prev && kr[j] > mine) mine = kr[j];
        const unsigned long long best = dev::block_reduce(mine, dev::MaxU64(), rs.k);
        if (best == 0ull) break;
        prev = kth = best;
    }
    const float vk = kth ? dev::key_value(kth) : -__int_as_float(0x7f800000);
    const float t_s = vk - 2.0f * eps - (fabsf(vk) * 0x1p-18f + 0x1p-20f);
    // S = union keys at or above t_s; a_below = best union value left out
    float a_below = -__int_as_float(0x7f800000);
#pragma unroll
    for (int j = 0; j < kFinKPT; ++j) {
        if (kr[j] == 0ull) continue;
        const float v = dev::key_value(kr[j]);
        if (v >= t_s) {
            const int pos = atomicAdd(&s_nsel, 1);
            if (pos < kCsMax) s_sel[pos] = kr[j];
        } else {
            a_below = fmaxf(a_below, v);
        }
    }
    a_below = dev::block_reduce(a_below, dev::MaxF(), rs.f);
    const int nsel = s_nsel;  // block_reduce synchronized
    const int ns = min(nsel, kCsMax);
    // canonical (descending) order, so every CTA of the row indexes S identically
    unsigned long long my_sel = tid < ns ? s_sel[tid] : 0ull;
    int my_rank = 0;
    for (int c = 0; c < ns; ++c) my_rank += s_sel[c] > my_sel;
    __syncthreads();
    if (tid < ns) s_sel[my_rank] = my_sel;
    __syncthreads();

    // ---- exact recompute of my slice S[8b, 8b + 8)
    const int c0 = b * kCandPerFinCta, c1 = min(ns, c0 + kCandPerFinCta);
    if (c0 < c1) {
        {  // all candidate-row loads in flight at once: 8 rows x d/8 uint4 over the CTA
            const int per_row = A.d / 8, total = (c1 - c0) * per_row;
            constexpr int MAXV = 16;  // 8 rows x 512 uint4 / 256 threads for d = 4096
            uint4 v[MAXV];
#pragma unroll
            for (int u = 0; u < MAXV; ++u) {
                const int e = tid + u * kFinThreads;
                if (e < total) {
                    const int c = c0 + e / per_row, off = e % per_row;
                    v[u] = __ldg(reinterpret_cast<const uint4 *>(A.slab + (size_t)dev::key_index(s_sel[c]) * A.d) + off);
                }
            }
#pragma unroll
            for (int u = 0; u < MAXV; ++u) {
                const int e = tid + u * kFinThreads;
                if (e < total) reinterpret_cast<uint4 *>(wrows)[e] = v[u];
            }
            for (int e = tid + MAXV * kFinThreads; e < total; e += kFinThreads) {  // d > 4096
                const int c = c0 + e / per_row, off = e % per_row;
                reinterpret_cast<uint4 *>(wrows)[e] =
                    __ldg(reinterpret_cast<const uint4 *>(A.slab + (size_t)dev::key_index(s_sel[c]) * A.d) + off);
            }
        }
        __syncthreads();
        if (warp_u < kCandPerFinCta * 8 / 32) {
            const int c = c0 + tid / 8;
            const int cc = c < c1 ? c : c0;
            const float v = dev::dot_f32_lanes8(sh, wrows + (size_t)(cc - c0) * A.d, A.d);
            if ((tid & 7) == 0 && c < c1) A.fin[(size_t)i * kCsMax + c] = v;
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned long long old = atomicAdd(&A.row_ctr[i], 1ull);
        s_last = (old % kFinCtas) == static_cast<unsigned long long>(kFinCtas - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- selection + certification (the last CTA of this row)
    const float a_bound = fmaxf(th, a_below);  // every row not recomputed has approx <= a_bound
    uint32_t flags = bad ? FRS_FLAG_NONFINITE : 0u;
    dev::load_exp_table(rs.tab);
    __syncthreads();
    if (warp_u == 0) {
        const bool overflow = nsel > kCsMax;
        float mx = -__int_as_float(0x7f800000);
        unsigned long long best_val = 0ull;
        for (int c = tid; c < ns; c += 32) {
            const float l = A.fin[(size_t)i * kCsMax + c];
            const float x = __fdiv_rn(l, A.temperature);
            mx = fmaxf(mx, x);
            const unsigned long long vkey = dev::value_key(l, dev::key_index(s_sel[c]));
            best_val = vkey > best_val ? vkey : best_val;
            s_ek[c] = __float_as_uint(x);  // stash x; replaced by the e-key below
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        best_val = warp_max_u64(best_val);
        bool cert = !bad && !overflow && ns >= kk;
        if (A.argmax) {
            // every non-recomputed row: exact <= a_bound + eps < the best exact logit
            if (tid == 0) {
                const float lb = dev::key_value(best_val);
                cert = cert && (a_bound + eps < lb || a_bound == -__int_as_float(0x7f800000));
                s_ek[0] = best_val;
                s_cert = cert;
            }
        } else {
            __syncwarp();
            for (int c = tid; c < ns; c += 32) {
                const float x = __uint_as_float(static_cast<uint32_t>(s_ek[c]));
                s_ek[c] = dev::prob_key(dev::expf_glibc(__fsub_rn(x, mx), rs.tab), dev::key_index(s_sel[c]));
            }
            __syncwarp();
            const int want = min(ns, kk + 1);
            for (int r = 0; r < want; ++r) {  // selection sort of the leading (kk + 1) e-keys
                unsigned long long best = 0ull;
                int where = -1;
                for (int c = r + tid; c < ns; c += 32)
                    if (s_ek[c] > best) {
                        best = s_ek[c];
                        where = c;
                    }
                const unsigned long long wbest = warp_max_u64(best);
                const unsigned ball = __ballot_sync(0xffffffffu, where >= 0 && best == wbest);
                const int w = __shfl_sync(0xffffffffu, where, __ffs(ball) - 1);
                if (tid == 0 && w != r) {
                    const unsigned long long tmp = s_ek[r];
                    s_ek[r] = s_ek[w];
                    s_ek[w] = tmp;
                }
                __syncwarp();
            }
            if (tid == 0) {
                // near ties (within 4 ulps) among the selected and at the k boundary: the
                // reference's (prob, index) order could depend on the exact denominator
                for (int r = 0; cert && r + 1 < want; ++r) {
                    const float ea = __uint_as_float(static_cast<uint32_t>(s_ek[r] >> 32));
                    const float eb = __uint_as_float(static_cast<uint32_t>(s_ek[r + 1] >> 32));
                    if (ea != eb && ea <= eb * (1.0f + 0x1p-21f)) cert = false;
                }
                if (cert && a_bound != -__int_as_float(0x7f800000)) {
                    const float x_ub = __fdiv_ru(a_bound + eps, A.temperature) * (1.0f + 0x1p-20f) + 0x1p-20f;
                    if (!(x_ub < mx)) {
                        cert = false;
                    } else {
                        const float e_ub = dev::expf_glibc(x_ub - mx, rs.tab) * (1.0f + 0x1p-20f);
                        const float e_k = __uint_as_float(static_cast<uint32_t>(s_ek[kk - 1] >> 32));
                        if (!(e_ub * (1.0f + 0x1p-21f) < e_k)) cert = false;
                    }
                }
                s_cert = cert;
                s_mx = mx;
            }
        }
    }
    __syncthreads();
    if (s_cert) {
        if (tid == 0) {
            if (A.argmax) {
                const unsigned long long best = s_ek[0];
                A.out_full[i] = A.id_offset + dev::key_index(best);
                if (A.out_prob) A.out_prob[i] = dev::key_value(best);
            } else {
                const float mx = s_mx;
                // tot = sum exp(x_j - M) in the approximate domain; rescale to the exact max
                const double total = tot * exp(static_cast<double>(mmax) - static_cast<double>(mx));
                const float inv = __double2float_rn(1.0 / total);
                for (int r = 0; r < kk; ++r) {
                    const int j = dev::key_index(s_ek[r]);
                    A.out_ridx[(size_t)i * A.k + r] = j;
                    A.out_full[(size_t)i * A.k + r] = A.ordered ? A.ordered[j] : j;
                    A.out_prob[(size_t)i * A.k + r] =
                        __fmul_rn(__uint_as_float(static_cast<uint32_t>(s_ek[r] >> 32)), inv);
                }
                for (int r = kk; r < A.k; ++r) {
                    A.out_ridx[(size_t)i * A.k + r] = -1;
                    A.out_full[(size_t)i * A.k + r] = -1;
                    A.out_prob[(size_t)i * A.k + r] = 0.0f;
                }
                if (A.out_rowmax) A.out_rowmax[i] = mx;
                if (A.out_total) A.out_total[i] = total;
            }
            if (A.out_flags) A.out_flags[i] = flags;
        }
        return;
    }
    // ---- fallback: the exact full row in this CTA (bit-identical to the EXACT path)
    float *L = A.scratch + (size_t)i * 2 * A.v_rows;
    if (!bad) {
        fallback_exact_logits(sh, A.slab, A.v_rows, A.d, L);
        flags |= FRS_FLAG_RECOMPUTED;
    } else {
        for (int j = tid; j < A.v_rows; j += nt) L[j] = __int_as_float(0x7fc00000);
    }
    __syncthreads();
    if (A.argmax) {
        unsigned long long cand = 0ull;
        for (int j = tid; j < A.v_rows; j += nt) {
            const unsigned long long kk2 = dev::value_key(L[j], j);
            cand = kk2 > cand ? kk2 : cand;
        }
        const unsigned long long best = dev::block_reduce(cand, dev::MaxU64(), rs.k);
        if (tid == 0) {
            A.out_full[i] = A.id_offset + dev::key_index(best);
            if (A.out_prob) A.out_prob[i] = L[dev::key_index(best)];
            if (A.out_flags) A.out_flags[i] = flags;
        }
        return;
    }
    const uint32_t f2 = dev::softmax_topk_row(L, A.v_rows, A.k, A.temperature, A.ordered, L + A.v_rows,
                                              A.out_ridx + (size_t)i * A.k, A.out_full + (size_t)i * A.k,
                                              A.out_prob + (size_t)i * A.k, A.out_rowmax ? A.out_rowmax + i : nullptr,
                                              A.out_total ? A.out_total + i : nullptr, rs);
    if (tid == 0 && A.out_flags) A.out_flags[i] = flags | f2;
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
    const size_t o_pm = take((size_t)NP * G * 4), o_ps = take((size_t)NP * G * 4), o_pth = take((size_t)NP * G * 4);
    const size_t o_pkey = take((size_t)NP * G * R * 8), o_pw2 = take((size_t)G * 4);
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
    static const bool tracing = std::getenv("FRS_TRACE") != nullptr;
    if (tracing) {
        if ((st = ctx->trace.ensure((size_t)G * 16 * 8))) return st;
        w.P.trace = static_cast<unsigned long long *>(ctx->trace.ptr);
    }
    if (!ctx->fast_ctr.ptr) {
        if ((st = ctx->fast_ctr.ensure(64 * sizeof(unsigned long long)))) return st;
        FRS_CUDA_TRY(cudaMemset(ctx->fast_ctr.ptr, 0, 64 * sizeof(unsigned long long)));
    }
    return FRS_OK;
}

template <int NP, bool SOFTMAX>
int launch_main(frs_ctx *ctx, const CUtensorMap &mapW, const CUtensorMap &mapH, int n, int v_rows, int d,
                float inv_t, const Partials &P, cudaStream_t s) {
    using C = MainCfg<NP, SOFTMAX>;
    auto kern = k_fast_main<NP, SOFTMAX>;
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
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
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, mapW, mapH, n, v_rows, d, inv_t, P));
    ++ctx->launches;
    return FRS_OK;
}

int launch_fin(frs_ctx *ctx, const FinArgs &A, int rows, cudaStream_t s) {
    auto kern = k_fast_finalize;
    const size_t smem = (size_t)((A.d + 7) & ~7) * 4 + (size_t)kCandPerFinCta * A.d * 2 + 64;
    if (smem > ctx->smem_optin) return fail(FRS_ENOTSUP, "FAST finalize: hidden_dim too large");
    FRS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows, kFinCtas);
    cfg.blockDim = dim3(kFinThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FRS_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, A));
    ++ctx->launches;
    return FRS_OK;
}

int launch_fast(frs_ctx *ctx, const float *h, int n, int d, const void *W, int v_rows, const int32_t *ordered_ids,
                int k, float temperature, bool argmax, int32_t id_offset, int32_t *out_ridx, int32_t *out_full,
                float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags, cudaStream_t s) {
    if (d % 8 != 0) return fail(FRS_ENOTSUP, "FAST head: hidden_dim must be a multiple of 8 (TMA row pitch)");
    if (n > 64) return fail(FRS_ENOTSUP, "FAST head: at most 64 hidden rows per call");
    if (!argmax && n > 16) {  // the fused softmax path takes 16 hidden rows per pass
        for (int r0 = 0; r0 < n; r0 += 16) {
            const int nr = std::min(16, n - r0);
            const int st = launch_fast(ctx, h + (size_t)r0 * d, nr, d, W, v_rows, ordered_ids, k, temperature, false, 0,
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
    if (G * R > kFinThreads * kFinKPT) return fail(FRS_ENOTSUP, "FAST head: too many SMs for the candidate merge");
    FastWs w;
    int st = fast_workspace(ctx, NP, d, n, v_rows, w);
    if (st) return st;
    CUtensorMap mapW, mapH;
    if ((st = make_map(&mapW, W, v_rows, d, BM))) return st;
    if ((st = make_map(&mapH, w.hs, 2 * NP, d, 2 * NP))) return st;

    timing_begin(ctx, s);
    struct EndTiming {
        frs_ctx *c;
        cudaStream_t s;
        ~EndTiming() { timing_end(c, s); }
    } end_timing{ctx, s};
    k_hsplit<<<std::min(ctx->sm_count, (NP * d + 255) / 256), 256, 0, s>>>(h, n, d, NP, w.hs);
    ++ctx->launches;
    FRS_CUDA_TRY(cudaGetLastError());
    const float inv_t = 1.0f / temperature;
    if (argmax) {
        st = NP == 16   ? launch_main<16, false>(ctx, mapW, mapH, n, v_rows, d, inv_t, w.P, s)
             : NP == 32 ? launch_main<32, false>(ctx, mapW, mapH, n, v_rows, d, inv_t, w.P, s)
                        : launch_main<64, false>(ctx, mapW, mapH, n, v_rows, d, inv_t, w.P, s);
    } else {
        st = launch_main<16, true>(ctx, mapW, mapH, n, v_rows, d, inv_t, w.P, s);
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
    A.scratch = w.scratch;
    A.out_ridx = out_ridx;
    A.out_full = out_full;
    A.out_prob = out_prob;
    A.out_rowmax = out_rowmax;
    A.out_total = out_total;
    A.out_flags = out_flags;
    A.argmax = argmax ? 1 : 0;
    A.id_offset = id_offset;
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
    FRS_CUDA_TRY(cudaMemcpy(pm, w.P.pm, sizeof(float) * n * G, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(ps, w.P.ps, sizeof(float) * n * G, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pth, w.P.pth, sizeof(float) * n * G, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pkey, w.P.pkey, sizeof(unsigned long long) * n * G * R, cudaMemcpyDeviceToHost));
    FRS_CUDA_TRY(cudaMemcpy(pw2, w.P.pw2, sizeof(float) * G, cudaMemcpyDeviceToHost));
    if (w.P.trace && ctx->trace.bytes >= (size_t)G * 16 * 8) {  // trailing [G][16] stamps
        FRS_CUDA_TRY(cudaMemcpy(pkey + (size_t)n * G * R, w.P.trace, (size_t)G * 16 * 8, cudaMemcpyDeviceToHost));
    }
    return FRS_OK;
}

int launch_fast_draft(frs_ctx *ctx, const float *h, int n, int d, const void *slab, int v_sub,
                      const int32_t *ordered_ids, int k, float temperature, int32_t *out_ridx, int32_t *out_full,
                      float *out_prob, float *out_rowmax, double *out_total, uint32_t *out_flags, cudaStream_t s) {
    return launch_fast(ctx, h, n, d, slab, v_sub, ordered_ids, k, temperature, false, 0, out_ridx, out_full,
                       out_prob, out_rowmax, out_total, out_flags, s);
}

int launch_fast_verify(frs_ctx *ctx, const float *h, int m, int d, const void *W, int v_rows, int32_t id_offset,
                       int32_t *out_id, float *out_val, uint32_t *out_flags, cudaStream_t s) {
    return launch_fast(ctx, h, m, d, W, v_rows, nullptr, 1, 1.0f, true, id_offset, nullptr, out_id, out_val,
                       nullptr, nullptr, out_flags, s);
}

namespace {

}  // namespace
}  // namespace frs
