// HBM read-bandwidth probe for the FAST draft head's access pattern (diagnostic tool, not
// product code). Streams a [rows x d] bf16 slab once per launch with:
//   ldg   : plain 16-byte loads, grid = SMs x B, U loads in flight per thread
//   tma2d : one CTA per SM, 32-row x 64-col SWIZZLE_128B boxes into an S-stage mbarrier ring,
//           the CTA's contiguous row range walked tile (4 boxes) by 64-column block — the
//           k_fast_main producer pattern with the consumers reduced to a bare arrive
//   bulk  : one CTA per SM, 1-D cp.async.bulk of contiguous C-byte pieces into the same ring
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
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
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__global__ void k_ldg(const uint4 *__restrict__ p, size_t n16, unsigned *out) {
    constexpr int U = 8;
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        const uint4 v = __ldcs(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

struct ProbeArgs {
    int rows, d, stages, mode;  // mode 0: tma2d, 1: bulk
    int piece;                  // bulk piece bytes
    const uint8_t *base;
};

__global__ void __launch_bounds__(128, 1) k_ring(const __grid_constant__ CUtensorMap map, ProbeArgs a, unsigned *out) {
    extern __shared__ uint8_t raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int STAGE = 16384;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + a.stages * STAGE), *empty = full + a.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int G = gridDim.x, cta = blockIdx.x;
    long long nstage_total;
    long long s_begin, s_end;
    if (a.mode == 0) {
        const int NCH = a.rows / 32, KB = a.d / 64;
        const int c_begin = (int)((long long)cta * NCH / G), c_end = (int)((long long)(cta + 1) * NCH / G);
        s_begin = c_begin;
        s_end = c_end;
        nstage_total = (long long)((c_end - c_begin + 3) / 4) * KB;
    } else {
        const long long bytes = (long long)a.rows * a.d * 2, np = bytes / a.piece;
        s_begin = np * cta / G;
        s_end = np * (cta + 1) / G;
        nstage_total = s_end - s_begin;
    }
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        int stage = 0;
        uint32_t phase = 0;
        if (a.mode == 0) {
            const int KB = a.d / 64;
            for (int c0 = (int)s_begin; c0 < s_end; c0 += 4) {
                const int nch = min(4, (int)s_end - c0);
                for (int kb = 0; kb < KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], nch * 4096);
                    for (int c = 0; c < nch; ++c)
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem + stage * STAGE + c * 4096)),
                            "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&full[stage])), "r"(kb * 64),
                            "r"((c0 + c) * 32), "l"(pol)
                            : "memory");
                    if (++stage == a.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        } else {
            for (long long p = s_begin; p < s_end; ++p) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_expect_tx(&full[stage], a.piece);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                        smem_u32(smem + stage * STAGE)),
                    "l"(a.base + p * a.piece), "r"(a.piece), "r"(smem_u32(&full[stage])), "l"(pol)
                    : "memory");
                if (++stage == a.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        uint32_t acc = 0;
        for (long long s = 0; s < nstage_total; ++s) {
            mbar_wait(&full[stage], phase);
            acc ^= *reinterpret_cast<volatile uint32_t *>(smem + stage * STAGE);
            mbar_arrive(&empty[stage]);
            if (++stage == a.stages) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (acc == 0x12345678u) out[0] = acc;
    }
}

int main(int argc, char **argv) {
    const int rows = argc > 1 ? atoi(argv[1]) : 32768, d = argc > 2 ? atoi(argv[2]) : 4096;
    const size_t bytes = (size_t)rows * d * 2;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int ncopy = 4;  // rotate copies: each launch reads a slab not touched by the previous one
    std::vector<uint8_t *> bufs(ncopy);
    for (auto &b : bufs) {
        CK(cudaMalloc(&b, bytes));
        CK(cudaMemset(b, 1, bytes));
    }
    unsigned *out;
    CK(cudaMalloc(&out, 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch, const char *name) {
        for (int w = 0; w < 8; ++w) launch(bufs[w % ncopy]);
        CK(cudaDeviceSynchronize());
        const int iters = 40;
        CK(cudaEventRecord(e0));
        for (int it = 0; it < iters; ++it) launch(bufs[it % ncopy]);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double us = 1000.0 * ms / iters;
        printf("{\"probe\": \"%s\", \"us\": %.2f, \"GBps\": %.1f}\n", name, us, bytes / (us * 1e-6) / 1e9);
        fflush(stdout);
    };
    for (int B : {2, 4, 8})
        for (int T : {256, 512}) {
            char name[64];
            snprintf(name, sizeof name, "ldg grid=%dxSM threads=%d", B, T);
            timeit([&](uint8_t *b) { k_ldg<<<sms * B, T>>>(reinterpret_cast<const uint4 *>(b), bytes / 16, out); }, name);
        }
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&enc), cudaEnableDefault, &q));
    std::vector<CUtensorMap> maps(ncopy);
    for (int c = 0; c < ncopy; ++c) {
        cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)d * 2};
        cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
        if (enc(&maps[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bufs[c], dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
    }
    for (int mode = 0; mode < 2; ++mode)
        for (int stages : {6, 10, 13}) {
            for (int piece : {4096, 16384}) {
                if (mode == 0 && piece != 16384) continue;
                const int smem = stages * 16384 + 2048;
                CK(cudaFuncSetAttribute(k_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                char name[96];
                snprintf(name, sizeof name, "%s stages=%d piece=%d", mode == 0 ? "tma2d(32x64 boxes, 4/stage)" : "bulk1d",
                         stages, mode == 0 ? 16384 : piece);
                int idx = 0;
                timeit(
                    [&](uint8_t *b) {
                        int c = 0;
                        for (; c < ncopy; ++c)
                            if (bufs[c] == b) break;
                        ProbeArgs a{rows, d, stages, mode, piece, b};
                        k_ring<<<sms, 128, smem>>>(maps[c], a, out);
                        ++idx;
                    },
                    name);
                CK(cudaGetLastError());
            }
        }
    return 0;
}
