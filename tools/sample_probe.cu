// DIAGNOSTIC: phase stamps of a copy of k_softmax_sample (frs_exact.cu) on n rows of v logits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2502_14856_b200/csrc \
//      tools/sample_probe.cu -o tools/sample_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "frs_device.cuh"
using namespace frs;
#define STAMP(q) do { if (blockIdx.x == 0 && threadIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); stamps[q] = t_; } } while (0)
__global__ void __launch_bounds__(1024)
    k_sample_probe(unsigned long long *stamps, const float *__restrict__ logits, int v, float temperature, const double *__restrict__ uniforms,
                     int w, const int32_t *__restrict__ ordered, float *__restrict__ probs, float *__restrict__ work,
                     int32_t *__restrict__ out_ridx, int32_t *__restrict__ out_full, float *__restrict__ out_prob,
                     int32_t *__restrict__ out_count, uint32_t *__restrict__ out_flags, int wk_in_smem) {
    __shared__ dev::ReduceScratch rs;
    __shared__ double s_cp[1024];
    extern __shared__ float s_wk[];  // the draw weights when v floats fit (wk_in_smem)
    const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const float *L = logits + (size_t)row * v;
    float *P = probs + (size_t)row * v, *Wk = wk_in_smem ? s_wk : work + (size_t)row * v;
    STAMP(0);
    uint32_t flags = dev::softmax_probs_row(L, v, temperature, P, rs);
    STAMP(1);
    __shared__ int s_pick;
    const int C = (v + 1023) / 1024, j0 = min(v, tid * C), j1 = min(v, j0 + C);
    // work = probs (coalesced; the chunk sums and the draws read other threads' chunks). A
    // per-thread chunk copy through global memory was a chain of dependent L2 round trips
    // (43 us at V_sub 32768) and so were its chunk sums (18 us); from shared memory both are ~1 us.
    for (int j = tid; j < v; j += 1024) Wk[j] = P[j];
    __syncthreads();
    STAMP(2);
    // Prefix bookkeeping: a fresh scan (chunk sums + block scan) is within errP = 2^-46 T of the
    // exact prefix; each later pick is subtracted in place (one rounding each, errP grows by
    // 2^-52 T). The reference's running sums are within (v + 64) 2^-53 T of the exact ones.
    // Rescan when the remaining mass halves, so the bounds stay relative to it.
    double errP = 0.0, t_scan = 0.0;
    bool need_scan = true;
    __shared__ int s_pchunk;
    int count = 0;
    for (int k = 0; k < w; ++k) {
        if (need_scan) {
            double cs = 0.0;
            // the chunk sum in a lane-rotated order (any order is within errP): chunks are
            // C floats apart, so lane l starting at offset l keeps the 32 lanes on distinct banks
            const int cnt = j1 - j0;
            for (int i = 0; i < cnt; ++i) {
                int o = i + lane;
                o = o >= cnt ? o - cnt : o;
                o = o >= cnt ? o % cnt : o;
                cs += static_cast<double>(Wk[j0 + o]);
            }
            __syncthreads();  // readers of the previous s_cp are done
            s_cp[tid] = cs;
            __syncthreads();
            for (int off = 1; off < 1024; off <<= 1) {  // inclusive scan of the chunk sums
                double x = s_cp[tid];
                if (tid >= off) x += s_cp[tid - off];
                __syncthreads();
                s_cp[tid] = x;
                __syncthreads();
            }
            t_scan = s_cp[1023];
            errP = t_scan * 0x1p-46;
            need_scan = false;
            STAMP(3);
        }
        const double T = s_cp[1023];
        if (!(T > 0.0)) break;  // all mass drawn: the reference breaks (total <= 0)
        if (tid < 32) {
            const double uni = uniforms[(size_t)row * w + k];
            const double eb = errP + static_cast<double>(v + 64) * 0x1p-53 * T;
            const double u_lo = __dmul_rd(uni, T - eb), u_hi = __dmul_ru(uni, T + eb);
            // first chunk with CP + eb > u_lo, first with CP - eb > u_hi (CP is non-decreasing)
            int c_lo = 1024, c_hi = 1024;
            for (int c0 = 0; c0 < 1024; c0 += 32) {
                const double cp = s_cp[c0 + lane];
                const unsigned bl = __ballot_sync(0xffffffffu, cp + eb > u_lo);
                const unsigned bh = __ballot_sync(0xffffffffu, cp - eb > u_hi);
                if (c_lo == 1024 && bl) c_lo = c0 + __ffs(bl) - 1;
                if (c_hi == 1024 && bh) c_hi = c0 + __ffs(bh) - 1;
                if (c_hi != 1024) break;
            }
            int pick = -1;
            if (c_lo == c_hi && c_hi < 1024) {  // inside chunk c: element prefixes base + warp scan
                const int c = c_lo, e0 = min(v, c * C), e1 = min(v, e0 + C);
                double base = c > 0 ? s_cp[c - 1] : 0.0;
                int i_lo = -1, i_hi = -1;
                for (int p0 = e0; p0 < e1 && i_hi < 0; p0 += 32) {
                    const int j = p0 + lane;
                    double x = j < e1 ? static_cast<double>(Wk[j]) : 0.0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const double y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    const double pj = base + x;
                    const unsigned bl = __ballot_sync(0xffffffffu, j < e1 && pj + eb > u_lo);
                    const unsigned bh = __ballot_sync(0xffffffffu, j < e1 && pj - eb > u_hi);
                    if (i_lo < 0 && bl) i_lo = p0 + __ffs(bl) - 1;
                    if (i_hi < 0 && bh) i_hi = p0 + __ffs(bh) - 1;
                    base += __shfl_sync(0xffffffffu, x, 31);
                }
                if (i_lo >= 0 && i_lo == i_hi) pick = i_lo;
            }
            if (lane == 0) {
                s_pick = pick;
                s_pchunk = c_lo;
                if (pick >= 0) {
                    out_ridx[(size_t)row * w + k] = pick;
                    out_full[(size_t)row * w + k] = ordered ? ordered[pick] : pick;
                    out_prob[(size_t)row * w + k] = P[pick];
                    Wk[pick] = 0.0f;
                }
            }
        }
        __syncthreads();
        if (s_pick < 0) {  // uncertain (or the reference's upper-edge guard): the host replays
            flags |= FRS_FLAG_SAMPLE_UNCERTIFIED;
            break;
        }
        ++count;
        // subtract the drawn mass from the prefixes at and after its chunk
        if (tid >= s_pchunk) s_cp[tid] -= static_cast<double>(P[s_pick]);
        errP += T * 0x1p-52;
        __syncthreads();
        need_scan = s_cp[1023] < 0.5 * t_scan;
        STAMP(4 + k);
    }
    if (tid == 0) {
        out_count[row] = count;
        if (out_flags) out_flags[row] = flags;
    }
}


int main(int argc, char **argv) {
    const int n = 10, v = 32768, w = 10;
    std::vector<float> h((size_t)n * v);
    srand(1);
    for (auto &x : h) { float s = 0; for (int i = 0; i < 12; ++i) s += (rand() & 0xffff) / 65536.0f; x = (s - 6.0f) * 1.28f; }
    std::vector<double> u(n * w);
    for (auto &x : u) x = (rand() & 0xffffff) / 16777216.0;
    float *L, *P, *Wk, *prob; int32_t *ridx, *full, *cnt; uint32_t *fl; double *ud; unsigned long long *st;
    cudaMalloc(&L, h.size() * 4); cudaMalloc(&P, h.size() * 4); cudaMalloc(&Wk, h.size() * 4);
    cudaMalloc(&prob, n * w * 4); cudaMalloc(&ridx, n * w * 4); cudaMalloc(&full, n * w * 4);
    cudaMalloc(&cnt, n * 4); cudaMalloc(&fl, n * 4); cudaMalloc(&ud, n * w * 8); cudaMalloc(&st, 64 * 8);
    cudaMemcpy(L, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ud, u.data(), u.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_sample_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, v * 4);
    for (int it = 0; it < 3; ++it)
        k_sample_probe<<<n, 1024, v * 4>>>(st, L, v, 1.0f, ud, w, nullptr, P, Wk, ridx, full, prob, cnt, fl, 1);
    cudaDeviceSynchronize();
    unsigned long long s[16];
    cudaMemcpy(s, st, sizeof(s), cudaMemcpyDeviceToHost);
    printf("softmax %.1f  copy %.1f  scan %.1f  draws:", (s[1] - s[0]) / 1e3, (s[2] - s[1]) / 1e3, (s[3] - s[2]) / 1e3);
    unsigned long long prev = s[3];
    for (int k = 0; k < w; ++k) { printf(" %.1f", (s[4 + k] - prev) / 1e3); prev = s[4 + k]; }
    printf("  total %.1f us  (%s)\n", (s[4 + w - 1] - s[0]) / 1e3, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
