// DIAGNOSTIC: per-phase time of dev::softmax_topk_row (max / exp+sum / list build / pops) on
// n rows of v random logits, one CTA per row, %globaltimer stamps from thread 0 of row 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2502_14856_b200/csrc \
//      tools/softmax_probe.cu -o tools/softmax_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "frs_device.cuh"

using namespace frs;

__global__ void __launch_bounds__(1024) k_probe(const float *L, int v, int k, float *E, int32_t *ridx, int32_t *full,
                                                float *prob, unsigned long long *stamps) {
    __shared__ dev::ReduceScratch rs;
    const int row = blockIdx.x;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    dev::softmax_topk_row(L + (size_t)row * v, v, k, 1.0f, nullptr, E + (size_t)row * v, ridx + row * k,
                          full + row * k, prob + row * k, nullptr, nullptr, rs, true,
                          row == 0 ? stamps + 1 : nullptr);
    if (row == 0 && threadIdx.x == 0) stamps[0] = t0;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 10, v = argc > 2 ? atoi(argv[2]) : 32768, k = 10;
    std::vector<float> h((size_t)n * v);
    srand(1);
    for (auto &x : h) x = ((rand() & 0xffff) / 65536.0f - 0.5f) * 6.0f;
    float *L, *E, *prob;
    int32_t *ridx, *full;
    unsigned long long *st;
    cudaMalloc(&L, h.size() * 4);
    cudaMalloc(&E, h.size() * 4);
    cudaMalloc(&prob, n * k * 4);
    cudaMalloc(&ridx, n * k * 4);
    cudaMalloc(&full, n * k * 4);
    cudaMalloc(&st, 64 * 8);
    cudaMemcpy(L, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 5; ++it) k_probe<<<n, 1024>>>(L, v, k, E, ridx, full, prob, st);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) k_probe<<<n, 1024>>>(L, v, k, E, ridx, full, prob, st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long s[6];
    cudaMemcpy(s, st, sizeof(s), cudaMemcpyDeviceToHost);
    printf("kernel %.1f us | max %.1f  exp+sum %.1f  inv %.1f  lists %.1f  pops %.1f (us) | err %s\n",
           ms * 1000 / 20, (s[1] - s[0]) / 1e3, (s[2] - s[1]) / 1e3, (s[3] - s[2]) / 1e3, (s[4] - s[3]) / 1e3,
           (s[5] - s[4]) / 1e3, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
