// Host->device copy bandwidth (pinned, fp64 vs fp32 bytes) and host fp64->fp32 conversion rate.
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
using clk = std::chrono::steady_clock;
int main() {
    const size_t n = 7ull << 20;  // 1M rows x 7
    double* h64; float* h32; void* d;
    cudaMallocHost(&h64, n * 8);
    cudaMallocHost(&h32, n * 4);
    cudaMalloc(&d, n * 8);
    for (size_t i = 0; i < n; ++i) h64[i] = 0.001 * (i % 1000);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0, s); cudaMemcpyAsync(d, h64, n * 8, cudaMemcpyHostToDevice, s); cudaEventRecord(e1, s);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("H2D %zu MB: %.3f ms = %.1f GB/s\n", n * 8 >> 20, ms, n * 8 / ms / 1e6);
        cudaEventRecord(e0, s); cudaMemcpyAsync(d, h32, n * 4, cudaMemcpyHostToDevice, s); cudaEventRecord(e1, s);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("H2D %zu MB: %.3f ms = %.1f GB/s\n", n * 4 >> 20, ms, n * 4 / ms / 1e6);
    }
    printf("hardware threads: %u\n", std::thread::hardware_concurrency());
    for (int T : {1, 2, 4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            auto t0 = clk::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([=] {
                    const size_t a = n * t / T, b = n * (t + 1) / T;
                    for (size_t i = a; i < b; ++i) h32[i] = static_cast<float>(h64[i]);
                });
            for (auto& x : th) x.join();
            double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
            if (rep) printf("convert T=%d: %.3f ms (%.1f GB/s read)\n", T, ms, n * 8 / ms / 1e6);
        }
    }
}
