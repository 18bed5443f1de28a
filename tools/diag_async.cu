// Per-call cost of stream-ordered allocation vs plain launches (lazy vs eager module loading).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_touch(int* p) { if (p) p[threadIdx.x] = threadIdx.x; }
int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int* q;
    cudaMalloc(&q, 4096);
    for (int round = 0; round < 3; ++round) {
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 20; ++i) {
            k_touch<<<1, 32, 0, s>>>(q);
            cudaStreamSynchronize(s);
        }
        auto t1 = std::chrono::steady_clock::now();
        for (int i = 0; i < 20; ++i) {
            int* p;
            cudaMallocAsync(&p, 4096, s);
            k_touch<<<1, 32, 0, s>>>(p);
            cudaFreeAsync(p, s);
            cudaStreamSynchronize(s);
        }
        auto t2 = std::chrono::steady_clock::now();
        printf("launch+sync %.3f ms/call   mallocAsync+launch+free+sync %.3f ms/call\n",
               std::chrono::duration<double, std::milli>(t1 - t0).count() / 20,
               std::chrono::duration<double, std::milli>(t2 - t1).count() / 20);
    }
}
