// ez_peak.cu — FP32 FMA throughput microbenchmark: the roofline denominator of
// the checker (FP32-FMA bound); MEASURED_PEAKS.json carries
// only HBM and bf16 tensor peaks.
#include "ez_common.h"

namespace ez {

__global__ void __launch_bounds__(256) k_fma_peak(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[blockIdx.x] = s;  // keep the chain alive
}

// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput: the roofline
// denominator of the hit-and-run walk, whose chord data is a DMMA GEMM.
__global__ void __launch_bounds__(512) k_dmma_peak(double* out, int iters) {
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.0) out[blockIdx.x] = s;
}

}  // namespace ez

extern "C" int32_t ez_fp64_tc_peak(int32_t device, double* tflops, double* ms_out) {
    using namespace ez;
    EZ_ON_DEVICE(device);
    int sms = 0;
    EZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    EZ_CUDA(cudaMalloc(&d, 4096 * sizeof(double)));
    cudaEvent_t e0, e1;
    EZ_CUDA(cudaEventCreate(&e0));
    EZ_CUDA(cudaEventCreate(&e1));
    const int blocks = sms, threads = 512, iters = 2048;
    k_dmma_peak<<<blocks, threads>>>(d, 16);  // warm-up
    EZ_CUDA(cudaEventRecord(e0));
    k_dmma_peak<<<blocks, threads>>>(d, iters);
    EZ_CUDA(cudaEventRecord(e1));
    EZ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    EZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // 8x8x4 FMA = 512 FLOP per warp-MMA
    const double flops = 512.0 * 8 * static_cast<double>(iters) * blocks * (threads / 32);
    *tflops = flops / (ms * 1e-3) / 1e12;
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return EZ_OK;
}

extern "C" int32_t ez_fp32_peak(int32_t device, double* tflops, double* ms_out) {
    using namespace ez;
    EZ_ON_DEVICE(device);
    int sms = 0;
    EZ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    float* d = nullptr;
    EZ_CUDA(cudaMalloc(&d, 4096 * sizeof(float)));
    cudaEvent_t e0, e1;
    EZ_CUDA(cudaEventCreate(&e0));
    EZ_CUDA(cudaEventCreate(&e1));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_fma_peak<<<blocks, threads>>>(d, 64, 0.999f, 1e-3f);  // warm-up
    EZ_CUDA(cudaEventRecord(e0));
    k_fma_peak<<<blocks, threads>>>(d, iters, 0.999f, 1e-3f);
    EZ_CUDA(cudaEventRecord(e1));
    EZ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    EZ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * blocks * threads;
    *tflops = flops / (ms * 1e-3) / 1e12;
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return EZ_OK;
}
