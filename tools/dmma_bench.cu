// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[16];
    for (int j = 0; j < 16; ++j) c[j] = j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) c[j] = fma(a, c[j], b);
    }
    double s = 0.0;
    for (int j = 0; j < 16; ++j) s += c[j];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        k_dmma<<<sms, 32 * warps>>>(out, 16);
        cudaEventRecord(e0);
        k_dmma<<<sms, 32 * warps>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 256 * 8 * (double)iters * warps * sms;
        printf("dmma warps/SM=%d  %.1f TFLOP/s\n", warps, fl / ms / 1e9);
        k_dfma<<<sms, 32 * warps>>>(out, 16);
        cudaEventRecord(e0);
        k_dfma<<<sms, 32 * warps>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl2 = 2.0 * 16 * 32 * (double)iters * warps * sms;
        printf("dfma warps/SM=%d  %.1f TFLOP/s\n", warps, fl2 / ms / 1e9);
    }
    return 0;
}
