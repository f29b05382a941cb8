// FP64 tensor-core (mma.sync m8n8k4 f64) throughput probe on the current GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[4][2] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    for (int warps = 4; warps <= 32; warps *= 2) {
        dmma_loop<<<sms * 4, warps * 32 / 4>>>(out, 16);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        dmma_loop<<<sms * 4, warps * 32 / 4>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma = (double)sms * 4 * (warps / 4) * iters * 4 * 256;
        printf("warps/SM %2d: %.1f TFLOP/s (mma.sync m8n8k4 f64)\n", warps, 2 * fma / (ms * 1e-3) / 1e12);
    }
    return 0;
}
