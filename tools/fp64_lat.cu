// FP64 DADD throughput vs (warps per SM, independent chains per thread): how much parallelism
// the FP64 pipe needs on this part.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double *out, int iters, double b) {
    double x[ILP];
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dadd_rn(x[i], b);
    }
    double s = 0;
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
template <int ILP>
void run(double *d, int warps_per_sm) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 40000 / ILP * 8;
    const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32), blocks = 148 * (warps_per_sm * 32 / threads);
    k<ILP><<<blocks, threads>>>(d, iters, 1e-7);
    cudaEventRecord(e0);
    k<ILP><<<blocks, threads>>>(d, iters, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("warps/SM=%2d ILP=%d: %.2f T DADD/s\n", warps_per_sm, ILP, (double)blocks * threads * iters * ILP / ms / 1e9);
}
int main() {
    double *d; cudaMalloc(&d, 8);
    for (int w : {4, 8, 12, 16, 24, 32}) { run<1>(d, w); run<2>(d, w); run<4>(d, w); run<8>(d, w); }
    return 0;
}
