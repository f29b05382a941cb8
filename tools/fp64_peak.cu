// FP64 pipe microbenchmark: independent DFMA / DADD chains, 148 x k CTAs.  Prints G instr/s.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = OP == 0 ? fma(x[i], a, b) : (OP == 1 ? __dadd_rn(x[i], b) : __dmul_rn(x[i], a));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;
}
int main() {
    double *d; cudaMalloc(&d, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int op = 0; op < 3; ++op) for (int bl : {2, 4, 8}) {
        const int blocks = 148 * bl, threads = 256;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
            if (op == 1) k<1><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
            if (op == 2) k<2><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double inst = (double)blocks * threads * iters * 8;
            if (rep) printf("op=%s ctas/SM=%d: %.2f T thread-instr/s\n", op == 0 ? "DFMA" : op == 1 ? "DADD" : "DMUL", bl, inst / ms / 1e9);
        }
    }
    return 0;
}
