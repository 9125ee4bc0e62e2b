#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, 1.0); x1 = fma(x1, a, 1.0); x2 = fma(x2, a, 1.0); x3 = fma(x3, a, 1.0);
        x4 = fma(x4, a, 1.0); x5 = fma(x5, a, 1.0); x6 = fma(x6, a, 1.0); x7 = fma(x7, a, 1.0);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void kdep(double* out, int iters, double a) {
    double x0 = threadIdx.x;
    for (int i = 0; i < iters; ++i) x0 = fma(x0, a, 1.0);
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
__global__ void ksqrt(double* out, int iters) {
    double x0 = threadIdx.x + 2.0;
    for (int i = 0; i < iters; ++i) x0 = sqrt(x0) + 1.5;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
__global__ void kdiv(double* out, int iters) {
    double x0 = threadIdx.x + 2.0;
    for (int i = 0; i < iters; ++i) x0 = 3.0 / x0 + 1.0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
int main() {
    double* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    int it = 1 << 14;
    k<<<148 * 8, 256>>>(o, 16, 0.999); cudaDeviceSynchronize();
    cudaEventRecord(a); k<<<148 * 8, 256>>>(o, it, 0.999); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("fp64 FMA throughput: %.2f TFLOP/s\n", 2.0 * 8 * it * 148 * 8 * 256 / (ms * 1e-3) / 1e12);
    cudaEventRecord(a); kdep<<<1, 32>>>(o, it, 0.999); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent DFMA latency: %.1f ns (%.1f cycles at 1.965 GHz)\n", ms * 1e6 / it, ms * 1e6 / it * 1.965);
    cudaEventRecord(a); ksqrt<<<1, 32>>>(o, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent fp64 sqrt+add: %.1f ns\n", ms * 1e6 / 4096);
    cudaEventRecord(a); kdiv<<<1, 32>>>(o, 4096); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent fp64 div+add: %.1f ns\n", ms * 1e6 / 4096);
    return 0;
}
