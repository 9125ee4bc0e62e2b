// Microbenchmark: cost of one colour step of a cluster-resident GS smoother on
// B200 (one 16-CTA cluster, clock64 per phase, CTA 0 thread 0 reports):
//   mode 0: barrier.cluster only
//   mode 1: + DSMEM pushes (PUSH rows x K doubles to 4 neighbour CTAs)
//   mode 2: + row compute from shared memory (ROWS rows / CTA, NNZ entries,
//           LPR lanes per row, fp64 division)
//   mode 3: mode 2 with reciprocal multiply instead of division
//   mode 4: mode 2 with a multiply by a constant (no division at all)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_step_bench tools/cluster_step_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned crank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned mapa(const void* p, unsigned cta) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(cta));
    return r;
}
__device__ __forceinline__ void st_remote(unsigned addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}

template <int LPR, int MODE>
__global__ void __launch_bounds__(512, 1) kbench(int steps, int rows, int nnz, int push, double* out) {
    constexpr int K = 3;
    __shared__ double xs[1000 * K];
    __shared__ double vs[2048];
    __shared__ unsigned short ls[2048];
    __shared__ int rps[65];
    const int tid = threadIdx.x, p = crank(), cs = gridDim.x;
    for (int i = tid; i < 1000 * K; i += blockDim.x) xs[i] = 1.0 + (i % 7) * 0.01;
    for (int i = tid; i < 2048; i += blockDim.x) {
        vs[i] = (i % 5 == 0) ? 4.0 : -0.1;
        ls[i] = (unsigned short)((i * 37) % 1000);
    }
    for (int i = tid; i <= rows; i += blockDim.x) rps[i] = i * nnz;
    __syncthreads();
    csync();
    unsigned long long t0 = clock64(), tc = 0, tp = 0, tb = 0;
    const int grp = tid / LPR, lane = tid % LPR, ngrp = blockDim.x / LPR;
    for (int s = 0; s < steps; ++s) {
        unsigned long long a = clock64();
        if (MODE >= 2) {
            for (int r = grp; r < rows; r += ngrp) {
                const int li = r;
                double sacc[K] = {0, 0, 0}, d = 0.0;
                for (int q = rps[r] + lane; q < rps[r + 1]; q += LPR) {
                    const int j = ls[q];
                    const double av = vs[q];
                    if (q == rps[r]) d += av;
                    else
#pragma unroll
                        for (int k = 0; k < K; ++k) sacc[k] = fma(av, xs[j * K + k], sacc[k]);
                }
#pragma unroll
                for (int off = LPR / 2; off > 0; off >>= 1) {
#pragma unroll
                    for (int k = 0; k < K; ++k) sacc[k] += __shfl_xor_sync(0xffffffffu, sacc[k], off, LPR);
                    d += __shfl_xor_sync(0xffffffffu, d, off, LPR);
                }
                if (lane == 0) {
                    if (MODE == 4) {
#pragma unroll
                        for (int k = 0; k < K; ++k) xs[li * K + k] = (1.0 - sacc[k]) * 0.25;
                    } else if (MODE == 3) {
                        const double id = 1.0 / d;
#pragma unroll
                        for (int k = 0; k < K; ++k) xs[li * K + k] = (1.0 - sacc[k]) * id;
                    } else {
#pragma unroll
                        for (int k = 0; k < K; ++k) xs[li * K + k] = (1.0 - sacc[k]) / d;
                    }
                }
            }
            __syncthreads();
        }
        unsigned long long b = clock64();
        if (MODE >= 1) {
            for (int q = tid; q < push; q += blockDim.x) {
                const unsigned dst = (p + 1 + (q & 3)) % cs;
                const unsigned ra = mapa(xs + (size_t)(q % 1000) * K, dst);
#pragma unroll
                for (int k = 0; k < K; ++k) st_remote(ra + 8u * k, xs[(q % 1000) * K + k]);
            }
        }
        unsigned long long c = clock64();
        csync();
        unsigned long long d2 = clock64();
        tc += b - a;
        tp += c - b;
        tb += d2 - c;
    }
    if (p == 0 && tid == 0) {
        out[0] = (double)(clock64() - t0) / steps;
        out[1] = (double)tc / steps;
        out[2] = (double)tp / steps;
        out[3] = (double)tb / steps;
    }
}

template <int LPR, int MODE>
void run(int rows, int nnz, int push, int threads) {
    double* d;
    cudaMalloc(&d, 64);
    auto kern = kbench<LPR, MODE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, 400, rows, nnz, push, d);
    cudaDeviceSynchronize();
    double h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("mode %d LPR %2d thr %d rows %4d nnz %2d push %4d: step %6.0f cyc = compute %6.0f + push %5.0f + barrier %5.0f  (%s)\n",
           MODE, LPR, threads, rows, nnz, push, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<32, 0>(0, 0, 0, 512);
    run<32, 1>(0, 0, 64, 512);
    run<32, 1>(0, 0, 512, 512);
    for (int rows : {8, 32, 64}) {
        run<32, 2>(rows, 30, 64, 512);
        run<32, 3>(rows, 30, 64, 512);
        run<32, 4>(rows, 30, 64, 512);
        run<8, 2>(rows, 30, 64, 512);
        run<8, 4>(rows, 30, 64, 512);
        run<4, 2>(rows, 30, 64, 512);
        run<4, 3>(rows, 30, 64, 512);
        run<4, 4>(rows, 30, 64, 512);
    }
    return 0;
}
