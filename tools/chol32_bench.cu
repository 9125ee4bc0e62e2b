// Micro-benchmark (tools only): latency of the 32x32 diagonal-block Cholesky
// factor + triangular inverse variants used on the critical path of k_chol_grid.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void chol32_shfl(double (*S)[33]) {
    const int lane = threadIdx.x & 31;
    double a[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = S[lane][c];
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        double piv = __shfl_sync(0xffffffffu, a[p], p);
        piv = piv > 0.0 ? piv : 1.0;
        const double d = sqrt(piv);
        const double rd = 1.0 / d;
        a[p] = lane == p ? d : (lane > p ? a[p] * rd : a[p]);
        const double lp = a[p];
#pragma unroll
        for (int c = p + 1; c < 32; ++c) {
            const double lcp = __shfl_sync(0xffffffffu, lp, c);
            const double upd = fma(-lp, lcp, a[c]);
            a[c] = lane >= c ? upd : a[c];
        }
    }
    __syncthreads();
    if (threadIdx.x < 32)
#pragma unroll
        for (int c = 0; c < 32; ++c) S[lane][c] = a[c];
    __syncthreads();
}

// variant: no sqrt/div on the dependent path: rsqrt via MUFU + Newton, column scaled by multiplication
__device__ __forceinline__ void chol32_fast(double (*S)[33]) {
    const int lane = threadIdx.x & 31;
    double a[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = S[lane][c];
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        double piv = __shfl_sync(0xffffffffu, a[p], p);
        piv = piv > 0.0 ? piv : 1.0;
        double r = rsqrt(piv);                       // 1/sqrt
        r = r * (1.5 - 0.5 * piv * r * r);           // one Newton step
        const double d = piv * r;
        a[p] = lane == p ? d : (lane > p ? a[p] * r : a[p]);
        const double lp = a[p];
#pragma unroll
        for (int c = 1; c < 32; ++c) {
            if (c <= p) continue;
            const double lcp = __shfl_sync(0xffffffffu, lp, c);
            const double upd = fma(-lp, lcp, a[c]);
            a[c] = lane >= c ? upd : a[c];
        }
    }
    __syncthreads();
    if (threadIdx.x < 32)
#pragma unroll
        for (int c = 0; c < 32; ++c) S[lane][c] = a[c];
    __syncthreads();
}

// column broadcast through shared memory (one STS + 31 broadcast LDS per step)
__device__ __forceinline__ void chol32_smem(double (*S)[33], double* colb) {
    const int lane = threadIdx.x & 31;
    double a[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) a[c] = S[lane][c];
    __syncthreads();
    if (threadIdx.x < 32) {
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            if (lane == p) colb[32] = a[p];
            __syncwarp();
            double piv = colb[32];
            piv = piv > 0.0 ? piv : 1.0;
            const double d = sqrt(piv);
            const double rd = 1.0 / d;
            a[p] = lane == p ? d : (lane > p ? a[p] * rd : a[p]);
            colb[lane] = a[p];
            __syncwarp();
            const double lp = a[p];
#pragma unroll
            for (int c = p + 1; c < 32; ++c) {
                const double upd = fma(-lp, colb[c], a[c]);
                a[c] = lane >= c ? upd : a[c];
            }
            __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) S[lane][c] = a[c];
    }
    __syncthreads();
}

// triangular inverse with reciprocal diagonal and 4 independent partial sums
__device__ __forceinline__ void trinv32_ilp(const double (*S)[33], double (*Li)[33]) {
    const int lane = threadIdx.x;
    if (lane >= 32) return;
    double rdg[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) rdg[i] = 1.0 / S[i][i];
    double xv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int q = 0; q < i; ++q) {
            const double t = S[i][q] * xv[q];
            if ((q & 3) == 0) s0 -= t;
            else if ((q & 3) == 1) s1 -= t;
            else if ((q & 3) == 2) s2 -= t;
            else s3 -= t;
        }
        xv[i] = ((s0 + s1) + (s2 + s3)) * rdg[i];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Li[i][lane] = xv[i];
}

__device__ __forceinline__ void trinv32(const double (*S)[33], double (*Li)[33]) {
    const int lane = threadIdx.x;
    if (lane >= 32) return;
    double xv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        double sacc = (i == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < i; ++q) sacc = fma(-S[i][q], xv[q], sacc);
        xv[i] = sacc / S[i][i];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Li[i][lane] = xv[i];
}

__device__ __forceinline__ double rsqrt_nr(double x) {
    double r = (double)rsqrtf((float)x);
    r = r * fma(-0.5 * x, r * r, 1.5);
    r = r * fma(-0.5 * x, r * r, 1.5);
    return r;
}
// factor AND inverse on one warp, registers only: lane i holds row i of A
// (a[]) and column i of L^{-1} (xv[]); step p broadcasts column p of L by
// shuffles (c = p+1 first: the next pivot's update), which serves both the
// rank-1 update of the factor and the forward-substitution step p of the
// inverse (xv_c -= L_cp * xv_p).
__device__ __forceinline__ void chol32_fused(double (*S)[33], double (*Li)[33]) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        double a[32], xv[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            a[c] = S[lane][c];
            xv[c] = c == lane ? 1.0 : 0.0;
        }
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            double piv = __shfl_sync(0xffffffffu, a[p], p);
            piv = piv > 0.0 ? piv : 1.0;
            const double r = rsqrt_nr(piv);
            const double l = lane == p ? piv * r : a[p] * r;   // column p of L (rows > p valid)
            a[p] = lane >= p ? l : a[p];
            xv[p] *= r;
#pragma unroll
            for (int c = 1; c < 32; ++c) {
                if (c <= p) continue;
                const double lcp = __shfl_sync(0xffffffffu, l, c);   // L_cp
                const double upd = fma(-l, lcp, a[c]);
                a[c] = lane >= c ? upd : a[c];
                xv[c] = fma(-lcp, xv[p], xv[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            S[lane][c] = a[c];
            Li[c][lane] = xv[c];
        }
    }
    __syncthreads();
}

template <int V>
__global__ void kbench(const double* A, double* out, long long* cyc, int reps) {
    __shared__ double S[32][33], Li[32][33], colb[40];
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        for (int q = threadIdx.x; q < 1024; q += blockDim.x) S[q >> 5][q & 31] = A[q];
        __syncthreads();
        if (V == 0) chol32_shfl(S);
        if (V == 1) chol32_fast(S);
        if (V == 2) { chol32_shfl(S); trinv32(S, Li); __syncthreads(); }
        if (V == 3) chol32_smem(S, colb);
        if (V == 4) { trinv32_ilp(S, Li); __syncthreads(); }
        if (V == 5) { trinv32(S, Li); __syncthreads(); }
        if (V == 6) chol32_fused(S, Li);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[V] = (t1 - t0) / reps;
    for (int q = threadIdx.x; q < 1024; q += blockDim.x) out[q] = S[q >> 5][q & 31] + Li[q >> 5][q & 31];
}

int main() {
    double h[1024];
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
    double *A, *o;
    long long* c;
    cudaMalloc(&A, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
    cudaMemcpy(A, h, 8192, cudaMemcpyHostToDevice);
    for (int threads : {32, 256}) {
        kbench<0><<<1, threads>>>(A, o, c, 20);
        kbench<1><<<1, threads>>>(A, o, c, 20);
        kbench<2><<<1, threads>>>(A, o, c, 20);
        kbench<3><<<1, threads>>>(A, o, c, 20);
        kbench<4><<<1, threads>>>(A, o, c, 20);
        kbench<5><<<1, threads>>>(A, o, c, 20);
        kbench<6><<<1, threads>>>(A, o, c, 20);
        long long hc[7];
        cudaMemcpy(hc, c, 56, cudaMemcpyDeviceToHost);
        printf("threads %d: chol32 shfl %lld cyc, rsqrt %lld, shfl+trinv32 %lld, chol32 smem %lld, trinv32 ilp %lld, trinv32 %lld, fused factor+inverse %lld\n",
               threads, hc[0], hc[1], hc[2], hc[3], hc[4], hc[5], hc[6]);
    }
    return 0;
}
