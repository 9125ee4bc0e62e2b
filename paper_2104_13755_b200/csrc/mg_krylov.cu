// libmg multigrid-preconditioned conjugate gradients ("use our
// multigrid solver as the pre-conditioner for ... the conjugate gradient
// method", §8).  Textbook PCG, every right-hand-side column
// independently, with z = M^{-1} r one symmetric V-cycle from a zero guess.
// One PCG iteration = [prep: b0 <- r, x0 <- 0] -> V-cycle body -> these
// kernels, all captured into one CUDA graph per K:
//   k_dot_partial(r, z) -> k_pcg_beta        rz = (r, z); beta = rz / rz_old (0 first)
//   k_pcg_p                                  p = z + beta p
//   k_spmv_dot                               q = A p, partial (p, q)
//   k_pcg_alpha                              alpha = rz / (p, q)
//   k_pcg_update                             x += alpha p, r -= alpha q, partial |r|^2
//   k_norm_finalize (mg_vcycle.cu)           rho = |r| / |b|
// Vectors use the internal layout [n][VS<K>::S] (pad lanes stay 0).  Every
// reduction is block partials + one fixed-order single-block finalisation:
// deterministic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mg_common.cuh"
#include "mg_internal.h"

namespace mg {
namespace {

constexpr int kDotBlocks = 1184;   // 8 x 148 SMs

template <int K>
__device__ __forceinline__ void block_partial_k(double (&acc)[K], double* partial) {
    __shared__ double red[kBlock / 32][K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const double v = warp_sum(acc[c]);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) v += red[w][threadIdx.x];
        partial[blockIdx.x * K + threadIdx.x] = v;
    }
}

// sum of the block partials per column, by one block in a fixed order
template <int K>
__device__ __forceinline__ void finalize_sum(const double* __restrict__ partial, int nb, double (&out)[K]) {
    __shared__ double red[kBlock / 32][K];
    __shared__ double res[K];
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int t = threadIdx.x; t < nb; t += kBlock)
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] += partial[t * K + c];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        const double v = warp_sum(acc[c]);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) v += red[w][threadIdx.x];
        res[threadIdx.x] = v;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < K; ++c) out[c] = res[c];
}

// b0 <- r (the preconditioner's right-hand side), x0 <- 0
template <int K>
__global__ void __launch_bounds__(kBlock) k_pcg_prep(const double* __restrict__ r, double* __restrict__ b0,
                                                     double* __restrict__ x0, int n) {
    pdl_launch_dependents();
    pdl_wait();
    const size_t tot = (size_t)n * VS<K>::S;
    for (size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x; t < tot; t += (size_t)gridDim.x * kBlock) {
        b0[t] = r[t];
        x0[t] = 0.0;
    }
}

// partial (u, v) per column
template <int K>
__global__ void __launch_bounds__(kBlock) k_dot_partial(const double* __restrict__ u, const double* __restrict__ v,
                                                        int n, double* __restrict__ partial) {
    pdl_launch_dependents();
    pdl_wait();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        double a[K], b[K];
        ldrow<K>(u + (size_t)i * VS<K>::S, a);
        ldrow<K>(v + (size_t)i * VS<K>::S, b);
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(a[c], b[c], acc[c]);
    }
    block_partial_k<K>(acc, partial);
}

// sc layout: [0,K) rz  [K,2K) beta  [2K,3K) alpha;  first: 1 before the first iteration
template <int K>
__global__ void __launch_bounds__(kBlock) k_pcg_beta(const double* __restrict__ partial, int nb,
                                                     double* __restrict__ sc, int* __restrict__ first) {
    pdl_launch_dependents();
    pdl_wait();
    double rz[K];
    finalize_sum<K>(partial, nb, rz);
    if (threadIdx.x == 0) {
        const bool f = *first != 0;
#pragma unroll
        for (int c = 0; c < K; ++c) {
            sc[K + c] = (f || sc[c] == 0.0) ? 0.0 : rz[c] / sc[c];   // reading A27
            sc[c] = rz[c];
        }
        *first = 0;
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_pcg_p(const double* __restrict__ z, double* __restrict__ p,
                                                  const double* __restrict__ sc, int n) {
    pdl_launch_dependents();
    pdl_wait();
    double beta[K];
#pragma unroll
    for (int c = 0; c < K; ++c) beta[c] = sc[K + c];
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        double zv[K], pv[K];
        ldrow<K>(z + (size_t)i * VS<K>::S, zv);
        ldrow<K>(p + (size_t)i * VS<K>::S, pv);
#pragma unroll
        for (int c = 0; c < K; ++c) pv[c] = fma(beta[c], pv[c], zv[c]);
        strow<K>(p + (size_t)i * VS<K>::S, pv);
    }
}

// q = A p (8 lanes per row), partial (p, q)
constexpr int kSpmvG = 8;
template <int K>
__global__ void __launch_bounds__(kBlock) k_spmv_dot(const int* __restrict__ rp, const int* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ p,
                                                     double* __restrict__ q, int n, double* __restrict__ partial) {
    pdl_launch_dependents();
    pdl_wait();
    const int lane = threadIdx.x & (kSpmvG - 1);
    const unsigned mask = group_mask(kSpmvG);
    const int groups = gridDim.x * (kBlock / kSpmvG);
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int base = 0; base < n; base += groups) {   // whole groups iterate together
        const int row = base + (blockIdx.x * kBlock + threadIdx.x) / kSpmvG;
        double s[K];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = 0.0;
        if (row < n) {
            for (int e = rp[row] + lane; e < rp[row + 1]; e += kSpmvG) {
                const int j = __ldg(col + e);
                const double a = __ldg(val + e);
                double pv[K];
                ldrow<K>(p + (size_t)j * VS<K>::S, pv);
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a, pv[c], s[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = group_sum<kSpmvG>(s[c], mask);
        if (row < n && lane == 0) {
            double pr[K];
            ldrow<K>(p + (size_t)row * VS<K>::S, pr);
            strow<K>(q + (size_t)row * VS<K>::S, s);
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = fma(pr[c], s[c], acc[c]);
        }
    }
    block_partial_k<K>(acc, partial);
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_pcg_alpha(const double* __restrict__ partial, int nb,
                                                      double* __restrict__ sc) {
    pdl_launch_dependents();
    pdl_wait();
    double pq[K];
    finalize_sum<K>(partial, nb, pq);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < K; ++c) sc[2 * K + c] = pq[c] == 0.0 ? 0.0 : sc[c] / pq[c];   // reading A27: solved column
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_pcg_update(double* __restrict__ x, double* __restrict__ r,
                                                       const double* __restrict__ p, const double* __restrict__ q,
                                                       const double* __restrict__ sc, int n,
                                                       double* __restrict__ partial) {
    pdl_launch_dependents();
    pdl_wait();
    double alpha[K], acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        alpha[c] = sc[2 * K + c];
        acc[c] = 0.0;
    }
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        double xv[K], rv[K], pv[K], qv[K];
        ldrow<K>(x + (size_t)i * VS<K>::S, xv);
        ldrow<K>(r + (size_t)i * VS<K>::S, rv);
        ldrow<K>(p + (size_t)i * VS<K>::S, pv);
        ldrow<K>(q + (size_t)i * VS<K>::S, qv);
#pragma unroll
        for (int c = 0; c < K; ++c) {
            xv[c] = fma(alpha[c], pv[c], xv[c]);
            rv[c] = fma(-alpha[c], qv[c], rv[c]);
            acc[c] = fma(rv[c], rv[c], acc[c]);
        }
        strow<K>(x + (size_t)i * VS<K>::S, xv);
        strow<K>(r + (size_t)i * VS<K>::S, rv);
    }
    block_partial_k<K>(acc, partial);
}

#define MG_KS(K, EXPR)                                    \
    switch (K) {                                          \
        case 1: { constexpr int KK = 1; EXPR; } break;   \
        case 2: { constexpr int KK = 2; EXPR; } break;   \
        case 3: { constexpr int KK = 3; EXPR; } break;   \
        default: { constexpr int KK = 4; EXPR; } break;  \
    }

inline int grid_for(int n) { return std::max(1, std::min(kDotBlocks, nblk(n, kBlock))); }

}  // namespace

int pcg_blocks() { return kDotBlocks; }

int pcg_prep(int K, const double* r, double* b0, double* x0, int n, bool pdl, cudaStream_t s) {
    MG_KS(K, (launch_k(pdl, k_pcg_prep<KK>, grid_for(n), kBlock, 0, s, r, b0, x0, n)));
    return 1;
}

int pcg_direction(int K, const double* r, const double* z, double* p, int n, double* partial, double* sc, int* first,
                  bool pdl, cudaStream_t s) {
    const int g = grid_for(n);
    MG_KS(K, (launch_k(pdl, k_dot_partial<KK>, g, kBlock, 0, s, r, z, n, partial),
              launch_k(pdl, k_pcg_beta<KK>, 1, kBlock, 0, s, (const double*)partial, g, sc, first),
              launch_k(pdl, k_pcg_p<KK>, g, kBlock, 0, s, z, p, (const double*)sc, n)));
    return 3;
}

int pcg_step(int K, const Level& L0, double* x, double* r, const double* p, double* q, double* partial, double* sc,
             bool pdl, cudaStream_t s) {
    const int n = L0.n;
    const int g = grid_for(n);
    const int gs = std::max(1, std::min(kDotBlocks, nblk((int64_t)n * kSpmvG, kBlock)));
    MG_KS(K, (launch_k(pdl, k_spmv_dot<KK>, gs, kBlock, 0, s, L0.rp.p, L0.col.p, L0.val.p, p, q, n, partial),
              launch_k(pdl, k_pcg_alpha<KK>, 1, kBlock, 0, s, (const double*)partial, gs, sc),
              launch_k(pdl, k_pcg_update<KK>, g, kBlock, 0, s, x, r, p, (const double*)q, (const double*)sc, n,
                       partial)));
    return 3;
}

int pcg_update_blocks(int n) { return grid_for(n); }

}  // namespace mg
