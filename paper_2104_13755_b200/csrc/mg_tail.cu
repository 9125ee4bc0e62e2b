// libmg "coarse tail": the part of the V-cycle on the small levels
// (Alg. 2, for levels lt..H) in ONE launch of one thread-block
// cluster (16 CTAs x 1024 threads when the device allows the non-portable
// size, else 8).  Every dependent phase (one colour class of the multicolour
// Gauss-Seidel sweep, residual, restriction, coarsest solve, prolongation)
// is separated by barrier.cluster (release/acquire at cluster scope) instead
// of a kernel boundary: on the small levels the ~2.5 us per dependent launch
// dominated, while one barrier costs a few hundred cycles.  Data produced
// inside the tail (x, b, r) is read with ld.global.cg (L2), so no stale L1
// line can be observed across CTAs.  Same arithmetic as the per-launch
// kernels of mg_vcycle.cu, row by row.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mg_common.cuh"
#include "mg_internal.h"

namespace mg {
namespace {

constexpr int kTailThreads = 1024;
constexpr int kTailLPR = 8;

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n"
        "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// MODE 0: GS rows [r0,r1); MODE 1: residual rows [r0,r1) into L.r
template <int K, int MODE>
__device__ __forceinline__ void tail_sweep(const TailLevel& L, int r0, int r1, int gtid, int nthreads) {
    constexpr int G = kTailLPR;
    const int lane = gtid & (G - 1);
    const int ngroups = nthreads / G;
    const unsigned mask = group_mask(G);
    for (int row = r0 + gtid / G; row < r1; row += ngroups) {
        const int e0 = L.rp[row], e1 = L.rp[row + 1];
        double s[K];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = 0.0;
        double d = 0.0;
#pragma unroll 2
        for (int e = e0 + lane; e < e1; e += G) {
            const int j = __ldg(L.col + e);
            const double a = __ldg(L.val + e);
            if (MODE == 0 && j == row) {
                d += a;
            } else {
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a, __ldcg(L.x + (size_t)j * VS<K>::S + c), s[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = group_sum<G>(s[c], mask);
        if (MODE == 0) d = group_sum<G>(d, mask);
        if (lane == 0) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double bv = __ldcg(L.b + (size_t)row * VS<K>::S + c);
                if (MODE == 0) L.x[(size_t)row * VS<K>::S + c] = (bv - s[c]) / d;
                else L.r[(size_t)row * VS<K>::S + c] = bv - s[c];
            }
        }
    }
}

// coarse.b = P^T fine.r (children lists), coarse.x = 0
template <int K>
__device__ __forceinline__ void tail_restrict(const TailLevel& F, const TailLevel& C, int gtid, int nthreads) {
    constexpr int G = kTailLPR;
    const int lane = gtid & (G - 1);
    const int ngroups = nthreads / G;
    const unsigned mask = group_mask(G);
    for (int I = gtid / G; I < C.n; I += ngroups) {
        double s[K];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = 0.0;
        for (int t = C.cptr[I] + lane; t < C.cptr[I + 1]; t += G) {
            const int i = __ldg(C.cidx + t);
            const double w = __ldg(C.cw + t);
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = fma(w, __ldcg(F.r + (size_t)i * VS<K>::S + c), s[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = group_sum<G>(s[c], mask);
        if (lane == 0) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
                C.b[(size_t)I * VS<K>::S + c] = s[c];
                C.x[(size_t)I * VS<K>::S + c] = 0.0;
            }
        }
    }
}

// fine.x += P coarse.x
template <int K>
__device__ __forceinline__ void tail_prolong(const TailLevel& F, const TailLevel& C, int gtid, int nthreads) {
    const int n = F.n;
    for (int i = gtid; i < n; i += nthreads) {
        const int c0 = __ldg(F.pc + i), c1 = __ldg(F.pc + n + i), c2 = __ldg(F.pc + 2 * n + i);
        const double w0 = __ldg(F.pw + i), w1 = __ldg(F.pw + n + i), w2 = __ldg(F.pw + 2 * n + i);
#pragma unroll
        for (int c = 0; c < K; ++c) {
            double v = w0 * __ldcg(C.x + (size_t)c0 * VS<K>::S + c);
            v = fma(w1, __ldcg(C.x + (size_t)c1 * VS<K>::S + c), v);
            v = fma(w2, __ldcg(C.x + (size_t)c2 * VS<K>::S + c), v);
            F.x[(size_t)i * VS<K>::S + c] = __ldcg(F.x + (size_t)i * VS<K>::S + c) + v;
        }
    }
}

// coarsest: x = Z b, one warp per row of the explicit inverse
template <int K>
__device__ __forceinline__ void tail_coarse(const TailLevel& H, const double* __restrict__ Z, int npad, int gtid,
                                            int nthreads) {
    const int lane = gtid & 31;
    const int nwarps = nthreads / 32;
    for (int row = gtid / 32; row < H.n; row += nwarps) {
        const double* Zr = Z + (size_t)row * npad;
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = 0.0;
        for (int j = lane; j < H.n; j += 32) {
            const double z = __ldg(Zr + j);
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = fma(z, __ldcg(H.b + (size_t)j * VS<K>::S + c), acc[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = warp_sum(acc[c]);
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < K; ++c) H.x[(size_t)row * VS<K>::S + c] = acc[c];
    }
}

template <int K>
__global__ void __launch_bounds__(kTailThreads, 1) k_tail(const TailParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const int nthreads = (int)cluster_nctarank() * kTailThreads;
    const int gtid = (int)cluster_ctarank() * kTailThreads + threadIdx.x;
    const int last = p.nl - 1;
    for (int li = 0; li < last; ++li) {
        const TailLevel& L = p.lv[li];
        for (int it = 0; it < p.mu_pre; ++it)
            for (int c = 0; c < L.ncol; ++c) {
                tail_sweep<K, 0>(L, __ldg(L.coff + c), __ldg(L.coff + c + 1), gtid, nthreads);
                cluster_sync_all();
            }
        tail_sweep<K, 1>(L, 0, L.n, gtid, nthreads);
        cluster_sync_all();
        tail_restrict<K>(L, p.lv[li + 1], gtid, nthreads);
        cluster_sync_all();
    }
    tail_coarse<K>(p.lv[last], p.Z, p.npad, gtid, nthreads);
    cluster_sync_all();
    for (int li = last - 1; li >= 0; --li) {
        const TailLevel& L = p.lv[li];
        tail_prolong<K>(L, p.lv[li + 1], gtid, nthreads);
        cluster_sync_all();
        for (int it = 0; it < p.mu_post; ++it)
            for (int c = 0; c < L.ncol; ++c) {
                tail_sweep<K, 0>(L, __ldg(L.coff + c), __ldg(L.coff + c + 1), gtid, nthreads);
                cluster_sync_all();
            }
    }
}

template <int K>
cudaError_t launch_tail_k(const TailParams& p, int cs, bool pdl, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kTailThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_tail<K>, p);
}

template <int K>
int max_cluster_k() {
    cudaFuncSetAttribute(k_tail<K>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {16, 8, 4, 2, 1}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kTailThreads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, k_tail<K>, &cfg) == cudaSuccess && nclusters >= 1) return cs;
        cudaGetLastError();
    }
    return 0;
}

}  // namespace

int tail_cluster_size() {
    static int cs = -1;
    if (cs < 0) {
        cs = max_cluster_k<1>();
        cs = std::min(cs, max_cluster_k<2>());
        cs = std::min(cs, max_cluster_k<3>());
        cs = std::min(cs, max_cluster_k<4>());
    }
    return cs;
}

int vc_tail(int K, const TailParams& p, int cs, bool pdl, cudaStream_t s) {
    cudaError_t e;
    switch (K) {
        case 1: e = launch_tail_k<1>(p, cs, pdl, s); break;
        case 2: e = launch_tail_k<2>(p, cs, pdl, s); break;
        case 3: e = launch_tail_k<3>(p, cs, pdl, s); break;
        default: e = launch_tail_k<4>(p, cs, pdl, s); break;
    }
    return e == cudaSuccess ? 1 : -1;
}

}  // namespace mg
