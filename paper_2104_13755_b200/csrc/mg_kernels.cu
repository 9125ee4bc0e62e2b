// libmg device kernels for sm_100a: the hot path of the Galerkin surface
// multigrid of arXiv 2104.13755.  fp64 throughout; HBM-bandwidth bound
// (SpMV-class intensity ~0.17 flop/B), so no tensor cores.
//
// Kernel map (SURVEY.md §2.3 K-numbers, PAPER.md lines):
//   K1 k_cotan_assemble   cotan L + lumped M -> A = mM + lL
//   K2 k_galerkin         A_{l+1} = P^T A_l P on a fixed pattern          (Eq. gca)
//   K3 k_resnorm_*        rho = ||b - A x|| / ||b|| per column            (reading A3)
//   K4 k_gs_colour        one colour class of multicolour Gauss-Seidel    (App. A)
//   K5 k_residual+k_restrict   r = b - A x', r_c = P^T r                 (Alg. 2)
//   K6 k_prolong          x <- x' + P c                                   (Alg. 2, reading A1)
//   K7 k_chol_*           coarsest dense Cholesky factor / solve          (Alg. 2, reading A12)
//   K9 k_gather/scatter   user <-> internal (colour-grouped) ordering
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mg_internal.h"

namespace mg {
namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ unsigned group_mask(int lpr) {
    if (lpr >= 32) return 0xffffffffu;
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << lpr) - 1u) << (lane & ~(unsigned)(lpr - 1));
}

template <int LPR>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) v += __shfl_xor_sync(mask, v, off, LPR);
    return v;
}

// Streaming (read-once) loads of matrix data: keep them out of L1 and mark
// them evict-first in L2 (cache-policy operand) so the gathered vector x
// stays resident.
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// ---------------------------------------------------------------------------
// K4: multicolour Gauss-Seidel, one colour class [r0, r1) (rows of one colour
// are contiguous in the internal order and mutually independent, App. A
// P:821-823).  x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii for K columns.
// LPR lanes cooperate on one row.
template <int K, int LPR>
__global__ void __launch_bounds__(kBlock) k_gs_colour(const int* __restrict__ rp, const int* __restrict__ col,
                                                      const double* __restrict__ val, const double* __restrict__ b,
                                                      double* __restrict__ x, int r0, int r1) {
    const int g = (blockIdx.x * kBlock + threadIdx.x) / LPR;
    const int lane = threadIdx.x & (LPR - 1);
    const int row = r0 + g;
    if (row >= r1) return;   // whole LPR-groups leave together
    const unsigned mask = group_mask(LPR);
    const uint64_t pol = evict_first_policy();
    const int e0 = rp[row], e1 = rp[row + 1];
    double s[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    double d = 0.0;
    for (int e = e0 + lane; e < e1; e += LPR) {
        const int j = ld_stream(col + e, pol);
        const double a = ld_stream(val + e, pol);
        if (j == row) {
            d = a;
        } else {
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = fma(a, x[(size_t)j * K + c], s[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], mask);
    d = group_sum<LPR>(d, mask);
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < K; ++c) x[(size_t)row * K + c] = (b[(size_t)row * K + c] - s[c]) / d;
    }
}

// K5a: r = b - A x over all rows.
template <int K, int LPR>
__global__ void __launch_bounds__(kBlock) k_residual(const int* __restrict__ rp, const int* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ b,
                                                     const double* __restrict__ x, double* __restrict__ r, int n) {
    const int row = (blockIdx.x * kBlock + threadIdx.x) / LPR;
    const int lane = threadIdx.x & (LPR - 1);
    if (row >= n) return;
    const unsigned mask = group_mask(LPR);
    const uint64_t pol = evict_first_policy();
    const int e0 = rp[row], e1 = rp[row + 1];
    double s[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    for (int e = e0 + lane; e < e1; e += LPR) {
        const int j = ld_stream(col + e, pol);
        const double a = ld_stream(val + e, pol);
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = fma(a, x[(size_t)j * K + c], s[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], mask);
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < K; ++c) r[(size_t)row * K + c] = b[(size_t)row * K + c] - s[c];
    }
}

// ---------------------------------------------------------------------------
// Tile-staged CSR kernels (used for every level whose tiles fit in shared
// memory).  A CTA owns a tile of kTile consecutive rows: the row pointers and
// the tile's contiguous run of (col, val) are staged into shared memory with
// fully coalesced streaming loads, then each thread processes one row from
// shared memory, issuing its x gathers in independent batches of UNR so the
// L2 latency of the gathers overlaps.  One HBM pass over A per sweep.
constexpr int kTile = 256;

__device__ __forceinline__ int tile_stage(const int* __restrict__ rp, const int* __restrict__ col,
                                          const double* __restrict__ val, int row0, int nrow, int* rps, int* cs,
                                          double* vs, uint64_t pol) {
    const int t = threadIdx.x;
    if (t < nrow) rps[t] = rp[row0 + t];
    if (t == 0) rps[nrow] = rp[row0 + nrow];
    __syncthreads();
    const int e0 = rps[0];
    const int cnt = rps[nrow] - e0;
    const int* cg = col + e0;
    const double* vg = val + e0;
    int q = t;
    for (; q + 3 * kTile < cnt; q += 4 * kTile) {
        const int c0 = ld_stream(cg + q, pol), c1 = ld_stream(cg + q + kTile, pol), c2 = ld_stream(cg + q + 2 * kTile, pol),
                  c3 = ld_stream(cg + q + 3 * kTile, pol);
        const double v0 = ld_stream(vg + q, pol), v1 = ld_stream(vg + q + kTile, pol), v2 = ld_stream(vg + q + 2 * kTile, pol),
                     v3 = ld_stream(vg + q + 3 * kTile, pol);
        cs[q] = c0;
        cs[q + kTile] = c1;
        cs[q + 2 * kTile] = c2;
        cs[q + 3 * kTile] = c3;
        vs[q] = v0;
        vs[q + kTile] = v1;
        vs[q + 2 * kTile] = v2;
        vs[q + 3 * kTile] = v3;
    }
    for (; q < cnt; q += kTile) {
        cs[q] = ld_stream(cg + q, pol);
        vs[q] = ld_stream(vg + q, pol);
    }
    __syncthreads();
    return e0;
}

// Row dot product from the staged tile: s[c] = sum_{j != row} a_rj x_jc, d = a_rr.
template <int K, int UNR>
__device__ __forceinline__ void tile_row(const int* cs, const double* vs, int qb, int qe, int row,
                                         const double* __restrict__ x, double (&s)[K], double& d) {
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    d = 0.0;
    for (int q = qb; q < qe; q += UNR) {
        int j[UNR];
        double a[UNR];
        double xv[UNR][K];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const bool ok = q + u < qe;
            j[u] = ok ? cs[q + u] : row;
            a[u] = ok ? vs[q + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int c = 0; c < K; ++c) xv[u][c] = x[(size_t)j[u] * K + c];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (j[u] == row) {
                d += a[u];
            } else {
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a[u], xv[u][c], s[c]);
            }
        }
    }
}

template <int K>
struct Unroll {
    static constexpr int value = K == 1 ? 8 : 4;
};

// K4 (tiled): one colour class [r0, r1), one tile per CTA.  Dynamic shared
// memory: cap doubles (values) then cap ints (columns), cap >= nnz of any tile.
template <int K>
__global__ void __launch_bounds__(kTile) k_gs_tiled(const int* __restrict__ rp, const int* __restrict__ col,
                                                    const double* __restrict__ val, const double* __restrict__ b,
                                                    double* __restrict__ x, int r0, int r1, int cap) {
    extern __shared__ double smem_d[];
    __shared__ int rps[kTile + 1];
    double* vs = smem_d;
    int* cs = reinterpret_cast<int*>(smem_d + cap);
    const uint64_t pol = evict_first_policy();
    const int row0 = r0 + blockIdx.x * kTile;
    const int nrow = min(kTile, r1 - row0);
    const int e0 = tile_stage(rp, col, val, row0, nrow, rps, cs, vs, pol);
    const int t = threadIdx.x;
    if (t >= nrow) return;
    const int row = row0 + t;
    double s[K], d;
    tile_row<K, Unroll<K>::value>(cs, vs, rps[t] - e0, rps[t + 1] - e0, row, x, s, d);
#pragma unroll
    for (int c = 0; c < K; ++c) x[(size_t)row * K + c] = (b[(size_t)row * K + c] - s[c]) / d;
}

// K5a (tiled): r = b - A x over all rows.
template <int K>
__global__ void __launch_bounds__(kTile) k_residual_tiled(const int* __restrict__ rp, const int* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ b, const double* __restrict__ x,
                                                          double* __restrict__ r, int n, int cap) {
    extern __shared__ double smem_d[];
    __shared__ int rps[kTile + 1];
    double* vs = smem_d;
    int* cs = reinterpret_cast<int*>(smem_d + cap);
    const uint64_t pol = evict_first_policy();
    const int row0 = blockIdx.x * kTile;
    const int nrow = min(kTile, n - row0);
    const int e0 = tile_stage(rp, col, val, row0, nrow, rps, cs, vs, pol);
    const int t = threadIdx.x;
    if (t >= nrow) return;
    const int row = row0 + t;
    double s[K], d;
    tile_row<K, Unroll<K>::value>(cs, vs, rps[t] - e0, rps[t + 1] - e0, row, x, s, d);
#pragma unroll
    for (int c = 0; c < K; ++c) r[(size_t)row * K + c] = b[(size_t)row * K + c] - fma(d, x[(size_t)row * K + c], s[c]);
}

// K3 (tiled, persistent): block partial sums of (b - A x)^2 per column.
template <int K>
__global__ void __launch_bounds__(kTile) k_resnorm_tiled(const int* __restrict__ rp, const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ b, const double* __restrict__ x,
                                                         double* __restrict__ partial, int n, int cap) {
    extern __shared__ double smem_d[];
    __shared__ int rps[kTile + 1];
    __shared__ double red[kTile / 32][K];
    double* vs = smem_d;
    int* cs = reinterpret_cast<int*>(smem_d + cap);
    const uint64_t pol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const int ntiles = (n + kTile - 1) / kTile;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row0 = tile * kTile;
        const int nrow = min(kTile, n - row0);
        const int e0 = tile_stage(rp, col, val, row0, nrow, rps, cs, vs, pol);
        const int t = threadIdx.x;
        if (t < nrow) {
            const int row = row0 + t;
            double s[K], d;
            tile_row<K, Unroll<K>::value>(cs, vs, rps[t] - e0, rps[t + 1] - e0, row, x, s, d);
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double rr = b[(size_t)row * K + c] - fma(d, x[(size_t)row * K + c], s[c]);
                acc[c] = fma(rr, rr, acc[c]);
            }
        }
        __syncthreads();   // smem reuse by the next tile
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double v = acc[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < kTile / 32; ++w) v += red[w][threadIdx.x];
        partial[blockIdx.x * K + threadIdx.x] = v;
    }
}

// K5b: r_c = P^T r, gathered through the transpose of P (children of each
// coarse vertex) so no atomics are needed and the result is deterministic.
// Also zeroes the coarse iterate: the recursive V-cycle starts from 0.
template <int K>
__global__ void __launch_bounds__(kBlock) k_restrict(const int* __restrict__ cptr, const int* __restrict__ cidx,
                                                     const double* __restrict__ cw, const double* __restrict__ r,
                                                     double* __restrict__ bc, double* __restrict__ xc, int nc) {
    const int I = blockIdx.x * kBlock + threadIdx.x;
    if (I >= nc) return;
    double s[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    for (int t = cptr[I]; t < cptr[I + 1]; ++t) {
        const int i = cidx[t];
        const double w = cw[t];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = fma(w, r[(size_t)i * K + c], s[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
        bc[(size_t)I * K + c] = s[c];
        xc[(size_t)I * K + c] = 0.0;
    }
}

// K6: x <- x + P c (ELL-3, SoA [3][n]).
template <int K>
__global__ void __launch_bounds__(kBlock) k_prolong(const int* __restrict__ pc, const double* __restrict__ pw,
                                                    const double* __restrict__ xc, double* __restrict__ x, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int c0 = pc[i], c1 = pc[n + i], c2 = pc[2 * n + i];
    const double w0 = pw[i], w1 = pw[n + i], w2 = pw[2 * n + i];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double v = w0 * xc[(size_t)c0 * K + c];
        v = fma(w1, xc[(size_t)c1 * K + c], v);
        v = fma(w2, xc[(size_t)c2 * K + c], v);
        x[(size_t)i * K + c] += v;
    }
}

// ---------------------------------------------------------------------------
// K3: residual norms.  Block partial sums of (b - Ax)^2 per column, then a
// single-block deterministic finalisation.
constexpr int kNormBlocks = 1184;   // 8 x 148 SMs

template <int K, int LPR>
__global__ void __launch_bounds__(kBlock) k_resnorm_partial(const int* __restrict__ rp, const int* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            const double* __restrict__ b,
                                                            const double* __restrict__ x, double* __restrict__ partial,
                                                            int n) {
    __shared__ double red[kBlock / 32][K];
    const int lane = threadIdx.x & (LPR - 1);
    const unsigned mask = group_mask(LPR);
    const uint64_t pol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const int groups_per_grid = gridDim.x * (kBlock / LPR);
    for (int row = (blockIdx.x * kBlock + threadIdx.x) / LPR; row < n; row += groups_per_grid) {
        const int e0 = rp[row], e1 = rp[row + 1];
        double s[K];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = 0.0;
        for (int e = e0 + lane; e < e1; e += LPR) {
            const int j = ld_stream(col + e, pol);
            const double a = ld_stream(val + e, pol);
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = fma(a, x[(size_t)j * K + c], s[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], mask);
        if (lane == 0) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double rr = b[(size_t)row * K + c] - s[c];
                acc[c] = fma(rr, rr, acc[c]);
            }
        }
    }
    // block reduction (fixed order: deterministic)
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double v = acc[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) v += red[w][threadIdx.x];
        partial[blockIdx.x * K + threadIdx.x] = v;
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_sumsq_partial(const double* __restrict__ v, int n,
                                                          double* __restrict__ partial) {
    __shared__ double red[kBlock / 32][K];
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double t = v[(size_t)i * K + c];
            acc[c] = fma(t, t, acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double t = acc[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = t;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) t += red[w][threadIdx.x];
        partial[blockIdx.x * K + threadIdx.x] = t;
    }
}

// out[c] = sqrt(sum_b partial[b][c]) / (denom[c] > 0 ? denom[c] : 1)   (denom may be null)
template <int K>
__global__ void __launch_bounds__(kBlock) k_norm_finalize(const double* __restrict__ partial, int nblk,
                                                          const double* __restrict__ denom,
                                                          double* __restrict__ out) {
    __shared__ double red[kBlock / 32][K];
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int t = threadIdx.x; t < nblk; t += kBlock)
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] += partial[t * K + c];
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double v = acc[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double v = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) v += red[w][threadIdx.x];
        v = sqrt(v);
        if (denom) {
            const double d = denom[threadIdx.x];
            v = v / (d > 0.0 ? d : 1.0);
        }
        out[threadIdx.x] = v;
    }
}

// ---------------------------------------------------------------------------
// K9: user <-> internal permutations (row blocks of K values).
template <int K>
__global__ void __launch_bounds__(kBlock) k_gather_rows(const int* __restrict__ perm, const double* __restrict__ src,
                                                        double* __restrict__ dst, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const size_t u = (size_t)perm[i];
#pragma unroll
    for (int c = 0; c < K; ++c) dst[(size_t)i * K + c] = src[u * K + c];
}
template <int K>
__global__ void __launch_bounds__(kBlock) k_scatter_rows(const int* __restrict__ perm, const double* __restrict__ src,
                                                         double* __restrict__ dst, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const size_t u = (size_t)perm[i];
#pragma unroll
    for (int c = 0; c < K; ++c) dst[u * K + c] = src[(size_t)i * K + c];
}
__global__ void __launch_bounds__(kBlock) k_gather_vals(const int64_t* __restrict__ i2u, const double* __restrict__ src,
                                                        double* __restrict__ dst, int64_t nnz) {
    const int64_t e = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    if (e < nnz) dst[e] = src[i2u[e]];
}

// B = M X (user order).
template <int K>
__global__ void __launch_bounds__(kBlock) k_apply_mass(const double* __restrict__ M, const double* __restrict__ X,
                                                       double* __restrict__ B, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const double m = M[i];
#pragma unroll
    for (int c = 0; c < K; ++c) B[(size_t)i * K + c] = m * X[(size_t)i * K + c];
}

// ---------------------------------------------------------------------------
// K1: cotangent Laplacian + lumped mass on the fixed 1-ring pattern (internal
// order).  Each off-diagonal (i,j) reads its <= 2 opposite vertices
// (opp[2e], opp[2e+1], -1 for a boundary edge: natural BC):
//   L_ij = -1/2 sum_o cot(angle at o),  cot = (vi-vo).(vj-vo) / |(vi-vo)x(vj-vo)|
//   L_ii = -sum_{j != i} L_ij
//   M_ii = 1/3 sum_{faces f at i} area_f = 1/6 sum_{(i,j)} sum_o |(vi-vo)x(vj-vo)|/2
// (every face at i is seen from both of its edges at i).  One thread per row,
// deterministic (no atomics).  A = mass_coeff M + lap_coeff L.
__global__ void __launch_bounds__(kBlock) k_cotan_assemble(const int* __restrict__ rp, const int* __restrict__ col,
                                                           const int* __restrict__ opp, const double* __restrict__ V,
                                                           double mass_coeff, double lap_coeff,
                                                           double* __restrict__ val, double* __restrict__ M, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const double xi = V[3 * (size_t)i], yi = V[3 * (size_t)i + 1], zi = V[3 * (size_t)i + 2];
    double lsum = 0.0, area2 = 0.0;
    int ediag = -1;
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
        const int j = col[e];
        if (j == i) {
            ediag = e;
            continue;
        }
        const double xj = V[3 * (size_t)j], yj = V[3 * (size_t)j + 1], zj = V[3 * (size_t)j + 2];
        double cot_sum = 0.0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int o = opp[2 * (size_t)e + s];
            if (o < 0) continue;
            const double xo = V[3 * (size_t)o], yo = V[3 * (size_t)o + 1], zo = V[3 * (size_t)o + 2];
            const double ax = xi - xo, ay = yi - yo, az = zi - zo;
            const double bx = xj - xo, by = yj - yo, bz = zj - zo;
            const double cx = ay * bz - az * by, cy = az * bx - ax * bz, cz = ax * by - ay * bx;
            const double cr = sqrt(cx * cx + cy * cy + cz * cz);
            cot_sum += (ax * bx + ay * by + az * bz) / cr;
            area2 += cr;
        }
        const double lij = -0.5 * cot_sum;
        lsum += lij;
        val[e] = lap_coeff * lij;
    }
    const double m = area2 / 12.0;   // (1/6) * sum (|cross| / 2)
    M[i] = m;
    if (ediag >= 0) val[ediag] = mass_coeff * m + lap_coeff * (-lsum);
}

__global__ void k_scatter_vec(const int* __restrict__ perm, const double* __restrict__ src, double* __restrict__ dst,
                              int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i < n) dst[perm[i]] = src[i];
}

// ---------------------------------------------------------------------------
// K2: Galerkin numeric phase.  One warp per coarse row I (taken in locality
// order):  A_c[I, J] = sum_{i in children(I)} P[i,I] sum_{j in row i} A[i,j] P[j,J].
// The (child, nonzero) pairs of the coarse row are flattened across the 32
// lanes; each contribution finds its slot J by binary search in the coarse
// row's (sorted) column list held in shared memory and is accumulated there.
// Rows wider than kGalMaxM accumulate into global memory instead.
constexpr int kGalWarps = 8;
constexpr int kGalMaxM = 96;

__device__ __forceinline__ int find_slot(const int* cols, int m, int J) {
    int lo = 0, hi = m - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < J) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kGalWarps * 32) k_galerkin(
    int nc, const int* __restrict__ order, const int* __restrict__ crp, const int* __restrict__ ccol,
    double* __restrict__ cval, const int* __restrict__ cptr, const int* __restrict__ cidx,
    const double* __restrict__ cw, const int* __restrict__ rp, const int* __restrict__ col,
    const double* __restrict__ val, const int* __restrict__ pc, const double* __restrict__ pw, int nf) {
    __shared__ double acc[kGalWarps][kGalMaxM];
    __shared__ int cols[kGalWarps][kGalMaxM];
    __shared__ int ch_start[kGalWarps][32];
    __shared__ int ch_scan[kGalWarps][32];
    __shared__ double ch_w[kGalWarps][32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kGalWarps + w;
    if (gw >= nc) return;
    const int I = order[gw];
    const int c0 = crp[I];
    const int m = crp[I + 1] - c0;
    const bool wide = m > kGalMaxM;
    const int* slots = wide ? (ccol + c0) : cols[w];
    double* accp = wide ? (cval + c0) : acc[w];
    for (int s = lane; s < m; s += 32) {
        if (!wide) cols[w][s] = ccol[c0 + s];
        accp[s] = 0.0;
    }
    __syncwarp();
    const int t0 = cptr[I], t1 = cptr[I + 1];
    for (int tb = t0; tb < t1; tb += 32) {
        const int nb = min(32, t1 - tb);
        int len = 0;
        if (lane < nb) {
            const int i = cidx[tb + lane];
            ch_w[w][lane] = cw[tb + lane];
            const int s = rp[i];
            ch_start[w][lane] = s;
            len = rp[i + 1] - s;
        }
        int incl = len;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        ch_scan[w][lane] = incl;
        const int total = __shfl_sync(0xffffffffu, incl, nb - 1);
        __syncwarp();
        for (int g = lane; g < total; g += 32) {
            int lo = 0, hi = nb - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (ch_scan[w][mid] > g) hi = mid;
                else lo = mid + 1;
            }
            const int excl = lo ? ch_scan[w][lo - 1] : 0;
            const int e = ch_start[w][lo] + (g - excl);
            const int j = col[e];
            const double a = ch_w[w][lo] * val[e];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double wq = pw[(size_t)q * nf + j];
                if (wq != 0.0) {
                    const int J = pc[(size_t)q * nf + j];
                    const int slot = find_slot(slots, m, J);
                    atomicAdd(accp + slot, a * wq);
                }
            }
        }
        __syncwarp();
    }
    if (!wide)
        for (int s = lane; s < m; s += 32) cval[c0 + s] = acc[w][s];
}

// ---------------------------------------------------------------------------
// K7: coarsest level.  Dense row-major npad x npad (npad multiple of 32,
// padding = identity), blocked right-looking Cholesky with 32-wide panels:
// one CTA factors the diagonal block, a grid solves the panel below it, then a
// grid of CTAs applies the rank-32 update to the trailing lower triangle.
__global__ void k_densify_zero(double* D, size_t total) {
    for (size_t t = (size_t)blockIdx.x * kBlock + threadIdx.x; t < total; t += (size_t)gridDim.x * kBlock) D[t] = 0.0;
}
__global__ void k_densify(const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                          int n, int npad, double* __restrict__ D) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= npad) return;
    if (i >= n) {
        D[(size_t)i * npad + i] = 1.0;
        return;
    }
    for (int e = rp[i]; e < rp[i + 1]; ++e) D[(size_t)i * npad + col[e]] = val[e];
}

__global__ void __launch_bounds__(1024) k_chol_diag(double* __restrict__ D, int npad, int kb, int* err) {
    __shared__ double Ld[32][33];
    const int tid = threadIdx.x, r = tid >> 5, c = tid & 31;
    const int base = kb * 32;
    Ld[r][c] = D[(size_t)(base + r) * npad + base + c];
    __syncthreads();
    for (int p = 0; p < 32; ++p) {
        if (tid == 0) {
            double d = Ld[p][p];
            if (!(d > 0.0)) {
                atomicExch(err, 1);
                d = 1.0;
            }
            Ld[p][p] = sqrt(d);
        }
        __syncthreads();
        if (tid > p && tid < 32) Ld[tid][p] /= Ld[p][p];
        __syncthreads();
        if (r > p && c > p && c <= r) Ld[r][c] -= Ld[r][p] * Ld[c][p];
        __syncthreads();
    }
    D[(size_t)(base + r) * npad + base + c] = (c <= r) ? Ld[r][c] : 0.0;
}

// panel below the diagonal block: l = a L_kk^{-T}, one thread per row
constexpr int kTrsmThreads = 64;
__global__ void __launch_bounds__(kTrsmThreads) k_chol_trsm(double* __restrict__ D, int npad, int kb) {
    __shared__ double Ld[32][33];
    const int base = kb * 32;
    for (int s = threadIdx.x; s < 1024; s += kTrsmThreads) Ld[s >> 5][s & 31] = D[(size_t)(base + (s >> 5)) * npad + base + (s & 31)];
    __syncthreads();
    const int i = base + 32 + blockIdx.x * kTrsmThreads + threadIdx.x;
    if (i >= npad) return;
    double a[32];
    double* Di = D + (size_t)i * npad + base;
#pragma unroll
    for (int p = 0; p < 32; ++p) a[p] = Di[p];
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        double s = a[p];
#pragma unroll
        for (int q = 0; q < p; ++q) s -= a[q] * Ld[p][q];
        a[p] = s / Ld[p][p];
    }
#pragma unroll
    for (int p = 0; p < 32; ++p) Di[p] = a[p];
}

__global__ void __launch_bounds__(256) k_chol_update(double* __restrict__ D, int npad, int kb) {
    __shared__ double Pi[32][33];
    __shared__ double Pj[32][33];
    const int t = blockIdx.x;
    int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    const int tj = t - ti * (ti + 1) / 2;
    const int bi = kb + 1 + ti, bj = kb + 1 + tj;
    const int base = kb * 32;
    for (int s = threadIdx.x; s < 1024; s += 256) {
        const int r = s >> 5, c = s & 31;
        Pi[r][c] = D[(size_t)(bi * 32 + r) * npad + base + c];
        Pj[r][c] = D[(size_t)(bj * 32 + r) * npad + base + c];
    }
    __syncthreads();
    for (int s = threadIdx.x; s < 1024; s += 256) {
        const int r = s >> 5, c = s & 31;
        if (bi == bj && c > r) continue;
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < 32; ++p) acc = fma(Pi[r][p], Pj[c][p], acc);
        D[(size_t)(bi * 32 + r) * npad + bj * 32 + c] -= acc;
    }
}

// Inverse of every 32x32 diagonal block of L (for the solve); thread t
// computes column t by forward substitution.
__global__ void __launch_bounds__(32) k_chol_diaginv(const double* __restrict__ D, int npad, double* __restrict__ Linv) {
    __shared__ double Ld[32][33];
    const int I = blockIdx.x, t = threadIdx.x;
    for (int r = 0; r < 32; ++r) Ld[r][t] = D[(size_t)(I * 32 + r) * npad + I * 32 + t];
    __syncwarp();
    double z[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        double s = (r == t) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < r; ++q) s -= Ld[r][q] * z[q];
        z[r] = (r >= t) ? s / Ld[r][r] : 0.0;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) Linv[(size_t)I * 1024 + r * 32 + t] = z[r];
}

// Coarsest solve L L^T x = b in ONE CTA (1024 threads): blocked forward and
// backward substitution; the off-diagonal blocks are streamed from L2 with
// coalesced row loads, the diagonal blocks applied through their inverses
// with warp-shuffle reductions; the iterate is staged in shared memory.
template <int K>
__global__ void __launch_bounds__(1024) k_chol_solve(const double* __restrict__ L, const double* __restrict__ Linv,
                                                     int npad, int n, const double* __restrict__ b,
                                                     double* __restrict__ x) {
    extern __shared__ double sm[];
    double* y = sm;                       // [npad][K]
    double* red = sm + (size_t)npad * K;  // [32][32][K]
    double* t = red + 32 * 32 * K;        // [32][K]
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < npad * K; i += 1024) y[i] = (i < n * K) ? b[i] : 0.0;
    __syncthreads();
    const int nb = npad / 32;
    for (int I = 0; I < nb; ++I) {
        // t_r = y_{32I+r} - sum_{j < 32I} L[32I+r][j] y_j      (warp w = row r)
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = 0.0;
        const double* Lr = L + (size_t)(32 * I + w) * npad;
        for (int j = lane; j < 32 * I; j += 32) {
            const double l = Lr[j];
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = fma(l, y[j * K + c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
        }
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < K; ++c) t[w * K + c] = y[(32 * I + w) * K + c] - acc[c];
        __syncthreads();
        // y_I = inv(L_II) t      (warp w = row r, lane = column q)
        const double li = Linv[(size_t)I * 1024 + w * 32 + lane];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            double v = li * t[lane * K + c];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            acc[c] = v;
        }
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < K; ++c) y[(32 * I + w) * K + c] = acc[c];
        __syncthreads();
    }
    for (int I = nb - 1; I >= 0; --I) {
        // t_r = y_{32I+r} - sum_{j >= 32(I+1)} L[j][32I+r] x_j   (lane = r, warps stride j)
        double acc[K];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = 0.0;
        for (int j = 32 * (I + 1) + w; j < npad; j += 32) {
            const double l = L[(size_t)j * npad + 32 * I + lane];
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = fma(l, y[j * K + c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) red[(w * 32 + lane) * K + c] = acc[c];
        __syncthreads();
        if (w == 0) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
                double s = 0.0;
                for (int v = 0; v < 32; ++v) s += red[(v * 32 + lane) * K + c];
                t[lane * K + c] = y[(32 * I + lane) * K + c] - s;
            }
        }
        __syncthreads();
        // x_I = inv(L_II)^T t : x_r = sum_q inv[q][r] t_q   (warp w = r, lane = q)
        const double li = Linv[(size_t)I * 1024 + lane * 32 + w];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            double v = li * t[lane * K + c];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            acc[c] = v;
        }
        if (lane == 0)
#pragma unroll
            for (int c = 0; c < K; ++c) y[(32 * I + w) * K + c] = acc[c];
        __syncthreads();
    }
    for (int i = tid; i < n * K; i += 1024) x[i] = y[i];
}

// Explicit inverse A_H^{-1} = L^{-T} L^{-1} from the factor: CTA b solves
// L L^T Z = I for columns [16b, 16b+16) by blocked forward/backward
// substitution (off-diagonal blocks streamed from L2 as warp-broadcast
// loads, diagonal blocks applied through their inverses).  Computed once per
// rebuild; afterwards every coarsest solve is one GEMV (k_coarse_gemv).
constexpr int kInvCols = 16;
__global__ void __launch_bounds__(512) k_chol_inverse(const double* __restrict__ L, const double* __restrict__ Linv,
                                                      int npad, double* __restrict__ Z) {
    extern __shared__ double sm[];
    double* Y = sm;                          // [npad][16]
    double* T = sm + (size_t)npad * kInvCols; // [32][16]
    const int tid = threadIdx.x, r = tid >> 4, c = tid & 15;
    const int c0 = blockIdx.x * kInvCols;
    const int nb = npad / 32;
    for (int I = 0; I < nb; ++I) {
        double acc = 0.0;
        const double* Lr = L + (size_t)(32 * I + r) * npad;
        for (int j = 0; j < 32 * I; ++j) acc = fma(Lr[j], Y[j * kInvCols + c], acc);
        T[r * kInvCols + c] = ((32 * I + r) == (c0 + c) ? 1.0 : 0.0) - acc;
        __syncthreads();
        double v = 0.0;
        const double* Li = Linv + (size_t)I * 1024 + r * 32;
#pragma unroll 8
        for (int q = 0; q < 32; ++q) v = fma(Li[q], T[q * kInvCols + c], v);
        Y[(32 * I + r) * kInvCols + c] = v;
        __syncthreads();
    }
    for (int I = nb - 1; I >= 0; --I) {
        double acc = 0.0;
        for (int j = 32 * (I + 1); j < npad; ++j) acc = fma(L[(size_t)j * npad + 32 * I + r], Y[j * kInvCols + c], acc);
        T[r * kInvCols + c] = Y[(32 * I + r) * kInvCols + c] - acc;
        __syncthreads();
        double v = 0.0;
#pragma unroll 8
        for (int q = 0; q < 32; ++q) v = fma(Linv[(size_t)I * 1024 + q * 32 + r], T[q * kInvCols + c], v);
        Y[(32 * I + r) * kInvCols + c] = v;
        __syncthreads();
    }
    for (int i = tid; i < npad * kInvCols; i += 512) Z[(size_t)(i / kInvCols) * npad + c0 + (i % kInvCols)] = Y[i];
}

// Coarsest solve x = A_H^{-1} b: one warp per row of the inverse (coalesced
// row reads from L2), K columns.
template <int K>
__global__ void __launch_bounds__(256) k_coarse_gemv(const double* __restrict__ Z, int npad, int n,
                                                     const double* __restrict__ b, double* __restrict__ x) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const double* Zr = Z + (size_t)row * npad;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double z = Zr[j];
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(z, b[(size_t)j * K + c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
    }
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < K; ++c) x[(size_t)row * K + c] = acc[c];
}

inline int nblk(int64_t n, int per) { return (int)((n + per - 1) / per); }

inline size_t tile_smem(int cap) { return (size_t)cap * (sizeof(double) + sizeof(int)); }

template <int K>
int gs_dispatch(int lpr, const Level& L, int r0, int r1, cudaStream_t s) {
    const int rows = r1 - r0;
    if (rows <= 0) return 0;
    if (L.tiled) {
        k_gs_tiled<K><<<nblk(rows, kTile), kTile, tile_smem(L.cap_gs), s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, r0,
                                                                            r1, L.cap_gs);
        return 1;
    }
    const int grid = nblk((int64_t)rows * lpr, kBlock);
    switch (lpr) {
        case 4: k_gs_colour<K, 4><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, r0, r1); break;
        case 8: k_gs_colour<K, 8><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, r0, r1); break;
        case 16: k_gs_colour<K, 16><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, r0, r1); break;
        default: k_gs_colour<K, 32><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, r0, r1); break;
    }
    return 1;
}

template <int K>
int residual_dispatch(int lpr, const Level& L, cudaStream_t s) {
    if (L.tiled) {
        k_residual_tiled<K><<<nblk(L.n, kTile), kTile, tile_smem(L.cap_all), s>>>(L.rp.p, L.col.p, L.val.p, L.b.p,
                                                                                  L.x.p, L.r.p, L.n, L.cap_all);
        return 1;
    }
    const int grid = nblk((int64_t)L.n * lpr, kBlock);
    switch (lpr) {
        case 4: k_residual<K, 4><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, L.r.p, L.n); break;
        case 8: k_residual<K, 8><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, L.r.p, L.n); break;
        case 16: k_residual<K, 16><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, L.r.p, L.n); break;
        default: k_residual<K, 32><<<grid, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, L.r.p, L.n); break;
    }
    return 1;
}

template <int K>
int resnorm_dispatch(int lpr, const Level& L, double* partial, int nb, const double* bnorm, double* rho,
                     cudaStream_t s) {
    if (L.tiled) {
        const int grid = std::min(nb, nblk(L.n, kTile));
        k_resnorm_tiled<K><<<grid, kTile, tile_smem(L.cap_all), s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial,
                                                                     L.n, L.cap_all);
        k_norm_finalize<K><<<1, kBlock, 0, s>>>(partial, grid, bnorm, rho);
        return 2;
    }
    switch (lpr) {
        case 4: k_resnorm_partial<K, 4><<<nb, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
        case 8: k_resnorm_partial<K, 8><<<nb, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
        case 16: k_resnorm_partial<K, 16><<<nb, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
        default: k_resnorm_partial<K, 32><<<nb, kBlock, 0, s>>>(L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
    }
    k_norm_finalize<K><<<1, kBlock, 0, s>>>(partial, nb, bnorm, rho);
    return 2;
}

template <template <int> class F, class... A>
int dispatch_k(int K, A... a) {
    switch (K) {
        case 1: return F<1>::run(a...);
        case 2: return F<2>::run(a...);
        case 3: return F<3>::run(a...);
        default: return F<4>::run(a...);
    }
}

template <int K>
struct GsF {
    static int run(int lpr, const Level* L, int r0, int r1, cudaStream_t s) { return gs_dispatch<K>(lpr, *L, r0, r1, s); }
};
template <int K>
struct ResF {
    static int run(int lpr, const Level* L, cudaStream_t s) { return residual_dispatch<K>(lpr, *L, s); }
};
template <int K>
struct RestrictF {
    static int run(const Level* C, const Level* F, cudaStream_t s) {
        k_restrict<K><<<nblk(C->n, kBlock), kBlock, 0, s>>>(C->cptr.p, C->cidx.p, C->cw.p, F->r.p, C->b.p, C->x.p, C->n);
        return 1;
    }
};
template <int K>
struct ProlongF {
    static int run(const Level* F, const Level* C, cudaStream_t s) {
        k_prolong<K><<<nblk(F->n, kBlock), kBlock, 0, s>>>(F->pc.p, F->pw.p, C->x.p, F->x.p, F->n);
        return 1;
    }
};
template <int K>
struct ResnormF {
    static int run(int lpr, const Level* L, double* partial, int nb, const double* bnorm, double* rho, cudaStream_t s) {
        return resnorm_dispatch<K>(lpr, *L, partial, nb, bnorm, rho, s);
    }
};
template <int K>
struct SumsqF {
    static int run(const double* v, int n, double* partial, int nb, double* out, cudaStream_t s) {
        k_sumsq_partial<K><<<nb, kBlock, 0, s>>>(v, n, partial);
        k_norm_finalize<K><<<1, kBlock, 0, s>>>(partial, nb, nullptr, out);
        return 2;
    }
};
template <int K>
struct GatherF {
    static int run(const int32_t* perm, const double* src, double* dst, int n, cudaStream_t s) {
        if (n <= 0) return 0;
        k_gather_rows<K><<<nblk(n, kBlock), kBlock, 0, s>>>(perm, src, dst, n);
        return 1;
    }
};
template <int K>
struct ScatterF {
    static int run(const int32_t* perm, const double* src, double* dst, int n, cudaStream_t s) {
        if (n <= 0) return 0;
        k_scatter_rows<K><<<nblk(n, kBlock), kBlock, 0, s>>>(perm, src, dst, n);
        return 1;
    }
};
template <int K>
struct MassF {
    static int run(const double* M, const double* X, double* B, int n, cudaStream_t s) {
        if (n <= 0) return 0;
        k_apply_mass<K><<<nblk(n, kBlock), kBlock, 0, s>>>(M, X, B, n);
        return 1;
    }
};
template <int K>
struct GemvF {
    static int run(const double* Z, int npad, int n, const double* b, double* x, cudaStream_t s) {
        k_coarse_gemv<K><<<nblk(n, 8), 256, 0, s>>>(Z, npad, n, b, x);
        return 1;
    }
};
template <int K>
struct CholSolveF {
    static int run(const double* D, const double* Linv, int npad, int n, const double* b, double* x, cudaStream_t s) {
        const size_t smem = sizeof(double) * ((size_t)npad * K + 32 * 32 * K + 32 * K);
        k_chol_solve<K><<<1, 1024, smem, s>>>(D, Linv, npad, n, b, x);
        return 1;
    }
};

template <int K>
void set_attrs() {
    const int big = 200 * 1024;
    cudaFuncSetAttribute(k_gs_tiled<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_residual_tiled<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_resnorm_tiled<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_chol_solve<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_chol_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

}  // namespace

int resnorm_blocks(int n) { return kNormBlocks; }
int tile_rows() { return kTile; }
size_t tile_smem_limit() { return 160 * 1024; }

void init_kernel_attributes() {
    set_attrs<1>();
    set_attrs<2>();
    set_attrs<3>();
    set_attrs<4>();
}

int launch_gs_colour(int K, int lpr, const Level& L, int r0, int r1, cudaStream_t s) {
    return dispatch_k<GsF>(K, lpr, &L, r0, r1, s);
}
int launch_residual(int K, int lpr, const Level& L, cudaStream_t s) { return dispatch_k<ResF>(K, lpr, &L, s); }
int launch_restrict(int K, const Level& coarse, const Level& fine, cudaStream_t s) {
    return dispatch_k<RestrictF>(K, &coarse, &fine, s);
}
int launch_prolong(int K, const Level& fine, const Level& coarse, cudaStream_t s) {
    return dispatch_k<ProlongF>(K, &fine, &coarse, s);
}
int launch_resnorm(int K, int lpr, const Level& L, double* partial, int nblk_max, const double* bnorm,
                   double* rho_out, cudaStream_t s) {
    return dispatch_k<ResnormF>(K, lpr, &L, partial, nblk_max, bnorm, rho_out, s);
}
int launch_sumsq(int K, const double* v, int n, double* partial, int nblk_max, double* out, cudaStream_t s) {
    return dispatch_k<SumsqF>(K, v, n, partial, nblk_max, out, s);
}
int launch_gather_rows(int K, const int32_t* perm, const double* src_user, double* dst_int, int n, cudaStream_t s) {
    return dispatch_k<GatherF>(K, perm, src_user, dst_int, n, s);
}
int launch_scatter_rows(int K, const int32_t* perm, const double* src_int, double* dst_user, int n, cudaStream_t s) {
    return dispatch_k<ScatterF>(K, perm, src_int, dst_user, n, s);
}
int launch_gather_vals(const int64_t* i2u, const double* src, double* dst, int64_t nnz, cudaStream_t s) {
    if (nnz <= 0) return 0;
    k_gather_vals<<<nblk(nnz, kBlock), kBlock, 0, s>>>(i2u, src, dst, nnz);
    return 1;
}
int launch_cotan(const Level& L0, const int32_t* opp, const double* Vint, double mass_coeff, double lap_coeff,
                 double* M_int, cudaStream_t s) {
    k_cotan_assemble<<<nblk(L0.n, kBlock), kBlock, 0, s>>>(L0.rp.p, L0.col.p, opp, Vint, mass_coeff, lap_coeff,
                                                            L0.val.p, M_int, L0.n);
    return 1;
}
int launch_apply_mass(int K, const double* M_user, const double* X, double* B, int n, cudaStream_t s) {
    return dispatch_k<MassF>(K, M_user, X, B, n, s);
}
int launch_scatter_vec(const int32_t* perm, const double* src_int, double* dst_user, int n, cudaStream_t s) {
    k_scatter_vec<<<nblk(n, kBlock), kBlock, 0, s>>>(perm, src_int, dst_user, n);
    return 1;
}
int launch_galerkin(const Level& fine, Level& coarse, cudaStream_t s) {
    const int nc = coarse.n;
    k_galerkin<<<nblk(nc, kGalWarps), kGalWarps * 32, 0, s>>>(
        nc, coarse.gal_order.p, coarse.rp.p, coarse.col.p, coarse.val.p, coarse.cptr.p, coarse.cidx.p, coarse.cw.p,
        fine.rp.p, fine.col.p, fine.val.p, fine.pc.p, fine.pw.p, fine.n);
    return 1;
}
int launch_densify(const Level& LH, double* D, int npad, cudaStream_t s) {
    const size_t total = (size_t)npad * npad;
    k_densify_zero<<<nblk((int64_t)std::min<size_t>(total, 1u << 20), kBlock), kBlock, 0, s>>>(D, total);
    k_densify<<<nblk(npad, kBlock), kBlock, 0, s>>>(LH.rp.p, LH.col.p, LH.val.p, LH.n, npad, D);
    return 2;
}
int launch_chol_factor(double* D, double* Linv, int npad, int* err, cudaStream_t s) {
    const int nb = npad / 32;
    int launches = 0;
    for (int kb = 0; kb < nb; ++kb) {
        k_chol_diag<<<1, 1024, 0, s>>>(D, npad, kb, err);
        ++launches;
        const int m = nb - kb - 1;
        if (m > 0) {
            k_chol_trsm<<<nblk(32 * m, kTrsmThreads), kTrsmThreads, 0, s>>>(D, npad, kb);
            ++launches;
            k_chol_update<<<m * (m + 1) / 2, 256, 0, s>>>(D, npad, kb);
            ++launches;
        }
    }
    k_chol_diaginv<<<nb, 32, 0, s>>>(D, npad, Linv);
    return launches + 1;
}
int launch_chol_inverse(const double* D, const double* Linv, int npad, double* Z, cudaStream_t s) {
    const size_t smem = sizeof(double) * ((size_t)npad * kInvCols + 32 * kInvCols);
    k_chol_inverse<<<npad / kInvCols, 512, smem, s>>>(D, Linv, npad, Z);
    return 1;
}
int launch_coarse_gemv(int K, const double* Z, int npad, int n, const double* b, double* x, cudaStream_t s) {
    return dispatch_k<GemvF>(K, Z, npad, n, b, x, s);
}
int launch_chol_solve(int K, const double* D, const double* Linv, int npad, int n, const double* b, double* x,
                      cudaStream_t s) {
    return dispatch_k<CholSolveF>(K, D, Linv, npad, n, b, x, s);
}

}  // namespace mg
