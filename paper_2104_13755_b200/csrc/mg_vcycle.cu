// libmg V-cycle kernels for sm_100a (Alg. 2).  fp64, HBM-bound
// (SpMV-class intensity ~0.17 flop/B): no tensor cores.
//
//   K4 multicolour Gauss-Seidel colour pass      (App. A, reading A2)
//   K5 residual r = b - A x' and restriction P^T r (Alg. 2)
//   K6 prolongation + correction x <- x' + P c     (Alg. 2, reading A1)
//   K7b coarsest solve x = A_H^{-1} b              (Alg. 2, reading A12)
//   K3 residual norm rho = ||b - A x|| / ||b||     (reading A3)
//
// Every kernel here is launched with programmatic dependent launch inside the
// captured V-cycle graph: a prologue loads what no earlier kernel of the
// solve writes (matrix structure/values, P, children lists), then
// griddepcontrol.wait, then the dependent part (x, b, r).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mg_common.cuh"
#include "mg_internal.h"

namespace mg {
namespace {

// Experiment builds (MG_NVCC_DEFINES=-DMG_GS_TRACE, tools/gs_trace.py): thread
// 0 of every CTA of a GS colour pass stamps %globaltimer at kernel entry,
// after griddepcontrol.wait and at its end.  Compiled out of the product.
#ifdef MG_GS_TRACE
constexpr unsigned kGsTraceCap = 1u << 20;
__device__ unsigned long long g_gs_trace[4 * kGsTraceCap];
__device__ unsigned g_gs_trace_n;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
struct GsTrace {
    unsigned long long t0, t1;
    __device__ __forceinline__ void start() { if (threadIdx.x == 0) t0 = gtime(); }
    __device__ __forceinline__ void waited() { if (threadIdx.x == 0) t1 = gtime(); }
    __device__ __forceinline__ void end(int kid, int key) {
        if (threadIdx.x == 0) {
            const unsigned long long t2 = gtime();
            const unsigned k = atomicAdd(&g_gs_trace_n, 1u);
            if (k < kGsTraceCap) {
                g_gs_trace[4 * k] = t0;
                g_gs_trace[4 * k + 1] = t1;
                g_gs_trace[4 * k + 2] = t2;
                g_gs_trace[4 * k + 3] = ((unsigned long long)kid << 56) | ((unsigned long long)(unsigned)key << 24) |
                                        (unsigned long long)(blockIdx.x & 0xffffff);
            }
        }
    }
};
#else
struct GsTrace {
    __device__ __forceinline__ void start() {}
    __device__ __forceinline__ void waited() {}
    __device__ __forceinline__ void end(int, int) {}
};
#endif

// ---------------------------------------------------------------------------
// Tile-staged CSR rows (levels with short rows): a CTA owns kTile consecutive
// rows; row pointers and the tile's contiguous run of (col, val) are staged
// into shared memory with coalesced streaming loads in the PDL prologue; each
// thread then processes one row, issuing its x gathers in independent batches.
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
        const int c0 = ld_stream(cg + q, pol), c1 = ld_stream(cg + q + kTile, pol),
                  c2 = ld_stream(cg + q + 2 * kTile, pol), c3 = ld_stream(cg + q + 3 * kTile, pol);
        const double v0 = ld_stream(vg + q, pol), v1 = ld_stream(vg + q + kTile, pol),
                     v2 = ld_stream(vg + q + 2 * kTile, pol), v3 = ld_stream(vg + q + 3 * kTile, pol);
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

// s[c] = sum_{j != row} a_rj x_jc and d = a_rr from the staged tile.
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
        for (int u = 0; u < UNR; ++u) ldrow<K>(x + (size_t)j[u] * VS<K>::S, xv[u]);
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

// gathers per batch in the pipelined tile kernel: one batch covers a whole
// 1-ring row (7 entries incl. the skipped diagonal) for every K
template <int K>
struct PipeUnroll {
    static constexpr int value = K >= 3 ? 4 : 8;
};

template <int K>
struct Unroll {
    static constexpr int value = K == 1 ? 8 : 4;
};

// MODE 0: GS colour pass  x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii  on rows [r0, r1)
// MODE 1: residual        r_i = b_i - sum_j a_ij x_j                   on rows [r0, r1)
// MODE 3: damped Jacobi   r_i = x_i + omega (b_i - sum_j a_ij x_j) / a_ii (App. E; into r)
template <int K, int MODE>
__global__ void __launch_bounds__(kTile) k_tile_sweep(const int* __restrict__ rp, const int* __restrict__ col,
                                                      const double* __restrict__ val, const double* __restrict__ b,
                                                      double* __restrict__ x, double* __restrict__ r, int r0, int r1,
                                                      int cap, double omega) {
    extern __shared__ double smem_d[];
    __shared__ int rps[kTile + 1];
    double* vs = smem_d;
    int* cs = reinterpret_cast<int*>(smem_d + cap);
    pdl_launch_dependents();
    const uint64_t pol = evict_first_policy();
    const int row0 = r0 + blockIdx.x * kTile;
    const int nrow = min(kTile, r1 - row0);
    const int e0 = tile_stage(rp, col, val, row0, nrow, rps, cs, vs, pol);
    pdl_wait();
    const int t = threadIdx.x;
    if (t >= nrow) return;
    const int row = row0 + t;
    double s[K], d;
    tile_row<K, Unroll<K>::value>(cs, vs, rps[t] - e0, rps[t + 1] - e0, row, x, s, d);
    const double inv = (MODE == 0 || MODE == 3) ? 1.0 / d : 0.0;
    if (MODE == 0) {
        double bv[K], xn[K];
        ldrow<K>(b + (size_t)row * VS<K>::S, bv);
#pragma unroll
        for (int c = 0; c < K; ++c) xn[c] = div_by(bv[c] - s[c], d, inv);
        strow<K>(x + (size_t)row * VS<K>::S, xn);
    } else {
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double xi = x[(size_t)row * VS<K>::S + c];
            const double rr = b[(size_t)row * VS<K>::S + c] - fma(d, xi, s[c]);
            r[(size_t)row * VS<K>::S + c] = MODE == 3 ? xi + div_by(omega * rr, d, inv) : rr;
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent, double-buffered variant of the tile kernel (default for levels
// with short rows).  Each CTA walks the tiles t = t_begin + blockIdx.x +
// i * gridDim.x; one thread streams tile i+2's row pointers, columns and
// values into shared memory with 1-D TMA bulk copies (cp.async.bulk, L2
// evict-first) completing on an mbarrier, while all threads compute tile i.
// Tile descriptors {row0, nrow, e0, e1} are precomputed per level, so no
// pointer chase precedes a copy.  Gathers of x skip the diagonal (predicated).
// MODE 0: GS pass, 1: residual r = b - A x, 2: residual-norm partial sums,
// 3: damped Jacobi r = x + omega D^{-1} (b - A x).
struct TileDesc {
    int row0, nrow, e0, e1;
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)), "l"(pol)
        : "memory");
}

// shared-memory layout of one stage: [rps: kTile+8 ints][cs: cap+8 ints][vs: cap+4 doubles]
__host__ __device__ inline int stage_ints(int cap) { return (kTile + 8) + (cap + 8); }
__host__ __device__ inline size_t stage_bytes(int cap) {
    const size_t ints = (size_t)stage_ints(cap);
    const size_t a = (ints * 4 + 15) / 16 * 16;
    return a + (size_t)(cap + 4) * 8;
}

struct StageView {
    const int* rps;   // rps[t] = row pointer of row0 + t
    const int* cs;    // cs[q] = col[e0 + q]
    const double* vs; // vs[q] = val[e0 + q]
};

__device__ __forceinline__ void issue_tile(const TileDesc& d, unsigned char* stage, int cap, uint64_t* bar,
                                           const int* rp, const int* col, const double* val, uint64_t pol) {
    const int ra = d.row0 & ~3;
    const int rcnt = (d.row0 + d.nrow + 1 - ra + 3) & ~3;
    const int ca = d.e0 & ~3;
    const int ccnt = (d.e1 - ca + 3) & ~3;
    const int va = d.e0 & ~1;
    const int vcnt = (d.e1 - va + 1) & ~1;
    int* rps = reinterpret_cast<int*>(stage);
    int* cs = rps + (kTile + 8);
    double* vs = reinterpret_cast<double*>(stage + ((size_t)stage_ints(cap) * 4 + 15) / 16 * 16);
    const unsigned bytes = (unsigned)(rcnt * 4 + ccnt * 4 + vcnt * 8);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(rps, rp + ra, rcnt * 4, bar, pol);
    if (ccnt > 0) bulk_g2s(cs, col + ca, ccnt * 4, bar, pol);
    if (vcnt > 0) bulk_g2s(vs, val + va, vcnt * 8, bar, pol);
}

__device__ __forceinline__ StageView view_tile(const TileDesc& d, const unsigned char* stage, int cap) {
    const int* rps = reinterpret_cast<const int*>(stage);
    const int* cs = rps + (kTile + 8);
    const double* vs = reinterpret_cast<const double*>(stage + ((size_t)stage_ints(cap) * 4 + 15) / 16 * 16);
    StageView v;
    v.rps = rps + (d.row0 - (d.row0 & ~3));
    v.cs = cs + (d.e0 - (d.e0 & ~3)) - d.e0;   // index with absolute nnz positions
    v.vs = vs + (d.e0 - (d.e0 & ~1)) - d.e0;
    return v;
}

// Tile schedule: CTA b takes tiles b, b + G, ... of [t_begin, t_end), walked
// backwards when rev != 0 (alternate passes over a level run in opposite
// directions, so a pass starts where the previous one left its lines in L2;
// the rows of one pass are independent, so the result does not change).
__device__ __forceinline__ int tile_ix(int t_begin, int t_end, int t, int rev) {
    return rev ? t_end - 1 - t : t_begin + t;
}

template <int K, int UNR>
__device__ __forceinline__ void stage_row(const StageView& v, int t, int row, const double* __restrict__ x,
                                          double (&s)[K], double& d, uint64_t xpol) {
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    d = 0.0;
    const int qb = v.rps[t], qe = v.rps[t + 1];
    for (int q = qb; q < qe; q += UNR) {
        int j[UNR];
        double a[UNR];
        double xv[UNR][K];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const bool ok = q + u < qe;
            j[u] = ok ? v.cs[q + u] : row;
            a[u] = ok ? v.vs[q + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (j[u] != row) {
                ldrow_pol<K>(x + (size_t)j[u] * VS<K>::S, xv[u], xpol);
            } else {
#pragma unroll
                for (int c = 0; c < K; ++c) xv[u][c] = 0.0;
            }
        }
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

template <int K, int MODE, int UNR = PipeUnroll<K>::value>
__global__ void __launch_bounds__(kTile, UNR >= 8 && K >= 3 ? 3 : 4) k_tile_pipe(const TileDesc* __restrict__ tiles, int t_begin, int t_end,
                                                     const int* __restrict__ rp, const int* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ b,
                                                     double* __restrict__ x, double* __restrict__ r,
                                                     double* __restrict__ partial, int cap, double omega, int rev) {
    extern __shared__ __align__(128) unsigned char smem_pipe[];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const size_t sb = (stage_bytes(cap) + 127) / 128 * 128;
    unsigned char* stage[2] = {smem_pipe, smem_pipe + sb};
    GsTrace trc;
    trc.start();
    pdl_launch_dependents();
    const int nt = t_end - t_begin;
    const int mine = nt > (int)blockIdx.x ? (nt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    uint64_t pol = 0;
    if (tid == 0) {
        pol = evict_first_policy();
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 0; i < 2 && i < mine; ++i) {
            const TileDesc d = tiles[tile_ix(t_begin, t_end, blockIdx.x + i * gridDim.x, rev)];
            issue_tile(d, stage[i], cap, &bar[i], rp, col, val, pol);
        }
    }
    pdl_wait();
    trc.waited();
    const uint64_t xpol = evict_last_policy();
    const uint64_t spol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int i = 0; i < mine; ++i) {
        const int sidx = i & 1;
        const TileDesc d = tiles[tile_ix(t_begin, t_end, blockIdx.x + i * gridDim.x, rev)];
        mbar_wait(&bar[sidx], (unsigned)((i >> 1) & 1));
        const StageView v = view_tile(d, stage[sidx], cap);
        if (tid < d.nrow) {
            const int row = d.row0 + tid;
            // b (and the row's own x for the residual modes) go out before the
            // neighbour gathers so all loads of the row share one round trip
            double bv[K], xr[K];
            ldrow_pol<K>(b + (size_t)row * VS<K>::S, bv, spol);
            if (MODE != 0) ldrow_pol<K>(x + (size_t)row * VS<K>::S, xr, xpol);
            double s[K], dg;
            stage_row<K, UNR>(v, tid, row, x, s, dg, xpol);
            const double inv = (MODE == 0 || MODE == 3) ? 1.0 / dg : 0.0;
            if (MODE == 0) {
                double xn[K];
#pragma unroll
                for (int c = 0; c < K; ++c) xn[c] = div_by(bv[c] - s[c], dg, inv);
                strow_pol<K>(x + (size_t)row * VS<K>::S, xn, xpol);
            } else {
                double rr[K];
#pragma unroll
                for (int c = 0; c < K; ++c) rr[c] = bv[c] - fma(dg, xr[c], s[c]);
                if (MODE == 1) {
                    strow_pol<K>(r + (size_t)row * VS<K>::S, rr, xpol);
                } else if (MODE == 3) {
                    double xo[K];
#pragma unroll
                    for (int c = 0; c < K; ++c) xo[c] = xr[c] + div_by(omega * rr[c], dg, inv);
                    strow_pol<K>(r + (size_t)row * VS<K>::S, xo, xpol);
                } else {
#pragma unroll
                    for (int c = 0; c < K; ++c) acc[c] = fma(rr[c], rr[c], acc[c]);
                }
            }
        }
        __syncthreads();   // stage sidx fully consumed
        if (tid == 0 && i + 2 < mine) {
            const TileDesc dn = tiles[tile_ix(t_begin, t_end, blockIdx.x + (i + 2) * gridDim.x, rev)];
            issue_tile(dn, stage[sidx], cap, &bar[sidx], rp, col, val, pol);
        }
    }
    if (MODE == 0) trc.end(1, t_begin);
    if (MODE == 2) {
        __shared__ double red[kTile / 32][K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double vsum = warp_sum(acc[c]);
            if ((tid & 31) == 0) red[tid >> 5][c] = vsum;
        }
        __syncthreads();
        if (tid < K) {
            double vsum = 0.0;
            for (int w = 0; w < kTile / 32; ++w) vsum += red[w][tid];
            partial[blockIdx.x * K + tid] = vsum;
        }
    }
}

// Pipelined tiles with LPR lanes per row (levels with longer rows, e.g. the
// first Galerkin level): the same TMA-bulk double-buffered stage ring as
// k_tile_pipe, tiles of kTile / LPR rows; lane l of a row takes the staged
// entries qb + l + u * LPR (the assignment and summation order of
// k_lpr_sweep), so nothing but x and b is loaded after the PDL wait.
template <int K, int LPR, int MODE>
__global__ void __launch_bounds__(kTile, 3) k_tile_pipe_lpr(const TileDesc* __restrict__ tiles, int t_begin, int t_end,
                                                         const int* __restrict__ rp, const int* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ b,
                                                         double* __restrict__ x, double* __restrict__ r,
                                                         double* __restrict__ partial, int cap, double omega, int rev) {
    extern __shared__ __align__(128) unsigned char smem_pipe[];
    __shared__ __align__(8) uint64_t bar[2];
    constexpr int GB = 4;   // gathers in flight per lane (8 with 2 CTAs/SM measured slower)
    const int tid = threadIdx.x;
    const int tr = tid / LPR;
    const int lane = tid & (LPR - 1);
    const size_t sb = (stage_bytes(cap) + 127) / 128 * 128;
    unsigned char* stage[2] = {smem_pipe, smem_pipe + sb};
    GsTrace trc;
    trc.start();
    pdl_launch_dependents();
    const int nt = t_end - t_begin;
    const int mine = nt > (int)blockIdx.x ? (nt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    uint64_t pol = 0;
    if (tid == 0) {
        pol = evict_first_policy();
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 0; i < 2 && i < mine; ++i) {
            const TileDesc d = tiles[tile_ix(t_begin, t_end, blockIdx.x + i * gridDim.x, rev)];
            issue_tile(d, stage[i], cap, &bar[i], rp, col, val, pol);
        }
    }
    pdl_wait();
    trc.waited();
    const uint64_t xpol = evict_last_policy();
    const uint64_t spol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int i = 0; i < mine; ++i) {
        const int sidx = i & 1;
        const TileDesc d = tiles[tile_ix(t_begin, t_end, blockIdx.x + i * gridDim.x, rev)];
        mbar_wait(&bar[sidx], (unsigned)((i >> 1) & 1));
        const StageView v = view_tile(d, stage[sidx], cap);
        const bool valid = tr < d.nrow;
        const int row = d.row0 + tr;
        double bv[K];
        if (valid && lane == 0) ldrow_pol<K>(b + (size_t)row * VS<K>::S, bv, spol);
        const int qb = valid ? v.rps[tr] : 0, qe = valid ? v.rps[tr + 1] : 0;
        double s[K], xi[K], dg = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = xi[c] = 0.0;
        for (int q0 = qb + lane; q0 < qe; q0 += GB * LPR) {
            int j[GB];
            double a[GB];
            double xv[GB][K];
#pragma unroll
            for (int u = 0; u < GB; ++u) {
                const int q = q0 + u * LPR;
                j[u] = q < qe ? v.cs[q] : -1;
                a[u] = q < qe ? v.vs[q] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < GB; ++u)
                if (j[u] >= 0 && (MODE != 0 || j[u] != row)) ldrow_pol<K>(x + (size_t)j[u] * VS<K>::S, xv[u], xpol);
#pragma unroll
            for (int u = 0; u < GB; ++u) {
                if (j[u] < 0) continue;
                if (MODE == 0 && j[u] == row) {
                    dg += a[u];
                } else {
                    if (MODE == 3 && j[u] == row) {
                        dg += a[u];
#pragma unroll
                        for (int c = 0; c < K; ++c) xi[c] = xv[u][c];
                    }
#pragma unroll
                    for (int c = 0; c < K; ++c) s[c] = fma(a[u], xv[u][c], s[c]);
                }
            }
        }
        // groups never straddle a warp; every lane of the warp takes part
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], 0xffffffffu);
        if (MODE == 0 || MODE == 3) dg = group_sum<LPR>(dg, 0xffffffffu);
        if (MODE == 3)
#pragma unroll
            for (int c = 0; c < K; ++c) xi[c] = group_sum<LPR>(xi[c], 0xffffffffu);
        if (valid && lane == 0) {
            double out[K];
            const double inv = (MODE == 0 || MODE == 3) ? 1.0 / dg : 0.0;
#pragma unroll
            for (int c = 0; c < K; ++c)
                out[c] = MODE == 0 ? div_by(bv[c] - s[c], dg, inv)
                                   : MODE == 3 ? xi[c] + div_by(omega * (bv[c] - s[c]), dg, inv) : bv[c] - s[c];
            if (MODE == 0) strow_pol<K>(x + (size_t)row * VS<K>::S, out, xpol);
            else if (MODE != 2) strow_pol<K>(r + (size_t)row * VS<K>::S, out, xpol);
            else
#pragma unroll
                for (int c = 0; c < K; ++c) acc[c] = fma(out[c], out[c], acc[c]);
        }
        __syncthreads();   // stage sidx fully consumed
        if (tid == 0 && i + 2 < mine) {
            const TileDesc dn = tiles[tile_ix(t_begin, t_end, blockIdx.x + (i + 2) * gridDim.x, rev)];
            issue_tile(dn, stage[sidx], cap, &bar[sidx], rp, col, val, pol);
        }
    }
    if (MODE == 0) trc.end(2, t_begin);
    if (MODE == 2) {
        __shared__ double red[kTile / 32][K];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double vsum = warp_sum(acc[c]);
            if ((tid & 31) == 0) red[tid >> 5][c] = vsum;
        }
        __syncthreads();
        if (tid < K) {
            double vsum = 0.0;
            for (int w = 0; w < kTile / 32; ++w) vsum += red[w][tid];
            partial[blockIdx.x * K + tid] = vsum;
        }
    }
}

// One-tile form of the k_tile_pipe_lpr GS pass, for colour classes whose
// tiles all fit the resident grid (one tile per CTA: levels 1-2 of the large
// configs).  One stage of shared memory and <= 64 registers, so 4 CTAs fit an
// SM and the CTAs of the NEXT colour pass (launched programmatically as soon
// as this pass's CTAs have started) are resident beside this pass's: their
// prologue - tile descriptor, TMA bulk copies of the row pointers / columns /
// values - runs under this pass, and after griddepcontrol.wait only the x
// gathers remain on the critical path.  With the two-stage kernel (3 CTAs of
// 80 registers and two stages per SM) most of the next pass's CTAs could not
// become resident before this pass's left.  Same lane assignment and
// summation order as k_tile_pipe_lpr: bitwise the same iterate.
template <int K, int LPR>
__global__ void __launch_bounds__(kTile, 4) k_tile_one_lpr(const TileDesc* __restrict__ tiles, int t_begin,
                                                           const int* __restrict__ rp, const int* __restrict__ col,
                                                           const double* __restrict__ val, const double* __restrict__ b,
                                                           double* __restrict__ x, int cap) {
    extern __shared__ __align__(128) unsigned char smem_pipe[];
    __shared__ __align__(8) uint64_t bar;
    constexpr int GB = 4;
    const int tid = threadIdx.x;
    const int tr = tid / LPR;
    const int lane = tid & (LPR - 1);
    GsTrace trc;
    trc.start();
    pdl_launch_dependents();
    const TileDesc d = tiles[t_begin + (int)blockIdx.x];
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue_tile(d, smem_pipe, cap, &bar, rp, col, val, evict_first_policy());
    }
    __syncthreads();
    const uint64_t xpol = evict_last_policy();
    const uint64_t spol = evict_first_policy();
    const StageView v = view_tile(d, smem_pipe, cap);
    const bool valid = tr < d.nrow;
    const int row = d.row0 + tr;
    // the tile lands under the previous pass; the diagonal's group sum and
    // reciprocal are formed before the wait (one nonzero term: exact)
    mbar_wait(&bar, 0u);
    const int qb = valid ? v.rps[tr] : 0, qe = valid ? v.rps[tr + 1] : 0;
    double dg = 0.0;
    for (int q = qb + lane; q < qe; q += LPR)
        if (v.cs[q] == row) dg = v.vs[q];
    dg = group_sum<LPR>(dg, 0xffffffffu);
    const double inv = 1.0 / dg;
    pdl_wait();
    trc.waited();
    double bv[K];
    if (valid && lane == 0) ldrow_pol<K>(b + (size_t)row * VS<K>::S, bv, spol);
    double s[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    for (int q0 = qb + lane; q0 < qe; q0 += GB * LPR) {
        int j[GB];
        double a[GB];
        double xv[GB][K];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
            const int q = q0 + u * LPR;
            j[u] = q < qe ? v.cs[q] : -1;
            a[u] = q < qe ? v.vs[q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GB; ++u)
            if (j[u] >= 0 && j[u] != row) ldrow_pol<K>(x + (size_t)j[u] * VS<K>::S, xv[u], xpol);
#pragma unroll
        for (int u = 0; u < GB; ++u) {
            if (j[u] < 0) continue;
            if (j[u] != row) {
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a[u], xv[u][c], s[c]);
            }
        }
    }
    // groups never straddle a warp; every lane of the warp takes part
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], 0xffffffffu);
    if (valid && lane == 0) {
        double out[K];
#pragma unroll
        for (int c = 0; c < K; ++c) out[c] = div_by(bv[c] - s[c], dg, inv);
        strow_pol<K>(x + (size_t)row * VS<K>::S, out, xpol);
    }
    trc.end(3, t_begin);
}

// ---------------------------------------------------------------------------
// LPR lanes per row (levels with long rows: Galerkin fill).  Each lane
// prefetches up to U = 32/LPR (col, val) of its row in the PDL prologue;
// after the wait its x gathers go out in batches of GB independent loads.
// The group width is chosen per level so that one colour pass is about one
// wave of the GPU (see choose_lpr in mg_host.cpp).
#ifndef MG_LPR_WIDE_ENTRIES
#define MG_LPR_WIDE_ENTRIES 64   // entries per row prefetched by the 16- and 32-lane groups
#endif
template <int K, int LPR, int MODE>
__global__ void __launch_bounds__(kBlock, LPR == 4 ? 4 : 1) k_lpr_sweep(const int* __restrict__ rp, const int* __restrict__ col,
                                                      const double* __restrict__ val, const double* __restrict__ b,
                                                      double* __restrict__ x, double* __restrict__ r, int r0, int r1,
                                                      double omega) {
    // entries prefetched per lane: 64 per row for the wide groups (Galerkin
    // rows reach ~40 entries; an entry left to the tail loop costs two more
    // dependent round trips after the wait - tools/gs_trace.py: the CTAs
    // holding such rows ended 1.1-1.3 us after the release against a median
    // of 0.7), 32 per row otherwise
    constexpr int U = LPR >= 16 ? MG_LPR_WIDE_ENTRIES / LPR : 32 / LPR;
    // gathers in flight per lane: the whole prefetch for LPR >= 8, batches of
    // 4 for LPR = 4 (8 entries per lane) to keep registers / occupancy
    constexpr int GB = U <= 4 ? U : 4;
    const int g = (int)(blockIdx.x * blockDim.x + threadIdx.x) / LPR;
    const int lane = threadIdx.x & (LPR - 1);
    const int row = r0 + g;
    GsTrace trc;
    trc.start();
    pdl_launch_dependents();
    const bool active = row < r1;
    const uint64_t pol = evict_first_policy();
    int e0 = 0, e1 = 0;
    int j[U];
    double a[U];
    if (active) {
        e0 = rp[row];
        e1 = rp[row + 1];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int e = e0 + lane + u * LPR;
        const bool ok = active && e < e1;
        j[u] = ok ? ld_stream(col + e, pol) : -1;
        a[u] = ok ? ld_stream(val + e, pol) : 0.0;
    }
    // the diagonal entry is among the lane's prefetched (or tail) entries:
    // its group sum and reciprocal are formed before the wait, off the
    // critical path of the colour pass (one nonzero term: exact)
    const unsigned mask = group_mask(LPR);
    double d = 0.0, inv = 0.0;
    if (MODE == 0 || MODE == 3) {
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j[u] == row) d = a[u];
        for (int e = e0 + lane + U * LPR; e < e1; e += LPR)
            if (ld_stream(col + e, pol) == row) d = ld_stream(val + e, pol);
        d = group_sum<LPR>(d, mask);
        inv = 1.0 / d;
    }
    pdl_wait();
    trc.waited();
    if (!active) return;   // whole groups leave together
    const uint64_t xpol = evict_last_policy();
    // the row's right-hand side goes out with the gathers (one round trip)
    double bv[K];
    if (lane == 0) ldrow<K>(b + (size_t)row * VS<K>::S, bv);
    double s[K], xi[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = xi[c] = 0.0;
#pragma unroll
    for (int u0 = 0; u0 < U; u0 += GB) {
        double xv[GB][K];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
            const int jj = j[u0 + u];
            if (jj >= 0 && (MODE != 0 || jj != row)) ldrow_pol<K>(x + (size_t)jj * VS<K>::S, xv[u], xpol);
        }
#pragma unroll
        for (int u = 0; u < GB; ++u) {
            const int jj = j[u0 + u];
            if (jj < 0) continue;
            if (MODE == 0 && jj == row) {
            } else {
                if (MODE == 3 && jj == row) {
#pragma unroll
                    for (int c = 0; c < K; ++c) xi[c] = xv[u][c];
                }
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a[u0 + u], xv[u][c], s[c]);
            }
        }
    }
    for (int e = e0 + lane + U * LPR; e < e1; e += LPR) {
        const int jj = ld_stream(col + e, pol);
        const double av = ld_stream(val + e, pol);
        if (MODE == 0 && jj == row) {
        } else {
            double xv[K];
            ldrow_pol<K>(x + (size_t)jj * VS<K>::S, xv, xpol);
            if (MODE == 3 && jj == row) {
#pragma unroll
                for (int c = 0; c < K; ++c) xi[c] = xv[c];
            }
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = fma(av, xv[c], s[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], mask);
    if (MODE == 3)
#pragma unroll
        for (int c = 0; c < K; ++c) xi[c] = group_sum<LPR>(xi[c], mask);   // only the diagonal's lane holds x_i
    if (lane == 0) {
        double out[K];
#pragma unroll
        for (int c = 0; c < K; ++c)
            out[c] = MODE == 0 ? div_by(bv[c] - s[c], d, inv)
                               : MODE == 3 ? xi[c] + div_by(omega * (bv[c] - s[c]), d, inv) : bv[c] - s[c];
        if (MODE == 0) strow_pol<K>(x + (size_t)row * VS<K>::S, out, xpol);
        else strow<K>(r + (size_t)row * VS<K>::S, out);
    }
    if (MODE == 0) trc.end(4, r0);
}

// ---------------------------------------------------------------------------
// K5b: r_c = P^T r gathered through the children lists of the coarse
// vertices (transpose of P): deterministic, no atomics.  G lanes per coarse
// row; children indices and weights prefetched before the wait.  Zeroes the
// coarse iterate (the recursive V-cycle starts from 0).
// G lanes per coarse row, U children per lane prefetched before the PDL wait;
// after it every lane issues its U residual gathers at once (children beyond
// G * U in a tail loop).  The kernel is latency-bound: ~30 waves of a 3-deep
// dependent chain (children offsets -> children -> residual rows), so fewer
// lanes per row (fewer waves) win while G * U still covers a typical coarse
// row (~12 children).  Measured on B200 (C4, residual + restriction ms/step,
// level 0 / level 1): 8 x 4 1.30 / 0.634, 8 x 2 1.13 / 0.601, 4 x 8 1.41 /
// 0.644, 4 x 4 1.06 / 0.614 (profiles/r02/restrict_ab.txt; round 1: 16 x 2
// 225 us/cycle against 8 x 4 191 at level 0).
#ifndef MG_RESTRICT_G
#define MG_RESTRICT_G 4
#endif
#ifndef MG_RESTRICT_U
#define MG_RESTRICT_U 4
#endif
constexpr int kRestrictG = MG_RESTRICT_G;
template <int K, int G, int U = 32 / G>
__global__ void __launch_bounds__(kBlock) k_restrict(const int* __restrict__ cptr, const int* __restrict__ cidx,
                                                     const double* __restrict__ cw, const double* __restrict__ r,
                                                     double* __restrict__ bc, double* __restrict__ xc, int nc,
                                                     const int* __restrict__ order) {
    const int g = (blockIdx.x * kBlock + threadIdx.x) / G;
    const int lane = threadIdx.x & (G - 1);
    pdl_launch_dependents();
    const bool active = g < nc;
    // coarse rows in locality order (all colours interleaved): the children's
    // residual rows are then gathered from a small spatial window (L2 hits)
    // ordered mode: the lists (cptr, cidx, cw) are already in visiting order
    // g; order[g] only names the output row
    const int I = active ? (order ? order[g] : g) : 0;
    const int L = order ? g : I;
    int t0 = 0, t1 = 0;
    int ii[U];
    double ww[U];
    if (active) {
        t0 = cptr[L];
        t1 = cptr[L + 1];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int t = t0 + lane + u * G;
        ii[u] = (active && t < t1) ? cidx[t] : -1;
        ww[u] = (active && t < t1) ? cw[t] : 0.0;
    }
    pdl_wait();
    if (!active) return;
    const unsigned mask = group_mask(G);
    double s[K];
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = 0.0;
    double rv[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ii[u] >= 0) ldrow<K>(r + (size_t)ii[u] * VS<K>::S, rv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
        if (ii[u] >= 0)
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = fma(ww[u], rv[u][c], s[c]);
    for (int t = t0 + lane + U * G; t < t1; t += G) {
        const int i = cidx[t];
        const double w = cw[t];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = fma(w, r[(size_t)i * VS<K>::S + c], s[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) s[c] = group_sum<G>(s[c], mask);
    if (lane < K) {
        double v = s[0];
#pragma unroll
        for (int c = 1; c < K; ++c)
            if (lane == c) v = s[c];
        bc[(size_t)I * VS<K>::S + lane] = v;
        xc[(size_t)I * VS<K>::S + lane] = 0.0;
    }
}

// K6: x <- x + P c (ELL-3, SoA [3][n]).
template <int K>
__global__ void __launch_bounds__(kBlock) k_prolong(const int* __restrict__ pc, const double* __restrict__ pw,
                                                    const double* __restrict__ xc, double* __restrict__ x, int n) {
    const int i = blockIdx.x * kBlock + threadIdx.x;
    pdl_launch_dependents();
    int c0 = 0, c1 = 0, c2 = 0;
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    if (i < n) {
        c0 = pc[i];
        c1 = pc[n + i];
        c2 = pc[2 * n + i];
        w0 = pw[i];
        w1 = pw[n + i];
        w2 = pw[2 * n + i];
    }
    pdl_wait();
    if (i >= n) return;
    double y0[K], y1[K], y2[K], xi[K];
    ldrow<K>(xc + (size_t)c0 * VS<K>::S, y0);
    ldrow<K>(xc + (size_t)c1 * VS<K>::S, y1);
    ldrow<K>(xc + (size_t)c2 * VS<K>::S, y2);
    ldrow<K>(x + (size_t)i * VS<K>::S, xi);
#pragma unroll
    for (int c = 0; c < K; ++c) {
        double v = w0 * y0[c];
        v = fma(w1, y1[c], v);
        v = fma(w2, y2[c], v);
        xi[c] += v;
    }
    strow<K>(x + (size_t)i * VS<K>::S, xi);
}

// K7b: coarsest solve x = A_H^{-1} b, one warp per row of the explicit
// inverse (prefetched into registers before the wait).
template <int K>
__global__ void __launch_bounds__(256) k_coarse_gemv(const double* __restrict__ Z, int npad, int n,
                                                     const double* __restrict__ b, double* __restrict__ x) {
    constexpr int U = 32;   // covers n <= 1024 from registers
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    pdl_launch_dependents();
    double z[U];
    const double* Zr = Z + (size_t)min(row, n - 1) * npad;
#pragma unroll
    for (int u = 0; u < U; ++u) z[u] = (lane + 32 * u < n) ? Zr[lane + 32 * u] : 0.0;
    pdl_wait();
    if (row >= n) return;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int j = lane + 32 * u;
        if (j < n)
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = fma(z[u], b[(size_t)j * VS<K>::S + c], acc[c]);
    }
    for (int j = lane + 32 * U; j < n; j += 32)
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(Zr[j], b[(size_t)j * VS<K>::S + c], acc[c]);
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < K; ++c) x[(size_t)row * VS<K>::S + c] = acc[c];
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
    pdl_launch_dependents();
    pdl_wait();
    double* y = sm;                       // [npad][K]
    double* red = sm + (size_t)npad * K;  // [32][32][K]
    double* t = red + 32 * 32 * K;        // [32][K]
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    for (int i = tid; i < npad * K; i += 1024) y[i] = (i < n * K) ? b[(size_t)(i / K) * VS<K>::S + i % K] : 0.0;
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
    for (int i = tid; i < n * K; i += 1024) x[(size_t)(i / K) * VS<K>::S + i % K] = y[i];
}

// ---------------------------------------------------------------------------
// K3: residual norms: block partial sums of (b - A x)^2 per column (tiled or
// LPR rows), then one deterministic single-block finalisation.
constexpr int kNormBlocks = 1184;   // 8 x 148 SMs

template <int K>
__device__ __forceinline__ void block_partial(double (&acc)[K], double* partial) {
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

template <int K>
__global__ void __launch_bounds__(kTile) k_resnorm_tiled(const int* __restrict__ rp, const int* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ b, const double* __restrict__ x,
                                                         double* __restrict__ partial, int n, int cap) {
    extern __shared__ double smem_d[];
    __shared__ int rps[kTile + 1];
    double* vs = smem_d;
    int* cs = reinterpret_cast<int*>(smem_d + cap);
    pdl_launch_dependents();
    const uint64_t pol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const int ntiles = (n + kTile - 1) / kTile;
    bool waited = false;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row0 = tile * kTile;
        const int nrow = min(kTile, n - row0);
        const int e0 = tile_stage(rp, col, val, row0, nrow, rps, cs, vs, pol);
        if (!waited) {
            pdl_wait();
            waited = true;
        }
        const int t = threadIdx.x;
        if (t < nrow) {
            const int row = row0 + t;
            double s[K], d;
            tile_row<K, Unroll<K>::value>(cs, vs, rps[t] - e0, rps[t + 1] - e0, row, x, s, d);
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double rr = b[(size_t)row * VS<K>::S + c] - fma(d, x[(size_t)row * VS<K>::S + c], s[c]);
                acc[c] = fma(rr, rr, acc[c]);
            }
        }
        __syncthreads();
    }
    if (!waited) pdl_wait();
    block_partial<K>(acc, partial);
}

template <int K, int LPR>
__global__ void __launch_bounds__(kBlock) k_resnorm_lpr(const int* __restrict__ rp, const int* __restrict__ col,
                                                        const double* __restrict__ val, const double* __restrict__ b,
                                                        const double* __restrict__ x, double* __restrict__ partial,
                                                        int n) {
    pdl_launch_dependents();
    pdl_wait();
    const int lane = threadIdx.x & (LPR - 1);
    const uint64_t pol = evict_first_policy();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    const int groups = gridDim.x * (kBlock / LPR);
    const int g0 = (blockIdx.x * kBlock + threadIdx.x) / LPR;
    // iterate whole groups together: every group runs the same trip count
    for (int base = 0; base < n; base += groups) {
        const int row = base + g0;
        const bool active = row < n;
        const unsigned mask = group_mask(LPR);
        double s[K];
#pragma unroll
        for (int c = 0; c < K; ++c) s[c] = 0.0;
        if (active) {
            for (int e = rp[row] + lane; e < rp[row + 1]; e += LPR) {
                const int j = ld_stream(col + e, pol);
                const double a = ld_stream(val + e, pol);
#pragma unroll
                for (int c = 0; c < K; ++c) s[c] = fma(a, x[(size_t)j * VS<K>::S + c], s[c]);
            }
        }
        if (active) {
#pragma unroll
            for (int c = 0; c < K; ++c) s[c] = group_sum<LPR>(s[c], mask);
            if (lane == 0)
#pragma unroll
                for (int c = 0; c < K; ++c) {
                    const double rr = b[(size_t)row * VS<K>::S + c] - s[c];
                    acc[c] = fma(rr, rr, acc[c]);
                }
        }
    }
    block_partial<K>(acc, partial);
}

// out[c] = sqrt(sum_b partial[b][c]) / (denom[c] > 0 ? denom[c] : 1)   (denom may be null)
template <int K>
__global__ void __launch_bounds__(kBlock) k_norm_finalize(const double* __restrict__ partial, int nblk_,
                                                          const double* __restrict__ denom,
                                                          double* __restrict__ out) {
    pdl_launch_dependents();
    pdl_wait();
    __shared__ double red[kBlock / 32][K];
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int t = threadIdx.x; t < nblk_; t += kBlock)
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
        v = sqrt(v);
        if (denom) {
            const double d = denom[threadIdx.x];
            v = v / (d > 0.0 ? d : 1.0);
        }
        out[threadIdx.x] = v;
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_sumsq_partial(const double* __restrict__ v, int n,
                                                          double* __restrict__ partial) {
    pdl_launch_dependents();
    pdl_wait();
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock)
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double t = v[(size_t)i * VS<K>::S + c];
            acc[c] = fma(t, t, acc[c]);
        }
    block_partial<K>(acc, partial);
}

// ---------------------------------------------------------------------------
inline size_t tile_smem(int cap) { return (size_t)cap * (sizeof(double) + sizeof(int)); }

inline int pipe_nsm() {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    return nsm;
}
// persistent grid: every CTA resident at once (registers: 4 CTAs/SM for the
// thread-per-row kernel, 3 for the lanes-per-row and 8-gather variants)
inline int pipe_per_sm(const Level& L, int K) { return (L.pipe_lpr > 1 || (K == 3 && L.pipe_unr8)) ? 3 : 4; }
// the tile set balanced for that residency (setup_pattern, mg_host.cpp)
inline const std::vector<int32_t>& pipe_tiles(const Level& L, int K) {
    return pipe_per_sm(L, K) == 3 ? L.tile_off : L.tile_off4;
}
inline int pipe_grid(const Level& L, int K, int ntiles) {
    const size_t smem = 2 * ((stage_bytes(L.pipe_cap) + 127) / 128 * 128) + 2048;
    const int by_regs = pipe_per_sm(L, K);
    const int per_sm = std::max(1, std::min<int>(by_regs, (int)((227 * 1024) / smem)));
    return std::max(1, std::min(ntiles, pipe_nsm() * per_sm));
}
inline size_t pipe_smem(int cap) { return 2 * ((stage_bytes(cap) + 127) / 128 * 128); }
// k_tile_one_lpr: every tile of the pass on its own resident CTA (4 per SM by
// registers, one stage of shared memory each)
#ifndef MG_ONE_TILE
#define MG_ONE_TILE 1
#endif
#ifndef MG_ONE_TILE_MIN_LPR
#define MG_ONE_TILE_MIN_LPR 2
#endif
inline bool one_tile_ok(const Level& L, int ntiles) {
    const size_t smem = pipe_smem(L.pipe_cap) / 2 + 1280;
    const int per_sm = std::min<int>(4, (int)((227 * 1024) / smem));
    return MG_ONE_TILE && ntiles <= pipe_nsm() * per_sm;
}

// MODE 0..3 over tiles [t0, t1) of level L (iterate read from xin)
template <int K, int MODE>
void pipe_launch(const Level& L, int t0, int t1, double* xin, double* r, double* partial, int grid, double omega,
                 bool pdl, cudaStream_t s) {
    const TileDesc* td = reinterpret_cast<const TileDesc*>(L.tiles.p);
    const size_t sm = pipe_smem(L.pipe_cap);
    const int rev = (MODE != 2 && L.serpentine) ? (L.pass_ctr++ & 1) : 0;   // norm partials keep one order
    if (MODE == 0 && L.pipe_lpr >= MG_ONE_TILE_MIN_LPR && one_tile_ok(L, t1 - t0)) {
        const size_t sm1 = sm / 2;
        const int g1 = t1 - t0;
        switch (L.pipe_lpr) {
            case 2: launch_k(pdl, k_tile_one_lpr<K, 2>, g1, kTile, sm1, s, td, t0, L.rp.p, L.col.p, L.val.p, L.b.p, xin, L.pipe_cap); break;
            case 4: launch_k(pdl, k_tile_one_lpr<K, 4>, g1, kTile, sm1, s, td, t0, L.rp.p, L.col.p, L.val.p, L.b.p, xin, L.pipe_cap); break;
            default: launch_k(pdl, k_tile_one_lpr<K, 8>, g1, kTile, sm1, s, td, t0, L.rp.p, L.col.p, L.val.p, L.b.p, xin, L.pipe_cap); break;
        }
        return;
    }
    switch (L.pipe_lpr) {
        case 1:
            if (K == 3 && L.pipe_unr8)
                launch_k(pdl, k_tile_pipe<K, MODE, 8>, grid, kTile, sm, s, td, t0, t1, L.rp.p, L.col.p, L.val.p, L.b.p, xin, r, partial, L.pipe_cap, omega, rev);
            else
                launch_k(pdl, k_tile_pipe<K, MODE>, grid, kTile, sm, s, td, t0, t1, L.rp.p, L.col.p, L.val.p, L.b.p, xin, r, partial, L.pipe_cap, omega, rev);
            break;
        case 2: launch_k(pdl, k_tile_pipe_lpr<K, 2, MODE>, grid, kTile, sm, s, td, t0, t1, L.rp.p, L.col.p, L.val.p, L.b.p, xin, r, partial, L.pipe_cap, omega, rev); break;
        case 4: launch_k(pdl, k_tile_pipe_lpr<K, 4, MODE>, grid, kTile, sm, s, td, t0, t1, L.rp.p, L.col.p, L.val.p, L.b.p, xin, r, partial, L.pipe_cap, omega, rev); break;
        default: launch_k(pdl, k_tile_pipe_lpr<K, 8, MODE>, grid, kTile, sm, s, td, t0, t1, L.rp.p, L.col.p, L.val.p, L.b.p, xin, r, partial, L.pipe_cap, omega, rev); break;
    }
}

// MODE 0: GS pass on rows [r0, r1) in place on L.x; MODE 1: r = b - A x;
// MODE 3: Jacobi out = x + omega D^{-1}(b - A x).  xin: iterate read (L.x if null).
template <int K, int MODE>
int sweep_k(const Level& L, int r0, int r1, double* r, bool pdl, cudaStream_t s, double* xin = nullptr,
            double omega = 0.0) {
    double* xp = xin ? xin : L.x.p;
    const int rows = r1 - r0;
    if (rows <= 0) return 0;
    if (L.pipe) {
        // tile range of this colour class (GS) or of the whole level (residual)
        int t0, t1;
        const std::vector<int32_t>& toff = pipe_tiles(L, K);
        if (MODE == 0) {
            int c = 0;
            while (L.colour_off[c] != r0) ++c;
            t0 = toff[c];
            t1 = toff[c + 1];
        } else {
            t0 = toff[toff.size() - 2];   // whole-level tiles are the last range
            t1 = toff.back();
        }
        pipe_launch<K, MODE>(L, t0, t1, xp, r, nullptr, pipe_grid(L, K, t1 - t0), omega, pdl, s);
        return 1;
    }
    if (L.tiled) {
        const int cap = MODE == 0 ? L.cap_gs : L.cap_all;
        launch_k(pdl, k_tile_sweep<K, MODE>, nblk(rows, kTile), kTile, tile_smem(cap), s, L.rp.p, L.col.p, L.val.p,
                 L.b.p, xp, r, r0, r1, cap, omega);
        return 1;
    }
    const int lpr = MODE == 0 ? L.lpr : L.lpr_all;
    // a GS colour pass that would not put a 256-thread CTA on every SM runs
    // 128-thread CTAs (its rows spread over twice the SMs: C4 levels 4 / 5
    // 1.08 / 0.96 -> 1.00 / 0.93 ms/step; passes of more CTAs than SMs measured
    // slower that way, C4 level 3 1.35 -> 1.42; profiles/r02/lpr_block_ab.txt)
    const int blk = (MODE == 0 && lpr >= 16 && nblk((int64_t)rows * lpr, kBlock) < pipe_nsm()) ? kBlock / 2 : kBlock;
    const int grid = nblk((int64_t)rows * lpr, blk);
    switch (lpr) {
        case 4: launch_k(pdl, k_lpr_sweep<K, 4, MODE>, grid, blk, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, xp, r, r0, r1, omega); break;
        case 8: launch_k(pdl, k_lpr_sweep<K, 8, MODE>, grid, blk, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, xp, r, r0, r1, omega); break;
        case 16: launch_k(pdl, k_lpr_sweep<K, 16, MODE>, grid, blk, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, xp, r, r0, r1, omega); break;
        default: launch_k(pdl, k_lpr_sweep<K, 32, MODE>, grid, blk, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, xp, r, r0, r1, omega); break;
    }
    return 1;
}

template <int K>
int resnorm_k(const Level& L, double* partial, int nb, const double* bnorm, double* rho, bool pdl, cudaStream_t s) {
    int grid;
    if (L.pipe) {
        const std::vector<int32_t>& toff = pipe_tiles(L, K);
        const int t0 = toff[toff.size() - 2], t1 = toff.back();
        grid = std::min(nb, pipe_grid(L, K, t1 - t0));
        pipe_launch<K, 2>(L, t0, t1, L.x.p, nullptr, partial, grid, 0.0, pdl, s);
    } else if (L.tiled) {
        grid = std::min(nb, nblk(L.n, kTile));
        launch_k(pdl, k_resnorm_tiled<K>, grid, kTile, tile_smem(L.cap_all), s, L.rp.p, L.col.p, L.val.p, L.b.p,
                 L.x.p, partial, L.n, L.cap_all);
    } else {
        grid = std::min(nb, nblk((int64_t)L.n * L.lpr_all, kBlock));
        switch (L.lpr_all) {
            case 4: launch_k(pdl, k_resnorm_lpr<K, 4>, grid, kBlock, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
            case 8: launch_k(pdl, k_resnorm_lpr<K, 8>, grid, kBlock, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
            case 16: launch_k(pdl, k_resnorm_lpr<K, 16>, grid, kBlock, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
            default: launch_k(pdl, k_resnorm_lpr<K, 32>, grid, kBlock, 0, s, L.rp.p, L.col.p, L.val.p, L.b.p, L.x.p, partial, L.n); break;
        }
    }
    launch_k(pdl, k_norm_finalize<K>, 1, kBlock, 0, s, (const double*)partial, grid, bnorm, rho);
    return 2;
}

template <int K>
void set_attrs_k() {
    const int big = 200 * 1024;
    cudaFuncSetAttribute(k_tile_sweep<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_sweep<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_resnorm_tiled<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_chol_solve<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 0, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe<K, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_one_lpr<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_one_lpr<K, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_one_lpr<K, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 4, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 4, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_pipe_lpr<K, 8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_tile_sweep<K, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
}

#define MG_K_SWITCH(K, EXPR_T)                  \
    switch (K) {                                \
        case 1: { constexpr int KK = 1; return EXPR_T; } \
        case 2: { constexpr int KK = 2; return EXPR_T; } \
        case 3: { constexpr int KK = 3; return EXPR_T; } \
        default: { constexpr int KK = 4; return EXPR_T; } \
    }

}  // namespace

int resnorm_blocks(int) { return kNormBlocks; }
int tile_rows() { return kTile; }
size_t pipe_smem_bytes(int cap) { return pipe_smem(cap); }
size_t tile_smem_limit() { return 160 * 1024; }

void init_vcycle_attributes() {
    set_attrs_k<1>();
    set_attrs_k<2>();
    set_attrs_k<3>();
    set_attrs_k<4>();
}

int vc_gs(int K, const Level& L, int r0, int r1, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (sweep_k<KK, 0>(L, r0, r1, nullptr, pdl, s)))
}
// Device-side V-cycle loop (conditional WHILE graph node): after each cycle's
// residual norm this kernel records rho into the history, applies mg_solve's
// stopping rule (non-finite -> stop; every column rho <= tol -> stop; cycle
// budget spent -> stop) and sets the loop condition, so a whole solve is one
// graph launch and one host synchronisation.
template <int K>
__global__ void k_loop_check(const double* __restrict__ rho, LoopState* st, double* __restrict__ hist,
                             cudaGraphConditionalHandle h) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    const int cyc = st->cyc + 1;
    st->cyc = cyc;
    bool finite = true, done = st->tol > 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const double r = rho[j];
        hist[(size_t)cyc * K + j] = r;
        finite &= isfinite(r);
        done &= r <= st->tol;
    }
    st->status = !finite ? 2 : done ? 1 : 0;
    cudaGraphSetConditional(h, (finite && !done && cyc < st->max_cycles) ? 1u : 0u);
}

int vc_loop_check(int K, const double* rho, LoopState* st, double* hist, cudaGraphConditionalHandle h, cudaStream_t s) {
    switch (K) {
        case 1: k_loop_check<1><<<1, 32, 0, s>>>(rho, st, hist, h); break;
        case 2: k_loop_check<2><<<1, 32, 0, s>>>(rho, st, hist, h); break;
        case 3: k_loop_check<3><<<1, 32, 0, s>>>(rho, st, hist, h); break;
        default: k_loop_check<4><<<1, 32, 0, s>>>(rho, st, hist, h); break;
    }
    return 1;
}

int vc_jacobi(int K, const Level& L, double* xin, double* xout, double omega, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (sweep_k<KK, 3>(L, 0, L.n, xout, pdl, s, xin, omega)))
}
int vc_residual(int K, const Level& L, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (sweep_k<KK, 1>(L, 0, L.n, L.r.p, pdl, s)))
}
int vc_restrict(int K, const Level& C, const Level& F, bool pdl, cudaStream_t s) {
    const int G = kRestrictG;
    const bool ordered = C.restrict_ordered && C.rcptr.p;
    const int* ord = ordered ? (const int*)C.gal_order.p : nullptr;
    const int* cp = ordered ? (const int*)C.rcptr.p : (const int*)C.cptr.p;
    const int* ci = ordered ? (const int*)C.rcidx.p : (const int*)C.cidx.p;
    const double* cwp = ordered ? (const double*)C.rcw.p : (const double*)C.cw.p;
    switch (G) {
        case 4: MG_K_SWITCH(K, (launch_k(pdl, k_restrict<KK, 4, MG_RESTRICT_U>, nblk((int64_t)C.n * 4, kBlock), kBlock, 0, s, cp, ci, cwp, F.r.p, C.b.p, C.x.p, C.n, ord), 1))
        case 8: MG_K_SWITCH(K, (launch_k(pdl, k_restrict<KK, 8, MG_RESTRICT_U>, nblk((int64_t)C.n * 8, kBlock), kBlock, 0, s, cp, ci, cwp, F.r.p, C.b.p, C.x.p, C.n, ord), 1))
        case 16: MG_K_SWITCH(K, (launch_k(pdl, k_restrict<KK, 16>, nblk((int64_t)C.n * 16, kBlock), kBlock, 0, s, cp, ci, cwp, F.r.p, C.b.p, C.x.p, C.n, ord), 1))
        default: MG_K_SWITCH(K, (launch_k(pdl, k_restrict<KK, 8>, nblk((int64_t)C.n * 8, kBlock), kBlock, 0, s, cp, ci, cwp, F.r.p, C.b.p, C.x.p, C.n, ord), 1))
    }
}
int vc_prolong(int K, const Level& F, const Level& C, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (launch_k(pdl, k_prolong<KK>, nblk(F.n, kBlock), kBlock, 0, s, F.pc.p, F.pw.p, C.x.p, F.x.p, F.n), 1))
}
int vc_coarse_gemv(int K, const double* Z, int npad, int n, const double* b, double* x, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (launch_k(pdl, k_coarse_gemv<KK>, nblk(n, 8), 256, 0, s, Z, npad, n, b, x), 1))
}
int vc_coarse_trsv(int K, const double* L, const double* Linv, int npad, int n, const double* b, double* x, bool pdl,
                   cudaStream_t s) {
    MG_K_SWITCH(K, (launch_k(pdl, k_chol_solve<KK>, 1, 1024, sizeof(double) * ((size_t)npad * KK + 32 * 32 * KK + 32 * KK),
                             s, L, Linv, npad, n, b, x), 1))
}
int vc_resnorm(int K, const Level& L, double* partial, int nb, const double* bnorm, double* rho, bool pdl,
               cudaStream_t s) {
    MG_K_SWITCH(K, (resnorm_k<KK>(L, partial, nb, bnorm, rho, pdl, s)))
}
int vc_norm_finalize(int K, const double* partial, int nb, const double* denom, double* out, bool pdl, cudaStream_t s) {
    MG_K_SWITCH(K, (launch_k(pdl, k_norm_finalize<KK>, 1, kBlock, 0, s, partial, nb, denom, out), 1))
}
int vc_sumsq(int K, const double* v, int n, double* partial, int nb, double* out, cudaStream_t s) {
    const int grid = std::min(nb, std::max(1, nblk(n, kBlock)));
    MG_K_SWITCH(K, (launch_k(false, k_sumsq_partial<KK>, grid, kBlock, 0, s, v, n, partial),
                    launch_k(false, k_norm_finalize<KK>, 1, kBlock, 0, s, (const double*)partial, grid,
                             (const double*)nullptr, out),
                    2))
}

}  // namespace mg

#ifdef MG_GS_TRACE
// experiment builds only: copy out / reset the GS pass trace
extern "C" int mg_debug_gs_trace(unsigned long long* out, int max_entries, int reset) {
    unsigned n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, mg::g_gs_trace_n, sizeof(n));
    n = std::min(n, mg::kGsTraceCap);
    const int m = std::min<int>((int)n, max_entries);
    if (out && m > 0) cudaMemcpyFromSymbol(out, mg::g_gs_trace, (size_t)m * 4 * sizeof(unsigned long long));
    if (reset) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(mg::g_gs_trace_n, &z, sizeof(z));
    }
    return m;
}
#endif
