// Device helpers shared by the libmg kernel translation units (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "mg_internal.h"

namespace mg {

constexpr int kBlock = 256;

__host__ __device__ inline int nblk(int64_t n, int per) { return (int)((n + per - 1) / per); }

// ---- programmatic dependent launch (PDL) --------------------------------
// Kernels of the V-cycle chain are launched with programmatic stream
// serialisation: the next kernel is scheduled while the previous one drains,
// runs its prologue (loads of data no earlier kernel of the solve writes:
// matrix structure and values, prolongation, children lists) and only then
// waits for its predecessor's memory with griddepcontrol.wait.  Both
// instructions are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- cache-policy loads ---------------------------------------------------
// Streaming (read-once per sweep) matrix data: no L1 allocation, evict-first
// in L2 so the gathered iterate x stays resident.
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

// ---- GS / Jacobi quotient ---------------------------------------------------
// num / d for the K right-hand sides of a row with ONE division: q = num *
// (1/d), refined by one residual step q + (num - q d)(1/d).  Within an ulp of
// IEEE division (round-off level, like the FMA contraction of reading A18),
// and the same arithmetic for every K, so a column's iterate does not depend
// on how many columns are solved together.  Measured on B200: K = 3 fp64
// divisions on a row's critical path cost ~340 cycles more than one
// (tools/cluster_step_bench.cu).
__device__ __forceinline__ double div_by(double num, double d, double inv) {
    const double q = num * inv;
    return fma(fma(-q, d, num), inv, q);
}

// ---- sub-warp groups ----------------------------------------------------
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
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// ---- internal vector layout ------------------------------------------------
// Internal iterate / right-hand side / residual vectors are row-major with a
// row stride of VS<K>::S doubles: K rounded up to an aligned vector width
// (k = 3 is padded to 4 so every row is one 32-byte sector and one 256-bit
// load).  The user-facing [n][k] layout is converted by the permutation
// kernels.
template <int K>
struct VS {
    static constexpr int S = (K == 3) ? 4 : K;
};

template <int K>
__device__ __forceinline__ void ldrow(const double* p, double (&v)[K]) {
    if constexpr (K == 1) {
        v[0] = *p;
    } else if constexpr (K == 2) {
        asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p));
    } else if constexpr (K == 3) {
        double pad;
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(pad) : "l"(p));
    } else {
        asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
    }
}
// 32-byte read-only load (one sector, 256-bit): packed {w0, w1, w2, 0} P rows
__device__ __forceinline__ double4 ldg_d4(const double4* p) {
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// row load / store with an L2 eviction-priority policy (x: evict_last so the
// iterate stays resident across the colour passes; streams: evict_first)
template <int K>
__device__ __forceinline__ void ldrow_pol(const double* p, double (&v)[K], uint64_t pol) {
    if constexpr (K == 1) {
        asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[0]) : "l"(p), "l"(pol));
    } else if constexpr (K == 2) {
        asm volatile("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v[0]), "=d"(v[1]) : "l"(p), "l"(pol));
    } else if constexpr (K == 3) {
        double pad;
        asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(pad)
                     : "l"(p), "l"(pol));
    } else {
        asm volatile("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
                     : "l"(p), "l"(pol));
    }
}
template <int K>
__device__ __forceinline__ void strow_pol(double* p, const double (&v)[K], uint64_t pol) {
    if constexpr (K == 1) {
        asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v[0]), "l"(pol) : "memory");
    } else if constexpr (K == 2) {
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p), "d"(v[0]), "d"(v[1]), "l"(pol)
                     : "memory");
    } else if constexpr (K == 3) {
        asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v[0]), "d"(v[1]),
                     "d"(v[2]), "d"(0.0), "l"(pol)
                     : "memory");
    } else {
        asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "d"(v[0]), "d"(v[1]),
                     "d"(v[2]), "d"(v[3]), "l"(pol)
                     : "memory");
    }
}

// same through L2 only (data produced by other CTAs inside one launch)
template <int K>
__device__ __forceinline__ void ldrow_cg(const double* p, double (&v)[K]) {
    if constexpr (K == 1) {
        v[0] = __ldcg(p);
    } else if constexpr (K == 2) {
        asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "l"(p));
    } else if constexpr (K == 3) {
        double pad;
        asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(pad) : "l"(p));
    } else {
        asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
    }
}
template <int K>
__device__ __forceinline__ void strow(double* p, const double (&v)[K]) {
    if constexpr (K == 1) {
        *p = v[0];
    } else if constexpr (K == 2) {
        asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v[0]), "d"(v[1]) : "memory");
    } else if constexpr (K == 3) {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(0.0)
                     : "memory");
    } else {
        asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                     : "memory");
    }
}

// ---- host launch helper -------------------------------------------------
template <typename... KArgs, typename... Args>
inline void launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
    if (!pdl) {
        kern<<<grid, block, smem, s>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace mg
