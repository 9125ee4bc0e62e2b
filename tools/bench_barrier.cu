// Micro-benchmark (tools only, not part of libmg): cost of one dependent
// phase on B200, to choose between (a) one PDL kernel launch per GS colour
// pass inside a CUDA graph and (b) a persistent cooperative kernel with a
// software grid barrier between passes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb tools/bench_barrier.cu && /tmp/bb
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Monotone counter barrier: epoch e completes when the counter reaches e * nblocks.
__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        atom_add_release(ctr, 1u);
        while (ld_acquire(ctr) < target) {
        }
    }
    __syncthreads();
}

// Each phase: every CTA reads one value written by another CTA in the previous phase.
__global__ void k_persistent(unsigned* ctr, double* buf, int phases) {
    const unsigned nb = gridDim.x;
    double acc = 0.0;
    for (int ph = 0; ph < phases; ++ph) {
        if (threadIdx.x == 0) buf[(ph & 1) * 4096 + blockIdx.x] = acc + ph;
        grid_sync(ctr, nb * (unsigned)(ph + 1));
        acc += buf[(ph & 1) * 4096 + (blockIdx.x + 1) % nb];
    }
    if (threadIdx.x == 0) buf[8192 + blockIdx.x] = acc;
}

__global__ void k_cluster(double* buf, int phases) {
    double acc = 0.0;
    for (int ph = 0; ph < phases; ++ph) {
        if (threadIdx.x == 0) buf[(ph & 1) * 4096 + blockIdx.x] = acc + ph;
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        acc += __ldcg(buf + (ph & 1) * 4096 + (blockIdx.x + 1) % gridDim.x);
    }
    if (threadIdx.x == 0) buf[8192 + blockIdx.x] = acc;
}

// Generation barrier (count + gen), reusable across launches without a reset.
__device__ __forceinline__ void grid_sync_gen(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire(gen);
        if (atom_add_release(count, 1u) == gridDim.x - 1) {
            *count = 0;
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            while (ld_acquire(gen) == g) {
            }
        }
    }
    __syncthreads();
}
__global__ void k_persistent_gen(unsigned* count, unsigned* gen, double* buf, int phases) {
    double acc = 0.0;
    for (int ph = 0; ph < phases; ++ph) {
        if (threadIdx.x == 0) buf[(ph & 1) * 4096 + blockIdx.x] = acc + ph;
        grid_sync_gen(count, gen);
        acc += __ldcg(buf + (ph & 1) * 4096 + (blockIdx.x + 1) % gridDim.x);
    }
    if (threadIdx.x == 0) buf[8192 + blockIdx.x] = acc;
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__global__ void k_phase(double* buf, int ph) {
    pdl_launch();
    pdl_wait();
    const double v = buf[((ph + 1) & 1) * 4096 + (blockIdx.x + 1) % gridDim.x];
    if (threadIdx.x == 0) buf[(ph & 1) * 4096 + blockIdx.x] = v + 1.0;
}

int main() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    unsigned* ctr;
    double* buf;
    CK(cudaMalloc(&ctr, 4));
    CK(cudaMalloc(&buf, 16384 * 8));
    CK(cudaMemset(buf, 0, 16384 * 8));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int phases = 4000;
    for (int per : {1, 2, 4}) {
        for (int thr : {256, 512, 1024}) {
            if (per * thr > 2048) continue;
            const int grid = nsm * per;
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaMemsetAsync(ctr, 0, 4, s));
                void* args[] = {&ctr, &buf, (void*)&phases};
                CK(cudaEventRecord(a, s));
                CK(cudaLaunchCooperativeKernel((void*)k_persistent, grid, thr, args, 0, s));
                CK(cudaEventRecord(b, s));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                if (rep) printf("persistent grid=%d x %d threads: %.3f us per grid barrier phase\n", grid, thr,
                                ms * 1e3 / phases);
            }
        }
    }
    {
        unsigned* cg;
        CK(cudaMalloc(&cg, 8));
        CK(cudaMemset(cg, 0, 8));
        for (int per : {1, 2}) {
            const int grid = nsm * per;
            for (int rep = 0; rep < 2; ++rep) {
                unsigned* c0 = cg;
                unsigned* g0 = cg + 1;
                void* args[] = {&c0, &g0, &buf, (void*)&phases};
                CK(cudaEventRecord(a, s));
                CK(cudaLaunchCooperativeKernel((void*)k_persistent_gen, grid, 512, args, 0, s));
                CK(cudaEventRecord(b, s));
                CK(cudaEventSynchronize(b));
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                if (rep) printf("generation barrier grid=%d x 512: %.3f us per phase\n", grid, ms * 1e3 / phases);
            }
        }
    }
    CK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs : {8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(1024);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaEventRecord(a, s));
            CK(cudaLaunchKernelEx(&cfg, k_cluster, buf, phases));
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep) printf("cluster barrier cs=%d x 1024: %.3f us per phase\n", cs, ms * 1e3 / phases);
        }
    }
    // PDL chain inside a graph
    for (int grid : {nsm, 2 * nsm, 8 * nsm}) {
        const int n = 1000;
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < n; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, k_phase, buf, i));
        }
        CK(cudaStreamEndCapture(s, &g));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a, s));
            CK(cudaGraphLaunch(ge, s));
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep == 2) printf("graph PDL chain grid=%d: %.3f us per dependent launch\n", grid, ms * 1e3 / n);
        }
        // without PDL
        cudaGraph_t g2;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < n; ++i) k_phase<<<grid, 256, 0, s>>>(buf, i);
        CK(cudaStreamEndCapture(s, &g2));
        cudaGraphExec_t ge2;
        CK(cudaGraphInstantiate(&ge2, g2, 0));
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(a, s));
            CK(cudaGraphLaunch(ge2, s));
            CK(cudaEventRecord(b, s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep == 2) printf("graph plain chain grid=%d: %.3f us per dependent launch\n", grid, ms * 1e3 / n);
        }
    }
    printf("done\n");
    return 0;
}
