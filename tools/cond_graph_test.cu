// Micro-test (tools only): conditional WHILE graph node with a device-side cudaGraphSetConditional.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cgt tools/cond_graph_test.cu && /tmp/cgt
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_check(cudaGraphConditionalHandle h, int* ctr, int maxc) {
    int c = ++(*ctr);
    cudaGraphSetConditional(h, c < maxc ? 1u : 0u);
}
__global__ void k_body(double* x) { x[threadIdx.x] += 1.0; }
int main() {
    cudaStream_t s; cudaStreamCreate(&s);
    int* ctr; double* x; cudaMalloc(&ctr, 4); cudaMalloc(&x, 8*32); cudaMemset(ctr, 0, 4); cudaMemset(x, 0, 256);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
    printf("add %s\n", cudaGetErrorString(e));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("cap %s\n", cudaGetErrorString(e));
    k_body<<<1, 32, 0, s>>>(x);
    k_check<<<1, 1, 0, s>>>(h, ctr, 7);
    e = cudaStreamEndCapture(s, &body);
    printf("end %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge; e = cudaGraphInstantiate(&ge, g, 0); printf("inst %s\n", cudaGetErrorString(e));
    e = cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); printf("launch %s\n", cudaGetErrorString(e));
    double hx; cudaMemcpy(&hx, x, 8, cudaMemcpyDeviceToHost); int hc; cudaMemcpy(&hc, ctr, 4, cudaMemcpyDeviceToHost);
    printf("x %g ctr %d\n", hx, hc);
    return 0;
}
