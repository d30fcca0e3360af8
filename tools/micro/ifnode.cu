// Microbenchmark: cost of a graph IF node (condition 0, body = 8 kernels) between two kernels,
// vs the same chain without it, vs an early-exit kernel in its place; chains of 200 substeps.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void work(float* x, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = x[i] * 0.999f + 1e-3f;
}
__global__ void plan(cudaGraphConditionalHandle h, int set) {
    if (set && threadIdx.x == 0) cudaGraphSetConditional(h, 0u);
}
__global__ void noop(const int* flag) {
    if (*flag == 0) return;
}
__global__ void __launch_bounds__(128, 2) coop_noop(const int* flag) {
    if (*flag == 0) return;
    __syncthreads();
}
int main() {
    const int n = 1 << 20, S = 200;
    float* x; int* flag;
    cudaMalloc(&x, n * 4); cudaMalloc(&flag, 4); cudaMemset(x, 0, n * 4); cudaMemset(flag, 0, 4);
    cudaStream_t s, s2; cudaStreamCreate(&s); cudaStreamCreate(&s2);
    for (int mode = 0; mode < 5; ++mode) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        for (int k = 0; k < S; ++k) {
            work<<<n / 256, 256, 0, s>>>(x, n);       // "density"
            work<<<n / 256, 256, 0, s>>>(x, n);       // "force"
            if (mode == 1) {                          // plan + IF node (condition 0)
                cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
                cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
                cudaGraphConditionalHandle h;
                cudaGraphConditionalHandleCreate(&h, cg, 0, 0);
                plan<<<1, 32, 0, s>>>(h, 1);
                cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
                cudaGraphNodeParams cp = {};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = h;
                cp.conditional.type = cudaGraphCondTypeIf;
                cp.conditional.size = 1;
                cudaGraphNode_t node;
                cudaGraphAddNode(&node, cg, deps, nd, &cp);
                cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies);
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
                for (int j = 0; j < 8; ++j) work<<<n / 256, 256, 0, s2>>>(x, n);
                cudaStreamEndCapture(s2, &body);
            } else if (mode == 2) {                   // plan only
                plan<<<1, 32, 0, s>>>(0, 0);
            } else if (mode == 3) {                   // 8 early-exit kernels
                for (int j = 0; j < 8; ++j) noop<<<4096, 256, 0, s>>>(flag);
            } else if (mode == 4) {                   // one early-exit cooperative launch
                void* args[] = {&flag};
                cudaLaunchCooperativeKernel((void*)coop_noop, dim3(296), dim3(128), args, 0, s);
            }
        }
        cudaStreamEndCapture(s, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed mode %d\n", mode); continue; }
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const char* names[] = {"2 kernels", "2 kernels + plan + IF(0)", "2 kernels + plan", "2 kernels + 8 early-exit", "2 kernels + coop early-exit"};
        printf("%-28s %.3f us per substep  (%s)\n", names[mode], ms * 1e3 / (10 * S), cudaGetErrorString(cudaGetLastError()));
    }
}
