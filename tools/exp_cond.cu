// Feasibility probe: IF/ELSE conditional graph nodes created during stream
// capture, with PDL launches inside the bodies; cost per level vs a plain chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/exp_cond tools/exp_cond.cu -lcuda
#include <cuda_runtime.h>
#include <cstdio>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void k_set(cudaGraphConditionalHandle h, const int* flag, int* out) {
    pdl_wait();
    if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, *flag ? 1u : 0u);
}
__global__ void k_body(int* out, int v) {
    pdl_wait();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = out[0] * 3 + v;
}
__global__ void k_after(int* out) {
    pdl_wait();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] += 1;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid; cfg.blockDim = block; cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

int build(cudaStream_t s, int levels, int nbody, bool cond, int* flag, int* out, cudaGraphExec_t* ex) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int l = 0; l < levels; ++l) {
        if (!cond) {
            for (int b = 0; b < nbody; ++b) launch_pdl(k_body, 148, 128, s, out, 1);
            launch_pdl(k_after, 148, 128, s, out);
            continue;
        }
        cudaStreamCaptureStatus st;
        cudaGraph_t cg;
        const cudaGraphNode_t* deps;
        size_t nd;
        CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
        launch_pdl(k_set, 1, 32, s, h, flag, out);
        CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 2;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, cg, deps, nd, &cp));
        CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
        cudaStream_t s2;
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        for (int br = 0; br < 2; ++br) {
            CK(cudaStreamBeginCaptureToGraph(s2, cp.conditional.phGraph_out[br], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
            for (int b = 0; b < (br ? nbody : 2); ++b) launch_pdl(k_body, 148, 128, s2, out, br ? 1 : 2);
            cudaGraph_t bg;
            CK(cudaStreamEndCapture(s2, &bg));
        }
        cudaStreamDestroy(s2);
        launch_pdl(k_after, 148, 128, s, out);
    }
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(ex, g, 0));
    return 0;
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int *flag, *out;
    CK(cudaMalloc(&flag, 4));
    CK(cudaMalloc(&out, 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int L = 13, NB = 12;
    for (int mode = 0; mode < 3; ++mode) {
        cudaGraphExec_t ex;
        const bool cond = mode > 0;
        if (build(s, L, NB, cond, flag, out, &ex)) return 1;
        const int fv = mode == 2 ? 1 : 0;  // 1: take the NB-kernel branch
        CK(cudaMemcpy(flag, &fv, 4, cudaMemcpyHostToDevice));
        int z[2] = {0, 0};
        CK(cudaMemcpy(out, z, 8, cudaMemcpyHostToDevice));
        CK(cudaGraphLaunch(ex, s));
        CK(cudaStreamSynchronize(s));
        int r[2];
        CK(cudaMemcpy(r, out, 8, cudaMemcpyDeviceToHost));
        for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ex, s));
        CK(cudaEventRecord(a, s));
        const int R = 50;
        for (int i = 0; i < R; ++i) CK(cudaGraphLaunch(ex, s));
        CK(cudaEventRecord(b, s));
        CK(cudaStreamSynchronize(s));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("mode %d (%s) out0=%d after=%d  graph %.2f us  per level %.2f us\n", mode,
               mode == 0 ? "plain chain NB+1 kernels" : mode == 1 ? "cond -> 2-kernel branch" : "cond -> NB-kernel branch",
               r[0], r[1], 1000 * ms / R, 1000 * ms / R / L);
    }
    return 0;
}
