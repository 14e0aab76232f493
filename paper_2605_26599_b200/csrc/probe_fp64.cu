// probe_fp64.cu -- FP64 pipe peak microbenchmark (MEASURED_PEAKS.json has no
// FP64 entry).  Independent DFMA chains per thread, persistent grid; reports
// DFMA lane-ops per second (1 per DFMA per thread) measured with CUDA events.
// Tooling only (libbrprobe.so); not part of the solver.
#include <cuda_runtime.h>

#include <cstdint>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x0 = __fma_rn(x0, a, b); x1 = __fma_rn(x1, a, b); x2 = __fma_rn(x2, a, b);
            x3 = __fma_rn(x3, a, b); x4 = __fma_rn(x4, a, b); x5 = __fma_rn(x5, a, b);
            x6 = __fma_rn(x6, a, b); x7 = __fma_rn(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1.2345) out[0] = s;  // keep live
}

extern "C" __attribute__((visibility("default"))) double brprobe_fp64_peak(int device, double* ms_out) {
    cudaSetDevice(device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out;
    cudaMalloc(&out, 8);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 256, 0.999999, 1e-7);  // warm up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms_out) *ms_out = best;
    const double lane_ops = (double)blocks * threads * iters * 64.0;
    return lane_ops / (best * 1e-3);  // DFMA lane-ops per second
}
