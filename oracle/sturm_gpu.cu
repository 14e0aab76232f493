// sturm_gpu.cu -- TEST-ONLY independent certificate (never linked into the
// product): Sturm counts (LDL^T inertia) of T - x I for many shifts x at once
// on the GPU, with exactly the arithmetic of the CPU checker's
// bro_sturm_count (oracle/br_oracle.c): q_0 = d_0 - x,
// q_i = (d_i - x) - e_{i-1} e_{i-1} / q_{i-1}, |q| < 4 DBL_MIN -> -4 DBL_MIN,
// count of negative q.  Compiled with --fmad=false and IEEE division, so every
// count equals the CPU count bit for bit; tests/ use it to certify EVERY
// eigenvalue index of the 2^18 / 2^20 configurations:
//     count(w_i - tol) <= i < count(w_i + tol)   for all i
// i.e. |w_i - lambda_i| <= tol for the exact i-th eigenvalue lambda_i.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

namespace {

constexpr int kThreads = 256;
constexpr int kTile = 2048;

// one shift per thread; d and e^2 staged through shared memory in tiles that
// every thread of the CTA walks in lockstep
__global__ void __launch_bounds__(kThreads) k_sturm(int64_t n, const double* __restrict__ d,
                                                    const double* __restrict__ e, const double* __restrict__ x,
                                                    int64_t nx, int64_t* __restrict__ out) {
    __shared__ double sd[kTile], se[kTile];
    const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const double xv = j < nx ? x[j] : 0.0;
    const double pivmin = DBL_MIN * 4.0;
    int64_t cnt = 0;
    double q = 1.0;
    for (int64_t t0 = 0; t0 < n; t0 += kTile) {
        const int len = (int)(n - t0 < kTile ? n - t0 : kTile);
        __syncthreads();
        for (int k = threadIdx.x; k < len; k += kThreads) {
            sd[k] = d[t0 + k];
            se[k] = (t0 + k >= 1) ? e[t0 + k - 1] : 0.0;
        }
        __syncthreads();
        for (int k = 0; k < len; ++k) {
            if (t0 + k == 0) {
                q = sd[0] - xv;
            } else {
                const double ek = se[k];
                q = (sd[k] - xv) - ek * ek / q;
            }
            if (fabs(q) < pivmin) q = -pivmin;
            cnt += q < 0.0;
        }
    }
    if (j < nx) out[j] = cnt;
}

}  // namespace

extern "C" {

// counts[j] = #{eigenvalues of T below x[j]} for j < nx (host arrays in and out).
// Returns 0 on success, the CUDA error code otherwise.
int brsturm_counts(int64_t n, const double* d, const double* e, const double* x, int64_t nx, int64_t* counts) {
    if (n <= 0 || nx <= 0) return 0;
    double *dd = nullptr, *de = nullptr, *dx = nullptr;
    int64_t* dc = nullptr;
    cudaError_t st = cudaMalloc(&dd, sizeof(double) * n);
    if (st == cudaSuccess) st = cudaMalloc(&de, sizeof(double) * (n > 1 ? n - 1 : 1));
    if (st == cudaSuccess) st = cudaMalloc(&dx, sizeof(double) * nx);
    if (st == cudaSuccess) st = cudaMalloc(&dc, sizeof(int64_t) * nx);
    if (st == cudaSuccess) st = cudaMemcpy(dd, d, sizeof(double) * n, cudaMemcpyHostToDevice);
    if (st == cudaSuccess && n > 1) st = cudaMemcpy(de, e, sizeof(double) * (n - 1), cudaMemcpyHostToDevice);
    if (st == cudaSuccess) st = cudaMemcpy(dx, x, sizeof(double) * nx, cudaMemcpyHostToDevice);
    if (st == cudaSuccess) {
        const int64_t grid = (nx + kThreads - 1) / kThreads;
        k_sturm<<<(unsigned)grid, kThreads>>>(n, dd, de, dx, nx, dc);
        st = cudaGetLastError();
    }
    if (st == cudaSuccess) st = cudaMemcpy(counts, dc, sizeof(int64_t) * nx, cudaMemcpyDeviceToHost);
    cudaFree(dd);
    cudaFree(de);
    cudaFree(dx);
    cudaFree(dc);
    return (int)st;
}

}  // extern "C"
