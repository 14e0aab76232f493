// Microbenchmark: cycles of one lane-arithmetic evaluation (eval_fast, K poles
// in shared memory) against one rs_consume (bracket, safeguards, model step),
// for a lone warp (the latency-bound top levels of the live tier).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17
//      -I include -I paper_2605_26599_b200/csrc tools/exp_consume.cu -o /tmp/exp_consume
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#include "internal.hpp"
#include "numerics.cuh"
using namespace brgpu;

// variant: the prefix snapshot as register selects (no shared-memory store per term)
template <typename P, int U>
__device__ __forceinline__ void eval_sel(const P& pairs, int K, int jsplit, double dorg, double tau,
                                         double& sum, double& sum_abs, double& sum_d, double& psi) {
    double s = 0.0, sd = 0.0, ps = 0.0, pd = 0.0;
    int i = 0;
    for (; i + U <= K; i += U) {
        double2 a[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = pairs(i + u);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double del = (a[u].x - dorg) - tau;
            const double r = rcp_nr(del);
            const double t = a[u].y * r;
            s += t;
            sd = __fma_rn(t, r, sd);
            const bool hit = i + u == jsplit;
            ps = hit ? s : ps;
            pd = hit ? sd : pd;
        }
    }
    for (; i < K; ++i) {
        const double2 a = pairs(i);
        const double del = (a.x - dorg) - tau;
        const double r = rcp_nr(del);
        const double t = a.y * r;
        s += t;
        sd = __fma_rn(t, r, sd);
        const bool hit = i == jsplit;
        ps = hit ? s : ps;
        pd = hit ? sd : pd;
    }
    if (jsplit >= K) { ps = s; pd = sd; }
    sum = s; sum_d = sd; psi = pd; sum_abs = s - 2.0 * ps;
}

template <int MODE>
__global__ void k_probe(const double2* __restrict__ g, int K, double rho, unsigned long long* out) {
    __shared__ double2 P[1024];
    __shared__ double2 snapb[32];
    for (int i = threadIdx.x; i < K; i += blockDim.x) P[i] = g[i];
    __syncthreads();
    const int j = threadIdx.x * (K / 32);
    RootSM st;
    rs_begin(st, K, j, rho, PolesPairs{P}, 0.0, Z2Pairs{P});
    long long tev = 0, tcon = 0;
    int nev = 0;
    while (st.phase != kRsDone && st.phase != kRsFail) {
        double sum, sum_abs, sum_d, psi;
        long long t0 = clock64();
        if (MODE == 0) eval_fast(SmemPairs{P}, st.K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi, snapb + threadIdx.x);
        else if (MODE == 1) eval_sel<SmemPairs, 4>(SmemPairs{P}, st.K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi);
        else eval_sel<SmemPairs, 8>(SmemPairs{P}, st.K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi);
        Ev ev;
        ev.f = 1.0 + st.rho * sum;
        ev.fp = st.rho * sum_d;
        ev.abs_sum = st.rho * sum_abs;
        ev.psi = st.rho * psi;
        ev.pole = false;
        long long t1 = clock64();
        rs_consume(st, ev, PolesPairs{P}, Z2Pairs{P}, true);
        long long t2 = clock64();
        tev += t1 - t0;
        tcon += t2 - t1;
        ++nev;
    }
    out[3 * threadIdx.x] = tev;
    out[3 * threadIdx.x + 1] = tcon;
    out[3 * threadIdx.x + 2] = nev;
}

int main() {
    for (int K : {32, 100, 400}) {
        std::vector<double2> h(K);
        std::vector<double> d(K);
        srand(7);
        for (int i = 0; i < K; ++i) d[i] = 6.0 * rand() / RAND_MAX - 3.0;
        std::sort(d.begin(), d.end());
        for (int i = 0; i < K; ++i) {
            const double z = (2.0 * rand() / RAND_MAX - 1.0) / std::sqrt((double)K);
            h[i] = make_double2(d[i], z * z);
        }
        double2* g; unsigned long long* o;
        cudaMalloc(&g, sizeof(double2) * K);
        cudaMalloc(&o, sizeof(unsigned long long) * 96);
        cudaMemcpy(g, h.data(), sizeof(double2) * K, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k_probe<0><<<1, 32>>>(g, K, 0.7, o);
                else if (mode == 1) k_probe<1><<<1, 32>>>(g, K, 0.7, o);
                else k_probe<2><<<1, 32>>>(g, K, 0.7, o);
            }
            unsigned long long ho[96];
            cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
            double se = 0, sc = 0, sn = 0;
            for (int l = 0; l < 32; ++l) { se += ho[3 * l]; sc += ho[3 * l + 1]; sn += ho[3 * l + 2]; }
            printf("K=%d mode %d (%s): per evaluation %.0f cycles pole loop (%.1f per term), %.0f cycles consume; evals/root %.2f\n",
                   K, mode, mode == 0 ? "snap store" : mode == 1 ? "selects x4" : "selects x8", se / sn, se / sn / K, sc / sn, sn / 32);
        }
        cudaFree(g); cudaFree(o);
    }
    return 0;
}
