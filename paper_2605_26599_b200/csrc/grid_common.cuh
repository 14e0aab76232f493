// grid_common.cuh -- helpers shared by the grid-tier level kernels
// (kernels.cu: dense pipeline; sparse.cu: sparse pipeline).
#pragma once

#include "internal.hpp"
#include "numerics.cuh"

namespace brgpu {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_merge(const LevelDev& L, int p) {
    const int t = p / kTile;
    int m = L.tileFirst[t];
    const int last = L.tileFirst[t + 1] < L.M ? L.tileFirst[t + 1] : L.M - 1;
    while (m < last && L.mOff[m + 1] <= p) ++m;
    if (m >= L.M || m < 0) return -1;
    const int off = L.mOff[m];
    if (p < off || p >= off + L.mSize[m]) return -1;
    return m;
}

__device__ __forceinline__ double merge_tol(const LevelDev& L, int m, double tol_scale) {
    const double mx = __longlong_as_double((long long)L.mTol[m]);
    return 8.0 * kU * mx * tol_scale;
}

// Active range [ks, ke) of merge m in the level-global compacted arrays.
__device__ __forceinline__ void active_range(const Work& w, const LevelDev& L, int m, int& ks, int& ke) {
    const int off = L.mOff[m];
    ks = w.survPre[w.nnPre[off]];
    ke = w.survPre[w.nnPre[off + L.mSize[m]]];
}

template <int BLOCK>
__device__ __forceinline__ int block_exclusive_scan(int v, int& total) {
    __shared__ int warp_tot[BLOCK / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int t = lane < BLOCK / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < BLOCK / 32) warp_tot[lane] = t;
    }
    __syncthreads();
    const int base = wid ? warp_tot[wid - 1] : 0;
    total = warp_tot[BLOCK / 32 - 1];
    __syncthreads();
    return base + x - v;
}

template <int BLOCK>
__device__ __forceinline__ int block_sum(int v) {
    __shared__ int red[BLOCK / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    int t = 0;
    if (threadIdx.x < 32) {
        t = lane < BLOCK / 32 ? red[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    return t;  // valid in thread 0
}

// Number of left-child elements among the first d outputs of the stable merge
// of sorted a[0..nl) (left) and b[0..nr) (right): left element i precedes
// right element j iff a_i <= b_j (std::stable_sort of the concatenation by
// '<', deflate.cpp:62-66).  Warp-cooperative 32-ary search (all lanes call it
// with the same arguments): about log32 of the child size dependent L2 round
// trips instead of log2.
__device__ __forceinline__ int warp_merge_split(const double* __restrict__ a, int nl,
                                                const double* __restrict__ b, int nr, int d) {
    const int lane = threadIdx.x & 31;
    int lo = max(0, d - nr), hi = min(d, nl);  // answer in [lo, hi]; pred(i) holds for i <= answer
    while (hi > lo) {
        const int span = hi - lo;
        const int step = (span + 31) >> 5;
        const int c = min(lo + (lane + 1) * step, hi);
        const bool pred = (d - c >= nr) || !(b[d - c] < a[c - 1]);  // a[c-1] is within the first d
        const unsigned bal = __ballot_sync(0xffffffffu, pred);
        const int k = __popc(bal);  // candidates are monotone: the first k hold
        if (step == 1) { lo = min(lo + k, hi); break; }  // capped duplicates of hi may add to k
        const int nlo = k ? min(lo + k * step, hi) : lo;
        hi = min(hi, lo + (k + 1) * step - 1);
        lo = nlo;
    }
    return lo;
}

// CTA-wide scans of the shared-memory level kernels (fused.cu, sparse.cu)
template <int kFuseThreads>
__device__ __forceinline__ int cta_excl_scan(int v, int& total, int* warp_tot) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = kFuseThreads / 32;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int t = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NW) warp_tot[lane] = t;
    }
    __syncthreads();
    const int base = wid ? warp_tot[wid - 1] : 0;
    total = warp_tot[NW - 1];
    __syncthreads();
    return base + x - v;
}

// exclusive prefix of flags[0..E) into pre[0..E]; each thread scans a contiguous chunk
template <int kFuseThreads>
__device__ __forceinline__ int cta_scan_flags(const unsigned char* flags, int E, int* pre, int* warp_tot) {
    const int per = (E + kFuseThreads - 1) / kFuseThreads;
    const int i0 = threadIdx.x * per;
    int local = 0;
    for (int k = 0; k < per; ++k) {
        const int i = i0 + k;
        if (i < E) local += flags[i];
    }
    int tot;
    int run = cta_excl_scan<kFuseThreads>(local, tot, warp_tot);
    for (int k = 0; k < per; ++k) {
        const int i = i0 + k;
        if (i < E) {
            pre[i] = run;
            run += flags[i];
        }
    }
    if (threadIdx.x == 0) pre[E] = tot;
    __syncthreads();
    return tot;
}

// largest t in [0, cnt) with a[t] <= x
__device__ __forceinline__ int upper_index(const int* a, int cnt, int x) {
    int lo = 0, hi = cnt;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid; else hi = mid;
    }
    return lo;
}

}  // namespace brgpu
