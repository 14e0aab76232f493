// tiled.cu -- large-K tier of the secular solver (Toeplitz / glued-Wilkinson
// top levels, K up to n/2).
//
// Same chunking of roots as k_secular (kernels.cu); this kernel owns exactly
// the chunks whose pole window does not fit in shared memory.  Every lane
// still runs its own resumable RootSM (numerics.cuh) and refills from the CTA
// queue, but evaluations are CTA-SYNCHRONOUS passes: the CTA streams the pole
// window through shared memory in tiles of (d, z^2) pairs (double-buffered,
// one coalesced load per tile per CTA instead of one L2 stream per warp) and
// every lane with a pending evaluation accumulates the tile's intersection
// with its merge, in pole order -- the checker's summation order, so results
// are bit-identical to k_secular / oracle/br_oracle.c.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"
#include "level_state.cuh"

namespace brgpu {

constexpr int kTiledThreads = 256;
constexpr int kTile2 = 1024;           // (d, z^2) pairs per tile (16 KB, double-buffered)
constexpr int kSecChunkBlock = 128;    // must match kSecBlock in kernels.cu (chunk formula)
constexpr int kSecWinFit = 2048;       // must match kSecWinQ in kernels.cu

__device__ __forceinline__ void tile_load(double2* dst, const double* __restrict__ d,
                                          const double* __restrict__ z2, int lo, int hi) {
    for (int i = lo + threadIdx.x; i < hi; i += kTiledThreads) dst[i - lo] = make_double2(d[i], z2[i]);
}

__global__ void __launch_bounds__(kTiledThreads, 2)
k_secular_tiled(Work w, LevelDev L, int n, int patched, int G) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ double2 s_tile[2][kTile2];
    __shared__ double2 s_snap[kTiledThreads];
    __shared__ int s_next;
    if (!(*w.levelModes & 1)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int R = max(kSecChunkBlock, (T + G - 1) / G);
    // this kernel's grid covers the same G chunks; CTA b owns chunk b
    const int c0 = blockIdx.x * R;
    if (c0 >= T) return;
    const int c1 = min(c0 + R, T);
    if (!chunk_has_mode(w, L, c0, c1, false)) return;
    int a0, a1, b0, b1;
    {
        const int m0 = w.aMerge[c0], m1 = w.aMerge[c1 - 1];
        const int o0 = L.mOff[m0], o1 = L.mOff[m1];
        a0 = w.survPre[w.nnPre[o0]];
        a1 = w.survPre[w.nnPre[o0 + L.mSize[m0]]];
        b0 = w.survPre[w.nnPre[o1]];
        b1 = w.survPre[w.nnPre[o1 + L.mSize[m1]]];
    }
    (void)a1; (void)b0;
    const int P0 = a0, P1 = b1;
    if (P1 - P0 <= kSecWinFit) return;  // k_secular owns it
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();

    RootSM st;
    int g = -1, ks = 0;
    bool exhausted = false;
    unsigned long long evals = 0, terms = 0;
    for (;;) {
        while (g < 0 && !exhausted) {
            const int q = atomicAdd(&s_next, 1);
            if (c0 + q >= c1) { exhausted = true; break; }
            if (!owns(w, c0 + q)) continue;  // another rank's root (root-range split)
            const int m = w.aMerge[c0 + q];
            int ke;
            const int off = L.mOff[m];
            ks = w.survPre[w.nnPre[off]];
            ke = w.survPre[w.nnPre[off + L.mSize[m]]];
            if (split_mode(L.mSize[m], ke - ks)) continue;  // warp-per-root tier (warp.cu)
            g = c0 + q;
            const double rho = fabs(w.ew[off + L.mNL[m] - 1]);
            rs_begin(st, ke - ks, g - ks, rho, PolesPtr{w.dA + ks}, w.zA[ks], Z2Ptr{w.z2A + ks});
            if (st.phase == kRsDone) {
                w.org[g] = ks + st.org;
                w.tau[g] = st.tau;
                g = -1;
            }
        }
        const bool need = g >= 0;
        if (!__syncthreads_or(need)) break;
        // one CTA-synchronous evaluation pass over the window
        double sum = 0.0, sum_abs = 0.0, sum_d = 0.0, psi = 0.0;
        const int K = need ? st.K : 0;
        const int j = st.j;
        const double dorg = st.dorg, tau = st.tau;
        const bool fast = need && !w.exact && eval_guard(GlobalPairs{w.dA + ks, w.z2A + ks}, K, j, dorg, tau);
        const unsigned sa = (unsigned)__cvta_generic_to_shared(s_snap + threadIdx.x);
        snap_if(sa, 0, j < 0 ? 0 : 1, 0.0, 0.0);
        int buf = 0;
        tile_load(s_tile[0], w.dA, w.z2A, P0, min(P0 + kTile2, P1));
        for (int tlo = P0; tlo < P1; tlo += kTile2) {
            const int thi = min(tlo + kTile2, P1);
            __syncthreads();  // tile `buf` complete; previous readers of buf^1 done
            if (thi < P1) tile_load(s_tile[buf ^ 1], w.dA, w.z2A, thi, min(thi + kTile2, P1));
            if (fast) {
                const int ilo = max(ks, tlo), ihi = min(ks + K, thi);
                const double2* __restrict__ tp = s_tile[buf] - tlo;
                const int jg = ks + j;
                auto term = [&](double2 dz, int i) {
                    const double r = rcp_nr((dz.x - dorg) - tau);
                    const double t = dz.y * r;
                    sum += t;
                    sum_d = __fma_rn(t, r, sum_d);
                    snap_if(sa, i, jg, sum, sum_d);
                };
                int i = ilo;
                for (; i + 4 <= ihi; i += 4) {
                    const double2 a0 = tp[i], a1 = tp[i + 1], a2 = tp[i + 2], a3 = tp[i + 3];
                    term(a0, i);
                    term(a1, i + 1);
                    term(a2, i + 2);
                    term(a3, i + 3);
                }
                for (; i < ihi; ++i) term(tp[i], i);
            }
            buf ^= 1;
        }
        __syncthreads();
        bool pole = false;
        if (need) {
            if (fast) {
                snap_if(sa, 0, j >= K ? 0 : 1, sum, sum_d);
                const double2 sn = ld_snap(sa);
                psi = sn.y;
                sum_abs = sum - 2.0 * sn.x;  // term signs are fixed by the bracket
            } else {  // rare: exact pass from global memory
                pole = eval_pass_exact(GlobalPairs{w.dA + ks, w.z2A + ks}, K, j, dorg, tau, sum, sum_abs,
                                       sum_d, psi);
            }
            Ev ev;
            ev.f = 1.0 + st.rho * sum;
            ev.fp = st.rho * sum_d;
            ev.abs_sum = st.rho * sum_abs;
            ev.psi = st.rho * psi;
            ev.pole = pole;
            ++evals;
            terms += (unsigned long long)K;
            rs_consume(st, ev, PolesPtr{w.dA + ks}, Z2Ptr{w.z2A + ks}, patched != 0);
            if (st.phase == kRsDone || st.phase == kRsFail) {
                if (st.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                w.org[g] = ks + st.org;
                w.tau[g] = st.tau;
                g = -1;
            }
        }
    }
    unsigned long long e = evals, t = terms;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if ((threadIdx.x & 31) == 0 && e) {
        atomicAdd(&w.counters[0], e);
        atomicAdd(&w.counters[1], t);
    }
}

void launch_secular_tiled(cudaStream_t s, const Work& w, const LevelDev& L, int n,
                          const SolveParams& prm) {
    launch_pdl(k_secular_tiled, prm.sec_grid, kTiledThreads, 0, s, w, L, n, prm.patched, prm.sec_grid);
}

}  // namespace brgpu
