// warp.cu -- warp-per-root tier for merges larger than the fused SMEM tier
// (size > kSplitMinSize): the upper levels of random inputs (few roots, latency
// bound) and the large-K top levels of Toeplitz / glued Wilkinson.
//
// One warp owns one root (secular, rows) or one pole (refreshed weights).  Lane
// l accumulates the terms l, l+32, ... in increasing order and the 32 partials
// meet in the xor butterfly (bfly_add / bfly_mul) -- the split arithmetic the
// checker states for these merges (oracle/br_oracle.c, BRO_SPLIT_MIN_SIZE), so
// results stay bit-identical.  Every lane runs the same RootSM update on the
// same butterfly result, so the per-root control flow has no divergence.  The
// CTA's pole window streams through shared memory in tiles shared by its 8
// warps (one coalesced L2 read per tile per CTA).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"

namespace brgpu {

constexpr int kWarpThreads = 256;  // 8 warps
constexpr int kWarpTile = 1024;    // (d, z^2) pairs per tile
#ifndef BRGPU_SECW_THREADS
#define BRGPU_SECW_THREADS 256
#endif
#ifndef BRGPU_SECW_MINB
#define BRGPU_SECW_MINB 3  // CTAs per SM: 80 registers, no spills (2: 107 registers, C3 +1%)
#endif
#ifndef BRGPU_SECW_TILE
#define BRGPU_SECW_TILE 2048  // 2 x 32 KB dynamic SMEM per CTA, 3 CTAs per SM
#endif
constexpr int kSecWThreads = BRGPU_SECW_THREADS;  // k_secular_warp: roots in flight per CTA x 32
constexpr int kSecWTile = BRGPU_SECW_TILE;        // k_secular_warp: (d, z^2) pairs per SMEM tile

__device__ __forceinline__ void merge_active(const Work& w, const LevelDev& L, int m, int& ks, int& ke) {
    const int off = L.mOff[m];
    ks = w.survPre[w.nnPre[off]];
    ke = w.survPre[w.nnPre[off + L.mSize[m]]];
}

// first index i >= lo with (i - ks) % 32 == lane
__device__ __forceinline__ int strided_start(int lo, int ks, int lane) {
    const int r = (lane - (lo - ks)) & 31;
    return lo + r;
}

// (d, z^2) pairs of poles [a, b) into a shared-memory tile with cp.async: the
// copies complete in the background (no register round trip, no stall on the
// global load) and cp_async_wait_all + a barrier publish them.
__device__ __forceinline__ void tile_fetch(double2* tile, const Work& w, int a, int b) {
    for (int i = a + (int)threadIdx.x; i < b; i += kSecWThreads) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + (i - a));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(w.dA + i) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u), "l"(w.z2A + i) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------------------
// secular roots, one warp per root
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSecWThreads, BRGPU_SECW_MINB) k_secular_warp(Work w, LevelDev L, int n, int patched) {
    pdl_entry();
    extern __shared__ __align__(16) double2 s_tiles[];  // two tiles of kSecWTile pairs (dynamic)
    __shared__ int s_next;
    if (!L.allSplit && !(*w.levelModes & 2)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int G = (int)gridDim.x;
    const int R = max(kSecWThreads / 32, (T + G - 1) / G);
    const int c0 = blockIdx.x * R;
    if (c0 >= T) return;
    const int c1 = min(c0 + R, T);
    if (!chunk_has_mode(w, L, c0, c1, true)) return;
    int P0, P1, tmp;
    merge_active(w, L, w.aMerge[c0], P0, tmp);
    merge_active(w, L, w.aMerge[c1 - 1], tmp, P1);
    if (threadIdx.x == 0) s_next = 0;
    // a window that fits one tile is loaded once for all evaluation rounds;
    // a larger one streams through the two tiles every round
    const bool resident = P1 - P0 <= kSecWTile;
    if (resident) tile_fetch(s_tiles, w, P0, P1);
    __syncthreads();
    const int lane = threadIdx.x & 31;

    RootSM st;
    int g = -1, ks = 0;
    bool exhausted = false;
    unsigned long long evals = 0, terms = 0;
    for (;;) {
        while (g < 0 && !exhausted) {
            int q = 0;
            if (lane == 0) q = atomicAdd(&s_next, 1);
            q = __shfl_sync(0xffffffffu, q, 0);
            if (c0 + q >= c1) { exhausted = true; break; }
            const int gg = c0 + q;
            if (!owns(w, gg)) continue;  // another rank's root (root-range split)
            const int m = w.aMerge[gg];
            int ke;
            merge_active(w, L, m, ks, ke);
            if (!split_mode(L.mSize[m], ke - ks)) continue;  // lane-per-root tier owns it
            g = gg;
            const int K = ke - ks, j = g - ks;
            const double rho = fabs(w.ew[L.mOff[m] + L.mNL[m] - 1]);
            double zsq = 0.0;
            if (j == K - 1 && K > 1) {
                for (int i = ks + lane; i < ke; i += 32) zsq += w.z2A[i];
                zsq = bfly_add(zsq);
            }
            rs_begin_zsq(st, K, j, rho, PolesPtr{w.dA + ks}, w.zA[ks], zsq, w.z2A[ks + K - 1]);
            if (st.phase == kRsDone) {
                if (lane == 0) { w.org[g] = st.org; w.tau[g] = st.tau; }
                g = -1;
            }
        }
        const bool need = g >= 0;
        if (!__syncthreads_or(need)) break;
        double sum = 0.0, sum_d = 0.0, psi = 0.0, psum = 0.0;
        const int K = need ? st.K : 0;
        const int j = st.j;
        const double dorg = st.dorg, tau = st.tau;
        // neighbour range guard (eval_guard, numerics.cuh); on failure the warp
        // skips the fast pass and runs the exact one below
        const bool fast = need && !w.exact && eval_guard(GlobalPairs{w.dA + ks, w.z2A + ks}, K, j, dorg, tau);
        int buf = 0;
        if (!resident) tile_fetch(s_tiles, w, P0, min(P0 + kSecWTile, P1));
        for (int tlo = P0; tlo < P1; tlo += kSecWTile) {
            const int thi = min(tlo + kSecWTile, P1);
            cp_async_wait_all();
            __syncthreads();
            if (thi < P1) tile_fetch(s_tiles + (buf ^ 1) * kSecWTile, w, thi, min(thi + kSecWTile, P1));
            if (fast) {
                const int lo = max(ks, tlo), hi = min(ks + K, thi);
                const double2* __restrict__ tp = s_tiles + buf * kSecWTile - tlo;
                // terms i <= j, then the prefix snapshot, then i > j: a lane's
                // strided terms are split at one point, so the two loops differ
                // across lanes by at most one trip (no per-term snapshot selects)
                const int mid = min(hi, ks + j + 1);
                int i = strided_start(lo, ks, lane);
#pragma unroll 4
                for (; i < mid; i += 32) {
                    const double2 dz = tp[i];
                    const double r = rcp_nr((dz.x - dorg) - tau);
                    const double t = dz.y * r;
                    sum += t;
                    sum_d = __fma_rn(t, r, sum_d);
                }
                if (lo < mid) { psi = sum_d; psum = sum; }
#pragma unroll 4
                for (; i < hi; i += 32) {
                    const double2 dz = tp[i];
                    const double r = rcp_nr((dz.x - dorg) - tau);
                    const double t = dz.y * r;
                    sum += t;
                    sum_d = __fma_rn(t, r, sum_d);
                }
            }
            buf ^= 1;
        }
        __syncthreads();
        if (need) {
            bool pole = false;
            if (!fast) {  // rare: exact strided pass from global memory
                sum = 0.0; sum_d = 0.0; psi = 0.0; psum = 0.0;
                for (int i = ks + lane; i < ks + K; i += 32) {
                    const double del = (w.dA[i] - dorg) - tau;
                    pole |= (del == 0.0);
                    const double r = __drcp_rn(del);
                    const double t = w.z2A[i] * r;
                    sum += t;
                    sum_d = __fma_rn(t, r, sum_d);
                    if (i - ks <= j) { psi = sum_d; psum = sum; }
                }
                pole = __any_sync(0xffffffffu, pole);
            }
            const double S = bfly_add(sum), SD = bfly_add(sum_d);
            const double PS = bfly_add(psi), PU = bfly_add(psum);
            Ev ev;
            ev.f = 1.0 + st.rho * S;
            ev.fp = st.rho * SD;
            ev.abs_sum = st.rho * (S - 2.0 * PU);
            ev.psi = st.rho * PS;
            ev.pole = pole;
            ++evals;
            terms += (unsigned long long)K;
            rs_consume(st, ev, PolesPtr{w.dA + ks}, Z2Ptr{w.z2A + ks}, patched != 0);
            if (st.phase == kRsDone || st.phase == kRsFail) {
                if (lane == 0) {
                    if (st.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                    w.org[g] = st.org;
                    w.tau[g] = st.tau;
                }
                g = -1;
            }
        }
    }
    if (lane == 0 && evals) {
        atomicAdd(&w.counters[0], evals);
        atomicAdd(&w.counters[1], terms);
    }
}

// ---------------------------------------------------------------------------
// refreshed weights, kZhatPerWarp poles per warp (product over roots, split by lane)
// ---------------------------------------------------------------------------
#ifndef BRGPU_ZHAT_PER_WARP
#define BRGPU_ZHAT_PER_WARP 2
#endif
constexpr int kZhatPerWarp = BRGPU_ZHAT_PER_WARP;

struct WarpZhatPole {
    int g, ks, K, i;
    bool act, fast;
    double di, prod;
};

// Poles of one warp share every root tile read from shared memory (d_org,
// tau, d_j: 24 B per term), which halves the SMEM traffic per FP64 term at 2
// poles per warp.  Each pole keeps its lane-strided product order and the
// butterfly, so results are bitwise those of one pole per warp.
#ifndef BRGPU_ZHAT_MINB
#define BRGPU_ZHAT_MINB 5  // CTAs per SM (48 registers): C3 zhat 2.97 -> 2.91 ms
#endif
__global__ void __launch_bounds__(kWarpThreads, BRGPU_ZHAT_MINB) k_zhat_warp(Work w, LevelDev L, int n) {
    pdl_entry();
    __shared__ double s_dorg[kWarpTile], s_tau[kWarpTile], s_dj[kWarpTile];
    if (!L.allSplit && !(*w.levelModes & 2)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int PPC = (kWarpThreads / 32) * kZhatPerWarp;  // poles per CTA step
    for (int base = blockIdx.x * PPC; base < T; base += gridDim.x * PPC) {  // uniform per CTA
        WarpZhatPole pl[kZhatPerWarp];
        bool any = false;
#pragma unroll
        for (int q = 0; q < kZhatPerWarp; ++q) {
            WarpZhatPole& P = pl[q];
            P.g = base + wid * kZhatPerWarp + q;
            P.ks = 0; P.K = 0; P.i = 0; P.act = false; P.fast = false; P.di = 0.0; P.prod = 1.0;
            if (P.g < T) {
                const int m = w.aMerge[P.g];
                int ke;
                merge_active(w, L, m, P.ks, ke);
                // a lone pole keeps its z (the checker refreshes only K > 1)
                P.act = split_mode(L.mSize[m], ke - P.ks) && !(L.mFlags[m] & kMergeRoot) && owns(w, P.g) &&
                        ke - P.ks > 1;
                P.K = ke - P.ks;
                P.i = P.g - P.ks;
                P.di = w.dA[P.g];
                P.fast = P.act && !w.exact && zhat_guard(PolesPtr{w.dA + P.ks}, P.K, P.i);
            }
            any = any || P.act;
        }
        if (!__syncthreads_or(any)) continue;
        const int gl = min(base + PPC, T) - 1;
        int P0, P1, tmp;
        merge_active(w, L, w.aMerge[base], P0, tmp);
        merge_active(w, L, w.aMerge[gl], tmp, P1);
        bool shared = true;  // every pole of the warp is fast and in the same merge
#pragma unroll
        for (int q = 0; q < kZhatPerWarp; ++q) shared = shared && pl[q].fast && pl[q].ks == pl[0].ks;
        for (int tlo = P0; tlo < P1; tlo += kWarpTile) {
            const int thi = min(tlo + kWarpTile, P1);
            __syncthreads();
            for (int r = tlo + (int)threadIdx.x; r < thi; r += kWarpThreads) {
                int rks, rke;
                merge_active(w, L, w.aMerge[r], rks, rke);
                s_dorg[r - tlo] = w.dA[rks + w.org[r]];
                s_tau[r - tlo] = w.tau[r];
                s_dj[r - tlo] = w.dA[r];
            }
            __syncthreads();
            if (shared) {
                // the poles' own indices (ascending: consecutive g of one merge)
                // split each lane's strided range; between them every factor is
                // del / (d_i - d_j), so the inner loop has no per-term select
                const int ks = pl[0].ks;
                const int lo = max(ks, tlo), hi = min(ks + pl[0].K, thi);
                int jg = strided_start(lo, ks, lane);
#pragma unroll
                for (int sp = 0; sp <= kZhatPerWarp; ++sp) {
                    const int stop = sp < kZhatPerWarp ? min(hi, ks + pl[sp].i) : hi;
#pragma unroll 2
                    for (; jg < stop; jg += 32) {
                        const int t = jg - tlo;
                        const double dorg = s_dorg[t], tau = s_tau[t], dj = s_dj[t];
#pragma unroll
                        for (int q = 0; q < kZhatPerWarp; ++q)
                            pl[q].prod = pl[q].prod * (((pl[q].di - dorg) - tau) * rcp_nr(pl[q].di - dj));
                    }
                    if (sp < kZhatPerWarp && jg == ks + pl[sp].i && jg < hi) {
                        const int t = jg - tlo;
                        const double dorg = s_dorg[t], tau = s_tau[t], dj = s_dj[t];
#pragma unroll
                        for (int q = 0; q < kZhatPerWarp; ++q) {
                            const double del = (pl[q].di - dorg) - tau;
                            pl[q].prod = pl[q].prod * (q == sp ? del : del * rcp_nr(pl[q].di - dj));
                        }
                        jg += 32;
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < kZhatPerWarp; ++q) {
                    WarpZhatPole& P = pl[q];
                    if (!P.fast) continue;
                    // roots before the pole, the pole's own factor, roots after:
                    // one split point per lane, so no per-term self select
                    const int ks = P.ks;
                    const double di = P.di;
                    const int lo = max(ks, tlo), hi = min(ks + P.K, thi);
                    const int mid = min(hi, ks + P.i);
                    int jg = strided_start(lo, ks, lane);
                    double prod = P.prod;
                    for (; jg < mid; jg += 32) {
                        const int t = jg - tlo;
                        prod = prod * (((di - s_dorg[t]) - s_tau[t]) * rcp_nr(di - s_dj[t]));
                    }
                    if (jg == ks + P.i && jg < hi) {
                        const int t = jg - tlo;
                        prod = prod * ((di - s_dorg[t]) - s_tau[t]);
                        jg += 32;
                    }
                    for (; jg < hi; jg += 32) {
                        const int t = jg - tlo;
                        prod = prod * (((di - s_dorg[t]) - s_tau[t]) * rcp_nr(di - s_dj[t]));
                    }
                    P.prod = prod;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kZhatPerWarp; ++q) {
            WarpZhatPole& P = pl[q];
            if (!P.act) continue;
            if (!P.fast) {  // exact redo
                P.prod = 1.0;
                for (int jg = P.ks + lane; jg < P.ks + P.K; jg += 32) {
                    const double del = (P.di - w.dA[P.ks + w.org[jg]]) - w.tau[jg];
                    if (jg - P.ks == P.i) P.prod = P.prod * del;
                    else P.prod = P.prod * (del * __drcp_rn(P.di - w.dA[jg]));
                }
            }
            const double W = bfly_mul(P.prod);
            if (lane == 0) {
                const double mag = sqrt(fmax(0.0, -W));
                w.zA[P.g] = w.zA[P.g] >= 0.0 ? mag : -mag;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// boundary rows + placement, kRowsPerWarp roots per warp
// ---------------------------------------------------------------------------
#ifndef BRGPU_ROWS_PER_WARP
#define BRGPU_ROWS_PER_WARP 2
#endif
constexpr int kRowsPerWarp = BRGPU_ROWS_PER_WARP;  // roots per warp in k_rows_warp
#ifndef BRGPU_ROWS_TILE
#define BRGPU_ROWS_TILE 512
#endif
constexpr int kRowsTile = BRGPU_ROWS_TILE;  // poles per k_rows_warp tile (2 buffers x 4 arrays: 32 KB)

__device__ __forceinline__ void rows_fetch(double (*tile)[kRowsTile], const Work& w, int a, int b) {
    for (int i = a + (int)threadIdx.x; i < b; i += kWarpThreads) {
        const double* src[4] = {w.dA + i, w.zA + i, w.r0A + i, w.r1A + i};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(&tile[c][i - a]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src[c]) : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// One root of k_rows_warp.
struct WarpRowRoot {
    int g, ks, K, p;
    bool rows, fast;
    double dorg, tau;
};

// Up to kRowsPerWarp roots per warp: a pole tile read from shared memory
// (d, zhat, r0, r1: 32 B per term) feeds every root of the warp, so the SMEM
// traffic per FP64 term halves (the 1-root loop moved 8 SMEM wavefronts per
// 5.5 FP64-issue cycles and was SMEM-bound).  Each root keeps its own lane-
// strided accumulation order and butterfly, so results are bitwise those of
// one root per warp.
#ifndef BRGPU_ROWS_MINB
#define BRGPU_ROWS_MINB 4  // CTAs per SM (64 registers): C3 rows 3.14 -> 3.02 ms
#endif
__global__ void __launch_bounds__(kWarpThreads, BRGPU_ROWS_MINB) k_rows_warp(Work w, LevelDev L, int n) {
    pdl_entry();
    // two buffers of (d, zhat, r0, r1) tiles: the next tile streams in by
    // cp.async while the current one is consumed
    __shared__ __align__(16) double s_rt[2][4][kRowsTile];
    if (!L.allSplit && !(*w.levelModes & 2)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int RPC = (kWarpThreads / 32) * kRowsPerWarp;  // roots per CTA step
    for (int base = blockIdx.x * RPC; base < T; base += gridDim.x * RPC) {
        WarpRowRoot rt[kRowsPerWarp];
        bool any = false;
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            WarpRowRoot& R = rt[q];
            R.g = base + wid * kRowsPerWarp + q;
            R.ks = 0; R.K = 0; R.p = 0; R.rows = false; R.fast = false; R.dorg = 0.0; R.tau = 0.0;
            if (R.g < T) {
                const int m = w.aMerge[R.g];
                int ke;
                merge_active(w, L, m, R.ks, ke);
                if (split_mode(L.mSize[m], ke - R.ks)) {
                    R.K = ke - R.ks;
                    const int j = R.g - R.ks;
                    const int off = L.mOff[m], size = L.mSize[m];
                    R.dorg = w.dA[R.ks + w.org[R.g]];
                    R.tau = w.tau[R.g];
                    const double lam = R.dorg + R.tau;
                    const int pos = j + count_leq(w.D + off, size, lam) - count_leq(w.dA + R.ks, R.K, lam);
                    R.p = off + pos;
                    if (lane == 0) {
                        w.lam[R.p] = lam;
                        w.tau[R.g] = lam;  // dead after the reads above: k_deflated_out searches root
                        w.org[R.g] = R.p;  // values, the root-range split exchange finds the position
                    }
                    R.rows = !(L.mFlags[m] & kMergeRoot) && owns(w, R.g);
                    R.fast = R.rows && !w.exact &&
                             eval_guard(GlobalPairs{w.dA + R.ks, w.z2A + R.ks}, R.K, j, R.dorg, R.tau);
                }
            }
            any = any || R.rows;
        }
        if (!__syncthreads_or(any)) continue;
        const int gl = min(base + RPC, T) - 1;
        int P0, P1, tmp;
        merge_active(w, L, w.aMerge[base], P0, tmp);
        merge_active(w, L, w.aMerge[gl], tmp, P1);
        double nn[kRowsPerWarp], s0[kRowsPerWarp], s1[kRowsPerWarp];
        bool shared = true;  // every fast root of the warp streams the same pole range
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            nn[q] = 0.0; s0[q] = 0.0; s1[q] = 0.0;
            shared = shared && rt[q].fast && rt[q].ks == rt[0].ks;
        }
        int buf = 0;
        rows_fetch(s_rt[0], w, P0, min(P0 + kRowsTile, P1));
        for (int tlo = P0; tlo < P1; tlo += kRowsTile) {
            const int thi = min(tlo + kRowsTile, P1);
            cp_async_wait_all();
            __syncthreads();
            if (thi < P1) rows_fetch(s_rt[buf ^ 1], w, thi, min(thi + kRowsTile, P1));
            const double* __restrict__ s_d = s_rt[buf][0];
            const double* __restrict__ s_zh = s_rt[buf][1];
            const double* __restrict__ s_r0 = s_rt[buf][2];
            const double* __restrict__ s_r1 = s_rt[buf][3];
            if (shared) {
                const int ks = rt[0].ks;
                const int lo = max(ks, tlo), hi = min(ks + rt[0].K, thi);
#pragma unroll 2
                for (int i = strided_start(lo, ks, lane); i < hi; i += 32) {
                    const int t = i - tlo;
                    const double d = s_d[t], zh = s_zh[t], a0 = s_r0[t], a1 = s_r1[t];
#pragma unroll
                    for (int q = 0; q < kRowsPerWarp; ++q) {
                        const double y = zh * rcp_nr((d - rt[q].dorg) - rt[q].tau);
                        nn[q] = __fma_rn(y, y, nn[q]);
                        s0[q] = __fma_rn(a0, y, s0[q]);
                        s1[q] = __fma_rn(a1, y, s1[q]);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q) {
                    if (!rt[q].fast) continue;
                    const int ks = rt[q].ks;
                    const double dorg = rt[q].dorg, tau = rt[q].tau;
                    const int lo = max(ks, tlo), hi = min(ks + rt[q].K, thi);
                    for (int i = strided_start(lo, ks, lane); i < hi; i += 32) {
                        const int t = i - tlo;
                        const double y = s_zh[t] * rcp_nr((s_d[t] - dorg) - tau);
                        nn[q] = __fma_rn(y, y, nn[q]);
                        s0[q] = __fma_rn(s_r0[t], y, s0[q]);
                        s1[q] = __fma_rn(s_r1[t], y, s1[q]);
                    }
                }
            }
            buf ^= 1;
        }
        __syncthreads();  // the last tile is consumed before the next step's prefetch
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            const WarpRowRoot& R = rt[q];
            if (!R.rows) continue;
            if (!R.fast) {  // exact redo; a zero delta is an error
                bool zero = false;
                nn[q] = 0.0; s0[q] = 0.0; s1[q] = 0.0;
                for (int i = R.ks + lane; i < R.ks + R.K; i += 32) {
                    const double del = (w.dA[i] - R.dorg) - R.tau;
                    zero |= (del == 0.0);
                    const double y = w.zA[i] * __drcp_rn(del);
                    nn[q] = __fma_rn(y, y, nn[q]);
                    s0[q] = __fma_rn(w.r0A[i], y, s0[q]);
                    s1[q] = __fma_rn(w.r1A[i], y, s1[q]);
                }
                if (__any_sync(0xffffffffu, zero) && lane == 0) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
            }
            const double NN = bfly_add(nn[q]), S0 = bfly_add(s0[q]), S1 = bfly_add(s1[q]);
            if (lane == 0) {
                const double inv = 1.0 / sqrt(NN);
                w.blo[R.p] = S0 * inv;
                w.bhi[R.p] = S1 * inv;
            }
        }
    }
}

// Grids of the warp tier (CTAs per SM, times the SM count): the secular kernel
// takes chunks of roots per CTA, the z-hat / rows kernels stride over roots.
#ifndef BRGPU_WARP_SEC_PER_SM
#define BRGPU_WARP_SEC_PER_SM 16
#endif
#ifndef BRGPU_WARP_ROW_PER_SM
#define BRGPU_WARP_ROW_PER_SM 24
#endif
constexpr int kWarpSecPerSm = BRGPU_WARP_SEC_PER_SM;
constexpr int kWarpRowPerSm = BRGPU_WARP_ROW_PER_SM;
static int warp_grid(const SolveParams& prm, int per_sm) { return prm.sms * per_sm; }

constexpr size_t kSecWSmem = 2 * kSecWTile * sizeof(double2);

void init_warp_attributes() {
    cudaFuncSetAttribute(k_secular_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSecWSmem);
}

void launch_secular_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_secular_warp, warp_grid(prm, kWarpSecPerSm), kSecWThreads, kSecWSmem, s, w, L, n, prm.patched);
}
void launch_zhat_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_zhat_warp, warp_grid(prm, kWarpRowPerSm), kWarpThreads, 0, s, w, L, n);
}
void launch_rows_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_rows_warp, warp_grid(prm, kWarpRowPerSm), kWarpThreads, 0, s, w, L, n);
}

}  // namespace brgpu
