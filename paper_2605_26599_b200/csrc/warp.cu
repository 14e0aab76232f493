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
#include "level_state.cuh"

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
#ifndef BRGPU_SECW_SLOTS
#define BRGPU_SECW_SLOTS 2
#endif
#ifndef BRGPU_SECW2_MINB
#define BRGPU_SECW2_MINB 2
#endif
constexpr int kSecWSlots = BRGPU_SECW_SLOTS;  // roots per warp in k_secular_warp (large-K levels)
#ifndef BRGPU_SECW2_MIN_ROOTS
#define BRGPU_SECW2_MIN_ROOTS 16384
#endif
constexpr int kSecW2MinRoots = kSecWSlots == 1 ? 0x7fffffff : BRGPU_SECW2_MIN_ROOTS;

// Partial sums of one root's evaluation (lane-strided terms, split at the
// root's own index for the prefix snapshot).
struct SecAcc {
    double sum, sum_d, psi, psum;
};

__device__ __forceinline__ void sec_terms(const double2* __restrict__ tp, int& i, int stop, double dorg, double tau,
                                          SecAcc& A) {
#pragma unroll 4
    for (; i < stop; i += 32) {
        const double2 dz = tp[i];
        const double r = rcp_nr((dz.x - dorg) - tau);
        const double t = dz.y * r;
        A.sum += t;
        A.sum_d = __fma_rn(t, r, A.sum_d);
    }
}

// Two roots of one merge: each (d, z^2) pair read from shared memory feeds
// both (half the SMEM traffic and barriers per root; 2 x 8 roots in flight per
// CTA).  Per root the terms and their order are those of sec_terms.
__device__ __forceinline__ void sec_terms2(const double2* __restrict__ tp, int& i, int stop, double dorg0,
                                           double tau0, double dorg1, double tau1, SecAcc& A, SecAcc& B) {
#pragma unroll 2
    for (; i < stop; i += 32) {
        const double2 dz = tp[i];
        const double r0 = rcp_nr((dz.x - dorg0) - tau0);
        const double r1 = rcp_nr((dz.x - dorg1) - tau1);
        const double t0 = dz.y * r0, t1 = dz.y * r1;
        A.sum += t0;
        A.sum_d = __fma_rn(t0, r0, A.sum_d);
        B.sum += t1;
        B.sum_d = __fma_rn(t1, r1, B.sum_d);
    }
}

// Secular roots, kSecWSlots roots per warp (split arithmetic: lane-strided
// terms + xor butterfly, bitwise the checker's BRO_SPLIT evaluation).  A CTA
// owns a chunk of roots and a CTA queue; every evaluation round streams the
// chunk's pole window through shared memory once for all its warps' roots.
template <int NS>
__global__ void __launch_bounds__(kSecWThreads, NS == 1 ? BRGPU_SECW_MINB : BRGPU_SECW2_MINB)
k_secular_warp(Work w, LevelDev L, int n, int patched) {
    pdl_entry();
    if (!dense_entry(L)) return;
    extern __shared__ __align__(16) double2 s_tiles[];  // two tiles of kSecWTile pairs (dynamic)
    __shared__ int s_next;
    if (!L.allSplit && !(*w.levelModes & 2)) return;
    const int T = w.survPre[w.nnPre[n]];
    // the second root slot of a warp is used only on large-K levels (Toeplitz /
    // glued Wilkinson tops: half the SMEM traffic and barriers per root); on a
    // level with few roots one root per warp keeps more warps busy
    const int nsl = T < kSecW2MinRoots ? 1 : NS;
    const int G = (int)gridDim.x;
    const int R = max(kSecWThreads / 32 * nsl, (T + G - 1) / G);
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
    if (resident) {
        tile_fetch(s_tiles, w, P0, P1);
        cp_async_wait_all();
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (resident) {
        // the whole window is in shared memory: every warp runs its roots to
        // convergence on its own (no per-evaluation block barriers; the few-root
        // top levels of random inputs were bound by those rounds)
        unsigned long long ev = 0, tm = 0;
        for (;;) {
            int qq = 0;
            if (lane == 0) qq = atomicAdd(&s_next, 1);
            qq = __shfl_sync(0xffffffffu, qq, 0);
            if (c0 + qq >= c1) break;
            const int gg = c0 + qq;
            if (!owns(w, gg)) continue;  // another rank's root (root-range split)
            const int m = w.aMerge[gg];
            int kss, ke;
            merge_active(w, L, m, kss, ke);
            if (!split_mode(L.mSize[m], ke - kss)) continue;  // lane-per-root tier owns it
            const double rho = fabs(w.ew[L.mOff[m] + L.mNL[m] - 1]);
            int o;
            double tu;
            root_warp(s_tiles + (kss - P0), w.zA + kss, ke - kss, gg - kss, rho, w.exact != 0, patched != 0,
                      w.status, o, tu, ev, tm);
            if (lane == 0) {
                w.org[gg] = kss + o;
                w.tau[gg] = tu;
            }
        }
        if (lane == 0 && ev) {
            atomicAdd(&w.counters[0], ev);
            atomicAdd(&w.counters[1], tm);
        }
        return;
    }

    RootSM st[NS];
    int g[NS], ks[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) { g[q] = -1; ks[q] = 0; }
    bool exhausted = false;
    unsigned long long evals = 0, terms = 0;
    for (;;) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            while (g[q] < 0 && !exhausted && q < nsl) {
                int qq = 0;
                if (lane == 0) qq = atomicAdd(&s_next, 1);
                qq = __shfl_sync(0xffffffffu, qq, 0);
                if (c0 + qq >= c1) { exhausted = true; break; }
                const int gg = c0 + qq;
                if (!owns(w, gg)) continue;  // another rank's root (root-range split)
                const int m = w.aMerge[gg];
                int ke;
                merge_active(w, L, m, ks[q], ke);
                if (!split_mode(L.mSize[m], ke - ks[q])) continue;  // lane-per-root tier owns it
                g[q] = gg;
                const int K = ke - ks[q], j = gg - ks[q];
                const double rho = fabs(w.ew[L.mOff[m] + L.mNL[m] - 1]);
                double zsq = 0.0;
                if (j == K - 1 && K > 1) {
                    for (int i = ks[q] + lane; i < ke; i += 32) zsq += w.z2A[i];
                    zsq = bfly_add(zsq);
                }
                rs_begin_zsq(st[q], K, j, rho, PolesPtr{w.dA + ks[q]}, w.zA[ks[q]], zsq, w.z2A[ks[q] + K - 1]);
                if (st[q].phase == kRsDone) {
                    if (lane == 0) { w.org[gg] = ks[q] + st[q].org; w.tau[gg] = st[q].tau; }
                    g[q] = -1;
                }
            }
        }
        bool need[NS], fast[NS];
        SecAcc acc[NS];
        bool any = false;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            need[q] = g[q] >= 0;
            any = any || need[q];
            acc[q] = SecAcc{0.0, 0.0, 0.0, 0.0};
            // neighbour range guard (eval_guard, numerics.cuh); on failure the
            // root skips the fast pass and runs the exact one below
            fast[q] = need[q] && !w.exact &&
                      eval_guard(GlobalPairs{w.dA + ks[q], w.z2A + ks[q]}, st[q].K, st[q].j, st[q].dorg, st[q].tau);
        }
        if (!__syncthreads_or(any)) break;
        // both roots fast and in one merge: one pass over the shared pole range,
        // split at both roots' own indices (prefix snapshots)
        const bool pair = NS == 2 && fast[0] && fast[NS - 1] && ks[0] == ks[NS - 1];
        int buf = 0;
        if (!resident) tile_fetch(s_tiles, w, P0, min(P0 + kSecWTile, P1));
        for (int tlo = P0; tlo < P1; tlo += kSecWTile) {
            const int thi = min(tlo + kSecWTile, P1);
            cp_async_wait_all();
            __syncthreads();
            if (thi < P1) tile_fetch(s_tiles + (buf ^ 1) * kSecWTile, w, thi, min(thi + kSecWTile, P1));
            const double2* __restrict__ tp = s_tiles + buf * kSecWTile - tlo;
            if (pair) {
                SecAcc& A = acc[0];
                SecAcc& B = acc[NS - 1];
                const int k0 = ks[0];
                const int lo = max(k0, tlo), hi = min(k0 + st[0].K, thi);
                const int m0 = min(hi, k0 + st[0].j + 1), m1 = min(hi, k0 + st[NS - 1].j + 1);
                const int midA = min(m0, m1), midB = max(m0, m1);
                const double d0 = st[0].dorg, t0 = st[0].tau, d1 = st[NS - 1].dorg, t1 = st[NS - 1].tau;
                int i = strided_start(lo, k0, lane);
                sec_terms2(tp, i, midA, d0, t0, d1, t1, A, B);
                if (lo < m0 && m0 == midA) { A.psi = A.sum_d; A.psum = A.sum; }
                if (lo < m1 && m1 == midA) { B.psi = B.sum_d; B.psum = B.sum; }
                sec_terms2(tp, i, midB, d0, t0, d1, t1, A, B);
                if (lo < m0 && m0 != midA) { A.psi = A.sum_d; A.psum = A.sum; }
                if (lo < m1 && m1 != midA) { B.psi = B.sum_d; B.psum = B.sum; }
                sec_terms2(tp, i, hi, d0, t0, d1, t1, A, B);
            } else {
#pragma unroll
                for (int q = 0; q < NS; ++q) {
                    if (!fast[q]) continue;
                    // terms i <= j, then the prefix snapshot, then i > j: a lane's
                    // strided terms are split at one point (no per-term selects)
                    const int lo = max(ks[q], tlo), hi = min(ks[q] + st[q].K, thi);
                    const int mid = min(hi, ks[q] + st[q].j + 1);
                    int i = strided_start(lo, ks[q], lane);
                    sec_terms(tp, i, mid, st[q].dorg, st[q].tau, acc[q]);
                    if (lo < mid) { acc[q].psi = acc[q].sum_d; acc[q].psum = acc[q].sum; }
                    sec_terms(tp, i, hi, st[q].dorg, st[q].tau, acc[q]);
                }
            }
            buf ^= 1;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            if (!need[q]) continue;
            RootSM& S = st[q];
            const int K = S.K, j = S.j;
            bool pole = false;
            if (!fast[q]) {  // rare: exact strided pass from global memory
                SecAcc& A = acc[q];
                A = SecAcc{0.0, 0.0, 0.0, 0.0};
                for (int i = ks[q] + lane; i < ks[q] + K; i += 32) {
                    const double del = (w.dA[i] - S.dorg) - S.tau;
                    pole |= (del == 0.0);
                    const double r = __drcp_rn(del);
                    const double t = w.z2A[i] * r;
                    A.sum += t;
                    A.sum_d = __fma_rn(t, r, A.sum_d);
                    if (i - ks[q] <= j) { A.psi = A.sum_d; A.psum = A.sum; }
                }
                pole = __any_sync(0xffffffffu, pole);
            }
            const double Sm = bfly_add(acc[q].sum), SD = bfly_add(acc[q].sum_d);
            const double PS = bfly_add(acc[q].psi), PU = bfly_add(acc[q].psum);
            Ev ev;
            ev.f = 1.0 + S.rho * Sm;
            ev.fp = S.rho * SD;
            ev.abs_sum = S.rho * (Sm - 2.0 * PU);
            ev.psi = S.rho * PS;
            ev.pole = pole;
            ++evals;
            terms += (unsigned long long)K;
            rs_consume(S, ev, PolesPtr{w.dA + ks[q]}, Z2Ptr{w.z2A + ks[q]}, patched != 0);
            if (S.phase == kRsDone || S.phase == kRsFail) {
                if (lane == 0) {
                    if (S.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                    w.org[g[q]] = ks[q] + S.org;
                    w.tau[g[q]] = S.tau;
                }
                g[q] = -1;
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
    if (!dense_entry(L)) return;
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
                s_dorg[r - tlo] = w.dA[w.org[r]];
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
                    const double del = (P.di - w.dA[w.org[jg]]) - w.tau[jg];
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
    if (!dense_entry(L)) return;
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
                    R.dorg = w.dA[w.org[R.g]];
                    R.tau = w.tau[R.g];
                    const double lam = R.dorg + R.tau;
                    const int pos = j + warp_count_leq(w.D + off, size, lam) - warp_count_leq(w.dA + R.ks, R.K, lam);
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
    cudaFuncSetAttribute(k_secular_warp<kSecWSlots>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSecWSmem);
}

int launch_secular_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_secular_warp<kSecWSlots>, warp_grid(prm, kWarpSecPerSm), kSecWThreads, kSecWSmem, s, w, L, n,
               prm.patched);
    return 1;
}
void launch_zhat_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_zhat_warp, warp_grid(prm, kWarpRowPerSm), kWarpThreads, 0, s, w, L, n);
}
void launch_rows_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm) {
    launch_pdl(k_rows_warp, warp_grid(prm, kWarpRowPerSm), kWarpThreads, 0, s, w, L, n);
}

}  // namespace brgpu
