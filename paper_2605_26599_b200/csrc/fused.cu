// fused.cu -- one-launch-per-level merge kernel for the bottom of the tree.
//
// A CTA owns a GROUP of consecutive whole merges of one level (<= kFuseMax
// elements, <= kFuseMaxMerges merges, contiguous in position).  Everything a
// merge does happens in shared memory: per-merge tolerance (deflate.cpp:55-60),
// the stable merge of the sorted children with z = (sign*bhi_L, blo_R)
// (deflate.cpp:31-41, 62-66), small-z compaction, the close-pole Givens walk
// with its replay on the two selected rows (deflate.cpp:70-107, 109-140), the
// survivor compaction, the secular roots (secular.cpp:80-241; resumable
// per-lane RootSM with a CTA root queue), the Gu-Eisenstat weights
// (secular.cpp:288-313) and the boundary-row streaming R_parent(:,j) =
// R_child y_j -- then the parent state is written to HBM
// once.  Arithmetic and every reduction order are those of the grid-tier
// kernels in kernels.cu (and of oracle/br_oracle.c): results are bit-identical.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"
#include "grid_common.cuh"

namespace brgpu {

// CTAs per SM of the 512-element shape: both bounds are instantiated.  3 CTAs
// (80 registers) when the launch fits one wave at 3 per SM: a short, latency-bound
// launch (n = 4096: 0.71 ms against 0.76 ms at 4); 4 CTAs (64 registers, ~90 B
// of root-state spills outside the pole loops) when it does not (glued Wilkinson
// 2^18: 7.96 -> 7.78 ms; random 2^20 4.09 -> 4.08 ms).
constexpr int kFuseMinbFew = 3;
constexpr int kFuseMinbMany = 4;
constexpr int kFuseMaxMerges = 128;   // merges per group
#ifndef BRGPU_SMALL_THREADS
#define BRGPU_SMALL_THREADS 256
#endif
constexpr int kSmallThreads = BRGPU_SMALL_THREADS;  // threads of the 512-element shape
#ifndef BRGPU_BIG_THREADS
#define BRGPU_BIG_THREADS 256
#endif
constexpr int kBigThreads = BRGPU_BIG_THREADS;  // threads of the 1024-element shape

// Two shapes: groups of <= 1024 elements on 256 threads (merges of 513..1024,
// two CTAs per SM) and groups of <= 512 on 256 threads (merges <= 512, four
// CTAs and 32 warps per SM at 64 registers, so one CTA's root-queue tail
// overlaps the others' work; random 2^20: 4.76 -> 4.66 ms).
template <int kFuseMax, int kFuseThreads>
struct FuseSmem {
    // sorted merge arrays (local positions)
    double D[kFuseMax];
    double Z[kFuseMax];
    double R0[kFuseMax];
    double R1[kFuseMax];
    // inputs (lam, blo, bhi); after the scatter: active (d, z^2) pairs + active z / z-hat
    double in[3 * kFuseMax];
    double r0A[kFuseMax];
    double r1A[kFuseMax];
    double tau[kFuseMax];
    int org[kFuseMax];
    int nnPre[kFuseMax + 1];
    int nnPos[kFuseMax];
    int survPre[kFuseMax + 1];
    unsigned char flag[kFuseMax];
    unsigned char surv[kFuseMax];
    // per-merge metadata
    int mo[kFuseMaxMerges + 1];  // local offsets (+ end)
    int ms[kFuseMaxMerges];
    int mnl[kFuseMaxMerges];
    int mf[kFuseMaxMerges];
    int kS[kFuseMaxMerges + 1];  // active ranges
    double rho[kFuseMaxMerges];
    double neg[kFuseMaxMerges];  // -1 when e_m < 0
    unsigned long long tolb[kFuseMaxMerges];
    int scan[kFuseThreads / 32];
    int ne[kFuseMaxMerges + 1];  // merges with K > 0 before t (root queue order)
    int next;
    int cnt;
    unsigned long long evals, terms;
};

// One group of merges of one level: merges m0 .. m0+cnt-1 (level-local
// indices) tile a contiguous range; state in and out through w.lam/blo/bhi.
template <int kFuseMax, int kFuseThreads>
__device__ __forceinline__ void fused_group(const Work& w, const LevelDev& L, const int m0, const int cnt,
                                            const SolveParams& prm, int* __restrict__ traceOut,
                                            FuseSmem<kFuseMax, kFuseThreads>& S) {
    const int tid = threadIdx.x;
    const int base = L.mOff[m0];
#ifdef BRGPU_PHASE_PROF
    // phase cycle accounting (profiling builds only): deflation / secular /
    // refreshed weights / rows + placement, summed over CTAs in counters[4..7]
    long long ph_t = clock64();
#define PHASE_MARK(k)                                                              \
    do {                                                                           \
        if (tid == 0) {                                                            \
            const long long t_ = clock64();                                        \
            atomicAdd(&w.counters[4 + (k)], (unsigned long long)(t_ - ph_t));      \
            ph_t = t_;                                                             \
        }                                                                          \
    } while (0)
#else
#define PHASE_MARK(k) do {} while (0)
#endif

    // ---- metadata + inputs -------------------------------------------------
    if (tid < cnt) {
        const int m = m0 + tid;
        const int off = L.mOff[m] - base, nl = L.mNL[m];
        S.mo[tid] = off;
        S.ms[tid] = L.mSize[m];
        S.mnl[tid] = nl;
        S.mf[tid] = L.mFlags[m];
        const double em = w.ew[L.mOff[m] + nl - 1];
        S.rho[tid] = fabs(em);
        S.neg[tid] = em < 0 ? -1.0 : 1.0;
        S.tolb[tid] = 0ULL;
        if (tid == cnt - 1) S.mo[cnt] = off + L.mSize[m];
    }
    if (tid == 0) {
        S.next = 0;
        S.evals = 0;
        S.terms = 0;
        S.cnt = cnt;
    }
    __syncthreads();
    const int E = S.mo[cnt];
    double* lamIn = S.in;
    double* bloIn = S.in + kFuseMax;
    double* bhiIn = S.in + 2 * kFuseMax;
    for (int i = tid; i < E; i += kFuseThreads) {
        lamIn[i] = w.lam[base + i];
        bloIn[i] = w.blo[base + i];
        bhiIn[i] = w.bhi[base + i];
    }
    __syncthreads();

    // ---- tolerance: max(|D|, |z|) per merge ---------------------------------
    // (segmented warp max over consecutive elements, one shared atomic per
    // merge segment: 64-bit shared atomics are CAS loops on sm_100a)
    for (int b0 = 0; b0 < E; b0 += kFuseThreads) {
        const int i = b0 + tid;
        const bool valid = i < E;
        int t = -1;
        unsigned long long v = 0ULL;
        if (valid) {
            t = upper_index(S.mo, cnt, i);
            const double zv = (i - S.mo[t] < S.mnl[t]) ? bhiIn[i] : bloIn[i];
            v = (unsigned long long)__double_as_longlong(fmax(fabs(lamIn[i]), fabs(zv)));
        }
        const int lane = tid & 31;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long v2 = __shfl_down_sync(0xffffffffu, v, off);
            const int t2 = __shfl_down_sync(0xffffffffu, t, off);
            if (lane + off < 32 && t2 == t && v2 > v) v = v2;
        }
        const int tp = __shfl_up_sync(0xffffffffu, t, 1);
        if (valid && (lane == 0 || tp != t)) atomicMax(&S.tolb[t], v);
    }
    __syncthreads();

    // ---- stable merge of the two sorted children + z ------------------------
    for (int i = tid; i < E; i += kFuseThreads) {
        const int t = upper_index(S.mo, cnt, i);
        const int off = S.mo[t], nl = S.mnl[t], nr = S.ms[t] - nl;
        const double v = lamIn[i];
        int sp;
        double z, r0, r1;
        if (i < off + nl) {
            sp = i + count_less(lamIn + off + nl, nr, v);
            const double b = bhiIn[i];
            z = S.neg[t] < 0 ? -b : b;
            r0 = bloIn[i];
            r1 = 0.0;
        } else {
            sp = (i - nl) + count_leq(lamIn + off, nl, v);
            z = bloIn[i];
            r0 = 0.0;
            r1 = bhiIn[i];
        }
        S.D[sp] = v;
        S.Z[sp] = z;
        S.R0[sp] = r0;
        S.R1[sp] = r1;
    }
    __syncthreads();

    // ---- small-z flags + NN compaction --------------------------------------
    for (int i = tid; i < E; i += kFuseThreads) {
        const int t = upper_index(S.mo, cnt, i);
        const double tol = 8.0 * kU * __longlong_as_double((long long)S.tolb[t]) * prm.tol_scale;
        S.flag[i] = fabs(S.Z[i]) > tol;
    }
    __syncthreads();
    const int NN = cta_scan_flags<kFuseThreads>(S.flag, E, S.nnPre, S.scan);
    for (int i = tid; i < E; i += kFuseThreads)
        if (S.flag[i]) S.nnPos[S.nnPre[i]] = i;
    __syncthreads();

    // ---- close-pole deflation: segment heads walk their runs ----------------
    // (group rotation chains from prefix sums, k_segment_walk's arithmetic;
    // member prefixes go to the dead input slots, members finish in parallel)
    {
        double* pQ = lamIn;
        double* pS0 = bloIn;
        double* pS1 = bhiIn;
        for (int q = tid; q < NN; q += kFuseThreads) {
            const int k = S.nnPos[q];
            const int t = upper_index(S.mo, cnt, k);
            const int qs = S.nnPre[S.mo[t]], qe = S.nnPre[S.mo[t] + S.ms[t]];
            const double tol = 8.0 * kU * __longlong_as_double((long long)S.tolb[t]) * prm.tol_scale;
            if (q > qs && fabs(S.D[k] - S.D[S.nnPos[q - 1]]) <= tol) continue;  // not a head
            S.surv[q] = 1;
            int prev = k, nmem = 0;
            double dp = S.D[k];
            const double zs = S.Z[k];
            double Q = zs * zs, S0 = zs * S.R0[k], S1 = zs * S.R1[k];
            double dprev_nn = dp;
            for (int q2 = q + 1; q2 < qe; ++q2) {
                const int k2 = S.nnPos[q2];
                const double d2 = S.D[k2];
                if (fabs(d2 - dprev_nn) > tol) break;
                dprev_nn = d2;
                const double zq = S.Z[k2];
                if (fabs(d2 - dp) <= tol) {
                    pQ[k2] = Q;
                    pS0[k2] = S0;
                    pS1[k2] = S1;
                    Q = Q + zq * zq;
                    S0 = S0 + zq * S.R0[k2];
                    S1 = S1 + zq * S.R1[k2];
                    ++nmem;
                    S.surv[q2] = 0;
                } else {
                    if (nmem) {
                        const double R = sqrt(Q), iR = 1.0 / R;
                        S.Z[prev] = R; S.R0[prev] = S0 * iR; S.R1[prev] = S1 * iR;
                    }
                    S.surv[q2] = 1;
                    prev = k2; dp = d2; nmem = 0;
                    Q = zq * zq; S0 = zq * S.R0[k2]; S1 = zq * S.R1[k2];
                }
            }
            if (nmem) {
                const double R = sqrt(Q), iR = 1.0 / R;
                S.Z[prev] = R; S.R0[prev] = S0 * iR; S.R1[prev] = S1 * iR;
            }
        }
        __syncthreads();
        for (int q = tid; q < NN; q += kFuseThreads) {
            if (S.surv[q]) continue;
            const int k = S.nnPos[q];
            double x0 = S.R0[k], x1 = S.R1[k];
            group_member(pQ[k], pS0[k], pS1[k], S.Z[k], x0, x1);
            S.R0[k] = x0;
            S.R1[k] = x1;
            S.Z[k] = 0.0;
        }
    }
    __syncthreads();

    // ---- survivor compaction: active (d, z^2) pairs, z, rows ----------------
    const int T = cta_scan_flags<kFuseThreads>(S.surv, NN, S.survPre, S.scan);
    double2* pairs = reinterpret_cast<double2*>(S.in);   // aliases lam/blo inputs (dead)
    double* zA = S.in + 2 * kFuseMax;                     // aliases bhi input (dead)
    for (int q = tid; q < NN; q += kFuseThreads) {
        if (!S.surv[q]) continue;
        const int g = S.survPre[q], k = S.nnPos[q];
        const double z = S.Z[k];
        pairs[g] = make_double2(S.D[k], z * z);
        zA[g] = z;
        S.r0A[g] = S.R0[k];
        S.r1A[g] = S.R1[k];
    }
    if (tid <= cnt) S.kS[tid] = S.survPre[S.nnPre[tid < cnt ? S.mo[tid] : E]];
    __syncthreads();
    // Root queue order: every merge's last root first (the one-pole model of the
    // root above the largest pole averages ~2.5x the evaluations of an interior
    // root: started last it would set the secular phase's tail), then the
    // interior roots in order.  The order never changes a result.  ne[t] = merges
    // with K > 0 before t; the order lives in nnPos (dead after the compaction).
    if (tid <= cnt) {
        int c = 0;
        for (int u = 0; u < tid; ++u) c += S.kS[u + 1] > S.kS[u];
        S.ne[tid] = c;
    }
    __syncthreads();
    int* qorder = S.nnPos;
    for (int g = tid; g < T; g += kFuseThreads) {
        const int t = upper_index(S.kS, cnt, g);
        qorder[g == S.kS[t + 1] - 1 ? S.ne[t] : S.ne[cnt] + g - S.ne[t]] = g;
    }
    __syncthreads();

    PHASE_MARK(0);
    // ---- secular roots: per-lane RootSM, CTA queue --------------------------
    {
        // per-thread prefix snapshot slot; S.Z is dead between compaction and sDorg
        double2* snap = reinterpret_cast<double2*>(S.Z) + tid;
        RootSM st;
        int g = -1, ks = 0;
        bool exhausted = false;
        unsigned long long evals = 0, terms = 0;
        for (;;) {
            while (g < 0 && !exhausted) {
                const int q = atomicAdd(&S.next, 1);
                if (q >= T) { exhausted = true; break; }
                g = qorder[q];
                const int t = upper_index(S.kS, cnt, g);
                ks = S.kS[t];
                const int K = S.kS[t + 1] - ks;
                rs_begin(st, K, g - ks, S.rho[t], PolesPairs{pairs + ks}, zA[ks], Z2Pairs{pairs + ks});
                if (st.phase == kRsDone) {
                    S.org[g] = st.org;
                    S.tau[g] = st.tau;
                    g = -1;
                }
            }
            if (!__any_sync(0xffffffffu, g >= 0)) break;
            if (g >= 0) {
                double sum, sum_abs, sum_d, psi;
                bool pole = false;
                const SmemPairs P{pairs + ks};
                if (!w.exact && eval_guard(P, st.K, st.j, st.dorg, st.tau))
                    eval_fast(P, st.K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi, snap);
                else
                    pole = eval_pass_exact(P, st.K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi);
                Ev ev;
                ev.f = 1.0 + st.rho * sum;
                ev.fp = st.rho * sum_d;
                ev.abs_sum = st.rho * sum_abs;
                ev.psi = st.rho * psi;
                ev.pole = pole;
                ++evals;
                terms += (unsigned long long)st.K;
                rs_consume(st, ev, PolesPairs{pairs + ks}, Z2Pairs{pairs + ks}, prm.patched != 0);
                if (st.phase == kRsDone || st.phase == kRsFail) {
                    if (st.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                    S.org[g] = st.org;
                    S.tau[g] = st.tau;
                    g = -1;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            evals += __shfl_xor_sync(0xffffffffu, evals, o);
            terms += __shfl_xor_sync(0xffffffffu, terms, o);
        }
        if ((tid & 31) == 0 && evals) {
            atomicAdd(&w.counters[2], evals);
            atomicAdd(&w.counters[3], terms);
        }
    }
    __syncthreads();

    double* sDorg = S.Z;  // d[origin] per root (lambda = dorg + tau); S.Z is dead after compaction
    for (int g = tid; g < T; g += kFuseThreads) {
        const int t = upper_index(S.kS, cnt, g);
        sDorg[g] = pairs[S.kS[t] + S.org[g]].x;
    }
    __syncthreads();

    PHASE_MARK(1);
    // ---- Gu-Eisenstat refreshed weights (non-root merges) --------------------
    if (prm.zhat) {
        for (int g = tid; g < T; g += kFuseThreads) {
            const int t = upper_index(S.kS, cnt, g);
            if (S.mf[t] & kMergeRoot) continue;
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if (K == 1) continue;  // a lone pole keeps its z (the checker refreshes only K > 1)
            const double di = pairs[g].x;
            double prod = 1.0;
            const bool fast = !w.exact && zhat_guard(PolesPairs{pairs + ks}, K, i);
            if (fast) {
#pragma unroll 4
                for (int j = 0; j < K; ++j) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    const double dd = di - pairs[ks + j].x;
                    const double f = (j == i) ? del : del * rcp_nr(dd);
                    prod = prod * f;
                }
            } else {
                prod = 1.0;
                for (int j = 0; j < K; ++j) {
                    const double del = (di - pairs[ks + S.org[ks + j]].x) - S.tau[ks + j];
                    if (j == i) prod = prod * del;
                    else prod = prod * (del * __drcp_rn(di - pairs[ks + j].x));
                }
            }
            const double mag = sqrt(fmax(0.0, -prod));
            zA[g] = zA[g] >= 0.0 ? mag : -mag;
        }
        __syncthreads();
    }

    PHASE_MARK(2);
    // ---- roots: boundary rows + placement; deflated columns: placement -------
    for (int g = tid; g < T; g += kFuseThreads) {
        const int t = upper_index(S.kS, cnt, g);
        const int ks = S.kS[t], K = S.kS[t + 1] - ks, j = g - ks;
        const int off = S.mo[t], size = S.ms[t];
        const double dorg = sDorg[g];
        const double tau = S.tau[g];
        const double lam = dorg + tau;
        // #{dA <= lam} over the merge's active poles
        int lo = 0, hi = K;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (!(lam < pairs[ks + mid].x)) lo = mid + 1; else hi = mid;
        }
        const int pos = j + count_leq(S.D + off, size, lam) - lo;
        const int p = base + off + pos;
        w.lam[p] = lam;
        if (S.mf[t] & kMergeRoot) continue;
        double nn = 0.0, s0 = 0.0, s1 = 0.0;
        if (!w.exact && eval_guard(SmemPairs{pairs + ks}, K, j, dorg, tau)) {
#pragma unroll 4
            for (int i = 0; i < K; ++i) {
                const double y = zA[ks + i] * rcp_nr((pairs[ks + i].x - dorg) - tau);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
        } else {
            bool zero = false;
            nn = 0.0; s0 = 0.0; s1 = 0.0;
            for (int i = 0; i < K; ++i) {
                const double del = (pairs[ks + i].x - dorg) - tau;
                zero |= (del == 0.0);
                const double y = zA[ks + i] * __drcp_rn(del);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
            if (zero) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
        }
        const double inv = 1.0 / sqrt(nn);
        w.blo[p] = s0 * inv;
        w.bhi[p] = s1 * inv;
    }
    for (int k = tid; k < E; k += kFuseThreads) {
        const int q = S.nnPre[k];
        if (S.flag[k] && S.surv[q]) continue;  // survivor: placed above
        const int t = upper_index(S.mo, cnt, k);
        const int off = S.mo[t];
        const int ks = S.kS[t], K = S.kS[t + 1] - ks;
        const int tt = (k - off) - (S.survPre[q] - ks);
        const double v = S.D[k];
        int lo = 0, hi = K;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const double lj = sDorg[ks + mid] + S.tau[ks + mid];
            if (lj < v) lo = mid + 1; else hi = mid;
        }
        const int p = base + off + tt + lo;
        w.lam[p] = v;
        if (!(S.mf[t] & kMergeRoot)) {
            w.blo[p] = S.R0[k];
            w.bhi[p] = S.R1[k];
        }
    }

#ifdef BRGPU_PHASE_PROF
    __syncthreads();
#endif
    PHASE_MARK(3);
#undef PHASE_MARK
    // ---- stats / trace -------------------------------------------------------
    if (traceOut && tid < cnt) {
        traceOut[2 * (m0 + tid)] = S.nnPre[S.mo[tid] + S.ms[tid]] - S.nnPre[S.mo[tid]];
        traceOut[2 * (m0 + tid) + 1] = S.kS[tid + 1] - S.kS[tid];
    }
}

template <int kFuseMax, int kFuseThreads, int MINB>
__global__ void __launch_bounds__(kFuseThreads, kFuseMax <= 512 ? MINB : 2048 / kFuseMax)
k_level_fused(Work w, LevelDev L, const int* __restrict__ gFirst, const int* __restrict__ gCount,
              SolveParams prm, int* __restrict__ traceOut) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char fuse_raw[];
    using Smem = FuseSmem<kFuseMax, kFuseThreads>;
    Smem& S = *reinterpret_cast<Smem*>(fuse_raw);
    fused_group<kFuseMax, kFuseThreads>(w, L, gFirst[blockIdx.x], gCount[blockIdx.x], prm, traceOut, S);
}

// Several consecutive levels in one launch: CTA b owns one group of the top
// level and, below it, the merges of every lower level of the run that tile
// the same range (tab[b*nlev + l] = (first, count)); a level's outputs are
// the next level's inputs, so the CTA moves from level to level with a block
// barrier instead of a grid-wide kernel boundary (the data stays in L1/L2),
// and different CTAs' root-queue tails overlap across levels.
template <int kFuseMax, int kFuseThreads, int MINB>
__global__ void __launch_bounds__(kFuseThreads, MINB)
k_levels_fused(Work w, FusedRun run, const int2* __restrict__ tab, SolveParams prm) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char fuse_raw[];
    using Smem = FuseSmem<kFuseMax, kFuseThreads>;
    Smem& S = *reinterpret_cast<Smem*>(fuse_raw);
    for (int l = 0; l < run.nlev; ++l) {
        const int2 fc = tab[blockIdx.x * run.nlev + l];
        fused_group<kFuseMax, kFuseThreads>(w, run.L[l], fc.x, fc.y, prm, run.trace[l], S);
        __syncthreads();
    }
}

void launch_level_fused(cudaStream_t s, const Work& w, const LevelDev& L, int ngroups, int cap,
                        const int* gFirst, const int* gCount, const SolveParams& prm, int* traceOut,
                        int* launches, Prof* prof) {
    if (cap <= 512 && ngroups > kFuseMinbFew * prm.sms)
        launch_pdl(k_level_fused<512, kSmallThreads, kFuseMinbMany>, ngroups, kSmallThreads, sizeof(FuseSmem<512, kSmallThreads>), s, w, L, gFirst, gCount, prm,
                                                                                 traceOut);
    else if (cap <= 512)
        launch_pdl(k_level_fused<512, kSmallThreads, kFuseMinbFew>, ngroups, kSmallThreads, sizeof(FuseSmem<512, kSmallThreads>), s, w, L, gFirst, gCount, prm,
                                                                                 traceOut);
    else
        launch_pdl(k_level_fused<1024, kBigThreads, 2>, ngroups, kBigThreads, sizeof(FuseSmem<1024, kBigThreads>), s, w, L, gFirst, gCount, prm,
                                                                                   traceOut);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_SUBTREE);
}

void launch_levels_fused(cudaStream_t s, const Work& w, const FusedRun& run, int ngroups, const int2* tab,
                         const SolveParams& prm, int* launches, Prof* prof) {
    if (ngroups > kFuseMinbFew * prm.sms)
        launch_pdl(k_levels_fused<512, kSmallThreads, kFuseMinbMany>, ngroups, kSmallThreads,
                   sizeof(FuseSmem<512, kSmallThreads>), s, w, run, tab, prm);
    else
        launch_pdl(k_levels_fused<512, kSmallThreads, kFuseMinbFew>, ngroups, kSmallThreads,
                   sizeof(FuseSmem<512, kSmallThreads>), s, w, run, tab, prm);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_SUBTREE);
}

static_assert(sizeof(FuseSmem<1024, kBigThreads>) <= 113 * 1024, "two fused CTAs must fit one SM (227 KB)");
static_assert(sizeof(FuseSmem<512, kSmallThreads>) <= 56 * 1024, "four small fused CTAs must fit one SM");

void init_fused_attributes() {
    const int small = (int)sizeof(FuseSmem<512, kSmallThreads>);
    cudaFuncSetAttribute(k_level_fused<1024, kBigThreads, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(FuseSmem<1024, kBigThreads>));
    cudaFuncSetAttribute(k_level_fused<512, kSmallThreads, kFuseMinbFew>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, small);
    cudaFuncSetAttribute(k_level_fused<512, kSmallThreads, kFuseMinbMany>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, small);
    cudaFuncSetAttribute(k_levels_fused<512, kSmallThreads, kFuseMinbFew>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, small);
    cudaFuncSetAttribute(k_levels_fused<512, kSmallThreads, kFuseMinbMany>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, small);
}

}  // namespace brgpu
