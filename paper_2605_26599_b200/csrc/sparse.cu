// sparse.cu -- the sparse grid-tier level: three launches per level when every
// merge of the level has at most C non-negligible poles (NN).
//
// Above the fused SMEM levels, random inputs deflate almost everything: at
// n = 2^20 every merge from size 256 up to 2^20 keeps K ~ 100 active poles.
// The dense pipeline (kernels.cu) still moves every element of the level
// through ~15 launches (merged copies, scans over n, per-tier secular, z-hat
// and row kernels over level-global arrays).  Here a level is:
//
//   k_sp_flag   one persistent pass over the level's elements, three phases
//               separated by grid barriers: per-merge max(|D|, |z|)
//               (deflate.cpp:55-60), small-z flags (deflate.cpp:70-75) and an
//               ORDERED compaction of the non-negligible elements, in element
//               order (per merge: left child ascending, then right child
//               ascending) -- no merged copy of the level is written.
//   k_sp_solve  one CTA per group of merges (whole merges, <= 2C entries):
//               stable merge of the two sorted NN lists (deflate.cpp:62-66
//               restricted to the NN entries: same relative order), close-pole
//               walk (deflate.cpp:76-140), survivor compaction, secular roots
//               (secular.cpp:80-241; lane-per-root RootSM with a CTA queue, or
//               warp-per-root split arithmetic for split merges), Gu-Eisenstat
//               weights (secular.cpp:288-313) and boundary rows
//               (PAPER.md:1384-1396), all in shared memory.  Publishes per
//               merge: survivor prefix + rotated rows per NN entry, and per
//               root lambda_j, its rows and #{active <= lambda_j}.
//   k_sp_place  merge path over the level (tiles of 256 merged positions):
//               every deflated element goes to t + #{roots < D_t}, every root
//               to j + #{deflated <= lambda_j} --
//               written to the OTHER state slot (level_state.cuh).
//
// Arithmetic and every reduction order are those of the dense grid tier and
// the fused kernel (and of oracle/br_oracle.c): results are bit-identical.
// The dense pipeline stays as the fallback for levels with a merge of more
// than C non-negligible poles (Toeplitz, the top of glued Wilkinson).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "grid_common.cuh"
#include "internal.hpp"
#include "launch.cuh"
#include "level_state.cuh"
#include "numerics.cuh"

namespace brgpu {

constexpr int kFlagThreads = 256;
constexpr int kPlaceThreads = 256;
constexpr int kPlaceTile = 1024;  // merged positions per k_sp_place CTA
constexpr int kKeyWeight = 4;  // group key of merge m: spCs[m] + 4 m (bounds merges per group)

#ifndef BRGPU_SP_CAP
#define BRGPU_SP_CAP 2048
#endif
#ifndef BRGPU_SP_THREADS
#define BRGPU_SP_THREADS 512
#endif
constexpr int kSpCap = BRGPU_SP_CAP;          // NN entries per k_sp_solve CTA (2C)
constexpr int kSpC = kSpCap / 2;              // sparse iff every merge has NN <= C
constexpr int kSpThreads = BRGPU_SP_THREADS;

int sparse_cap() { return kSpC; }

// ---------------------------------------------------------------------------
// grid barrier of the persistent k_sp_flag (every CTA is resident: the grid is
// at most the co-resident CTA count, and a PDL dependent's CTAs are scheduled
// only after all of this grid's CTAs have started)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (*(volatile unsigned*)ctr < target) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
}

// Segmented (by merge) warp reduction; returns true in the lane that heads
// its merge's run within the warp, with the run's reduction in v.
template <typename T, typename Op>
__device__ __forceinline__ bool warp_seg_reduce(int m, T& v, Op op) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T v2 = __shfl_down_sync(0xffffffffu, v, o);
        const int m2 = __shfl_down_sync(0xffffffffu, m, o);
        if (lane + o < 32 && m2 == m) v = op(v, v2);
    }
    const int mp = __shfl_up_sync(0xffffffffu, m, 1);
    return m >= 0 && (lane == 0 || mp != m);
}

struct MaxU64 {
    __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a > b ? a : b; }
};
struct AddI {
    __device__ int operator()(int a, int b) const { return a + b; }
};

__device__ __forceinline__ double elem_z(const Work& w, const LevelDev& L, int m, int p) {
    return (p - L.mOff[m] < L.mNL[m]) ? w.bhi[p] : w.blo[p];  // |z| source (sign irrelevant)
}

// ---------------------------------------------------------------------------
// k_sp_flag
// ---------------------------------------------------------------------------
// CTA b owns nsc super-chunks of kFlagRows x 256 consecutive positions; thread
// tid owns positions base + r*256 + tid of each.  The merges a super-chunk
// touches (levels with merges >= 8 elements: at most kFlagMM) are staged in a
// shared table once per CTA -- per-element reads of the same merge words by
// every warp of the grid are an L2 hot spot at the top levels.  With one
// super-chunk (n up to the resident CTAs x 2048) table indices and |z| stay in
// registers across the three phases.
constexpr int kFlagRows = 8;
constexpr int kFlagChunk = kFlagRows * kFlagThreads;
constexpr int kSpMinMerge = 8;  // sparse levels need merges of >= 8 elements (table / segment bounds)
constexpr int kFlagMM = kFlagChunk / kSpMinMerge + 2;

struct FlagTab {
    int m0, cnt;
    int off[kFlagMM];
    int nl[kFlagMM];
    int end[kFlagMM];
    int cs[kFlagMM];
    double tol[kFlagMM];
};

// merges touching positions [base, lim): m0 = first merge ending after base
__device__ __forceinline__ void flag_table(const LevelDev& L, int base, int lim, FlagTab& T) {
    if (threadIdx.x == 0) {
        T.m0 = base < lim ? L.tileFirst[base / kTile] : L.M;
        T.cnt = 0;
    }
    __syncthreads();
    const int m0 = T.m0;
    for (int i = threadIdx.x; i < kFlagMM; i += kFlagThreads) {
        const int m = m0 + i;
        if (m < L.M) {
            const int off = L.mOff[m];
            if (off < lim) {
                T.off[i] = off;
                T.nl[i] = L.mNL[m];
                T.end[i] = off + L.mSize[m];
                atomicMax(&T.cnt, i + 1);  // valid entries form a prefix (merges ascend)
            }
        }
    }
    __syncthreads();
}

// table index of the merge holding position p, or -1
__device__ __forceinline__ int flag_lookup(const FlagTab& T, int p) {
    int lo = 0, hi = T.cnt;
    if (hi == 0) return -1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (T.off[mid] <= p) lo = mid; else hi = mid;
    }
    return (p >= T.off[lo] && p < T.end[lo]) ? lo : -1;
}

struct FlagRows {
    int i[kFlagRows];  // table index
    double z[kFlagRows];
    unsigned long long v[kFlagRows];
};

__device__ __forceinline__ void flag_rows_load(const Work& w, const FlagTab& T, int base, int c1, FlagRows& R) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int r = 0; r < kFlagRows; ++r) {
        const int p = base + r * kFlagThreads + tid;
        const int i = p < c1 ? flag_lookup(T, p) : -1;
        R.i[r] = i;
        R.z[r] = 0.0;
        R.v[r] = 0ULL;
        if (i >= 0) {
            R.z[r] = fabs((p - T.off[i] < T.nl[i]) ? w.bhi[p] : w.blo[p]);
            R.v[r] = (unsigned long long)__double_as_longlong(fmax(fabs(w.lam[p]), R.z[r]));
        }
    }
}

// per-merge tolerances of the table (after the max phase)
__device__ __forceinline__ void flag_table_tol(const LevelDev& L, double tol_scale, FlagTab& T) {
    for (int i = threadIdx.x; i < T.cnt; i += kFlagThreads)
        T.tol[i] = 8.0 * kU * __longlong_as_double((long long)__ldcg(&L.mTol[T.m0 + i])) * tol_scale;
    __syncthreads();
}

__global__ void __launch_bounds__(kFlagThreads) k_sp_flag(Work w0, LevelDev L, int n, double tol_scale,
                                                          int* __restrict__ blockCnt, int ngroups, int nsc) {
    pdl_entry();
    __shared__ unsigned long long s_maxA, s_maxB;
    __shared__ int s_cntA, s_cntB, s_mA, s_mB;
    __shared__ int s_red[kFlagThreads / 32];
    __shared__ int s_wt[kFlagRows][kFlagThreads / 32];
    __shared__ FlagTab T;
    const Work& w = w0;  // the children are in (lam, blo, bhi)
    const int G = (int)gridDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = nsc * kFlagChunk;  // the launcher sizes the grid: G * per >= n
    const int c0 = (int)min((long long)n, (long long)blockIdx.x * per), c1 = min(n, c0 + per);
    unsigned* bar = reinterpret_cast<unsigned*>(L.ctl + 2);

    // ---- phase 0: level words, per-merge accumulators, group table ---------
    if (blockIdx.x == 0 && tid == 0) L.ctl[1] = 0;
    for (int m = blockIdx.x * kFlagThreads + tid; m < L.M; m += G * kFlagThreads) {
        L.mTol[m] = 0ULL;
        L.spNN[m] = 0;
    }
    for (int g = blockIdx.x * kFlagThreads + tid; g <= ngroups; g += G * kFlagThreads) L.spGroup[g] = L.M;
    if (tid == 0) {
        s_maxA = 0ULL; s_maxB = 0ULL;
        s_cntA = 0; s_cntB = 0;
        s_mA = c0 < c1 ? find_merge(L, c0) : -1;      // merges shared with other CTAs:
        s_mB = c0 < c1 ? find_merge(L, c1 - 1) : -1;  // accumulated in shared memory first
    }
    flag_table(L, c0, min(c1, c0 + kFlagChunk), T);
    FlagRows R;
    flag_rows_load(w, T, c0, c1, R);
    // k_sp_place tile records (one warp per tile start; overlaps the barrier wait)
    {
        const int tiles = (n + kPlaceTile - 1) / kPlaceTile;
        for (int tt = blockIdx.x * (kFlagThreads / 32) + wid; tt <= tiles; tt += G * (kFlagThreads / 32)) {
            const int pe = tt * kPlaceTile;
            const int m = pe < n ? find_merge(L, pe) : -1;
            int sp = 0;
            if (m >= 0) {
                const int off = L.mOff[m];
                if (pe > off) {
                    const int nl = L.mNL[m], nr = L.mSize[m] - nl;
                    const double* la = w.lam + off;
                    sp = warp_merge_split(la, nl, la + nl, nr, pe - off);
                }
            }
            if (lane == 0) {
                L.spTileM[tt] = m;
                L.spTileSplit[tt] = sp;
            }
        }
    }
    grid_barrier(bar, (unsigned)G);
    const int mA = s_mA, mB = s_mB;

    // ---- phase A: max(|lambda|, |z|) per merge -----------------------------
    for (int sc = 0; sc < nsc; ++sc) {
        if (sc) {
            const int base = c0 + sc * kFlagChunk;
            __syncthreads();
            flag_table(L, base, min(c1, base + kFlagChunk), T);
            flag_rows_load(w, T, base, c1, R);
        }
#pragma unroll
        for (int r = 0; r < kFlagRows; ++r) {
            const int m = R.i[r] >= 0 ? T.m0 + R.i[r] : -1;
            unsigned long long v = R.v[r];
            if (warp_seg_reduce(m, v, MaxU64{})) {
                if (m == mA) atomicMax(&s_maxA, v);
                else if (m == mB) atomicMax(&s_maxB, v);
                else atomicMax(&L.mTol[m], v);  // merge inside this CTA's chunk
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (mA >= 0) atomicMax(&L.mTol[mA], s_maxA);
        if (mB >= 0 && mB != mA) atomicMax(&L.mTol[mB], s_maxB);
    }
    grid_barrier(bar, 2u * (unsigned)G);

    // ---- phase B: small-z flags, per-merge and per-CTA counts --------------
    int mine = 0;
    for (int sc = 0; sc < nsc; ++sc) {
        if (nsc > 1) {
            const int base = c0 + sc * kFlagChunk;
            __syncthreads();
            flag_table(L, base, min(c1, base + kFlagChunk), T);
            flag_rows_load(w, T, base, c1, R);
        }
        flag_table_tol(L, tol_scale, T);
#pragma unroll
        for (int r = 0; r < kFlagRows; ++r) {
            const int i = R.i[r];
            const int m = i >= 0 ? T.m0 + i : -1;
            const int f = i >= 0 && R.z[r] > T.tol[i];
            mine += f;
            int c = f;
            if (warp_seg_reduce(m, c, AddI{}) && c) {
                if (m == mA) atomicAdd(&s_cntA, c);
                else if (m == mB) atomicAdd(&s_cntB, c);
                else atomicAdd(&L.spNN[m], c);
            }
        }
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if (lane == 0) s_red[wid] = mine;
    __syncthreads();
    if (tid == 0) {
        int t = 0;
#pragma unroll
        for (int k = 0; k < kFlagThreads / 32; ++k) t += s_red[k];
        blockCnt[blockIdx.x] = t;
        if (mA >= 0 && s_cntA) atomicAdd(&L.spNN[mA], s_cntA);
        if (mB >= 0 && mB != mA && s_cntB) atomicAdd(&L.spNN[mB], s_cntB);
    }
    grid_barrier(bar, 3u * (unsigned)G);

    // ---- phase C: ordered compaction ----------------------------------------
    {
        int s = 0;
        for (int k = tid; k < (int)blockIdx.x; k += kFlagThreads) s += __ldcg(&blockCnt[k]);
        s = __reduce_add_sync(0xffffffffu, s);
        if (lane == 0) s_red[wid] = s;
    }
    __syncthreads();
    int run = 0;
#pragma unroll
    for (int k = 0; k < kFlagThreads / 32; ++k) run += s_red[k];
    const unsigned ltmask = (1u << lane) - 1u;
    const int span = L.spSpan;
    for (int sc = 0; sc < nsc; ++sc) {
        const int base = c0 + sc * kFlagChunk;
        if (nsc > 1) {
            __syncthreads();
            flag_table(L, base, min(c1, base + kFlagChunk), T);
            flag_rows_load(w, T, base, c1, R);
            flag_table_tol(L, tol_scale, T);
        }
        // per-merge NN counts of the table (final after the barrier)
        for (int i = tid; i < T.cnt; i += kFlagThreads) T.cs[i] = __ldcg(&L.spNN[T.m0 + i]);
        unsigned fbits = 0;
#pragma unroll
        for (int r = 0; r < kFlagRows; ++r) {
            const int i = R.i[r];
            const int f = i >= 0 && R.z[r] > T.tol[i];
            fbits |= (unsigned)f << r;
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (lane == 0) s_wt[r][wid] = __popc(bal);
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kFlagRows; ++r) {
            const int i = R.i[r];
            const int p = base + r * kFlagThreads + tid;
            const int f = (fbits >> r) & 1;
            int before = 0, all = 0;
#pragma unroll
            for (int k = 0; k < kFlagThreads / 32; ++k) {
                before += k < wid ? s_wt[r][k] : 0;
                all += s_wt[r][k];
            }
            const int c = run + before + __popc(__ballot_sync(0xffffffffu, f) & ltmask);
            run += all;
            if (p < c1) w0.nnPre[p] = c;  // exclusive NN prefix by position (k_sp_place's NN ranks)
            if (i < 0) continue;
            const int m = T.m0 + i;
            const int off = T.off[i], nl = T.nl[i];
            if (p == off) {
                L.spCs[m] = c;
                atomicMax(&L.ctl[1], T.cs[i]);
                // k_sp_solve groups: merge m belongs to group key(m) / span,
                // key(m) = spCs[m] + 4m; group g starts at its first merge
                const int gm = (c + kKeyWeight * m) / span;
                const int gp = m > 0 ? (c - __ldcg(&L.spNN[m - 1]) + kKeyWeight * (m - 1)) / span : -1;
                for (int g = gp + 1; g <= gm && g <= ngroups; ++g) L.spGroup[g] = m;
            }
            if (p == off + nl) L.spCsR[m] = c;
            if (f) {
                double z, r0, r1;
                if (p - off < nl) {
                    const double bh = w.bhi[p];
                    z = w.ew[off + nl - 1] < 0 ? -bh : bh;
                    r0 = w.blo[p];
                    r1 = 0.0;
                } else {
                    z = w.blo[p];
                    r0 = 0.0;
                    r1 = w.bhi[p];
                }
                w.dA[c] = w.lam[p];
                w.zA[c] = z;
                w.r0A[c] = r0;
                w.r1A[c] = r1;
                w.nnPos[c] = p;
            }
        }
    }
    if (blockIdx.x == G - 1 && tid == 0) {
        L.ctl[3] = run;  // level total NN (planning statistics)
        w0.nnPre[n] = run;
    }
}

// ---------------------------------------------------------------------------
// k_sp_solve
// ---------------------------------------------------------------------------
template <int CAP, int NT>
struct SpSmem {
    static constexpr int MM = CAP / (2 * kKeyWeight) + 2;  // merges per group (key weight 4, span C)
    double D[CAP];       // merged NN order: poles, z, rows
    double Z[CAP];       // (then: secular prefix snapshots; then d[origin] per root)
    double R0[CAP];
    double R1[CAP];
    double2 pairs[CAP];  // active (d, z^2); first: NN values (merge ranks), walk prefixes Q, S0
    double zA[CAP];      // active z / z-hat; walk prefix S1
    double r0A[CAP];
    double r1A[CAP];
    double tau[CAP];
    int org[CAP];
    int survPre[CAP + 1];
    unsigned char surv[CAP];
    int mo[MM + 1];  // local NN offsets (+ end)
    int mnL[MM];     // left-child NN entries
    int mg[MM];      // first position
    int ms[MM];      // size
    int mf[MM];      // flags
    int mcs[MM];     // compacted start
    int kS[MM + 1];  // active ranges
    double rho[MM];
    double tol[MM];
    int scan[NT / 32];
    int next, nextW, nextLast;
};

// One group of whole merges [mfirst, mend) of a sparse level.
template <int CAP, int NT>
__device__ __forceinline__ void sp_group(const Work& w, const LevelDev& L, const SolveParams& prm,
                                         int* __restrict__ traceOut, const int mfirst, const int mend,
                                         SpSmem<CAP, NT>& S) {
    const int cnt = mend - mfirst;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    const int cs0 = L.spCs[mfirst];

    // ---- metadata ------------------------------------------------------------
    for (int t = tid; t < cnt; t += NT) {
        const int m = mfirst + t;
        const int cs = L.spCs[m], nn = L.spNN[m];
        const int off = L.mOff[m], nl = L.mNL[m];
        S.mo[t] = cs - cs0;
        S.mnL[t] = L.spCsR[m] - cs;
        S.mg[t] = off;
        S.ms[t] = L.mSize[m];
        S.mf[t] = L.mFlags[m];
        S.mcs[t] = cs;
        S.rho[t] = fabs(w.ew[off + nl - 1]);
        S.tol[t] = 8.0 * kU * __longlong_as_double((long long)L.mTol[m]) * prm.tol_scale;
        if (t == cnt - 1) S.mo[cnt] = cs + nn - cs0;
    }
    if (tid == 0) {
        S.next = 0;
        S.nextW = 0;
        S.nextLast = 0;
    }
    __syncthreads();
    const int E = S.mo[cnt];

    // ---- stable merge of the two sorted NN lists of each merge ---------------
    double* val = reinterpret_cast<double*>(S.pairs);
    for (int e = tid; e < E; e += NT) val[e] = w.dA[cs0 + e];
    __syncthreads();
    for (int e = tid; e < E; e += NT) {
        const int t = upper_index(S.mo, cnt, e);
        const int base = S.mo[t], nL = S.mnL[t], nR = S.mo[t + 1] - base - nL;
        const int a = e - base;
        const double v = val[e];
        const int rank = a < nL ? a + count_less(val + base + nL, nR, v) : (a - nL) + count_leq(val + base, nL, v);
        const int k = base + rank;
        S.D[k] = v;
        S.Z[k] = w.zA[cs0 + e];
        S.R0[k] = w.r0A[cs0 + e];
        S.R1[k] = w.r1A[cs0 + e];
    }
    __syncthreads();

    // ---- close-pole deflation (fused.cu / k_segment_walk arithmetic) ---------
    {
        double* pQ = reinterpret_cast<double*>(S.pairs);
        double* pS0 = pQ + CAP;
        double* pS1 = S.zA;
        for (int q = tid; q < E; q += NT) {
            const int t = upper_index(S.mo, cnt, q);
            const int qs = S.mo[t], qe = S.mo[t + 1];
            const double tol = S.tol[t];
            if (q > qs && fabs(S.D[q] - S.D[q - 1]) <= tol) continue;  // not a head
            S.surv[q] = 1;
            int prev = q, nmem = 0;
            double dp = S.D[q];
            const double zs = S.Z[q];
            double Q = zs * zs, S0 = zs * S.R0[q], S1 = zs * S.R1[q];
            double dprev_nn = dp;
            for (int q2 = q + 1; q2 < qe; ++q2) {
                const double d2 = S.D[q2];
                if (fabs(d2 - dprev_nn) > tol) break;
                dprev_nn = d2;
                const double zq = S.Z[q2];
                if (fabs(d2 - dp) <= tol) {
                    pQ[q2] = Q;
                    pS0[q2] = S0;
                    pS1[q2] = S1;
                    Q = Q + zq * zq;
                    S0 = S0 + zq * S.R0[q2];
                    S1 = S1 + zq * S.R1[q2];
                    ++nmem;
                    S.surv[q2] = 0;
                } else {
                    if (nmem) {
                        const double R = sqrt(Q), iR = 1.0 / R;
                        S.Z[prev] = R; S.R0[prev] = S0 * iR; S.R1[prev] = S1 * iR;
                    }
                    S.surv[q2] = 1;
                    prev = q2; dp = d2; nmem = 0;
                    Q = zq * zq; S0 = zq * S.R0[q2]; S1 = zq * S.R1[q2];
                }
            }
            if (nmem) {
                const double R = sqrt(Q), iR = 1.0 / R;
                S.Z[prev] = R; S.R0[prev] = S0 * iR; S.R1[prev] = S1 * iR;
            }
        }
        __syncthreads();
        for (int q = tid; q < E; q += NT) {
            if (S.surv[q]) continue;
            double x0 = S.R0[q], x1 = S.R1[q];
            group_member(pQ[q], pS0[q], pS1[q], S.Z[q], x0, x1);
            S.R0[q] = x0;
            S.R1[q] = x1;
            S.Z[q] = 0.0;
        }
    }
    __syncthreads();

    // ---- survivor compaction; NN results for k_sp_place ----------------------
    const int T = cta_scan_flags<NT>(S.surv, E, S.survPre, S.scan);
    for (int q = tid; q < E; q += NT) {
        if (!S.surv[q]) continue;
        const int g = S.survPre[q];
        const double z = S.Z[q];
        S.pairs[g] = make_double2(S.D[q], z * z);
        S.zA[g] = z;
        S.r0A[g] = S.R0[q];
        S.r1A[g] = S.R1[q];
    }
    if (tid <= cnt) S.kS[tid] = S.survPre[S.mo[tid]];
    __syncthreads();
    for (int q = tid; q < E; q += NT) {
        const int t = upper_index(S.mo, cnt, q);
        w.survPre[cs0 + q] = S.survPre[q] - S.kS[t];
        w.survFlag[cs0 + q] = S.surv[q];
        w.r0A[cs0 + q] = S.R0[q];
        w.r1A[cs0 + q] = S.R1[q];
    }

    // ---- secular roots -------------------------------------------------------
    unsigned long long evals = 0, terms = 0;
    // split merges (size > 8192 or K > 1024): one warp per root
    for (;;) {
        int g = 0;
        if (lane == 0) g = atomicAdd(&S.nextW, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= T) break;
        const int t = upper_index(S.kS, cnt, g);
        const int ks = S.kS[t], K = S.kS[t + 1] - ks;
        if (!split_mode(S.ms[t], K)) continue;
        int o;
        double tu;
        root_warp(S.pairs + ks, S.zA + ks, K, g - ks, S.rho[t], w.exact != 0, prm.patched != 0, w.status, o, tu,
                  evals, terms);
        if (lane == 0) {
            S.org[g] = o;
            S.tau[g] = tu;
        }
    }
    if (lane) evals = terms = 0;  // the warp's counts live in lane 0
    // lane-per-root merges: per-lane RootSM, CTA queue (fused.cu)
    {
        double2* snap = reinterpret_cast<double2*>(S.Z) + tid;
        RootSM st;
        int g = -1, ks = 0;
        bool exhausted = false, lastDone = false;
        for (;;) {
            while (g < 0 && !exhausted) {  // last roots first (fused.cu), then interior roots
                int t, q;
                if (!lastDone) {
                    t = atomicAdd(&S.nextLast, 1);
                    if (t >= cnt) { lastDone = true; continue; }
                    if (S.kS[t + 1] == S.kS[t]) continue;
                    q = S.kS[t + 1] - 1;
                } else {
                    q = atomicAdd(&S.next, 1);
                    if (q >= T) { exhausted = true; break; }
                    t = upper_index(S.kS, cnt, q);
                    if (q == S.kS[t + 1] - 1) continue;
                }
                ks = S.kS[t];
                const int K = S.kS[t + 1] - ks;
                if (split_mode(S.ms[t], K)) continue;
                g = q;
                rs_begin(st, K, g - ks, S.rho[t], PolesPairs{S.pairs + ks}, S.zA[ks], Z2Pairs{S.pairs + ks});
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
                const SmemPairs P{S.pairs + ks};
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
                rs_consume(st, ev, PolesPairs{S.pairs + ks}, Z2Pairs{S.pairs + ks}, prm.patched != 0);
                if (st.phase == kRsDone || st.phase == kRsFail) {
                    if (st.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                    S.org[g] = st.org;
                    S.tau[g] = st.tau;
                    g = -1;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        evals += __shfl_xor_sync(0xffffffffu, evals, o);
        terms += __shfl_xor_sync(0xffffffffu, terms, o);
    }
    if (lane == 0 && evals) {
        atomicAdd(&w.counters[0], evals);
        atomicAdd(&w.counters[1], terms);
    }
    __syncthreads();
    double* sDorg = S.Z;  // d[origin] per root
    for (int g = tid; g < T; g += NT) {
        const int t = upper_index(S.kS, cnt, g);
        sDorg[g] = S.pairs[S.kS[t] + S.org[g]].x;
    }
    __syncthreads();

    // ---- Gu-Eisenstat refreshed weights (non-root merges, K > 1) --------------
    if (prm.zhat) {
        for (int g = tid; g < T; g += NT) {  // lane-per-pole merges: sequential product
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if ((S.mf[t] & kMergeRoot) || K == 1 || split_mode(S.ms[t], K)) continue;
            const double di = S.pairs[g].x;
            double prod = 1.0;
            if (!w.exact && zhat_guard(PolesPairs{S.pairs + ks}, K, i)) {
#pragma unroll 4
                for (int j = 0; j < K; ++j) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    const double dd = di - S.pairs[ks + j].x;
                    const double f = (j == i) ? del : del * rcp_nr(dd);
                    prod = prod * f;
                }
            } else {
                for (int j = 0; j < K; ++j) {
                    const double del = (di - S.pairs[ks + S.org[ks + j]].x) - S.tau[ks + j];
                    if (j == i) prod = prod * del;
                    else prod = prod * (del * __drcp_rn(di - S.pairs[ks + j].x));
                }
            }
            const double mag = sqrt(fmax(0.0, -prod));
            S.zA[g] = S.zA[g] >= 0.0 ? mag : -mag;
        }
        for (int g = wid; g < T; g += NW) {  // split merges: one warp per pole
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if ((S.mf[t] & kMergeRoot) || K == 1 || !split_mode(S.ms[t], K)) continue;
            const double di = S.pairs[g].x;
            double prod = 1.0;
            if (!w.exact && zhat_guard(PolesPairs{S.pairs + ks}, K, i)) {
                for (int j = lane; j < K; j += 32) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    prod = prod * (j == i ? del : del * rcp_nr(di - S.pairs[ks + j].x));
                }
            } else {
                for (int j = lane; j < K; j += 32) {
                    const double del = (di - S.pairs[ks + S.org[ks + j]].x) - S.tau[ks + j];
                    if (j == i) prod = prod * del;
                    else prod = prod * (del * __drcp_rn(di - S.pairs[ks + j].x));
                }
            }
            const double W = bfly_mul(prod);
            if (lane == 0) {
                const double mag = sqrt(fmax(0.0, -W));
                S.zA[g] = S.zA[g] >= 0.0 ? mag : -mag;
            }
        }
        __syncthreads();
    }

    // ---- roots: lambda_j, #{active <= lambda_j}, boundary rows ----------------
    for (int g = tid; g < T; g += NT) {  // lane-per-root merges (and every root's lambda)
        const int t = upper_index(S.kS, cnt, g);
        const int ks = S.kS[t], K = S.kS[t + 1] - ks, j = g - ks;
        const double dorg = sDorg[g], tau = S.tau[g];
        const double lam = dorg + tau;
        int lo = 0, hi = K;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (!(lam < S.pairs[ks + mid].x)) lo = mid + 1; else hi = mid;
        }
        const int oj = S.mcs[t] + j;
        w.tau[oj] = lam;
        w.org[oj] = lo;
        if ((S.mf[t] & kMergeRoot) || split_mode(S.ms[t], K)) continue;
        double nn = 0.0, s0 = 0.0, s1 = 0.0;
        if (!w.exact && eval_guard(SmemPairs{S.pairs + ks}, K, j, dorg, tau)) {
#pragma unroll 4
            for (int i = 0; i < K; ++i) {
                const double y = S.zA[ks + i] * rcp_nr((S.pairs[ks + i].x - dorg) - tau);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
        } else {
            bool zero = false;
            for (int i = 0; i < K; ++i) {
                const double del = (S.pairs[ks + i].x - dorg) - tau;
                zero |= (del == 0.0);
                const double y = S.zA[ks + i] * __drcp_rn(del);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
            if (zero) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
        }
        const double inv = 1.0 / sqrt(nn);
        w.z2A[oj] = s0 * inv;
        w.zA[oj] = s1 * inv;
    }
    for (int g = wid; g < T; g += NW) {  // split merges: one warp per root
        const int t = upper_index(S.kS, cnt, g);
        const int ks = S.kS[t], K = S.kS[t + 1] - ks, j = g - ks;
        if ((S.mf[t] & kMergeRoot) || !split_mode(S.ms[t], K)) continue;
        const double dorg = sDorg[g], tau = S.tau[g];
        double nn = 0.0, s0 = 0.0, s1 = 0.0;
        if (!w.exact && eval_guard(SmemPairs{S.pairs + ks}, K, j, dorg, tau)) {
            for (int i = lane; i < K; i += 32) {
                const double y = S.zA[ks + i] * rcp_nr((S.pairs[ks + i].x - dorg) - tau);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
        } else {
            bool zero = false;
            for (int i = lane; i < K; i += 32) {
                const double del = (S.pairs[ks + i].x - dorg) - tau;
                zero |= (del == 0.0);
                const double y = S.zA[ks + i] * __drcp_rn(del);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(S.r0A[ks + i], y, s0);
                s1 = __fma_rn(S.r1A[ks + i], y, s1);
            }
            if (__any_sync(0xffffffffu, zero) && lane == 0) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
        }
        const double NNs = bfly_add(nn), S0 = bfly_add(s0), S1 = bfly_add(s1);
        if (lane == 0) {
            const double inv = 1.0 / sqrt(NNs);
            const int oj = S.mcs[t] + j;
            w.z2A[oj] = S0 * inv;
            w.zA[oj] = S1 * inv;
        }
    }
    for (int t = tid; t < cnt; t += NT) {
        const int K = S.kS[t + 1] - S.kS[t];
        L.spK[mfirst + t] = K;
        if (traceOut) {
            traceOut[2 * (mfirst + t)] = S.mo[t + 1] - S.mo[t];
            traceOut[2 * (mfirst + t) + 1] = K;
        }
    }
}

// Persistent: one CTA per SM walks the level's groups (group g = merges with
// key in [g*span, (g+1)*span)); the host picks span from the previous solve's
// deflation profile so that the group count fills the SMs evenly.
template <int CAP, int NT>
__global__ void __launch_bounds__(NT, 1) k_sp_solve(Work w, LevelDev L, SolveParams prm, int* __restrict__ traceOut,
                                                  int ngroups) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char sp_raw[];
    SpSmem<CAP, NT>& S = *reinterpret_cast<SpSmem<CAP, NT>*>(sp_raw);
    if (!level_sparse(L)) return;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int mfirst = L.spGroup[g];
        if (mfirst >= L.M) break;
        const int mend = min(L.spGroup[g + 1], L.M);
        if (mfirst >= mend) continue;
        const int E = L.spCs[mend - 1] + L.spNN[mend - 1] - L.spCs[mfirst];
        if (E > CAP || mend - mfirst > SpSmem<CAP, NT>::MM) {  // cannot happen when the level is sparse
#ifdef BRGPU_SP_DEBUG
            if (threadIdx.x == 0)
                printf("k_sp_solve: group %d merges [%d,%d) E %d M %d span %d cap %d maxNN %d\n", g, mfirst, mend, E,
                       L.M, L.spSpan, L.spCap, L.ctl[1]);
#endif
            if (threadIdx.x == 0) set_status(w.status, BRGPU_ERR_MALFORMED_COMPACT_ROOT);
            continue;
        }
        sp_group<CAP, NT>(w, L, prm, traceOut, mfirst, mend, S);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// k_sp_place
// ---------------------------------------------------------------------------
// A CTA owns kPlaceTile consecutive merged positions; thread t owns positions
// 4t .. 4t+3 of the tile.  The merges overlapping the tile are its segments
// (levels whose merges have >= 8 elements: at most kPlaceSegs).  Per segment,
// the merge's root values and its NN survivor prefixes/flags are staged in
// shared memory once, so every per-element search is a shared-memory search.
constexpr int kPlacePer = kPlaceTile / kPlaceThreads;
constexpr int kPlaceSegs = kPlaceTile / 8 + 2;
constexpr int kPlaceStage = 1024;  // staged roots (and NN entries) per tile; larger: global fallback

struct PlaceSmem {
    double v[kPlaceTile];   // inputs in segment input order, then merged D
    double b0[kPlaceTile];  // ... blo, then merged R0
    double b1[kPlaceTile];  // ... bhi, then merged R1
    double za[kPlaceTile];  // merged |z|
    int ex[kPlaceTile];     // exclusive NN prefix over the tile (position order)
    double roots[kPlaceStage];
    int pre[kPlaceStage];
    unsigned char sflag[kPlaceStage];
    int nseg, split0, split1, stRoots, stNN, sparse;
    // per segment
    int soff[kPlaceSegs], snl[kPlaceSegs], ssize[kPlaceSegs], scs[kPlaceSegs], snn[kPlaceSegs], sK[kPlaceSegs];
    int sh[kPlaceSegs], slen[kPlaceSegs], si0[kPlaceSegs], sla[kPlaceSegs], sqb[kPlaceSegs];
    int sr[kPlaceSegs + 1], sn[kPlaceSegs + 1], sjlo[kPlaceSegs], sjn[kPlaceSegs + 1];
    double svb[kPlaceSegs];
    double stol[kPlaceSegs];
    int smf[kPlaceSegs];
    int sroot[kPlaceSegs];
};

// first index in [lo, hi) of an ascending int array with a[i] >= x, or hi
// (warp-cooperative, 32-ary; every lane returns the same value)
__device__ __forceinline__ int warp_lower_bound(const int* __restrict__ a, int lo, int hi, int x) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) >> 5;
        const int c = lo + lane * step;
        const int k = __popc(__ballot_sync(0xffffffffu, c < hi && a[c] < x));  // monotone prefix
        if (k == 0) return lo;
        const int nlo = lo + (k - 1) * step + 1;  // a[lo + (k-1) step] < x
        hi = min(hi, lo + k * step);               // a[lo + k step] >= x (or out of range)
        lo = nlo;
    }
    const bool lt = lo + lane < hi && a[lo + lane] < x;
    return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

__global__ void __launch_bounds__(kPlaceThreads) k_sp_place(Work w0, LevelDev L, int n, double tol_scale) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char pl_raw[];
    PlaceSmem& S = *reinterpret_cast<PlaceSmem*>(pl_raw);
    const int t = threadIdx.x;
    if (t == 0) {  // one thread reads the level and tile words (grid-wide hot lines)
        S.sparse = level_sparse(L);
        S.split0 = L.spTileSplit[blockIdx.x];
        S.split1 = L.spTileSplit[blockIdx.x + 1];
    }
    __syncthreads();
    if (!S.sparse) return;
    // children in (lam, blo, bhi); parents to (D, R0, R1), copied back by k_sp_home
    const Work& wi = w0;
    struct { double *lam, *blo, *bhi; } wo = {w0.D, w0.R0, w0.R1};
    const int p0 = blockIdx.x * kPlaceTile;
    const int pend = min(n, p0 + kPlaceTile);

    // ---- segment table: the merges touching this tile (m0 = first ending after p0)
    const int sm0 = L.tileFirst[p0 / kTile];
    if (t == 0) S.nseg = 0;
    __syncthreads();
    for (int s = t; s < kPlaceSegs; s += kPlaceThreads) {
        const int m = sm0 + s;
        if (m >= L.M) continue;
        const int off = L.mOff[m];
        if (off >= pend) continue;
        atomicMax(&S.nseg, s + 1);  // merges ascend: the valid entries form a prefix
        const int nl = L.mNL[m], size = L.mSize[m];
        const int q0 = max(p0, off), q1 = min(pend, off + size);
        const int i0 = q0 == off ? 0 : S.split0;
        const int i1 = q1 == off + size ? nl : S.split1;
        S.soff[s] = off; S.snl[s] = nl; S.ssize[s] = size;
        S.scs[s] = L.spCs[m]; S.snn[s] = L.spNN[m]; S.sK[s] = L.spK[m];
        S.sh[s] = q0 - p0; S.slen[s] = q1 - q0; S.si0[s] = i0; S.sla[s] = i1 - i0;
        S.sqb[s] = 0;
        S.stol[s] = 8.0 * kU * __longlong_as_double((long long)L.mTol[m]) * tol_scale;
        S.smf[s] = L.mFlags[m];
        // v_b: the merged element right after the segment (first of the next tile)
        double vb = 0.0;
        if (q1 < off + size) {
            const int ib = S.split1, jb = (q1 - off) - ib;
            const double* lc = wi.lam + off;
            vb = (ib < nl && (jb >= size - nl || !(lc[nl + jb] < lc[ib]))) ? lc[ib] : lc[nl + jb];
        }
        S.svb[s] = vb;
    }
    __syncthreads();
    const int nseg = S.nseg;
    // segment of each of this thread's positions (-1: not merged at this level --
    // the state moves to the other slot unchanged)
    int mk[kPlacePer];
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        const int p = p0 + kPlacePer * t + k;
        int sg = -1;
        if (p < pend && nseg > 0) {
            int lo = 0, hi = nseg;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (S.soff[mid] <= p) lo = mid; else hi = mid;
            }
            if (p >= S.soff[lo] && p < S.soff[lo] + S.ssize[lo]) sg = lo;
        }
        mk[k] = sg >= 0 ? sm0 + sg : -1;
        if (p < pend && sg < 0) {
            wo.lam[p] = wi.lam[p];
            wo.blo[p] = wi.blo[p];
            wo.bhi[p] = wi.bhi[p];
        }
    }
    if (nseg == 0) return;  // uniform
    // NN entries of the first segment's merge before the tile (warp 0; the only
    // segment that can start inside its merge), staging offsets (thread 32)
    if (t == 0) {
        const int off = S.soff[0];
        if (S.sh[0] == 0 && p0 > off) {  // NN entries before the tile: by position prefix (k_sp_flag)
            const int nl = S.snl[0], i0 = S.si0[0], j0 = (p0 - off) - i0;
            S.sqb[0] = (w0.nnPre[off + i0] - S.scs[0]) + (w0.nnPre[off + nl + j0] - L.spCsR[sm0]);
        }
    } else if (t == 32) {
        int r = 0, q = 0;
        for (int s = 0; s < nseg; ++s) {
            S.sr[s] = r; S.sn[s] = q;
            r += S.sK[s]; q += S.snn[s];
        }
        S.sr[nseg] = r; S.sn[nseg] = q;
        S.stRoots = r <= kPlaceStage;
        S.stNN = q <= kPlaceStage;
    }
    __syncthreads();
    // stage root values and NN survivor prefixes / flags
    const bool stR = S.stRoots, stN = S.stNN;
    if (stR || stN) {
        for (int s = 0; s < nseg; ++s) {
            const int cs = S.scs[s];
            if (stR) for (int j = t; j < S.sK[s]; j += kPlaceThreads) S.roots[S.sr[s] + j] = w0.tau[cs + j];
            if (stN)
                for (int q = t; q < S.snn[s]; q += kPlaceThreads) {
                    S.pre[S.sn[s] + q] = w0.survPre[cs + q];
                    S.sflag[S.sn[s] + q] = w0.survFlag[cs + q];
                }
        }
    }

    // ---- merge path inside each segment: inputs, then merged order ----------------
    double v[kPlacePer], r0[kPlacePer], r1[kPlacePer], za[kPlacePer];
    int o[kPlacePer];
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        const int u = kPlacePer * t + k;  // tile-local input slot = merged position - p0
        o[k] = -1;
        if (mk[k] < 0) continue;
        const int s = mk[k] - sm0;
        const int off = S.soff[s], nl = S.snl[s], h = S.sh[s], la = S.sla[s], i0 = S.si0[s];
        const int j0 = (h + p0 - off) - i0;
        const int uu = u - h;
        const int src = uu < la ? off + i0 + uu : off + nl + j0 + (uu - la);
        S.v[u] = wi.lam[src];
        S.b0[u] = wi.blo[src];
        S.b1[u] = wi.bhi[src];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        const int u = kPlacePer * t + k;
        if (mk[k] < 0) continue;
        const int s = mk[k] - sm0;
        const int off = S.soff[s], h = S.sh[s], la = S.sla[s], i0 = S.si0[s], len = S.slen[s];
        const int j0 = (h + p0 - off) - i0;
        const int uu = u - h;
        v[k] = S.v[u];
        int sp;
        if (uu < la) {
            sp = (i0 + uu) + j0 + count_less(S.v + h + la, len - la, v[k]);
            za[k] = fabs(S.b1[u]);
            r0[k] = S.b0[u];
            r1[k] = 0.0;
        } else {
            sp = (j0 + uu - la) + i0 + count_leq(S.v + h, la, v[k]);
            za[k] = fabs(S.b0[u]);
            r0[k] = 0.0;
            r1[k] = S.b1[u];
        }
        o[k] = off + sp - p0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        if (o[k] < 0) continue;
        S.v[o[k]] = v[k];
        S.b0[o[k]] = r0[k];
        S.b1[o[k]] = r1[k];
        S.za[o[k]] = za[k];
    }
    __syncthreads();

    // ---- NN flags in merged order, exclusive prefix over the tile -------------------
    int f[kPlacePer];
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        const int u = kPlacePer * t + k;
        f[k] = 0;
        if (mk[k] >= 0) {
            f[k] = S.za[u] > S.stol[mk[k] - sm0];
        }
        cnt += f[k];
    }
    int tot;
    int run = block_exclusive_scan<kPlaceThreads>(cnt, tot);
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        S.ex[kPlacePer * t + k] = run;
        run += f[k];
    }
    // roots owned by each segment: insertion index #{merged <= lambda_j} in (a, b]
    // (or 0 when the segment starts its merge)
    for (int s = t; s < nseg; s += kPlaceThreads) {
        const int K = S.sK[s], off = S.soff[s], h = S.sh[s];
        const double* rv = stR ? S.roots + S.sr[s] : w0.tau + S.scs[s];
        const int a = h + p0 - off, b = a + S.slen[s];
        int jlo = 0, jhi = K;
        if (a > 0) jlo = count_less(rv, K, S.v[h]);
        if (b < S.ssize[s]) jhi = count_less(rv, K, S.svb[s]);
        S.sjlo[s] = jlo;
        S.sroot[s] = max(0, jhi - jlo);
    }
    __syncthreads();
    if (t == 0) {
        int r = 0;
        for (int s = 0; s < nseg; ++s) { S.sjn[s] = r; r += S.sroot[s]; }
        S.sjn[nseg] = r;
    }

    // ---- deflated elements: t + #{roots < v} ------------------------------------------
#pragma unroll
    for (int k = 0; k < kPlacePer; ++k) {
        const int u = kPlacePer * t + k;
        if (mk[k] < 0) continue;
        const int m = mk[k], s = m - sm0;
        const int off = S.soff[s], cs = S.scs[s], nn = S.snn[s], K = S.sK[s], h = S.sh[s];
        const int q = S.sqb[s] + (S.ex[u] - S.ex[h]);
        const bool member = f[k] && (stN ? S.sflag[S.sn[s] + q] : w0.survFlag[cs + q]) == 0;
        if (f[k] && !member) continue;  // survivor: its slot goes to a root
        const int survBefore = q < nn ? (stN ? S.pre[S.sn[s] + q] : w0.survPre[cs + q]) : K;
        const int tt = (u + p0 - off) - survBefore;
        const double vv = S.v[u];
        const int lo = count_less(stR ? S.roots + S.sr[s] : w0.tau + cs, K, vv);
        const int dst = off + tt + lo;
        wo.lam[dst] = vv;
        if (!(S.smf[s] & kMergeRoot)) {
            wo.blo[dst] = member ? w0.r0A[cs + q] : S.b0[u];
            wo.bhi[dst] = member ? w0.r1A[cs + q] : S.b1[u];
        }
    }
    __syncthreads();
    // ---- roots: j + #{deflated <= lambda_j} ----------------------------------------------
    const int nroots = S.sjn[nseg];
    for (int r = t; r < nroots; r += kPlaceThreads) {
        const int s = upper_index(S.sjn, nseg, r);
        const int m = sm0 + s;
        const int j = S.sjlo[s] + (r - S.sjn[s]);
        const int off = S.soff[s], cs = S.scs[s], h = S.sh[s];
        const double lam = stR ? S.roots[S.sr[s] + j] : w0.tau[cs + j];
        const int ins = (h + p0 - off) + count_leq(S.v + h, S.slen[s], lam);
        const int dst = off + j + ins - w0.org[cs + j];
        wo.lam[dst] = lam;
        if (!(S.smf[s] & kMergeRoot)) {
            wo.blo[dst] = w0.z2A[cs + j];
            wo.bhi[dst] = w0.zA[cs + j];
        }
    }
}

// Parents back to (lam, blo, bhi): every level boundary keeps the state there,
// so the dense and fused kernels never need to know which path a level took.
__global__ void __launch_bounds__(256) k_sp_home(Work w, LevelDev L, int n) {
    pdl_entry();
    __shared__ int s_sp;
    if (threadIdx.x == 0) s_sp = level_sparse(L);
    __syncthreads();
    if (!s_sp) return;
    const int n2 = n >> 1;  // 16-byte vectors
    const double2* __restrict__ D = reinterpret_cast<const double2*>(w.D);
    const double2* __restrict__ R0 = reinterpret_cast<const double2*>(w.R0);
    const double2* __restrict__ R1 = reinterpret_cast<const double2*>(w.R1);
    double2* lam = reinterpret_cast<double2*>(w.lam);
    double2* blo = reinterpret_cast<double2*>(w.blo);
    double2* bhi = reinterpret_cast<double2*>(w.bhi);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x) {
        lam[i] = D[i];
        blo[i] = R0[i];
        bhi[i] = R1[i];
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        w.lam[n - 1] = w.D[n - 1];
        w.blo[n - 1] = w.R0[n - 1];
        w.bhi[n - 1] = w.R1[n - 1];
    }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static int g_flag_grid_per_sm = 0;

void init_sparse_attributes() {
    cudaFuncSetAttribute(k_sp_solve<kSpCap, kSpThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(SpSmem<kSpCap, kSpThreads>));
    int nb = 0;
    cudaFuncSetAttribute(k_sp_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PlaceSmem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sp_flag, kFlagThreads, 0);
    g_flag_grid_per_sm = nb < 1 ? 1 : nb;
}

int sparse_groups_max(int n, int M, int span) { return (n + kKeyWeight * M) / span + 2; }
int sparse_min_merge() { return kSpMinMerge; }
// k_sp_flag's grid: all CTAs co-resident (grid barriers), each owning nsc
// super-chunks of kFlagChunk positions
int sparse_flag_nsc(int n, int sms) {
    const long long res = (long long)sms * (g_flag_grid_per_sm ? g_flag_grid_per_sm : 1);
    const long long chunks = ((long long)n + kFlagChunk - 1) / kFlagChunk;
    return (int)std::max<long long>(1, (chunks + res - 1) / res);
}
int sparse_flag_grid(int n, int sms) {
    const int nsc = sparse_flag_nsc(n, sms);
    const long long per = (long long)nsc * kFlagChunk;
    return (int)std::max<long long>(1, ((long long)n + per - 1) / per);
}

void launch_level_sparse(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm,
                         int* blockCnt, int* traceOut, int* launches, Prof* prof) {
    const int ng = sparse_groups_max(n, L.M, L.spSpan);
    launch_pdl(k_sp_flag, sparse_flag_grid(n, prm.sms), kFlagThreads, 0, s, w, L, n, prm.tol_scale, blockCnt, ng,
               sparse_flag_nsc(n, prm.sms));
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_SPFLAG);
    launch_pdl(k_sp_solve<kSpCap, kSpThreads>, std::min(ng, prm.sms), kSpThreads, sizeof(SpSmem<kSpCap, kSpThreads>),
               s, w, L, prm, traceOut, ng);
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_SPSOLVE);
    launch_pdl(k_sp_place, (n + kPlaceTile - 1) / kPlaceTile, kPlaceThreads, sizeof(PlaceSmem), s, w, L, n,
               prm.tol_scale);
    launch_pdl(k_sp_home, std::max(1, std::min((n / 2 + 255) / 256, prm.sms * 8)), 256, 0, s, w, L, n);
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_SPPLACE);
    *launches += 4;
}

static_assert(sizeof(SpSmem<kSpCap, kSpThreads>) <= 227 * 1024, "k_sp_solve shared memory");

}  // namespace brgpu
