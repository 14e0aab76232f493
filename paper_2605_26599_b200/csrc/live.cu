// live.cu -- live-list tier for the top levels of a large single-block solve.
//
// Above the bottom levels of a deflation-heavy input (random n = 2^20: every
// merge from size 256 up keeps K ~ 100 active poles of its 256 .. 2^20
// elements), almost every element is a pole whose two boundary-row entries are
// below the deflation tolerance of every later merge: it deflates by small z
// (deflate.cpp:31-41) at every level up to the root and its eigenvalue never
// changes.  The dense grid tier still moves every element through ~15 launches
// per level.  This tier keeps, per node, only the LIVE elements (a boundary-row
// entry above theta = tol/2 of the merge that produced them), in the node's
// order, at the start of the node's position range; the eigenvalues of the
// other (dead) elements go to a pool, and three maxima per node summarise them
// (|lambda|, |first row|, |last row|):
//  * a merge's tolerance 8u max(|D|, |z|) (deflate.cpp:55-60) is order-free:
//    the live elements' terms plus the children's dead maxima (|lambda| of
//    both, the left child's last row, the right child's first row) -- the dense
//    value exactly;
//  * the dead elements are small-z deflations iff the left child's dead
//    last-row maximum and the right child's dead first-row maximum are <= tol.
//    Checked per merge; when it fails (or a merge's live lists exceed shared
//    memory, or a bucket of the final sort overflows) the fallback word is set
//    and api.cpp redoes the solve on the dense tiers;
//  * the non-negligible elements, their merged order (the dense merge restricted
//    to the live elements is the stable merge of the live lists), the close-pole
//    walk, the secular problem, refreshed weights and boundary rows are then
//    those of the dense tiers -- same operations in the same order, so every
//    root, weight and row is bit-identical -- and the parent's live list is the
//    restriction of the parent's order (deflated first on ties);
//  * merges larger than kSplitMinSize use the warp tier's 32-way split
//    arithmetic (root_warp, lane-strided products / sums + xor butterflies), one
//    merge per 1024-thread CTA so that every root / pole gets its own warp.
// At the root the live list joins the pool (n values), which a bucket sort
// (value buckets, rank sort per bucket in shared memory) puts in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"
#include "grid_common.cuh"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace brgpu {

constexpr int kLiveMax = 512;      // live elements of one merge (both children)
#ifndef BRGPU_LIVE_THREADS
#define BRGPU_LIVE_THREADS 256
#endif
constexpr int kLiveThreads = BRGPU_LIVE_THREADS;
constexpr int kLiveInitThreads = 256;
constexpr int kBucketCap = 4096;   // elements of one final-sort bucket (shared memory)
constexpr int kBucketThreads = 256;
constexpr int kLiveCtasPerSm = 3;
#ifndef BRGPU_LIVE_SPLIT_THREADS
#define BRGPU_LIVE_SPLIT_THREADS 1024
#endif
constexpr int kLiveSplitThreads = BRGPU_LIVE_SPLIT_THREADS;  // split-rule levels: a warp per root  // resident live CTAs per SM (launch bounds, shared memory)
#ifndef BRGPU_LIVE_GROUP_MAX
#define BRGPU_LIVE_GROUP_MAX 4
#endif
constexpr int kLiveGroupMax = BRGPU_LIVE_GROUP_MAX;

constexpr int kLiveGroup = 4;      // merges of one batch

struct LiveSmem {
    double D[kLiveMax];
    double Z[kLiveMax];
    double R0[kLiveMax];
    double R1[kLiveMax];
    double in[3 * kLiveMax];   // inputs (lam, blo, bhi); then active (d, z^2) pairs + z / z-hat
    double r0A[kLiveMax];
    double r1A[kLiveMax];
    double tau[kLiveMax];
    double oLam[kLiveMax];     // parent outputs at their live-order positions
    double oR0[kLiveMax];
    double oR1[kLiveMax];
    int org[kLiveMax];
    int nnPre[kLiveMax + 1];
    int nnPos[kLiveMax];
    int survPre[kLiveMax + 1];
    unsigned char flag[kLiveMax];
    unsigned char surv[kLiveMax];
    int scan[32];              // warp totals of a CTA scan (<= 1024 threads)
    // per merge of the batch
    int mo[kLiveGroup + 1];    // local offsets (+ end)
    int me[kLiveGroup];        // live inputs
    int ml[kLiveGroup];        // ... of the left child
    int mb[kLiveGroup];        // first position of the merge
    int mblk[kLiveGroup];      // its block (pool)
    int mnlF[kLiveGroup];      // left child's size
    int kS[kLiveGroup + 1];    // active ranges
    int ne[kLiveGroup + 1];    // merges with K > 0 before t (root queue order)
    int outc[kLiveGroup];
    double rho[kLiveGroup];
    double tol[kLiveGroup];
    double dead[6 * kLiveGroup];  // children's dead maxima: L (lam, blo, bhi), R (lam, blo, bhi)
    unsigned long long tolb[kLiveGroup];
    unsigned long long dmx[3 * kLiveGroup];  // demoted maxima bits: |lambda|, |first row|, |last row|
    bool neg[kLiveGroup];
    int next, bail, root, batch;
};

__device__ __forceinline__ unsigned long long dbits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ double bitsd(unsigned long long b) { return __longlong_as_double((long long)b); }

__device__ __forceinline__ void live_fail(const LiveDev& V) { atomicExch(&V.ctl[1], 1); }

// block of position p (one block: 0)
__device__ __forceinline__ int live_block(const LiveDev& V, int p) {
    int lo = 0, hi = V.nblk;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (V.bstart[mid] <= p) lo = mid; else hi = mid;
    }
    return lo;
}

// warp-aggregated append of v to block blk's pool (blk uniform per warp)
__device__ __forceinline__ void pool_push(const LiveDev& V, int blk, bool push, double v) {
    const unsigned m = __ballot_sync(0xffffffffu, push);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = V.bstart[blk] + atomicAdd(&V.bctr[blk], __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (push) V.pool[base + __popc(m & ((1u << lane) - 1u))] = v;
}

template <int BLOCK>
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = red[0];
#pragma unroll
    for (int q = 1; q < BLOCK / 32; ++q) r = fmax(r, red[q]);
    return r;
}

// ---------------------------------------------------------------------------
// Entry of the tier: every frontier node (a child of a live merge computed by
// the dense tiers) keeps its live elements, in order, at the start of its range.
// theta = half the smallest tolerance a later merge can have on the node's own
// |lambda| scale; the per-merge check makes the choice a performance matter only.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLiveInitThreads) k_live_init(Work w, LiveDev V, const int2* __restrict__ front,
                                                                double tol_scale) {
    pdl_entry();
    __shared__ double s_red[kLiveInitThreads / 32];
    // the final sort's bucket counts are zeroed here (the dense levels used the array)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * V.nb + 2; i += gridDim.x * blockDim.x)
        V.bcount[i] = 0;
    const int2 f = front[blockIdx.x];
    const int off = f.x, size = f.y;
    const int blk = live_block(V, off);
    double mx = 0.0;
    for (int i = threadIdx.x; i < size; i += kLiveInitThreads) mx = fmax(mx, fabs(w.lam[off + i]));
    mx = block_max<kLiveInitThreads>(mx, s_red);
    const double theta = 0.5 * (8.0 * kU * mx * tol_scale);
    double dl = 0.0, d0 = 0.0, d1 = 0.0;
    int out = 0;
    for (int c0 = 0; c0 < size; c0 += kLiveInitThreads) {
        const int i = c0 + threadIdx.x;
        const bool valid = i < size;
        double v = 0.0, b0 = 0.0, b1 = 0.0;
        if (valid) {
            v = w.lam[off + i];
            b0 = w.blo[off + i];
            b1 = w.bhi[off + i];
        }
        const bool live = valid && fmax(fabs(b0), fabs(b1)) > theta;
        const bool dead = valid && !live;
        pool_push(V, blk, dead, v);
        if (dead) {
            dl = fmax(dl, fabs(v));
            d0 = fmax(d0, fabs(b0));
            d1 = fmax(d1, fabs(b1));
        }
        int tot;
        const int ex = block_exclusive_scan<kLiveInitThreads>(live ? 1 : 0, tot);  // all loads of the chunk are done
        if (live) {
            const int p = off + out + ex;
            w.lam[p] = v;
            w.blo[p] = b0;
            w.bhi[p] = b1;
        }
        out += tot;
    }
    dl = block_max<kLiveInitThreads>(dl, s_red);
    d0 = block_max<kLiveInitThreads>(d0, s_red);
    d1 = block_max<kLiveInitThreads>(d1, s_red);
    if (threadIdx.x == 0) {
        V.cnt[off] = out;
        V.dLam[off] = dl;
        V.dBlo[off] = d0;
        V.dBhi[off] = d1;
    }
}

// ---------------------------------------------------------------------------
// A batch of consecutive merges of a live level per CTA pass (live inputs of
// the batch <= kLiveMax): the fused tier's shared-memory pipeline (fused.cu
// holds the commented dense original) on the children's live lists.  A CTA owns
// up to G merges and cuts them into batches greedily, so one CTA's 256 lanes
// hold the roots of several merges of K ~ 100.
// ---------------------------------------------------------------------------
//
// CLU: one merge per thread-block CLUSTER (k_live_cluster; split arithmetic):
// every CTA of the cluster runs the deflation on its own copy of the inputs
// (same operations, same results), then the CTAs share the roots, refreshed
// weights and boundary rows by index (CTA r of C takes root queue entries
// r, r + C, ...; warp slices for the weights and rows) and publish each result
// into every CTA's shared memory over DSMEM, a cluster barrier per phase; CTA 0
// writes the parent.  Every root / weight / row is computed by the same code on
// the same shared-memory operands, so the results are bitwise those of one CTA.
// LPR < 32: the split arithmetic on groups of LPR lanes (LaneGroup, numerics.cuh;
// bitwise the warp-per-root form), 32 / LPR roots / poles per warp.
#ifdef BRGPU_LIVE_PROF
// CTAs whose phase cycles are recorded: cluster rank 0 of the split-rule levels
// and one-CTA few-merge levels (or, with -DBRGPU_LIVE_PROF_ONLY=G, only the
// levels launched on G CTAs)
__device__ __forceinline__ bool live_prof_cta(bool clu, int crank) {
#ifdef BRGPU_LIVE_PROF_ONLY
    return !clu && gridDim.x == BRGPU_LIVE_PROF_ONLY;
#else
    return clu ? crank == 0 : gridDim.x <= 64;
#endif
}
#endif

template <bool SPLIT, int NT, bool CLU = false, int LPR = 32>
__device__ __forceinline__ void live_group(const Work& w, const LevelDev& L, const LiveDev& V, const int m0,
                                           const int cnt, const SolveParams& prm, int* __restrict__ traceOut,
                                           LiveSmem& S) {
    static_assert(SPLIT || NT <= kLiveMax / 2, "lane mode: one double2 snapshot slot per thread in S.Z");
    static_assert(!CLU || SPLIT, "cluster mode runs the split arithmetic");
    static_assert(LPR == 32 || SPLIT, "lane groups run the split arithmetic");
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    // cluster rank / size (1 CTA: 0 / 1)
    int crank = 0, csize = 1;
    if constexpr (CLU) {
        crank = (int)cg::this_cluster().block_rank();
        csize = (int)cg::this_cluster().num_blocks();
    }
#ifdef BRGPU_LIVE_PROF
    // phase cycles of the few-merge (latency-bound) levels, summed over CTAs in
    // counters[4..7]: deflation / secular / refreshed weights / rows + output
    long long ph_t = clock64();
#define LIVE_MARK(k)                                                                          \
    do {                                                                                      \
        __syncthreads();                                                                      \
        if (tid == 0 && live_prof_cta(CLU, crank)) {                                          \
            const long long t_ = clock64();                                                   \
            atomicAdd(&w.counters[4 + (k)], (unsigned long long)(t_ - ph_t));                 \
            ph_t = t_;                                                                        \
        }                                                                                     \
    } while (0)
#else
#define LIVE_MARK(k) do {} while (0)
#endif
    // ---- batch metadata ---------------------------------------------------------
    if (tid < cnt) {
        const int m = m0 + tid;
        const int base = L.mOff[m], nlF = L.mNL[m];
        const int cl = V.cnt[base], cr = V.cnt[base + nlF];
        S.mb[tid] = base;
        S.mblk[tid] = live_block(V, base);
        S.mnlF[tid] = nlF;
        S.ml[tid] = cl;
        S.me[tid] = cl + cr;
        const double em = w.ew[base + nlF - 1];
        S.rho[tid] = fabs(em);
        S.neg[tid] = em < 0;
        double* dd = S.dead + 6 * tid;
        dd[0] = V.dLam[base];
        dd[1] = V.dBlo[base];
        dd[2] = V.dBhi[base];
        dd[3] = V.dLam[base + nlF];
        dd[4] = V.dBlo[base + nlF];
        dd[5] = V.dBhi[base + nlF];
        // tolerance terms of the dead elements: |lambda| of both children, |z| =
        // the left child's last row, the right child's first row
        S.tolb[tid] = dbits(fmax(fmax(dd[0], dd[3]), fmax(dd[2], dd[4])));
        S.dmx[3 * tid] = S.dmx[3 * tid + 1] = S.dmx[3 * tid + 2] = 0ULL;
    }
    if (tid == 0) {
        S.next = 0;
        S.root = (L.mFlags[m0] & kMergeRoot) != 0;
    }
    __syncthreads();
    if (tid == 0) {
        int o = 0;
        for (int t = 0; t < cnt; ++t) { S.mo[t] = o; o += S.me[t]; }
        S.mo[cnt] = o;
        S.bail = (!CLU && *(volatile int*)&V.ctl[1] != 0) || o > kLiveMax;
        if (o > kLiveMax) live_fail(V);
    }
    __syncthreads();
    if (S.bail) return;
    const int E = S.mo[cnt];
    const bool isRoot = S.root;
    double* lamIn = S.in;
    double* bloIn = S.in + kLiveMax;
    double* bhiIn = S.in + 2 * kLiveMax;
    for (int i = tid; i < E; i += NT) {
        const int t = upper_index(S.mo, cnt, i);
        const int li = i - S.mo[t], nl = S.ml[t];
        const int src = li < nl ? S.mb[t] + li : S.mb[t] + S.mnlF[t] + (li - nl);
        lamIn[i] = w.lam[src];
        bloIn[i] = w.blo[src];
        bhiIn[i] = w.bhi[src];
    }
    __syncthreads();

    // ---- tolerance: max(|D|, |z|) over the live and dead elements ------------
    for (int b0 = 0; b0 < E; b0 += NT) {
        const int i = b0 + tid;
        int t = -1;
        double v = 0.0;
        if (i < E) {
            t = upper_index(S.mo, cnt, i);
            v = fmax(fabs(lamIn[i]), fabs(i - S.mo[t] < S.ml[t] ? bhiIn[i] : bloIn[i]));
        }
        const int t0 = __shfl_sync(0xffffffffu, t, 0);
        if (__all_sync(0xffffffffu, t == t0)) {  // one merge per warp: reduce, one shared atomic
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0 && t0 >= 0 && v > 0.0) atomicMax(&S.tolb[t0], dbits(v));
        } else if (t >= 0 && v > 0.0) {
            atomicMax(&S.tolb[t], dbits(v));
        }
    }
    __syncthreads();
    if (tid < cnt) {
        const double tol = 8.0 * kU * bitsd(S.tolb[tid]) * prm.tol_scale;
        S.tol[tid] = tol;
        const double* dd = S.dead + 6 * tid;
        if (!(dd[2] <= tol && dd[4] <= tol)) {  // a dead element would be non-negligible
            S.bail = 1;
            live_fail(V);
        }
    }
    __syncthreads();
    if (S.bail) return;

    // ---- stable merge of each merge's two sorted live lists + z --------------
    for (int i = tid; i < E; i += NT) {
        const int t = upper_index(S.mo, cnt, i);
        const int off = S.mo[t], nl = S.ml[t], Et = S.me[t];
        const int li = i - off;
        const double v = lamIn[i];
        int sp;
        double z, r0, r1;
        if (li < nl) {
            sp = li + count_less(lamIn + off + nl, Et - nl, v);
            const double b = bhiIn[i];
            z = S.neg[t] ? -b : b;
            r0 = bloIn[i];
            r1 = 0.0;
        } else {
            sp = (li - nl) + count_leq(lamIn + off, nl, v);
            z = bloIn[i];
            r0 = 0.0;
            r1 = bhiIn[i];
        }
        S.D[off + sp] = v;
        S.Z[off + sp] = z;
        S.R0[off + sp] = r0;
        S.R1[off + sp] = r1;
    }
    __syncthreads();

    // ---- small-z flags + NN compaction ---------------------------------------
    for (int i = tid; i < E; i += NT) S.flag[i] = fabs(S.Z[i]) > S.tol[upper_index(S.mo, cnt, i)];
    __syncthreads();
    const int NN = cta_scan_flags<NT>(S.flag, E, S.nnPre, S.scan);
    for (int i = tid; i < E; i += NT)
        if (S.flag[i]) S.nnPos[S.nnPre[i]] = i;
    __syncthreads();

    // ---- close-pole deflation (k_segment_walk / fused.cu arithmetic) ---------
    {
        double* pQ = lamIn;
        double* pS0 = bloIn;
        double* pS1 = bhiIn;
        for (int q = tid; q < NN; q += NT) {
            const int k = S.nnPos[q];
            const int t = upper_index(S.mo, cnt, k);
            const int qs = S.nnPre[S.mo[t]], qe = S.nnPre[S.mo[t + 1]];
            const double tol = S.tol[t];
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
        for (int q = tid; q < NN; q += NT) {
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

    // ---- survivor compaction: active (d, z^2) pairs, z, rows ------------------
    const int T = cta_scan_flags<NT>(S.surv, NN, S.survPre, S.scan);
    double2* pairs = reinterpret_cast<double2*>(S.in);  // aliases lam/blo inputs (dead)
    double* zA = S.in + 2 * kLiveMax;                    // aliases the bhi input (dead)
    for (int q = tid; q < NN; q += NT) {
        if (!S.surv[q]) continue;
        const int g = S.survPre[q], k = S.nnPos[q];
        const double z = S.Z[k];
        pairs[g] = make_double2(S.D[k], z * z);
        zA[g] = z;
        S.r0A[g] = S.R0[k];
        S.r1A[g] = S.R1[k];
    }
    if (tid <= cnt) S.kS[tid] = S.survPre[S.nnPre[S.mo[tid]]];
    __syncthreads();
    // root queue: every merge's last root first, then the interior roots in order
    // (the order never changes a result); ne[t] = merges with K > 0 before t
    if (tid <= cnt) {
        int c = 0;
        for (int u = 0; u < tid; ++u) c += S.kS[u + 1] > S.kS[u];
        S.ne[tid] = c;
    }
    __syncthreads();
    int* qorder = S.nnPos;  // dead after the compaction
    for (int g = tid; g < T; g += NT) {
        const int t = upper_index(S.kS, cnt, g);
        qorder[g == S.kS[t + 1] - 1 ? S.ne[t] : S.ne[cnt] + g - S.ne[t]] = g;
    }
    __syncthreads();
    LIVE_MARK(0);

    // ---- secular roots ---------------------------------------------------------
    if (SPLIT && LPR < 32) {  // a lane group per root, group queue
        const LaneGroup<LPR> G;
        RootSM st;
        int g = -1, ks = 0;
        bool exhausted = false;
        unsigned long long ev = 0, tm = 0;
        for (;;) {
            while (g < 0 && !exhausted) {
                int q = 0;
                if (G.gl == 0) q = atomicAdd(&S.next, 1) * csize + crank;
                q = __shfl_sync(G.mask, q, G.base);
                if (q >= T) { exhausted = true; break; }
                g = qorder[q];
                const int t = upper_index(S.kS, cnt, g);
                ks = S.kS[t];
                const int K = S.kS[t + 1] - ks, j = g - ks;
                const double2* P = pairs + ks;
                const double zsq = (j == K - 1 && K > 1) ? grp_zsq(G, P, K) : 0.0;
                rs_begin_zsq(st, K, j, S.rho[t], PolesPairs{P}, zA[ks], zsq, P[K - 1].y);
                if (st.phase == kRsDone) {
                    if constexpr (CLU) {
                        for (int rr = G.gl; rr < csize; rr += LPR) {
                            *cg::this_cluster().map_shared_rank(&S.org[g], rr) = st.org;
                            *cg::this_cluster().map_shared_rank(&S.tau[g], rr) = st.tau;
                        }
                    } else if (G.gl == 0) {
                        S.org[g] = st.org;
                        S.tau[g] = st.tau;
                    }
                    g = -1;
                }
            }
            if (!__any_sync(0xffffffffu, g >= 0)) break;
            if (g >= 0) {
                const double2* P = pairs + ks;
                const Ev e = grp_eval(G, P, st, w.exact != 0);
                if (G.gl == 0) {
                    ++ev;
                    tm += (unsigned long long)st.K;
                }
                rs_consume(st, e, PolesPairs{P}, Z2Pairs{P}, prm.patched != 0);
                if (st.phase == kRsDone || st.phase == kRsFail) {
                    if (st.phase == kRsFail && G.gl == 0) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                    if constexpr (CLU) {
                        for (int rr = G.gl; rr < csize; rr += LPR) {
                            *cg::this_cluster().map_shared_rank(&S.org[g], rr) = st.org;
                            *cg::this_cluster().map_shared_rank(&S.tau[g], rr) = st.tau;
                        }
                    } else if (G.gl == 0) {
                        S.org[g] = st.org;
                        S.tau[g] = st.tau;
                    }
                    g = -1;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ev += __shfl_xor_sync(0xffffffffu, ev, o);
            tm += __shfl_xor_sync(0xffffffffu, tm, o);
        }
        if (lane == 0 && ev) {
            atomicAdd(&w.counters[8], ev);
            atomicAdd(&w.counters[9], tm);
        }
    } else if (SPLIT) {  // warp per root, 32-way split arithmetic (k_secular_warp), warp queue
        unsigned long long ev = 0, tm = 0;
        for (;;) {
            int q = 0;
            if (lane == 0) q = atomicAdd(&S.next, 1) * csize + crank;
            q = __shfl_sync(0xffffffffu, q, 0);
            if (q >= T) break;
            const int g = qorder[q];
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks;
            int o;
            double tu;
            root_warp(pairs + ks, zA + ks, K, g - ks, S.rho[t], w.exact != 0, prm.patched != 0, w.status, o, tu,
                      ev, tm);
            if constexpr (CLU) {
                if (lane < csize) {  // lane r publishes into CTA r's shared memory
                    *cg::this_cluster().map_shared_rank(&S.org[g], lane) = o;
                    *cg::this_cluster().map_shared_rank(&S.tau[g], lane) = tu;
                }
            } else if (lane == 0) {
                S.org[g] = o;
                S.tau[g] = tu;
            }
        }
        if (lane == 0 && ev) {  // every lane counted its warp's evaluations: lane 0 reports
            atomicAdd(&w.counters[8], ev);
            atomicAdd(&w.counters[9], tm);
        }
    } else {  // lane per root, CTA queue
        double2* snap = reinterpret_cast<double2*>(S.Z) + tid;  // S.Z is dead after the compaction
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
        if (lane == 0 && evals) {  // live-tier work counters (api.cpp kCounters)
            atomicAdd(&w.counters[8], evals);
            atomicAdd(&w.counters[9], terms);
        }
    }
    if constexpr (CLU) cg::this_cluster().sync();
    else __syncthreads();

    double* sDorg = S.Z;  // d[origin] per root (S.Z is dead after the compaction)
    for (int g = tid; g < T; g += NT) sDorg[g] = pairs[S.kS[upper_index(S.kS, cnt, g)] + S.org[g]].x;
    __syncthreads();
    LIVE_MARK(1);

    // ---- Gu-Eisenstat refreshed weights (non-root merges, K > 1) -------------
    if (prm.zhat && !isRoot && SPLIT && LPR < 32) {  // a lane group per pole
        const LaneGroup<LPR> G;
        constexpr int GPW = 32 / LPR;  // groups per warp
        for (int g = (crank * (NT / 32) + wid) * GPW + lane / LPR; g < T; g += csize * (NT / LPR)) {
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if (K == 1) continue;  // a lone pole keeps its z (the checker refreshes only K > 1)
            const double W = grp_zhat_prod(G, pairs + ks, sDorg + ks, S.tau + ks, K, i, w.exact != 0);
            const double mag = sqrt(fmax(0.0, -W));
            const double zh = zA[g] >= 0.0 ? mag : -mag;
            __syncwarp(G.mask);
            if constexpr (CLU) {
                for (int rr = G.gl; rr < csize; rr += LPR) *cg::this_cluster().map_shared_rank(&zA[g], rr) = zh;
            } else if (G.gl == 0) {
                zA[g] = zh;
            }
        }
        if constexpr (CLU) cg::this_cluster().sync();
        else __syncthreads();
    } else if (prm.zhat && !isRoot && SPLIT) {  // warp per pole: lane-strided products + butterfly (k_zhat_warp)
        for (int g = wid + crank * (NT / 32); g < T; g += csize * (NT / 32)) {
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if (K == 1) continue;  // a lone pole keeps its z (the checker refreshes only K > 1)
            const double di = pairs[g].x;
            double prod = 1.0;
            if (!w.exact && zhat_guard(PolesPairs{pairs + ks}, K, i)) {
                for (int j = lane; j < K; j += 32) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    prod = prod * (j == i ? del : del * rcp_nr(di - pairs[ks + j].x));
                }
            } else {
                for (int j = lane; j < K; j += 32) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    if (j == i) prod = prod * del;
                    else prod = prod * (del * __drcp_rn(di - pairs[ks + j].x));
                }
            }
            const double W = bfly_mul(prod);
            const double mag = sqrt(fmax(0.0, -W));
            const double zh = zA[g] >= 0.0 ? mag : -mag;
            __syncwarp();
            if constexpr (CLU) {
                if (lane < csize) *cg::this_cluster().map_shared_rank(&zA[g], lane) = zh;
            } else if (lane == 0) {
                zA[g] = zh;
            }
        }
        if constexpr (CLU) cg::this_cluster().sync();
        else __syncthreads();
    } else if (prm.zhat && !isRoot) {
        for (int g = tid; g < T; g += NT) {
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, i = g - ks;
            if (K == 1) continue;  // a lone pole keeps its z (the checker refreshes only K > 1)
            const double di = pairs[g].x;
            double prod = 1.0;
            if (!w.exact && zhat_guard(PolesPairs{pairs + ks}, K, i)) {
#pragma unroll 4
                for (int j = 0; j < K; ++j) {
                    const double del = (di - sDorg[ks + j]) - S.tau[ks + j];
                    const double dd = di - pairs[ks + j].x;
                    const double f = (j == i) ? del : del * rcp_nr(dd);
                    prod = prod * f;
                }
            } else {
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
    LIVE_MARK(2);

    // ---- roots: position in the parent's live order + boundary rows ----------
    if (SPLIT) {  // warp per root: lane-strided sums + butterflies (k_rows_warp)
        // (cluster: CTA r's warp slice; every result goes to CTA 0's shared memory)
        double* oLam = S.oLam;
        double* oR0 = S.oR0;
        double* oR1 = S.oR1;
        if constexpr (CLU) {
            oLam = cg::this_cluster().map_shared_rank(S.oLam, 0);
            oR0 = cg::this_cluster().map_shared_rank(S.oR0, 0);
            oR1 = cg::this_cluster().map_shared_rank(S.oR1, 0);
        }
        const LaneGroup<LPR> G;
        for (int g = (crank * (NT / 32) + wid) * (32 / LPR) + lane / LPR; g < T; g += csize * (NT / LPR)) {
            const int t = upper_index(S.kS, cnt, g);
            const int ks = S.kS[t], K = S.kS[t + 1] - ks, j = g - ks;
            const int off = S.mo[t];
            const double dorg = sDorg[g], tau = S.tau[g];
            const double lam = dorg + tau;
            int lo = 0, hi = K;  // #{dA <= lam}
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (!(lam < pairs[ks + mid].x)) lo = mid + 1; else hi = mid;
            }
            const int p = off + j + count_leq(S.D + off, S.me[t], lam) - lo;
            if (G.gl == 0) oLam[p] = lam;
            if (isRoot) continue;
            if constexpr (LPR < 32) {
                double NNs, S0, S1;
                if (!grp_rows(G, pairs + ks, zA + ks, S.r0A + ks, S.r1A + ks, K, j, dorg, tau, w.exact != 0, NNs, S0,
                              S1) && G.gl == 0)
                    set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
                if (G.gl == 0) {
                    const double inv = 1.0 / sqrt(NNs);
                    oR0[p] = S0 * inv;
                    oR1[p] = S1 * inv;
                }
                continue;
            }
            double nn = 0.0, s0 = 0.0, s1 = 0.0;
            if (!w.exact && eval_guard(SmemPairs{pairs + ks}, K, j, dorg, tau)) {
                for (int i = lane; i < K; i += 32) {
                    const double y = zA[ks + i] * rcp_nr((pairs[ks + i].x - dorg) - tau);
                    nn = __fma_rn(y, y, nn);
                    s0 = __fma_rn(S.r0A[ks + i], y, s0);
                    s1 = __fma_rn(S.r1A[ks + i], y, s1);
                }
            } else {
                bool zero = false;
                for (int i = lane; i < K; i += 32) {
                    const double del = (pairs[ks + i].x - dorg) - tau;
                    zero |= (del == 0.0);
                    const double y = zA[ks + i] * __drcp_rn(del);
                    nn = __fma_rn(y, y, nn);
                    s0 = __fma_rn(S.r0A[ks + i], y, s0);
                    s1 = __fma_rn(S.r1A[ks + i], y, s1);
                }
                if (__any_sync(0xffffffffu, zero) && lane == 0) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
            }
            const double NNs = bfly_add(nn), S0 = bfly_add(s0), S1 = bfly_add(s1);
            if (lane == 0) {
                const double inv = 1.0 / sqrt(NNs);
                oR0[p] = S0 * inv;
                oR1[p] = S1 * inv;
            }
        }
    } else
    for (int g = tid; g < T; g += NT) {
        const int t = upper_index(S.kS, cnt, g);
        const int ks = S.kS[t], K = S.kS[t + 1] - ks, j = g - ks;
        const int off = S.mo[t];
        const double dorg = sDorg[g], tau = S.tau[g];
        const double lam = dorg + tau;
        int lo = 0, hi = K;  // #{dA <= lam}
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (!(lam < pairs[ks + mid].x)) lo = mid + 1; else hi = mid;
        }
        const int p = off + j + count_leq(S.D + off, S.me[t], lam) - lo;
        S.oLam[p] = lam;
        if (isRoot) continue;
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
        S.oR0[p] = s0 * inv;
        S.oR1[p] = s1 * inv;
    }
    // deflated live elements: t + #{roots < D}
    for (int k = tid; k < (crank == 0 ? E : 0); k += NT) {
        const int q = S.nnPre[k];
        if (S.flag[k] && S.surv[q]) continue;  // survivor: its column became a root
        const int t = upper_index(S.mo, cnt, k);
        const int off = S.mo[t], ks = S.kS[t], K = S.kS[t + 1] - ks;
        const int tt = (k - off) - (S.survPre[q] - ks);
        const double v = S.D[k];
        int lo = 0, hi = K;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const double lj = sDorg[ks + mid] + S.tau[ks + mid];
            if (lj < v) lo = mid + 1; else hi = mid;
        }
        S.oLam[off + tt + lo] = v;
        S.oR0[off + tt + lo] = S.R0[k];
        S.oR1[off + tt + lo] = S.R1[k];
    }
    if constexpr (CLU) {
        cg::this_cluster().sync();  // every output is in CTA 0's shared memory; no DSMEM access after this
        if (crank != 0) return;
    } else {
        __syncthreads();
    }

    // ---- parents' live lists: demote outputs with both rows <= tol / 2 --------
    if (isRoot) {  // the roots' eigenvalues join their blocks' pools for the final sort
        for (int t = 0; t < cnt; ++t)
            for (int c0 = 0; c0 < S.me[t]; c0 += NT) {
                const int i = c0 + tid;
                pool_push(V, S.mblk[t], i < S.me[t], i < S.me[t] ? S.oLam[S.mo[t] + i] : 0.0);
            }
    } else {
        for (int t = 0; t < cnt; ++t) {
            const int off = S.mo[t], Et = S.me[t], base = S.mb[t];
            const double theta = 0.5 * S.tol[t];
            int out = 0;
            double dl = 0.0, d0 = 0.0, d1 = 0.0;
            for (int c0 = 0; c0 < Et; c0 += NT) {
                const int i = c0 + tid;
                const bool valid = i < Et;
                double v = 0.0, b0 = 0.0, b1 = 0.0;
                if (valid) { v = S.oLam[off + i]; b0 = S.oR0[off + i]; b1 = S.oR1[off + i]; }
                const bool live = valid && fmax(fabs(b0), fabs(b1)) > theta;
                const bool dead = valid && !live;
                pool_push(V, S.mblk[t], dead, v);
                if (dead) {
                    dl = fmax(dl, fabs(v));
                    d0 = fmax(d0, fabs(b0));
                    d1 = fmax(d1, fabs(b1));
                }
                int tot;
                const int ex = block_exclusive_scan<NT>(live ? 1 : 0, tot);
                if (live) {
                    const int p = base + out + ex;
                    w.lam[p] = v;
                    w.blo[p] = b0;
                    w.bhi[p] = b1;
                }
                out += tot;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                dl = fmax(dl, __shfl_xor_sync(0xffffffffu, dl, o));
                d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
                d1 = fmax(d1, __shfl_xor_sync(0xffffffffu, d1, o));
            }
            if (lane == 0) {
                if (dl > 0.0) atomicMax(&S.dmx[3 * t], dbits(dl));
                if (d0 > 0.0) atomicMax(&S.dmx[3 * t + 1], dbits(d0));
                if (d1 > 0.0) atomicMax(&S.dmx[3 * t + 2], dbits(d1));
            }
            if (tid == 0) S.outc[t] = out;
        }
        __syncthreads();
        if (tid < cnt) {
            // parent rows of the children's dead elements: left (first row, 0), right (0, last row)
            const int base = S.mb[tid];
            const double* dd = S.dead + 6 * tid;
            V.cnt[base] = S.outc[tid];
            V.dLam[base] = fmax(fmax(dd[0], dd[3]), bitsd(S.dmx[3 * tid]));
            V.dBlo[base] = fmax(dd[1], bitsd(S.dmx[3 * tid + 1]));
            V.dBhi[base] = fmax(dd[5], bitsd(S.dmx[3 * tid + 2]));
        }
    }
    LIVE_MARK(3);
#undef LIVE_MARK
    if (traceOut && tid < cnt) {
        traceOut[2 * (m0 + tid)] = S.nnPre[S.mo[tid + 1]] - S.nnPre[S.mo[tid]];
        traceOut[2 * (m0 + tid) + 1] = S.kS[tid + 1] - S.kS[tid];
    }
}

// Split-rule levels: NT threads per cluster CTA, LPR lanes per root / pole / row
// (LaneGroup; 16 measured best against 8, 32 and 4 at C5).
#ifndef BRGPU_CLUSTER_THREADS
#define BRGPU_CLUSTER_THREADS 512
#endif
#ifndef BRGPU_CLUSTER_LPR
#define BRGPU_CLUSTER_LPR 16
#endif
constexpr int kClThreads = BRGPU_CLUSTER_THREADS;
constexpr int kClLpr = BRGPU_CLUSTER_LPR;
#ifndef BRGPU_LIVE_M3_THREADS
#define BRGPU_LIVE_M3_THREADS 256
#endif
constexpr int kLiveM3Threads = BRGPU_LIVE_M3_THREADS;  // many-merge split levels (MODE 3)

// A CTA owns merges [blockIdx.x * G, +G) and processes them in batches of
// consecutive merges whose live inputs fit kLiveMax.  MODE 0: lane arithmetic
// (256 threads), 1: split arithmetic, every merge > kSplitMinSize (one merge per
// 1024-thread CTA: a warp per root / pole), 2: per merge (one merge per CTA),
// 3: split arithmetic on lane groups (many-merge split-rule levels, G merges per CTA).
template <int MODE, int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 3 : 1)
k_live_level(Work w, LevelDev L, LiveDev V, SolveParams prm, int* __restrict__ traceOut, int G) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char live_raw[];
    LiveSmem& S = *reinterpret_cast<LiveSmem*>(live_raw);
    const int mEnd = min(L.M, (blockIdx.x + 1) * G);
    for (int m = blockIdx.x * G; m < mEnd;) {
        if (threadIdx.x == 0) {
            int c = 0, sum = 0;
            while (m + c < mEnd && c < kLiveGroup) {
                const int base = L.mOff[m + c];
                const int e = V.cnt[base] + V.cnt[base + L.mNL[m + c]];
                if (c > 0 && sum + e > kLiveMax) break;
                sum += e;
                ++c;
            }
            S.batch = c;
        }
        __syncthreads();
        const int c = S.batch;
        if constexpr (MODE == 2) {
            if (L.mSize[m] > kSplitMinSize) live_group<true, NT>(w, L, V, m, c, prm, traceOut, S);
            else live_group<false, NT>(w, L, V, m, c, prm, traceOut, S);
        } else if constexpr (MODE == 3) {
            live_group<true, NT, false, kClLpr>(w, L, V, m, c, prm, traceOut, S);
        } else {
            live_group<MODE == 1, NT>(w, L, V, m, c, prm, traceOut, S);
        }
        __syncthreads();
        m += c;
    }
}

// The few-merge top levels as one launch: merges start when their children are
// done instead of at level boundaries, so the critical path is the slowest chain
// of merges rather than the sum of each level's slowest merge (one merge per
// CTA, split arithmetic; the children of merge m of level l are merges 2m and
// 2m + 1 of level l - 1 -- api.cpp checks the run is that complete binary
// tree and that every CTA of the run is co-resident).
__global__ void __launch_bounds__(kLiveSplitThreads, 1) k_live_top(Work w, LiveRun R, LiveDev V, SolveParams prm) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char live_raw[];
    LiveSmem& S = *reinterpret_cast<LiveSmem*>(live_raw);
    const int b = blockIdx.x;
    const int l = upper_index(R.first, R.nlev, b);
    const int m = b - R.first[l];
    if (l > 0 && threadIdx.x == 0) {
        const volatile int* c = R.done + R.first[l - 1] + 2 * m;
        while (c[0] == 0 || c[1] == 0) __nanosleep(200);
        __threadfence();
    }
    __syncthreads();
    live_group<true, kLiveSplitThreads>(w, R.L[l], V, m, 1, prm, R.trace[l], S);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(R.done + b, 1);
    }
}

// A few-merge split-rule level with one merge per thread-block cluster of C CTAs
// on C SMs (cluster size chosen per launch): a merge's ~100-200 roots then run
// at ~one root per warp instead of ~5 per warp on one SM, whose FP64 pipe the
// split arithmetic (bracket / model replicated on 32 lanes) saturates.
template <int NT, int LPR>
__global__ void __launch_bounds__(NT, 1) k_live_cluster(Work w, LevelDev L, LiveDev V, SolveParams prm,
                                                        int* __restrict__ traceOut) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char live_raw[];
    LiveSmem& S = *reinterpret_cast<LiveSmem*>(live_raw);
    cg::this_cluster().sync();  // every CTA of the cluster runs before any DSMEM store
    const int m = (int)(blockIdx.x / cg::this_cluster().num_blocks());
    live_group<true, NT, true, LPR>(w, L, V, m, 1, prm, traceOut, S);
}

// Lane-mode live levels as one dataflow launch: persistent CTAs take work items
// (G consecutive merges of one level, the per-level launch's CTA share) by
// ticket, in level order; an item waits until its merges' children (level l - 1
// merges 2m, 2m + 1 -- api.cpp checks the run is that complete binary tree) have
// set their done words, so each merge starts when its own inputs are ready and
// the levels' root tails overlap instead of adding up.  Tickets hand out items
// children-first, so every awaited item is held by a running CTA.
__global__ void __launch_bounds__(kLiveThreads, kLiveCtasPerSm) k_live_flow(Work w, LiveRun R, LiveDev V,
                                                                            SolveParams prm) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char live_raw[];
    LiveSmem& S = *reinterpret_cast<LiveSmem*>(live_raw);
    __shared__ int s_item;
    const int tid = threadIdx.x;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(R.ticket, 1);
        __syncthreads();
        const int it = s_item;
        if (it >= R.nitems) return;
        const int4 I = R.items[it];
        const int l = I.x, m0 = I.y, cnt = I.z;
        if (l > 0) {
            if (tid < 2 * cnt) {
                const volatile int* f = R.done + R.first[l - 1] + 2 * m0 + tid;
                while (*f == 0) __nanosleep(128);
            }
            __threadfence();
        }
        __syncthreads();
        for (int m = m0; m < m0 + cnt;) {  // batches of the item's merges (k_live_level, MODE 0)
            if (tid == 0) {
                int c = 0, sum = 0;
                while (m + c < m0 + cnt && c < kLiveGroup) {
                    const int base = R.L[l].mOff[m + c];
                    const int e = V.cnt[base] + V.cnt[base + R.L[l].mNL[m + c]];
                    if (c > 0 && sum + e > kLiveMax) break;
                    sum += e;
                    ++c;
                }
                S.batch = c;
            }
            __syncthreads();
            const int c = S.batch;
            live_group<false, kLiveThreads>(w, R.L[l], V, m, c, prm, R.trace[l], S);
            __syncthreads();
            m += c;
        }
        __threadfence();
        __syncthreads();
        if (tid < cnt) atomicExch(R.done + R.first[l] + m0 + tid, 1);
    }
}

// ---------------------------------------------------------------------------
// Final order: bucket sort of the pool (n values).  Buckets split the value
// range uniformly (a monotone bucket function, so concatenated buckets are in
// order); each bucket is rank-sorted in shared memory (ties by pool index:
// equal doubles are interchangeable).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long okey(double v) {
    const unsigned long long b = dbits(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double okey_val(unsigned long long k) {
    return bitsd((k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k);
}
struct Buckets {
    double vmin, scale;
    int nb;
    __device__ __forceinline__ int operator()(double x) const {
        if (!(scale > 0.0)) return 0;
        const double t = (x - vmin) * scale;
        return t >= (double)(nb - 1) ? nb - 1 : (int)t;
    }
};
__device__ __forceinline__ Buckets buckets_of(const LiveDev& V) {
    Buckets B;
    B.nb = V.nb;
    B.vmin = okey_val(~V.keys[0]);
    const double vmax = okey_val(V.keys[1]);
    B.scale = vmax > B.vmin ? (double)V.nb / (vmax - B.vmin) : 0.0;
    if (!(B.scale < 1e300)) B.scale = 0.0;  // (vmax - vmin) underflow: one bucket
    return B;
}

__global__ void k_live_bounds(LiveDev V, int n) {
    pdl_entry();
    if (V.ctl[1]) return;
    unsigned long long lo = 0ULL, hi = 0ULL;  // lo holds ~min
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = okey(V.pool[i]);
        lo = ~k > lo ? ~k : lo;
        hi = k > hi ? k : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a > lo ? a : lo;
        hi = b > hi ? b : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&V.keys[0], lo);
        atomicMax(&V.keys[1], hi);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && V.ctl[0] != n) live_fail(V);  // every value reached the pool
}

constexpr int kHistShared = 8192;
__global__ void k_live_hist(LiveDev V, int n) {
    pdl_entry();
    if (V.ctl[1]) return;
    __shared__ int s_h[kHistShared];
    const Buckets B = buckets_of(V);
    const bool sh = B.nb <= kHistShared;
    if (sh)
        for (int b = threadIdx.x; b < B.nb; b += blockDim.x) s_h[b] = 0;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int b = B(V.pool[i]);
        if (sh) atomicAdd(&s_h[b], 1); else atomicAdd(&V.bcount[b], 1);
    }
    __syncthreads();
    if (sh)
        for (int b = threadIdx.x; b < B.nb; b += blockDim.x)
            if (s_h[b]) atomicAdd(&V.bcount[b], s_h[b]);
}

// exclusive scan of the bucket counts (one CTA): starts in bcount[nb ..], cursors in bcur
__global__ void __launch_bounds__(1024) k_live_scan(LiveDev V) {
    pdl_entry();
    if (V.ctl[1]) return;
    __shared__ int s_wt[32];
    const int nb = V.nb;
    const int per = (nb + 1023) / 1024;
    const int i0 = threadIdx.x * per;
    int local = 0, big = 0;
    for (int k = 0; k < per; ++k)
        if (i0 + k < nb) {
            const int c = V.bcount[i0 + k];
            local += c;
            big = max(big, c);
        }
    if (__syncthreads_or(big > kBucketCap)) {
        if (threadIdx.x == 0) live_fail(V);
        return;
    }
    int tot;
    int run = cta_excl_scan<1024>(local, tot, s_wt);
    for (int k = 0; k < per; ++k)
        if (i0 + k < nb) {
            V.bcount[nb + i0 + k] = run;
            V.bcur[i0 + k] = run;
            run += V.bcount[i0 + k];
        }
    if (threadIdx.x == 0) V.bcount[2 * nb] = tot;
}

__global__ void k_live_scatter(LiveDev V, int n) {
    pdl_entry();
    if (V.ctl[1]) return;
    const Buckets B = buckets_of(V);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double x = V.pool[i];
        V.tmp[atomicAdd(&V.bcur[B(x)], 1)] = x;
    }
}

__global__ void __launch_bounds__(kBucketThreads) k_live_bucket(LiveDev V, double* __restrict__ out) {
    pdl_entry();
    if (V.ctl[1]) return;
    __shared__ double s_v[kBucketCap];
    const int b = blockIdx.x;
    const int start = V.bcount[V.nb + b], cnt = V.bcount[b];
    for (int i = threadIdx.x; i < cnt; i += kBucketThreads) s_v[i] = V.tmp[start + i];
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += kBucketThreads) {
        const double x = s_v[i];
        int r = 0;
        for (int j = 0; j < cnt; ++j) {
            const double y = s_v[j];
            r += (y < x) || (y == x && j < i);
        }
        out[start + r] = x;
    }
}

// Several blocks (a batch): every live block (<= kBucketCap elements) is sorted
// from its own pool by one CTA -- a bitonic network over order-preserving 64-bit
// keys in shared memory (padded to a power of two with +inf); a pool that did
// not fill its block is a fallback.
__global__ void __launch_bounds__(kBucketThreads) k_live_blocksort(LiveDev V, const int* __restrict__ blocks,
                                                                   double* __restrict__ out) {
    pdl_entry();
    if (V.ctl[1]) return;
    __shared__ unsigned long long s_k[kBucketCap];
    const int b = blocks[blockIdx.x];
    const int start = V.bstart[b], cnt = V.bstart[b + 1] - start;
    if (V.bctr[b] != cnt) {
        if (threadIdx.x == 0) live_fail(V);
        return;
    }
    int P = 1;
    while (P < cnt) P <<= 1;
    for (int i = threadIdx.x; i < P; i += kBucketThreads) s_k[i] = i < cnt ? okey(V.pool[start + i]) : ~0ULL;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < P / 2; t += kBucketThreads) {
                const int i = 2 * t - (t & (j - 1));  // lower index of the pair (i, i + j)
                const int q = i + j;
                const bool up = (i & k) == 0;
                const unsigned long long a = s_k[i], c = s_k[q];
                if ((a > c) == up) {
                    s_k[i] = c;
                    s_k[q] = a;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < cnt; i += kBucketThreads) out[start + i] = okey_val(s_k[i]);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void launch_live_init(cudaStream_t s, const Work& w, const LiveDev& V, const int2* front, int nfront,
                      double tol_scale, int* launches, Prof* prof) {
    launch_pdl(k_live_init, nfront, kLiveInitThreads, 0, s, w, V, front, tol_scale);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE);
}

void launch_level_live(cudaStream_t s, const Work& w, const LevelDev& L, const LiveDev& V,
                       const SolveParams& prm, int* traceOut, int* launches, Prof* prof) {
    const size_t sm = sizeof(LiveSmem);
    if (L.allSplit && L.M > prm.sms) {  // many split-rule merges: lane groups, G merges per CTA
        const int per = std::max(1, std::min(kLiveGroup, L.M / (prm.sms * kLiveCtasPerSm)));
        const int G = std::min(per, kLiveGroupMax);
        launch_pdl(k_live_level<3, kLiveM3Threads>, (L.M + G - 1) / G, kLiveM3Threads, sm, s, w, L, V, prm, traceOut, G);
    } else if (L.allSplit) {  // few large merges: one per CTA, a warp per root
        launch_pdl(k_live_level<1, kLiveSplitThreads>, L.M, kLiveSplitThreads, sm, s, w, L, V, prm, traceOut, 1);
    } else if (L.maxSize > kSplitMinSize) {  // both sides of the split rule (unbalanced tree)
        launch_pdl(k_live_level<2, kLiveThreads>, L.M, kLiveThreads, sm, s, w, L, V, prm, traceOut, 1);
    } else {
        // merges per CTA: a level of many merges packs up to kLiveGroup per CTA
        // (a merge keeps K ~ 100 roots for 256 lanes), a few-merge level keeps one
        const int per = std::max(1, std::min(kLiveGroup, L.M / (prm.sms * kLiveCtasPerSm)));
        const int G = std::min(per, kLiveGroupMax);
        launch_pdl(k_live_level<0, kLiveThreads>, (L.M + G - 1) / G, kLiveThreads, sm, s, w, L, V, prm, traceOut, G);
    }
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE);
}

// merges per work item of a lane-mode live level of M merges (the per-level
// launch's CTA share, launch_level_live)
int live_lane_group(int M, int sms) {
    const int per = std::max(1, std::min(kLiveGroup, M / (sms * kLiveCtasPerSm)));
    return std::min(per, kLiveGroupMax);
}

void launch_live_flow(cudaStream_t s, const Work& w, const LiveRun& R, const LiveDev& V, const SolveParams& prm,
                      int* launches, Prof* prof) {
    launch_pdl(k_live_flow, std::min(R.nitems, prm.sms * kLiveCtasPerSm), kLiveThreads, sizeof(LiveSmem), s, w, R,
               V, prm);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE);
}

void launch_live_top(cudaStream_t s, const Work& w, const LiveRun& R, const LiveDev& V, const SolveParams& prm,
                     int* launches, Prof* prof) {
    launch_pdl(k_live_top, R.first[R.nlev], kLiveSplitThreads, sizeof(LiveSmem), s, w, R, V, prm);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE);
}

// cluster size of a split-rule live level of M merges: the largest power of two
// c <= 16 for which all M clusters are co-resident (cudaOccupancyMaxActiveClusters:
// a cluster must fit one GPC, so 16 clusters of 8 need not fit 148 SMs) -- a
// second wave would double the level's time.  Probed once per device.
static int g_cluster_active[64][5];  // [device][log2 c]: co-resident clusters of c CTAs (0: unprobed)
static bool g_cluster_probed[64];
int live_cluster_max(int device) {
    if (device < 0 || device >= 64) return 1;
    if (!g_cluster_probed[device]) {
        cudaFuncSetAttribute(k_live_cluster<kClThreads, kClLpr>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k_live_cluster<kClThreads, kClLpr>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(LiveSmem));
        for (int l = 1; l <= 4; ++l) {
            const int c = 1 << l;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(c);
            cfg.blockDim = dim3(kClThreads);
            cfg.dynamicSmemBytes = sizeof(LiveSmem);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, k_live_cluster<kClThreads, kClLpr>, &cfg) != cudaSuccess) {
                cudaGetLastError();
                nc = 0;
            }
            g_cluster_active[device][l] = nc;
        }
        g_cluster_probed[device] = true;
    }
    int best = 1;
    for (int l = 1; l <= 4; ++l)
        if (g_cluster_active[device][l] > 0) best = 1 << l;
    return best;
}

int live_cluster_size(int device, int M, int cmax) {
    int c = 1;
    for (int l = 1; l <= 4 && (1 << l) <= cmax; ++l)
        if (device >= 0 && device < 64 && M <= g_cluster_active[device][l]) c = 1 << l;
    return c;
}

void launch_level_live_cluster(cudaStream_t s, const Work& w, const LevelDev& L, const LiveDev& V,
                               const SolveParams& prm, int* traceOut, int C, int* launches, Prof* prof) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(L.M * C);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = sizeof(LiveSmem);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = C;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, k_live_cluster<kClThreads, kClLpr>, w, L, V, prm, traceOut);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE);
}

// co-resident CTAs of k_live_top (the run's merges must all fit at once)
int live_top_capacity(int sms) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_live_top, kLiveSplitThreads, sizeof(LiveSmem));
    return per * sms;
}

void launch_live_sort(cudaStream_t s, const LiveDev& V, int n, double* out, int sms, int* launches, Prof* prof) {
    const int g = sms * 4;
    launch_pdl(k_live_bounds, g, 256, 0, s, V, n);
    launch_pdl(k_live_hist, g, 256, 0, s, V, n);
    launch_pdl(k_live_scan, 1, 1024, 0, s, V);
    launch_pdl(k_live_scatter, g, 256, 0, s, V, n);
    launch_pdl(k_live_bucket, V.nb, kBucketThreads, 0, s, V, out);
    *launches += 5;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE_SORT);
}

int live_buckets(int n) { return n / 128 > 1 ? n / 128 : 1; }
int live_block_cap() { return kBucketCap; }

void launch_live_blocksort(cudaStream_t s, const LiveDev& V, const int* blocks, int nlive, double* out,
                           int* launches, Prof* prof) {
    launch_pdl(k_live_blocksort, nlive, kBucketThreads, 0, s, V, blocks, out);
    *launches += 1;
    if (prof) prof_mark(prof, (void*)s, BRGPU_K_LIVE_SORT);
}

void init_live_attributes() {
    const int sm = (int)sizeof(LiveSmem);
    cudaFuncSetAttribute(k_live_level<0, kLiveThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_level<1, kLiveSplitThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_level<2, kLiveThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_level<3, kLiveM3Threads>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_top, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_cluster<kClThreads, kClLpr>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_live_cluster<kClThreads, kClLpr>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

static_assert(sizeof(LiveSmem) <= 75 * 1024, "three live CTAs per SM");

}  // namespace brgpu
