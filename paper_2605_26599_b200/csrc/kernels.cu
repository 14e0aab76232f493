// kernels.cu -- sm_100a kernels of the boundary-row (BR) eigenvalue-only
// divide-and-conquer tridiagonal eigensolver.  Built with --fmad=false (see
// numerics.cuh).  Every kernel is launched by the host planner in api.cpp.
//
// Level pipeline (grid tier; one launch per step covers ALL merges of a
// level, positions are level-global so no host round trip is needed):
//   k_merge_prep     per-merge max(|D|,|z|) + merge-path splits  deflate.cpp:55-60
//   k_merge_nn       stable merge of the sorted children deflate.cpp:62-66, build_z deflate.cpp:31-41,
//                    small-z flags + compaction, 1 pass  deflate.cpp:70-75
//   k_segment_walk   close-pole groups per segment       deflate.cpp:76-95, 109-140
//   k_surv_scan      survivor compaction, 1 pass         deflate.cpp:100-105
//   k_secular        lane-per-root RootSM + CTA queue    secular.cpp:80-241 (tiled.cu, warp.cu: other tiers)
//   k_zhat           refreshed weights, one pole/thread  secular.cpp:288-313
//   k_rows           R_parent(:,j) = R_child y_j + parent placement
//   k_deflated_out   deflated columns to parent order
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"
#include "grid_common.cuh"
#include "level_state.cuh"

namespace brgpu {

constexpr int kScanBlock = 1024;

// ---------------------------------------------------------------------------
// input validation + irreducible block split (tridiagonal.cpp:17-30, 45-58)
// ---------------------------------------------------------------------------
__global__ void k_copy_input(int n, const double* __restrict__ d, const double* __restrict__ e,
                             double* __restrict__ dw, double* __restrict__ ew) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dw[i] = d[i];
    ew[i] = i + 1 < n ? e[i] : 0.0;
}

// dw/ew hold the input; flags split points |e_i| <= u(|d_i|+|d_{i+1}|)
__global__ void k_scan_input(int n, const double* __restrict__ d, const double* __restrict__ e,
                             uint8_t* __restrict__ split, int* __restrict__ nsplit,
                             int* __restrict__ status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int cnt = 0;
    if (i < n) {
        const double di = d[i];
        bool bad = !isfinite(di);
        uint8_t s = 0;
        if (i + 1 < n) {
            const double ei = e[i];
            bad |= !isfinite(ei);
            s = fabs(ei) <= kU * (fabs(di) + fabs(d[i + 1]));
        }
        if (bad) set_status(status, BRGPU_ERR_INVALID_ARGUMENT);
        split[i] = s;
        cnt = s;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nsplit, cnt);
}

// batch of independent matrices laid end to end; matrix ends are implied
// block boundaries (not flagged), natural split points are flagged.
__global__ void k_scan_input_batched(int batch, int n, const double* __restrict__ d,
                                     const double* __restrict__ e, double* __restrict__ dw,
                                     double* __restrict__ ew, uint8_t* __restrict__ split,
                                     int* __restrict__ nsplit, int* __restrict__ status) {
    const long long N = (long long)batch * n;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int cnt = 0;
    if (i < N) {
        const int b = (int)(i / n), j = (int)(i - (long long)b * n);
        const double di = d[i];
        dw[i] = di;
        bool bad = !isfinite(di);
        uint8_t s = 0;
        double ei = 0.0;
        if (j + 1 < n) {
            ei = e[(long long)b * (n - 1) + j];
            bad |= !isfinite(ei);
            s = fabs(ei) <= kU * (fabs(di) + fabs(d[i + 1]));
        }
        ew[i] = ei;
        if (bad) set_status(status, BRGPU_ERR_INVALID_ARGUMENT);
        split[i] = s;
        cnt = s;
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nsplit, cnt);
}

// block id of position i (bstart ascending, nblk+1 entries)
__device__ __forceinline__ int find_block(const int* __restrict__ bstart, int nblk, int i) {
    int lo = 0, hi = nblk;  // last b with bstart[b] <= i
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bstart[mid] <= i) lo = mid; else hi = mid;
    }
    return lo;
}

// per-block scale = max(1, |d|, |e internal|), computed on dw/ew
__global__ void k_block_scale(int n, const double* __restrict__ d, const double* __restrict__ e,
                              const int* __restrict__ bstart, int nblk,
                              unsigned long long* __restrict__ sbits) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = (i < n && nblk > 1) ? find_block(bstart, nblk, i) : 0;
    double v = 0.0;
    if (i < n) {
        v = fabs(d[i]);
        if (i + 1 < bstart[b + 1]) v = fmax(v, fabs(e[i]));
    }
    unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    // a warp inside one block reduces first and issues one atomic (batches: one
    // atomic per element on ~n/1024 words was a 0.33 ms hot spot at 4096 x 1024)
    const int b0 = __shfl_sync(0xffffffffu, b, 0);
    if (__all_sync(0xffffffffu, i >= n || b == b0)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long y = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = y > bits ? y : bits;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(&sbits[b0], bits);
    } else if (i < n) {
        atomicMax(&sbits[b], bits);
    }
}

// in place: dw /= s, ew /= s inside the block, 0 at block boundaries
// Block scale: max(1, |d|, |e|); tiny blocks (max < 2^-500) are
// lifted by the power of two 2^ilogb(max) instead -- exact, and it keeps the
// boundary-row sums from overflowing (the checker's GPU-mode rule).
__device__ __forceinline__ double block_scale_of(unsigned long long bits) {
    const double mx = __longlong_as_double((long long)bits);
    if (mx > 0.0 && mx < 0x1p-500) return ldexp(1.0, ilogb(mx));
    return fmax(1.0, mx);
}

__global__ void k_apply_scale(int n, const int* __restrict__ bstart, int nblk,
                              const unsigned long long* __restrict__ sbits,
                              double* __restrict__ dw, double* __restrict__ ew) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = nblk == 1 ? 0 : find_block(bstart, nblk, i);
    const double s = block_scale_of(sbits[b]);
    dw[i] = dw[i] / s;
    ew[i] = (i + 1 < bstart[b + 1]) ? ew[i] / s : 0.0;
}

// Cuppen cuts (merge_tree.cpp:78-92).  With leaf cutoff >= 3 every cut
// position is strictly interior to its node, so no position is cut twice and
// the cuts commute: one thread per internal node, bitwise equal to pre-order.
__global__ void k_cuts(int ncut, const int* __restrict__ cutPos, const double* __restrict__ ew,
                       double* __restrict__ dw) {
    pdl_entry();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncut) return;
    const int m = cutPos[t];
    const double rho = fabs(ew[m]);
    dw[m] -= rho;
    dw[m + 1] -= rho;
}

// ---------------------------------------------------------------------------
// leaves (qrql.cpp:396-413) and small blocks (qrql.cpp:386-394): one per thread
// ---------------------------------------------------------------------------
// Per-thread arrays live in shared memory ([i][thread] layout): a leaf's QL
// sweeps are a serial chain of dependent loads/stores, so they must hit SMEM
// latency, not L1-thrashing local memory (4 x MAXM doubles per thread).
constexpr int kLeafThreads = 64;
constexpr int kLeafSpreadWarps = 148 * 4;  // warps to spread a small leaf set over
// per-thread SMEM doubles: d[MAXM], e[MAXM-1] (e[m-1] is never read), r0, r1.
// At MAXM = 16 this is 63 doubles = 32256 B per 64-thread CTA, so 7 CTAs fit in
// one SM (7 x (32256 + 1024 reserved) <= 233472 B) and the 65536 leaves of an
// n = 2^20 problem (1024 CTAs <= 7 x 148) run in ONE wave instead of two.
template <int MAXM>
constexpr int leaf_smem_bytes() { return (4 * MAXM - 1) * kLeafThreads * (int)sizeof(double); }

template <int MAXM>
__global__ void __launch_bounds__(kLeafThreads) k_leaf(int ntask, const int* __restrict__ tOff,
                                                       const int* __restrict__ tSize,
                                                       const int* __restrict__ tFlags,
                                                       const double* __restrict__ dw,
                                                       const double* __restrict__ ew,
                                                       double* __restrict__ lam,
                                                       double* __restrict__ blo,
                                                       double* __restrict__ bhi,
                                                       int* __restrict__ status, int per_warp) {
    pdl_entry();
    extern __shared__ double leaf_sm[];
    // per_warp leaves per warp (lanes >= per_warp idle): 32 packs the machine
    // when there are many leaves; fewer shorten the latency of small solves,
    // where one warp's divergent leaves would otherwise run back to back
    const int lane = threadIdx.x & 31;
    if (lane >= per_warp) return;
    const int t = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * per_warp + lane;
    if (t >= ntask) return;
    const int off = tOff[t], m = tSize[t];
    const bool values_only = tFlags[t] & 1;
    constexpr int S = kLeafThreads;
    const Strided<S> d{leaf_sm + threadIdx.x};
    const Strided<S> e{leaf_sm + MAXM * S + threadIdx.x};
    const Strided<S> r0{leaf_sm + (2 * MAXM - 1) * S + threadIdx.x};
    const Strided<S> r1{leaf_sm + (3 * MAXM - 1) * S + threadIdx.x};
    for (int i = 0; i < m; ++i) {
        d[i] = dw[off + i];
        if (i + 1 < m) e[i] = ew[off + i];
        r0[i] = 0.0;
        r1[i] = 0.0;
    }
    r0[0] = 1.0;
    r1[m - 1] = 1.0;
    const int st = values_only ? steqr_leaf<false>(m, d, e, r0, r1) : steqr_leaf<true>(m, d, e, r0, r1);
    if (st) set_status(status, st);
    // stable ascending sort (qrql.cpp:348-364): rank = #{d_j < d_i} + #{j<i: d_j == d_i},
    // on a register copy of the eigenvalues (unrolled; entries j >= m never count)
    double dv[MAXM];
#pragma unroll
    for (int j = 0; j < MAXM; ++j) dv[j] = j < m ? d[j] : 0.0;
#pragma unroll
    for (int i = 0; i < MAXM; ++i) {
        if (i < m) {
            const double di = dv[i];
            int rank = 0;
#pragma unroll
            for (int j = 0; j < MAXM; ++j) rank += j < m && ((dv[j] < di) || (j < i && dv[j] == di));
            lam[off + rank] = di;
            if (!values_only) {
                blo[off + rank] = r0[i];
                bhi[off + rank] = r1[i];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// level pipeline
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// single-pass compaction scans (decoupled look-back).  Tile states are packed
// 64-bit words: bits 62-63 status (1 aggregate, 2 inclusive), low 32 the count;
// tiles are taken in ticket order so every predecessor is resident or done.
// ---------------------------------------------------------------------------
constexpr unsigned long long kTileAgg = 1ULL << 62, kTileInc = 2ULL << 62;

// Warp 0 only: publish the tile aggregate, look back, return the exclusive
// prefix (valid in every lane of warp 0).
__device__ __forceinline__ int warp_lookback(unsigned long long* state, int tile, int aggregate) {
    const int lane = threadIdx.x & 31;
    if (lane == 0)
        atomicExch(&state[tile], ((tile == 0 ? 2ULL : 1ULL) << 62) | (unsigned)aggregate);
    int prefix = 0;
    if (tile > 0) {
        int j = tile - 1;
        for (;;) {
            const int idx = j - lane;
            unsigned long long v = idx >= 0 ? *(volatile unsigned long long*)&state[idx] : (2ULL << 62);
            while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
                if ((v >> 62) == 0) v = *(volatile unsigned long long*)&state[idx];
            }
            const unsigned incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
            const int k = incl ? __ffs(incl) - 1 : 31;
            int c = lane <= k ? (int)(unsigned)(v & 0xffffffffULL) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            prefix += c;
            if (incl) break;
            j -= 32;
        }
        if (lane == 0) atomicExch(&state[tile], kTileInc | (unsigned)(prefix + aggregate));
    }
    return prefix;
}

__device__ __forceinline__ int cta_lookback(unsigned long long* state, int tile, int aggregate,
                                            int* s_bcast) {
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors per step
        const int lane = threadIdx.x;
        if (lane == 0)
            atomicExch(&state[tile], ((tile == 0 ? 2ULL : 1ULL) << 62) | (unsigned)aggregate);
        int prefix = 0;
        if (tile > 0) {
            int j = tile - 1;
            for (;;) {
                const int idx = j - lane;
                unsigned long long v = idx >= 0 ? *(volatile unsigned long long*)&state[idx] : (2ULL << 62);
                while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
                    if ((v >> 62) == 0) v = *(volatile unsigned long long*)&state[idx];
                }
                const unsigned incl = __ballot_sync(0xffffffffu, (v >> 62) == 2);
                // closest inclusive predecessor = lowest set lane; sum lanes [0, k]
                const int k = incl ? __ffs(incl) - 1 : 31;
                int c = lane <= k ? (int)(unsigned)(v & 0xffffffffULL) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                prefix += c;
                if (incl) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&state[tile], kTileInc | (unsigned)(prefix + aggregate));
        }
        if (lane == 0) *s_bcast = prefix;
    }
    __syncthreads();
    return *s_bcast;
}

constexpr int kMergeTile = 256;
constexpr int kPrepVec = 4;  // merge tiles per k_merge_prep CTA: the whole level is one wave

// Merge preparation over kPrepVec merge tiles per CTA (one pass, one wave):
//  * the per-merge deflation scale max(|D|, |z|) (deflate.cpp:55-60), an
//    order-free max: segmented warp reduction, then one atomicMax per merge
//    segment of each tile (a tile inside one merge reduces through shared
//    memory first);
//  * the merge-path diagonal split at each tile's first position (warp k for
//    tile k, 32-ary search), kept in split[tile] for k_merge_nn.
__global__ void __launch_bounds__(kMergeTile) k_merge_prep(Work w, LevelDev L, int n, int* __restrict__ split) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ unsigned long long s_max[kPrepVec][kMergeTile / 32];
    __shared__ int s_m[kPrepVec][kMergeTile / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tile0 = blockIdx.x * kPrepVec;
    int mk[kPrepVec];
    unsigned long long bk[kPrepVec];
#pragma unroll
    for (int k = 0; k < kPrepVec; ++k) {  // independent loads of the CTA's positions
        const int p = (tile0 + k) * kMergeTile + threadIdx.x;
        const int m = p < n ? find_merge(L, p) : -1;
        mk[k] = m;
        bk[k] = 0ULL;
        if (m >= 0) {
            const int off = L.mOff[m], nl = L.mNL[m];
            const double zs = p < off + nl ? w.bhi[p] : w.blo[p];
            bk[k] = (unsigned long long)__double_as_longlong(fmax(fabs(w.lam[p]), fabs(zs)));
        }
    }
#pragma unroll
    for (int k = 0; k < kPrepVec; ++k) {
        const int m = mk[k];
        unsigned long long bits = bk[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long b2 = __shfl_down_sync(0xffffffffu, bits, o);
            const int m2 = __shfl_down_sync(0xffffffffu, m, o);
            if (lane + o < 32 && m2 == m && b2 > bits) bits = b2;
        }
        const int m31 = __shfl_sync(0xffffffffu, m, 31);
        const bool whole = __all_sync(0xffffffffu, m == m31) && m31 >= 0;
        if (lane == 0) {
            s_m[k][wid] = whole ? m : -2;
            s_max[k][wid] = bits;
        }
        bk[k] = bits;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPrepVec; ++k) {
        bool tile_whole = true;
#pragma unroll
        for (int q = 0; q < kMergeTile / 32; ++q) tile_whole = tile_whole && s_m[k][q] == s_m[k][0] && s_m[k][q] >= 0;
        if (tile_whole) {
            if (threadIdx.x == 0) {
                unsigned long long b = s_max[k][0];
#pragma unroll
                for (int q = 1; q < kMergeTile / 32; ++q) b = s_max[k][q] > b ? s_max[k][q] : b;
                atomicMax(&L.mTol[s_m[k][0]], b);
            }
        } else {
            const int m = mk[k];
            const int mp = __shfl_up_sync(0xffffffffu, m, 1);
            if (m >= 0 && (lane == 0 || mp != m)) atomicMax(&L.mTol[m], bk[k]);
        }
    }
    if (wid < kPrepVec) {
        const int tile = tile0 + wid;
        const int p0 = tile * kMergeTile;
        const int m0 = p0 < n ? find_merge(L, p0) : -1;
        if (m0 >= 0) {
            const int off = L.mOff[m0], nl = L.mNL[m0], nr = L.mSize[m0] - nl;
            const double* la = w.lam + off;
            const int sp = warp_merge_split(la, nl, la + nl, nr, p0 - off);
            if (lane == 0) split[tile] = sp;
        }
    }
}

// Stable merge of the sorted children (merge path), z = (sign*bhi_L, blo_R)
// and the non-negligible flags |z| > tol (deflate.cpp:31-41, 62-72) with their
// single-pass prefix (nnPre) and list (nnPos).  A CTA owns kMergeTile output
// positions; the diagonal splits bounding each merge segment's inputs come
// from k_merge_prep (tile start) or are the merge's ends, so the inputs are
// loaded coalesced at once, placed by searches in shared memory and written
// back coalesced in merged order.  The tile's flag count (order-free: the same
// elements) is published before the placement so the look-back overlaps it.
__global__ void __launch_bounds__(kMergeTile) k_merge_nn(Work w, LevelDev L, int n, double tol_scale,
                                                         const int* __restrict__ split,
                                                         unsigned long long* state, int* ticket) {
    pdl_entry();
    if (!dense_entry(L)) return;
    // inputs (lam, blo, bhi), then the merged tile (D, Z, R0 alias them; R1)
    __shared__ double s_v[kMergeTile], s_b0[kMergeTile], s_b1[kMergeTile], s_R1[kMergeTile];
    double* s_D = s_v;
    double* s_Z = s_b0;
    double* s_R0 = s_b1;
    __shared__ int s_red[kMergeTile / 32];
    __shared__ int s_tile, s_pref;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    const int t = threadIdx.x;
    const int lane = t & 31, wid = t >> 5;
    const int p0 = tile * kMergeTile;
    const int p = p0 + t;
    const int m = p < n ? find_merge(L, p) : -1;
    int off = 0, nl = 0, q0 = 0, q1 = 0, i0 = 0, j0 = 0, la = 0, u = 0, f = 0;
    double tol = 0.0;
    if (m >= 0) {
        off = L.mOff[m];
        nl = L.mNL[m];
        const int size = L.mSize[m];
        q0 = max(p0, off);
        q1 = min(min(p0 + kMergeTile, n), off + size);
        i0 = q0 == off ? 0 : split[tile];                      // a segment starting mid-tile starts its merge
        const int i1 = q1 == off + size ? nl : split[tile + 1];  // ... and one ending mid-tile ends it
        la = i1 - i0;
        j0 = (q0 - off) - i0;
        u = p - q0;
        const bool left = u < la;
        const int src = left ? off + i0 + u : off + nl + j0 + (u - la);
        const double b0 = w.blo[src], b1 = w.bhi[src];
        s_v[t] = w.lam[src];
        s_b0[t] = b0;
        s_b1[t] = b1;
        tol = merge_tol(L, m, tol_scale);
        f = fabs(left ? b1 : b0) > tol;  // |z| (the sign does not matter)
    }
    // tile flag count: published before the placement so the look-back overlaps it
    int c = __reduce_add_sync(0xffffffffu, f);
    if (lane == 0) s_red[wid] = c;
    __syncthreads();
    if (wid == 0) {
        c = lane < kMergeTile / 32 ? s_red[lane] : 0;
        c = __reduce_add_sync(0xffffffffu, c);
        const int pref = warp_lookback(state, tile, c);
        if (lane == 0) s_pref = pref;
    }
    int o = -1;
    double v = 0.0, z = 0.0, r0 = 0.0, r1 = 0.0;
    if (m >= 0) {
        const int h = q0 - p0;
        v = s_v[t];
        int sp;  // merge-local output index
        if (u < la) {  // left element i0+u: right elements before it are b[0..j0) + local ones < v
            sp = (i0 + u) + j0 + count_less(s_v + h + la, (q1 - q0) - la, v);
            const double em = w.ew[off + nl - 1];
            const double b = s_b1[t];
            z = em < 0 ? -b : b;
            r0 = s_b0[t];
            r1 = 0.0;
        } else {       // right element j0+u-la: left elements before it are a[0..i0) + local ones <= v
            sp = (j0 + u - la) + i0 + count_leq(s_v + h, la, v);
            z = s_b0[t];
            r0 = 0.0;
            r1 = s_b1[t];
        }
        o = off + sp - p0;
    }
    __syncthreads();  // every search is done: the input slots become the merged tile
    if (o >= 0) {
        s_D[o] = v;
        s_Z[o] = z;
        s_R0[o] = r0;
        s_R1[o] = r1;
    }
    __syncthreads();
    f = 0;
    if (m >= 0) {
        z = s_Z[t];
        w.D[p] = s_D[t];
        w.Z[p] = z;
        w.R0[p] = s_R0[t];
        w.R1[p] = s_R1[t];
        f = fabs(z) > tol;
    }
    if (p < n) w.nnFlag[p] = (uint8_t)f;
    int tot;
    const int ex = block_exclusive_scan<kMergeTile>(f, tot);
    const int base = s_pref;
    if (p < n) {
        w.nnPre[p] = base + ex;
        if (f) w.nnPos[base + ex] = p;
    }
    if (t == kMergeTile - 1 && (tile + 1) * kMergeTile >= n) w.nnPre[n] = base + tot;
}

// Close-pole deflation (deflate.cpp:76-95, 109-140).  A segment is a maximal
// run of consecutive non-negligible sorted poles whose neighbour gaps are
// <= tol; its first pole is always a survivor (its gap to any earlier survivor
// exceeds tol), so segments are independent.  The segment head walks its run
// with the reference's rule (a pole within tol of the last survivor is
// absorbed by it) and evaluates each group's rotation chain from prefix sums
// (the checker's deflate_walk / group_member): the walk carries only
// Q = sum z^2, S0/S1 = sum z x -- one add per member on the dependency chain --
// and records each member's prefix (Q, S0, S1) at its position in the free
// lam/blo/bhi slots; k_surv_scan finishes the members in parallel.
// Long segments are walked by the whole warp: 32 NN entries are loaded at once
// (one coalesced position load, one gather of their data), then every lane
// replays the walk over the chunk in lane order from shuffles (the same
// operations in the same order as a sequential walk, so every lane holds the
// same Q/S0/S1) and each lane keeps the prefix at its own entry -- a run of
// 10^4 close poles (glued Wilkinson) costs two dependent L2 round trips per 32
// entries.  A segment of length 1 (random inputs: almost all) is decided by its
// head's first probe, with no warp work.
__device__ __forceinline__ void walk_retire(const Work& w, int prev, double Q, double S0, double S1) {
    const double R = sqrt(Q), iR = 1.0 / R;
    w.Z[prev] = R; w.R0[prev] = S0 * iR; w.R1[prev] = S1 * iR;
}

__global__ void __launch_bounds__(256) k_segment_walk(Work w, LevelDev L, int n, double tol_scale) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int NN = w.nnPre[n];
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int c0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; c0 < NN; c0 += nwarps * 32) {
        const int q = c0 + lane;
        bool lng = false;
        int k = 0, qe = 0;
        double tol = 0.0, dk = 0.0;
        if (q < NN) {
            k = w.nnPos[q];
            const int m = find_merge(L, k);
            const int off = L.mOff[m];
            const int qs = w.nnPre[off];
            qe = w.nnPre[off + L.mSize[m]];
            tol = merge_tol(L, m, tol_scale);
            dk = w.D[k];
            const bool head = !(q > qs && fabs(dk - w.D[w.nnPos[q - 1]]) <= tol);
            if (head) {
                w.survFlag[q] = 1;
                lng = q + 1 < qe && fabs(w.D[w.nnPos[q + 1]] - dk) <= tol;
            }
        }
        unsigned heads = __ballot_sync(0xffffffffu, lng);
        while (heads) {
            const int src = __ffs(heads) - 1;
            heads &= heads - 1;
            const int hq = __shfl_sync(0xffffffffu, q, src);
            const int hqe = __shfl_sync(0xffffffffu, qe, src);
            const double htol = __shfl_sync(0xffffffffu, tol, src);
            int prev = __shfl_sync(0xffffffffu, k, src);
            double dp = __shfl_sync(0xffffffffu, dk, src);
            const double zs = w.Z[prev];
            double Q = zs * zs, S0 = zs * w.R0[prev], S1 = zs * w.R1[prev];
            double dprev_nn = dp;
            int nmem = 0;
            bool done = false;
            // two-stage prefetch: the next chunk's data and the chunk after's
            // positions are in flight while this chunk replays (a long segment is
            // then bound by the replay, not by dependent L2 round trips); loads
            // ahead are safe: the walk only writes the survivors' Z / R0 / R1,
            // which precede every entry still to come
            int kc = hq + 1 + lane < hqe ? w.nnPos[hq + 1 + lane] : 0;
            double d2 = 0.0, z2 = 0.0, x0 = 0.0, x1 = 0.0;
            if (hq + 1 + lane < hqe) { d2 = w.D[kc]; z2 = w.Z[kc]; x0 = w.R0[kc]; x1 = w.R1[kc]; }
            int kn = hq + 33 + lane < hqe ? w.nnPos[hq + 33 + lane] : 0;
            for (int cb = hq + 1; !done && cb < hqe; cb += 32) {
                const int q2 = cb + lane;
                const int k2 = kc;
                const bool nin = cb + 32 + lane < hqe;
                double nd = 0.0, nz = 0.0, nx0 = 0.0, nx1 = 0.0;
                if (nin) { nd = w.D[kn]; nz = w.Z[kn]; nx0 = w.R0[kn]; nx1 = w.R1[kn]; }
                const int knn = cb + 64 + lane < hqe ? w.nnPos[cb + 64 + lane] : 0;
                const int cnt = min(32, hqe - cb);
                int role = -1;  // this lane's entry: 0 member (prefix below), 1 group head
                double mQ = 0.0, mS0 = 0.0, mS1 = 0.0;
                for (int u = 0; u < cnt; ++u) {  // warp-uniform replay in lane order
                    const double du = __shfl_sync(0xffffffffu, d2, u);
                    if (fabs(du - dprev_nn) > htol) { done = true; break; }  // next segment head
                    dprev_nn = du;
                    const double zu = __shfl_sync(0xffffffffu, z2, u);
                    const double xu0 = __shfl_sync(0xffffffffu, x0, u);
                    const double xu1 = __shfl_sync(0xffffffffu, x1, u);
                    if (fabs(du - dp) <= htol) {  // member of prev's group
                        if (lane == u) { role = 0; mQ = Q; mS0 = S0; mS1 = S1; }
                        Q = Q + zu * zu;
                        S0 = S0 + zu * xu0;
                        S1 = S1 + zu * xu1;
                        ++nmem;
                    } else {  // a new group head inside the segment: retire the survivor
                        if (nmem && lane == 0) walk_retire(w, prev, Q, S0, S1);
                        if (lane == u) role = 1;
                        prev = __shfl_sync(0xffffffffu, k2, u);
                        dp = du;
                        nmem = 0;
                        Q = zu * zu; S0 = zu * xu0; S1 = zu * xu1;
                    }
                }
                if (role == 0) {
                    w.lam[k2] = mQ;
                    w.blo[k2] = mS0;
                    w.bhi[k2] = mS1;
                    w.survFlag[q2] = 0;
                } else if (role == 1) {
                    w.survFlag[q2] = 1;
                }
                kc = kn; d2 = nd; z2 = nz; x0 = nx0; x1 = nx1;
                kn = knn;
            }
            if (nmem && lane == 0) walk_retire(w, prev, Q, S0, S1);
        }
    }
}

// survivor prefix over NN indices + compacted active problem (deflate.cpp:100-105),
// one pass; tile 0 always runs so survPre[NN] is written even when NN == 0
__global__ void __launch_bounds__(kScanBlock) k_surv_scan(Work w, LevelDev L, int n,
                                                          unsigned long long* state, int* ticket) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ int s_tile, s_pref;
    const int NN = w.nnPre[n];
    // persistent: tiles in ticket order (the look-back waits only on earlier
    // tickets, held by resident CTAs); tile 0 always runs so survPre[NN] is written
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
        __syncthreads();
        const int tile = s_tile;
        if (tile > 0 && tile * kScanBlock >= NN) break;  // uniform per CTA
        const int q = tile * kScanBlock + threadIdx.x;
        const int f = q < NN ? w.survFlag[q] : 0;
        if (q < NN && !f) {  // group member: rotation-chain update from its prefix (k_segment_walk)
            const int k = w.nnPos[q];
            double x0 = w.R0[k], x1 = w.R1[k];
            group_member(w.lam[k], w.blo[k], w.bhi[k], w.Z[k], x0, x1);
            w.R0[k] = x0;
            w.R1[k] = x1;
            w.Z[k] = 0.0;
        }
        int tot;
        const int ex = block_exclusive_scan<kScanBlock>(f, tot);
        const int base = cta_lookback(state, tile, tot, &s_pref);
        const int g = base + ex;
        if (q < NN) {
            w.survPre[q] = g;
            if (f) {
                const int k = w.nnPos[q];
                const double z = w.Z[k];
                w.dA[g] = w.D[k];
                w.zA[g] = z;
                w.z2A[g] = z * z;
                w.r0A[g] = w.R0[k];
                w.r1A[g] = w.R1[k];
                w.aMerge[g] = find_merge(L, k);
            }
        }
        if (threadIdx.x == kScanBlock - 1 && (tile + 1) * kScanBlock >= NN) w.survPre[NN] = base + tot;
        __syncthreads();  // s_tile / s_pref reuse
    }
}

// Start of a grid-tier level: zero the per-merge scale words, the look-back
// tile states + tickets and the tier-mode word.  On a dense-only level this is
// the level's first kernel: it publishes the state slot (level_state.cuh).
__global__ void k_level_zero(LevelDev L, unsigned long long* __restrict__ st, int words, int* __restrict__ modes,
                             int modes0) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < L.M) L.mTol[i] = 0ULL;
    if (i < words) st[i] = 0ULL;
    if (i == 0) *modes = modes0;
}

// Which secular tiers a level needs (merges with K > 0): bit0 lane-per-root,
// bit1 warp-per-root.  Kernels of an absent tier exit on their first load.
__global__ void k_level_modes(Work w, LevelDev L) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    int bits = 0;
    if (m < L.M) {
        const int off = L.mOff[m];
        const int K = w.survPre[w.nnPre[off + L.mSize[m]]] - w.survPre[w.nnPre[off]];
        if (K > 0) bits = split_mode(L.mSize[m], K) ? 2 : 1;
    }
    bits = __reduce_or_sync(0xffffffffu, bits);
    if ((threadIdx.x & 31) == 0 && bits) atomicOr(w.levelModes, bits);
}

constexpr int kSecBlock = 128;
constexpr int kWin = 1024;

struct Window {
    int P0, P1;
    bool fits;
};

__device__ __forceinline__ Window range_window(const Work& w, const LevelDev& L, int c0, int c1,
                                               int cap) {
    int a, b, c, d;
    active_range(w, L, w.aMerge[c0], a, b);
    active_range(w, L, w.aMerge[c1 - 1], c, d);
    Window win;
    win.P0 = a;
    win.P1 = d;
    win.fits = (d - a) <= cap;
    return win;
}

__device__ __forceinline__ Window cta_window(const Work& w, const LevelDev& L, int T) {
    const int g0 = blockIdx.x * kSecBlock;
    return range_window(w, L, g0, min(g0 + kSecBlock, T), kWin);
}

// Secular roots (secular.cpp:80-241, tau-relative stop when patched).
// A CTA owns a chunk of roots; each lane runs one root's iteration as a
// resumable state machine (RootSM) and pulls the next root from a CTA queue
// as soon as its root converges.  Every evaluation is one warp-uniform loop
// over the poles (shared-memory broadcast reads), so lanes never wait on
// a neighbour's slower root and the pole loop has no divergence.
#ifndef BRGPU_SEC_WIN
#define BRGPU_SEC_WIN 2048
#endif
constexpr int kSecWinQ = BRGPU_SEC_WIN;
#ifndef BRGPU_SEC_MINB
#define BRGPU_SEC_MINB 6
#endif
#ifndef BRGPU_SEC_MINB_SMALL
#define BRGPU_SEC_MINB_SMALL 4
#endif
constexpr int kSecMinbSmall = BRGPU_SEC_MINB_SMALL;  // k_secular CTAs per SM below kSecBigLevel elements
constexpr int kSecBigLevel = 1 << 21;
constexpr int kSecMeta = 256;  // merges of a chunk staged in shared memory (more: global lookups)
// Secular roots (secular.cpp:80-241, tau-relative stop when patched).
// A CTA owns a chunk of roots; each lane runs one root's iteration as a
// resumable state machine (RootSM) and pulls the next root from a CTA queue
// as soon as its root converges.  Evaluations are branch-free pole loops over
// shared-memory (d, z^2) pairs (one LDS.128 per term, broadcast within a merge).
template <int MINB>
__global__ void __launch_bounds__(kSecBlock, MINB) k_secular(Work w, LevelDev L, int n, int patched) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ double2 s_dz[kSecWinQ];
    __shared__ double2 s_snap[kSecBlock];
    // per-merge table of the chunk's merges (active range start, rho, size):
    // the root queue and the iteration then touch no global metadata
    __shared__ int s_ks[kSecMeta + 1], s_sz[kSecMeta];
    __shared__ double s_rho[kSecMeta];
    __shared__ int s_next, s_nextLast;
    if (!(*w.levelModes & 1)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int R = max(kSecBlock, (T + (int)gridDim.x - 1) / (int)gridDim.x);
    const int c0 = blockIdx.x * R;
    if (c0 >= T) return;  // uniform per CTA
    const int c1 = min(c0 + R, T);
    const int m0 = w.aMerge[c0];
    const int nm = w.aMerge[c1 - 1] - m0 + 1;
    const bool meta = nm <= kSecMeta;  // uniform per CTA
    Window win;
    if (meta) {
        int lane_mode = 0;
        for (int t = threadIdx.x; t <= nm; t += kSecBlock) {
            const int m = m0 + min(t, nm - 1);
            const int off = L.mOff[m], size = L.mSize[m];
            s_ks[t] = w.survPre[w.nnPre[t < nm ? off : off + size]];
            if (t < nm) {
                s_sz[t] = size;
                s_rho[t] = fabs(w.ew[off + L.mNL[m] - 1]);
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nm; t += kSecBlock) {
            const int K = s_ks[t + 1] - s_ks[t];
            lane_mode |= K > 0 && !split_mode(s_sz[t], K);
        }
        if (!__syncthreads_or(lane_mode)) return;  // all roots belong to warp.cu
        win.P0 = s_ks[0];
        win.P1 = s_ks[nm];
        win.fits = win.P1 - win.P0 <= kSecWinQ;
    } else {
        if (!chunk_has_mode(w, L, c0, c1, false)) return;  // all roots belong to warp.cu
        win = range_window(w, L, c0, c1, kSecWinQ);
    }
    if (!win.fits) return;  // large-K chunk: k_secular_tiled (tiled.cu) owns it
    for (int i = threadIdx.x; i < win.P1 - win.P0; i += kSecBlock)
        s_dz[i] = make_double2(w.dA[win.P0 + i], w.z2A[win.P0 + i]);
    if (threadIdx.x == 0) {
        s_next = 0;
        s_nextLast = 0;
    }
    __syncthreads();

    RootSM st;
    int g = -1, ks = 0;
    bool exhausted = false, lastDone = false;
    int evals = 0;
    unsigned long long terms = 0;
    for (;;) {
        // refill: take roots from the CTA queue until one needs an evaluation.
        // Queue order: the last root of every merge of the chunk first (its
        // one-pole iteration averages ~2.5x the evaluations of an interior root),
        // then the interior roots in order -- never changes a result
        while (g < 0 && !exhausted) {
            int m = 0, t = 0, ke, gg;
            if (!lastDone) {
                t = atomicAdd(&s_nextLast, 1);
                if (t >= nm) { lastDone = true; continue; }
                m = m0 + t;
                if (meta) { ks = s_ks[t]; ke = s_ks[t + 1]; } else active_range(w, L, m, ks, ke);
                gg = ke - 1;
                if (gg < c0 || gg >= c1 || gg < ks) continue;  // not in this chunk (or K = 0)
            } else {
                const int q = atomicAdd(&s_next, 1);
                if (c0 + q >= c1) { exhausted = true; break; }
                gg = c0 + q;
                if (meta) {
                    t = upper_index(s_ks, nm, gg);
                    ks = s_ks[t];
                    ke = s_ks[t + 1];
                } else {
                    m = w.aMerge[gg];
                    active_range(w, L, m, ks, ke);
                }
                if (gg == ke - 1) continue;  // a last root: already taken
            }
            if (!owns(w, gg)) continue;  // another rank's root (root-range split)
            const int K = ke - ks;
            if (split_mode(meta ? s_sz[t] : L.mSize[m], K)) continue;  // warp-per-root tier (warp.cu)
            g = gg;
            const double rho = meta ? s_rho[t] : fabs(w.ew[L.mOff[m] + L.mNL[m] - 1]);
            const double2* pz = s_dz + (ks - win.P0);
            rs_begin(st, K, g - ks, rho, PolesPairs{pz}, K == 1 ? w.zA[ks] : 0.0, Z2Pairs{pz});
            if (st.phase == kRsDone) {
                w.org[g] = ks + st.org;
                w.tau[g] = st.tau;
                g = -1;
            }
        }
        if (!__any_sync(0xffffffffu, g >= 0)) break;
        if (g >= 0) {
            double sum, sum_abs, sum_d, psi;
            bool pole = false;
            const int K = st.K;
            const SmemPairs P{s_dz + (ks - win.P0)};
            if (!w.exact && eval_guard(P, K, st.j, st.dorg, st.tau))
                eval_fast(P, K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi, s_snap + threadIdx.x);
            else
                pole = eval_pass_exact(P, K, st.j, st.dorg, st.tau, sum, sum_abs, sum_d, psi);
            Ev ev;
            ev.f = 1.0 + st.rho * sum;
            ev.fp = st.rho * sum_d;
            ev.abs_sum = st.rho * sum_abs;
            ev.psi = st.rho * psi;
            ev.pole = pole;
            ++evals;
            terms += (unsigned long long)K;
            rs_consume(st, ev, PolesPairs{s_dz + (ks - win.P0)}, Z2Pairs{s_dz + (ks - win.P0)}, patched != 0);
            if (st.phase == kRsDone || st.phase == kRsFail) {
                if (st.phase == kRsFail) set_status(w.status, BRGPU_ERR_NO_CONVERGENCE);
                w.org[g] = ks + st.org;
                w.tau[g] = st.tau;
                g = -1;
            }
        }
    }
    evals = __reduce_add_sync(0xffffffffu, evals);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) terms += __shfl_xor_sync(0xffffffffu, terms, o);
    if ((threadIdx.x & 31) == 0 && evals) {
        atomicAdd(&w.counters[0], (unsigned long long)evals);
        atomicAdd(&w.counters[1], terms);
    }
}

// Self-test of rcp_nr against __drcp_rn (bitwise) over x = m * 2^e.
__global__ void k_selftest_rcp(long long count, unsigned long long seed, unsigned long long* bad) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    unsigned long long s = seed ^ (0x9E3779B97F4A7C15ULL * (unsigned long long)(i + 1));
    s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
    s *= 0x2545F4914F6CDD1DULL;
    const int ex = (int)((s >> 52) % 2001) - 1000;          // exponent in [-1000, 1000]
    unsigned long long mant = s & 0xFFFFFFFFFFFFFULL;         // random mantissa
    if (i & 1) {  // low-entropy mantissas: only the top k bits set (powers of two, 1.5, ...)
        const int k = (int)((s >> 20) % 53);
        mant &= ~((1ULL << (52 - k)) - 1ULL);
    }
    if ((i & 3) == 2) mant |= (1ULL << ((s >> 8) % 52)) - 1ULL;  // trailing ones
    double x = __longlong_as_double((long long)((1023ULL << 52) | mant));
    x = ldexp(x, ex);
    if (s & (1ULL << 63)) x = -x;
    if (__double_as_longlong(rcp_nr(x)) != __double_as_longlong(__drcp_rn(x))) atomicAdd(bad, 1ULL);
}

// Gu-Eisenstat refreshed weights, one pole per thread, roots in order
// (secular.cpp:288-313); replaces zA in place by sign(z)*sqrt(max(0,-w)).
// The roots' (d_origin, tau, d_j) triples stream through shared memory in
// tiles of kWin covering the CTA's window (one tile when it fits), in root
// order, so the product order is the checker's.
__global__ void __launch_bounds__(kSecBlock) k_zhat(Work w, LevelDev L, int n) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ double s_dorg[kWin], s_tau[kWin], s_dj[kWin];
    if (!(*w.levelModes & 1)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int g0 = blockIdx.x * kSecBlock;
    if (g0 >= T) return;  // uniform per CTA
    const Window win = cta_window(w, L, T);
    const int g = g0 + threadIdx.x;
    bool act = g < T;
    int ks = 0, K = 0, i = 0;
    double di = 0.0;
    if (act) {
        const int m = w.aMerge[g];
        int ke;
        active_range(w, L, m, ks, ke);
        // a lone pole keeps its z (the checker refreshes only K > 1)
        if ((L.mFlags[m] & kMergeRoot) || split_mode(L.mSize[m], ke - ks) || !owns(w, g) || ke - ks == 1)
            act = false;
        K = ke - ks;
        i = g - ks;
        di = w.dA[g];
    }
    double prod = 1.0;
    if (!__syncthreads_or(act)) return;
    const bool fast = act && !w.exact && zhat_guard(PolesPtr{w.dA + ks}, K, i);
    for (int tlo = win.P0; tlo < win.P1; tlo += kWin) {
        const int thi = min(tlo + kWin, win.P1);
        __syncthreads();
        for (int r = tlo + threadIdx.x; r < thi; r += kSecBlock) {
            s_dorg[r - tlo] = w.dA[w.org[r]];
            s_tau[r - tlo] = w.tau[r];
            s_dj[r - tlo] = w.dA[r];
        }
        __syncthreads();
        if (fast) {
            const int jlo = max(ks, tlo), jhi = min(ks + K, thi);
            for (int jg = jlo; jg < jhi; ++jg) {
                const int t = jg - tlo;
                const double del = (di - s_dorg[t]) - s_tau[t];
                const double dd = di - s_dj[t];
                const double f = ((jg - ks) == i) ? del : del * rcp_nr(dd);
                prod = prod * f;
            }
        }
    }
    if (!act) return;
    if (!fast) {  // exact redo (global memory)
        const double* __restrict__ dA = w.dA + ks;
        const double* __restrict__ tau = w.tau + ks;
        const int* __restrict__ org = w.org + ks;
        prod = 1.0;
        for (int j = 0; j < K; ++j) {
            const double del = (di - w.dA[org[j]]) - tau[j];
            if (j == i) prod = prod * del;
            else prod = prod * (del * __drcp_rn(di - dA[j]));
        }
    }
    const double mag = sqrt(fmax(0.0, -prod));
    w.zA[g] = w.zA[g] >= 0.0 ? mag : -mag;
}

// Parent boundary rows for root j: R_parent(:,j) = R_child y_j with
// y = zhat/Delta_j / ||zhat/Delta_j|| streamed (never stored),
// plus placement of lambda_j in the parent's ascending order.  Poles (d, zhat,
// r0, r1) stream through shared memory in tiles, in pole order.
__global__ void __launch_bounds__(kSecBlock) k_rows(Work w, LevelDev L, int n) {
    pdl_entry();
    if (!dense_entry(L)) return;
    __shared__ double s_d[kWin], s_zh[kWin], s_r0[kWin], s_r1[kWin];
    if (!(*w.levelModes & 1)) return;
    const int T = w.survPre[w.nnPre[n]];
    const int g0 = blockIdx.x * kSecBlock;
    if (g0 >= T) return;  // uniform per CTA
    const Window win = cta_window(w, L, T);
    const int g = g0 + threadIdx.x;
    bool act = g < T;
    int ks = 0, K = 0, p = 0;
    double dorg = 0.0, tau = 0.0;
    if (act) {  // warp-per-root tier owns split merges
        int a0, a1;
        active_range(w, L, w.aMerge[g], a0, a1);
        if (split_mode(L.mSize[w.aMerge[g]], a1 - a0)) act = false;
    }
    if (!__syncthreads_or(act)) return;
    if (act) {
        const int m = w.aMerge[g];
        int ke;
        active_range(w, L, m, ks, ke);
        K = ke - ks;
        const int j = g - ks;
        const int off = L.mOff[m], size = L.mSize[m];
        dorg = w.dA[w.org[g]];
        tau = w.tau[g];
        const double lam = dorg + tau;
        // parent position: j + #{deflated <= lam} = j + #{D <= lam} - #{dA <= lam}
        const int pos = j + count_leq(w.D + off, size, lam) - count_leq(w.dA + ks, K, lam);
        p = off + pos;
        w.lam[p] = lam;
        w.tau[g] = lam;  // tau, org are dead after these reads: k_deflated_out searches the
        w.org[g] = p;    // root values, the root-range split exchange finds the position
        if ((L.mFlags[m] & kMergeRoot) || !owns(w, g)) act = false;
    }
    double nn = 0.0, s0 = 0.0, s1 = 0.0;
    if (!__syncthreads_or(act)) return;
    const bool fast = act && !w.exact && eval_guard(GlobalPairs{w.dA + ks, w.z2A + ks}, K, g - ks, dorg, tau);
    for (int tlo = win.P0; tlo < win.P1; tlo += kWin) {
        const int thi = min(tlo + kWin, win.P1);
        __syncthreads();
        for (int r = tlo + threadIdx.x; r < thi; r += kSecBlock) {
            s_d[r - tlo] = w.dA[r];
            s_zh[r - tlo] = w.zA[r];
            s_r0[r - tlo] = w.r0A[r];
            s_r1[r - tlo] = w.r1A[r];
        }
        __syncthreads();
        if (fast) {
            const int ilo = max(ks, tlo) - tlo, ihi = min(ks + K, thi) - tlo;
#pragma unroll 4
            for (int t = ilo; t < ihi; ++t) {
                const double y = s_zh[t] * rcp_nr((s_d[t] - dorg) - tau);
                nn = __fma_rn(y, y, nn);
                s0 = __fma_rn(s_r0[t], y, s0);
                s1 = __fma_rn(s_r1[t], y, s1);
            }
        }
    }
    if (!act) return;
    if (!fast) {  // exact redo; a zero delta is an error
        const double* __restrict__ dA = w.dA + ks;
        const double* __restrict__ zh = w.zA + ks;
        const double* __restrict__ r0 = w.r0A + ks;
        const double* __restrict__ r1 = w.r1A + ks;
        bool zero = false;
        nn = 0.0; s0 = 0.0; s1 = 0.0;
        for (int i = 0; i < K; ++i) {
            const double del = (dA[i] - dorg) - tau;
            zero |= (del == 0.0);
            const double y = zh[i] * __drcp_rn(del);
            nn = __fma_rn(y, y, nn);
            s0 = __fma_rn(r0[i], y, s0);
            s1 = __fma_rn(r1[i], y, s1);
        }
        if (zero) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
    }
    const double inv = 1.0 / sqrt(nn);
    w.blo[p] = s0 * inv;
    w.bhi[p] = s1 * inv;
}

// deflated columns: parent position t + #{roots < D}
__global__ void k_deflated_out(Work w, LevelDev L, int n) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int m = find_merge(L, k);
    if (m < 0) return;
    const int q = w.nnPre[k];
    if (w.nnFlag[k] && w.survFlag[q]) return;  // survivor: placed by k_rows
    const int off = L.mOff[m];
    int ks, ke;
    active_range(w, L, m, ks, ke);
    const int K = ke - ks;
    const int t = (k - off) - (w.survPre[q] - ks);
    const double v = w.D[k];
    // #{roots j: lambda_j < v}; roots ascend (interlacing); the rows kernels
    // left lambda_j = d[org_j] + tau_j in tau[j]
    int lo = 0, hi = K;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const double lj = w.tau[ks + mid];
        if (lj < v) lo = mid + 1; else hi = mid;
    }
    const int p = off + t + lo;
    w.lam[p] = v;
    if (!(L.mFlags[m] & kMergeRoot)) {
        w.blo[p] = w.R0[k];
        w.bhi[p] = w.R1[k];
    }
}

// Secular-problem trace (brgpu_set_secular_trace): the level's active problem
// (dA, zA before the refreshed weights replace zA) and rho per merge.
__global__ void k_dump_active(Work w, LevelDev L, int n, double* __restrict__ out, double* __restrict__ rho) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int T = w.survPre[w.nnPre[n]];
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < T; g += gridDim.x * blockDim.x) {
        out[2 * g] = w.dA[g];
        out[2 * g + 1] = w.zA[g];
    }
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L.M; m += gridDim.x * blockDim.x)
        rho[m] = fabs(w.ew[L.mOff[m] + L.mNL[m] - 1]);
}

void launch_dump_active(cudaStream_t s, const Work& w, const LevelDev& L, int n, double* out, double* rho,
                        int* launches) {
    launch_pdl(k_dump_active, 64, 256, 0, s, w, L, n, out, rho);
    *launches += 1;
}

// per-merge (nn, K) for the trace
__global__ void k_level_trace(Work w, LevelDev L, int* __restrict__ out) {
    pdl_entry();
    if (!dense_entry(L)) return;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= L.M) return;
    const int off = L.mOff[m], end = off + L.mSize[m];
    const int a = w.nnPre[off], b = w.nnPre[end];
    out[2 * m] = b - a;
    out[2 * m + 1] = w.survPre[b] - w.survPre[a];
}

// ---------------------------------------------------------------------------
// rescale + cross-block merge
// ---------------------------------------------------------------------------
__global__ void k_rescale(int n, const int* __restrict__ bstart, int nblk,
                          const unsigned long long* __restrict__ sbits, double* __restrict__ lam) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = nblk == 1 ? 0 : find_block(bstart, nblk, i);
    const double s = block_scale_of(sbits[b]);
    lam[i] = lam[i] * s;
}

// one pass of a bottom-up stable merge sort over runs [rs[r], rs[r+1])
__global__ void k_merge_runs(int n, const double* __restrict__ src, double* __restrict__ dst,
                             const int* __restrict__ rs, int nruns) {
    pdl_entry();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = find_block(rs, nruns, i);
    const double v = src[i];
    const int pr = r ^ 1;
    const int pair0 = rs[r & ~1];
    if (pr >= nruns) { dst[i] = v; return; }
    const int ps = rs[pr], pn = rs[pr + 1] - ps;
    const int own = i - rs[r];
    const int other = (r & 1) ? count_leq(src + ps, pn, v) : count_less(src + ps, pn, v);
    dst[pair0 + own + other] = v;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static inline int cdiv(int a, int b) { return (a + b - 1) / b; }

void launch_secular_tiled(cudaStream_t s, const Work& w, const LevelDev& L, int n,
                          const SolveParams& prm);
int launch_secular_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm);
void launch_zhat_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm);
void launch_rows_warp(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm);

int selftest_rcp(long long count, unsigned long long seed, unsigned long long* host_bad) {
    unsigned long long* d;
    if (cudaMalloc(&d, sizeof(unsigned long long)) != cudaSuccess) return BRGPU_ERR_CUDA;
    cudaMemset(d, 0, sizeof(unsigned long long));
    k_selftest_rcp<<<(int)((count + 255) / 256), 256>>>(count, seed, d);
    cudaError_t e = cudaMemcpy(host_bad, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? BRGPU_OK : BRGPU_ERR_CUDA;
}

int sec_ctas_per_sm() { return BRGPU_SEC_MINB; }

void init_kernel_attributes() {
    cudaFuncSetAttribute(k_leaf<26>, cudaFuncAttributeMaxDynamicSharedMemorySize, leaf_smem_bytes<26>());
    cudaFuncSetAttribute(k_leaf<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, leaf_smem_bytes<32>());
}

void launch_copy_input(cudaStream_t s, int n, const double* d, const double* e, double* dw,
                       double* ew) {
    k_copy_input<<<cdiv(n, 256), 256, 0, s>>>(n, d, e, dw, ew);
}

void launch_scan_input(cudaStream_t s, int n, const double* d, const double* e, uint8_t* split,
                       int* nsplit, int* status) {
    k_scan_input<<<cdiv(n, 256), 256, 0, s>>>(n, d, e, split, nsplit, status);
}

void launch_scan_input_batched(cudaStream_t s, int batch, int n, const double* d, const double* e,
                               double* dw, double* ew, uint8_t* split, int* nsplit, int* status) {
    const int N = batch * n;
    k_scan_input_batched<<<cdiv(N, 256), 256, 0, s>>>(batch, n, d, e, dw, ew, split, nsplit, status);
}

#define PMARK(c) do { if (prof) prof_mark(prof, (void*)s, (c)); } while (0)

void launch_prepare(cudaStream_t s, int n, const int* bstart, int nblk, unsigned long long* sbits,
                    double* dw, double* ew, int ncut, const int* cutPos, int* launches, Prof* prof) {
    launch_pdl(k_block_scale, cdiv(n, 256), 256, 0, s, n, dw, ew, bstart, nblk, sbits);
    launch_pdl(k_apply_scale, cdiv(n, 256), 256, 0, s, n, bstart, nblk, sbits, dw, ew);
    *launches += 2;
    if (ncut > 0) {
        launch_pdl(k_cuts, cdiv(ncut, 256), 256, 0, s, ncut, cutPos, ew, dw);
        *launches += 1;
    }
    PMARK(BRGPU_K_PREPARE);
}

void launch_leaves(cudaStream_t s, int ntask, int maxm, const int* tOff, const int* tSize,
                   const int* tFlags, const Work& w, int* launches, Prof* prof) {
    if (ntask <= 0) return;
    // leaves per warp: fill ~4 warps per SM first, then pack up to 32 per warp
    int per_warp = 1;
    while (per_warp < 32 && (long long)ntask > (long long)per_warp * kLeafSpreadWarps) per_warp <<= 1;
    const int warps = cdiv(ntask, per_warp);
    const int grid = cdiv(warps * 32, kLeafThreads);
    if (maxm <= 16) {
        const size_t sm = leaf_smem_bytes<16>();
        launch_pdl(k_leaf<16>, grid, kLeafThreads, sm, s, ntask, tOff, tSize, tFlags, w.dw, w.ew, w.lam,
                                                  w.blo, w.bhi, w.status, per_warp);
    } else if (maxm <= 26) {
        const size_t sm = leaf_smem_bytes<26>();
        launch_pdl(k_leaf<26>, grid, kLeafThreads, sm, s, ntask, tOff, tSize, tFlags, w.dw, w.ew, w.lam,
                                                  w.blo, w.bhi, w.status, per_warp);
    } else {
        const size_t sm = leaf_smem_bytes<32>();
        launch_pdl(k_leaf<32>, grid, kLeafThreads, sm, s, ntask, tOff, tSize, tFlags, w.dw, w.ew, w.lam,
                                                  w.blo, w.bhi, w.status, per_warp);
    }
    *launches += 1;
    PMARK(BRGPU_K_LEAF);
}

// Root-range split exchange: a rank packs the results of the
// active indices it owns (g = k*P + r) into slot r of the gather buffers, the
// buffers are all-gathered in place (NCCL, or device copies for virtual
// ranks), and every rank unpacks the other slots.  kind 0: roots (tau, org);
// 1: refreshed weights; 2: boundary rows (at the parent position in org).
__global__ void k_xpack(Work w, int n, int kind, int c, double* __restrict__ xA, double* __restrict__ xB) {
    pdl_entry();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int T = w.survPre[w.nnPre[n]];
    const int g = k * w.own_P + w.own_r;
    if (k >= c || g >= T) return;
    const int slot = w.own_r * c + k;
    if (kind == 0) {
        xA[slot] = w.tau[g];
        xB[slot] = (double)w.org[g];
    } else if (kind == 1) {
        xA[slot] = w.zA[g];
    } else {
        const int p = w.org[g];
        xA[slot] = w.blo[p];
        xB[slot] = w.bhi[p];
    }
}

__global__ void k_xunpack(Work w, int n, int kind, int c, const double* __restrict__ xA,
                          const double* __restrict__ xB) {
    pdl_entry();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int P = w.own_P;
    if (idx >= P * c) return;
    const int rr = idx / c, k = idx - rr * c;
    const int T = w.survPre[w.nnPre[n]];
    const int g = k * P + rr;
    if (rr == w.own_r || g >= T) return;
    if (kind == 0) {
        w.tau[g] = xA[idx];
        w.org[g] = (int)xB[idx];
    } else if (kind == 1) {
        w.zA[g] = xA[idx];
    } else {
        const int p = w.org[g];
        w.blo[p] = xA[idx];
        w.bhi[p] = xB[idx];
    }
}

// One level of the grid tier, in four parts separated by the points where a
// root-range split exchanges results (prm.xsplit): 0 deflation + secular roots,
// 1 refreshed weights, 2 boundary rows + root placement, 3 deflated placement.
// Without a split the parts run back to back.
void launch_sigma_stage(cudaStream_t s, const Work& w, const LevelDev& L, const SigmaDev& sg, int maxSize,
                        int stage, int* launches);

void launch_level_part(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm,
                       int part, int* launches, Prof* prof) {
    const bool lane_tier = !L.allSplit;  // all merges > kSplitMinSize: warp tier only
    // merges of at most kSplitMinK elements can never reach the split rule
    // (size > kSplitMinSize or K > kSplitMinK): no warp-tier launches
    const bool warp_tier = L.maxSize > kSplitMinK;
    const bool x = prm.xsplit != 0;
    const int xg = cdiv(prm.xc, 256), xu = cdiv(prm.xc * w.own_P, 256);
    int nl = 0;
    if (part == 0) {
        const int ntiles = cdiv(n, kScanBlock);
        const int mtiles = cdiv(n, kMergeTile);  // >= ntiles
        // per-merge scales, tile states + tickets of the two single-pass scans
        // (mtiles + ntiles + 2 words) and the mode word: zeroed by a kernel so the
        // level's launches form one programmatic-dependency chain
        // a level without warp-tier merges needs no k_level_modes: its mode word is
        // the lane bit (the lane kernels exit on an empty level by its root count)
        launch_pdl(k_level_zero, cdiv(max(L.M, mtiles + ntiles + 2), 256), 256, 0, s, L, w.scanState,
                   mtiles + ntiles + 2, w.levelModes, warp_tier ? 0 : 1);
        unsigned long long* st1 = w.scanState;
        unsigned long long* st2 = w.scanState + mtiles;
        int* tk = reinterpret_cast<int*>(w.scanState + mtiles + ntiles);
        launch_pdl(k_merge_prep, cdiv(mtiles, kPrepVec), kMergeTile, 0, s, w, L, n, w.org);  // org: free until the secular pass
        PMARK(BRGPU_K_SCATTER);
        launch_pdl(k_merge_nn, mtiles, kMergeTile, 0, s, w, L, n, prm.tol_scale, w.org, st1, tk);
        PMARK(BRGPU_K_NNFLAG);
        if (prm.sigma) launch_sigma_stage(s, w, L, *prm.sigma, L.maxSize, 0, &nl);
        launch_pdl(k_segment_walk, min(cdiv(n, 256), prm.sms * 8), 256, 0, s, w, L, n, prm.tol_scale);
        PMARK(BRGPU_K_WALK);
        launch_pdl(k_surv_scan, min(ntiles, prm.sms * 2), kScanBlock, 0, s, w, L, n, st2, tk + 1);
        PMARK(BRGPU_K_SURVWRITE);
        if (prm.sigma) launch_sigma_stage(s, w, L, *prm.sigma, L.maxSize, 1, &nl);
        nl += 4;
        if (lane_tier) {
            if (warp_tier) { launch_pdl(k_level_modes, cdiv(L.M, 256), 256, 0, s, w, L); ++nl; }
            // CTAs per SM (= the launch bounds' minimum and the grid): 4 on levels up to
            // 2M elements (random 2^20 4.52 -> 4.46 ms), 6 on larger batched levels
            // (4096 x 1024: 12.12 -> 11.67 ms at 6)
            // (k_secular_tiled takes the same chunks: same grid)
            SolveParams ps = prm;
            if (n >= kSecBigLevel) {
                ps.sec_grid = prm.sms * BRGPU_SEC_MINB;
                launch_pdl(k_secular<BRGPU_SEC_MINB>, ps.sec_grid, kSecBlock, 0, s, w, L, n, prm.patched);
            } else {
                ps.sec_grid = prm.sms * kSecMinbSmall;
                launch_pdl(k_secular<kSecMinbSmall>, ps.sec_grid, kSecBlock, 0, s, w, L, n, prm.patched);
            }
            launch_secular_tiled(s, w, L, n, ps);
            nl += 2;
        }
        if (warp_tier) nl += launch_secular_warp(s, w, L, n, prm);
        if (x) { launch_pdl(k_xpack, xg, 256, 0, s, w, n, 0, prm.xc, prm.xA, prm.xB); ++nl; }
        PMARK(BRGPU_K_SECULAR);
    } else if (part == 1) {
        if (x) { launch_pdl(k_xunpack, xu, 256, 0, s, w, n, 0, prm.xc, prm.xA, prm.xB); ++nl; }
        if (prm.zhat) {
            if (lane_tier) { launch_pdl(k_zhat, cdiv(n, kSecBlock), kSecBlock, 0, s, w, L, n); ++nl; }
            if (warp_tier) { launch_zhat_warp(s, w, L, n, prm); ++nl; }
            if (x) { launch_pdl(k_xpack, xg, 256, 0, s, w, n, 1, prm.xc, prm.xA, prm.xB); ++nl; }
            PMARK(BRGPU_K_ZHAT);
        }
    } else if (part == 2) {
        if (x && prm.zhat) { launch_pdl(k_xunpack, xu, 256, 0, s, w, n, 1, prm.xc, prm.xA, prm.xB); ++nl; }
        // requested rows need the roots (tau, org) that the rows kernels overwrite
        if (prm.sigma) launch_sigma_stage(s, w, L, *prm.sigma, L.maxSize, 2, &nl);
        if (lane_tier) { launch_pdl(k_rows, cdiv(n, kSecBlock), kSecBlock, 0, s, w, L, n); ++nl; }
        if (warp_tier) { launch_rows_warp(s, w, L, n, prm); ++nl; }
        if (x) { launch_pdl(k_xpack, xg, 256, 0, s, w, n, 2, prm.xc, prm.xA, prm.xB); ++nl; }
        PMARK(BRGPU_K_ROWS);
    } else {
        if (x) { launch_pdl(k_xunpack, xu, 256, 0, s, w, n, 2, prm.xc, prm.xA, prm.xB); ++nl; }
        launch_pdl(k_deflated_out, cdiv(n, 256), 256, 0, s, w, L, n);
        ++nl;
        PMARK(BRGPU_K_DEFLATED);
    }
    *launches += nl + (part == 0 ? 1 : 0);  // + k_level_zero
}

// Does a split level exchange after `part` (and which arrays: 1 = xA, 2 = xA + xB)?
int level_exchange_arrays(const SolveParams& prm, int part) {
    if (!prm.xsplit) return 0;
    if (part == 0) return 2;             // roots: tau, org
    if (part == 1) return prm.zhat ? 1 : 0;  // refreshed weights
    if (part == 2) return 2;             // rows: blo, bhi
    return 0;
}

void launch_level(cudaStream_t s, const Work& w, const LevelDev& L, int n,
                  const SolveParams& prm, int* launches, Prof* prof) {
    for (int part = 0; part < 4; ++part) launch_level_part(s, w, L, n, prm, part, launches, prof);
}

void launch_level_trace(cudaStream_t s, const Work& w, const LevelDev& L, int n, int* out,
                        int* launches, Prof* prof) {
    (void)n;
    launch_pdl(k_level_trace, cdiv(L.M, 128), 128, 0, s, w, L, out);
    *launches += 1;
    PMARK(BRGPU_K_TRACE);
}

void launch_finish(cudaStream_t s, int n, const int* bstart, int nblk,
                   const unsigned long long* sbits, double* lam, int* launches, Prof* prof) {
    launch_pdl(k_rescale, cdiv(n, 256), 256, 0, s, n, bstart, nblk, sbits, lam);
    *launches += 1;
    PMARK(BRGPU_K_FINISH);
}

void launch_merge_runs(cudaStream_t s, int n, const double* src, double* dst, const int* rs,
                       int nruns, int* launches, Prof* prof) {
    launch_pdl(k_merge_runs, cdiv(n, 256), 256, 0, s, n, src, dst, rs, nruns);
    *launches += 1;
    PMARK(BRGPU_K_FINISH);
}

}  // namespace brgpu
