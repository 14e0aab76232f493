// sigma.cu -- requested eigenvector rows (Algorithm 1's sigma; SPEC.md:317-337,
// PAPER.md:1786, 1799-1817): besides the eigenvalues, rows Q(sigma_r, :) of the
// eigenvector matrix of T for any list of row indices (duplicates, any order).
//
// The rows ride on the grid tier of the level pipeline (kernels.cu): the
// planner runs every level through it (no fused SMEM levels) and keeps the
// block roots out of root-only mode, so each merge leaves its merged order,
// deflation groups, active problem, roots and refreshed weights in the level-
// global arrays.  Four kernels per level then carry each requested row:
//   k_sig_gather  after k_merge_nn:    child row -> merged order (the other
//                                      child's columns are 0: split_row_request)
//   k_sig_group   after k_surv_scan:   close-pole group rotations (the checker's
//                                      group_member), active compaction
//   k_sig_out     after the refreshed weights: R_parent(r, j) = R_child(r,:) y_j
//                                      for the roots, deflated columns passed
//                                      through, both at their parent positions
// plus k_sig_leaf (leaf QL/QR tracking row sigma_r) and k_sig_final (block
// columns -> global eigenvalue order).  Storage per requested row is one
// n-vector per stage (S: node rows, X: merged order, XA: active order), the
// O(|sigma| n) of PAPER.md:1799-1817.  Arithmetic = the checker's
// bro_eigvals_rows (oracle/br_oracle.c), bit for bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.hpp"
#include "launch.cuh"
#include "numerics.cuh"

namespace brgpu {

namespace {

__device__ __forceinline__ int sig_find_merge(const LevelDev& L, int p) {
    const int t = p / kTile;
    int m = L.tileFirst[t];
    const int last = L.tileFirst[t + 1] < L.M ? L.tileFirst[t + 1] : L.M - 1;
    while (m < last && L.mOff[m + 1] <= p) ++m;
    if (m >= L.M || m < 0) return -1;
    const int off = L.mOff[m];
    if (p < off || p >= off + L.mSize[m]) return -1;
    return m;
}

constexpr int kSigLeafThreads = 32;

// Leaf (or block <= cutoff) of row sigma_r: the leaf QL/QR of kernels.cu
// (steqr_leaf, same sweeps and shifts) tracking e_{sigma_r - off}, then the
// leaf's stable ascending order (qrql.cpp:348-364).
template <int MAXM>
__global__ void __launch_bounds__(kSigLeafThreads) k_sig_leaf(SigmaDev sg, const int* __restrict__ taskOf,
                                                              const int* __restrict__ tOff,
                                                              const int* __restrict__ tSize,
                                                              const double* __restrict__ dw,
                                                              const double* __restrict__ ew, int* status) {
    pdl_entry();
    extern __shared__ double sig_sm[];
    const int r = blockIdx.x * kSigLeafThreads + threadIdx.x;
    if (r >= sg.nsel) return;
    const int t = taskOf[r];
    const int off = tOff[t], m = tSize[t];
    const int row = sg.sel[r] - off;
    constexpr int S = kSigLeafThreads;
    const Strided<S> d{sig_sm + threadIdx.x};
    const Strided<S> e{sig_sm + MAXM * S + threadIdx.x};
    const Strided<S> x{sig_sm + (2 * MAXM - 1) * S + threadIdx.x};
    const Strided<S> y{sig_sm + (3 * MAXM - 1) * S + threadIdx.x};
    for (int i = 0; i < m; ++i) {
        d[i] = dw[off + i];
        if (i + 1 < m) e[i] = ew[off + i];
        x[i] = i == row ? 1.0 : 0.0;
        y[i] = 0.0;
    }
    const int st = steqr_leaf<true>(m, d, e, x, y);
    if (st) set_status(status, st);
    double* Sr = sg.S + (long long)r * sg.stride;
    for (int i = 0; i < m; ++i) {
        const double di = d[i];
        int rank = 0;
        for (int j = 0; j < m; ++j) rank += (d[j] < di) || (j < i && d[j] == di);
        Sr[off + rank] = x[i];
    }
}

// Child row -> merged order.  Thread u owns child element off+u; its merged
// position is the stable-merge rank k_merge_nn gives it.  Also keeps the
// merged z (before the close-pole walk rotates it) for k_sig_group.
__global__ void k_sig_gather(Work w, LevelDev L, SigmaDev sg) {
    pdl_entry();
    const int r = blockIdx.y;
    const int i = sg.sel[r];
    const int m = sig_find_merge(L, i);
    if (m < 0) return;
    const int off = L.mOff[m], size = L.mSize[m], nl = L.mNL[m];
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= size) return;
    const double* la = w.lam + off;
    const bool left = u < nl;
    const double v = la[u];
    const int sp = left ? u + count_less(la + nl, size - nl, v) : (u - nl) + count_leq(la, nl, v);
    const bool mine = left == (i < off + nl);
    sg.X[(long long)r * sg.stride + off + sp] = mine ? sg.S[(long long)r * sg.stride + off + u] : 0.0;
    sg.Z0[off + u] = w.Z[off + u];
}

// Close-pole groups (k_segment_walk's groups: a survivor followed by its
// members in NN order) applied to the requested row, then the survivors'
// values compacted into the active order.
__global__ void k_sig_group(Work w, LevelDev L, SigmaDev sg) {
    pdl_entry();
    const int r = blockIdx.y;
    const int m = sig_find_merge(L, sg.sel[r]);
    if (m < 0) return;
    const int off = L.mOff[m], size = L.mSize[m];
    const int qs = w.nnPre[off], qe = w.nnPre[off + size];
    const int q = qs + blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= qe || !w.survFlag[q]) return;
    double* X = sg.X + (long long)r * sg.stride;
    const int k = w.nnPos[q];
    double x = X[k];
    if (q + 1 < qe && !w.survFlag[q + 1]) {
        const double zs = sg.Z0[k];
        double Q = zs * zs, S = zs * x;
        for (int q2 = q + 1; q2 < qe && !w.survFlag[q2]; ++q2) {
            const int k2 = w.nnPos[q2];
            const double zk = sg.Z0[k2], xk = X[k2];
            double xm = xk, unused = 0.0;
            group_member(Q, S, S, zk, xm, unused);
            X[k2] = xm;
            Q = Q + zk * zk;
            S = S + zk * xk;
        }
        const double R = sqrt(Q), iR = 1.0 / R;
        x = S * iR;
        X[k] = x;
    }
    sg.XA[(long long)r * sg.stride + w.survPre[q]] = x;
}

// Parent row: thread u computes root j = u (if u < K) and places merged
// column off+u if it was deflated.  Roots: y_j = zhat / Delta_j streamed in
// pole order, R(r, j) = <x, y_j> / ||y_j|| (the checker's sigma_root_row);
// positions as k_rows / k_deflated_out.
__global__ void k_sig_out(Work w, LevelDev L, SigmaDev sg) {
    pdl_entry();
    const int r = blockIdx.y;
    const int m = sig_find_merge(L, sg.sel[r]);
    if (m < 0) return;
    const int off = L.mOff[m], size = L.mSize[m];
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= size) return;
    const int ks = w.survPre[w.nnPre[off]], ke = w.survPre[w.nnPre[off + size]];
    const int K = ke - ks;
    double* Sr = sg.S + (long long)r * sg.stride;
    const double* X = sg.X + (long long)r * sg.stride;
    const double* XA = sg.XA + (long long)r * sg.stride + ks;
    const double* dA = w.dA + ks;
    if (u < K) {
        const int g = ks + u;
        const double dorg = w.dA[w.org[g]], tau = w.tau[g];
        const double lam = dorg + tau;
        const int pos = u + count_leq(w.D + off, size, lam) - count_leq(dA, K, lam);
        const double* zh = w.zA + ks;
        double nn = 0.0, s = 0.0;
        bool zero = false;
        for (int i = 0; i < K; ++i) {
            const double del = (dA[i] - dorg) - tau;
            zero |= del == 0.0;
            const double y = zh[i] * (1.0 / del);
            nn = __fma_rn(y, y, nn);
            s = __fma_rn(XA[i], y, s);
        }
        if (zero) set_status(w.status, BRGPU_ERR_ZERO_DENOMINATOR);
        Sr[off + pos] = s * (1.0 / sqrt(nn));
    }
    const int k = off + u;
    const int q = w.nnPre[k];
    if (w.nnFlag[k] && w.survFlag[q]) return;  // survivor: its column became a root
    const int t = u - (w.survPre[q] - ks);
    const double v = w.D[k];
    int lo = 0, hi = K;  // #{roots j: lambda_j < v}
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int g = ks + mid;
        if (w.dA[w.org[g]] + w.tau[g] < v) lo = mid + 1; else hi = mid;
    }
    Sr[off + t + lo] = X[k];
}

// Block columns -> global order: element i of block b lands at its stable
// rank over the rescaled block spectra (the order of the cross-block merge
// passes, left-first ties); columns of other blocks stay 0.
__global__ void k_sig_final(SigmaDev sg, const double* __restrict__ lam, const int* __restrict__ bstart,
                            int nblk, const int* __restrict__ blkOf, double* __restrict__ out, int n) {
    pdl_entry();
    const int r = blockIdx.y;
    const int b = blkOf[r];
    const int i = bstart[b] + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= bstart[b + 1]) return;
    const double v = lam[i];
    int pos = i - bstart[b];
    for (int c = 0; c < nblk; ++c) {
        if (c == b) continue;
        const int o = bstart[c], sz = bstart[c + 1] - o;
        pos += c < b ? count_leq(lam + o, sz, v) : count_less(lam + o, sz, v);
    }
    out[(long long)r * n + pos] = sg.S[(long long)r * sg.stride + i];
}

int cdiv(int a, int b) { return (a + b - 1) / b; }

}  // namespace

void launch_sigma_leaves(cudaStream_t s, const SigmaDev& sg, int maxm, const int* taskOf, const int* tOff,
                         const int* tSize, const Work& w, int* launches) {
    if (sg.nsel <= 0) return;
    const int grid = cdiv(sg.nsel, kSigLeafThreads);
    if (maxm <= 16)  // leaf cutoff <= 32 (BRGPU_OPT_LEAF_CUTOFF): 32 KiB of SMEM at most
        launch_pdl(k_sig_leaf<16>, grid, kSigLeafThreads, (size_t)4 * 16 * kSigLeafThreads * 8, s, sg, taskOf,
                   tOff, tSize, w.dw, w.ew, w.status);
    else
        launch_pdl(k_sig_leaf<32>, grid, kSigLeafThreads, (size_t)4 * 32 * kSigLeafThreads * 8, s, sg, taskOf,
                   tOff, tSize, w.dw, w.ew, w.status);
    ++*launches;
}

// stage 0: after k_merge_nn; 1: after k_surv_scan; 2: after the refreshed weights
void launch_sigma_stage(cudaStream_t s, const Work& w, const LevelDev& L, const SigmaDev& sg, int maxSize,
                        int stage, int* launches) {
    if (sg.nsel <= 0) return;
    const dim3 grid(cdiv(maxSize, 256), sg.nsel);
    if (stage == 0) launch_pdl(k_sig_gather, grid, 256, 0, s, w, L, sg);
    else if (stage == 1) launch_pdl(k_sig_group, grid, 256, 0, s, w, L, sg);
    else launch_pdl(k_sig_out, grid, 256, 0, s, w, L, sg);
    ++*launches;
}

void launch_sigma_final(cudaStream_t s, const SigmaDev& sg, const double* lam, const int* bstart, int nblk,
                        const int* blkOf, int maxBlock, double* out, int n, int* launches) {
    if (sg.nsel <= 0) return;
    const dim3 grid(cdiv(maxBlock, 256), sg.nsel);
    launch_pdl(k_sig_final, grid, 256, 0, s, sg, lam, bstart, nblk, blkOf, out, n);
    ++*launches;
}

}  // namespace brgpu
