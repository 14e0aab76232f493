// internal.hpp -- structures shared by the host planner (api.cpp) and the
// sm_100a kernels (kernels.cu).  Positions are int32 (n < 2^31).
#pragma once

#include <cstdint>

#include "brgpu.h"

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#endif
#endif

namespace brgpu {

// Tile width used to map a position to the merge containing it: tileFirst[t]
// is the first merge (of a level) that ends after position t*kTile.
constexpr int kTile = 256;

// Merge flags.
constexpr int kMergeRoot = 1;   // block root: root-only mode

// Device-resident workspace (all arrays sized for the reserved capacity).
// Doubles: dw, ew, lam, blo, bhi, D, Z, R0, R1, dA, zA, z2A, r0A, r1A, tau  (15n)
// Ints   : nnPre(n+1), nnPos, survPre(n+1), aMerge, org, + byte flags (~5.5n)
struct Work {
    double* dw;      // scaled, Cuppen-cut diagonal
    double* ew;      // scaled off-diagonal
    double* lam;     // node eigenvalues (ascending per node); final output
    double* blo;     // node first eigenvector row
    double* bhi;     // node last eigenvector row
    double* D;       // merged (sorted) poles
    double* Z;       // merged z (rotated in place by close-pole deflation)
    double* R0;      // merged first selected row
    double* R1;      // merged last selected row
    double* dA;      // compacted active poles (global active index)
    double* zA;      // compacted active weights; replaced by z-hat
    double* z2A;     // zA^2
    double* r0A;
    double* r1A;
    double* tau;     // root offsets
    int* nnPre;      // exclusive prefix of non-negligible flags over positions (n+1)
    int* nnPos;      // NN index -> sorted position
    int* survPre;    // exclusive prefix of survivor flags over NN indices (n+1)
    int* aMerge;     // active index -> merge id (within level)
    int* org;        // root origin (level-global active pole index; k_rows reuses it for the parent position)
    uint8_t* nnFlag;
    uint8_t* survFlag;
    int* tileCnt;    // per-1024 tile counts (scan scratch)
    int* tileOff;
    int* status;     // first error code
    unsigned long long* scanState;  // look-back tile states (2*ntiles) + 2 tickets
    int* levelModes;  // bit0: level has lane-per-root merges, bit1: warp-per-root merges
    unsigned long long* counters;  // [0] evals
    int exact;       // test hook (BRGPU_OPT_EXACT_PASSES): every pole pass takes the exact path
    // root-range split of the shared top merges: this rank
    // solves the roots (and refreshed weights, boundary rows) of the active
    // indices g with g % own_P == own_r; 1/0 outside split levels
    int own_P, own_r;
};

// One level's merges (device pointers into the plan arrays).
struct LevelDev {
    const int* mOff;
    const int* mSize;
    const int* mNL;
    const int* mFlags;
    unsigned long long* mTol;  // max(|D|,|z|) bits per merge (atomicMax)
    const int* tileFirst;      // ceil(n/kTile)+1 entries
    int M;
    int allSplit;              // every merge of the level is larger than kSplitMinSize (warp tier only)
    int maxSize;               // largest merge of the level
    // Level control words of a sparse-capable level (sparse.cu): ctl[1] = largest
    // non-negligible count of a merge (k_sp_flag), ctl[2] = k_sp_flag's
    // grid-barrier counter, ctl[3] = the level's total non-negligible count.
    int* ctl;
    int spCap;        // this level's sparse cap C: sparse iff every merge has NN <= C (0: dense only)
    int spStatic;     // every merge has size <= C: sparse always, no dense kernels launched
    int spSpan;       // k_sp_solve group key span (host-chosen from the previous solve's profile)
    // per-merge sparse tables (level-local merge index)
    int* spCs;        // compacted start of the merge's non-negligible entries
    int* spCsR;       // ... of its right-child entries
    int* spNN;        // non-negligible count
    int* spK;         // active rank K
    int* spGroup;     // k_sp_solve group starts (first merge of group g)
    int* spTileM;     // k_sp_place tile records (k_sp_flag): merge at each tile start (-1: none) ...
    int* spTileSplit; // ... and the merge-path split there (left elements before the tile start)
};

// Requested eigenvector rows (Algorithm 1's sigma, sigma.cu).  Per requested
// row r: S = the row in the current nodes' eigenvalue order (node positions),
// X = merged order, XA = active order; each nsel x stride doubles.
struct SigmaDev {
    int nsel;
    long long stride;
    const int* sel;  // global row index per request
    double* S;
    double* X;
    double* XA;
    double* Z0;      // merged z before the close-pole walk (stride doubles)
};

// Live-list tier (live.cu): the top levels of a large single-block solve keep,
// per node, only the elements with a boundary-row entry above the deflation
// threshold ("live"), sorted, at the start of the node's position range; the
// other ("dead") eigenvalues go to a pool, summarised per node by three maxima.
// Per-node words are indexed by the node's first position.
struct LiveDev {
    int* cnt;        // live count per node
    double* dLam;    // max |lambda| of the node's dead elements
    double* dBlo;    // max |first row| of the node's dead elements
    double* dBhi;    // max |last row| of the node's dead elements
    double* pool;    // dead eigenvalues, then the root's list (n values, any order)
    double* tmp;     // bucket-sort scatter buffer (n)
    int* bcount;     // bucket counts (nb), bucket starts (nb + 1)
    int* bcur;       // bucket cursors (nb)
    int* ctl;        // [0] pool fill (one block), [1] fallback (redo the solve on the dense tiers)
    unsigned long long* keys;  // [0] ~min key, [1] max key of the pool (order-preserving)
    int nb;          // buckets of the final sort
    // blocks (irreducible blocks / batch matrices): block b's pool is
    // pool[bstart[b] ..), filled through bctr[b] (one block: bctr = ctl)
    const int* bstart;
    int nblk;
    int* bctr;
};

// The top levels of the live tier as one dataflow launch (k_live_top): CTA b
// solves merge b - first[l] of level l once its two children (merges of level
// l - 1, or nodes completed before the launch) have set their done words.
constexpr int kMaxLiveTop = 16;
struct LiveRun {
    LevelDev L[kMaxLiveTop];
    int* trace[kMaxLiveTop];
    int first[kMaxLiveTop + 1];  // CTA offset of each level
    int nlev;
    int* done;                   // one word per merge of the run (zeroed per solve)
    // lane-mode dataflow run (k_live_flow): work items (level, first merge, merges)
    // in level order, taken by ticket, so an item only waits on lower tickets
    const int4* items = nullptr;
    int nitems = 0;
    int* ticket = nullptr;       // zeroed per solve
};

// A run of consecutive fused levels launched as one kernel (k_levels_fused).
constexpr int kMaxFusedRun = 8;
struct FusedRun {
    LevelDev L[kMaxFusedRun];
    int* trace[kMaxFusedRun];
    int nlev;
};

// Optional per-kernel profiling (brgpu_profile_kernels): the launchers call
// prof_mark after every launch; api.cpp records a CUDA event per mark.
struct Prof;
void prof_mark(Prof* p, void* stream, int cls);

struct SolveParams {
    int n;
    int zhat;
    int patched;
    double tol_scale;
    int sec_grid;  // CTAs of the secular kernel (fills the GPU; chunks adapt to the root count)
    int sms;       // SM count (grid sizing of the warp tier)
    // root-range split exchange: results of owned indices are packed into slot
    // own_r (xc entries) of the gather buffers xA/xB, which are all-gathered in place
    int xsplit;
    int xc;
    double* xA;
    double* xB;
    const SigmaDev* sigma;  // requested rows (grid tier only), or null
};

}  // namespace brgpu
