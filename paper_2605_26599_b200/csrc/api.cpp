// api.cpp -- C ABI (include/brgpu.h), handle, workspace ledger and the host
// planner of the B200 BR solver.
//
// Host responsibilities (everything O(#nodes), never O(n) per solve once the
// plan is cached):
//   * irreducible-block plan (tridiagonal.cpp:45-58): the device flags split
//     points (k_scan_input); the host receives only their count, and the flag
//     array when it is non-zero;
//   * split trees per block (merge_tree.cpp:34-60), Cuppen cut list
//     (merge_tree.cpp:78-92), leaf tasks, per-level merge tables;
//   * the launch sequence (optionally replayed as one CUDA graph).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen'ed (torch's copy when already loaded)

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "internal.hpp"

namespace brgpu {

// kernels.cu
void launch_scan_input(cudaStream_t s, int n, const double* d, const double* e, uint8_t* split,
                       int* nsplit, int* status);
void launch_scan_input_batched(cudaStream_t s, int batch, int n, const double* d, const double* e,
                               double* dw, double* ew, uint8_t* split, int* nsplit, int* status);
void launch_copy_input(cudaStream_t s, int n, const double* d, const double* e, double* dw, double* ew);
void launch_prepare(cudaStream_t s, int n, const int* bstart, int nblk, unsigned long long* sbits,
                    double* dw, double* ew, int ncut, const int* cutPos, int* launches, Prof* prof);
void launch_leaves(cudaStream_t s, int ntask, int maxm, const int* tOff, const int* tSize,
                   const int* tFlags, const Work& w, int* launches, Prof* prof);
void launch_level(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm,
                  int* launches, Prof* prof);
void launch_level_part(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm,
                       int part, int* launches, Prof* prof);
int level_exchange_arrays(const SolveParams& prm, int part);
void launch_level_trace(cudaStream_t s, const Work& w, const LevelDev& L, int n, int* out,
                        int* launches, Prof* prof);
void launch_level_sparse(cudaStream_t s, const Work& w, const LevelDev& L, int n, const SolveParams& prm,
                         int* blockCnt, int* traceOut, int* launches, Prof* prof);
void init_sparse_attributes();
void launch_dump_active(cudaStream_t s, const Work& w, const LevelDev& L, int n, double* out, double* rho,
                        int* launches);
int sparse_cap();
int sparse_groups_max(int n, int M, int span);
int sparse_min_merge();
int sparse_flag_grid(int n, int sms);
void launch_finish(cudaStream_t s, int n, const int* bstart, int nblk,
                   const unsigned long long* sbits, double* lam, int* launches, Prof* prof);
void launch_merge_runs(cudaStream_t s, int n, const double* src, double* dst, const int* rs,
                       int nruns, int* launches, Prof* prof);
void launch_level_fused(cudaStream_t s, const Work& w, const LevelDev& L, int ngroups, int cap,
                        const int* gFirst, const int* gCount, const SolveParams& prm, int* traceOut,
                        int* launches, Prof* prof);
void launch_levels_fused(cudaStream_t s, const Work& w, const FusedRun& run, int ngroups, const int2* tab,
                         const SolveParams& prm, int* launches, Prof* prof);
void init_fused_attributes();
void init_warp_attributes();
void launch_live_init(cudaStream_t s, const Work& w, const LiveDev& V, const int2* front, int nfront,
                      double tol_scale, int* launches, Prof* prof);
void launch_level_live(cudaStream_t s, const Work& w, const LevelDev& L, const LiveDev& V,
                       const SolveParams& prm, int* traceOut, int* launches, Prof* prof);
void launch_live_sort(cudaStream_t s, const LiveDev& V, int n, double* out, int sms, int* launches, Prof* prof);
void launch_live_top(cudaStream_t s, const Work& w, const LiveRun& R, const LiveDev& V, const SolveParams& prm,
                     int* launches, Prof* prof);
int live_top_capacity(int sms);
int live_lane_group(int M, int sms);
void launch_live_flow(cudaStream_t s, const Work& w, const LiveRun& R, const LiveDev& V, const SolveParams& prm,
                      int* launches, Prof* prof);
int live_cluster_max(int device);
int live_cluster_size(int device, int M, int cmax);
void launch_level_live_cluster(cudaStream_t s, const Work& w, const LevelDev& L, const LiveDev& V,
                               const SolveParams& prm, int* traceOut, int C, int* launches, Prof* prof);
int live_block_cap();
void launch_live_blocksort(cudaStream_t s, const LiveDev& V, const int* blocks, int nlive, double* out,
                           int* launches, Prof* prof);
int live_buckets(int n);
void init_live_attributes();
// Live-list tier (live.cu): single-block solves of at least kLiveMinN elements
// run every level above the last fused / small one on live lists when all those
// levels' merges are >= kLiveMinSize (random 2^20: levels 5..16).  512 since the
// lane levels run as one dataflow launch (C5 -0.015 ms against 1024; 256 +0.03 ms)
#ifndef BRGPU_LIVE_MIN_SIZE
#define BRGPU_LIVE_MIN_SIZE 512
#endif
constexpr int kLiveMinSize = BRGPU_LIVE_MIN_SIZE;
constexpr int kLiveMinN = 1 << 15;
constexpr int kRetryDense = 1000;  // internal: the live tier fell back, redo the solve densely
constexpr int kLiveBackoff0 = 64;  // dense solves of an order after its first live-tier fallback
// work counters (Work::counters): [0,1] grid-tier evaluations / pole terms, [2,3]
// fused tier, [4..7] phase cycles of profiling builds, [8,9] live tier
constexpr int kCounters = 12;
#ifndef BRGPU_FUSE_MAX_ELEMS
#define BRGPU_FUSE_MAX_ELEMS 1024
#endif
constexpr int kFuseMaxElems = BRGPU_FUSE_MAX_ELEMS;
constexpr int kGridMinN = 32768;  // below this order, underfilled 1024-shape levels stay fused
constexpr int kGridManyPerSm = 4;  // 1024-shape levels with >= 4 merges per SM run on the grid tier
#ifndef BRGPU_GRID_MANY_MIN_SIZE
#define BRGPU_GRID_MANY_MIN_SIZE 128
#endif
constexpr int kGridManyMinSize = BRGPU_GRID_MANY_MIN_SIZE;  // ... when their merges exceed this size  // largest merge of a fused SMEM level (512 or 1024)
constexpr int kFuseSmallElems = 512;  // small fused shape (fused.cu)
constexpr int kSpMinSpan = 16;        // smallest k_sp_solve group key span (group table size)
#ifndef BRGPU_SPLIT_MIN_SIZE
#define BRGPU_SPLIT_MIN_SIZE 8192
#endif
#ifndef BRGPU_LIVE_FLOW_GMAX
#define BRGPU_LIVE_FLOW_GMAX 4
#endif
constexpr int kLiveFlowGMax = BRGPU_LIVE_FLOW_GMAX;  // merges per dataflow work item (cap)
constexpr int kSplitMinSizeHost = BRGPU_SPLIT_MIN_SIZE;  // == kSplitMinSize (numerics.cuh): warp-per-root merges
constexpr int kFuseMaxMergesHost = 128;
// A fused level with fewer merges than this many per SM x SMs gives every merge
// its own CTA (one merge's roots per 256 lanes instead of a group's) and runs as
// its own launch: small solves are bound by the per-level latency of a CTA's
// root queue (n = 4096: 8 CTAs for levels 1-5 as one run)
#ifndef BRGPU_FEW_MERGES_PER_SM
#define BRGPU_FEW_MERGES_PER_SM 1
#endif
constexpr int kFewMergesPerSm = BRGPU_FEW_MERGES_PER_SM;

void init_kernel_attributes();
void launch_sigma_leaves(cudaStream_t s, const SigmaDev& sg, int maxm, const int* taskOf, const int* tOff,
                         const int* tSize, const Work& w, int* launches);
void launch_sigma_final(cudaStream_t s, const SigmaDev& sg, const double* lam, const int* bstart, int nblk,
                        const int* blkOf, int maxBlock, double* out, int n, int* launches);
int sec_ctas_per_sm();
int selftest_rcp(long long count, unsigned long long seed, unsigned long long* host_bad);

struct Prof {
    std::vector<cudaEvent_t> ev;
    std::vector<int> cls;
};

void prof_mark(Prof* p, void* stream, int cls) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, (cudaStream_t)stream);
    p->ev.push_back(e);
    p->cls.push_back(cls);
}

}  // namespace brgpu

using namespace brgpu;

namespace {

const char* kVersion = "brgpu 0.1 sm_100a fp64 (--fmad=false)";

struct LevelHost {
    int level;
    int m0;      // first merge index (global across levels)
    int M;       // merges at this level
    int tile0;   // offset of this level's tileFirst table
    bool fused;  // all merges <= kFuseMaxElems: one fused SMEM launch (fused.cu)
    int g0, G;   // groups of the fused launch
    int cap;     // group capacity (elements): 512 (small shape) or 1024
    int minSize; // smallest merge of the level
    int maxSize; // largest merge of the level
    int sp = 0;        // sparse-capable grid level (sparse.cu; device-side decision)
    int spStatic = 0;  // every merge <= the sparse cap: sparse always, no dense kernels
    int spCap = 0;     // sparse iff every merge has NN <= spCap
    int spSpan = 0;    // k_sp_solve group key span
    int ctl = 0;       // index of the level's control words (4 ints)
    bool live = false; // live-list level (live.cu)
};

struct Plan {
    int n = 0;
    int cutoff = 0;
    std::vector<int> bstart;  // blocks (nblk + 1)
    std::vector<int> segs;    // segment (matrix) boundaries for the final merge
    // host tables
    std::vector<int> tOff, tSize, tFlags;
    std::vector<int> cutPos;
    std::vector<int> mOff, mSize, mNL, mFlags, mLevel;
    std::vector<int> tileFirst;
    std::vector<int> gFirst, gCount;  // fused groups (level-local first merge, count)
    // runs of consecutive small-shape fused levels launched as one kernel:
    // (first level index in `levels`, level count, groups, offset in mlTab)
    struct MultiRun { int lev0, nlev, G, tab0; };
    std::vector<MultiRun> multi;
    std::vector<int> mlTab;           // (first, count) per (group, level), level-local
    int2* d_mlTab = nullptr;
    std::vector<LevelHost> levels;    // phase 1: merges owned by this rank (all, when nranks == 1)
    std::vector<LevelHost> levels2;   // phase 2: top merges shared by all ranks (after the exchange)
    int nranks = 1, rank = 0;
    // owned[k] = ranges [off, off+len) whose phase-1 state rank k computes and broadcasts
    std::vector<std::vector<std::pair<int, int>>> owned;
    std::vector<std::vector<int>> runPasses;  // run boundaries before each merge pass
    int height = 0;
    int maxM = 0;
    int maxLeaf = 0;
    int sms = 148;       // SM count of the device (fused-tier fill rule)
    bool sigma = false;  // requested-rows plan: grid tier everywhere, no root-only merges
    std::vector<int> tByOff;  // leaf tasks in offset order (requested-rows plans)
    // device copies
    int* dev = nullptr;  // one int buffer
    size_t devInts = 0;
    int *d_tOff = nullptr, *d_tSize = nullptr, *d_tFlags = nullptr, *d_cut = nullptr;
    int *d_mOff = nullptr, *d_mSize = nullptr, *d_mNL = nullptr, *d_mFlags = nullptr;
    int *d_tileFirst = nullptr, *d_bstart = nullptr, *d_gFirst = nullptr, *d_gCount = nullptr;
    std::vector<int*> d_runs;
    // sparse levels: control words (4 per level + a zero block), per-merge
    // tables (spCs, spCsR, spNN, spK: 4 per merge), group starts, per-CTA counts
    int* d_ctl = nullptr;
    int nctl = 0;
    int* d_spTab = nullptr;
    int* d_spGroup = nullptr;
    int* d_blockCnt = nullptr;
    int* d_spTiles = nullptr;  // k_sp_place tile records: merge + split per 1024 positions
    int* h_ctl = nullptr;  // pinned copy of the control words after a solve (deflation profile)
    int dbgStop = 0;       // debug (BRGPU_DEBUG_STOP_LEVEL): run only the first k levels of phase 1
    bool anySp = false;
    // live-list tier: first live level (index in `levels`, -1: none), frontier
    // nodes (off, size) entering it, control words + key words, final-sort buckets
    bool liveWanted = false;
    int liveLev = -1;
    std::vector<int> liveFront;
    int2* d_liveFront = nullptr;
    int* d_liveCtl = nullptr;
    unsigned long long* d_liveKeys = nullptr;
    int liveNb = 0;
    std::vector<int> liveBlocks;  // several blocks: the blocks whose top levels are live
    int* d_liveBlocks = nullptr;
    int* d_liveBctr = nullptr;    // per-block pool counters (several blocks)
    int liveTop = -1;        // first level of the dataflow top run (k_live_top), -1: none
    int liveTopMerges = 0;
    int liveCl = 1;          // > 1: split-rule live levels run one merge per cluster of up to liveCl CTAs
    int liveFlow = -1, liveFlowLevels = 0;  // lane-mode live levels as one dataflow launch (k_live_flow)
    std::vector<int> liveFlowItems;         // int4 (level in run, first merge, merges, 0)
    int liveFlowMerges = 0;
    int* d_liveFlowItems = nullptr;
    int* d_liveFlowDone = nullptr;          // flowMerges done words + the ticket
    int* d_liveDone = nullptr;
    cudaGraphExec_t graph = nullptr;
    bool graph_trace = false;
    uint64_t graph_gen = 0;
    int launches = 0;
};

struct Handle {
    int device = 0;
    int sms = 148;
    int sec_grid = 148 * 8;
    cudaStream_t stream = nullptr;
    int leaf_cutoff = 25;
    int zhat = 1;
    int patched = 1;
    int use_graph = 1;
    int subtree = 1;
    int sparse = 0;  // sparse grid-tier levels (BRGPU_OPT_SPARSE; opt-in)
    int live = 1;    // live-list top levels (BRGPU_OPT_LIVE)
    int liveCluster = 1;  // split-rule live levels on thread-block clusters (BRGPU_OPT_LIVE_CLUSTER)
    int liveFlow = 1;     // lane-mode live levels as one dataflow launch (BRGPU_OPT_LIVE_FLOW)
    // live-tier fallback back-off: after a fallback at order liveVeto the next
    // liveSkip solves of that order plan densely (64, doubling per repeated fallback:
    // a failed attempt costs ~40% of a solve, so inputs that never hold pay < 1%)
    int liveVeto = 0, liveSkip = 0, liveBackoff = kLiveBackoff0;
    int strace = 0;  // secular-problem trace (brgpu_set_secular_trace): grid tier, dump per level
    double* strBuf = nullptr;  // per level 2n doubles (d, z) + rho per merge
    int64_t strCap = 0;
    int exact = 0;
    int trace = 0;
    double tol_scale = 1.0;
    std::string err;
    // workspace
    int64_t cap = 0;
    Work w{};
    uint8_t* split = nullptr;
    unsigned long long* sbits = nullptr;  // per block scale bits
    int64_t sbitsCap = 0;
    unsigned long long* mTol = nullptr;
    int64_t mTolCap = 0;
    int* traceBuf = nullptr;  // 2 ints per merge
    int64_t traceCap = 0;
    double* pinned = nullptr;
    int64_t pinnedCap = 0;
    int* hsmall = nullptr;  // pinned: [0]=nsplit [1]=status
    unsigned long long* hcnt = nullptr;
    int* dsmall = nullptr;  // device: [0]=nsplit [1..]=unused
    // ledger
    int64_t ledger_doubles = 0, ledger_ints = 0, peak_doubles = 0, peak_ints = 0, limit_n = 0;
    // plan cache
    std::unique_ptr<Plan> plan;
    cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t pev[2] = {nullptr, nullptr};  // after stage A, after the exchange (graph record nodes)
    brgpu_timing timing{};
    Prof* prof = nullptr;
    uint64_t bufgen = 1;  // bumped whenever a buffer baked into a graph moves
    brgpu_stats stats{};
    std::vector<brgpu_trace> traceRecs;
    // distribution: one process per GPU over NCCL, or P virtual ranks on this device
    int nranks = 1, rank = 0;
    ncclComm_t comm = nullptr;
    int virt = 1;
    int root_split = 1;  // split the roots of shared top merges across ranks (BRGPU_OPT_ROOT_SPLIT)
    int xerr = 0;        // first exchange error of the current solve (run_plan returns it)
    std::vector<std::unique_ptr<Handle>> subs;
    // requested eigenvector rows of the current solve (brgpu_eigvals_rows), or null
    struct SigmaRun {
        SigmaDev dev{};
        std::vector<int> sel;  // host copy of the request
        int* dTask = nullptr;  // leaf task per request
        int* dBlk = nullptr;   // block per request
        int maxBlock = 0;
        double* out = nullptr; // nsel x n, global column order
    };
    SigmaRun* sig = nullptr;
    double* sigDbl = nullptr;  // grow-only buffers of the requested-rows solves (never in a graph)
    int64_t sigDblCap = 0;
    int* sigInt = nullptr;
    int64_t sigIntCap = 0;
};

int fail(Handle* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

#define CUDA_TRY(h, call)                                                              \
    do {                                                                               \
        cudaError_t e__ = (call);                                                      \
        if (e__ != cudaSuccess)                                                        \
            return fail((h), BRGPU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
    } while (0)

// ---------------------------------------------------------------------------
// planning
// ---------------------------------------------------------------------------
struct NodeRec {
    int off, size, nl, level, root, owner;  // owner: rank, or -1 for the shared top of a split block
};

struct LeafRec {
    int off, size, owner;
};

// Split tree of one block (merge_tree.cpp:34-60).  For a block split across
// ranks, nodes at depth < D are "top" (owner -1, all ranks after the
// exchange) and the depth-D nodes, left to right, are owned by ranks 0..2^D-1
// together with their whole subtrees.
int build_node(int off, int size, int cutoff, bool root, int depth, int D, int owner, int* nextOwner,
               std::vector<NodeRec>& internal, std::vector<LeafRec>& leaves,
               std::vector<std::pair<int, int>>* ownedBig) {
    if (depth == D && owner < 0 && nextOwner) {
        owner = (*nextOwner)++;
        if (ownedBig) ownedBig[owner].emplace_back(off, size);
    }
    if (size <= cutoff) {
        leaves.push_back({off, size, owner});
        return 0;
    }
    const int nl = size / 2;
    const int idx = (int)internal.size();
    internal.push_back({off, size, nl, 0, root ? 1 : 0, owner});
    const int ll = build_node(off, nl, cutoff, false, depth + 1, D, owner, nextOwner, internal, leaves, ownedBig);
    const int rl = build_node(off + nl, size - nl, cutoff, false, depth + 1, D, owner, nextOwner, internal,
                              leaves, ownedBig);
    const int lev = 1 + std::max(ll, rl);
    internal[idx].level = lev;
    return lev;
}

// Level tables of a set of merges (grouped by level, offset order) appended to
// the plan's merge arrays; fused SMEM groups where every merge of the level fits.
void add_levels(Plan* p, std::vector<NodeRec> nodes, bool fuse, std::vector<LevelHost>& out) {
    std::stable_sort(nodes.begin(), nodes.end(), [](const NodeRec& a, const NodeRec& b) {
        return a.level != b.level ? a.level < b.level : a.off < b.off;
    });
    const int ntiles = (p->n + kTile - 1) / kTile;
    size_t i = 0;
    while (i < nodes.size()) {
        const int lev = nodes[i].level;
        LevelHost L;
        L.level = lev;
        L.m0 = (int)p->mOff.size();
        L.tile0 = (int)p->tileFirst.size();
        size_t j = i;
        while (j < nodes.size() && nodes[j].level == lev) {
            p->mOff.push_back(nodes[j].off);
            p->mSize.push_back(nodes[j].size);
            p->mNL.push_back(nodes[j].nl);
            p->mFlags.push_back(nodes[j].root ? kMergeRoot : 0);
            p->mLevel.push_back(lev);
            ++j;
        }
        L.M = (int)(j - i);
        p->maxM = std::max(p->maxM, L.M);
        int maxSize = 0, minSize = INT32_MAX;
        for (int q = 0; q < L.M; ++q) {
            maxSize = std::max(maxSize, p->mSize[L.m0 + q]);
            minSize = std::min(minSize, p->mSize[L.m0 + q]);
        }
        L.minSize = minSize;
        L.maxSize = maxSize;
        // A 1024-shape level runs 2 CTAs per SM; with fewer merges than SMs most
        // of the GPU idles (Toeplitz 2^16, level 6: 64 merges of K ~ 512), and the
        // grid tier, which spreads every merge over the whole GPU, is faster
        // once n is large enough to amortise its ~15 launches per level
        // (A/B: Toeplitz 2^16 20.7 -> 20.1 ms; glued Wilkinson 2^18, 256 merges,
        // and n = 4096 stay fused).
        const bool underfilled = maxSize > kFuseSmallElems && L.M < p->sms && p->n >= kGridMinN;
        // ... and a level of many merges (>= 4 per SM) larger than 128 runs on
        // the grid tier too: its lane-per-root secular kernel packs the roots
        // of all merges onto full warps, where a fused CTA holds only K ~ 100-140
        // roots of one or two merges for its 256 lanes (A/B, levels 4-6 on the
        // grid tier: random 2^20 4.59 -> 4.52 ms, 4096 x 1024 batch 12.30 ->
        // 11.66 ms; glued Wilkinson 2^18 8.04 -> 8.15 ms, its few-root level 4
        // prefers the fused tier; merges <= 128 stay fused everywhere).
        // 512-shape levels (4 CTAs per SM) need twice as many merges (glued
        // Wilkinson 2^18, level 4 with 1024 merges: 8.11 -> 7.99 ms fused)
        const int perSm = maxSize > kFuseSmallElems ? kGridManyPerSm : 2 * kGridManyPerSm;
        const bool many = maxSize > kGridManyMinSize && L.M >= perSm * p->sms && p->n >= kGridMinN;
        L.fused = fuse && maxSize <= kFuseMaxElems && !underfilled && !many;
        L.cap = maxSize <= kFuseSmallElems ? kFuseSmallElems : kFuseMaxElems;
        L.g0 = (int)p->gFirst.size();
        L.G = 0;
        if (L.fused) {
            int q = 0;
            const bool few = L.M < kFewMergesPerSm * p->sms;
            while (q < L.M) {
                int c = 1, tot = p->mSize[L.m0 + q];
                while (!few && q + c < L.M && c < kFuseMaxMergesHost &&
                       p->mOff[L.m0 + q + c] == p->mOff[L.m0 + q + c - 1] + p->mSize[L.m0 + q + c - 1] &&
                       tot + p->mSize[L.m0 + q + c] <= L.cap) {
                    tot += p->mSize[L.m0 + q + c];
                    ++c;
                }
                p->gFirst.push_back(q);
                p->gCount.push_back(c);
                q += c;
                ++L.G;
            }
        }
        // tileFirst[t] = first merge whose end exceeds t*kTile
        int m = 0;
        for (int t = 0; t <= ntiles; ++t) {
            const long long start = (long long)t * kTile;
            while (m < L.M && (long long)p->mOff[L.m0 + m] + p->mSize[L.m0 + m] <= start) ++m;
            p->tileFirst.push_back(m);
        }
        out.push_back(L);
        i = j;
    }
}

// Runs of >= 2 consecutive small-shape fused levels in which every group of
// the run's top level is exactly tiled by whole merges at each lower level
// (true for complete trees such as n = 2^k; otherwise the levels stay
// separate launches): one k_levels_fused launch per run.
void plan_fused_runs(Plan* p) {
    auto& lv = p->levels;
    size_t i = 0;
    while (i < lv.size()) {
        size_t j = i;
        while (j < lv.size() && lv[j].fused && lv[j].cap == kFuseSmallElems &&
               (j == i || lv[j].level == lv[j - 1].level + 1) && j - i < (size_t)kMaxFusedRun &&
               lv[j].M >= kFewMergesPerSm * p->sms)  // few-merge levels launch on their own
            ++j;
        if (j - i < 2) { i = std::max(j, i + 1); continue; }
        const LevelHost& top = lv[j - 1];
        const int nlev = (int)(j - i);
        std::vector<int> tab;
        std::vector<int> covered(j - i, 0);  // every merge of every level of the run must be in a group
        bool ok = true;
        for (int q = 0; q < top.G && ok; ++q) {
            const int gf = p->gFirst[(size_t)top.g0 + q], gc = p->gCount[(size_t)top.g0 + q];
            const int a = top.m0 + gf, z = top.m0 + gf + gc - 1;
            const int start = p->mOff[(size_t)a], end = p->mOff[(size_t)z] + p->mSize[(size_t)z];
            for (size_t l = i; l < j && ok; ++l) {
                const LevelHost& L = lv[l];
                const int* mo = p->mOff.data() + L.m0;
                const int* ms = p->mSize.data() + L.m0;
                const int first = (int)(std::lower_bound(mo, mo + L.M, start) - mo);
                int pos = start, c = 0;
                while (first + c < L.M && mo[first + c] < end) {
                    if (mo[first + c] != pos) { ok = false; break; }
                    pos += ms[first + c];
                    ++c;
                }
                ok = ok && pos == end && c >= 1 && c <= kFuseMaxMergesHost;
                covered[l - i] += c;
                tab.push_back(first);
                tab.push_back(c);
            }
        }
        for (size_t l = i; l < j && ok; ++l) ok = covered[l - i] == lv[l].M;
        if (ok) {
            p->multi.push_back({(int)i, nlev, top.G, (int)p->mlTab.size() / 2});
            p->mlTab.insert(p->mlTab.end(), tab.begin(), tab.end());
        }
        i = j;
    }
}

// Plan of rank `rank` out of `nranks` (1: the whole solve).  Blocks of at
// least 2^D * 2(cutoff+1) elements (D = floor(log2 nranks)) are split by
// subtree; smaller blocks go to ranks in contiguous chunks of the total size.
std::unique_ptr<Plan> make_plan(int n, int cutoff, const std::vector<int>& bstart,
                                const std::vector<int>& segs, bool fuse, int nranks = 1, int rank = 0,
                                int sms = 148, bool sparse = false, bool live = false, int liveCl = 1,
                                bool liveFlowOn = false) {
    auto p = std::make_unique<Plan>();
    p->n = n;
    p->sms = sms;
    p->cutoff = cutoff;
    p->bstart = bstart;
    p->segs = segs;
    p->nranks = nranks;
    p->rank = rank;
    p->owned.assign((size_t)nranks, {});
    int D = 0;
    while ((2 << D) <= nranks) ++D;
    const int Peff = 1 << D;
    const long long bigMin = (long long)Peff * 2 * (cutoff + 1);
    std::vector<NodeRec> internal;
    std::vector<LeafRec> leaves;
    const int nblk = (int)bstart.size() - 1;
    long long smallTotal = 0;
    if (nranks > 1)
        for (int b = 0; b < nblk; ++b) {
            const int sz = bstart[b + 1] - bstart[b];
            if (sz < bigMin) smallTotal += sz;
        }
    long long smallSeen = 0;
    for (int b = 0; b < nblk; ++b) {
        const int off = bstart[b], sz = bstart[b + 1] - off;
        const bool big = nranks > 1 && sz >= bigMin;
        int owner = 0;  // small blocks: contiguous chunks by cumulative size
        if (nranks > 1 && !big) {
            owner = (int)std::min<long long>(nranks - 1, smallTotal ? smallSeen * nranks / smallTotal : 0);
            smallSeen += sz;
            auto& ow = p->owned[(size_t)owner];
            if (!ow.empty() && ow.back().first + ow.back().second == off) ow.back().second += sz;
            else ow.emplace_back(off, sz);
        }
        if (sz <= cutoff) {
            if (owner == rank || nranks == 1) {
                p->tOff.push_back(off);
                p->tSize.push_back(sz);
                p->tFlags.push_back(1);  // values only
                p->maxLeaf = std::max(p->maxLeaf, sz);
            }
            continue;
        }
        int next = 0;
        const int h = build_node(off, sz, cutoff, true, 0, big ? D : -1, big ? -1 : owner,
                                 big ? &next : nullptr, internal, leaves, big ? p->owned.data() : nullptr);
        p->height = std::max(p->height, h);
    }
    for (auto& lf : leaves) {
        if (nranks > 1 && lf.owner != rank) continue;
        p->tOff.push_back(lf.off);
        p->tSize.push_back(lf.size);
        p->tFlags.push_back(0);
        p->maxLeaf = std::max(p->maxLeaf, lf.size);
    }
    for (auto& nd : internal) p->cutPos.push_back(nd.off + nd.nl - 1);  // prepare is full on every rank
    std::vector<NodeRec> mine, top;
    for (auto& nd : internal) {
        if (nranks == 1 || nd.owner == rank) mine.push_back(nd);
        else if (nd.owner < 0) top.push_back(nd);
    }
    add_levels(p.get(), mine, fuse, p->levels);
    add_levels(p.get(), top, fuse, p->levels2);
    plan_fused_runs(p.get());
    // live-list tier: the top run of non-fused levels whose merges are all >= kLiveMinSize
    p->liveWanted = live;
    if (live && nranks == 1 && n >= kLiveMinN) {
        size_t li = p->levels.size();
        while (li > 0 && !p->levels[li - 1].fused && p->levels[li - 1].minSize >= kLiveMinSize) --li;
        // one live level does not pay for the tier's entry and final sort (4096 x 1024
        // batch: only the block roots, 10.67 ms against 10.58 dense; 1024 x 4096: three
        // live levels, 11.35 against 11.60)
        if (p->levels.size() - li < 2) li = p->levels.size();
        // several blocks (a batch, natural splits): every block with live merges is
        // sorted by one CTA at the end, so it must fit its shared memory
        if (li < p->levels.size() && nblk > 1) {
            std::vector<char> isLive((size_t)nblk, 0);
            for (size_t l = li; l < p->levels.size(); ++l) {
                const LevelHost& lh = p->levels[l];
                for (int q = 0; q < lh.M; ++q) {
                    const int o = p->mOff[(size_t)(lh.m0 + q)];
                    const int b = (int)(std::upper_bound(bstart.begin(), bstart.end(), o) - bstart.begin()) - 1;
                    isLive[(size_t)b] = 1;
                }
            }
            bool fits = true;
            for (int b = 0; b < nblk; ++b)
                if (isLive[(size_t)b]) {
                    p->liveBlocks.push_back(b);
                    fits = fits && bstart[b + 1] - bstart[b] <= live_block_cap();
                }
            if (!fits) { li = p->levels.size(); p->liveBlocks.clear(); }
        }
        if (li < p->levels.size()) {
            p->liveLev = (int)li;
            std::set<std::pair<int, int>> liveM;
            for (size_t l = li; l < p->levels.size(); ++l) {
                LevelHost& lh = p->levels[l];
                lh.live = true;
                for (int q = 0; q < lh.M; ++q) liveM.emplace(p->mOff[(size_t)(lh.m0 + q)], p->mSize[(size_t)(lh.m0 + q)]);
            }
            std::vector<std::pair<int, int>> front;
            for (size_t l = li; l < p->levels.size(); ++l) {
                const LevelHost& lh = p->levels[l];
                for (int q = 0; q < lh.M; ++q) {
                    const int o = p->mOff[(size_t)(lh.m0 + q)], sz = p->mSize[(size_t)(lh.m0 + q)];
                    const int nl = p->mNL[(size_t)(lh.m0 + q)];
                    if (!liveM.count({o, nl})) front.emplace_back(o, nl);
                    if (!liveM.count({o + nl, sz - nl})) front.emplace_back(o + nl, sz - nl);
                }
            }
            std::sort(front.begin(), front.end());
            for (auto& f : front) { p->liveFront.push_back(f.first); p->liveFront.push_back(f.second); }
            p->liveNb = live_buckets(n);
            p->liveCl = liveCl;
            // lane-mode dataflow run: the live levels from the tier's first level
            // up to the split rule, each the complete binary child level of the next
            if (liveFlowOn) {
                size_t t = li;
                while (t < p->levels.size() && p->levels[t].maxSize <= kSplitMinSizeHost && t - li < (size_t)kMaxLiveTop) {
                    if (t > li) {
                        const LevelHost& lo = p->levels[t - 1];
                        const LevelHost& up = p->levels[t];
                        bool ok = lo.M == 2 * up.M;
                        for (int q = 0; ok && q < up.M; ++q) {
                            const size_t a = (size_t)(up.m0 + q), c0 = (size_t)(lo.m0 + 2 * q), c1 = c0 + 1;
                            ok = p->mOff[a] == p->mOff[c0] && p->mNL[a] == p->mSize[c0] &&
                                 p->mOff[c1] == p->mOff[a] + p->mNL[a] && p->mSize[c1] == p->mSize[a] - p->mNL[a];
                        }
                        if (!ok) break;
                    }
                    ++t;
                }
                if (t - li >= 2) {
                    p->liveFlow = (int)li;
                    p->liveFlowLevels = (int)(t - li);
                    for (size_t l = li; l < t; ++l) {
                        const int M = p->levels[l].M, G = std::min(live_lane_group(M, sms), kLiveFlowGMax);
                        for (int m = 0; m < M; m += G) {
                            p->liveFlowItems.push_back((int)(l - li));
                            p->liveFlowItems.push_back(m);
                            p->liveFlowItems.push_back(std::min(G, M - m));
                            p->liveFlowItems.push_back(0);
                        }
                        p->liveFlowMerges += M;
                    }
                }
            }
            // dataflow top run (clusters off): the longest tail of split-arithmetic
            // levels that form a complete binary tree (merge m of level l = merges
            // 2m, 2m+1 of l - 1) whose merges are all co-resident
            const int cap = liveCl > 1 ? 0 : live_top_capacity(sms);  // clusters replace the dataflow run
            size_t t = p->levels.size();
            int merges = 0;
            while (t > li && p->levels.size() - t < (size_t)kMaxLiveTop) {
                const LevelHost& lh = p->levels[t - 1];
                if (lh.minSize <= kSplitMinSizeHost || merges + lh.M > cap) break;
                if (t < p->levels.size()) {  // lh must be the complete child level of levels[t]
                    const LevelHost& up = p->levels[t];
                    bool ok = lh.M == 2 * up.M;
                    for (int q = 0; ok && q < up.M; ++q) {
                        const size_t a = (size_t)(up.m0 + q), c0 = (size_t)(lh.m0 + 2 * q), c1 = c0 + 1;
                        ok = p->mOff[a] == p->mOff[c0] && p->mNL[a] == p->mSize[c0] &&
                             p->mOff[c1] == p->mOff[a] + p->mNL[a] && p->mSize[c1] == p->mSize[a] - p->mNL[a];
                    }
                    if (!ok) break;
                }
                merges += lh.M;
                --t;
            }
            if (p->levels.size() - t >= 2) {
                p->liveTop = (int)t;
                p->liveTopMerges = merges;
            }
        }
    }
    // control words per level; phase-1 grid levels may run the sparse pipeline
    // (sparse.cu); the shared top merges of a multi-rank plan stay dense (their
    // roots are split across ranks by the dense kernels)
    {
        int ci = 0;
        for (LevelHost& lh : p->levels) {
            lh.ctl = 4 * ci++;
            // k_sp_place bounds its merge segments per tile by the smallest merge
            lh.sp = sparse && !lh.fused && !lh.live && lh.minSize >= sparse_min_merge() ? 1 : 0;
            lh.spCap = sparse_cap();
            lh.spSpan = 2 * sparse_cap() - lh.spCap;
            lh.spStatic = lh.sp && lh.maxSize <= lh.spCap ? 1 : 0;
        }
        for (LevelHost& lh : p->levels2) lh.ctl = 4 * ci++;
    }
    // final merge passes: runs = blocks, merged pairwise inside each segment;
    // a segment with an odd run count gets an empty partner so that pairs
    // (2k, 2k+1) of a pass table never straddle segments.
    {
        std::vector<int> runs = bstart;
        for (;;) {
            bool any = false;
            std::vector<int> pass{0};
            size_t r = 0;
            const size_t nr = runs.size() - 1;
            for (size_t sg = 0; sg + 1 < segs.size(); ++sg) {
                const int segEnd = segs[sg + 1];
                size_t cnt = 0;
                while (r < nr && runs[r + 1] <= segEnd) { pass.push_back(runs[r + 1]); ++r; ++cnt; }
                if (cnt > 1) any = true;
                if (cnt % 2) pass.push_back(segEnd);
            }
            if (!any) break;
            p->runPasses.push_back(pass);
            std::vector<int> nxt;
            for (size_t k = 0; k < pass.size(); k += 2)
                if (nxt.empty() || nxt.back() != pass[k]) nxt.push_back(pass[k]);
            runs = nxt;
        }
    }
    return p;
}

// Pageable host table -> device on the handle's (non-blocking) stream, then
// wait: a plain cudaMemcpy runs on the legacy stream, which a non-blocking
// stream is not ordered after, and may return before its DMA lands.
int h2d_sync(Handle* h, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return BRGPU_OK;
    CUDA_TRY(h, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    return BRGPU_OK;
}

int upload_plan(Handle* h, Plan* p) {
    std::vector<int> buf;
    auto put = [&](const std::vector<int>& v) {
        const size_t o = buf.size();
        buf.insert(buf.end(), v.begin(), v.end());
        while (buf.size() % 4) buf.push_back(0);
        return o;
    };
    const size_t oTOff = put(p->tOff), oTSize = put(p->tSize), oTFlags = put(p->tFlags);
    const size_t oCut = put(p->cutPos);
    const size_t oMOff = put(p->mOff), oMSize = put(p->mSize), oMNL = put(p->mNL), oMF = put(p->mFlags);
    const size_t oTile = put(p->tileFirst);
    const size_t oB = put(p->bstart);
    const size_t oGF = put(p->gFirst), oGC = put(p->gCount);
    const size_t oML = put(p->mlTab);  // int2 pairs: 8-byte aligned (offsets are multiples of 4 ints)
    std::vector<size_t> oRuns;
    for (auto& rp : p->runPasses) oRuns.push_back(put(rp));
    p->nctl = 4 * (int)(p->levels.size() + p->levels2.size() + 1);
    const size_t oCtl = put(std::vector<int>((size_t)p->nctl, 0));
    int ngMax = 1;
    bool anySp = false;
    for (const auto* lv : {&p->levels, &p->levels2})
        for (const LevelHost& lh : *lv)
            if (lh.sp) { anySp = true; ngMax = std::max(ngMax, sparse_groups_max(p->n, lh.M, kSpMinSpan)); }
    p->anySp = anySp;
    const size_t oSpTab = put(std::vector<int>(anySp ? 4 * p->mOff.size() : 0, 0));
    const size_t oSpGroup = put(std::vector<int>(anySp ? (size_t)ngMax + 1 : 0, 0));
    const size_t oBlk = put(std::vector<int>(anySp ? (size_t)sparse_flag_grid(p->n, p->sms) : 0, 0));
    const size_t oTiles = put(std::vector<int>(anySp ? 2 * (size_t)(p->n / 1024 + 2) : 0, 0));
    const size_t oFront = put(p->liveFront);  // int2 pairs
    const size_t oLiveCtl = put(std::vector<int>(p->liveLev >= 0 ? 4 : 0, 0));
    const size_t oLiveKeys = put(std::vector<int>(p->liveLev >= 0 ? 4 : 0, 0));  // 2 u64 (16-byte aligned offsets)
    const size_t oLiveDone = put(std::vector<int>((size_t)p->liveTopMerges, 0));
    const size_t oFlowItems = put(p->liveFlowItems);  // int4: 16-byte aligned offsets
    const size_t oFlowDone = put(std::vector<int>(p->liveFlowMerges ? (size_t)p->liveFlowMerges + 1 : 0, 0));
    const size_t oLiveBlocks = put(p->liveBlocks);
    const size_t oLiveBctr = put(std::vector<int>(p->liveBlocks.empty() ? 0 : p->bstart.size(), 0));
    if (anySp) CUDA_TRY(h, cudaMallocHost(&p->h_ctl, sizeof(int) * (size_t)p->nctl));
    p->devInts = buf.size();
    CUDA_TRY(h, cudaMalloc(&p->dev, sizeof(int) * std::max<size_t>(buf.size(), 1)));
    if (int r = h2d_sync(h, p->dev, buf.data(), sizeof(int) * buf.size())) return r;
    p->d_tOff = p->dev + oTOff; p->d_tSize = p->dev + oTSize; p->d_tFlags = p->dev + oTFlags;
    p->d_cut = p->dev + oCut;
    p->d_mOff = p->dev + oMOff; p->d_mSize = p->dev + oMSize; p->d_mNL = p->dev + oMNL;
    p->d_mFlags = p->dev + oMF; p->d_tileFirst = p->dev + oTile; p->d_bstart = p->dev + oB;
    p->d_gFirst = p->dev + oGF; p->d_gCount = p->dev + oGC;
    p->d_mlTab = reinterpret_cast<int2*>(p->dev + oML);
    for (size_t o : oRuns) p->d_runs.push_back(p->dev + o);
    p->d_ctl = p->dev + oCtl;
    p->d_spTab = p->dev + oSpTab;
    p->d_spGroup = p->dev + oSpGroup;
    p->d_blockCnt = p->dev + oBlk;
    p->d_spTiles = p->dev + oTiles;
    p->d_liveFront = reinterpret_cast<int2*>(p->dev + oFront);
    p->d_liveCtl = p->dev + oLiveCtl;
    p->d_liveKeys = reinterpret_cast<unsigned long long*>(p->dev + oLiveKeys);
    p->d_liveDone = p->dev + oLiveDone;
    p->d_liveFlowItems = p->dev + oFlowItems;
    p->d_liveFlowDone = p->dev + oFlowDone;
    p->d_liveBlocks = p->dev + oLiveBlocks;
    p->d_liveBctr = p->dev + oLiveBctr;
    return BRGPU_OK;
}

void free_plan(Plan* p) {
    if (!p) return;
    if (p->graph) cudaGraphExecDestroy(p->graph);
    if (p->dev) cudaFree(p->dev);
    if (p->h_ctl) cudaFreeHost(p->h_ctl);
    p->h_ctl = nullptr;
    p->graph = nullptr;
    p->dev = nullptr;
}

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------
void free_work(Handle* h) {
    if (h->cap == 0) return;
    cudaFree(h->w.dw);
    cudaFree(h->w.nnPre);
    cudaFree(h->w.nnFlag);
    h->w = Work{};
    h->cap = 0;
    h->ledger_doubles = h->ledger_ints = 0;
}

int ensure_work(Handle* h, int64_t n) {
    if (n <= h->cap) return BRGPU_OK;
    if (h->plan) { free_plan(h->plan.get()); h->plan.reset(); }
    free_work(h);
    const int64_t c = (std::max<int64_t>(n, 1024) + 1023) / 1024 * 1024;
    const int64_t nd = 15 * c;
    double* dbl = nullptr;
    CUDA_TRY(h, cudaMalloc(&dbl, sizeof(double) * nd));
    Work& w = h->w;
    w.exact = h->exact;
    w.own_P = 1;
    w.own_r = 0;
    w.dw = dbl; w.ew = dbl + c; w.lam = dbl + 2 * c; w.blo = dbl + 3 * c; w.bhi = dbl + 4 * c;
    w.D = dbl + 5 * c; w.Z = dbl + 6 * c; w.R0 = dbl + 7 * c; w.R1 = dbl + 8 * c;
    w.dA = dbl + 9 * c; w.zA = dbl + 10 * c; w.z2A = dbl + 11 * c; w.r0A = dbl + 12 * c;
    w.r1A = dbl + 13 * c; w.tau = dbl + 14 * c;
    const int64_t ntiles = (c + 1023) / 1024 + 1;
    // look-back states: merge tiles (256 positions) + scan tiles (1024) + tickets
    const int64_t ni = 5 * c + 2 + 2 * ntiles + 8 + 2 * (6 * ntiles + 8);
    int* ib = nullptr;
    CUDA_TRY(h, cudaMalloc(&ib, sizeof(int) * ni));
    w.nnPre = ib; w.nnPos = ib + c + 1; w.survPre = ib + 2 * c + 1; w.aMerge = ib + 3 * c + 2;
    w.org = ib + 4 * c + 2; w.tileCnt = ib + 5 * c + 2; w.tileOff = ib + 5 * c + 2 + ntiles;
    w.status = ib + 5 * c + 2 + 2 * ntiles;
    {
        // 8-byte aligned look-back states after status (+2 ints of padding)
        int* sp = ib + 5 * c + 2 + 2 * ntiles + 8;
        if (reinterpret_cast<uintptr_t>(sp) % 8) ++sp;
        w.scanState = reinterpret_cast<unsigned long long*>(sp);
        w.levelModes = ib + 5 * c + 2 + 2 * ntiles + 1;
    }
    uint8_t* bb = nullptr;
    CUDA_TRY(h, cudaMalloc(&bb, 3 * c + 128));
    w.nnFlag = bb; w.survFlag = bb + c; h->split = bb + 2 * c;
    w.counters = reinterpret_cast<unsigned long long*>(bb + 3 * c);  // 8-byte aligned (c%8==0? pad)
    h->cap = c;
    ++h->bufgen;
    h->ledger_doubles = nd;
    h->ledger_ints = ni + (3 * c + 128 + 3) / 4;
    h->peak_doubles = std::max(h->peak_doubles, h->ledger_doubles);
    h->peak_ints = std::max(h->peak_ints, h->ledger_ints);
    h->limit_n = c;
    return BRGPU_OK;
}

template <typename T>
int ensure_buf(Handle* h, T*& p, int64_t& cap, int64_t need) {
    if (need <= cap) return BRGPU_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    CUDA_TRY(h, cudaMalloc(&p, sizeof(T) * std::max<int64_t>(need, 1)));
    cap = need;
    ++h->bufgen;
    return BRGPU_OK;
}

// Every device allocation a handle holds, in 8-byte words (doubles and the
// u64 scale/tolerance words) and 4-byte words (ints; byte arrays rounded up):
// the main arena, the per-block scale bits, per-merge tolerance words, the
// plan tables, the trace buffer, the requested-rows buffers and the small
// status words -- plus the same for every virtual-rank sub-handle.  The
// requested-rows buffers (O(|sigma| n)) are reported separately.
void ledger_now(const Handle* h, int64_t& dbl, int64_t& ints) {
    dbl += h->ledger_doubles + h->sbitsCap + h->mTolCap;
    ints += h->ledger_ints + (h->plan ? (int64_t)h->plan->devInts : 0) + h->traceCap + 4;
    for (const auto& u : h->subs) ledger_now(u.get(), dbl, ints);
}

void ledger_peak(Handle* h) {
    int64_t dbl = 0, ints = 0;
    ledger_now(h, dbl, ints);
    h->peak_doubles = std::max(h->peak_doubles, dbl);
    h->peak_ints = std::max(h->peak_ints, ints);
}

// ---------------------------------------------------------------------------
// solve
// ---------------------------------------------------------------------------
int status_message(Handle* h, int st) {
    switch (st) {
        case BRGPU_ERR_INVALID_ARGUMENT: return fail(h, st, "tridiagonal: non-finite entry");
        case BRGPU_ERR_NO_CONVERGENCE: return fail(h, st, "no convergence (QL/QR sweep limit or secular iteration)");
        case BRGPU_ERR_ZERO_DENOMINATOR: return fail(h, st, "secular_column: reconstructed delta is zero");
        default: return fail(h, st, "device error " + std::to_string(st));
    }
}

LevelDev level_dev(Handle* h, Plan* p, const LevelHost& lh, const LevelHost* prev = nullptr) {
    LevelDev L{};
    L.mOff = p->d_mOff + lh.m0;
    L.mSize = p->d_mSize + lh.m0;
    L.mNL = p->d_mNL + lh.m0;
    L.mFlags = p->d_mFlags + lh.m0;
    L.mTol = h->mTol;
    L.tileFirst = p->d_tileFirst + lh.tile0;
    L.M = lh.M;
    L.allSplit = lh.minSize > kSplitMinSizeHost ? 1 : 0;
    L.maxSize = lh.maxSize;
    (void)prev;
    L.ctl = lh.sp ? p->d_ctl + lh.ctl : nullptr;
    L.spCap = lh.sp ? lh.spCap : 0;
    L.spStatic = lh.spStatic;
    L.spSpan = lh.spSpan;
    if (lh.sp) {
        const size_t M = p->mOff.size();
        L.spCs = p->d_spTab + lh.m0;
        L.spCsR = p->d_spTab + M + lh.m0;
        L.spNN = p->d_spTab + 2 * M + lh.m0;
        L.spK = p->d_spTab + 3 * M + lh.m0;
        L.spGroup = p->d_spGroup;
        L.spTileM = p->d_spTiles;
        L.spTileSplit = p->d_spTiles + (p->n / 1024 + 2);
    }
    return L;
}

SolveParams solve_params(Handle* h, int n) {
    SolveParams prm{};
    prm.n = n;
    prm.zhat = h->zhat;
    prm.patched = h->patched;
    prm.tol_scale = h->tol_scale;
    prm.sec_grid = h->sec_grid;
    prm.sms = h->sms;
    prm.sigma = h->sig ? &h->sig->dev : nullptr;
    return prm;
}

// Root-range split of the shared top merges: rank r of P
// owns active indices g = k*P + r, k < c; results travel through the gather
// buffers (the dead dw and Z arrays of phase 2) in slot r.
struct SplitCfg {
    int P = 1, r = 0, c = 0;
};

// Workspace a solve of order n needs.  A distributed handle reserves n + P so
// that the split exchange buffers (P slots of ceil(n/P)) always fit: whether a
// level's roots are split must depend on (n, P) only, never on one rank's
// reservation history, or the ranks would disagree on the collectives.
int64_t work_need(const Handle* h, int64_t n) { return n + (h->nranks > 1 ? h->nranks : 0); }

// chunk per rank, or 0 when the gather buffers (capacity cap) cannot hold P*c
int split_chunk(const Handle* h, int n, int P) {
    const int c = (n + P - 1) / P;
    return (int64_t)c * P <= h->cap ? c : 0;
}

void set_split(Handle* h, const SplitCfg* sc, SolveParams& prm) {
    h->w.own_P = sc ? sc->P : 1;
    h->w.own_r = sc ? sc->r : 0;
    prm.xsplit = sc ? 1 : 0;
    prm.xc = sc ? sc->c : 0;
    prm.xA = h->w.dw;
    prm.xB = h->w.Z;
}

int exchange_allgather(Handle* h, const SplitCfg& sc, int arrays);

// live-list tier state (live.cu) in arrays the dense tiers no longer use above
// the frontier: counts in nnPre, dead maxima in D / Z / R0, the pool in R1, the
// sort's scatter buffer in dA and its bucket tables in nnPos / survPre
LiveDev live_dev(Handle* h, Plan* p) {
    LiveDev V{};
    V.cnt = h->w.nnPre;
    V.dLam = h->w.D;
    V.dBlo = h->w.Z;
    V.dBhi = h->w.R0;
    V.pool = h->w.R1;
    V.tmp = h->w.dA;
    V.bcount = h->w.nnPos;
    V.bcur = h->w.survPre;
    V.ctl = p->d_liveCtl;
    V.keys = p->d_liveKeys;
    V.nb = p->liveNb;
    V.bstart = p->d_bstart;
    V.nblk = (int)p->bstart.size() - 1;
    V.bctr = p->liveBlocks.empty() ? p->d_liveCtl : p->d_liveBctr;  // one block: ctl[0]
    return V;
}

// the live tier's last step: one block -> value-bucket sort of the pool; several
// -> one CTA per live block
void live_final_sort(Handle* h, Plan* p, const LiveDev& V, int* launches, Prof* prof) {
    if (p->liveBlocks.empty())
        launch_live_sort(h->stream, V, p->n, h->w.lam, h->sms, launches, prof);
    else
        launch_live_blocksort(h->stream, V, p->d_liveBlocks, (int)p->liveBlocks.size(), h->w.lam, launches, prof);
}

void run_levels(Handle* h, Plan* p, const std::vector<LevelHost>& levels, int* launches, Prof* prof,
                const SplitCfg* sc = nullptr) {
    cudaStream_t s = h->stream;
    const int n = p->n;
    SolveParams prm = solve_params(h, n);
    const bool phase1 = &levels == &p->levels;
    size_t mr = 0;
    {
        const char* ev = std::getenv("BRGPU_DEBUG_STOP_LEVEL");
        p->dbgStop = ev ? std::atoi(ev) : 0;
    }
    for (size_t li = 0; li < levels.size(); ++li) {
        if (phase1 && p->dbgStop > 0 && li >= (size_t)p->dbgStop) break;
        const LevelHost& lh = levels[li];
        const LevelHost* prev = li ? &levels[li - 1] : nullptr;
        if (phase1 && mr < p->multi.size() && p->multi[mr].lev0 == (int)li) {
            const Plan::MultiRun& run = p->multi[mr++];
            FusedRun fr{};
            fr.nlev = run.nlev;
            for (int l = 0; l < run.nlev; ++l) {
                const LevelHost& ll = levels[li + (size_t)l];
                fr.L[l] = level_dev(h, p, ll, l ? &levels[li + (size_t)l - 1] : prev);
                fr.trace[l] = h->trace ? h->traceBuf + 2 * ll.m0 : nullptr;
            }
            set_split(h, nullptr, prm);
            launch_levels_fused(s, h->w, fr, run.G, p->d_mlTab + run.tab0, prm,
                                launches, prof);
            li += (size_t)run.nlev - 1;
            continue;
        }
        const LevelDev L = level_dev(h, p, lh, prev);
        if (lh.live) {
            const LiveDev V = live_dev(h, p);
            set_split(h, nullptr, prm);
            if ((int)li == p->liveLev)
                launch_live_init(s, h->w, V, p->d_liveFront, (int)p->liveFront.size() / 2, prm.tol_scale,
                                 launches, prof);
            if (phase1 && (int)li == p->liveFlow) {  // lane-mode live levels as one dataflow launch
                LiveRun R{};
                R.nlev = p->liveFlowLevels;
                R.first[0] = 0;
                for (int l = 0; l < R.nlev; ++l) {
                    const LevelHost& ll = levels[li + (size_t)l];
                    R.L[l] = level_dev(h, p, ll, l ? &levels[li + (size_t)l - 1] : prev);
                    R.trace[l] = h->trace ? h->traceBuf + 2 * ll.m0 : nullptr;
                    R.first[l + 1] = R.first[l] + ll.M;
                }
                R.done = p->d_liveFlowDone;
                R.ticket = p->d_liveFlowDone + p->liveFlowMerges;
                R.items = reinterpret_cast<const int4*>(p->d_liveFlowItems);
                R.nitems = (int)p->liveFlowItems.size() / 4;
                launch_live_flow(s, h->w, R, V, prm, launches, prof);
                li += (size_t)R.nlev - 1;
                if (li + 1 == levels.size()) live_final_sort(h, p, V, launches, prof);
                continue;
            }
            if (phase1 && (int)li == p->liveTop) {  // the rest of the tree as one dataflow launch
                LiveRun R{};
                R.nlev = (int)(levels.size() - li);
                R.first[0] = 0;
                for (int l = 0; l < R.nlev; ++l) {
                    const LevelHost& ll = levels[li + (size_t)l];
                    R.L[l] = level_dev(h, p, ll);
                    R.trace[l] = h->trace ? h->traceBuf + 2 * ll.m0 : nullptr;
                    R.first[l + 1] = R.first[l] + ll.M;
                }
                R.done = p->d_liveDone;
                launch_live_top(s, h->w, R, V, prm, launches, prof);
                live_final_sort(h, p, V, launches, prof);
                break;
            }
            const int C = L.allSplit && p->liveCl > 1 ? live_cluster_size(h->device, lh.M, p->liveCl) : 1;
            if (C > 1)
                launch_level_live_cluster(s, h->w, L, V, prm, h->trace ? h->traceBuf + 2 * lh.m0 : nullptr, C,
                                          launches, prof);
            else
                launch_level_live(s, h->w, L, V, prm, h->trace ? h->traceBuf + 2 * lh.m0 : nullptr, launches, prof);
            if (li + 1 == levels.size()) live_final_sort(h, p, V, launches, prof);
            continue;
        }
        if (lh.fused) {
            set_split(h, nullptr, prm);
            launch_level_fused(s, h->w, L, lh.G, lh.cap, p->d_gFirst + lh.g0, p->d_gCount + lh.g0, prm,
                               h->trace ? h->traceBuf + 2 * lh.m0 : nullptr, launches, prof);
            continue;
        }
        if (lh.sp) {
            set_split(h, nullptr, prm);
            launch_level_sparse(s, h->w, L, n, prm, p->d_blockCnt, h->trace ? h->traceBuf + 2 * lh.m0 : nullptr,
                                launches, prof);
            if (lh.spStatic) continue;
        }
        set_split(h, sc, prm);
        for (int part = 0; part < 4; ++part) {
            launch_level_part(s, h->w, L, n, prm, part, launches, prof);
            if (part == 0 && h->strace && h->strBuf) {  // active problem before the refreshed weights
                const size_t li2 = (phase1 ? 0 : p->levels.size()) + li;
                launch_dump_active(s, h->w, L, n, h->strBuf + 2 * (size_t)n * li2,
                                   h->strBuf + 2 * (size_t)n * (p->levels.size() + p->levels2.size()) + lh.m0,
                                   launches);
            }
            if (const int k = level_exchange_arrays(prm, part))
                if (const int e = exchange_allgather(h, *sc, k)) h->xerr = h->xerr ? h->xerr : e;
        }
        set_split(h, nullptr, prm);
        if (h->trace) launch_level_trace(s, h->w, L, n, h->traceBuf + 2 * lh.m0, launches, prof);
    }
}

// Stage A: scale + cuts (full), this rank's leaves and phase-1 merges.
void run_stage_a(Handle* h, Plan* p, int* launches, Prof* prof) {
    cudaStream_t s = h->stream;
    if (prof) prof_mark(prof, (void*)s, -1);
    const int n = p->n;
    const int nblk = (int)p->bstart.size() - 1;
    if (p->anySp) cudaMemsetAsync(p->d_ctl, 0, sizeof(int) * (size_t)p->nctl, s);  // level words (barrier counters)
    if (p->liveLev >= 0) cudaMemsetAsync(p->d_liveCtl, 0, sizeof(int) * 8, s);   // live words + key words
    if (p->liveTopMerges) cudaMemsetAsync(p->d_liveDone, 0, sizeof(int) * (size_t)p->liveTopMerges, s);
    if (p->liveFlowMerges)
        cudaMemsetAsync(p->d_liveFlowDone, 0, sizeof(int) * ((size_t)p->liveFlowMerges + 1), s);
    if (!p->liveBlocks.empty()) cudaMemsetAsync(p->d_liveBctr, 0, sizeof(int) * p->bstart.size(), s);
    launch_prepare(s, n, p->d_bstart, nblk, h->sbits, h->w.dw, h->w.ew, (int)p->cutPos.size(),
                   p->d_cut, launches, prof);
    launch_leaves(s, (int)p->tOff.size(), p->maxLeaf, p->d_tOff, p->d_tSize, p->d_tFlags, h->w,
                  launches, prof);
    if (h->sig)
        launch_sigma_leaves(s, h->sig->dev, p->maxLeaf, h->sig->dTask, p->d_tOff, p->d_tSize, h->w, launches);
    run_levels(h, p, p->levels, launches, prof);
}

// Stage B: shared top merges (roots split across ranks when enabled),
// rescale, cross-block merge passes.
void finish_stage_b(Handle* h, Plan* p, int* launches, Prof* prof);
void run_stage_b(Handle* h, Plan* p, int* launches, Prof* prof) {
    SplitCfg sc;
    const bool split = p->nranks > 1 && h->root_split && (sc.c = split_chunk(h, p->n, p->nranks)) > 0;
    sc.P = p->nranks;
    sc.r = p->rank;
    run_levels(h, p, p->levels2, launches, prof, split ? &sc : nullptr);
    finish_stage_b(h, p, launches, prof);
}

void finish_stage_b(Handle* h, Plan* p, int* launches, Prof* prof) {
    cudaStream_t s = h->stream;
    const int n = p->n;
    const int nblk = (int)p->bstart.size() - 1;
    launch_finish(s, n, p->d_bstart, nblk, h->sbits, h->w.lam, launches, prof);
    if (h->sig)
        launch_sigma_final(s, h->sig->dev, h->w.lam, p->d_bstart, nblk, h->sig->dBlk, h->sig->maxBlock,
                           h->sig->out, n, launches);
    double* src = h->w.lam;
    double* dst = h->w.D;
    for (size_t q = 0; q < p->runPasses.size(); ++q) {
        launch_merge_runs(s, n, src, dst, p->d_runs[q], (int)p->runPasses[q].size() - 1, launches,
                          prof);
        std::swap(src, dst);
    }
    if (src != h->w.lam) cudaMemcpyAsync(h->w.lam, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
}

int exchange_nccl(Handle* h, Plan* p);

// phase boundary marks: external record nodes when captured into the graph
void phase_mark(Handle* h, int k) {
    if (!h->pev[k]) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(h->stream, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(h->pev[k], h->stream, cudaEventRecordExternal);
    else
        cudaEventRecord(h->pev[k], h->stream);
}

int run_plan(Handle* h, Plan* p, int* launches, Prof* prof = nullptr) {
    h->xerr = 0;
    run_stage_a(h, p, launches, prof);
    phase_mark(h, 0);
    if (p->nranks > 1) {
        const int r = exchange_nccl(h, p);
        if (r) return r;
    }
    phase_mark(h, 1);
    run_stage_b(h, p, launches, prof);
    return h->xerr;
}

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed) and the phase-1 -> phase-2 exchange
// ---------------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return a;
        a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))dlsym(lib, "ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))dlsym(lib, "ncclCommDestroy");
        a.Broadcast = (decltype(a.Broadcast))dlsym(lib, "ncclBroadcast");
        a.AllGather = (decltype(a.AllGather))dlsym(lib, "ncclAllGather");
        a.GroupStart = (decltype(a.GroupStart))dlsym(lib, "ncclGroupStart");
        a.GroupEnd = (decltype(a.GroupEnd))dlsym(lib, "ncclGroupEnd");
        a.GetErrorString = (decltype(a.GetErrorString))dlsym(lib, "ncclGetErrorString");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Broadcast && a.AllGather && a.GroupStart &&
               a.GroupEnd && a.GetErrorString;
        return a;
    }();
    return api;
}

// Every rank ends phase 1 with the state (lam, blo, bhi) of the ranges it
// owns; one grouped in-place broadcast per owned range replicates the full
// state on all ranks for the shared top merges.
int exchange_nccl(Handle* h, Plan* p) {
    NcclApi& N = nccl_api();
    if (!h->comm || !N.ok) return fail(h, BRGPU_ERR_NCCL, "distributed plan without an NCCL communicator");
    double* arrs[3] = {h->w.lam, h->w.blo, h->w.bhi};
    ncclResult_t r = N.GroupStart();
    for (int k = 0; k < p->nranks && r == ncclSuccess; ++k)
        for (const auto& rg : p->owned[(size_t)k])
            for (double* a : arrs) {
                r = N.Broadcast(a + rg.first, a + rg.first, (size_t)rg.second, ncclDouble, k, h->comm, h->stream);
                if (r != ncclSuccess) break;
            }
    const ncclResult_t r2 = N.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(h, BRGPU_ERR_NCCL, std::string("ncclBroadcast: ") + N.GetErrorString(r != ncclSuccess ? r : r2));
    return BRGPU_OK;
}

// In-place all-gather of the split exchange buffers (slot r of c doubles per
// rank): one grouped call per array.  Virtual ranks copy between workspaces
// instead (solve_virtual).
int exchange_allgather(Handle* h, const SplitCfg& sc, int arrays) {
    NcclApi& N = nccl_api();
    if (!h->comm || !N.ok) return fail(h, BRGPU_ERR_NCCL, "root-range split without an NCCL communicator");
    double* bufs[2] = {h->w.dw, h->w.Z};
    ncclResult_t r = N.GroupStart();
    for (int k = 0; k < arrays && r == ncclSuccess; ++k)
        r = N.AllGather(bufs[k] + (size_t)sc.r * sc.c, bufs[k], (size_t)sc.c, ncclDouble, h->comm, h->stream);
    const ncclResult_t r2 = N.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return fail(h, BRGPU_ERR_NCCL, std::string("ncclAllGather: ") + N.GetErrorString(r != ncclSuccess ? r : r2));
    return BRGPU_OK;
}

int ensure_buf_sizes(Handle* h, Plan* p);

// P virtual ranks on this device (test mode): each runs its own phase-1 plan
// in its own workspace; the exchange is device copies; phase 2 on rank 0.
// Bitwise identical to the single-rank solve by construction (tested).
int solve_virtual(Handle* h, int n, const std::vector<int>& bstart, const std::vector<int>& segs) {
    const int P = h->virt;
    cudaStream_t s = h->stream;
    CUDA_TRY(h, cudaEventRecord(h->tev[2], s));
    while ((int)h->subs.size() < P) {
        auto sub = std::make_unique<Handle>();
        sub->device = h->device;
        sub->sms = h->sms;
        sub->stream = h->stream;
        h->subs.push_back(std::move(sub));
    }
    std::vector<std::unique_ptr<Plan>> plans;
    for (int k = 0; k < P; ++k) {
        Handle* u = h->subs[(size_t)k].get();
        u->leaf_cutoff = h->leaf_cutoff; u->zhat = h->zhat; u->patched = h->patched;
        u->use_graph = 0; u->subtree = h->subtree; u->trace = 0; u->exact = h->exact; u->w.exact = h->exact; u->tol_scale = h->tol_scale;
        u->sec_grid = h->sec_grid;
        u->root_split = h->root_split;
        u->sparse = h->sparse;
        if (int r = ensure_work(u, (int64_t)n + P)) return fail(h, r, u->err);  // split slots always fit
        u->w.status = h->w.status;
        u->w.counters = h->w.counters;
        CUDA_TRY(h, cudaMemcpyAsync(u->w.dw, h->w.dw, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        CUDA_TRY(h, cudaMemcpyAsync(u->w.ew, h->w.ew, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        plans.push_back(make_plan(n, h->leaf_cutoff, bstart, segs, h->subtree != 0, P, k, h->sms, h->sparse != 0));
        if (int r = upload_plan(u, plans.back().get())) return fail(h, r, u->err);
        if (int r = ensure_buf_sizes(u, plans.back().get())) return fail(h, r, u->err);
        CUDA_TRY(h, cudaMemsetAsync(u->sbits, 0, sizeof(unsigned long long) * bstart.size(), s));
        int launches = 0;
        run_stage_a(u, plans.back().get(), &launches, nullptr);
    }
    for (int k = 0; k < P; ++k)
        for (const auto& rg : plans[(size_t)k]->owned[(size_t)k])
            for (int j = 0; j < P; ++j) {
                if (j == k) continue;
                Handle* a = h->subs[(size_t)k].get();
                Handle* b = h->subs[(size_t)j].get();
                const size_t bytes = sizeof(double) * (size_t)rg.second;
                CUDA_TRY(h, cudaMemcpyAsync(b->w.lam + rg.first, a->w.lam + rg.first, bytes, cudaMemcpyDeviceToDevice, s));
                CUDA_TRY(h, cudaMemcpyAsync(b->w.blo + rg.first, a->w.blo + rg.first, bytes, cudaMemcpyDeviceToDevice, s));
                CUDA_TRY(h, cudaMemcpyAsync(b->w.bhi + rg.first, a->w.bhi + rg.first, bytes, cudaMemcpyDeviceToDevice, s));
            }
    int launches = 0;
    const int c = split_chunk(h->subs[0].get(), n, P);
    if (h->root_split && c > 0) {
        // phase 2 with the roots split across the P virtual ranks, in lockstep;
        // the all-gathers are device copies of each rank's slot
        const auto& L2 = plans[0]->levels2;
        for (size_t li = 0; li < L2.size(); ++li) {
            if (L2[li].fused) {
                for (int k = 0; k < P; ++k) {
                    Handle* u = h->subs[(size_t)k].get();
                    run_levels(u, plans[(size_t)k].get(), {plans[(size_t)k]->levels2[li]}, &launches, nullptr);
                }
                continue;
            }
            for (int part = 0; part < 4; ++part) {
                int arrays = 0;
                for (int k = 0; k < P; ++k) {
                    Handle* u = h->subs[(size_t)k].get();
                    Plan* pk = plans[(size_t)k].get();
                    SolveParams prm = solve_params(u, n);
                    SplitCfg sc;
                    sc.P = P; sc.r = k; sc.c = c;
                    set_split(u, &sc, prm);
                    launch_level_part(s, u->w, level_dev(u, pk, pk->levels2[li]), n, prm, part, &launches, nullptr);
                    arrays = level_exchange_arrays(prm, part);
                    set_split(u, nullptr, prm);
                }
                for (int k = 0; k < P && arrays; ++k)
                    for (int j = 0; j < P; ++j) {
                        if (j == k) continue;
                        Handle* a = h->subs[(size_t)k].get();
                        Handle* b = h->subs[(size_t)j].get();
                        const size_t off = (size_t)k * c, bytes = sizeof(double) * (size_t)c;
                        CUDA_TRY(h, cudaMemcpyAsync(b->w.dw + off, a->w.dw + off, bytes, cudaMemcpyDeviceToDevice, s));
                        if (arrays > 1)
                            CUDA_TRY(h, cudaMemcpyAsync(b->w.Z + off, a->w.Z + off, bytes, cudaMemcpyDeviceToDevice, s));
                    }
            }
        }
        finish_stage_b(h->subs[0].get(), plans[0].get(), &launches, nullptr);
    } else {
        run_stage_b(h->subs[0].get(), plans[0].get(), &launches, nullptr);
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->w.lam, h->subs[0]->w.lam, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(h, cudaEventRecord(h->tev[3], s));
    CUDA_TRY(h, cudaGetLastError());
    CUDA_TRY(h, cudaStreamSynchronize(s));
    for (auto& pl : plans) free_plan(pl.get());
    h->stats.n = n;
    h->stats.blocks = (int)bstart.size() - 1;
    h->stats.graph_replayed = 0;
    return BRGPU_OK;
}

int ensure_buf_sizes(Handle* h, Plan* p) {
    if (int r = ensure_buf(h, h->sbits, h->sbitsCap, (int64_t)p->bstart.size())) return r;
    if (int r = ensure_buf(h, h->mTol, h->mTolCap, std::max(p->maxM, 1))) return r;
    if (h->trace)
        if (int r = ensure_buf(h, h->traceBuf, h->traceCap, 2 * (int64_t)std::max<size_t>(p->mOff.size(), 1))) return r;
    if (h->strace)
        if (int r = ensure_buf(h, h->strBuf, h->strCap,
                               2 * (int64_t)p->n * (int64_t)std::max<size_t>(p->levels.size() + p->levels2.size(), 1) +
                                   (int64_t)std::max<size_t>(p->mOff.size(), 1)))
            return r;
    return BRGPU_OK;
}

// After the input has been copied to dw/ew and split flags computed, finish the solve.
int solve_prepared(Handle* h, int n, const std::vector<int>& segs) {
    cudaStream_t s = h->stream;
    CUDA_TRY(h, cudaMemcpyAsync(h->hsmall, h->dsmall, sizeof(int) * 2, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->hsmall + 1, h->w.status, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    if (h->hsmall[1]) return status_message(h, h->hsmall[1]);
    const int nsplit = h->hsmall[0];
    std::vector<int> bstart;
    if (nsplit == 0) {
        bstart = segs;
    } else {
        // split flags mark natural splits; segment (matrix) ends are implied
        std::vector<uint8_t> fl((size_t)n);
        CUDA_TRY(h, cudaMemcpy(fl.data(), h->split, (size_t)n, cudaMemcpyDeviceToHost));
        size_t sg = 1;
        bstart.push_back(0);
        for (int i = 0; i + 1 < n; ++i) {
            const bool segEnd = sg + 1 < segs.size() && segs[sg] == i + 1;
            if (segEnd) ++sg;
            if (fl[(size_t)i] || segEnd) bstart.push_back(i + 1);
        }
        bstart.push_back(n);
    }
    if (h->virt > 1) return solve_virtual(h, n, bstart, segs);
    Plan* p = h->plan.get();
    const bool sig = h->sig != nullptr;
    bool vetoed = false;
    if (h->liveVeto == n && h->liveSkip > 0) {
        vetoed = true;
        --h->liveSkip;
    }
    const bool wantLive = !sig && h->live != 0 && !h->strace && h->subtree != 0 && !vetoed;
    if (!p || p->n != n || p->cutoff != h->leaf_cutoff || p->bstart != bstart || p->segs != segs ||
        p->sigma != sig || p->liveWanted != wantLive) {
        if (h->plan) free_plan(h->plan.get());
        h->plan = make_plan(n, h->leaf_cutoff, bstart, segs, !sig && h->subtree != 0 && !h->strace, h->nranks,
                            h->rank, h->sms, !sig && h->sparse != 0 && !h->strace, wantLive,
                            h->liveCluster ? live_cluster_max(h->device) : 1, h->liveFlow != 0);
        p = h->plan.get();
        if (sig) {  // every merge propagates the requested rows: no root-only mode
            p->sigma = true;
            for (int& f : p->mFlags) f &= ~kMergeRoot;
        }
        int r = upload_plan(h, p);
        if (r) return r;
    }
    if (sig) {  // leaf task and block of every requested row
        Handle::SigmaRun& sr = *h->sig;
        const int ns = (int)sr.sel.size();
        std::vector<int> task((size_t)ns, -1), blk((size_t)ns, 0);
        std::vector<int>& byOff = p->tByOff;
        if (byOff.size() != p->tOff.size()) {
            byOff.resize(p->tOff.size());
            for (size_t t = 0; t < byOff.size(); ++t) byOff[t] = (int)t;
            std::sort(byOff.begin(), byOff.end(), [&](int a, int b) { return p->tOff[a] < p->tOff[b]; });
        }
        sr.maxBlock = 0;
        for (size_t b = 0; b + 1 < bstart.size(); ++b) sr.maxBlock = std::max(sr.maxBlock, bstart[b + 1] - bstart[b]);
        for (int r = 0; r < ns; ++r) {
            const int i = sr.sel[(size_t)r];
            auto it = std::upper_bound(byOff.begin(), byOff.end(), i,
                                       [&](int v, int t) { return v < p->tOff[t]; });
            task[(size_t)r] = *(it - 1);
            blk[(size_t)r] = (int)(std::upper_bound(bstart.begin(), bstart.end(), i) - bstart.begin()) - 1;
        }
        if (int r = h2d_sync(h, sr.dTask, task.data(), sizeof(int) * ns)) return r;
        if (int r = h2d_sync(h, sr.dBlk, blk.data(), sizeof(int) * ns)) return r;
    }
    if (int r = ensure_buf_sizes(h, p)) return r;
    CUDA_TRY(h, cudaMemsetAsync(h->sbits, 0, sizeof(unsigned long long) * bstart.size(), s));
    CUDA_TRY(h, cudaMemsetAsync(h->w.counters, 0, sizeof(unsigned long long) * kCounters, s));
    int launches = 0;
    const bool want_graph = h->use_graph != 0 && h->prof == nullptr && !sig;
    CUDA_TRY(h, cudaEventRecord(h->tev[2], s));
    if (want_graph) {
        if (!p->graph || p->graph_trace != (h->trace != 0) || p->graph_gen != h->bufgen) {
            if (p->graph) { cudaGraphExecDestroy(p->graph); p->graph = nullptr; }
            cudaGraph_t g;
            CUDA_TRY(h, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int r = run_plan(h, p, &launches);
            cudaError_t ce = cudaStreamEndCapture(s, &g);
            if (r) return r;
            if (ce != cudaSuccess) return fail(h, BRGPU_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
            CUDA_TRY(h, cudaGraphInstantiate(&p->graph, g, 0));
            cudaGraphDestroy(g);
            p->graph_trace = h->trace != 0;
            p->graph_gen = h->bufgen;
            p->launches = launches;
        }
        launches = p->launches;
        CUDA_TRY(h, cudaGraphLaunch(p->graph, s));
        h->stats.graph_replayed = 1;
    } else {
        int r = run_plan(h, p, &launches, h->prof);
        if (r) return r;
        h->stats.graph_replayed = 0;
    }
    CUDA_TRY(h, cudaEventRecord(h->tev[3], s));
    if (p->anySp && p->h_ctl)  // the deflation profile of this solve (adapt_sparse, after the sync)
        CUDA_TRY(h, cudaMemcpyAsync(p->h_ctl, p->d_ctl, sizeof(int) * (size_t)p->nctl, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaGetLastError());
    h->stats.kernel_launches = launches + 2;  // + input copy and scan
    h->stats.n = n;
    h->stats.blocks = (int)bstart.size() - 1;
    h->stats.height = p->height;
    h->stats.merges = (int64_t)p->mOff.size();
    return BRGPU_OK;
}

// Sparse-level configuration from the deflation profile of the last solve
// (k_sp_flag's per-level words: largest NN of a merge, total NN): the cap C
// becomes the next power of two >= max NN (>= the level's merge size when that
// is <= 1024, so such levels stay dense-free), and the group span fills the SMs
// with whole waves of k_sp_solve groups.  Results never depend on it: a level
// whose merges exceed its cap runs the dense pipeline.  A changed configuration
// drops the captured graph (re-captured by the next solve).
void adapt_sparse(Handle* h, Plan* p) {
    if (!p || !p->anySp || !p->h_ctl) return;
    const int capMax = sparse_cap(), room0 = 2 * sparse_cap();
    bool changed = false;
    for (LevelHost& lh : p->levels) {
        if (!lh.sp) continue;
        const int maxNN = p->h_ctl[lh.ctl + 1], tot = p->h_ctl[lh.ctl + 3];
        int cap = capMax, span = room0 - capMax;
        if (maxNN <= capMax && tot >= 0) {
            cap = 64;
            while (cap < maxNN) cap <<= 1;
            if (lh.maxSize <= capMax) while (cap < lh.maxSize) cap <<= 1;
            cap = std::min(cap, capMax);
            const int room = room0 - cap;
            const long long keys = (long long)tot + 4LL * lh.M;
            long long groups = std::max<long long>(1, (keys + room - 1) / room);
            groups = (groups + h->sms - 1) / h->sms * h->sms;
            span = (int)std::max<long long>(kSpMinSpan, std::min<long long>(room, keys / groups));
        }
        if (cap != lh.spCap || span != lh.spSpan) {
            lh.spCap = cap;
            lh.spSpan = span;
            lh.spStatic = lh.maxSize <= cap ? 1 : 0;
            changed = true;
        }
    }
    if (changed && p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
    }
}

int finish_solve(Handle* h) {
    cudaStream_t s = h->stream;
    ledger_peak(h);
    Plan* lp = h->virt <= 1 && h->plan && h->plan->liveLev >= 0 ? h->plan.get() : nullptr;
    h->hsmall[2] = 0;
    CUDA_TRY(h, cudaMemcpyAsync(h->hsmall + 1, h->w.status, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (lp) CUDA_TRY(h, cudaMemcpyAsync(h->hsmall + 2, lp->d_liveCtl + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaMemcpyAsync(h->hcnt, h->w.counters, sizeof(unsigned long long) * kCounters, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    if (lp && h->hsmall[2]) {  // the live tier could not prove this solve exact: redo it densely
        h->liveBackoff = h->liveVeto == lp->n ? std::min(h->liveBackoff * 2, 1 << 16) : kLiveBackoff0;
        h->liveVeto = lp->n;
        h->liveSkip = h->liveBackoff + 1;  // + the retry itself
        return kRetryDense;
    }
    if (lp && h->liveVeto == lp->n) h->liveBackoff = kLiveBackoff0;  // the tier held at this order again
    if (h->virt <= 1) adapt_sparse(h, h->plan.get());
    {
        // both pairs are recorded on every path; a failure here must not leave a
        // pending error for the next CUDA_TRY (of this or any other handle)
        float a = 0.f, b = 0.f;
        if (cudaEventElapsedTime(&a, h->tev[0], h->tev[1]) != cudaSuccess) { a = 0.f; cudaGetLastError(); }
        if (cudaEventElapsedTime(&b, h->tev[2], h->tev[3]) != cudaSuccess) { b = 0.f; cudaGetLastError(); }
        h->timing.pre_ms = a;
        h->timing.main_ms = b;
        h->timing.device_ms = (double)a + (double)b;
        float p1 = 0.f, x = 0.f, p2 = 0.f;
        const bool ok = h->virt <= 1 && h->pev[0] && h->pev[1] &&
                        cudaEventElapsedTime(&p1, h->tev[2], h->pev[0]) == cudaSuccess &&
                        cudaEventElapsedTime(&x, h->pev[0], h->pev[1]) == cudaSuccess &&
                        cudaEventElapsedTime(&p2, h->pev[1], h->tev[3]) == cudaSuccess;
        if (!ok) { cudaGetLastError(); p1 = b; x = 0.f; p2 = 0.f; }
        h->timing.phase1_ms = p1;
        h->timing.exchange_ms = x;
        h->timing.phase2_ms = p2;
    }
    h->stats.evals = (int64_t)(h->hcnt[0] + h->hcnt[2] + h->hcnt[8]);
    h->stats.pole_terms = (double)(h->hcnt[1] + h->hcnt[3] + h->hcnt[9]);
    h->stats.evals_live = (int64_t)h->hcnt[8];
    h->stats.pole_terms_live = (double)h->hcnt[9];
    h->stats.evals_fused = (int64_t)h->hcnt[2];
    h->stats.pole_terms_fused = (double)h->hcnt[3];
    if (h->trace && h->plan) {
        Plan* p = h->plan.get();
        const size_t M = p->mOff.size();
        std::vector<int> tb(2 * M);
        if (M) CUDA_TRY(h, cudaMemcpy(tb.data(), h->traceBuf, sizeof(int) * 2 * M, cudaMemcpyDeviceToHost));
        h->traceRecs.resize(M);
        double sk2 = 0, szt = 0, k2f = 0, k2g = 0, k2l = 0;
        int64_t sk = 0, snn = 0, mk = 0, nng = 0, kg = 0;
        std::vector<char> fusedMerge(M, 0);  // 1 fused tier, 2 live tier
        for (const auto* lv : {&p->levels, &p->levels2})
            for (const LevelHost& lh : *lv)
                for (int q = 0; q < lh.M; ++q) fusedMerge[(size_t)(lh.m0 + q)] = lh.fused ? 1 : lh.live ? 2 : 0;
        for (size_t m = 0; m < M; ++m) {
            brgpu_trace& t = h->traceRecs[m];
            t.level = p->mLevel[m];
            t.is_root = p->mFlags[m] & kMergeRoot;
            t.offset = p->mOff[m];
            t.size = p->mSize[m];
            t.nn = tb[2 * m];
            t.k = tb[2 * m + 1];
            sk += t.k; snn += t.nn; sk2 += (double)t.k * (double)t.k;
            if (!fusedMerge[m]) { nng += t.nn; kg += t.k; }
            if (!t.is_root) {
                szt += (double)t.k * (double)t.k;
                (fusedMerge[m] == 1 ? k2f : fusedMerge[m] == 2 ? k2l : k2g) += (double)t.k * (double)t.k;
            }
            mk = std::max<int64_t>(mk, t.k);
        }
        h->stats.sum_k = sk; h->stats.sum_k2 = sk2; h->stats.sum_nn = snn;
        h->stats.row_terms = szt; h->stats.zhat_terms = h->zhat ? szt : 0.0; h->stats.max_k = mk;
        h->stats.rotations = snn - sk;
        h->stats.k2_nonroot_fused = k2f;
        h->stats.k2_nonroot_grid = k2g;
        h->stats.k2_nonroot_live = k2l;
        h->stats.nn_grid = nng;
        h->stats.k_grid = kg;
    }
    if (h->hsmall[1]) return status_message(h, h->hsmall[1]);
    return BRGPU_OK;
}

int solve_device(Handle* h, int64_t n64, const double* d, const double* e, double* w_out,
                 bool w_host) {
    if (n64 <= 0 || n64 >= (int64_t)1 << 31) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "tridiagonal: order must be positive (and < 2^31)");
    const int n = (int)n64;
    if (int r = ensure_work(h, work_need(h, n64))) return r;
    cudaStream_t s = h->stream;
    CUDA_TRY(h, cudaMemsetAsync(h->dsmall, 0, sizeof(int) * 2, s));
    CUDA_TRY(h, cudaMemsetAsync(h->w.status, 0, sizeof(int), s));
    CUDA_TRY(h, cudaEventRecord(h->tev[0], s));
    launch_copy_input(s, n, d, e, h->w.dw, h->w.ew);
    launch_scan_input(s, n, h->w.dw, h->w.ew, h->split, h->dsmall, h->w.status);
    CUDA_TRY(h, cudaEventRecord(h->tev[1], s));
    int r = solve_prepared(h, n, {0, n});
    if (r) return r;
    if (w_host)
        CUDA_TRY(h, cudaMemcpyAsync(w_out, h->w.lam, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    else if (w_out != h->w.lam)
        CUDA_TRY(h, cudaMemcpyAsync(w_out, h->w.lam, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    r = finish_solve(h);
    // the live tier fell back (liveSkip: the next plans of this order are dense); inputs
    // staged in the workspace (brgpu_eigvals) are re-staged by the caller
    if (r == kRetryDense && d != h->w.D && e != h->w.Z) return solve_device(h, n64, d, e, w_out, w_host);
    return r;
}

}  // namespace

struct brgpu_handle {
    Handle h;
};

extern "C" {

const char* brgpu_version(void) { return kVersion; }

const char* brgpu_status_string(int st) {
    switch (st) {
        case BRGPU_OK: return "ok";
        case BRGPU_ERR_INVALID_ARGUMENT: return "InvalidArgument";
        case BRGPU_ERR_NO_CONVERGENCE: return "NoConvergence";
        case BRGPU_ERR_BUDGET_EXCEEDED: return "BudgetExceeded";
        case BRGPU_ERR_POLE_HIT: return "PoleHit";
        case BRGPU_ERR_ZERO_DENOMINATOR: return "ZeroDenominator";
        case BRGPU_ERR_MALFORMED_COMPACT_ROOT: return "MalformedCompactRoot";
        case BRGPU_ERR_DIMENSION_MISMATCH: return "DimensionMismatch";
        case BRGPU_ERR_DOMAIN_ERROR: return "DomainError";
        case BRGPU_ERR_OUT_OF_MEMORY: return "OutOfMemory";
        case BRGPU_ERR_CUDA: return "CudaError";
        case BRGPU_ERR_NCCL: return "NcclError";
        case BRGPU_ERR_NO_DEVICE: return "NoDevice";
        default: return "unknown";
    }
}

int brgpu_create(brgpu_handle** out, int device) {
    if (!out) return BRGPU_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return BRGPU_ERR_NO_DEVICE;
    }
    if (device < 0 || device >= ndev) return BRGPU_ERR_INVALID_ARGUMENT;
    auto* hh = new brgpu_handle();
    Handle* h = &hh->h;
    h->device = device;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMallocHost(&h->hsmall, sizeof(int) * 4) != cudaSuccess ||
        cudaMallocHost(&h->hcnt, sizeof(unsigned long long) * kCounters) != cudaSuccess ||
        cudaMalloc(&h->dsmall, sizeof(int) * 4) != cudaSuccess ||
        cudaEventCreate(&h->tev[0]) != cudaSuccess || cudaEventCreate(&h->tev[1]) != cudaSuccess ||
        cudaEventCreate(&h->tev[2]) != cudaSuccess || cudaEventCreate(&h->tev[3]) != cudaSuccess ||
        cudaEventCreate(&h->pev[0]) != cudaSuccess || cudaEventCreate(&h->pev[1]) != cudaSuccess) {
        delete hh;
        return BRGPU_ERR_CUDA;
    }
    brgpu::init_kernel_attributes();
    brgpu::init_fused_attributes();
    brgpu::init_sparse_attributes();
    brgpu::init_warp_attributes();
    brgpu::init_live_attributes();
    cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
    h->sec_grid = h->sms * brgpu::sec_ctas_per_sm();
    *out = hh;
    return BRGPU_OK;
}

int brgpu_destroy(brgpu_handle* hh) {
    if (!hh) return BRGPU_OK;
    Handle* h = &hh->h;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (auto& u : h->subs) {
        if (u->plan) free_plan(u->plan.get());
        free_work(u.get());
        if (u->sbits) cudaFree(u->sbits);
        if (u->mTol) cudaFree(u->mTol);
        if (u->traceBuf) cudaFree(u->traceBuf);
        if (u->strBuf) cudaFree(u->strBuf);
    }
    h->subs.clear();
    if (h->comm && nccl_api().ok) nccl_api().CommDestroy(h->comm);
    h->comm = nullptr;
    if (h->plan) free_plan(h->plan.get());
    free_work(h);
    if (h->sbits) cudaFree(h->sbits);
    if (h->mTol) cudaFree(h->mTol);
    if (h->traceBuf) cudaFree(h->traceBuf);
    if (h->strBuf) cudaFree(h->strBuf);
    if (h->pinned) cudaFreeHost(h->pinned);
    if (h->hsmall) cudaFreeHost(h->hsmall);
    if (h->hcnt) cudaFreeHost(h->hcnt);
    if (h->dsmall) cudaFree(h->dsmall);
    if (h->sigDbl) cudaFree(h->sigDbl);
    if (h->sigInt) cudaFree(h->sigInt);
    for (auto& e : h->tev) if (e) cudaEventDestroy(e);
    for (auto& e : h->pev) if (e) cudaEventDestroy(e);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete hh;
    return BRGPU_OK;
}

const char* brgpu_last_error_message(const brgpu_handle* hh) { return hh ? hh->h.err.c_str() : "null handle"; }

static void set_plan_opt(Handle* h, int& field, int v) {
    if (field == v) return;
    field = v;
    if (h->plan) { free_plan(h->plan.get()); h->plan.reset(); }
}

int brgpu_set_option(brgpu_handle* hh, int opt, int64_t v) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    switch (opt) {
        case BRGPU_OPT_LEAF_CUTOFF:
            if (v < 5 || v > 32) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "leaf cutoff must be in [5, 32]");
            h->leaf_cutoff = (int)v;
            return BRGPU_OK;
        // options that change the plan drop the cached plan (and its graph) only
        // when their value actually changes, so re-applying the same options is free
        case BRGPU_OPT_ZHAT: set_plan_opt(h, h->zhat, v != 0); return BRGPU_OK;
        case BRGPU_OPT_PATCHED_STOP: set_plan_opt(h, h->patched, v != 0); return BRGPU_OK;
        case BRGPU_OPT_USE_GRAPH: h->use_graph = v != 0; return BRGPU_OK;
        case BRGPU_OPT_SUBTREE: set_plan_opt(h, h->subtree, v != 0); return BRGPU_OK;
        case BRGPU_OPT_EXACT_PASSES:
            set_plan_opt(h, h->exact, v != 0);
            h->w.exact = h->exact;
            return BRGPU_OK;
        case BRGPU_OPT_ROOT_SPLIT: set_plan_opt(h, h->root_split, v != 0); return BRGPU_OK;
        case BRGPU_OPT_SPARSE: set_plan_opt(h, h->sparse, v != 0); return BRGPU_OK;
        case BRGPU_OPT_LIVE: set_plan_opt(h, h->live, v != 0); h->liveVeto = h->liveSkip = 0; return BRGPU_OK;
        case BRGPU_OPT_LIVE_CLUSTER: set_plan_opt(h, h->liveCluster, v != 0); return BRGPU_OK;
        case BRGPU_OPT_LIVE_FLOW: set_plan_opt(h, h->liveFlow, v != 0); return BRGPU_OK;
        case BRGPU_OPT_VIRTUAL_RANKS:
            if (v < 1 || v > 64) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "virtual ranks must be in [1, 64]");
            if (h->nranks > 1) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "virtual ranks on a distributed handle");
            h->virt = (int)v;
            return BRGPU_OK;
        default: return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "unknown option");
    }
}

int brgpu_get_option(const brgpu_handle* hh, int opt, int64_t* v) {
    if (!hh || !v) return BRGPU_ERR_INVALID_ARGUMENT;
    const Handle* h = &hh->h;
    switch (opt) {
        case BRGPU_OPT_LEAF_CUTOFF: *v = h->leaf_cutoff; return BRGPU_OK;
        case BRGPU_OPT_ZHAT: *v = h->zhat; return BRGPU_OK;
        case BRGPU_OPT_PATCHED_STOP: *v = h->patched; return BRGPU_OK;
        case BRGPU_OPT_USE_GRAPH: *v = h->use_graph; return BRGPU_OK;
        case BRGPU_OPT_SUBTREE: *v = h->subtree; return BRGPU_OK;
        case BRGPU_OPT_VIRTUAL_RANKS: *v = h->virt; return BRGPU_OK;
        case BRGPU_OPT_ROOT_SPLIT: *v = h->root_split; return BRGPU_OK;
        case BRGPU_OPT_EXACT_PASSES: *v = h->exact; return BRGPU_OK;
        case BRGPU_OPT_SPARSE: *v = h->sparse; return BRGPU_OK;
        case BRGPU_OPT_LIVE: *v = h->live; return BRGPU_OK;
        case BRGPU_OPT_LIVE_CLUSTER: *v = h->liveCluster; return BRGPU_OK;
        case BRGPU_OPT_LIVE_FLOW: *v = h->liveFlow; return BRGPU_OK;
        default: return BRGPU_ERR_INVALID_ARGUMENT;
    }
}

int brgpu_workspace_query(int64_t n, int64_t* doubles, int64_t* ints) {
    if (n <= 0) return BRGPU_ERR_INVALID_ARGUMENT;
    if (doubles) *doubles = 16 * n;
    if (ints) *ints = 7 * n;
    return BRGPU_OK;
}

int brgpu_reserve(brgpu_handle* hh, int64_t n) {
    if (!hh || n <= 0) return BRGPU_ERR_INVALID_ARGUMENT;
    cudaSetDevice(hh->h.device);
    return ensure_work(&hh->h, work_need(&hh->h, n));
}

int brgpu_get_ledger(const brgpu_handle* hh, brgpu_ledger* out) {
    if (!hh || !out) return BRGPU_ERR_INVALID_ARGUMENT;
    const Handle* h = &hh->h;
    int64_t dbl = 0, ints = 0;
    ledger_now(h, dbl, ints);
    out->live_doubles = dbl;
    out->peak_doubles = std::max(h->peak_doubles, dbl);
    out->live_ints = ints;
    out->peak_ints = std::max(h->peak_ints, ints);
    out->limit_doubles = 16 * h->limit_n;
    out->limit_ints = 7 * h->limit_n;
    out->rows_doubles = h->sigDblCap + h->strCap;  // requested rows + the secular-trace diagnostic buffer
    out->rows_ints = h->sigIntCap;
    return BRGPU_OK;
}

int brgpu_eigvals(brgpu_handle* hh, int64_t n, const double* d, const double* e, double* w) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (n <= 0 || !d || !w || (n > 1 && !e)) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "tridiagonal: order must be positive");
    if (n >= (int64_t)1 << 31) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "tridiagonal: order must be < 2^31");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (int r = ensure_work(h, work_need(h, n))) return r;
    // host buffers are staged in workspace arrays that are dead until the first
    // merge (D, Z), so the host path needs no memory beyond the 15N arena
    cudaStream_t s = h->stream;
    int r = BRGPU_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {  // a live-tier fallback re-stages the input
        CUDA_TRY(h, cudaMemcpyAsync(h->w.D, d, sizeof(double) * n, cudaMemcpyHostToDevice, s));
        if (n > 1) CUDA_TRY(h, cudaMemcpyAsync(h->w.Z, e, sizeof(double) * (n - 1), cudaMemcpyHostToDevice, s));
        r = solve_device(h, n, h->w.D, h->w.Z, w, true);
        if (r != kRetryDense) break;
    }
    return r;
}

int brgpu_eigvals_device(brgpu_handle* hh, int64_t n, const double* d, const double* e, double* w,
                         void* stream) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (n <= 0 || !d || !w || (n > 1 && !e)) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "tridiagonal: order must be positive");
    CUDA_TRY(h, cudaSetDevice(h->device));
    cudaStream_t user = (cudaStream_t)stream;
    cudaEvent_t ev = nullptr;
    if (user) {
        // order the handle stream after the caller's stream
        CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventRecord(ev, user));
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, ev, 0));
        cudaEventDestroy(ev);
    }
    return solve_device(h, n, d, e, w, false);
}

// Eigenvalues plus requested eigenvector rows (Algorithm 1's sigma,
// SPEC.md:317-337): rows[r*n + j] = Q(sel[r], j), columns in the order of w.
// The solve runs every level through the grid tier with the sigma kernels
// (sigma.cu) attached, outside the cached eigenvalue-only graph.
int brgpu_eigvals_rows(brgpu_handle* hh, int64_t n, const double* d, const double* e, int64_t nsel,
                       const int64_t* sel, double* w, double* rows) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (n <= 0 || n >= ((int64_t)1 << 31) || !d || !w || (n > 1 && !e))
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "tridiagonal: order must be positive (and < 2^31)");
    if (nsel < 0 || (nsel > 0 && (!sel || !rows)))
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "selected rows: negative count or null pointers");
    for (int64_t r = 0; r < nsel; ++r)
        if (sel[r] < 0 || sel[r] >= n)
            return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "selected rows: row index " + std::to_string(sel[r]) +
                                                           " outside [0, " + std::to_string(n) + ")");
    if (nsel == 0) return brgpu_eigvals(hh, n, d, e, w);
    if (h->nranks > 1 || h->virt > 1)
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "selected rows: single-device handles only");
    if (nsel > ((int64_t)1 << 30) / std::max<int64_t>(n, 1))
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "selected rows: nsel * n too large");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (int r = ensure_work(h, n)) return r;
    const int64_t c = h->cap;
    Handle::SigmaRun sr;
    sr.sel.assign(sel, sel + nsel);
    auto grow = [&](auto*& p, int64_t& cap, int64_t need) -> bool {
        if (need <= cap) return true;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, sizeof(*p) * (size_t)need) != cudaSuccess) { cudaGetLastError(); return false; }
        cap = need;
        return true;
    };
    if (!grow(h->sigDbl, h->sigDblCap, (3 * nsel + 1) * c + nsel * n) || !grow(h->sigInt, h->sigIntCap, 3 * nsel))
        return fail(h, BRGPU_ERR_CUDA, "selected rows: out of device memory");
    double* dbl = h->sigDbl;
    int* ib = h->sigInt;
    std::vector<int> s32(sr.sel.begin(), sr.sel.end());
    int rc = BRGPU_OK;
    if (cudaMemcpyAsync(ib, s32.data(), sizeof(int) * (size_t)nsel, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
        cudaStreamSynchronize(h->stream) != cudaSuccess)
        rc = fail(h, BRGPU_ERR_CUDA, "selected rows: copy of the request failed");
    sr.dev.nsel = (int)nsel;
    sr.dev.stride = c;
    sr.dev.sel = ib;
    sr.dev.S = dbl;
    sr.dev.X = dbl + nsel * c;
    sr.dev.XA = dbl + 2 * nsel * c;
    sr.dev.Z0 = dbl + 3 * nsel * c;
    sr.out = dbl + (3 * nsel + 1) * c;
    sr.dTask = ib + nsel;
    sr.dBlk = ib + 2 * nsel;
    if (!rc && cudaMemsetAsync(sr.out, 0, sizeof(double) * (size_t)(nsel * n), h->stream) != cudaSuccess)
        rc = fail(h, BRGPU_ERR_CUDA, "selected rows: memset failed");
    if (!rc) {
        h->sig = &sr;
        rc = brgpu_eigvals(hh, n, d, e, w);
        h->sig = nullptr;
        if (!rc && (cudaMemcpyAsync(rows, sr.out, sizeof(double) * (size_t)(nsel * n), cudaMemcpyDeviceToHost,
                                    h->stream) != cudaSuccess || cudaStreamSynchronize(h->stream) != cudaSuccess))
            rc = fail(h, BRGPU_ERR_CUDA, "selected rows: copy of the rows failed");
    }
    return rc;
}

// ---------------------------------------------------------------------------
// Upstream neighbour ("reduced dense"):
// dense symmetric -> tridiagonal by cuSOLVER dsytrd (library call, dlopen'ed so
// the product has no link-time dependency), then the BR solve.
// ---------------------------------------------------------------------------
struct CusolverApi {
    bool ok = false;
    using H = void*;
    int (*Create)(H*) = nullptr;
    int (*Destroy)(H) = nullptr;
    int (*SetStream)(H, cudaStream_t) = nullptr;
    int (*BufSize)(H, int, int, const double*, int, const double*, const double*, const double*, int*) = nullptr;
    int (*Sytrd)(H, int, int, double*, int, double*, double*, double*, double*, int, int*) = nullptr;
};

CusolverApi& cusolver_api() {
    static CusolverApi api = [] {
        CusolverApi a;
        void* lib = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) return a;
        a.Create = (decltype(a.Create))dlsym(lib, "cusolverDnCreate");
        a.Destroy = (decltype(a.Destroy))dlsym(lib, "cusolverDnDestroy");
        a.SetStream = (decltype(a.SetStream))dlsym(lib, "cusolverDnSetStream");
        a.BufSize = (decltype(a.BufSize))dlsym(lib, "cusolverDnDsytrd_bufferSize");
        a.Sytrd = (decltype(a.Sytrd))dlsym(lib, "cusolverDnDsytrd");
        a.ok = a.Create && a.Destroy && a.SetStream && a.BufSize && a.Sytrd;
        return a;
    }();
    return api;
}

int brgpu_eigvals_dense_device(brgpu_handle* hh, int64_t n64, double* A, int64_t lda, double* w, void* stream) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (n64 <= 0 || n64 >= (int64_t)1 << 31 || !A || !w || lda < n64)
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "dense: order must be positive and lda >= n");
    CusolverApi& C = cusolver_api();
    if (!C.ok) return fail(h, BRGPU_ERR_CUDA, "dense: libcusolver not available");
    CUDA_TRY(h, cudaSetDevice(h->device));
    const int n = (int)n64;
    cudaStream_t user = (cudaStream_t)stream;
    if (user) {
        cudaEvent_t ev = nullptr;
        CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventRecord(ev, user));
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, ev, 0));
        cudaEventDestroy(ev);
    }
    void* sh = nullptr;
    if (C.Create(&sh) != 0) return fail(h, BRGPU_ERR_CUDA, "dense: cusolverDnCreate failed");
    C.SetStream(sh, h->stream);
    double *buf = nullptr;
    int* info = nullptr;
    int lwork = 0;
    constexpr int kLower = 0;  // CUBLAS_FILL_MODE_LOWER
    int rc = BRGPU_OK;
    if (C.BufSize(sh, kLower, n, A, (int)lda, nullptr, nullptr, nullptr, &lwork) != 0) {
        rc = fail(h, BRGPU_ERR_CUDA, "dense: dsytrd_bufferSize failed");
    } else if (cudaMalloc(&buf, sizeof(double) * ((size_t)3 * n + (size_t)lwork)) != cudaSuccess ||
               cudaMalloc(&info, sizeof(int)) != cudaSuccess) {
        rc = fail(h, BRGPU_ERR_CUDA, "dense: workspace allocation failed");
    } else {
        double* d = buf;
        double* e = buf + n;
        double* tau = buf + 2 * (size_t)n;
        double* work = buf + 3 * (size_t)n;
        if (C.Sytrd(sh, kLower, n, A, (int)lda, d, e, tau, work, lwork, info) != 0)
            rc = fail(h, BRGPU_ERR_CUDA, "dense: dsytrd failed");
        else
            rc = solve_device(h, n, d, e, w, false);  // synchronises the handle stream
    }
    cudaFree(buf);
    cudaFree(info);
    C.Destroy(sh);
    return rc;
}

int brgpu_eigvals_batched_device(brgpu_handle* hh, int64_t batch, int64_t n, const double* d,
                                 const double* e, double* w, void* stream) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (batch <= 0 || n <= 0 || !d || !w || (n > 1 && !e)) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "batched: bad sizes");
    const int64_t N = batch * n;
    if (N >= (int64_t)1 << 31) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "batched: batch*n must be < 2^31");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (stream) {
        cudaEvent_t ev;
        CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CUDA_TRY(h, cudaEventRecord(ev, (cudaStream_t)stream));
        CUDA_TRY(h, cudaStreamWaitEvent(h->stream, ev, 0));
        cudaEventDestroy(ev);
    }
    if (int r = ensure_work(h, work_need(h, N))) return r;
    cudaStream_t s = h->stream;
    CUDA_TRY(h, cudaMemsetAsync(h->dsmall, 0, sizeof(int) * 2, s));
    CUDA_TRY(h, cudaMemsetAsync(h->w.status, 0, sizeof(int), s));
    CUDA_TRY(h, cudaEventRecord(h->tev[0], s));
    launch_scan_input_batched(s, (int)batch, (int)n, d, e, h->w.dw, h->w.ew, h->split, h->dsmall, h->w.status);
    CUDA_TRY(h, cudaEventRecord(h->tev[1], s));
    std::vector<int> segs;
    for (int64_t b = 0; b <= batch; ++b) segs.push_back((int)(b * n));
    int r = solve_prepared(h, (int)N, segs);
    if (r) return r;
    if (w != h->w.lam)
        CUDA_TRY(h, cudaMemcpyAsync(w, h->w.lam, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    r = finish_solve(h);
    // live-tier fallback: redo densely (inputs staged in the workspace: the caller re-stages)
    if (r == kRetryDense && d != h->w.D && e != h->w.Z) return brgpu_eigvals_batched_device(hh, batch, n, d, e, w, nullptr);
    return r;
}

int brgpu_eigvals_batched(brgpu_handle* hh, int64_t batch, int64_t n, const double* d,
                          const double* e, double* w) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (batch <= 0 || n <= 0 || !d || !w || (n > 1 && !e)) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "batched: bad sizes");
    const int64_t N = batch * n;
    if (N >= (int64_t)1 << 31) return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "batched: batch*n must be < 2^31");
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (int r = ensure_work(h, work_need(h, N))) return r;
    // staged in the workspace's D / Z arrays (dead until the first merge); the
    // result is read straight from lam
    cudaStream_t s = h->stream;
    int r = BRGPU_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {  // a live-tier fallback re-stages the input
        CUDA_TRY(h, cudaMemcpyAsync(h->w.D, d, sizeof(double) * N, cudaMemcpyHostToDevice, s));
        if (n > 1) CUDA_TRY(h, cudaMemcpyAsync(h->w.Z, e, sizeof(double) * batch * (n - 1), cudaMemcpyHostToDevice, s));
        r = brgpu_eigvals_batched_device(hh, batch, n, h->w.D, h->w.Z, h->w.lam, nullptr);
        if (r != kRetryDense) break;
    }
    if (r) return r;
    CUDA_TRY(h, cudaMemcpyAsync(w, h->w.lam, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(h, cudaStreamSynchronize(s));
    return BRGPU_OK;
}

int brgpu_get_stats(const brgpu_handle* hh, brgpu_stats* out) {
    if (!hh || !out) return BRGPU_ERR_INVALID_ARGUMENT;
    *out = hh->h.stats;
    return BRGPU_OK;
}

int brgpu_phase_cycles(brgpu_handle* hh, uint64_t* out4) {
    if (!hh || !out4) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (!h->w.counters) { for (int k = 0; k < 4; ++k) out4[k] = 0; return BRGPU_OK; }
    CUDA_TRY(h, cudaMemcpy(out4, h->w.counters + 4, sizeof(uint64_t) * 4, cudaMemcpyDeviceToHost));
    return BRGPU_OK;
}

int brgpu_get_timing(const brgpu_handle* hh, brgpu_timing* out) {
    if (!hh || !out) return BRGPU_ERR_INVALID_ARGUMENT;
    *out = hh->h.timing;
    return BRGPU_OK;
}

const char* brgpu_kernel_class_name(int c) {
    static const char* names[BRGPU_NCLASS] = {
        "prepare(scale+cuts)", "leaf", "merge_tol", "merge_scatter", "nn_flag", "scan_tiles",
        "nn_write", "segment_walk", "surv_count", "surv_write", "secular", "zhat", "rows",
        "deflated_out", "trace", "finish", "fused_level", "sparse_flag", "sparse_solve", "sparse_place",
        "live_level", "live_sort"};
    return (c >= 0 && c < BRGPU_NCLASS) ? names[c] : "?";
}

static int profile_impl(brgpu_handle* hh, int64_t batch, int64_t n, const double* d, const double* e,
                        double* class_ms, int32_t* class_launches) {
    if (!hh || !class_ms || !class_launches) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    CUDA_TRY(h, cudaSetDevice(h->device));
    if (n <= 0 || batch < 0 || (batch && n > (((int64_t)1 << 31) - 1) / batch))
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "profile: bad sizes");
    // the result lands in the workspace's own lam array: size the workspace
    // first, so a fresh (or smaller) handle never hands out a null or stale pointer
    if (int r0 = ensure_work(h, work_need(h, batch ? batch * n : n))) return r0;
    Prof prof;
    h->prof = &prof;
    const int r = batch ? brgpu_eigvals_batched_device(hh, batch, n, d, e, h->w.lam, nullptr)
                        : solve_device(h, n, d, e, h->w.lam, false);
    h->prof = nullptr;
    for (int c = 0; c < BRGPU_NCLASS; ++c) { class_ms[c] = 0.0; class_launches[c] = 0; }
    if (r == BRGPU_OK) {
        cudaStreamSynchronize(h->stream);
        const bool dump = std::getenv("BRGPU_PROF_DUMP") != nullptr;  // per-mark listing (tooling)
        for (size_t i = 1; i < prof.ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, prof.ev[i - 1], prof.ev[i]);
            const int c = prof.cls[i];
            if (dump) std::fprintf(stderr, "[prof] %zu %s %.4f\n", i, brgpu_kernel_class_name(c), ms);
            if (c >= 0 && c < BRGPU_NCLASS) { class_ms[c] += ms; class_launches[c] += 1; }
        }
    }
    for (auto e2 : prof.ev) cudaEventDestroy(e2);
    return r;
}

int brgpu_profile_kernels(brgpu_handle* hh, int64_t n, const double* d, const double* e,
                          double* class_ms, int32_t* class_launches) {
    return profile_impl(hh, 0, n, d, e, class_ms, class_launches);
}

int brgpu_profile_kernels_batched(brgpu_handle* hh, int64_t batch, int64_t n, const double* d,
                                  const double* e, double* class_ms, int32_t* class_launches) {
    if (batch <= 0) return BRGPU_ERR_INVALID_ARGUMENT;
    return profile_impl(hh, batch, n, d, e, class_ms, class_launches);
}

int brgpu_selftest_rcp(brgpu_handle* hh, int64_t count, uint64_t seed, uint64_t* mismatches) {
    if (!hh || !mismatches || count <= 0) return BRGPU_ERR_INVALID_ARGUMENT;
    cudaSetDevice(hh->h.device);
    unsigned long long bad = 0;
    const int r = brgpu::selftest_rcp(count, seed, &bad);
    *mismatches = bad;
    return r;
}

int brgpu_nccl_unique_id(void* out) {
    NcclApi& N = nccl_api();
    if (!out) return BRGPU_ERR_INVALID_ARGUMENT;
    if (!N.ok) return BRGPU_ERR_NCCL;
    ncclUniqueId id;
    if (N.GetUniqueId(&id) != ncclSuccess) return BRGPU_ERR_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return BRGPU_OK;
}

int brgpu_create_distributed(brgpu_handle** out, int device, int rank, int nranks, const void* unique_id) {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !unique_id))
        return BRGPU_ERR_INVALID_ARGUMENT;
    int rc = brgpu_create(out, device);
    if (rc) return rc;
    Handle* h = &(*out)->h;
    h->nranks = nranks;
    h->rank = rank;
    if (nranks > 1) {
        NcclApi& N = nccl_api();
        if (!N.ok) { brgpu_destroy(*out); *out = nullptr; return BRGPU_ERR_NCCL; }
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof(id));
        if (N.CommInitRank(&h->comm, nranks, id, rank) != ncclSuccess) {
            brgpu_destroy(*out);
            *out = nullptr;
            return BRGPU_ERR_NCCL;
        }
    }
    return BRGPU_OK;
}

int brgpu_plan_owned(int64_t n, int32_t leaf_cutoff, int32_t nranks, const int32_t* bstart, int32_t nblk,
                     int32_t* counts, int32_t* ranges, int32_t cap) {
    if (n <= 0 || nranks < 1 || !counts || leaf_cutoff < 5) return BRGPU_ERR_INVALID_ARGUMENT;
    std::vector<int> b;
    if (bstart && nblk > 0) b.assign(bstart, bstart + nblk + 1);
    else b = {0, (int)n};
    auto p = make_plan((int)n, leaf_cutoff, b, {0, (int)n}, true, nranks, 0);
    for (int k = 0; k < nranks; ++k) {
        const auto& ow = p->owned[(size_t)k];
        counts[k] = (int32_t)ow.size();
        for (int q = 0; q < (int)ow.size() && q < cap && ranges; ++q) {
            ranges[2 * (k * cap + q)] = ow[(size_t)q].first;
            ranges[2 * (k * cap + q) + 1] = ow[(size_t)q].second;
        }
    }
    return BRGPU_OK;
}

int brgpu_set_trace(brgpu_handle* hh, int enable) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    hh->h.trace = enable != 0;
    return BRGPU_OK;
}

int brgpu_set_secular_trace(brgpu_handle* hh, int enable) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    Handle* h = &hh->h;
    if (enable && (h->nranks > 1 || h->virt > 1))
        return fail(h, BRGPU_ERR_INVALID_ARGUMENT, "secular trace: single-device handles only");
    set_plan_opt(h, h->strace, enable != 0);
    if (enable) h->trace = 1;  // the per-merge K's locate each merge's entries
    return BRGPU_OK;
}

int brgpu_get_secular_trace(const brgpu_handle* hh, double* out, int64_t cap, int64_t* len) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    const Handle* h = &hh->h;
    const Plan* p = h->plan.get();
    if (!h->strace || !p || !h->strBuf) return BRGPU_ERR_INVALID_ARGUMENT;
    const int64_t n = p->n;
    const size_t nlev = p->levels.size() + p->levels2.size();
    const int64_t M = (int64_t)p->mOff.size();
    std::vector<double> buf((size_t)(2 * n * (int64_t)nlev + M));
    if (!buf.empty() && cudaMemcpy(buf.data(), h->strBuf, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return BRGPU_ERR_CUDA;
    // rho per merge, then each merge's (d, z) pairs in trace order
    std::vector<double> res(buf.begin() + 2 * n * (int64_t)nlev, buf.end());
    size_t li2 = 0;
    for (const auto* lv : {&p->levels, &p->levels2})
        for (const LevelHost& lh : *lv) {
            int64_t g = 0;  // level-global active index (merges in offset order)
            for (int q = 0; q < lh.M; ++q) {
                const int64_t K = h->traceRecs.size() > (size_t)(lh.m0 + q) ? h->traceRecs[(size_t)(lh.m0 + q)].k : 0;
                for (int64_t j = 0; j < K; ++j) {
                    res.push_back(buf[(size_t)(2 * n * (int64_t)li2 + 2 * (g + j))]);
                    res.push_back(buf[(size_t)(2 * n * (int64_t)li2 + 2 * (g + j) + 1)]);
                }
                g += K;
            }
            ++li2;
        }
    if (len) *len = (int64_t)res.size();
    if (out) std::copy(res.begin(), res.begin() + std::min<int64_t>(cap, (int64_t)res.size()), out);
    return BRGPU_OK;
}

int brgpu_get_trace(const brgpu_handle* hh, brgpu_trace* out, int64_t cap, int64_t* len) {
    if (!hh) return BRGPU_ERR_INVALID_ARGUMENT;
    const auto& v = hh->h.traceRecs;
    if (len) *len = (int64_t)v.size();
    if (out) for (int64_t i = 0; i < cap && i < (int64_t)v.size(); ++i) out[i] = v[(size_t)i];
    return BRGPU_OK;
}

}  // extern "C"
