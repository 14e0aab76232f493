// level_state.cuh -- which slot holds a level's node state, and which path runs it.
//
// The node state (lam, blo, bhi) of the current tree level lives in one of two
// slots of the workspace: slot 0 = (lam, blo, bhi), slot 1 = (D, R0, R1).  The
// dense grid pipeline and the fused kernels work in place (the merged copies
// they need go to the other slot's arrays); the sparse pipeline (sparse.cu)
// reads the children from one slot and writes the parents to the other.  Which
// path a level takes is decided on the device (k_sp_flag: every merge has at
// most C non-negligible poles), so the slot is a device word too: the first
// kernel of a level derives it from the previous level's words and publishes
// it in ctl[0]; every later kernel of the level reads ctl[0] and views the
// workspace through with_slot().
#pragma once

#include "internal.hpp"

namespace brgpu {

__device__ __forceinline__ bool prev_sparse(const LevelDev& L) {
    return L.pctl && L.pcap > 0 && L.pctl[1] <= L.pcap;
}

// slot at the start of this level, from the previous level's words (first kernel)
__device__ __forceinline__ int slot_from_prev(const LevelDev& L) {
    if (!L.pctl) return 0;
    return L.pctl[0] ^ (prev_sparse(L) ? 1 : 0);
}

// slot at the start of this level (any kernel after the level's first)
__device__ __forceinline__ int level_slot(const LevelDev& L) { return L.ctl ? L.ctl[0] : 0; }

// does this level run the sparse pipeline? (valid after k_sp_flag)
__device__ __forceinline__ bool level_sparse(const LevelDev& L) {
    return L.spCap > 0 && (L.spStatic || L.ctl[1] <= L.spCap);
}

__device__ __forceinline__ Work with_slot(Work w, int slot) {
    if (slot) {
        double* t;
        t = w.lam; w.lam = w.D; w.D = t;
        t = w.blo; w.blo = w.R0; w.R0 = t;
        t = w.bhi; w.bhi = w.R1; w.R1 = t;
    }
    return w;
}

// Entry of a dense-path level kernel (kernels.cu, tiled.cu, warp.cu): false
// when the level runs sparse (the kernel exits); w = the level's view.  Every
// thread of the CTA calls it; one thread reads the level words (a grid-wide
// read of one L2 line by every warp is a hot spot at the top levels).
__device__ __forceinline__ bool dense_entry(const Work& w0, const LevelDev& L, Work& w) {
    __shared__ int s_ctl[2];
    if (threadIdx.x == 0) {
        s_ctl[0] = L.ctl ? L.ctl[0] : 0;
        s_ctl[1] = L.spCap > 0 ? L.ctl[1] : 0;
    }
    __syncthreads();
    if (L.spCap > 0 && (L.spStatic || s_ctl[1] <= L.spCap)) return false;
    w = with_slot(w0, s_ctl[0]);
    return true;
}

}  // namespace brgpu
