// level_state.cuh -- which path a grid level takes (sparse.cu or the dense pipeline).
//
// A sparse-capable level (LevelDev::spCap > 0) is decided on the device by
// k_sp_flag (every merge has at most spCap non-negligible poles, ctl[1]); the
// dense kernels of such a level exit at once when it runs sparse.  The node
// state is in (lam, blo, bhi) at every level boundary: the sparse pipeline
// places the parents in (D, R0, R1) and copies them back (k_sp_home).
#pragma once

#include "internal.hpp"

namespace brgpu {

// does this level run the sparse pipeline? (valid after k_sp_flag)
__device__ __forceinline__ bool level_sparse(const LevelDev& L) {
    return L.spCap > 0 && (L.spStatic || L.ctl[1] <= L.spCap);
}

// Entry of a dense-path level kernel: false when the level runs sparse (the
// kernel exits).  Every thread of the CTA calls it; on sparse-capable levels one
// thread reads the level word (a grid-wide read of one L2 line by every warp is
// a hot spot at the top levels).
__device__ __forceinline__ bool dense_entry(const LevelDev& L) {
    if (L.spCap == 0) return true;  // uniform: dense-only level
    __shared__ int s_sp;
    if (threadIdx.x == 0) s_sp = level_sparse(L);
    __syncthreads();
    return !s_sp;
}

}  // namespace brgpu
