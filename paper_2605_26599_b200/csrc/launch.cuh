// launch.cuh -- programmatic dependent launch (PDL) for the level pipeline.
//
// Every kernel of a solve is launched with programmatic stream serialization
// and starts with pdl_entry(): it lets its own dependents begin launching at
// once (griddepcontrol.launch_dependents) and then waits until its
// predecessor grid has completed and its memory is visible
// (griddepcontrol.wait).  A dependent's CTAs are scheduled only after every
// CTA of the predecessor has started, so they never take resources the
// predecessor still needs; the launch and ramp latency of the ~15 small
// kernels per grid-tier level overlaps the tail of the previous one.  Inside
// a captured CUDA graph the serialization becomes programmatic edges.
#pragma once

#include <cuda_runtime.h>

#include <utility>

namespace brgpu {

__device__ __forceinline__ void pdl_entry() {
#ifdef BRGPU_PDL_EARLY
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace brgpu
