// Programmatic dependent launch (PDL): every libaxonn kernel is launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so it may start while the previous
// kernel of its stream is still draining.  Each kernel does its set-up (barrier init, TMEM
// allocation, descriptor prefetch), then pdl_wait()s for the previous grid to complete
// before its first global-memory access, and calls pdl_launch_dependents() so the next
// kernel can be scheduled early.  Hides per-launch prologue and tail time.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace axonn {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                     size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace axonn
