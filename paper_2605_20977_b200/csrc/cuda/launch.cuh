// Programmatic dependent launch (PDL). Every kernel of the decode path is
// launched with cudaLaunchAttributeProgrammaticStreamSerialization and begins
// with pdl_wait() before its first global-memory access, so the next kernel's
// launch and register/smem/TMEM prologue overlap the tail of the previous one
// (inside the captured CUDA graphs too). PSWA_NO_PDL=1 disables it.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

#include "check.h"

namespace pswa_dev {

__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = std::getenv("PSWA_NO_PDL") == nullptr;
  return on;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PSWA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace pswa_dev
