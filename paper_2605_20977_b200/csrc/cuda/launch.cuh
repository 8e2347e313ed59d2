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

// cluster_x > 1 launches thread-block clusters of cluster_x CTAs along x.
template <typename... KArgs, typename... Args>
void launch_kc(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  PSWA_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
              Args&&... args) {
  launch_kc(kernel, grid, block, smem, st, 1u, std::forward<Args>(args)...);
}

}  // namespace pswa_dev
