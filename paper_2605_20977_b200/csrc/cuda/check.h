#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace pswa_dev {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    throw CudaError(std::string("cuda: ") + what + ": " + cudaGetErrorString(e) + " (" +
                    file + ":" + std::to_string(line) + ")");
  }
}

}  // namespace pswa_dev

#define PSWA_CUDA(x) ::pswa_dev::cuda_check((x), #x, __FILE__, __LINE__)
#define PSWA_LAUNCH_CHECK() ::pswa_dev::cuda_check(cudaGetLastError(), "launch", __FILE__, __LINE__)
