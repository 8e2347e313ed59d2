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

// Makes `device` current for a scope and restores the caller's device on
// exit: a handle may be used from any host thread, whatever device that
// thread has current (each handle's allocations, streams and graphs belong to
// its own device).
class DeviceScope {
 public:
  explicit DeviceScope(int device) {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
    if (prev_ != device) cuda_check(cudaSetDevice(device), "cudaSetDevice", __FILE__, __LINE__);
    else prev_ = -1;
  }
  ~DeviceScope() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;

 private:
  int prev_ = -1;
};

}  // namespace pswa_dev

#define PSWA_CUDA(x) ::pswa_dev::cuda_check((x), #x, __FILE__, __LINE__)
#define PSWA_LAUNCH_CHECK() ::pswa_dev::cuda_check(cudaGetLastError(), "launch", __FILE__, __LINE__)
