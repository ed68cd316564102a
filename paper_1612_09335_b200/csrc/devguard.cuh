// Scoped current-device switch for the device-side entry points of libcwreco.
#pragma once
#include <cuda_runtime.h>

namespace cwr {

// Makes the context's device current for one library call and restores the
// caller's current device afterwards (contexts on several GPUs in one process).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      cudaGetLastError();
      prev = -1;
    }
    if (dev >= 0 && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace cwr
