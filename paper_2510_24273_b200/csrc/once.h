// Per-device one-time setup of kernel function attributes.
//
// cudaFuncSetAttribute (MaxDynamicSharedMemorySize, NonPortableClusterSizeAllowed)
// acts on the function in the CURRENT device's context, so a process that drives
// several GPUs (one thread per GPU, sals.h) must set it once per device.  The
// done-bits are per device (bit = device ordinal < 64, atomics), the setup runs
// under a mutex, so concurrent first calls from several threads are safe.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>

namespace sals {

class DeviceOnce {
 public:
  template <class F>
  cudaError_t run(F&& setup) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;   // >= 64 devices: set every time
    if (bit && (done_.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    std::lock_guard<std::mutex> lock(mu_);
    if (bit && (done_.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
    e = setup();
    if (e == cudaSuccess && bit) done_.fetch_or(bit, std::memory_order_release);
    return e;
  }

 private:
  std::atomic<uint64_t> done_{0};
  std::mutex mu_;
};

// Number of SMs of the current device (cached per device).
inline cudaError_t device_sm_count(int* n) {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) { *n = c; return cudaSuccess; }
  }
  e = cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess && dev < 64) cache[dev].store(*n, std::memory_order_relaxed);
  return e;
}

}  // namespace sals
