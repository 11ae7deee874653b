// common.h -- host-side launch accounting shared by the .cu files.
#pragma once
#include <atomic>

namespace psd {
// number of kernels this library has enqueued (captured launches count once,
// at capture; GpuBackend multiplies by graph replays)
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launches(int n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }
}  // namespace psd
