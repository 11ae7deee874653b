// common.h -- launch helpers shared by the .cu files: launch accounting and
// programmatic dependent launch (PDL).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <utility>

namespace psd {
// number of kernels this library has enqueued (captured launches count once,
// at capture; GpuBackend multiplies by graph replays)
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launches(int n = 1) { launch_counter().fetch_add(n, std::memory_order_relaxed); }

// PDL: a kernel may start (prologue: barrier init, TMEM alloc, descriptor
// prefetch, weight loads) while its stream predecessor drains; it calls
// pdl_wait() before touching the predecessor's outputs.  PSD_PDL=0 disables.
inline int pdl_enabled() {
  static int v = [] {
    const char* e = getenv("PSD_PDL");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <typename... Params, typename... Args>
inline cudaError_t launch(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args&&... args) {
  count_launches();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace psd

#ifdef __CUDACC__
// wait until the programmatic predecessor grid completed (its writes visible)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// allow the dependent grid to be scheduled once every CTA of this grid got here
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif
