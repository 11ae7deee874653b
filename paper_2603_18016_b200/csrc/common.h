// common.h -- launch helpers shared by the .cu files: launch accounting and
// programmatic dependent launch (PDL).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdio>
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

// PSD_DEBUG_LAUNCH=1: report launches that fail or find their stream's
// capture already invalidated (names the previous launch) on stderr
inline int debug_launch() {
  static int v = [] {
    const char* e = getenv("PSD_DEBUG_LAUNCH");
    return e ? atoi(e) : 0;
  }();
  return v;
}
inline void debug_before(const void* k, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusInvalidated)
    fprintf(stderr, "[psd] capture invalidated before %p\n", k);
}
inline void debug_after(const void* k, cudaError_t e, dim3 g, size_t smem, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess || cs == cudaStreamCaptureStatusInvalidated)
    fprintf(stderr, "[psd] launch %p grid (%u,%u,%u) smem %zu: %s%s\n", k, g.x, g.y, g.z, smem,
            cudaGetErrorString(e), cs == cudaStreamCaptureStatusInvalidated ? " (capture invalidated)"
                                                                           : "");
}

// raise a kernel's dynamic shared memory limit (call once per kernel, outside
// stream capture: the first launch of every kernel is eager)
inline cudaError_t set_smem_limit(const void* k, int bytes, cudaStream_t st = nullptr) {
  const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (debug_launch()) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (st) cudaStreamIsCapturing(st, &cs);
    fprintf(stderr, "[psd] smem limit %p = %d: %s%s\n", k, bytes, cudaGetErrorString(e),
            cs == cudaStreamCaptureStatusNone ? "" : " (during capture)");
  }
  return e;
}

// set_smem_limit once per (device, kernel): function attributes belong to the
// kernel's instance on the current device, so a process driving several GPUs
// sets them on each (kernels sharing a signature share a function-pointer
// type, so a per-type static flag would not do either)
inline cudaError_t ensure_smem_limit(const void* k, int bytes, cudaStream_t st = nullptr) {
  static std::mutex mu;
  static const void* done_k[256];
  static int done_dev[256];
  static int n = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; ++i)
    if (done_k[i] == k && done_dev[i] == dev) return cudaSuccess;
  e = set_smem_limit(k, bytes, st);
  if (e == cudaSuccess && n < 256) {
    done_k[n] = k;
    done_dev[n++] = dev;
  }
  return e;
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
  if (debug_launch()) debug_before(reinterpret_cast<const void*>(kernel), st);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (debug_launch()) debug_after(reinterpret_cast<const void*>(kernel), e, grid, smem, st);
  return e;
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
