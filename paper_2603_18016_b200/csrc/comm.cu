// comm.cu -- peer-memory communicator: tensor-parallel all-reduce and the
// point-to-point mailbox of the dedicated-draft-GPU hand-off, over NVLink /
// NVSwitch load-stores (no NCCL on these paths).
//
// Replaces what the reference only charges as a scalar: `comm_overhead`
// (pkg/src/specsim/request_model.py:128, added to the PSD step at
// engine.py:435-442) -- here the real exchanges: the row-parallel O / down
// sums of a tensor-parallel target and the draft-id
// hand-off between a draft GPU and its target GPU (C1).
//
// Every rank allocates one region (cudaMalloc) and exports it with a CUDA IPC
// handle; the host layer exchanges the handles (torch.distributed
// all_gather_object) and every rank maps all peers' regions.  Region layout:
//   ctrl  [4 KB]  ready[src] (u64): the all-reduce epoch rank src published
//                 seq[src] / ack[dst] (u64): mailbox message counters
//                 (written by peers, system scope), then local counters
//   data  [2][buf_bytes]  all-reduce staging, double-buffered by epoch parity
//   mbox  [world][mbox_bytes]  one payload slot per source rank
//
// All-reduce (psd_tp_allreduce_partials), one kernel, G resident CTAs:
//   1. each rank sums its S local split-K partials (fixed split order) into
//      its own staging buffer (parity = epoch & 1);
//   2. the last CTA to finish (ticket) publishes ready = epoch + 1 into every
//      peer's region (release, system scope); every CTA waits until all peers
//      published that epoch;
//   3. each CTA sums its slice of the W staging buffers in rank order 0..W-1,
//      so every rank computes bit-identical sums (deterministic TP numerics);
//   4. the last CTA out advances the device-resident epoch.  Seeing a peer's
//      epoch e + 1 implies that peer finished call e (stream order), so the
//      staging buffer of parity e is free again two calls later: one barrier
//      per call.  The epoch lives in device memory, so the kernel can be
//      captured in a CUDA graph and replayed.
// Every wait has a %globaltimer watchdog (trap after 10 s) instead of a hang.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>

#include "../../include/psd.h"
#include "common.h"

namespace {

constexpr int kMaxWorld = PSD_COMM_MAX_WORLD;
constexpr size_t kCtrl = 4096;
// ctrl offsets (u64 words)
constexpr int kReady = 0;          // [kMaxWorld] written by peers
constexpr int kSeq = 64;           // [kMaxWorld] mailbox: messages src has put here
constexpr int kAck = 128;          // [kMaxWorld] mailbox: messages dst consumed from me
constexpr int kEpoch = 192;        // local: all-reduce calls completed
constexpr int kArrive = 193;       // local: CTA tickets of phase 1 (reset per call)
constexpr int kDone = 194;         // local: CTA tickets of phase 3 (reset per call)
constexpr int kSent = 256;         // local [kMaxWorld]: messages I put to dst
constexpr int kConsumed = 320;     // local [kMaxWorld]: messages I consumed from src
constexpr int kThreads = 256;

struct Comm {
  int rank, world;
  size_t buf_bytes, mbox_bytes, region_bytes;
  char* local;
  char* peer[kMaxWorld];
  bool opened;
  int device;
  bool local_group;  // psd_comm_create_local: peers are this process's own regions
};

struct Handle {
  cudaIpcMemHandle_t ipc;
  uint64_t region_bytes;
  int32_t rank, world;
};

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// spin until *p >= want (system scope), trap after 10 s
__device__ __forceinline__ void wait_geq(const uint64_t* p, uint64_t want) {
  const uint64_t t0 = gtimer();
  while (ld_acquire_sys(p) < want) {
    if (gtimer() - t0 > 10000000000ull) __trap();
    __nanosleep(64);
  }
}

struct ARArgs {
  char* region[kMaxWorld];  // [world]: every rank's region (own included)
  int rank, world;
  const float* part;
  int S;
  size_t stride, n, buf_bytes;
  float* out;
  int gather;  // 0: out = sum over ranks; 1: out[r * n + i] = rank r's data
};

__global__ void __launch_bounds__(kThreads) allreduce_kernel(const ARArgs a) {
  uint64_t* ctrl = reinterpret_cast<uint64_t*>(a.region[a.rank]);
  __shared__ uint64_t s_epoch;
  __shared__ int s_last;
  pdl_wait();
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint64_t*>(ctrl + kEpoch);
  __syncthreads();
  const uint64_t e = s_epoch, E = e + 1;
  const int par = (int)(e & 1);
  const size_t nv = a.n / 4;  // float4 elements (n % 4 == 0, checked on the host)
  const size_t tid0 = (size_t)blockIdx.x * kThreads + threadIdx.x;
  const size_t step = (size_t)gridDim.x * kThreads;
  // 1. local split-K reduction into my staging buffer
  {
    float4* mine = reinterpret_cast<float4*>(a.region[a.rank] + kCtrl + par * a.buf_bytes);
    const float4* p = reinterpret_cast<const float4*>(a.part);
    const size_t sv = a.stride / 4;
    for (size_t i = tid0; i < nv; i += step) {
      float4 v = p[i];
      for (int s = 1; s < a.S; ++s) {
        const float4 w = p[s * sv + i];
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      mine[i] = v;
    }
  }
  // 2. publish (last CTA), then wait for every peer
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    // per-call ticket (grids differ between calls): the last CTA resets it;
    // no other CTA of this call touches it again, and the next call starts
    // after this one completed (stream order)
    const unsigned long long t =
        atomicAdd(reinterpret_cast<unsigned long long*>(ctrl + kArrive), 1ull);
    s_last = t == gridDim.x - 1;
    if (s_last) *reinterpret_cast<volatile uint64_t*>(ctrl + kArrive) = 0;
  }
  __syncthreads();
  if (s_last && threadIdx.x < a.world) {
    uint64_t* peer_ctrl = reinterpret_cast<uint64_t*>(a.region[threadIdx.x]);
    st_release_sys(peer_ctrl + kReady + a.rank, E);
  }
  if (threadIdx.x < a.world) wait_geq(ctrl + kReady + threadIdx.x, E);
  __syncthreads();
  // 3. sum the ranks' buffers in rank order (identical on every rank), or
  //    gather them rank after rank
  if (a.gather) {
    for (int r = 0; r < a.world; ++r) {
      const float4* src =
          reinterpret_cast<const float4*>(a.region[r] + kCtrl + par * a.buf_bytes);
      float4* dst = reinterpret_cast<float4*>(a.out) + r * nv;
      for (size_t i = tid0; i < nv; i += step) dst[i] = __ldcv(src + i);
    }
  }
  for (size_t i = tid0; i < nv && !a.gather; i += step) {
    float4 v = __ldcv(reinterpret_cast<const float4*>(a.region[0] + kCtrl + par * a.buf_bytes) +
                      i);
    for (int r = 1; r < a.world; ++r) {
      const float4 w =
          __ldcv(reinterpret_cast<const float4*>(a.region[r] + kCtrl + par * a.buf_bytes) + i);
      v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    }
    reinterpret_cast<float4*>(a.out)[i] = v;
  }
  // 4. the last CTA out advances the epoch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long t =
        atomicAdd(reinterpret_cast<unsigned long long*>(ctrl + kDone), 1ull);
    if (t == gridDim.x - 1) {
      *reinterpret_cast<volatile uint64_t*>(ctrl + kDone) = 0;
      *reinterpret_cast<volatile uint64_t*>(ctrl + kEpoch) = E;
    }
  }
  pdl_trigger();
}

struct P2PArgs {
  char* mine;
  char* peer;
  int rank, peer_rank;
  size_t mbox_off, mbox_bytes;  // mailbox area offset in a region, slot size
  int32_t* buf;
  int n;
};

// put: wait until the peer consumed my previous message (depth-1 slot), copy
// the payload into my slot of the peer's mailbox, publish the new sequence
__global__ void __launch_bounds__(kThreads) p2p_put_kernel(const P2PArgs a) {
  uint64_t* my = reinterpret_cast<uint64_t*>(a.mine);
  uint64_t* pc = reinterpret_cast<uint64_t*>(a.peer);
  __shared__ uint64_t s_sent;
  pdl_wait();
  if (threadIdx.x == 0) {
    s_sent = *reinterpret_cast<volatile uint64_t*>(my + kSent + a.peer_rank);
    wait_geq(my + kAck + a.peer_rank, s_sent);
  }
  __syncthreads();
  int32_t* slot = reinterpret_cast<int32_t*>(a.peer + a.mbox_off + a.rank * a.mbox_bytes);
  for (int i = threadIdx.x; i < a.n; i += kThreads) slot[i] = a.buf[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(pc + kSeq + a.rank, s_sent + 1);
    *reinterpret_cast<volatile uint64_t*>(my + kSent + a.peer_rank) = s_sent + 1;
  }
  pdl_trigger();
}

// get: wait for the next message from the peer, copy it out, acknowledge
__global__ void __launch_bounds__(kThreads) p2p_get_kernel(const P2PArgs a) {
  uint64_t* my = reinterpret_cast<uint64_t*>(a.mine);
  uint64_t* pc = reinterpret_cast<uint64_t*>(a.peer);
  __shared__ uint64_t s_cons;
  pdl_wait();
  if (threadIdx.x == 0) {
    s_cons = *reinterpret_cast<volatile uint64_t*>(my + kConsumed + a.peer_rank);
    wait_geq(my + kSeq + a.peer_rank, s_cons + 1);
  }
  __syncthreads();
  const int32_t* slot =
      reinterpret_cast<const int32_t*>(a.mine + a.mbox_off + a.peer_rank * a.mbox_bytes);
  for (int i = threadIdx.x; i < a.n; i += kThreads) a.buf[i] = __ldcv(slot + i);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile uint64_t*>(my + kConsumed + a.peer_rank) = s_cons + 1;
    st_release_sys(pc + kAck + a.rank, s_cons + 1);
  }
  pdl_trigger();
}

int sm_count_dev() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

extern "C" {

size_t psd_comm_handle_bytes(void) { return sizeof(Handle); }

int psd_comm_create(int rank, int world, size_t buf_bytes, size_t mbox_bytes, void** comm,
                    void* handle_out) {
  if (!comm || !handle_out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return (int)cudaErrorInvalidValue;
  buf_bytes = (buf_bytes + 255) & ~size_t(255);
  mbox_bytes = (mbox_bytes + 255) & ~size_t(255);
  // the mailbox slots sit after the two staging buffers
  Comm* c = new (std::nothrow) Comm();
  if (!c) return (int)cudaErrorMemoryAllocation;
  c->rank = rank;
  c->world = world;
  c->buf_bytes = buf_bytes;
  c->mbox_bytes = mbox_bytes;
  c->region_bytes = kCtrl + 2 * buf_bytes + (size_t)world * mbox_bytes;
  cudaGetDevice(&c->device);
  cudaError_t e = cudaMalloc(&c->local, c->region_bytes);
  if (e != cudaSuccess) {
    delete c;
    return (int)e;
  }
  cudaMemset(c->local, 0, kCtrl);
  Handle h{};
  e = cudaIpcGetMemHandle(&h.ipc, c->local);
  if (e != cudaSuccess) {
    cudaFree(c->local);
    delete c;
    return (int)e;
  }
  h.region_bytes = c->region_bytes;
  h.rank = rank;
  h.world = world;
  memcpy(handle_out, &h, sizeof(h));
  for (int r = 0; r < kMaxWorld; ++r) c->peer[r] = nullptr;
  c->peer[rank] = c->local;
  *comm = c;
  return (int)cudaDeviceSynchronize();
}

int psd_comm_create_local(int world, const int* devices, size_t buf_bytes, size_t mbox_bytes,
                          void** comms) {
  if (!comms || !devices || world < 1 || world > kMaxWorld) return (int)cudaErrorInvalidValue;
  buf_bytes = (buf_bytes + 255) & ~size_t(255);
  mbox_bytes = (mbox_bytes + 255) & ~size_t(255);
  int prev = 0;
  cudaGetDevice(&prev);
  Comm* cs[kMaxWorld] = {};
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < world && e == cudaSuccess; ++r) {
    cs[r] = new (std::nothrow) Comm();
    if (!cs[r]) { e = cudaErrorMemoryAllocation; break; }
    cs[r]->rank = r;
    cs[r]->world = world;
    cs[r]->buf_bytes = buf_bytes;
    cs[r]->mbox_bytes = mbox_bytes;
    cs[r]->region_bytes = kCtrl + 2 * buf_bytes + (size_t)world * mbox_bytes;
    cs[r]->device = devices[r];
    cs[r]->local_group = true;
    e = cudaSetDevice(devices[r]);
    if (e == cudaSuccess) e = cudaMalloc(&cs[r]->local, cs[r]->region_bytes);
    if (e == cudaSuccess) e = cudaMemset(cs[r]->local, 0, kCtrl);
    // direct peer access between distinct devices (same-device ranks need none)
    for (int q = 0; q < r && e == cudaSuccess; ++q) {
      if (devices[q] == devices[r]) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, devices[r], devices[q]);
      if (!ok) { e = cudaErrorPeerAccessUnsupported; break; }
      cudaSetDevice(devices[r]);
      cudaError_t pe = cudaDeviceEnablePeerAccess(devices[q], 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) e = pe;
      cudaSetDevice(devices[q]);
      pe = cudaDeviceEnablePeerAccess(devices[r], 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) e = pe;
      cudaGetLastError();  // clear a sticky "already enabled"
    }
  }
  if (e == cudaSuccess) {
    for (int r = 0; r < world; ++r) {
      for (int q = 0; q < kMaxWorld; ++q) cs[r]->peer[q] = q < world ? cs[q]->local : nullptr;
      cs[r]->opened = true;
      comms[r] = cs[r];
    }
    e = cudaDeviceSynchronize();
  } else {
    for (int r = 0; r < world; ++r)
      if (cs[r]) {
        if (cs[r]->local) cudaFree(cs[r]->local);
        delete cs[r];
      }
  }
  cudaSetDevice(prev);
  return (int)e;
}

int psd_comm_open(void* comm, const void* handles) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !handles) return (int)cudaErrorInvalidValue;
  const Handle* hs = static_cast<const Handle*>(handles);
  for (int r = 0; r < c->world; ++r) {
    if (hs[r].rank != r || hs[r].world != c->world || hs[r].region_bytes != c->region_bytes)
      return (int)cudaErrorInvalidValue;
    if (r == c->rank) continue;
    void* p = nullptr;
    cudaError_t e =
        cudaIpcOpenMemHandle(&p, hs[r].ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return (int)e;
    c->peer[r] = static_cast<char*>(p);
  }
  c->opened = true;
  return 0;
}

int psd_comm_destroy(void* comm) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c) return 0;
  cudaDeviceSynchronize();
  if (!c->local_group)
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  cudaFree(c->local);
  delete c;
  return 0;
}

static int launch_ar(void* comm, const float* partials, int S, size_t stride, size_t n,
                     float* out, int gather, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !c->opened || !partials || !out || S < 1) return (int)cudaErrorInvalidValue;
  if ((n & 3) || (stride & 3) || n * sizeof(float) > c->buf_bytes ||
      (reinterpret_cast<uintptr_t>(partials) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
    return (int)cudaErrorInvalidValue;
  ARArgs a{};
  for (int r = 0; r < c->world; ++r) a.region[r] = c->peer[r];
  a.rank = c->rank;
  a.world = c->world;
  a.part = partials;
  a.S = S;
  a.stride = stride;
  a.n = n;
  a.buf_bytes = c->buf_bytes;
  a.out = out;
  a.gather = gather;
  // resident grid (the CTAs wait on each other's tickets): half the SMs
  const size_t want = (n / 4 + kThreads - 1) / kThreads;
  int grid = sm_count_dev() / 2;
  if ((size_t)grid > want) grid = (int)(want > 0 ? want : 1);
  return (int)psd::launch(allreduce_kernel, dim3(grid), dim3(kThreads), 0,
                          (cudaStream_t)stream, a);
}

int psd_tp_allreduce_partials(void* comm, const float* partials, int S, size_t stride, size_t n,
                              float* out, void* stream) {
  return launch_ar(comm, partials, S, stride, n, out, 0, stream);
}

int psd_tp_allreduce_f32(void* comm, float* data, size_t n, void* stream) {
  return psd_tp_allreduce_partials(comm, data, 1, n, n, data, stream);
}

int psd_tp_allgather_f32(void* comm, const float* src, size_t n, float* out, void* stream) {
  if (out == src) return (int)cudaErrorInvalidValue;
  return launch_ar(comm, src, 1, n, n, out, 1, stream);
}

int psd_p2p_put_i32(void* comm, int peer, const int32_t* src, int n, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !c->opened || peer < 0 || peer >= c->world || peer == c->rank || n < 0 ||
      (size_t)n * 4 > c->mbox_bytes)
    return (int)cudaErrorInvalidValue;
  P2PArgs a{c->local, c->peer[peer], c->rank, peer, kCtrl + 2 * c->buf_bytes, c->mbox_bytes,
            const_cast<int32_t*>(src), n};
  return (int)psd::launch(p2p_put_kernel, dim3(1), dim3(kThreads), 0, (cudaStream_t)stream, a);
}

int psd_p2p_get_i32(void* comm, int peer, int32_t* dst, int n, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !c->opened || peer < 0 || peer >= c->world || peer == c->rank || n < 0 ||
      (size_t)n * 4 > c->mbox_bytes)
    return (int)cudaErrorInvalidValue;
  P2PArgs a{c->local, c->peer[peer], c->rank, peer, kCtrl + 2 * c->buf_bytes, c->mbox_bytes,
            dst, n};
  return (int)psd::launch(p2p_get_kernel, dim3(1), dim3(kThreads), 0, (cudaStream_t)stream, a);
}

}  // extern "C"
