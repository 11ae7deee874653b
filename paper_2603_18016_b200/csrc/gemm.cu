// gemm.cu -- K2: bf16 GEMM on tcgen05 tensor cores (TMEM accumulators, TMA
// operand staging, mbarrier pipeline), swap-AB for skinny token counts.
//
//   Y[m, n] = sum_k X[m, k] * W[n, k]          X: [M, K] bf16, W: [N, K] bf16
//
// Replaces the reference's virtual pass durations
// (verify_latency / draft_latency .duration, pkg/src/specsim/engine.py:338,
// 359-360, 378, 402, 429) with the real dense contractions of the target
// verify forward (M = B (k+1) tokens) and the draft decode (M = B tokens).
//
// Design (B200-first):
//   * swap-AB: the weight tile is the UMMA "A" operand (M = 128 weight rows),
//     the token tile is "B" (N = 32..256 tokens).  Decode / verify token counts
//     are 32..320, so one UMMA N covers the whole batch and every weight byte
//     is read from HBM exactly once per GEMM (weights are the HBM roofline).
//   * warp specialisation, 6 warps: warp 0 = TMA producer (one elected lane),
//     warp 1 = MMA issuer (one lane issues tcgen05.mma, commits release smem
//     stages), warps 2-5 = epilogue (tcgen05.ld TMEM -> registers -> global).
//   * multi-stage smem ring (4-8 stages of 16 KB weights + BN*128 B tokens),
//     128-byte swizzle matching the UMMA descriptors; weights are loaded with an
//     L2 evict-first policy (streamed once), tokens evict-last (re-read by
//     every weight tile).
//   * split-K over blockIdx.z when the weight-tile count cannot fill 148 SMs;
//     fp32 partials are reduced by psd_gemm_reduce with the same epilogue.
// Epilogues: bf16 store, fp32 store (LM-head logits), residual add (x += W o),
// fused SiLU(gate) * up (weights packed gate/up per 64-row half tile).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include "../../include/psd.h"
#include "../../include/psd_experimental.h"
#include "common.h"
#include "sm100.cuh"

namespace {
using namespace psd;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;
constexpr int kMaxTiles = 1 << 16;  // stream-K tickets reserved at the workspace head
struct GemmArgs {
  int M, N, K;
  int kb_total, kb_per_split;
  void* Y;
  int ldy;
  const __nv_bfloat16* R;
  int ldr;
  int tma_y;        // the tile leaves through TMA stores of tmY
  CUtensorMap tmY;  // Y [M][N_out] (2-D) or the partials [S][M][N] (3-D); box 16 tokens
};

// epilogue staging for TMA stores: 24 KB of rotating 16-token buffers (SiLU:
// 12 of 16 x 64 bf16, bf16: 6 of 16 x 128, fp32 / partials: 3 of 16 x 128)
constexpr int kEpBytes = 24 * 1024;
template <int EPI>
constexpr int ep_buf_bytes() {
  return EPI == PSD_EPI_SILU ? 16 * 64 * 2
       : (EPI == PSD_EPI_F32 || EPI == PSD_EPI_PARTIAL) ? 16 * 128 * 4 : 16 * 128 * 2;
}
// staging bytes of an epilogue kind (0: per-thread global stores)
template <int EPI>
constexpr int ep_stage_bytes() {
  return (EPI == PSD_EPI_RESID || EPI == PSD_EPI_ARGMAX) ? 0 : kEpBytes;
}

// NT token tiles of BN rows per weight tile (NT = 2 for 256 < M <= 512: every
// weight byte is streamed once instead of once per token tile)
template <int BN, int NT = 1, int SMEM_KB = 200>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = NT * BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int MAXS = (SMEM_KB * 1024) / STAGE;
  static constexpr int STAGES = MAXS > 8 ? 8 : MAXS;
  static constexpr int TMEM_COLS = NT * BN <= 32 ? 32 : NT * BN <= 64 ? 64
                                 : NT * BN <= 128 ? 128 : NT * BN <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
};

// silu(x) = x * sigmoid(x) = 0.5 x (1 + tanh(x / 2)): one MUFU.TANH per element
// (an IEEE reciprocal here measured +27 us on the 8B gate/up GEMM epilogue)
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float silu(float x) {
  const float h = 0.5f * x;
  return fmaf(h, tanh_approx(h), h);
}

// epilogue of one 128 x BN accumulator tile (warps 2-5; TMEM lane quarter q):
// weight rows n0 + 32q + lane, token columns m0 ..; split z for partials
template <int BN, int EPI>
__device__ __forceinline__ void tile_epilogue(const GemmArgs& g, uint32_t tmem, int n0, int m0,
                                              int z, int q, int lane, int tile_x) {
    const int n = n0 + 32 * q + lane;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c, r);
      tmem_ld_wait();
      if constexpr (EPI == PSD_EPI_SILU) {
        // packed weights: in quarter q, rows 32q..32q+15 = gate f, rows
        // 32q+16..32q+31 = up f (f = tile*64 + 16q + lane%16): one shuffle
        // pairs them inside the warp
        const int jo = tile_x * 64 + 16 * q + (lane & 15);
        __nv_bfloat16* Y = static_cast<__nv_bfloat16*>(g.Y);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float mine = __uint_as_float(r[j]);
          const float up = __shfl_down_sync(0xffffffffu, mine, 16);
          const int m = m0 + c + j;
          if (lane < 16 && m < g.M) Y[(size_t)m * g.ldy + jo] = __float2bfloat16(silu(mine) * up);
        }
      } else {
        if (n < g.N) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = m0 + c + j;
            if (m >= g.M) break;
            const float v = __uint_as_float(r[j]);
            if constexpr (EPI == PSD_EPI_PARTIAL) {
              float* P = static_cast<float*>(g.Y) + (size_t)z * g.M * g.N;
              P[(size_t)m * g.N + n] = v;
            } else if constexpr (EPI == PSD_EPI_F32) {
              static_cast<float*>(g.Y)[(size_t)m * g.ldy + n] = v;
            } else if constexpr (EPI == PSD_EPI_RESID) {
              __nv_bfloat16* Y = static_cast<__nv_bfloat16*>(g.Y);
              const float rv = __bfloat162float(g.R[(size_t)m * g.ldr + n]);
              Y[(size_t)m * g.ldy + n] = __float2bfloat16(v + rv);
            } else {
              static_cast<__nv_bfloat16*>(g.Y)[(size_t)m * g.ldy + n] = __float2bfloat16(v);
            }
          }
        }
      }
    }
}

// the same epilogue through shared memory and TMA stores (warps 2-5, one
// 16-token group per store; thread 64 issues)
template <int BN, int EPI>
__device__ __forceinline__ void tile_epilogue_tma(const GemmArgs& g, uint32_t tmem, int n0,
                                                  int m0, int z, int q, int lane, int tile_x,
                                                  uint8_t* sEp) {
  constexpr int EG = 4;
  constexpr int EPB = ep_buf_bytes<EPI>();
  constexpr int NEPB = ep_stage_bytes<EPI>() / EPB;
  const int row = 32 * q + lane;
  const uint32_t tbase = tmem + ((uint32_t)(32 * q) << 16);
  int eq = 0;
#pragma unroll 1
  for (int col0 = 0; col0 < BN; col0 += 16 * EG) {
    uint32_t r[EG][16];
#pragma unroll
    for (int e = 0; e < EG; ++e)
      if (col0 + 16 * e < BN) tmem_ld16(tbase + (uint32_t)(col0 + 16 * e), r[e]);
    tmem_ld_wait();
#pragma unroll
    for (int e = 0; e < EG; ++e) {
      const int col = col0 + 16 * e;
      if (col >= BN) break;
      uint8_t* buf = sEp + (eq % NEPB) * EPB;
      const uint32_t b0 = smem_u32(buf);
      if constexpr (EPI == PSD_EPI_SILU) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float mine = __uint_as_float(r[e][k]);
          const float up = __shfl_down_sync(0xffffffffu, mine, 16);
          v[k] = silu(mine) * up;
        }
        if (lane < 16) {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            sts_b16(b0 + 2 * (16 * q + lane) + k * 128, __float2bfloat16(v[k]));
        }
      } else if constexpr (EPI == PSD_EPI_BF16) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
          sts_b16(b0 + 2 * row + k * 2 * BM, __float2bfloat16(__uint_as_float(r[e][k])));
      } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) sts_f32(b0 + 4 * row + k * 4 * BM, __uint_as_float(r[e][k]));
      }
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) {
        if constexpr (EPI == PSD_EPI_PARTIAL)
          tma_store_3d(&g.tmY, buf, n0, m0 + col, z);
        else
          tma_store_2d(&g.tmY, buf, EPI == PSD_EPI_SILU ? tile_x * 64 : n0, m0 + col);
        bulk_commit();
        bulk_wait_read<NEPB - 2>();
      }
      ++eq;
    }
  }
  if (threadIdx.x == 64) bulk_wait<0>();
}

template <int BN, int EPI, int NT = 1, int SMEM_KB = 200>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
            const __grid_constant__ GemmArgs g) {
  using C = Cfg<BN, NT, SMEM_KB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sEp = sB + C::STAGES * C::B_BYTES;  // epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sEp + ep_stage_bytes<EPI>());
  uint64_t* empty = full + C::STAGES;
  uint64_t* accum = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BM, m0 = blockIdx.y * (NT * BN), z = blockIdx.z;
  const int kb0 = z * g.kb_per_split;
  const int nkb = min(g.kb_total, kb0 + g.kb_per_split) - kb0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(accum, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  constexpr int TB = BN * BK * 2;  // bytes of one token tile's k-block
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      // PDL: weights do not depend on the predecessor kernel -> the first
      // stages' weight tiles stream while it drains; tokens after pdl_wait()
      const int npre = min(nkb, C::STAGES);
      for (int i = 0; i < npre; ++i) {
        mbar_arrive_expect_tx(full + i, C::STAGE);
        tma_load_2d(sA + i * C::A_BYTES, &tmW, full + i, (kb0 + i) * BK, n0, pol_w);
      }
      pdl_wait();
      for (int i = 0; i < npre; ++i)
#pragma unroll
        for (int h = 0; h < NT; ++h)
          tma_load_2d(sB + i * C::B_BYTES + h * TB, &tmX, full + i, (kb0 + i) * BK, m0 + h * BN,
                      pol_x);
      for (int i = npre; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        mbar_wait(empty + s, ph ^ 1);
        mbar_arrive_expect_tx(full + s, C::STAGE);
        const int kc = (kb0 + i) * BK;
        tma_load_2d(sA + s * C::A_BYTES, &tmW, full + s, kc, n0, pol_w);
#pragma unroll
        for (int h = 0; h < NT; ++h)
          tma_load_2d(sB + s * C::B_BYTES + h * TB, &tmX, full + s, kc, m0 + h * BN, pol_x);
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        mbar_wait(full + s, ph);
        tc_fence_after();
        const uint32_t a = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
#pragma unroll
          for (int h = 0; h < NT; ++h)
            mma_bf16(tmem + h * BN, umma_desc_sw128(a + kk * 32),
                     umma_desc_sw128(b + h * TB + kk * 32), idesc, (i | kk) != 0);
        mma_commit(empty + s);
      }
      mma_commit(accum);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    pdl_wait();  // the residual R is the predecessor's output
    mbar_wait(accum, 0);
    tc_fence_after();
    // the NT token tiles are contiguous in tokens and in TMEM columns: one
    // NT * BN wide epilogue
    if constexpr (ep_stage_bytes<EPI>() > 0) {
      if (g.tma_y) {
        tile_epilogue_tma<NT * BN, EPI>(g, tmem, n0, m0, z, q, lane, blockIdx.x, sEp);
      } else {
        tile_epilogue<NT * BN, EPI>(g, tmem, n0, m0, z, q, lane, blockIdx.x);
      }
    } else {
      tile_epilogue<NT * BN, EPI>(g, tmem, n0, m0, z, q, lane, blockIdx.x);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ---- stream-K persistent variant ---------------------------------------------
// Work = tiles x k-blocks "units" in tile-major order (tile t = n_tile * MT +
// m_tile, so neighbouring units share weights); CTA c of G takes units
// [c U / G, (c+1) U / G).  Every SM gets the same number of weight k-blocks,
// so there are no wave-quantisation tails (224 gate/up tiles on 148 SMs
// would otherwise run 1.51 waves) and no separate split-K launch.  A tile cut
// by a CTA boundary is finished by whichever of its contributors arrives
// last (atomic ticket): it sums every contributor's fp32 partial in CTA order
// (deterministic), applies the epilogue and resets the ticket.  Nobody waits,
// so concurrent persistent kernels on two streams cannot deadlock.  The TMEM
// accumulator is double buffered: segment j+1's MMAs overlap j's epilogue.
struct SKArgs {
  int M, N, K;
  int KB, MT, tiles, G;
  // token-tile groups: every group of ACC_COLS tokens runs the same schedule
  // of G1 virtual CTAs over its T1 = N / 128 weight tiles (G = G1 * MT), so a
  // tile's k-split -- and every output element's summation order -- depends
  // on (N, K) and the SM count only, never on M (batch-invariant at any M)
  int G1, T1;
  long long U;
  void* Y;
  int ldy;
  const __nv_bfloat16* R;
  int ldr;
  float* part;    // [G][2][BN * 128]
  int* tickets;   // [tiles], zero between launches
  const __nv_bfloat16* Wt;  // pre-tiled weights (TILED variant)
  unsigned long long* trace;  // optional [G][16] globaltimer ns (psd_gemm_set_trace)
  int D;                      // tiles 0..D-1 whole per CTA (c, c+G, ..), after its stream-K units
  int tma_y;                  // finished tiles leave through TMA stores of tmY
  CUtensorMap tmY;            // Y [M][N_out] (bf16 / f32), box 16 tokens x 128 (64 SiLU) rows
  // PSD_EPI_ARGMAX (K6, the draft's greedy LM head): Y = float2 [M][N / 128]
  // (max, first argmax index) per (vocabulary tile, token); token m's logit at
  // column succ[tok[rows[m]]] gets + beta first (the synthetic-language bias,
  // as psd_bigram_bias adds it to stored logits)
  const int32_t* am_tok;
  const int32_t* am_rows;
  const int32_t* am_succ;
  float am_beta;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Seg {
  int t, kb0, kb1, first;  // tile, k-block range, is the (virtual) CTA's first segment
  int v;                   // virtual CTA the segment belongs to
  int tl, vb;              // group-local tile, first virtual CTA of the group
};

// first stream-K unit of a group's virtual CTA c (0 <= c <= G1)
__device__ __forceinline__ long long sk_bound(long long c, const SKArgs& g) {
  return c * g.U / g.G1;
}
// group-local virtual CTA holding unit u
__device__ __forceinline__ int sk_owner(long long u, const SKArgs& g) {
  long long c = u * g.G1 / g.U;
  while (c + 1 < g.G1 && sk_bound(c + 1, g) <= u) ++c;
  while (c > 0 && sk_bound(c, g) > u) --c;
  return (int)c;
}

template <int BN, int EPI, bool TILED, int NT = 1, int SMEM_KB = 200>
__global__ void __launch_bounds__(kThreads, 1)
gemm_sk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
               const __grid_constant__ SKArgs g) {
  using C = Cfg<BN, NT, SMEM_KB>;
  constexpr int ACC_COLS = NT * BN;           // one accumulator slot (NT token tiles)
  constexpr int NACC = NT == 1 ? 2 : 1;       // TMEM double buffer when it fits
  constexpr int TB = BN * BK * 2;             // bytes of one token tile's k-block
  constexpr int EG = 4;                       // epilogue: 16-column groups per round
  constexpr int TMEM_COLS = NACC * ACC_COLS <= 32 ? 32 : NACC * ACC_COLS <= 64 ? 64
                          : NACC * ACC_COLS <= 128 ? 128 : NACC * ACC_COLS <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  constexpr int EPS = ep_stage_bytes<EPI>();
  uint8_t* sEp = sB + C::STAGES * C::B_BYTES;  // EPS bytes of epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sEp + EPS);
  constexpr int EPB = ep_buf_bytes<EPI>();
  constexpr int NEPB = EPS / EPB;  // >= 3: a buffer is rewritten NEPB groups later
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;          // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Virtual CTAs: the work split (G shares, their k-block boundaries, the
  // fix-up order) depends only on the GEMM shape and the SM count, never on how
  // many CTAs actually run (psd_gemm_set_max_ctas): a capped launch's CTA c
  // processes virtual CTAs c, c + gridDim.x, ...  So every output element is
  // summed in the same order whatever the cap or the batch -- batch-invariant
  // numerics (greedy PSD == SD token for token).
  const int c = blockIdx.x;

  if (warp == 0 && lane == 0) {
    if (g.trace) g.trace[c * 16 + 0] = gtimer();
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // segment iterator (identical sequence in every role)
  // first this CTA's stream-K units over tiles D.., then its whole tiles
  // c, c+G, .. < D: a CTA ends on a whole tile, whose epilogue reads no partials
  // virtual CTA v = group * G1 + v1 works on group `group`'s tiles (tile
  // index group * T1 + local tile; token tile group = tile / T1).  A physical
  // CTA walks its group-local virtual CTAs v1 = c, c + grid, ...; each local
  // segment (weight tile, k-range) is run for every token group back to back,
  // so the groups re-read a weight k-block from L2 right after its first
  // fetch (the weights stream from HBM once at any M)
  struct SegIt {
    int v1;
    long long u, u0, u1;
    int dp;
    int gi, have;  // next token group of the current local segment
    int tl, kb0, kb1, first;
  };
  auto seg_begin = [&](int v1) -> SegIt {
    SegIt it;
    it.v1 = v1;
    it.u = it.u0 = sk_bound(v1, g);
    it.u1 = sk_bound(v1 + 1, g);
    it.dp = v1;
    it.gi = 0;
    it.have = 0;
    it.tl = it.kb0 = it.kb1 = it.first = 0;
    return it;
  };
  auto next_seg = [&](SegIt& it, Seg& sg) -> bool {
    while (true) {
      if (it.have && it.gi < g.MT) {
        sg.tl = it.tl;
        sg.kb0 = it.kb0;
        sg.kb1 = it.kb1;
        sg.first = it.first;
        sg.vb = it.gi * g.G1;
        sg.v = sg.vb + it.v1;
        sg.t = it.gi * g.T1 + it.tl;
        ++it.gi;
        return true;
      }
      it.have = 0;
      it.gi = 0;
      if (it.v1 >= g.G1) return false;
      if (it.u < it.u1) {
        it.tl = g.D + (int)(it.u / g.KB);
        it.kb0 = (int)(it.u % g.KB);
        it.kb1 = (int)min((long long)g.KB, it.kb0 + (it.u1 - it.u));
        it.first = it.u == it.u0;
        it.u += it.kb1 - it.kb0;
        it.have = 1;
        continue;
      }
      if (it.dp < g.D) {
        it.tl = it.dp;
        it.kb0 = 0;
        it.kb1 = g.KB;
        it.first = 0;
        it.dp += g.G1;
        it.have = 1;
        continue;
      }
      it = seg_begin(it.v1 + (int)gridDim.x);
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      SegIt it = seg_begin(c);
      Seg sg;
      int i = 0;
      // PDL: the first stages' weight tiles stream before pdl_wait()
      int npre = 0;
      {
        SegIt i0 = seg_begin(c);
        Seg s0;
        if (next_seg(i0, s0)) {
          const int n0 = (s0.t % g.T1) * BM;
          npre = min(s0.kb1 - s0.kb0, C::STAGES);
          for (int j = 0; j < npre; ++j) {
            mbar_arrive_expect_tx(full + j, C::STAGE);
            if constexpr (TILED) {
              const __nv_bfloat16* src =
                  g.Wt + ((size_t)(n0 / BM) * g.KB + s0.kb0 + j) * (size_t)(BM * BK);
              bulk_load(sA + j * C::A_BYTES, src, C::A_BYTES, full + j, pol_w);
            } else {
              tma_load_2d(sA + j * C::A_BYTES, &tmW, full + j, (s0.kb0 + j) * BK, n0, pol_w);
            }
          }
        }
      }
      pdl_wait();
      while (next_seg(it, sg)) {
        const int n0 = (sg.t % g.T1) * BM, m0 = (sg.t / g.T1) * ACC_COLS;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++i) {
          const int s = i % C::STAGES;
          const uint32_t ph = (i / C::STAGES) & 1;
          if (i < npre) {  // weight tile already in flight
#pragma unroll
            for (int h = 0; h < NT; ++h)
              tma_load_2d(sB + s * C::B_BYTES + h * TB, &tmX, full + s, kb * BK, m0 + h * BN,
                          pol_x);
            continue;
          }
          mbar_wait(empty + s, ph ^ 1);
          mbar_arrive_expect_tx(full + s, C::STAGE);
          if constexpr (TILED) {
            // pre-tiled, pre-swizzled weights: one contiguous 16 KB block
            const __nv_bfloat16* src =
                g.Wt + ((size_t)(n0 / BM) * g.KB + kb) * (size_t)(BM * BK);
            bulk_load(sA + s * C::A_BYTES, src, C::A_BYTES, full + s, pol_w);
          } else {
            tma_load_2d(sA + s * C::A_BYTES, &tmW, full + s, kb * BK, n0, pol_w);
          }
#pragma unroll
          for (int h = 0; h < NT; ++h)
            tma_load_2d(sB + s * C::B_BYTES + h * TB, &tmX, full + s, kb * BK, m0 + h * BN,
                        pol_x);
        }
      }
      pdl_trigger();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      SegIt it = seg_begin(c);
      Seg sg;
      int i = 0, j = 0;
      while (next_seg(it, sg)) {
        const int a = j % NACC;
        const uint32_t aph = (j / NACC) & 1;
        mbar_wait(tempty + a, aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * ACC_COLS;
        for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++i) {
          const int s = i % C::STAGES;
          const uint32_t ph = (i / C::STAGES) & 1;
          mbar_wait(full + s, ph);
          tc_fence_after();
          if (i == 0 && g.trace) g.trace[c * 16 + 1] = gtimer();
          const uint32_t sa = smem_u32(sA + s * C::A_BYTES);
          const uint32_t sb = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
#pragma unroll
            for (int h = 0; h < NT; ++h)
              mma_bf16(d + h * BN, umma_desc_sw128(sa + kk * 32),
                       umma_desc_sw128(sb + h * TB + kk * 32), idesc,
                       (kb != sg.kb0 || kk != 0) ? 1u : 0u);
          mma_commit(empty + s);
        }
        mma_commit(tfull + a);
        ++j;
      }
      if (g.trace) g.trace[c * 16 + 2] = gtimer();
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const int row = 32 * q + lane;  // tile row (weight row) of this thread
    pdl_wait();  // residual / partial workspace belong to the predecessor's epoch
    __shared__ int s_bcol[EPI == PSD_EPI_ARGMAX ? 512 : 1];
    __shared__ float s_amv[EPI == PSD_EPI_ARGMAX ? 16 * 136 : 1];
    if constexpr (EPI == PSD_EPI_ARGMAX) {
      // biased column of every token (three dependent loads, off the MMAs' path)
      for (int m = threadIdx.x - 64; m < 512; m += 128) {
        int col = -1;
        if (m < g.M && g.am_succ && g.am_beta != 0.f) {
          const int t = g.am_tok[g.am_rows ? g.am_rows[m] : m];
          if (t >= 0 && t < g.N) col = g.am_succ[t];
        }
        s_bcol[m] = col;
      }
      named_bar_sync(1, 128);
    }
    SegIt it = seg_begin(c);
    Seg sg;
    int j = 0, eq = 0;
    while (next_seg(it, sg)) {
      const int a = j % NACC;
      const uint32_t aph = (j / NACC) & 1;
      const int n0 = (sg.t % g.T1) * BM, m0 = (sg.t / g.T1) * ACC_COLS;
      const bool split = sg.kb0 != 0 || sg.kb1 != g.KB;
      const int me = sg.v;  // virtual CTA of this segment
      int owner = me, last = me;
      bool finisher = true;
      int* flag = s_flag + (j & 1);
      if (split) {
        owner = sg.vb + sk_owner((long long)(sg.tl - g.D) * g.KB, g);
        last = sg.vb + sk_owner((long long)(sg.tl - g.D) * g.KB + g.KB - 1, g);
        // every other contributor already published: finish without
        // publishing (the usual case for the tile a CTA ends on, i.e. the
        // tail).  Checked while this segment's MMAs are still running.
        if (threadIdx.x == 64) *flag = ld_acquire_gpu(g.tickets + sg.t) == last - owner;
        named_bar_sync(1, 128);
        finisher = *flag;
        if (finisher) __threadfence();
      }
      mbar_wait(tfull + a, aph);
      tc_fence_after();
      if (g.trace && threadIdx.x == 64) g.trace[c * 16 + 3] = gtimer();
      const uint32_t tbase = tmem + a * ACC_COLS + ((uint32_t)(32 * q) << 16);
      if (split) {
        if (g.trace && finisher && threadIdx.x == 64) g.trace[c * 16 + 6] += 1;
        if (!finisher) {
          // publish this segment's partial, take a ticket
          float* mine = g.part + ((size_t)me * 2 + (sg.first ? 0 : 1)) * (ACC_COLS * BM);
#pragma unroll 1
          for (int col0 = 0; col0 < ACC_COLS; col0 += 16 * EG) {
            uint32_t r[EG][16];
#pragma unroll
            for (int e = 0; e < EG; ++e)
              if (col0 + 16 * e < ACC_COLS) tmem_ld16(tbase + (uint32_t)(col0 + 16 * e), r[e]);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < EG; ++e)
              if (col0 + 16 * e < ACC_COLS) {
#pragma unroll
                for (int k = 0; k < 16; ++k)
                  mine[(col0 + 16 * e + k) * BM + row] = __uint_as_float(r[e][k]);
              }
          }
          __threadfence();
          named_bar_sync(1, 128);
          if (threadIdx.x == 64) {
            const int tk = atomicAdd(g.tickets + sg.t, 1);
            *flag = tk == last - owner;
          }
          named_bar_sync(1, 128);
          finisher = *flag;
          if (finisher) __threadfence();
        }
      }
      if (g.trace && threadIdx.x == 64) g.trace[c * 16 + 7] = gtimer();
      if (finisher) {
        // EG column groups per round: one TMEM wait and one L2 round trip for
        // the contributors' partials per 16*EG columns (the finisher of the
        // last tile is the kernel's tail)
#pragma unroll 1
        for (int col0 = 0; col0 < ACC_COLS; col0 += 16 * EG) {
          const int rnd = col0 / (16 * EG);
          uint32_t r[EG][16];
#pragma unroll
          for (int e = 0; e < EG; ++e)
            if (col0 + 16 * e < ACC_COLS) tmem_ld16(tbase + (uint32_t)(col0 + 16 * e), r[e]);
          tmem_ld_wait();
          if (g.trace && threadIdx.x == 64 && rnd < 4) g.trace[c * 16 + 8 + 2 * rnd] = gtimer();
          float v[EG][16];
          if (split) {
            // sum contributors in CTA order (own values from TMEM)
#pragma unroll
            for (int e = 0; e < EG; ++e)
#pragma unroll
              for (int k = 0; k < 16; ++k) v[e][k] = 0.f;
            for (int cc = owner; cc <= last; ++cc) {
              if (cc == me) {
#pragma unroll
                for (int e = 0; e < EG; ++e)
#pragma unroll
                  for (int k = 0; k < 16; ++k) v[e][k] += __uint_as_float(r[e][k]);
              } else {
                const bool first_of_cc =
                    sk_bound(cc - sg.vb, g) >= (long long)(sg.tl - g.D) * g.KB;
                const float* pp = g.part + ((size_t)cc * 2 + (first_of_cc ? 0 : 1)) * (ACC_COLS * BM);
                float w[EG][16];
#pragma unroll
                for (int e = 0; e < EG; ++e)
                  if (col0 + 16 * e < ACC_COLS) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) w[e][k] = __ldcg(pp + (col0 + 16 * e + k) * BM + row);
                  }
#pragma unroll
                for (int e = 0; e < EG; ++e)
#pragma unroll
                  for (int k = 0; k < 16; ++k) v[e][k] += w[e][k];
              }
            }
          } else {
#pragma unroll
            for (int e = 0; e < EG; ++e)
#pragma unroll
              for (int k = 0; k < 16; ++k) v[e][k] = __uint_as_float(r[e][k]);
          }
#pragma unroll
          for (int e = 0; e < EG; ++e) {
            const int col = col0 + 16 * e;
            if (col >= ACC_COLS) break;
            if constexpr (EPI == PSD_EPI_ARGMAX) {
              // per token column: max over the tile's 128 rows and the lowest
              // row attaining it.  Rows go through shared memory transposed
              // ([16 columns][136]: conflict-free both ways); 8 threads per
              // column scan rows p, p + 8, ... and merge by shuffles
              const int n = n0 + row;
#pragma unroll
              for (int k = 0; k < 16; ++k)
                s_amv[k * 136 + row] = n < g.N ? v[e][k] : -INFINITY;
              named_bar_sync(1, 128);
              {
                const int t = threadIdx.x - 64;
                const int k = t >> 3, p = t & 7;
                const int m = m0 + col + k;
                const int brow = m < g.M ? s_bcol[m] - n0 : -1;
                float bv = -INFINITY;
                int bi = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const int r = i * 8 + p;
                  float x = s_amv[k * 136 + r];
                  if (r == brow) x += g.am_beta;
                  if (x > bv) { bv = x; bi = r; }
                }
#pragma unroll
                for (int off = 4; off >= 1; off >>= 1) {
                  const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
                  const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
                }
                if (p == 0 && m < g.M)
                  static_cast<float2*>(g.Y)[(size_t)m * (g.N / BM) + n0 / BM] =
                      make_float2(bv, __int_as_float(n0 + bi));
              }
              named_bar_sync(1, 128);
              continue;
            }
            if constexpr (EPS > 0) {
              if (g.tma_y) {
                // stage 16 tokens x the tile's output rows in smem, one TMA
                // store per group (rows m >= M are clipped by the tensor map)
                uint8_t* buf = sEp + (eq % NEPB) * EPB;
                if constexpr (EPI == PSD_EPI_SILU) {
#pragma unroll
                  for (int k = 0; k < 16; ++k) {
                    const float up = __shfl_down_sync(0xffffffffu, v[e][k], 16);
                    v[e][k] = silu(v[e][k]) * up;
                  }
                  if (lane < 16) {
                    const uint32_t b = smem_u32(buf) + 2 * (16 * q + lane);
#pragma unroll
                    for (int k = 0; k < 16; ++k) sts_b16(b + k * 128, __float2bfloat16(v[e][k]));
                  }
                } else if constexpr (EPI == PSD_EPI_F32) {
                  const uint32_t b = smem_u32(buf) + 4 * row;
#pragma unroll
                  for (int k = 0; k < 16; ++k) sts_f32(b + k * 4 * BM, v[e][k]);
                } else {
                  const uint32_t b = smem_u32(buf) + 2 * row;
#pragma unroll
                  for (int k = 0; k < 16; ++k) sts_b16(b + k * 2 * BM, __float2bfloat16(v[e][k]));
                }
                fence_proxy_async_smem();
                named_bar_sync(1, 128);
                if (threadIdx.x == 64) {
                  tma_store_2d(&g.tmY, buf, EPI == PSD_EPI_SILU ? (n0 / BM) * 64 : n0, m0 + col);
                  bulk_commit();
                  // <= NEPB-2 stores still reading smem: the buffer the
                  // group after next writes is free
                  bulk_wait_read<NEPB - 2>();
                }
                ++eq;
                continue;
              }
            }
            if constexpr (EPI == PSD_EPI_SILU) {
              const int jo = (n0 / BM) * 64 + 16 * q + (lane & 15);
              __nv_bfloat16* Y = static_cast<__nv_bfloat16*>(g.Y);
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const float up = __shfl_down_sync(0xffffffffu, v[e][k], 16);
                v[e][k] = silu(v[e][k]) * up;  // all lanes: no divergence in the math
              }
              if (lane < 16) {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                  const int m = m0 + col + k;
                  if (m < g.M) Y[(size_t)m * g.ldy + jo] = __float2bfloat16(v[e][k]);
                }
              }
            } else {
              const int n = n0 + row;
              if (n < g.N) {
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                  const int m = m0 + col + k;
                  if (m >= g.M) break;
                  if constexpr (EPI == PSD_EPI_F32) {
                    static_cast<float*>(g.Y)[(size_t)m * g.ldy + n] = v[e][k];
                  } else if constexpr (EPI == PSD_EPI_RESID) {
                    __nv_bfloat16* Y = static_cast<__nv_bfloat16*>(g.Y);
                    const float rv = __bfloat162float(g.R[(size_t)m * g.ldr + n]);
                    Y[(size_t)m * g.ldy + n] = __float2bfloat16(v[e][k] + rv);
                  } else {
                    static_cast<__nv_bfloat16*>(g.Y)[(size_t)m * g.ldy + n] =
                        __float2bfloat16(v[e][k]);
                  }
                }
              }
            }
          }
          if (g.trace && threadIdx.x == 64 && rnd < 4) g.trace[c * 16 + 9 + 2 * rnd] = gtimer();
        }
        if (split && threadIdx.x == 64) g.tickets[sg.t] = 0;  // reusable next launch
      }
      // release this accumulator slot
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + a);
      ++j;
    }
    if (threadIdx.x == 64) bulk_wait<0>();  // TMA stores complete before exit
    if (g.trace && threadIdx.x == 64) {
      g.trace[c * 16 + 4] = gtimer();
      g.trace[c * 16 + 5] = j;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ---- split-K reduction with the same epilogues ------------------------------
__global__ void gemm_reduce_kernel(const float* __restrict__ P, int splits, int M, int N, int epi,
                                   void* Y, int ldy, const __nv_bfloat16* R, int ldr) {
  pdl_wait();
  pdl_trigger();
  const int Nout = epi == PSD_EPI_SILU ? N / 2 : N;
  const size_t total = (size_t)M * Nout;
  const size_t slice = (size_t)M * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int m = idx / Nout, n = idx % Nout;
    if (epi == PSD_EPI_SILU) {
      const int t = n / 64, r = n % 64;
      const size_t ig = (size_t)m * N + t * 128 + (r / 16) * 32 + r % 16, iu = ig + 16;
      float gs = 0.f, us = 0.f;
      for (int s = 0; s < splits; ++s) {
        gs += P[s * slice + ig];
        us += P[s * slice + iu];
      }
      static_cast<__nv_bfloat16*>(Y)[(size_t)m * ldy + n] = __float2bfloat16(silu(gs) * us);
      continue;
    }
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += P[s * slice + (size_t)m * N + n];
    if (epi == PSD_EPI_F32) {
      static_cast<float*>(Y)[(size_t)m * ldy + n] = acc;
    } else if (epi == PSD_EPI_RESID) {
      const float rv = __bfloat162float(R[(size_t)m * ldr + n]);
      static_cast<__nv_bfloat16*>(Y)[(size_t)m * ldy + n] = __float2bfloat16(acc + rv);
    } else {
      static_cast<__nv_bfloat16*>(Y)[(size_t)m * ldy + n] = __float2bfloat16(acc);
    }
  }
}

// ---- host side -----------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D bf16 tensor [rows, K] (row pitch ld elements), box = 64 x box_rows, SW128
int make_map(CUtensorMap* map, const void* base, int rows, int K, int ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// Y [M][N_out] for the stream-K finisher's TMA stores: box 16 tokens x box_cols
int make_out_map(CUtensorMap* map, void* Y, int M, int n_out, int ldy, int elt, int box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)n_out, (cuuint64_t)M};
  cuuint64_t strides[1] = {(cuuint64_t)ldy * elt};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, 16};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  2, Y, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// PSD_GEMM_TMA_STORE=0 keeps the per-thread global stores (A/B switch)
bool tma_store_enabled() {
  static bool v = [] {
    const char* e = getenv("PSD_GEMM_TMA_STORE");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

// split-K partials [S][M][N] fp32 as a 3-D tensor (rows m >= M of a split clip)
int make_part_map(CUtensorMap* map, void* P, int M, int N, int S) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)M * N * 4};
  cuuint32_t box[3] = {(cuuint32_t)BM, 16, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, P, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

// grid kernels: partials (kernel epilogue PARTIAL) or the final output
void set_grid_out_map(GemmArgs& g, int epi, void* Y, int M, int N, int ldy, int splits) {
  g.tma_y = 0;
  if (epi == PSD_EPI_RESID || !tma_store_enabled() || (reinterpret_cast<uintptr_t>(Y) & 15))
    return;
  if (epi == PSD_EPI_PARTIAL) {
    if (make_part_map(&g.tmY, Y, M, N, splits) == 0) g.tma_y = 1;
    return;
  }
  const int elt = epi == PSD_EPI_F32 ? 4 : 2;
  const int n_out = epi == PSD_EPI_SILU ? N / 2 : N;
  if (((size_t)ldy * elt) % 16) return;
  if (make_out_map(&g.tmY, Y, M, n_out, ldy, elt, epi == PSD_EPI_SILU ? 64 : BM) == 0)
    g.tma_y = 1;
}

void set_out_map(SKArgs& g, int epi, void* Y, int M, int N, int ldy) {
  g.tma_y = 0;
  if (epi == PSD_EPI_RESID || !tma_store_enabled()) return;
  const int elt = epi == PSD_EPI_F32 ? 4 : 2;
  const int n_out = epi == PSD_EPI_SILU ? N / 2 : N;
  if ((reinterpret_cast<uintptr_t>(Y) & 15) || ((size_t)ldy * elt) % 16) return;
  if (make_out_map(&g.tmY, Y, M, n_out, ldy, elt, epi == PSD_EPI_SILU ? 64 : BM) == 0)
    g.tma_y = 1;
}

template <int BN, int EPI, int SMEM_KB>
int launch_bn_s(const CUtensorMap& mw, const CUtensorMap& mx, const GemmArgs& g, dim3 grid,
                cudaStream_t st) {
  using C = Cfg<BN, 1, SMEM_KB>;
  {
    const cudaError_t e = psd::ensure_smem_limit((const void*)gemm_kernel<BN, EPI, 1, SMEM_KB>,
                                                 C::SMEM + ep_stage_bytes<EPI>(), st);
    if (e != cudaSuccess) return (int)e;
  }
  return (int)psd::launch(gemm_kernel<BN, EPI, 1, SMEM_KB>, grid, dim3(kThreads),
                          C::SMEM + ep_stage_bytes<EPI>(), st, mw, mx, g);
}

// Decode-width GEMMs of the draft (split-K QKV / O / down with <= 16
// k-blocks per CTA at <= 64 tokens, the whole-K gate/up at <= 32 tokens) run
// an 80 KB ring instead of 200 KB, so their CTAs fit on an SM beside the
// neighbouring kernel's (the decode attention, the next small GEMM):
// launched early by PDL they stream their weights while the predecessor
// still runs.  cfg2 draft phase -2.5 %, PSD +3.2 %, SD(2m) unchanged
// (profiles/r02_small_ring.txt).  PSD_GEMM_SMALL_RING: 0 = the full ring for
// every shape, 1 = split-K with <= 8 k-blocks only, 2 = default
int small_ring_enabled() {
  static int v = [] {
    const char* e = getenv("PSD_GEMM_SMALL_RING");
    return e ? atoi(e) : 2;
  }();
  return v;
}

template <int BN, int EPI>
int launch_bn(const CUtensorMap& mw, const CUtensorMap& mx, const GemmArgs& g, dim3 grid,
              cudaStream_t st) {
  if constexpr (EPI == PSD_EPI_PARTIAL && BN <= 64) {
    if (small_ring_enabled() && g.kb_per_split <= (small_ring_enabled() >= 2 ? 16 : 8))
      return launch_bn_s<BN, EPI, 80>(mw, mx, g, grid, st);
  }
  if constexpr (EPI == PSD_EPI_SILU && BN <= 32) {
    if (small_ring_enabled() >= 2) return launch_bn_s<BN, EPI, 80>(mw, mx, g, grid, st);
  }
  return launch_bn_s<BN, EPI, 200>(mw, mx, g, grid, st);
}


int sk_physical(int G);

template <int BN, int EPI, bool TILED, int NT = 1, int SMEM_KB = 200>
int launch_sk_bn_s(const CUtensorMap& mw, const CUtensorMap& mx, const SKArgs& g,
                   cudaStream_t st) {
  using C = Cfg<BN, NT, SMEM_KB>;
  constexpr int SMEM = C::SMEM + ep_stage_bytes<EPI>();
  static_assert(SMEM <= 227 * 1024, "stream-K GEMM shared memory");
  {
    const cudaError_t e = psd::ensure_smem_limit(
        (const void*)gemm_sk_kernel<BN, EPI, TILED, NT, SMEM_KB>, SMEM, st);
    if (e != cudaSuccess) return (int)e;
  }
  return (int)psd::launch(gemm_sk_kernel<BN, EPI, TILED, NT, SMEM_KB>, dim3(sk_physical(g.G1)),
                          dim3(kThreads), SMEM, st, mw, mx, g);
}

template <int BN, int EPI, bool TILED, int NT = 1>
int launch_sk_bn(const CUtensorMap& mw, const CUtensorMap& mx, const SKArgs& g, cudaStream_t st) {
  // the draft's stream-K gate/up at <= 32 tokens (small models whose FFN
  // tiles do not fill one wave): the same 80 KB ring as launch_bn's
  if constexpr (EPI == PSD_EPI_SILU && BN <= 32 && NT == 1 && !TILED) {
    static const int on = [] {
      const char* e = getenv("PSD_GEMM_SK_SMALL");
      return e ? atoi(e) : 1;
    }();
    if (on && small_ring_enabled() >= 2) return launch_sk_bn_s<BN, EPI, TILED, NT, 80>(mw, mx, g, st);
  }
  return launch_sk_bn_s<BN, EPI, TILED, NT, 200>(mw, mx, g, st);
}

// two token tiles per weight tile (256 < M <= 512)
template <int EPI>
int launch_sk_nt2(int bn, const CUtensorMap& mw, const CUtensorMap& mx, const SKArgs& g,
                  cudaStream_t st) {
  switch (bn) {
    case 128: return launch_sk_bn<128, EPI, false, 2>(mw, mx, g, st);
    case 160: return launch_sk_bn<160, EPI, false, 2>(mw, mx, g, st);
    case 192: return launch_sk_bn<192, EPI, false, 2>(mw, mx, g, st);
    case 224: return launch_sk_bn<224, EPI, false, 2>(mw, mx, g, st);
    case 256: return launch_sk_bn<256, EPI, false, 2>(mw, mx, g, st);
  }
  return (int)cudaErrorInvalidValue;
}

template <int BN, int EPI, int NT>
int launch_bn_nt(const CUtensorMap& mw, const CUtensorMap& mx, const GemmArgs& g, dim3 grid,
                 cudaStream_t st) {
  using C = Cfg<BN, NT>;
  {
    const cudaError_t e = psd::ensure_smem_limit((const void*)gemm_kernel<BN, EPI, NT>,
                                                 C::SMEM + ep_stage_bytes<EPI>(), st);
    if (e != cudaSuccess) return (int)e;
  }
  return (int)psd::launch(gemm_kernel<BN, EPI, NT>, grid, dim3(kThreads),
                          C::SMEM + ep_stage_bytes<EPI>(), st, mw, mx, g);
}

template <int EPI>
int launch_epi_nt2(int bn, const CUtensorMap& mw, const CUtensorMap& mx, const GemmArgs& g,
                   dim3 grid, cudaStream_t st) {
  switch (bn) {
    case 128: return launch_bn_nt<128, EPI, 2>(mw, mx, g, grid, st);
    case 160: return launch_bn_nt<160, EPI, 2>(mw, mx, g, grid, st);
    case 192: return launch_bn_nt<192, EPI, 2>(mw, mx, g, grid, st);
    case 224: return launch_bn_nt<224, EPI, 2>(mw, mx, g, grid, st);
    case 256: return launch_bn_nt<256, EPI, 2>(mw, mx, g, grid, st);
  }
  return (int)cudaErrorInvalidValue;
}

template <int EPI, bool TILED = false>
int launch_sk(int bn, const CUtensorMap& mw, const CUtensorMap& mx, const SKArgs& g,
              cudaStream_t st) {
  switch (bn) {
    case 32: return launch_sk_bn<32, EPI, TILED>(mw, mx, g, st);
    case 64: return launch_sk_bn<64, EPI, TILED>(mw, mx, g, st);
    case 96: return launch_sk_bn<96, EPI, TILED>(mw, mx, g, st);
    case 128: return launch_sk_bn<128, EPI, TILED>(mw, mx, g, st);
    case 160: return launch_sk_bn<160, EPI, TILED>(mw, mx, g, st);
    case 192: return launch_sk_bn<192, EPI, TILED>(mw, mx, g, st);
    case 224: return launch_sk_bn<224, EPI, TILED>(mw, mx, g, st);
    case 256: return launch_sk_bn<256, EPI, TILED>(mw, mx, g, st);
  }
  return (int)cudaErrorInvalidValue;
}

#if PSD_EXPERIMENTAL
// [N, K] row-major -> [N/128][KB][128][64] with the 128-byte swizzle applied
// (16-byte chunk j of row r stored at chunk j ^ (r & 7)), K zero-padded
__global__ void tile_weights_kernel(const __nv_bfloat16* __restrict__ W, int N, int K, int ldw,
                                    __nv_bfloat16* __restrict__ T) {
  const int KB = (K + BK - 1) / BK;
  const size_t nchunks = (size_t)N * KB * 8;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nchunks;
       q += (size_t)gridDim.x * blockDim.x) {
    const int jd = q & 7;
    const int r = (q >> 3) & 127;
    const size_t tk = q >> 10;  // (tile, kb)
    const int kb = (int)(tk % KB);
    const int tile = (int)(tk / KB);
    const int j = jd ^ (r & 7);
    const int n = tile * BM + r;
    const int k = kb * BK + j * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (k + 8 <= K) {
      v = *reinterpret_cast<const uint4*>(W + (size_t)n * ldw + k);
    } else if (k < K) {
      __nv_bfloat16 tmp[8];
      for (int e = 0; e < 8; ++e) tmp[e] = k + e < K ? W[(size_t)n * ldw + k + e] : __float2bfloat16(0.f);
      v = *reinterpret_cast<uint4*>(tmp);
    }
    reinterpret_cast<uint4*>(T)[q] = v;
  }
}
#endif  // PSD_EXPERIMENTAL

int token_tile(int M) {
  if (M > 256) {
    // fewest tiles, then least padding
    int best = 256, best_pad = 1 << 30;
    for (int bn = 256; bn >= 128; bn -= 32) {
      const int tiles = (M + bn - 1) / bn;
      const int pad = tiles * bn - M + tiles * 8;  // mild preference for fewer tiles
      if (pad < best_pad) { best_pad = pad; best = bn; }
    }
    return best;
  }
  return std::max(32, (M + 31) / 32 * 32);
}

// token geometry: bn rows per token tile, nt token tiles per weight tile (2
// above 256 tokens), mt token-tile groups (1 up to 512 tokens).  PSD_GEMM_NT2=0
// keeps one token tile per CTA (A/B runs)
struct TokGeo {
  int bn, nt, mt;
};
int nt2_enabled() {
  static int v = [] {
    const char* e = getenv("PSD_GEMM_NT2");
    return e ? atoi(e) : 1;
  }();
  return v;
}
TokGeo tok_geo(int M, bool allow_nt2 = true) {
  TokGeo t;
  if (allow_nt2 && M > 256 && nt2_enabled()) {
    // above 512 tokens: groups of <= 512 (two token tiles each), each group
    // running the one-group schedule (sk_plan), so fewer groups re-read the
    // weights and fix up split tiles than with single token tiles
    const int groups = (M + 511) / 512;
    t.bn = std::min(256, ((M + 2 * groups - 1) / (2 * groups) + 31) / 32 * 32);
    t.nt = 2;
  } else {
    t.bn = token_tile(M);
    t.nt = 1;
  }
  t.mt = (M + t.nt * t.bn - 1) / (t.nt * t.bn);
  return t;
}

// CTA budget of the GEMM grids (0 = every SM); psd_gemm_set_max_ctas.  Capping
// the verify GEMMs leaves SMs free for the concurrently running draft kernels.
std::atomic<int>& max_ctas_cap() {
  static std::atomic<int> v{0};
  return v;
}

// whole-K geometry (psd_gemm_set_whole_k): no k-splitting at all -- grid
// split-K runs one split, stream-K GEMMs run whole tiles only -- so every
// output element is one CTA's sequential accumulation over K whatever M is
// (prefill chunks of any composition give a prompt the same KV cache)
std::atomic<int>& whole_k() {
  static std::atomic<int> v{0};
  return v;
}

// stream-K timeline buffer (psd_gemm_set_trace; null = off)
std::atomic<unsigned long long*>& sk_trace() {
  static std::atomic<unsigned long long*> v{nullptr};
  return v;
}

int num_sms_raw();

// CTAs a stream-K launch of G virtual CTAs runs on: the cap, rounded so that
// every physical CTA gets the same number of virtual ones when possible
int sk_physical(int G) {
  const int cap = max_ctas_cap().load(std::memory_order_relaxed);
  if (cap <= 0 || cap >= G) return G;
  const int per = (G + cap - 1) / cap;  // virtual CTAs per physical CTA
  return (G + per - 1) / per;
}

int num_sms_raw() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// stream-K geometry + workspace bytes (partials, then tickets)
// PSD_GEMM_SK_DP=0: pure stream-K over all tiles (A/B switch)
bool sk_dp_enabled() {
  static bool v = [] {
    const char* e = getenv("PSD_GEMM_SK_DP");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

struct SKPlan {
  int bn, nt, KB, MT, tiles, G, D, G1, T1;
  long long U;
  size_t part_bytes, ticket_bytes;
};
// stream-K keeps one TMEM accumulator when it holds two token tiles (no epilogue
// overlap), which only pays when a CTA covers >= 2 weight tiles
// (70B gate/up at M = 320: 426 -> 294 us; 8B gate/up at M = 384: 110 -> 117 us)
SKPlan sk_plan(int M, int N, int K, bool allow_nt2 = true) {
  SKPlan p;
  // batch-invariant geometry: the k-block split of every tile depends only on
  // (N, K) and the SM count -- not on the CTA cap, and not on M.  One group's
  // schedule (G1 virtual CTAs over the T1 = N / 128 weight tiles) is planned
  // as for a single token tile; M > 512 runs MT groups of it (G = G1 * MT
  // virtual CTAs, a physical CTA runs a segment for every group in turn),
  // 256 < M <= 512 one group with two token tiles per weight tile
  const TokGeo tg = tok_geo(M, allow_nt2);
  p.bn = tg.bn;
  p.nt = tg.nt;
  p.KB = (K + BK - 1) / BK;
  p.MT = tg.mt;
  p.T1 = N / BM;
  p.tiles = p.T1 * p.MT;
  p.G1 = (int)std::min<long long>(num_sms_raw(), (long long)p.T1 * p.KB);
  p.G = p.G1 * p.MT;
  // data-parallel + stream-K: each CTA takes T1 / G1 whole tiles and an
  // equal share of the remaining tiles' k-blocks; a remainder that would cut
  // every tile into more than ~2 pieces gets one more stream-K wave instead
  p.D = sk_dp_enabled() ? p.G1 * (p.T1 / p.G1) : 0;
  if (p.D > 0 && p.D < p.T1 && (long long)(p.T1 - p.D) * p.KB < (long long)p.G1 * (p.KB / 2))
    p.D -= p.G1;
  if (whole_k().load(std::memory_order_relaxed)) p.D = p.T1;
  p.U = (long long)(p.T1 - p.D) * p.KB;
  p.part_bytes = (size_t)p.G * 2 * p.nt * p.bn * BM * sizeof(float);
  // tickets live at a FIXED offset (start of the workspace) so GEMMs of any
  // shape can share one workspace: each leaves its tickets zeroed
  p.ticket_bytes = (size_t)kMaxTiles * sizeof(int);
  return p;
}

template <int EPI>
int launch_epi(int bn, const CUtensorMap& mw, const CUtensorMap& mx, const GemmArgs& g, dim3 grid,
               cudaStream_t st) {
  switch (bn) {
    case 32: return launch_bn<32, EPI>(mw, mx, g, grid, st);
    case 64: return launch_bn<64, EPI>(mw, mx, g, grid, st);
    case 96: return launch_bn<96, EPI>(mw, mx, g, grid, st);
    case 128: return launch_bn<128, EPI>(mw, mx, g, grid, st);
    case 160: return launch_bn<160, EPI>(mw, mx, g, grid, st);
    case 192: return launch_bn<192, EPI>(mw, mx, g, grid, st);
    case 224: return launch_bn<224, EPI>(mw, mx, g, grid, st);
    case 256: return launch_bn<256, EPI>(mw, mx, g, grid, st);
  }
  return (int)cudaErrorInvalidValue;
}


// K6 fold: token m's argmax over the vocabulary tiles' (max, index) partials
// (ties -> lowest index, as K1's canonical argmax); optionally scattered into
// dst[dst_idx[m]] (the draft token into its slot; a negative index skips)
__global__ void __launch_bounds__(256)
argmax_fold_kernel(const float2* __restrict__ part, int ntiles, int M, int32_t* __restrict__ out,
                   int32_t* __restrict__ dst, const int32_t* __restrict__ dst_idx) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x, tid = threadIdx.x;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = tid; t < ntiles; t += 256) {
    const float2 p = __ldcg(part + (size_t)m * ntiles + t);
    const int i = __float_as_int(p.y);
    if (p.x > bv || (p.x == bv && i < bi)) { bv = p.x; bi = i; }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  __shared__ float sv[8];
  __shared__ int si[8];
  if ((tid & 31) == 0) { sv[tid >> 5] = bv; si[tid >> 5] = bi; }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < 8; ++w)
      if (sv[w] > bv || (sv[w] == bv && si[w] < bi)) { bv = sv[w]; bi = si[w]; }
    if (out) out[m] = bi;
    if (dst && dst_idx) {
      const int d = dst_idx[m];
      if (d >= 0) dst[d] = bi;
    }
  }
}

}  // namespace

extern "C" {

void psd_gemm_set_max_ctas(int n) { max_ctas_cap().store(n > 0 ? n : 0); }

void psd_gemm_set_whole_k(int on) { whole_k().store(on ? 1 : 0); }

void psd_gemm_set_trace(void* trace) {
  sk_trace().store(static_cast<unsigned long long*>(trace));
}

int psd_gemm_plan(int M, int N, int K, int epi, int splits_hint, int* splits_out,
                  size_t* workspace_bytes) {
  if (M <= 0 || N <= 0 || K <= 0 || (K % 8) || (N % BM)) return (int)cudaErrorInvalidValue;
  // weight tiles of ONE token tile: the split (and so the summation order of
  // every output element) depends on (N, K) and the SM count -- not on M, and
  // not on the CTA cap or what runs beside the GEMM
  const int tiles = N / BM;
  const int kb_total = (K + BK - 1) / BK;
  int splits = splits_hint;
  if (splits <= 0) {
    splits = 1;
    if (tiles < 120) splits = std::max(1, std::min(num_sms_raw() / tiles, kb_total / 4));
    if (whole_k().load(std::memory_order_relaxed)) splits = 1;
  }
  splits = std::max(1, std::min(splits, kb_total));
  const int per = (kb_total + splits - 1) / splits;
  splits = (kb_total + per - 1) / per;
  if (splits_out) *splits_out = splits;
  if (workspace_bytes) {
    if (splits_hint == 0 && epi != PSD_EPI_PARTIAL) {
      const SKPlan p = sk_plan(M, N, K);  // stream-K path
      *workspace_bytes = p.part_bytes + p.ticket_bytes;
    } else {
      *workspace_bytes = splits > 1 ? (size_t)splits * M * N * sizeof(float) : 0;
    }
  }
  return 0;
}

#if PSD_EXPERIMENTAL
size_t psd_tiled_weight_bytes(int N, int K) {
  return (size_t)N * ((K + BK - 1) / BK) * BK * sizeof(__nv_bfloat16);
}

int psd_tile_weights(const void* W, int N, int K, int ldw, void* tiled, void* stream) {
  if (!W || !tiled || N % BM || K % 8 || ldw % 8) return (int)cudaErrorInvalidValue;
  psd::count_launches();
  tile_weights_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(W), N, K, ldw, static_cast<__nv_bfloat16*>(tiled));
  return (int)cudaGetLastError();
}

int psd_gemm_tiled(const void* X, int ldx, int M, int K, const void* W_tiled, int N, void* Y,
                   int ldy, int epi, const void* R, int ldr, void* workspace,
                   size_t workspace_bytes, void* stream) {
  if (!X || !W_tiled || !Y || epi < 0 || epi > PSD_EPI_SILU) return (int)cudaErrorInvalidValue;
  if (epi == PSD_EPI_RESID && !R) return (int)cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W_tiled)) & 15)
    return (int)cudaErrorMisalignedAddress;
  if (ldx % 8) return (int)cudaErrorMisalignedAddress;
  if (M <= 0 || N <= 0 || K <= 0 || (K % 8) || (N % BM)) return (int)cudaErrorInvalidValue;
  const SKPlan p = sk_plan(M, N, K, false);  // pre-tiled weights: one token tile per CTA
  if (!workspace || workspace_bytes < p.part_bytes + p.ticket_bytes || p.tiles > kMaxTiles)
    return (int)cudaErrorInvalidValue;
  CUtensorMap mx;
  int rc;
  if ((rc = make_map(&mx, X, M, K, ldx, p.bn))) return rc;
  SKArgs g;
  g.M = M; g.N = N; g.K = K;
  g.KB = p.KB; g.MT = p.MT; g.tiles = p.tiles; g.G = p.G; g.U = p.U; g.D = p.D;
  g.G1 = p.G1; g.T1 = p.T1;
  g.Y = Y; g.ldy = ldy; g.R = static_cast<const __nv_bfloat16*>(R); g.ldr = ldr;
  g.tickets = static_cast<int*>(workspace);
  g.part = reinterpret_cast<float*>(static_cast<char*>(workspace) + p.ticket_bytes);
  g.trace = sk_trace().load(std::memory_order_relaxed);
  g.Wt = static_cast<const __nv_bfloat16*>(W_tiled);
  set_out_map(g, epi, Y, M, N, ldy);
  cudaStream_t st = (cudaStream_t)stream;
  switch (epi) {
    case PSD_EPI_BF16: return launch_sk<PSD_EPI_BF16, true>(p.bn, mx, mx, g, st);
    case PSD_EPI_F32: return launch_sk<PSD_EPI_F32, true>(p.bn, mx, mx, g, st);
    case PSD_EPI_RESID: return launch_sk<PSD_EPI_RESID, true>(p.bn, mx, mx, g, st);
    case PSD_EPI_SILU: return launch_sk<PSD_EPI_SILU, true>(p.bn, mx, mx, g, st);
  }
  return (int)cudaErrorInvalidValue;
}
#endif  // PSD_EXPERIMENTAL

size_t psd_argmax_partials_bytes(int M, int N) {
  return (size_t)(N / BM) * M * sizeof(float2);
}

int psd_gemm_argmax(const void* X, int ldx, int M, int K, const void* W, int ldw, int N,
                    const int32_t* tokens, const int32_t* rows, const int32_t* successor,
                    float beta, void* partials, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (!X || !W || !partials || M <= 0 || M > 512 || N <= 0 || K <= 0 || (K % 8) || (N % BM))
    return (int)cudaErrorInvalidValue;
  if (successor && beta != 0.f && !tokens) return (int)cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
    return (int)cudaErrorMisalignedAddress;
  if ((ldx % 8) || (ldw % 8)) return (int)cudaErrorMisalignedAddress;
  const SKPlan p = sk_plan(M, N, K);
  if (p.MT != 1) return (int)cudaErrorInvalidValue;
  if (!workspace || workspace_bytes < p.part_bytes + p.ticket_bytes || p.tiles > kMaxTiles)
    return (int)cudaErrorInvalidValue;
  CUtensorMap mw, mx;
  int rc;
  if ((rc = make_map(&mw, W, N, K, ldw, BM))) return rc;
  if ((rc = make_map(&mx, X, M, K, ldx, p.bn))) return rc;
  SKArgs g;
  memset(&g, 0, sizeof(g));
  g.M = M; g.N = N; g.K = K;
  g.KB = p.KB; g.MT = p.MT; g.tiles = p.tiles; g.G = p.G; g.U = p.U; g.D = p.D;
  g.G1 = p.G1; g.T1 = p.T1;
  g.Y = partials; g.ldy = M;
  g.tickets = static_cast<int*>(workspace);
  g.part = reinterpret_cast<float*>(static_cast<char*>(workspace) + p.ticket_bytes);
  g.trace = nullptr;
  g.Wt = nullptr;
  g.tma_y = 0;
  g.am_tok = tokens; g.am_rows = rows; g.am_succ = successor; g.am_beta = beta;
  cudaStream_t st = (cudaStream_t)stream;
  if (p.nt == 2) return launch_sk_nt2<PSD_EPI_ARGMAX>(p.bn, mw, mx, g, st);
  switch (p.bn) {
    case 32: return launch_sk_bn<32, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 64: return launch_sk_bn<64, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 96: return launch_sk_bn<96, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 128: return launch_sk_bn<128, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 160: return launch_sk_bn<160, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 192: return launch_sk_bn<192, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 224: return launch_sk_bn<224, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
    case 256: return launch_sk_bn<256, PSD_EPI_ARGMAX, false>(mw, mx, g, st);
  }
  return (int)cudaErrorInvalidValue;
}

int psd_argmax_fold(const void* partials, int M, int N, int32_t* out_tokens, int32_t* dst,
                    const int32_t* dst_idx, void* stream) {
  if (!partials || M <= 0 || N <= 0 || (N % BM) || (!out_tokens && !(dst && dst_idx)))
    return (int)cudaErrorInvalidValue;
  return (int)psd::launch(argmax_fold_kernel, dim3(M), dim3(256), 0, (cudaStream_t)stream,
                          static_cast<const float2*>(partials), N / BM, M, out_tokens, dst,
                          dst_idx);
}

int psd_gemm_partials(const void* X, int ldx, int M, int K, const void* W, int ldw, int N,
                      float* P, size_t p_bytes, int splits_hint, int* splits_used, void* stream) {
  if (!X || !W || !P) return (int)cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
    return (int)cudaErrorMisalignedAddress;
  if ((ldx % 8) || (ldw % 8)) return (int)cudaErrorMisalignedAddress;
  int splits = 1;
  int rc = psd_gemm_plan(M, N, K, PSD_EPI_PARTIAL, splits_hint, &splits, nullptr);
  if (rc) return rc;
  while (splits > 1 && (size_t)splits * M * N * sizeof(float) > p_bytes) --splits;
  if ((size_t)splits * M * N * sizeof(float) > p_bytes) return (int)cudaErrorInvalidValue;
  rc = psd_gemm_plan(M, N, K, PSD_EPI_PARTIAL, splits, &splits, nullptr);
  if (rc) return rc;
  const TokGeo tg = tok_geo(M);
  const int bn = tg.bn;
  CUtensorMap mw, mx;
  if ((rc = make_map(&mw, W, N, K, ldw, BM))) return rc;
  if ((rc = make_map(&mx, X, M, K, ldx, bn))) return rc;
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.kb_total = (K + BK - 1) / BK;
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  g.Y = P; g.ldy = N; g.R = nullptr; g.ldr = 0;
  set_grid_out_map(g, PSD_EPI_PARTIAL, P, M, N, N, splits);
  if (splits_used) *splits_used = splits;
  dim3 grid(N / BM, tg.mt, splits);
  if (tg.nt == 2)
    return launch_epi_nt2<PSD_EPI_PARTIAL>(bn, mw, mx, g, grid, (cudaStream_t)stream);
  return launch_epi<PSD_EPI_PARTIAL>(bn, mw, mx, g, grid, (cudaStream_t)stream);
}

int psd_gemm_bf16(const void* X, int ldx, int M, int K, const void* W, int ldw, int N, void* Y,
                  int ldy, int epi, const void* R, int ldr, int splits_hint, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (!X || !W || !Y || epi < 0 || epi > PSD_EPI_SILU) return (int)cudaErrorInvalidValue;
  if (epi == PSD_EPI_RESID && !R) return (int)cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(W)) & 15)
    return (int)cudaErrorMisalignedAddress;
  if ((ldx % 8) || (ldw % 8)) return (int)cudaErrorMisalignedAddress;
  if (splits_hint == 0 && M > 0 && N % BM == 0) {
    // one wave of whole-K tiles (>= 3/4 of the SMs busy, no tail): the plain
    // grid kernel beats stream-K, whose fix-ups buy nothing here (1B draft
    // gate/up at M = 32: 14.3 vs 19.8 us, profiles/r01b_kbench_gemm_splits.txt).
    // Decided on the weight tiles of one token tile so that every M takes the
    // same path (batch-invariant summation order)
    // Short-K GEMMs (K <= 1024: a few k-blocks per tile) take it from half a
    // wave: their stream-K fix-ups would cost more than the idle SMs (Qwen2.5-
    // 0.5B gate/up, 76 tiles x 14 k-blocks)
    const int tiles = N / BM;
    static const int short_k = [] {
      const char* e = getenv("PSD_GEMM_SHORTK_WAVE");
      return e ? atoi(e) : 1;
    }();
    if (tiles <= num_sms_raw() &&
        (4 * tiles >= 3 * num_sms_raw() || (short_k && K <= 1024 && 2 * tiles >= num_sms_raw())))
      splits_hint = 1;
  }
  if (splits_hint == 0) {
    // stream-K persistent path (default)
    if (M <= 0 || N <= 0 || K <= 0 || (K % 8) || (N % BM)) return (int)cudaErrorInvalidValue;
    const SKPlan p = sk_plan(M, N, K);
    if (!workspace || workspace_bytes < p.part_bytes + p.ticket_bytes || p.tiles > kMaxTiles)
      return (int)cudaErrorInvalidValue;
    CUtensorMap mw, mx;
    int rc;
    if ((rc = make_map(&mw, W, N, K, ldw, BM))) return rc;
    if ((rc = make_map(&mx, X, M, K, ldx, p.bn))) return rc;
    SKArgs g;
    g.M = M; g.N = N; g.K = K;
    g.KB = p.KB; g.MT = p.MT; g.tiles = p.tiles; g.G = p.G; g.U = p.U; g.D = p.D;
    g.G1 = p.G1; g.T1 = p.T1;
    g.Y = Y; g.ldy = ldy; g.R = static_cast<const __nv_bfloat16*>(R); g.ldr = ldr;
    g.tickets = static_cast<int*>(workspace);
    g.part = reinterpret_cast<float*>(static_cast<char*>(workspace) + p.ticket_bytes);
    g.trace = sk_trace().load(std::memory_order_relaxed);
    g.Wt = nullptr;
    set_out_map(g, epi, Y, M, N, ldy);
    cudaStream_t st = (cudaStream_t)stream;
    if (p.nt == 2) {
      switch (epi) {
        case PSD_EPI_BF16: return launch_sk_nt2<PSD_EPI_BF16>(p.bn, mw, mx, g, st);
        case PSD_EPI_F32: return launch_sk_nt2<PSD_EPI_F32>(p.bn, mw, mx, g, st);
        case PSD_EPI_RESID: return launch_sk_nt2<PSD_EPI_RESID>(p.bn, mw, mx, g, st);
        case PSD_EPI_SILU: return launch_sk_nt2<PSD_EPI_SILU>(p.bn, mw, mx, g, st);
      }
      return (int)cudaErrorInvalidValue;
    }
    switch (epi) {
      case PSD_EPI_BF16: return launch_sk<PSD_EPI_BF16>(p.bn, mw, mx, g, st);
      case PSD_EPI_F32: return launch_sk<PSD_EPI_F32>(p.bn, mw, mx, g, st);
      case PSD_EPI_RESID: return launch_sk<PSD_EPI_RESID>(p.bn, mw, mx, g, st);
      case PSD_EPI_SILU: return launch_sk<PSD_EPI_SILU>(p.bn, mw, mx, g, st);
    }
    return (int)cudaErrorInvalidValue;
  }
  int splits = 1;
  size_t need = 0;
  int rc = psd_gemm_plan(M, N, K, epi, splits_hint, &splits, &need);
  if (rc) return rc;
  if (splits > 1 && (!workspace || workspace_bytes < need)) {
    // not enough workspace: fall back to fewer splits that fit (or none)
    while (splits > 1 && (size_t)splits * M * N * sizeof(float) > workspace_bytes) --splits;
    rc = psd_gemm_plan(M, N, K, epi, splits, &splits, &need);
    if (rc) return rc;
    if (splits > 1 && (!workspace || workspace_bytes < need)) splits = 1;
  }
  const TokGeo tg = tok_geo(M);
  const int bn = tg.bn;
  CUtensorMap mw, mx;
  if ((rc = make_map(&mw, W, N, K, ldw, BM))) return rc;
  if ((rc = make_map(&mx, X, M, K, ldx, bn))) return rc;
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.kb_total = (K + BK - 1) / BK;
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;
  g.Y = splits > 1 ? workspace : Y;
  g.ldy = ldy; g.R = static_cast<const __nv_bfloat16*>(R); g.ldr = ldr;
  if (splits > 1)
    set_grid_out_map(g, PSD_EPI_PARTIAL, workspace, M, N, N, splits);
  else
    set_grid_out_map(g, epi, Y, M, N, ldy, 1);
  dim3 grid(N / BM, tg.mt, splits);
  cudaStream_t st = (cudaStream_t)stream;
  if (splits > 1) {
    rc = tg.nt == 2 ? launch_epi_nt2<PSD_EPI_PARTIAL>(bn, mw, mx, g, grid, st)
                    : launch_epi<PSD_EPI_PARTIAL>(bn, mw, mx, g, grid, st);
    if (rc) return rc;
    const int Nout = epi == PSD_EPI_SILU ? N / 2 : N;
    const size_t total = (size_t)M * Nout;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
    psd::count_launches();
    gemm_reduce_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(workspace), splits, M, N,
                                               epi, Y, ldy, static_cast<const __nv_bfloat16*>(R),
                                               ldr);
    return (int)cudaGetLastError();
  }
  if (tg.nt == 2) {
    switch (epi) {
      case PSD_EPI_BF16: return launch_epi_nt2<PSD_EPI_BF16>(bn, mw, mx, g, grid, st);
      case PSD_EPI_F32: return launch_epi_nt2<PSD_EPI_F32>(bn, mw, mx, g, grid, st);
      case PSD_EPI_RESID: return launch_epi_nt2<PSD_EPI_RESID>(bn, mw, mx, g, grid, st);
      case PSD_EPI_SILU: return launch_epi_nt2<PSD_EPI_SILU>(bn, mw, mx, g, grid, st);
    }
    return (int)cudaErrorInvalidValue;
  }
  switch (epi) {
    case PSD_EPI_BF16: return launch_epi<PSD_EPI_BF16>(bn, mw, mx, g, grid, st);
    case PSD_EPI_F32: return launch_epi<PSD_EPI_F32>(bn, mw, mx, g, grid, st);
    case PSD_EPI_RESID: return launch_epi<PSD_EPI_RESID>(bn, mw, mx, g, grid, st);
    case PSD_EPI_SILU: return launch_epi<PSD_EPI_SILU>(bn, mw, mx, g, grid, st);
  }
  return (int)cudaErrorInvalidValue;
}

}  // extern "C"
