// decode_mk.cu -- the draft model's k-step greedy decode loop as ONE persistent
// kernel (a dataflow "megakernel").
//
// Replaces the draft pass duration of the reference (draft_latency.duration,
// pkg/src/specsim/engine.py:355-364, 376-380, 400-404) with the real draft
// model's k autoregressive decode steps.  The per-kernel forward (model.py
// Forward.run: ~130 launches per step, each paying launch, pipeline fill and
// drain at 32 tokens) is latency-bound at ~3x the HBM roofline; here every SM
// runs one CTA for the whole loop:
//
//   warp 0  TMA producer: streams the weight tiles of every GEMM this CTA owns,
//           in program order, into a smem ring.  Weights never depend on
//           activations, so they run ahead across op boundaries (norms,
//           attention, argmax) limited only by the ring; the token tile of a
//           k-block is issued once the op producing it has completed.
//   warp 1  MMA issuer: tcgen05.mma (swap-AB: 128 weight rows x 64 tokens),
//           fp32 accumulators double-buffered in TMEM.
//   warps 2-5  compute: GEMM epilogues (tcgen05.ld -> split-K partials, fused
//           SiLU*up, fused LM-head bias+argmax partials) and the non-GEMM ops
//           (embedding+RMSNorm, residual add+RMSNorm, RoPE+paged-KV write+
//           attention, argmax reduction + scatter of the draft token).
//
// The program is a list of ops (host-built, per batch bucket and depth); unit
// u of op j runs on CTA (first_cta + u) % G.  An op's inputs are ready when the
// op it depends on has finished all its units (one global counter per op,
// release/acquire); the last CTA to exit zeroes the counters for the next
// launch.  All CTAs are co-resident (grid <= #SMs, 1 CTA per SM), so the
// in-order waits cannot deadlock.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/psd.h"
#include "../../include/psd_experimental.h"
#include "common.h"
#include "sm100.cuh"

namespace {
using namespace psd;
using bf16 = __nv_bfloat16;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int BN = 64;  // token tile: decode passes carry <= 64 tokens
constexpr int kThreads = 192;
constexpr int kCompute = 128;  // warps 2..5
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int STAGES = 6;
constexpr int TMEM_COLS = 2 * BN;
// attention (head_dim <= 64, <= 16 query rows per (sequence, kv head))
constexpr int ATT_D = 64;
constexpr int ATT_P = ATT_D + 8;
constexpr int ATT_KT = 32;
constexpr int ATT_KG = 4;
constexpr int ATT_NS = 2;
constexpr int ATT_ROWS = 16;
constexpr int ATT_MAX_BLOCKS = 512;
constexpr int SMEM_RING = STAGES * STAGE;
constexpr int SMEM_SQ = ATT_ROWS * ATT_P * 2;
constexpr int SMEM_ATT = ATT_NS * ATT_KG * 2 * ATT_KT * ATT_P * 2;
constexpr int SMEM_TOTAL = 1024 + SMEM_RING + SMEM_SQ + SMEM_ATT;

enum OpType { OP_GEMM = 0, OP_EMBED_NORM = 1, OP_ADD_NORM = 2, OP_ROPE_ATTN = 3, OP_ARGMAX = 4 };
enum Epi { E_PART = 0, E_SILU = 1, E_ARG = 2 };

struct Op {
  int type, units, dep, first;
  // GEMM
  int tmw, tmx, epi, M, N, KB, kb_per_unit, tiles;
  void* out;
  // norms
  const float* P;
  int S, write_back;
  const bf16* w;
  bf16* y;
  int rows_field;  // meta field index of a row indirection (-1: identity)
  // per-step metadata set / layer
  int set, layer;
};

struct LayerPtrs {
  const bf16* bqkv;
  bf16* kc;
  bf16* vc;
};

// meta field indices (model.py META_FIELDS order)
enum { F_TOKENS = 0, F_POS, F_SLOTS, F_SEQ_SLOT, F_Q_START, F_Q_LEN, F_Q_POS0, F_KV_LEN,
       F_LOGIT_ROWS, F_GATHER, F_SCATTER, F_COUNT };

struct Params {
  const Op* ops;
  int n_ops;
  const CUtensorMap* maps;
  int* counters;  // [n_ops + 1], zero between launches
  int G;
  int H, Hq, Hkv, D, V, nseq;
  float eps, scale_log2, beta;
  int bs, max_blocks;
  const int32_t* block_table;
  const float* inv_freq;
  const bf16* embed;
  const int32_t* succ;
  bf16* x;
  float2* argpart;  // [tiles][R]
  int32_t* slot_tok;
  int32_t* meta;  // sets x set_stride
  int set_stride;
  int off[F_COUNT];
  const LayerPtrs* layers;
  unsigned long long* trace;  // optional [G][n_ops][3] globaltimer ns: entry, inputs ready, done
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int32_t* field(const Params& p, int set, int f) {
  return p.meta + (size_t)set * p.set_stride + p.off[f];
}

__device__ __forceinline__ int ld_acquire(const int* ptr) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void wait_op(const Params& p, int j) {
  const int need = p.ops[j].units;
  uint32_t spins = 0;
  while (ld_acquire(p.counters + j) < need) {
    __nanosleep(32);
    if (++spins > (1u << 27)) __trap();
  }
}
__device__ __forceinline__ void cbar() { named_bar_sync(1, kCompute); }

// sum of S <= 16 split-K partials (base[z * slice], z ascending: P0 + P1 + ...)
// with every load issued before the first add (one L2 latency, not S)
__device__ __forceinline__ float sum_splits(const float* base, size_t slice, int S) {
  float v[16];
#pragma unroll
  for (int z = 0; z < 16; ++z) v[z] = z < S ? __ldcg(base + z * slice) : 0.f;
  float a = v[0];
#pragma unroll
  for (int z = 1; z < 16; ++z)
    if (z < S) a += v[z];
  return a;
}
__device__ __forceinline__ float4 sum_splits4(const float* base, size_t slice, int S) {
  float4 v[16];
#pragma unroll
  for (int z = 0; z < 16; ++z)
    v[z] = z < S ? __ldcg(reinterpret_cast<const float4*>(base + z * slice))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 a = v[0];
#pragma unroll
  for (int z = 1; z < 16; ++z)
    if (z < S) {
      a.x += v[z].x; a.y += v[z].y; a.z += v[z].z; a.w += v[z].w;
    }
  return a;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// units of op j owned by CTA c: u = (c - first) mod G, then + G ...
__device__ __forceinline__ int first_unit(const Op& op, int c, int G) {
  return ((c - op.first) % G + G) % G;
}

// ---- GEMM unit geometry ----------------------------------------------------------
struct Unit {
  int n0, kb0, kb1, z;
};
__device__ __forceinline__ Unit gemm_unit(const Op& op, int u) {
  Unit r;
  const int t = u % op.tiles;
  r.z = u / op.tiles;
  r.n0 = t * BM;
  r.kb0 = r.z * op.kb_per_unit;
  r.kb1 = min(op.KB, r.kb0 + op.kb_per_unit);
  return r;
}

// cursor over the (op, unit, k-block) sequence of this CTA's GEMM work
struct Cursor {
  int op, u, kb;
  Unit un;
  bool done;
  __device__ void seek(const Params& p, int c) {
    // advance to the first GEMM op with a unit here, starting at (op, u)
    while (op < p.n_ops) {
      const Op& o = p.ops[op];
      if (o.type == OP_GEMM && u < o.units) {
        un = gemm_unit(o, u);
        if (un.kb1 > un.kb0) {
          kb = un.kb0;
          done = false;
          return;
        }
        u += p.G;
        continue;
      }
      ++op;
      if (op < p.n_ops) u = first_unit(p.ops[op], c, p.G);
    }
    done = true;
  }
  __device__ void start(const Params& p, int c) {
    op = 0;
    u = p.n_ops ? first_unit(p.ops[0], c, p.G) : 0;
    seek(p, c);
  }
  __device__ void next(const Params& p, int c) {
    if (++kb < un.kb1) return;
    u += p.G;
    seek(p, c);
  }
};

// ---- producer -------------------------------------------------------------------
__device__ void producer(const Params& p, uint8_t* sA, uint8_t* sB, uint64_t* full,
                         uint64_t* empty) {
  const int c = blockIdx.x;
  const uint64_t pol_w = policy_evict_first();
  const uint64_t pol_x = policy_evict_last();
  Cursor ca, cb;
  ca.start(p, c);
  cb.start(p, c);
  int ia = 0, ib = 0;
  int ready_op = -1;  // last op whose dependency was observed complete (B side)
  uint32_t idle = 0;
  while (true) {
    bool prog = false;
    if (!ca.done && ia - ib < STAGES) {
      const int s = ia % STAGES;
      const uint32_t ph = (ia / STAGES) & 1;
      if (mbar_try_wait(empty + s, ph ^ 1)) {
        const Op& o = p.ops[ca.op];
        mbar_arrive_expect_tx(full + s, STAGE);
        tma_load_2d(sA + s * A_BYTES, p.maps + o.tmw, full + s, ca.kb * BK, ca.un.n0, pol_w);
        ++ia;
        ca.next(p, c);
        prog = true;
      }
    }
    if (ib < ia) {
      const Op& o = p.ops[cb.op];
      bool ok = ready_op == cb.op || o.dep < 0;
      if (!ok && ld_acquire(p.counters + o.dep) >= p.ops[o.dep].units) {
        fence_proxy_async();
        ready_op = cb.op;
        ok = true;
      }
      if (ok) {
        const int s = ib % STAGES;
        tma_load_2d(sB + s * B_BYTES, p.maps + o.tmx, full + s, cb.kb * BK, 0, pol_x);
        ++ib;
        cb.next(p, c);
        prog = true;
      }
    }
    if (ca.done && ib == ia) break;
    if (!prog) {
      __nanosleep(20);
      if (++idle > (1u << 28)) __trap();
    }
  }
}

// ---- MMA issuer -----------------------------------------------------------------
__device__ void mma_issuer(const Params& p, uint8_t* sA, uint8_t* sB, uint64_t* full,
                           uint64_t* empty, uint64_t* tfull, uint64_t* tempty, uint32_t tmem) {
  const int c = blockIdx.x;
  constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
  int i = 0, j = 0;
  for (int oi = 0; oi < p.n_ops; ++oi) {
    const Op& o = p.ops[oi];
    if (o.type != OP_GEMM) continue;
    for (int u = first_unit(o, c, p.G); u < o.units; u += p.G) {
      const Unit un = gemm_unit(o, u);
      if (un.kb1 <= un.kb0) continue;
      const int a = j & 1;
      mbar_wait(tempty + a, ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + a * BN;
      for (int kb = un.kb0; kb < un.kb1; ++kb, ++i) {
        const int s = i % STAGES;
        mbar_wait(full + s, (i / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(sA + s * A_BYTES);
        const uint32_t sb = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          mma_bf16(d, umma_desc_sw128(sa + kk * 32), umma_desc_sw128(sb + kk * 32), idesc,
                   (kb != un.kb0 || kk != 0) ? 1u : 0u);
        mma_commit(empty + s);
      }
      mma_commit(tfull + a);
      ++j;
    }
  }
}

__device__ __forceinline__ float silu(float x) {
  float t;
  const float h = 0.5f * x;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
  return fmaf(h, t, h);
}

// ---- compute warps: one op unit each ----------------------------------------------
struct Smem {
  bf16 (*sQ)[ATT_P];
  bf16 (*ring)[ATT_P];
  float* red;      // 32 floats
  float2* argx;    // [4][BN]
  int* bt;         // block-table row
  float* sc;       // cos [32], sin [32]
};

// GEMM epilogue of one unit (accumulator a)
__device__ void epilogue(const Params& p, const Op& o, const Unit& un, uint32_t tbase,
                         const Smem& sm) {
  const int ct = threadIdx.x - 64;
  const int q = (threadIdx.x >> 5) & 3;  // TMEM lane quarter of this warp
  const int lane = threadIdx.x & 31;
  const int row = 32 * q + lane;
  const uint32_t tq = tbase + ((uint32_t)(32 * q) << 16);
  if (o.epi == E_ARG) {
    // LM head: v = logit (+beta at succ[prev token]); per token column the
    // first-max over this tile's 128 vocab rows -> argpart[tile][m]
    const int n = un.n0 + row;
    const int32_t* toks = field(p, o.set, F_TOKENS);
    const int32_t* lrows = field(p, o.set, F_LOGIT_ROWS);
    for (int c0 = 0; c0 < BN && c0 < o.M; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tq + (uint32_t)c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int m = c0 + k;
        if (m >= o.M) break;
        float v = __uint_as_float(r[k]);
        if (p.beta != 0.0f) {
          const int prev = toks[lrows[m]];
          if (prev >= 0 && prev < p.V && p.succ[prev] == n) v += p.beta;
        }
        int idx = n;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
          if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (lane == 0) sm.argx[q * BN + m] = make_float2(v, __int_as_float(idx));
      }
    }
    cbar();
    if (ct < o.M) {
      float2 best = sm.argx[ct];
#pragma unroll
      for (int w = 1; w < 4; ++w) {
        const float2 c = sm.argx[w * BN + ct];
        if (c.x > best.x || (c.x == best.x && __float_as_int(c.y) < __float_as_int(best.y)))
          best = c;
      }
      p.argpart[(size_t)(un.n0 / BM) * o.M + ct] = best;
    }
    return;
  }
  for (int c0 = 0; c0 < BN && c0 < o.M; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tq + (uint32_t)c0, r);
    tmem_ld_wait();
    if (o.epi == E_SILU) {
      const int jo = (un.n0 / BM) * 64 + 16 * q + (lane & 15);
      bf16* Y = static_cast<bf16*>(o.out);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float mine = __uint_as_float(r[k]);
        const float up = __shfl_down_sync(0xffffffffu, mine, 16);
        const int m = c0 + k;
        if (lane < 16 && m < o.M) Y[(size_t)m * (o.N / 2) + jo] = __float2bfloat16(silu(mine) * up);
      }
    } else {
      float* P = static_cast<float*>(o.out) + (size_t)un.z * o.M * o.N;
      const int n = un.n0 + row;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int m = c0 + k;
        if (m >= o.M) break;
        P[(size_t)m * o.N + n] = __uint_as_float(r[k]);
      }
    }
  }
}

// v = bf16(x[src] (+ sum_z P[z][src])) written back, y = v * rsqrt(mean v^2 + eps) * w
__device__ void norm_row(const Params& p, const bf16* xsrc, bf16* xdst, const float* P, int S,
                         size_t slice, const bf16* w, bf16* y, const Smem& sm) {
  const int ct = threadIdx.x - 64;
  constexpr int MAXC = 4;  // 8-wide chunks per thread: H <= 4096
  float v[MAXC][8];
  float ss = 0.f;
  const int nch = p.H / 8;
#pragma unroll
  for (int k = 0; k < MAXC; ++k) {
    const int ch = ct + k * kCompute;
    if (ch < nch) {
      const int e = ch * 8;
      uint4 u = *reinterpret_cast<const uint4*>(xsrc + e);
      const bf16* b8 = reinterpret_cast<const bf16*>(&u);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[k][t] = __bfloat162float(b8[t]);
      if (P) {
        float acc[8];
        const float4 a0 = sum_splits4(P + e, slice, S), a1 = sum_splits4(P + e + 4, slice, S);
        acc[0] = a0.x; acc[1] = a0.y; acc[2] = a0.z; acc[3] = a0.w;
        acc[4] = a1.x; acc[5] = a1.y; acc[6] = a1.z; acc[7] = a1.w;
        uint4 o;
        bf16* o8 = reinterpret_cast<bf16*>(&o);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          o8[t] = __float2bfloat16(acc[t] + v[k][t]);
          v[k][t] = __bfloat162float(o8[t]);
        }
        if (xdst) *reinterpret_cast<uint4*>(xdst + e) = o;
      } else if (xdst && xdst != xsrc) {
        *reinterpret_cast<uint4*>(xdst + e) = u;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) ss += v[k][t] * v[k][t];
    }
  }
  ss = warp_sum(ss);
  const int cw = ct >> 5;
  if ((ct & 31) == 0) sm.red[cw] = ss;
  cbar();
  const float tot = (sm.red[0] + sm.red[1]) + (sm.red[2] + sm.red[3]);
  const float inv = rsqrtf(tot / p.H + p.eps);
#pragma unroll
  for (int k = 0; k < MAXC; ++k) {
    const int ch = ct + k * kCompute;
    if (ch < nch) {
      const int e = ch * 8;
      uint4 wu = *reinterpret_cast<const uint4*>(w + e);
      const bf16* w8 = reinterpret_cast<const bf16*>(&wu);
      uint4 o;
      bf16* o8 = reinterpret_cast<bf16*>(&o);
#pragma unroll
      for (int t = 0; t < 8; ++t) o8[t] = __float2bfloat16(v[k][t] * inv * __bfloat162float(w8[t]));
      *reinterpret_cast<uint4*>(y + e) = o;
    }
  }
  cbar();  // sm.red reuse
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], const void* ptr) {
  const uint32_t a = smem_u32(ptr);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// RoPE + paged KV write of this (sequence, kv head)'s new tokens, Q rows into
// smem, then causal attention over the paged cache (mma.sync, 4 key groups)
template <int D>
__device__ void rope_attn(const Params& p, const Op& o, int unit, const Smem& sm) {
  const int ct = threadIdx.x - 64, lane = threadIdx.x & 31, cw = ct >> 5;
  const int seq = unit / p.Hkv, hk = unit % p.Hkv;
  const int G = p.Hq / p.Hkv;
  const int set = o.set;
  const int ql = field(p, set, F_Q_LEN)[seq];
  const int qs = field(p, set, F_Q_START)[seq];
  const int p0 = field(p, set, F_Q_POS0)[seq];
  const int kvl = field(p, set, F_KV_LEN)[seq];
  const int srow = field(p, set, F_SEQ_SLOT)[seq];
  const int32_t* pos = field(p, set, F_POS);
  const int32_t* slots = field(p, set, F_SLOTS);
  const LayerPtrs L = p.layers[o.layer];
  const int NQKV = (p.Hq + 2 * p.Hkv) * D;
  const int M = o.M;  // tokens of this pass (partials row count)
  const size_t slice = (size_t)M * NQKV;
  const int R = ql * G;
  constexpr int half = D / 2;
  // ---- block table + earlier steps' keys of the first tile group ------------
  const int last_key = min(p0 + ql - 1, kvl - 1);
  const int* btg = p.block_table + (size_t)srow * p.max_blocks;
  const int nblk = min(last_key / p.bs + 1, ATT_MAX_BLOCKS);
  for (int i = ct; i < nblk; i += kCompute) sm.bt[i] = btg[i];
  cbar();
  typedef bf16 Row[ATT_P];
  Row* ring = sm.ring;
  auto sK = [&](int st, int j) { return ring + ((st * ATT_KG + j) * 2) * ATT_KT; };
  auto sV = [&](int st, int j) { return ring + ((st * ATT_KG + j) * 2 + 1) * ATT_KT; };
  const int ntiles = last_key / ATT_KT + 1;
  const int ngroups = (ntiles + ATT_KG - 1) / ATT_KG;
  // part: 0 all rows, 1 keys of earlier steps only (< p0), 2 the complement
  auto load_group = [&](int gi, int st, int part) {
    constexpr int per = ATT_KT * (D / 8);
    for (int idx = ct; idx < ATT_KG * per; idx += kCompute) {
      const int j = idx / per, rem = idx % per;
      const int r = rem / (D / 8), cc = rem % (D / 8);
      const int key = (gi * ATT_KG + j) * ATT_KT + r;
      const bool ok = key <= last_key;
      const bool old = ok && key < p0;
      if ((part == 1 && !old) || (part == 2 && old)) continue;
      size_t off = 0;
      if (ok) off = (((size_t)sm.bt[key / p.bs] * p.bs + key % p.bs) * p.Hkv + hk) * D + cc * 8;
      cp16(&sK(st, j)[r][cc * 8], L.kc + off, ok);
      cp16(&sV(st, j)[r][cc * 8], L.vc + off, ok);
    }
    asm volatile("cp.async.commit_group;");
  };
  load_group(0, 0, 1);
  if (ngroups > 1) load_group(1, 1, 1);
  else asm volatile("cp.async.commit_group;");
  // ---- RoPE + KV write + Q into smem --------------------------------------
  for (int t = 0; t < ql; ++t) {
    const int m = qs + t;
    const int ps = pos[m];
    const int sl = slots[m];
    if (ct < half) {
      float sn, cs;
      sincosf((float)ps * p.inv_freq[ct], &sn, &cs);
      sm.sc[ct] = cs;
      sm.sc[32 + ct] = sn;
    }
    cbar();
    // work items: (G q heads + 1 k head) x half pairs, then V (D)
    const int nrot = (G + 1) * half;
    for (int idx = ct; idx < nrot + D; idx += kCompute) {
      if (idx >= nrot) {
        const int i = idx - nrot;
        const int col = (p.Hq + p.Hkv + hk) * D + i;
        float a = sum_splits(o.P + (size_t)m * NQKV + col, slice, o.S);
        a = __bfloat162float(__float2bfloat16(a));
        if (L.bqkv) a = a + __bfloat162float(L.bqkv[col]);
        if (sl >= 0) L.vc[((size_t)sl * p.Hkv + hk) * D + i] = __float2bfloat16(a);
        continue;
      }
      const int hh = idx / half, i = idx % half;  // hh < G: q head hk*G+hh; hh == G: k head
      const int head = hh < G ? hk * G + hh : p.Hq + hk;
      const int col = head * D + i;
      float a = sum_splits(o.P + (size_t)m * NQKV + col, slice, o.S);
      float b = sum_splits(o.P + (size_t)m * NQKV + col + half, slice, o.S);
      a = __bfloat162float(__float2bfloat16(a));
      b = __bfloat162float(__float2bfloat16(b));
      if (L.bqkv) {
        a = __bfloat162float(__float2bfloat16(a + __bfloat162float(L.bqkv[col])));
        b = __bfloat162float(__float2bfloat16(b + __bfloat162float(L.bqkv[col + half])));
      }
      const float cs = sm.sc[i], sn = sm.sc[32 + i];
      const bf16 ra = __float2bfloat16(a * cs - b * sn);
      const bf16 rb = __float2bfloat16(b * cs + a * sn);
      if (hh < G) {
        sm.sQ[t * G + hh][i] = ra;
        sm.sQ[t * G + hh][i + half] = rb;
      } else if (sl >= 0) {
        bf16* dst = L.kc + ((size_t)sl * p.Hkv + hk) * D;
        dst[i] = ra;
        dst[i + half] = rb;
      }
    }
    cbar();
  }
  for (int idx = ct; idx < (ATT_ROWS - R) * D; idx += kCompute)
    sm.sQ[R + idx / D][idx % D] = __float2bfloat16(0.f);
  __threadfence();  // this step's K / V rows are read back below (through L2)
  cbar();
  // ---- attention ------------------------------------------------------------
  load_group(0, 0, 2);  // this step's keys (and the zero fill) of groups 0, 1
  if (ngroups > 1) load_group(1, 1, 2);
  else asm volatile("cp.async.commit_group;");
  const int g = lane >> 2, c = lane & 3;
  const int r0 = g, r1 = g + 8;
  const int lim0 = r0 < R ? min(p0 + r0 / G, kvl - 1) : -1;
  const int lim1 = r1 < R ? min(p0 + r1 / G, kvl - 1) : -1;
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    qf[kk][0] = *reinterpret_cast<const uint32_t*>(&sm.sQ[r0][kk * 16 + 2 * c]);
    qf[kk][1] = *reinterpret_cast<const uint32_t*>(&sm.sQ[r1][kk * 16 + 2 * c]);
    qf[kk][2] = *reinterpret_cast<const uint32_t*>(&sm.sQ[r0][kk * 16 + 8 + 2 * c]);
    qf[kk][3] = *reinterpret_cast<const uint32_t*>(&sm.sQ[r1][kk * 16 + 8 + 2 * c]);
  }
  float oacc[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) oacc[n][0] = oacc[n][1] = oacc[n][2] = oacc[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int kg = cw;
  // groups 0 and 1 are in flight (4 commit groups); group gi + 2 is issued
  // once group gi's stage is consumed
  for (int gi = 0; gi < ngroups; ++gi) {
    const int st = gi % ATT_NS;
    // outstanding after group gi: group gi + 1's last commit (gi = 0: part 2 of
    // group 1; gi >= 1: group gi + 1, issued at the end of iteration gi - 1)
    if (gi + 1 < ngroups) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    cbar();
    const int kt = gi * ATT_KG + kg;
    if (kt < ntiles) {
      Row* K = sK(st, kg);
      Row* V = sV(st, kg);
      float sacc[ATT_KT / 8][4];
#pragma unroll
      for (int n = 0; n < ATT_KT / 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < ATT_KT / 8; ++n) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&K[n * 8 + g][kk * 16 + 2 * c]);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&K[n * 8 + g][kk * 16 + 8 + 2 * c]);
          mma16816(sacc[n], qf[kk], b0, b1);
        }
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int n = 0; n < ATT_KT / 8; ++n) {
        const int key = kt * ATT_KT + n * 8 + 2 * c;
        sacc[n][0] = key <= lim0 ? sacc[n][0] * p.scale_log2 : -INFINITY;
        sacc[n][1] = key + 1 <= lim0 ? sacc[n][1] * p.scale_log2 : -INFINITY;
        sacc[n][2] = key <= lim1 ? sacc[n][2] * p.scale_log2 : -INFINITY;
        sacc[n][3] = key + 1 <= lim1 ? sacc[n][3] * p.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, fmaxf(sacc[n][0], sacc[n][1]));
        mx1 = fmaxf(mx1, fmaxf(sacc[n][2], sacc[n][3]));
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      const float base0 = mn0 == -INFINITY ? 0.f : mn0;
      const float base1 = mn1 == -INFINITY ? 0.f : mn1;
      const float al0 = exp2f(m0 - base0), al1 = exp2f(m1 - base1);
      m0 = mn0;
      m1 = mn1;
      float ps0 = 0.f, ps1 = 0.f;
      uint32_t pf[ATT_KT / 16][4];
#pragma unroll
      for (int n = 0; n < ATT_KT / 8; ++n) {
        const float e0 = exp2f(sacc[n][0] - base0), e1 = exp2f(sacc[n][1] - base0);
        const float e2 = exp2f(sacc[n][2] - base1), e3 = exp2f(sacc[n][3] - base1);
        ps0 += e0 + e1;
        ps1 += e2 + e3;
        const int kk = n >> 1;
        if ((n & 1) == 0) {
          pf[kk][0] = pack2(e0, e1);
          pf[kk][1] = pack2(e2, e3);
        } else {
          pf[kk][2] = pack2(e0, e1);
          pf[kk][3] = pack2(e2, e3);
        }
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        oacc[n][0] *= al0; oacc[n][1] *= al0; oacc[n][2] *= al1; oacc[n][3] *= al1;
      }
#pragma unroll
      for (int kk = 0; kk < ATT_KT / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < D / 8; n += 2) {
          uint32_t vb[4];
          const int mat = lane >> 3, rr = lane & 7;
          const int krow = kk * 16 + (mat & 1) * 8 + rr;
          const int dcol = (n + (mat >> 1)) * 8;
          ldsm_x4_trans(vb, &V[krow][dcol]);
          mma16816(oacc[n], pf[kk], vb[0], vb[1]);
          mma16816(oacc[n + 1], pf[kk], vb[2], vb[3]);
        }
      }
    }
    cbar();
    if (gi + 2 < ngroups) load_group(gi + 2, st, 0);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  // merge the 4 key groups through smem (the ring is free now)
  cbar();
  float* scr = reinterpret_cast<float*>(ring);
  constexpr int slot_floats = 16 * D + 32;
  if (kg > 0) {
    float* sp = scr + kg * slot_floats;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int d = n * 8 + 2 * c;
      sp[g * D + d] = oacc[n][0];
      sp[g * D + d + 1] = oacc[n][1];
      sp[(g + 8) * D + d] = oacc[n][2];
      sp[(g + 8) * D + d + 1] = oacc[n][3];
    }
    if (c == 0) {
      sp[16 * D + g] = m0;
      sp[16 * D + g + 8] = m1;
      sp[16 * D + 16 + g] = l0;
      sp[16 * D + 16 + g + 8] = l1;
    }
  }
  cbar();
  if (kg == 0) {
    float M0 = m0, M1 = m1;
    for (int j = 1; j < ATT_KG; ++j) {
      const float* sp = scr + j * slot_floats;
      M0 = fmaxf(M0, sp[16 * D + g]);
      M1 = fmaxf(M1, sp[16 * D + g + 8]);
    }
    const float w00 = M0 == -INFINITY ? 0.f : exp2f(m0 - M0);
    const float w10 = M1 == -INFINITY ? 0.f : exp2f(m1 - M1);
    l0 *= w00;
    l1 *= w10;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      oacc[n][0] *= w00; oacc[n][1] *= w00; oacc[n][2] *= w10; oacc[n][3] *= w10;
    }
    for (int j = 1; j < ATT_KG; ++j) {
      const float* sp = scr + j * slot_floats;
      const float mj0 = sp[16 * D + g], mj1 = sp[16 * D + g + 8];
      const float wj0 = mj0 == -INFINITY ? 0.f : exp2f(mj0 - M0);
      const float wj1 = mj1 == -INFINITY ? 0.f : exp2f(mj1 - M1);
      l0 += sp[16 * D + 16 + g] * wj0;
      l1 += sp[16 * D + 16 + g + 8] * wj1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int d = n * 8 + 2 * c;
        oacc[n][0] += sp[g * D + d] * wj0;
        oacc[n][1] += sp[g * D + d + 1] * wj0;
        oacc[n][2] += sp[(g + 8) * D + d] * wj1;
        oacc[n][3] += sp[(g + 8) * D + d + 1] * wj1;
      }
    }
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
    bf16* out = static_cast<bf16*>(o.out);
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int d = n * 8 + 2 * c;
      if (r0 < R) {
        const int t = r0 / G, gg = r0 % G;
        *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t) * p.Hq + hk * G + gg) * D + d) =
            __floats2bfloat162_rn(oacc[n][0] * inv0, oacc[n][1] * inv0);
      }
      if (r1 < R) {
        const int t = r1 / G, gg = r1 % G;
        *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t) * p.Hq + hk * G + gg) * D + d) =
            __floats2bfloat162_rn(oacc[n][2] * inv1, oacc[n][3] * inv1);
      }
    }
  }
  cbar();  // the ring / sQ are reused by the next unit
}

__device__ void argmax_row(const Params& p, const Op& o, int r, const Smem& sm) {
  const int ct = threadIdx.x - 64, lane = threadIdx.x & 31, cw = ct >> 5;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int t = ct; t < o.tiles; t += kCompute) {
    const float2 c = __ldcg(p.argpart + (size_t)t * o.M + r);
    const int ci = __float_as_int(c.y);
    if (c.x > bv || (c.x == bv && ci < bi)) { bv = c.x; bi = ci; }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) sm.argx[cw] = make_float2(bv, __int_as_float(bi));
  cbar();
  if (ct == 0) {
    float2 best = sm.argx[0];
    for (int w = 1; w < 4; ++w) {
      const float2 c = sm.argx[w];
      if (c.x > best.x || (c.x == best.x && __float_as_int(c.y) < __float_as_int(best.y))) best = c;
    }
    const int dst = field(p, o.set, F_SCATTER)[r];
    if (dst >= 0) p.slot_tok[dst] = __float_as_int(best.y);
  }
  cbar();
}

__device__ void compute_warps(const Params& p, uint64_t* tfull, uint64_t* tempty, uint32_t tmem,
                              const Smem& sm) {
  const int c = blockIdx.x;
  const int ct = threadIdx.x - 64;
  int j = 0;  // GEMM units seen (TMEM slot)
  unsigned long long* tr = p.trace ? p.trace + (size_t)c * p.n_ops * 3 : nullptr;
  for (int oi = 0; oi < p.n_ops; ++oi) {
    const Op& o = p.ops[oi];
    int mine = 0;
    if (tr && ct == 0) tr[oi * 3] = tr[oi * 3 + 1] = gtimer();
    if (o.type == OP_GEMM) {
      for (int u = first_unit(o, c, p.G); u < o.units; u += p.G) {
        const Unit un = gemm_unit(o, u);
        if (un.kb1 > un.kb0) {
          const int a = j & 1;
          mbar_wait(tfull + a, (j >> 1) & 1);
          tc_fence_after();
          if (tr && ct == 0 && mine == 0) tr[oi * 3 + 1] = gtimer();
          epilogue(p, o, un, tmem + a * BN, sm);
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive(tempty + a);
          ++j;
        }
        ++mine;
      }
    } else {
      bool waited = false;
      for (int u = first_unit(o, c, p.G); u < o.units; u += p.G) {
        if (!waited && o.dep >= 0) {
          if (ct == 0) {
            wait_op(p, o.dep);
            if (tr) tr[oi * 3 + 1] = gtimer();
          }
          cbar();
          waited = true;
        }
        switch (o.type) {
          case OP_EMBED_NORM: {
            const int32_t src = field(p, o.set, F_GATHER)[u];
            const int tok = p.slot_tok[src];
            if (ct == 0) field(p, o.set, F_TOKENS)[u] = tok;
            const int tk = tok < 0 ? 0 : tok;
            norm_row(p, p.embed + (size_t)tk * p.H, p.x + (size_t)u * p.H, nullptr, 0, 0, o.w,
                     o.y + (size_t)u * p.H, sm);
            break;
          }
          case OP_ADD_NORM: {
            const int src = o.rows_field >= 0 ? field(p, o.set, o.rows_field)[u] : u;
            const size_t slice = (size_t)o.M * p.H;
            norm_row(p, p.x + (size_t)src * p.H, o.write_back ? p.x + (size_t)src * p.H : nullptr,
                     o.P ? o.P + (size_t)src * p.H : nullptr, o.S, slice, o.w,
                     o.y + (size_t)u * p.H, sm);
            break;
          }
          case OP_ROPE_ATTN:
            if (p.D == 64) rope_attn<64>(p, o, u, sm);
            else rope_attn<32>(p, o, u, sm);
            break;
          case OP_ARGMAX:
            argmax_row(p, o, u, sm);
            break;
        }
        ++mine;
      }
    }
    if (mine) {
      // publish this CTA's units of op oi
      cbar();
      if (ct == 0) {
        fence_proxy_async();
        __threadfence();
        atomicAdd(p.counters + oi, mine);
      }
    }
    if (tr && ct == 0) tr[oi * 3 + 2] = gtimer();
  }
}

__global__ void __launch_bounds__(kThreads, 1) decode_mk_kernel(const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + STAGES * A_BYTES;
  Smem sm;
  sm.sQ = reinterpret_cast<bf16(*)[ATT_P]>(base + SMEM_RING);
  sm.ring = reinterpret_cast<bf16(*)[ATT_P]>(base + SMEM_RING + SMEM_SQ);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ float red[32];
  __shared__ float2 argx[4 * BN];
  __shared__ int bt[ATT_MAX_BLOCKS];
  __shared__ float sc[64];
  __shared__ int s_last;
  sm.red = red;
  sm.argx = argx;
  sm.bt = bt;
  sm.sc = sc;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();  // counters, metadata and caches belong to the predecessor's epoch
  if (warp == 0) {
    if ((threadIdx.x & 31) == 0) producer(p, sA, sB, full, empty);
  } else if (warp == 1) {
    if ((threadIdx.x & 31) == 0) mma_issuer(p, sA, sB, full, empty, tfull, tempty, tmem);
    __syncwarp();
  } else {
    compute_warps(p, tfull, tempty, tmem, sm);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
  // the last CTA out zeroes the op counters for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(p.counters + p.n_ops, 1) == p.G - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    for (int i = threadIdx.x; i <= p.n_ops; i += kThreads) p.counters[i] = 0;
  }
  pdl_trigger();
}

// ---- host side -------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const void* gptr, int rows, int K, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(gptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Program {
  Op* d_ops = nullptr;
  int n_ops = 0;
};

struct Handle {
  psd_mk_model m;
  std::vector<LayerPtrs> layers_h;
  LayerPtrs* d_layers = nullptr;
  CUtensorMap* d_maps = nullptr;
  int n_maps = 0;
  int* d_counters = nullptr;
  int counters_cap = 0;
  int G = 0;
  std::map<long long, Program> programs;
};

int split_count(int tiles, int KB, int G) {
  int S = std::max(1, std::min(G / std::max(tiles, 1), KB / 4));
  const int per = (KB + S - 1) / S;
  return (KB + per - 1) / per;
}

}  // namespace

extern "C" {

size_t psd_mk_smem_bytes(void) { return SMEM_TOTAL; }

void* psd_mk_create(const psd_mk_model* model) {
  if (!model || model->head_dim > ATT_D || (model->head_dim != 64 && model->head_dim != 32) ||
      model->heads / model->kv_heads * 2 > ATT_ROWS || model->hidden > 4096 ||
      model->hidden % 128 || model->vocab % 128 || model->max_blocks > ATT_MAX_BLOCKS)
    return nullptr;
  Handle* h = new Handle();
  h->m = *model;
  const psd_mk_model& m = h->m;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  h->G = m.grid > 0 ? std::min(m.grid, sms) : sms;
  // tensor maps: per layer qkv, o, gu, down; lm head; activations xn, attn, act, xf
  const int L = m.layers;
  std::vector<CUtensorMap> maps(4 * L + 5);
  const int qkv_out = (m.heads + 2 * m.kv_heads) * m.head_dim;
  const int dq = m.heads * m.head_dim;
  bool ok = true;
  h->layers_h.resize(L);
  for (int l = 0; l < L; ++l) {
    const void* const* lp = m.layer_ptrs + 9 * l;
    ok &= make_map(&maps[4 * l + 0], lp[0], qkv_out, m.hidden, BM);
    ok &= make_map(&maps[4 * l + 1], lp[1], m.hidden, dq, BM);
    ok &= make_map(&maps[4 * l + 2], lp[2], 2 * m.ffn, m.hidden, BM);
    ok &= make_map(&maps[4 * l + 3], lp[3], m.hidden, m.ffn, BM);
    h->layers_h[l].bqkv = static_cast<const bf16*>(lp[6]);
    h->layers_h[l].kc = static_cast<bf16*>(const_cast<void*>(lp[7]));
    h->layers_h[l].vc = static_cast<bf16*>(const_cast<void*>(lp[8]));
  }
  ok &= make_map(&maps[4 * L + 0], m.lm_head, m.vocab, m.hidden, BM);
  ok &= make_map(&maps[4 * L + 1], m.xn, m.max_tokens, m.hidden, BN);
  ok &= make_map(&maps[4 * L + 2], m.attn, m.max_tokens, dq, BN);
  ok &= make_map(&maps[4 * L + 3], m.act, m.max_tokens, m.ffn, BN);
  ok &= make_map(&maps[4 * L + 4], m.xf, m.max_tokens, m.hidden, BN);
  if (!ok) {
    delete h;
    return nullptr;
  }
  h->n_maps = (int)maps.size();
  if (cudaMalloc(&h->d_maps, sizeof(CUtensorMap) * maps.size()) != cudaSuccess ||
      cudaMemcpy(h->d_maps, maps.data(), sizeof(CUtensorMap) * maps.size(),
                 cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMalloc(&h->d_layers, sizeof(LayerPtrs) * L) != cudaSuccess ||
      cudaMemcpy(h->d_layers, h->layers_h.data(), sizeof(LayerPtrs) * L,
                 cudaMemcpyHostToDevice) != cudaSuccess) {
    delete h;
    return nullptr;
  }
  // op counters for the deepest program (PSD_MAX_K steps), allocated once so
  // captured graphs never see them move
  h->counters_cap = PSD_MAX_K * (7 * L + 4) + 2;
  if (cudaMalloc(&h->d_counters, sizeof(int) * h->counters_cap) != cudaSuccess ||
      cudaMemset(h->d_counters, 0, sizeof(int) * h->counters_cap) != cudaSuccess) {
    delete h;
    return nullptr;
  }
  cudaFuncSetAttribute(decode_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
  cudaDeviceSynchronize();
  return h;
}

void psd_mk_destroy(void* handle) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return;
  cudaFree(h->d_maps);
  cudaFree(h->d_layers);
  cudaFree(h->d_counters);
  for (auto& kv : h->programs) cudaFree(kv.second.d_ops);
  delete h;
}

int psd_mk_grid(void* handle) { return handle ? static_cast<Handle*>(handle)->G : 0; }

// k greedy draft steps over nb sequences: step 0 carries 2 tokens per sequence
// (the last two committed tokens), steps 1.. one; metadata set i describes step i
int psd_mk_launch(void* handle, int nb, int steps, void* stream) {
  return psd_mk_launch_traced(handle, nb, steps, nullptr, stream);
}

int psd_mk_n_ops(void* handle, int nb, int steps) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h) return -1;
  auto it = h->programs.find((long long)nb * 1024 + steps);
  return it == h->programs.end() ? -1 : it->second.n_ops;
}

int psd_mk_launch_traced(void* handle, int nb, int steps, void* trace, void* stream) {
  Handle* h = static_cast<Handle*>(handle);
  if (!h || nb <= 0 || 2 * nb > BN || steps <= 0 || steps > PSD_MAX_K)
    return (int)cudaErrorInvalidValue;
  const psd_mk_model& m = h->m;
  const long long key = (long long)nb * 1024 + steps;
  auto it = h->programs.find(key);
  if (it == h->programs.end()) {
    std::vector<Op> ops;
    const int G = h->G;
    const int L = m.layers;
    const int qkv_out = (m.heads + 2 * m.kv_heads) * m.head_dim;
    const int dq = m.heads * m.head_dim;
    int rot = 0;  // rotate first CTAs so small ops spread over the grid
    auto push = [&](Op o) {
      o.first = rot;
      rot = (rot + o.units) % G;
      ops.push_back(o);
      return (int)ops.size() - 1;
    };
    auto gemm = [&](int tmw, int tmx, int epi, int M, int N, int K, int dep, void* out,
                    bool split, int set) {
      Op o = {};
      o.type = OP_GEMM;
      o.tmw = tmw; o.tmx = tmx; o.epi = epi; o.M = M; o.N = N;
      o.KB = (K + BK - 1) / BK;
      o.tiles = N / BM;
      const int S = split ? split_count(o.tiles, o.KB, G) : 1;
      o.kb_per_unit = (o.KB + S - 1) / S;
      o.S = (o.KB + o.kb_per_unit - 1) / o.kb_per_unit;
      o.units = o.tiles * o.S;
      o.dep = dep;
      o.out = out;
      o.set = set;
      return o;
    };
    int last = -1;
    for (int st = 0; st < steps; ++st) {
      const int M = st == 0 ? 2 * nb : nb;
      // embedding + attention norm of layer 0
      Op e = {};
      e.type = OP_EMBED_NORM;
      e.units = M;
      e.dep = last;
      e.w = static_cast<const bf16*>(m.layer_ptrs[4]);
      e.y = static_cast<bf16*>(m.xn);
      e.set = st;
      e.rows_field = -1;
      last = push(e);
      for (int l = 0; l < L; ++l) {
        const void* const* lp = m.layer_ptrs + 9 * l;
        Op g1 = gemm(4 * l + 0, 4 * L + 1, E_PART, M, qkv_out, m.hidden, last, m.part, true, st);
        const int iq = push(g1);
        Op ra = {};
        ra.type = OP_ROPE_ATTN;
        ra.units = nb * m.kv_heads;
        ra.dep = iq;
        ra.P = m.part;
        ra.S = g1.S;
        ra.M = M;
        ra.out = m.attn;
        ra.set = st;
        ra.layer = l;
        const int ia = push(ra);
        Op g2 = gemm(4 * l + 1, 4 * L + 2, E_PART, M, m.hidden, dq, ia, m.part, true, st);
        const int io = push(g2);
        Op n2 = {};
        n2.type = OP_ADD_NORM;
        n2.units = M;
        n2.dep = io;
        n2.P = m.part;
        n2.S = g2.S;
        n2.M = M;
        n2.write_back = 1;
        n2.w = static_cast<const bf16*>(lp[5]);
        n2.y = static_cast<bf16*>(m.xn);
        n2.rows_field = -1;
        n2.set = st;
        const int in2 = push(n2);
        Op g3 = gemm(4 * l + 2, 4 * L + 1, E_SILU, M, 2 * m.ffn, m.hidden, in2, m.act, false, st);
        const int ig = push(g3);
        Op g4 = gemm(4 * l + 3, 4 * L + 3, E_PART, M, m.hidden, m.ffn, ig, m.part, true, st);
        const int id = push(g4);
        Op n3 = {};
        n3.type = OP_ADD_NORM;
        n3.dep = id;
        n3.P = m.part;
        n3.S = g4.S;
        n3.M = M;
        n3.set = st;
        if (l + 1 < L) {
          n3.units = M;
          n3.write_back = 1;
          n3.w = static_cast<const bf16*>(m.layer_ptrs[9 * (l + 1) + 4]);
          n3.y = static_cast<bf16*>(m.xn);
          n3.rows_field = -1;
        } else {  // final norm of the logit rows
          n3.units = nb;
          n3.write_back = 0;
          n3.w = static_cast<const bf16*>(m.final_norm);
          n3.y = static_cast<bf16*>(m.xf);
          n3.rows_field = F_LOGIT_ROWS;
        }
        last = push(n3);
      }
      Op lm = gemm(4 * L + 0, 4 * L + 4, E_ARG, nb, m.vocab, m.hidden, last, nullptr, false, st);
      const int il = push(lm);
      Op am = {};
      am.type = OP_ARGMAX;
      am.units = nb;
      am.dep = il;
      am.M = nb;
      am.tiles = m.vocab / BM;
      am.set = st;
      last = push(am);
    }
    Program pr;
    pr.n_ops = (int)ops.size();
    if (cudaMalloc(&pr.d_ops, sizeof(Op) * ops.size()) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
    if (cudaMemcpy(pr.d_ops, ops.data(), sizeof(Op) * ops.size(), cudaMemcpyHostToDevice) !=
        cudaSuccess)
      return (int)cudaErrorUnknown;
    if (pr.n_ops + 1 > h->counters_cap) {
      cudaFree(pr.d_ops);
      return (int)cudaErrorInvalidValue;
    }
    it = h->programs.emplace(key, pr).first;
  }
  Params p = {};
  p.ops = it->second.d_ops;
  p.n_ops = it->second.n_ops;
  p.maps = h->d_maps;
  p.counters = h->d_counters;
  p.G = h->G;
  p.H = m.hidden; p.Hq = m.heads; p.Hkv = m.kv_heads; p.D = m.head_dim; p.V = m.vocab;
  p.nseq = nb;
  p.eps = m.eps;
  p.scale_log2 = m.attn_scale * 1.44269504088896341f;
  p.beta = m.beta;
  p.bs = m.block_size;
  p.max_blocks = m.max_blocks;
  p.block_table = m.block_table;
  p.inv_freq = m.inv_freq;
  p.embed = static_cast<const bf16*>(m.embed);
  p.succ = m.successor;
  p.x = static_cast<bf16*>(m.x);
  p.argpart = static_cast<float2*>(m.argpart);
  p.slot_tok = m.slot_tok;
  p.meta = m.meta;
  p.set_stride = m.set_stride;
  for (int f = 0; f < F_COUNT; ++f) p.off[f] = m.field_offsets[f];
  p.layers = h->d_layers;
  p.trace = static_cast<unsigned long long*>(trace);

  return (int)psd::launch(decode_mk_kernel, dim3(h->G), dim3(kThreads), SMEM_TOTAL,
                          (cudaStream_t)stream, p);
}

}  // extern "C"
