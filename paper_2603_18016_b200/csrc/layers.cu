// layers.cu -- the non-GEMM kernels of the draft / target forwards (K3, K3',
// K4) and the small device-side glue of the PSD step (K5, K6 helpers).
//
// Replaces the virtual pass durations of the reference (verify_latency /
// draft_latency .duration, pkg/src/specsim/engine.py:338, 359-360, 378, 402,
// 429) together with gemm.cu.  All of these are HBM / latency bound and run
// on CUDA cores with 128-bit accesses; none is GEMM-shaped enough to pay for
// tensor-core staging at the BASELINE shapes (<= 64 query rows per KV head).
#include <cstdlib>
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/psd.h"
#include "common.h"
#include "sm100.cuh"

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- embedding gather -------------------------------------------------------
__global__ void embed_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ E,
                             __nv_bfloat16* __restrict__ out, int H) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int t = tok[m];
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)(t < 0 ? 0 : t) * H);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)m * H);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x)
    dst[i] = t < 0 ? make_uint4(0, 0, 0, 0) : src[i];
}

// ---- residual add of split-K partials + RMSNorm (fp32 statistics) ---------------
// v = bf16(x[src] + sum_s P[s][src]) (sum in s order; skipped when P == null),
// optionally written back to x (the residual stream), y[m] = v * rsqrt(mean(v^2)
// + eps) * w.  src = rows ? rows[m] : m.  The GEMMs before a norm (O proj, down
// proj) leave fp32 split-K partials, so this one kernel is their reduction,
// the residual add and the norm.
constexpr int NORM_THREADS = 256;
constexpr int NORM_MAX_PER_THREAD = 32;  // H <= 8192

// v[0..7] = sum over z < S of P[z * slice + off + 0..7], summed in z order.
// Loads go out four splits at a time (independent 32-byte loads) instead of
// one dependent L2 round trip per split; the additions keep the z order.
__device__ __forceinline__ void sum_partials8(const float* __restrict__ P, size_t slice, int S,
                                              size_t off, float (&v)[8]) {
  const float4* p4 = reinterpret_cast<const float4*>(P + off);
  float4 a = p4[0], b = p4[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  int z = 1;
#pragma unroll 1
  for (; z + 4 <= S; z += 4) {
    float4 c[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4* q4 = reinterpret_cast<const float4*>(P + (size_t)(z + u) * slice + off);
      c[u][0] = q4[0];
      c[u][1] = q4[1];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[0] += c[u][0].x; v[1] += c[u][0].y; v[2] += c[u][0].z; v[3] += c[u][0].w;
      v[4] += c[u][1].x; v[5] += c[u][1].y; v[6] += c[u][1].z; v[7] += c[u][1].w;
    }
  }
  for (; z < S; ++z) {
    const float4* q4 = reinterpret_cast<const float4*>(P + (size_t)z * slice + off);
    a = q4[0];
    b = q4[1];
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
    v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
  }
}

// all S <= 16 partials of one 8-wide chunk requested at once (one L2 round
// trip), then summed in z order -- same arithmetic as sum_partials8
__device__ __forceinline__ void sum_partials8_all(const float* __restrict__ P, size_t slice, int S,
                                                  size_t off, float (&v)[8]) {
  float4 c[16][2];
#pragma unroll
  for (int z = 0; z < 16; ++z)
    if (z < S) {
      const float4* q4 = reinterpret_cast<const float4*>(P + (size_t)z * slice + off);
      c[z][0] = q4[0];
      c[z][1] = q4[1];
    }
  v[0] = c[0][0].x; v[1] = c[0][0].y; v[2] = c[0][0].z; v[3] = c[0][0].w;
  v[4] = c[0][1].x; v[5] = c[0][1].y; v[6] = c[0][1].z; v[7] = c[0][1].w;
#pragma unroll
  for (int z = 1; z < 16; ++z)
    if (z < S) {
      v[0] += c[z][0].x; v[1] += c[z][0].y; v[2] += c[z][0].z; v[3] += c[z][0].w;
      v[4] += c[z][1].x; v[5] += c[z][1].y; v[6] += c[z][1].z; v[7] += c[z][1].w;
    }
}

template <int NV>  // NV = 8-wide chunks per thread (H / 8 / NORM_THREADS rounded up)
__global__ void __launch_bounds__(NORM_THREADS)
add_rmsnorm_kernel(__nv_bfloat16* __restrict__ x, int ldx, const float* __restrict__ P, int S,
                   size_t slice, int ldp, const int32_t* __restrict__ rows,
                   const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ y, int ldy,
                   int H, float eps, int write_back) {
  // the norm weights and the row map do not depend on the predecessor:
  // fetched before griddepcontrol.wait
  const int m = blockIdx.x;
  const int src = rows ? rows[m] : m;
  uint4 wv[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int e = (threadIdx.x + k * NORM_THREADS) * 8;
    if (e < H) wv[k] = *reinterpret_cast<const uint4*>(w + e);
  }
  pdl_wait();
  pdl_trigger();
  __nv_bfloat16* xr = x + (size_t)src * ldx;
  const float* pr = P ? P + (size_t)src * ldp : nullptr;
  float v[NV][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int e = (threadIdx.x + k * NORM_THREADS) * 8;
    if (e < H) {
      uint4 u = *reinterpret_cast<const uint4*>(xr + e);
      const __nv_bfloat16* b8 = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[k][t] = __bfloat162float(b8[t]);
      if (pr) {
        float acc[8];
        if (NV == 1 && S <= 16) sum_partials8_all(pr, slice, S, e, acc);
        else sum_partials8(pr, slice, S, e, acc);
        uint4 o;
        __nv_bfloat16* o8 = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          o8[t] = __float2bfloat16(acc[t] + v[k][t]);
          v[k][t] = __bfloat162float(o8[t]);
        }
        if (write_back) *reinterpret_cast<uint4*>(xr + e) = o;
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) ss += v[k][t] * v[k][t];
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (NORM_THREADS >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / H + eps);
  __nv_bfloat16* yr = y + (size_t)m * ldy;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int e = (threadIdx.x + k * NORM_THREADS) * 8;
    if (e < H) {
      const __nv_bfloat16* w8 = reinterpret_cast<const __nv_bfloat16*>(&wv[k]);
      uint4 o;
      __nv_bfloat16* o8 = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
      for (int t = 0; t < 8; ++t) o8[t] = __float2bfloat16(v[k][t] * inv * __bfloat162float(w8[t]));
      *reinterpret_cast<uint4*>(yr + e) = o;
    }
  }
}

// ---- RoPE + paged KV write ------------------------------------------------------
// qkv [M, (Hq + 2 Hkv) D]; q_out [M, Hq, D]; caches [blocks, bs, Hkv, D].
// rotate-half convention: pairs (i, i + D/2), angle = pos * inv_freq[i].
// One CTA per token.  Work item = (head, 8-wide chunk of the first half):
// one 16-byte load of x[i..i+7] and one of x[i+half..], 8 rotations, 16-byte
// stores -- every load of a thread is independent (no serial latency chain).
// 8 consecutive qkv values of token-row `row` starting at column e: bf16 input,
// or bf16(sum of S fp32 split-K partials) -- the QKV GEMM's reduction fused here
struct QkvSrc {
  const __nv_bfloat16* bf;
  const float* P;
  int S;
  size_t slice;
  __device__ __forceinline__ void load8(size_t off, float (&v)[8]) const {
    if (P) {
      sum_partials8(P, slice, S, off, v);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __bfloat162float(__float2bfloat16(v[k]));
    } else {
      uint4 u = *reinterpret_cast<const uint4*>(bf + off);
      const __nv_bfloat16* h8 = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __bfloat162float(h8[k]);
    }
  }
};

__global__ void __launch_bounds__(256)
rope_kv_kernel(const QkvSrc src, int Hq, int Hkv, int D,
               const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
               const float* __restrict__ inv_freq, const __nv_bfloat16* __restrict__ bias,
               __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kc,
               __nv_bfloat16* __restrict__ vc) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x;
  const int p = pos[m];
  const int s = slot[m];
  const int half = D / 2;
  const int cpr = half / 8;  // 8-wide chunks per half row
  __shared__ float s_cos[128], s_sin[128];
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    float sn, cs;
    sincosf((float)p * inv_freq[i], &sn, &cs);
    s_cos[i] = cs;
    s_sin[i] = sn;
  }
  __syncthreads();
  const size_t row = (size_t)m * (Hq + 2 * Hkv) * D;
  const int nrot = (s >= 0 ? Hq + Hkv : Hq) * cpr;
  const int nv = s >= 0 ? Hkv * D / 8 : 0;
  for (int idx = threadIdx.x; idx < nrot + nv; idx += blockDim.x) {
    if (idx >= nrot) {  // V: copy (+ bias)
      const int e = (idx - nrot) * 8;
      float vf[8];
      src.load8(row + (size_t)(Hq + Hkv) * D + e, vf);
      uint4 v;
      __nv_bfloat16* vv = reinterpret_cast<__nv_bfloat16*>(&v);
      const __nv_bfloat16* bb = bias ? bias + (size_t)(Hq + Hkv) * D + e : nullptr;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        vv[k] = __float2bfloat16(bb ? vf[k] + __bfloat162float(bb[k]) : vf[k]);
      *reinterpret_cast<uint4*>(vc + (size_t)s * Hkv * D + e) = v;
      continue;
    }
    const int h = idx / cpr, i0 = (idx % cpr) * 8;
    float a8[8], b8[8];
    src.load8(row + h * D + i0, a8);
    src.load8(row + h * D + i0 + half, b8);
    uint4 ra, rb;
    __nv_bfloat16* ra8 = reinterpret_cast<__nv_bfloat16*>(&ra);
    __nv_bfloat16* rb8 = reinterpret_cast<__nv_bfloat16*>(&rb);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float a = a8[k], b = b8[k];
      if (bias) {  // qkv bias (Qwen2), rounded to bf16 like the projection output
        a = __bfloat162float(__float2bfloat16(a + __bfloat162float(bias[h * D + i0 + k])));
        b = __bfloat162float(__float2bfloat16(b + __bfloat162float(bias[h * D + i0 + k + half])));
      }
      const float cs = s_cos[i0 + k], sn = s_sin[i0 + k];
      ra8[k] = __float2bfloat16(a * cs - b * sn);
      rb8[k] = __float2bfloat16(b * cs + a * sn);
    }
    __nv_bfloat16* dst = h < Hq ? q_out + ((size_t)m * Hq + h) * D
                                : kc + ((size_t)s * Hkv + (h - Hq)) * D;
    *reinterpret_cast<uint4*>(dst + i0) = ra;
    *reinterpret_cast<uint4*>(dst + i0 + half) = rb;
  }
}

// ---- paged multi-query attention (causal within the query window, GQA) ---------
// One CTA (4 warps) per (sequence, kv head, query chunk).  Query rows of the
// chunk = its tokens x the G = Hq / Hkv heads sharing this kv head (<= 64
// rows; warp w owns rows 16w..16w+15).  Keys stream through shared memory in
// tiles of 64 (cp.async, double buffered, zero-filled past the last key);
// S = Q K^T and O += P V run on tensor cores (mma.sync m16n8k16 bf16 -> fp32),
// softmax is online in fp32 registers (FlashAttention-2 register layout).
constexpr int ATT_THREADS = 128;
constexpr int ATT_MAXR = 64;   // query rows per CTA
constexpr int ATT_STAGES = 2;  // tile groups in flight (each group = one tile per key group)
constexpr int ATT_MAX_BLOCKS = 512;  // block-table entries staged in smem (8192 tokens)

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4],
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Warp roles: RG = ceil(rows / 16) row groups x KG = 4 / RG key groups.  Warp
// (rg, kg) owns query rows 16rg..16rg+15 and every KG-th key tile; tiles are
// streamed in groups of KG (one per key group) through an NS-stage cp.async
// ring, so a decode step (4-8 rows) keeps all 4 warps busy on 4 tiles at a
// time.  The key groups' (max, sum, O) states are merged through shared
// memory at the end (same math as split-KV flash decoding, no global traffic).
// Fused RoPE (decode / verify passes, one query chunk per sequence): the CTA of
// (sequence, kv head) reduces the QKV split-K partials of its G query heads and
// its K / V head for the sequence's tokens, rotates Q and K, writes this step's
// K / V rows into the paged cache and Q straight into shared memory -- no
// separate RoPE launch and no Q round trip through HBM.
__device__ __forceinline__ void vc_w(const __nv_bfloat16* vc, size_t off, float a) {
  const_cast<__nv_bfloat16*>(vc)[off] = __float2bfloat16(a);
}

struct RopeSrc {
  const float* P;  // QKV split-K partials [S][M][(Hq + 2 Hkv) D]
  int S;
  size_t slice;
  const int32_t* positions;
  const int32_t* slots;
  const float* inv_freq;
  const __nv_bfloat16* bias;  // qkv bias or null
};

__device__ __forceinline__ float sum_parts(const RopeSrc& rs, size_t off) {
  float v[16];
#pragma unroll
  for (int z = 0; z < 16; ++z) v[z] = z < rs.S ? __ldcg(rs.P + z * rs.slice + off) : 0.f;
  float a = v[0];
#pragma unroll
  for (int z = 1; z < 16; ++z)
    if (z < rs.S) a += v[z];
  return __bfloat162float(__float2bfloat16(a));  // the projection output is bf16
}

template <int D, int KT, int NS, bool ROPE>
__global__ void __launch_bounds__(ATT_THREADS)
attention_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                 const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ block_table,
                 int max_blocks, const int32_t* __restrict__ seq_slot,
                 const int32_t* __restrict__ q_start, const int32_t* __restrict__ q_len,
                 const int32_t* __restrict__ q_pos0, const int32_t* __restrict__ kv_len, int Hq,
                 int Hkv, int bs, float scale_log2, int tok_per_chunk, int RG, int S,
                 float* __restrict__ ws, int* __restrict__ tickets,
                 __nv_bfloat16* __restrict__ out, const RopeSrc rs) {
  // PDL: metadata, the block table and the keys of earlier steps (positions <
  // q_pos0) do not depend on the predecessor (RoPE writes this step's keys and
  // the queries), so they are fetched before griddepcontrol.wait
  constexpr int P = D + 8;  // smem row pitch (conflict-free fragment loads)
  const int KG = 4 / RG;
  const int seq = blockIdx.x, hk = blockIdx.y, chunk = blockIdx.z / S, split = blockIdx.z % S;
  const int G = Hq / Hkv;
  const int ql = q_len[seq];
  const int t0 = chunk * tok_per_chunk;
  if (t0 >= ql) return;
  const int nt = min(tok_per_chunk, ql - t0);
  const int R = nt * G;
  const int kvl = kv_len[seq];
  const int qs = q_start[seq];
  const int first_pos = q_pos0[seq];
  const int last_key = min(first_pos + t0 + nt - 1, kvl - 1);
  const int* btg = block_table + (size_t)seq_slot[seq] * max_blocks;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int rg = warp % RG, kg = warp / RG;
  __shared__ int bt[ATT_MAX_BLOCKS];
  const int nblk_used = min((last_key >> (__ffs(bs) - 1)) + 1, ATT_MAX_BLOCKS);
  for (int i = tid; i < nblk_used; i += ATT_THREADS) bt[i] = btg[i];

  extern __shared__ __align__(16) uint8_t att_smem[];
  typedef __nv_bfloat16 Row[P];
  Row* sQ = reinterpret_cast<Row*>(att_smem);
  Row* ring = reinterpret_cast<Row*>(att_smem + sizeof(Row) * RG * 16);  // sQ: RG x 16 rows
  // stage s, key group j: K rows at ring[((s*KG + j)*2) * KT], V rows right after
  auto sK = [&](int st, int j) { return ring + ((st * KG + j) * 2) * KT; };
  auto sV = [&](int st, int j) { return ring + ((st * KG + j) * 2 + 1) * KT; };

  const int ntiles_all = last_key / KT + 1;
  // this split's key tiles [ta, tb)
  const int ta = split * ntiles_all / S, tb = (split + 1) * ntiles_all / S;
  const int ntiles = tb - ta;
  const int ngroups = (ntiles + KG - 1) / KG;
  __syncthreads();  // bt staged
  // part: 0 = every row of the group, 1 = rows of earlier steps' keys only,
  // 2 = the complement of 1 (this step's keys and the zero fill past the end)
  // every thread copies the same (row, 16-byte chunk) positions of each tile:
  // KT * D / 8 chunks per tile over 128 threads (a whole multiple for D >= 32),
  // so the index math is hoisted and the block-table lookup is a shift / mask
  // (block_size is a power of two)
  constexpr int CPR = D / 8;                       // 16-byte chunks per row
  constexpr int PER_T = KT * CPR / ATT_THREADS;    // chunks per thread per tile
  static_assert(KT * CPR % ATT_THREADS == 0, "tile chunks must tile the CTA");
  const int bs_shift = __ffs(bs) - 1;
  // per-thread constants of its PER_T chunk positions (row r, chunk cc):
  // element offset inside a cache block, block step, shared-memory offset --
  // per tile only the block-table entry and one wide multiply-add remain
  uint32_t c_off[PER_T], c_soff[PER_T];
  int c_row[PER_T], c_blk[PER_T];
#pragma unroll
  for (int i = 0; i < PER_T; ++i) {
    const int idx = tid + ATT_THREADS * i;
    const int r = idx / CPR, cc = idx % CPR;  // compile-time divisors
    c_row[i] = r;
    c_blk[i] = r >> bs_shift;
    c_off[i] = (uint32_t)(((r & (bs - 1)) * Hkv + hk) * D + cc * 8);
    c_soff[i] = (uint32_t)(r * P + cc * 8) * 2u;
  }
  const uint32_t blk_elems = (uint32_t)(bs * Hkv * D);
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  auto load_group = [&](int gi, int st, int part) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j >= KG) break;
      const int tile = ta + gi * KG + j;
      const uint32_t sk = ring_s + (uint32_t)(((st * KG + j) * 2) * KT * P * 2);
      const uint32_t sv = sk + (uint32_t)(KT * P * 2);
      const int blk0 = (tile * KT) >> bs_shift;
#pragma unroll
      for (int i = 0; i < PER_T; ++i) {
        const int key = tile * KT + c_row[i];
        const bool ok = key <= last_key && tile < tb;
        const bool old = ok && key < first_pos;
        if ((part == 1 && !old) || (part == 2 && old)) continue;
        const uint64_t o = ok ? (uint64_t)(uint32_t)bt[blk0 + c_blk[i]] * blk_elems + c_off[i] : 0ull;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sk + c_soff[i]),
                     "l"(kc + o), "r"(ok ? 16 : 0));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sv + c_soff[i]),
                     "l"(vc + o), "r"(ok ? 16 : 0));
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < NS - 1; ++t) {
    if (t < ngroups) load_group(t, t, 1);
    else cp_async_commit();
  }
  pdl_wait();
  pdl_trigger();
  if constexpr (ROPE) {
    // rotate-half RoPE of (token t, head h, pair i): G query heads + the K head,
    // then the V head copied; bf16 rounding points as in rope_kv_kernel
    constexpr int half = D / 2;
    const int NQKV = (Hq + 2 * Hkv) * D;
    const int nrot = nt * (G + 1) * half;
    for (int idx = tid; idx < nrot + nt * D; idx += ATT_THREADS) {
      if (idx >= nrot) {
        const int t = (idx - nrot) / D, i = (idx - nrot) % D;
        const int m = qs + t0 + t;
        const int sl = rs.slots[m];
        if (sl < 0) continue;
        const int col = (Hq + Hkv + hk) * D + i;
        float a = sum_parts(rs, (size_t)m * NQKV + col);
        if (rs.bias) a = a + __bfloat162float(rs.bias[col]);
        vc_w(vc, ((size_t)sl * Hkv + hk) * D + i, a);
        continue;
      }
      const int t = idx / ((G + 1) * half), rem = idx % ((G + 1) * half);
      const int hh = rem / half, i = rem % half;
      const int m = qs + t0 + t;
      const int head = hh < G ? hk * G + hh : Hq + hk;
      const int col = head * D + i;
      float a = sum_parts(rs, (size_t)m * NQKV + col);
      float b = sum_parts(rs, (size_t)m * NQKV + col + half);
      if (rs.bias) {
        a = __bfloat162float(__float2bfloat16(a + __bfloat162float(rs.bias[col])));
        b = __bfloat162float(__float2bfloat16(b + __bfloat162float(rs.bias[col + half])));
      }
      float sn, cs;
      sincosf((float)rs.positions[m] * rs.inv_freq[i], &sn, &cs);
      const __nv_bfloat16 ra = __float2bfloat16(a * cs - b * sn);
      const __nv_bfloat16 rb = __float2bfloat16(b * cs + a * sn);
      if (hh < G) {
        sQ[t * G + hh][i] = ra;
        sQ[t * G + hh][i + half] = rb;
      } else {
        const int sl = rs.slots[m];
        if (sl >= 0) {
          __nv_bfloat16* dst = const_cast<__nv_bfloat16*>(kc) + ((size_t)sl * Hkv + hk) * D;
          dst[i] = ra;
          dst[i + half] = rb;
        }
      }
    }
    for (int idx = tid; idx < (RG * 16 - R) * D; idx += ATT_THREADS)
      sQ[R + idx / D][idx % D] = __float2bfloat16(0.f);
    __threadfence();  // this step's K / V rows are read back below through L2
    __syncthreads();
  } else {
    for (int idx = tid; idx < RG * 16 * (D / 8); idx += ATT_THREADS) {
      const int r = idx / (D / 8), cc = idx % (D / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < R) {
        const int t = r / G, gg = r % G;
        v = *reinterpret_cast<const uint4*>(q + ((size_t)(qs + t0 + t) * Hq + hk * G + gg) * D +
                                            cc * 8);
      }
      *reinterpret_cast<uint4*>(&sQ[r][cc * 8]) = v;
    }
  }
  // this step's keys of the prefetched groups (one extra commit group; the
  // first iteration waits for everything)
#pragma unroll
  for (int t = 0; t < NS - 1; ++t)
    if (t < ngroups) load_group(t, t, 2);
  cp_async_commit();
  __syncthreads();

  const bool active = kg < KG && rg * 16 < R;
  const int r0 = rg * 16 + g, r1 = r0 + 8;
  const int lim0 = r0 < R ? min(first_pos + t0 + r0 / G, kvl - 1) : -1;
  const int lim1 = r1 < R ? min(first_pos + t0 + r1 / G, kvl - 1) : -1;
  uint32_t qf[D / 16][4];
  if (active) {
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qf[kk][0] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 2 * c]);
      qf[kk][1] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 2 * c]);
      qf[kk][2] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 8 + 2 * c]);
      qf[kk][3] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 8 + 2 * c]);
    }
  }
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int gi = 0; gi < ngroups; ++gi) {
    const int st = gi % NS;
    if (gi + NS - 1 < ngroups) load_group(gi + NS - 1, (gi + NS - 1) % NS, 0);
    else cp_async_commit();
    if (gi == 0) cp_async_wait<1>();  // prologue groups (both parts) landed
    else cp_async_wait<NS - 1>();
    __syncthreads();
    const int kt = ta + gi * KG + kg;
    if (active && kt < tb) {
      Row* K = sK(st, kg);
      Row* V = sV(st, kg);
      float sacc[KT / 8][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
      // K fragments with ldmatrix.x4: matrices (keys 8n.., dims 16kk..), (.., 16kk+8..),
      // (keys 8n+8.., 16kk..), (.., 16kk+8..) -> b0/b1 of key blocks n and n+1
      const int lrow = lane & 7, lmat = lane >> 3;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < KT / 8; n += 2) {
          uint32_t kb[4];
          ldmatrix_x4(kb, &K[(n + (lmat >> 1)) * 8 + lrow][kk * 16 + (lmat & 1) * 8]);
          mma_bf16_16816(sacc[n], qf[kk], kb[0], kb[1]);
          mma_bf16_16816(sacc[n + 1], qf[kk], kb[2], kb[3]);
        }
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const int key = kt * KT + n * 8 + 2 * c;
        sacc[n][0] = key <= lim0 ? sacc[n][0] * scale_log2 : -INFINITY;
        sacc[n][1] = key + 1 <= lim0 ? sacc[n][1] * scale_log2 : -INFINITY;
        sacc[n][2] = key <= lim1 ? sacc[n][2] * scale_log2 : -INFINITY;
        sacc[n][3] = key + 1 <= lim1 ? sacc[n][3] * scale_log2 : -INFINITY;
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
      uint32_t pf[KT / 16][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const float p0 = exp2f(sacc[n][0] - base0), p1 = exp2f(sacc[n][1] - base0);
        const float p2 = exp2f(sacc[n][2] - base1), p3 = exp2f(sacc[n][3] - base1);
        ps0 += p0 + p1;
        ps1 += p2 + p3;
        const int kk = n >> 1;
        if ((n & 1) == 0) {
          pf[kk][0] = pack_bf16(p0, p1);
          pf[kk][1] = pack_bf16(p2, p3);
        } else {
          pf[kk][2] = pack_bf16(p0, p1);
          pf[kk][3] = pack_bf16(p2, p3);
        }
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= al0; o[n][1] *= al0; o[n][2] *= al1; o[n][3] *= al1;
      }
#pragma unroll
      for (int kk = 0; kk < KT / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < D / 8; n += 2) {
          uint32_t vb[4];
          const int mat = lane >> 3, rr = lane & 7;
          const int krow = kk * 16 + (mat & 1) * 8 + rr;
          const int dcol = (n + (mat >> 1)) * 8;
          ldmatrix_x4_trans(vb, &V[krow][dcol]);
          mma_bf16_16816(o[n], pf[kk], vb[0], vb[1]);
          mma_bf16_16816(o[n + 1], pf[kk], vb[2], vb[3]);
        }
      }
    }
    __syncthreads();
  }
  // the 4 threads of a row quad hold disjoint key columns: reduce l
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (KG > 1) {
    // merge key-group states: warp (rg, kg>0) publishes, warp (rg, 0) merges
    cp_async_wait<0>();
    __syncthreads();
    float* scr = reinterpret_cast<float*>(ring);  // ring is free now
    const int slot_floats = 16 * D + 32;          // o[16][D], m[16], l[16]
    if (active && kg > 0) {
      float* sp = scr + (rg * KG + kg) * slot_floats;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int d = n * 8 + 2 * c;
        sp[g * D + d] = o[n][0];
        sp[g * D + d + 1] = o[n][1];
        sp[(g + 8) * D + d] = o[n][2];
        sp[(g + 8) * D + d + 1] = o[n][3];
      }
      if (c == 0) {
        sp[16 * D + g] = m0;
        sp[16 * D + g + 8] = m1;
        sp[16 * D + 16 + g] = l0;
        sp[16 * D + 16 + g + 8] = l1;
      }
    }
    __syncthreads();
    if (active && kg == 0) {
      float M0 = m0, M1 = m1;
      for (int j = 1; j < KG; ++j) {
        const float* sp = scr + (rg * KG + j) * slot_floats;
        M0 = fmaxf(M0, sp[16 * D + g]);
        M1 = fmaxf(M1, sp[16 * D + g + 8]);
      }
      const float w00 = M0 == -INFINITY ? 0.f : exp2f(m0 - M0);
      const float w10 = M1 == -INFINITY ? 0.f : exp2f(m1 - M1);
      l0 *= w00;
      l1 *= w10;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= w00; o[n][1] *= w00; o[n][2] *= w10; o[n][3] *= w10;
      }
      for (int j = 1; j < KG; ++j) {
        const float* sp = scr + (rg * KG + j) * slot_floats;
        const float mj0 = sp[16 * D + g], mj1 = sp[16 * D + g + 8];
        const float wj0 = mj0 == -INFINITY ? 0.f : exp2f(mj0 - M0);
        const float wj1 = mj1 == -INFINITY ? 0.f : exp2f(mj1 - M1);
        l0 += sp[16 * D + 16 + g] * wj0;
        l1 += sp[16 * D + 16 + g + 8] * wj1;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          const int d = n * 8 + 2 * c;
          o[n][0] += sp[g * D + d] * wj0;
          o[n][1] += sp[g * D + d + 1] * wj0;
          o[n][2] += sp[(g + 8) * D + d] * wj1;
          o[n][3] += sp[(g + 8) * D + d + 1] * wj1;
        }
      }
    }
  }
  if (S > 1) {
    // split-KV: publish this split's (o, m, l) per row; the last split to
    // arrive merges all S in split order (deterministic) and writes the output
    const int unit = (seq * Hkv + hk) * (gridDim.z / S) + chunk;
    const int RW = D + 2;
    float* base = ws + (size_t)unit * S * ATT_MAXR * RW;
    if (active && kg == 0) {
      float* mine = base + (size_t)split * ATT_MAXR * RW;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int d = n * 8 + 2 * c;
        mine[r0 * RW + d] = o[n][0];
        mine[r0 * RW + d + 1] = o[n][1];
        mine[r1 * RW + d] = o[n][2];
        mine[r1 * RW + d + 1] = o[n][3];
      }
      if (c == 0) {
        mine[r0 * RW + D] = m0;
        mine[r0 * RW + D + 1] = l0;
        mine[r1 * RW + D] = m1;
        mine[r1 * RW + D + 1] = l1;
      }
    }
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (tid == 0) s_last = atomicAdd(tickets + unit, 1) == S - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // every split's R rows of (o, m, l), staged in the (now idle) key ring:
    // one wave of independent 8-byte L2 loads instead of a dependent L2
    // chain per output element; same split-order arithmetic either way
    float* sm = reinterpret_cast<float*>(ring);
    const bool staged = S * R * RW * 4 <= 2 * NS * KG * KT * P * 2;
    if (staged) {
      for (int sp = 0; sp < S; ++sp) {
        const float2* src = reinterpret_cast<const float2*>(base + (size_t)sp * ATT_MAXR * RW);
        float2* dst = reinterpret_cast<float2*>(sm + sp * R * RW);
#pragma unroll 4
        for (int i = tid; i < R * RW / 2; i += ATT_THREADS) dst[i] = __ldcg(src + i);
      }
      __syncthreads();
    }
    auto part = [&](int sp, int r) -> const float* {
      return staged ? sm + (sp * R + r) * RW : base + ((size_t)sp * ATT_MAXR + r) * RW;
    };
    for (int idx = tid; idx < R * (D / 2); idx += ATT_THREADS) {
      const int r = idx / (D / 2), d = (idx % (D / 2)) * 2;
      float M = -INFINITY;
      for (int sp = 0; sp < S; ++sp) M = fmaxf(M, staged ? part(sp, r)[D] : __ldcg(part(sp, r) + D));
      float L = 0.f, a0 = 0.f, a1 = 0.f;
      for (int sp = 0; sp < S; ++sp) {
        const float* pr = part(sp, r);
        const float ms = staged ? pr[D] : __ldcg(pr + D);
        const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
        L += (staged ? pr[D + 1] : __ldcg(pr + D + 1)) * w;
        a0 += (staged ? pr[d] : __ldcg(pr + d)) * w;
        a1 += (staged ? pr[d + 1] : __ldcg(pr + d + 1)) * w;
      }
      const float inv = L > 0.f ? 1.f / L : 0.f;
      const int t = r / G, gg = r % G;
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t0 + t) * Hq + hk * G + gg) * D + d) =
          __floats2bfloat162_rn(a0 * inv, a1 * inv);
    }
    if (tid == 0) tickets[unit] = 0;
    return;
  }
  if (!active || kg != 0) return;
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    const int d = n * 8 + 2 * c;
    if (r0 < R) {
      const int t = r0 / G, gg = r0 % G;
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t0 + t) * Hq + hk * G + gg) * D + d) =
          __floats2bfloat162_rn(o[n][0] * inv0, o[n][1] * inv0);
    }
    if (r1 < R) {
      const int t = r1 / G, gg = r1 % G;
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t0 + t) * Hq + hk * G + gg) * D + d) =
          __floats2bfloat162_rn(o[n][2] * inv1, o[n][3] * inv1);
    }
  }
}

// ---- paged attention with TMA key / value tiles ------------------------------
// Verify and prefill passes (no fused RoPE), D in {64, 128}, 16-token blocks.
// The cp.async form issues one 16-byte copy per thread per key-row chunk:
// ncu showed the verify kernel issue-bound on that copy + address stream
// (profiles/r02_attn_tma.txt).  Here one elected thread moves each
// (16-token block, kv head, 64-dim half) box with a 3-D TMA copy over the
// cache viewed as [slots][Hkv][D]: the box lands 128-byte swizzled (SW128),
// which is exactly the XOR pattern the ldmatrix addressing below undoes, and
// blocks past the sequence load with a negative slot coordinate (zero fill).
// Ring stages complete on mbarriers (expect_tx).  Math, warp roles and the
// key-group merge as in attention_kernel.
template <int D, int NS>
__global__ void __launch_bounds__(ATT_THREADS)
attention_tma_kernel(const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __nv_bfloat16* __restrict__ q,
                     const int32_t* __restrict__ block_table, int max_blocks,
                     const int32_t* __restrict__ seq_slot, const int32_t* __restrict__ q_start,
                     const int32_t* __restrict__ q_len, const int32_t* __restrict__ q_pos0,
                     const int32_t* __restrict__ kv_len, int Hq, int Hkv, float scale_log2,
                     int tok_per_chunk, int RG, __nv_bfloat16* __restrict__ out) {
  constexpr int KT = 32;                 // keys per tile = two 16-token blocks
  constexpr int NB64 = D / 64;           // 64-dim boxes per key row
  constexpr int BOXB = 16 * 128;         // one box: 16 keys x 64 dims bf16
  constexpr int TILEB = 2 * NB64 * BOXB; // one K (or V) tile
  constexpr int P = D + 8;
  const int KG = 4 / RG;
  const int seq = blockIdx.x, hk = blockIdx.y, chunk = blockIdx.z;
  const int G = Hq / Hkv;
  const int ql = q_len[seq];
  const int t0 = chunk * tok_per_chunk;
  if (t0 >= ql) return;
  const int nt = min(tok_per_chunk, ql - t0);
  const int R = nt * G;
  const int kvl = kv_len[seq];
  const int qs = q_start[seq];
  const int first_pos = q_pos0[seq];
  const int last_key = min(first_pos + t0 + nt - 1, kvl - 1);
  const int* btg = block_table + (size_t)seq_slot[seq] * max_blocks;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, c = lane & 3;
  const int rg = warp % RG, kg = warp / RG;
  __shared__ int bt[ATT_MAX_BLOCKS];
  __shared__ __align__(8) uint64_t full[NS];
  const int nblk_used = min((last_key >> 4) + 1, max_blocks);
  for (int i = tid; i < nblk_used; i += ATT_THREADS) bt[i] = btg[i];
  extern __shared__ __align__(1024) uint8_t at_smem[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(at_smem) + 1023) &
                                             ~uintptr_t(1023));
  typedef __nv_bfloat16 Row[P];
  Row* sQ = reinterpret_cast<Row*>(ring + (size_t)NS * KG * 2 * TILEB);
  if (tid == 0) {
    psd::tma_prefetch(&tmK);
    psd::tma_prefetch(&tmV);
    for (int s = 0; s < NS; ++s) psd::mbar_init(full + s, 1);
    psd::fence_barrier_init();
  }
  const int ntiles = last_key / KT + 1;
  const int ngroups = (ntiles + KG - 1) / KG;
  __syncthreads();  // bt staged, barriers initialised
  const uint32_t ring_s = psd::smem_u32(ring);
  auto kbase = [&](int st, int j) { return ring + (size_t)((st * KG + j) * 2) * TILEB; };
  // group gi -> stage st (thread 0): KG tiles x 2 blocks x NB64 boxes, K and V
  auto issue = [&](int gi, int st) {
    psd::mbar_arrive_expect_tx(full + st, (uint32_t)(KG * 2 * TILEB));
    for (int j = 0; j < KG; ++j) {
      const int tile = gi * KG + j;
      uint8_t* kd = kbase(st, j);
      uint8_t* vd = kd + TILEB;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int blk = tile * 2 + b;
        const int slot = (tile < ntiles && blk < nblk_used) ? bt[blk] * 16 : -16;
#pragma unroll
        for (int x = 0; x < NB64; ++x) {
          psd::tma_load_3d(kd + (b * NB64 + x) * BOXB, &tmK, full + st, x * 64, hk, slot);
          psd::tma_load_3d(vd + (b * NB64 + x) * BOXB, &tmV, full + st, x * 64, hk, slot);
        }
      }
    }
  };
  // prefetch groups whose blocks hold only keys of earlier steps before
  // griddepcontrol.wait: the predecessor (the RoPE / KV-write kernel) writes
  // only this step's keys, so these loads overlap its tail
  int npre = 0;
  if (tid == 0) {
    while (npre < NS - 1 && npre < ngroups && (npre + 1) * KG * KT <= first_pos) {
      issue(npre, npre);
      ++npre;
    }
  }
  pdl_wait();
  pdl_trigger();
  if (tid == 0) {
    for (int t = npre; t < NS - 1 && t < ngroups; ++t) issue(t, t);
  }
  for (int idx = tid; idx < RG * 16 * (D / 8); idx += ATT_THREADS) {
    const int r = idx / (D / 8), cc = idx % (D / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < R) {
      const int t = r / G, gg = r % G;
      v = *reinterpret_cast<const uint4*>(q + ((size_t)(qs + t0 + t) * Hq + hk * G + gg) * D +
                                          cc * 8);
    }
    *reinterpret_cast<uint4*>(&sQ[r][cc * 8]) = v;
  }
  __syncthreads();

  const bool active = kg < KG && rg * 16 < R;
  const int r0 = rg * 16 + g, r1 = r0 + 8;
  const int lim0 = r0 < R ? min(first_pos + t0 + r0 / G, kvl - 1) : -1;
  const int lim1 = r1 < R ? min(first_pos + t0 + r1 / G, kvl - 1) : -1;
  uint32_t qf[D / 16][4];
  if (active) {
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      qf[kk][0] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 2 * c]);
      qf[kk][1] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 2 * c]);
      qf[kk][2] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 8 + 2 * c]);
      qf[kk][3] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 8 + 2 * c]);
    }
  }
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int lrow = lane & 7, lmat = lane >> 3;
  // byte offset of (key row, 16-byte dim chunk) inside a SW128 tile
  auto toff = [](int row, int ch) -> uint32_t {
    return (uint32_t)(((((row >> 4) * NB64 + (ch >> 3)) * 16 + (row & 15)) << 7) +
                      (((ch & 7) ^ (row & 7)) << 4));
  };

  for (int gi = 0; gi < ngroups; ++gi) {
    const int st = gi % NS;
    if (tid == 0 && gi + NS - 1 < ngroups) issue(gi + NS - 1, (gi + NS - 1) % NS);
    psd::mbar_wait(full + st, (uint32_t)((gi / NS) & 1));
    const int kt = gi * KG + kg;
    if (active && kt < ntiles) {
      const uint32_t sk = ring_s + (uint32_t)((st * KG + kg) * 2) * TILEB;
      const uint32_t sv = sk + TILEB;
      float sacc[KT / 8][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < KT / 8; n += 2) {
          uint32_t kb[4];
          const uint32_t a = sk + toff((n + (lmat >> 1)) * 8 + lrow, 2 * kk + (lmat & 1));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(a));
          mma_bf16_16816(sacc[n], qf[kk], kb[0], kb[1]);
          mma_bf16_16816(sacc[n + 1], qf[kk], kb[2], kb[3]);
        }
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const int key = kt * KT + n * 8 + 2 * c;
        sacc[n][0] = key <= lim0 ? sacc[n][0] * scale_log2 : -INFINITY;
        sacc[n][1] = key + 1 <= lim0 ? sacc[n][1] * scale_log2 : -INFINITY;
        sacc[n][2] = key <= lim1 ? sacc[n][2] * scale_log2 : -INFINITY;
        sacc[n][3] = key + 1 <= lim1 ? sacc[n][3] * scale_log2 : -INFINITY;
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
      uint32_t pf[KT / 16][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const float p0 = exp2f(sacc[n][0] - base0), p1 = exp2f(sacc[n][1] - base0);
        const float p2 = exp2f(sacc[n][2] - base1), p3 = exp2f(sacc[n][3] - base1);
        ps0 += p0 + p1;
        ps1 += p2 + p3;
        const int kk = n >> 1;
        if ((n & 1) == 0) {
          pf[kk][0] = pack_bf16(p0, p1);
          pf[kk][1] = pack_bf16(p2, p3);
        } else {
          pf[kk][2] = pack_bf16(p0, p1);
          pf[kk][3] = pack_bf16(p2, p3);
        }
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= al0; o[n][1] *= al0; o[n][2] *= al1; o[n][3] *= al1;
      }
#pragma unroll
      for (int kk = 0; kk < KT / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < D / 8; n += 2) {
          uint32_t vb[4];
          const uint32_t a = sv + toff(kk * 16 + (lmat & 1) * 8 + lrow, n + (lmat >> 1));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(a));
          mma_bf16_16816(o[n], pf[kk], vb[0], vb[1]);
          mma_bf16_16816(o[n + 1], pf[kk], vb[2], vb[3]);
        }
      }
    }
    __syncthreads();  // stage st is free for the group NS - 1 ahead
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  if (KG > 1) {
    // merge key-group states through the (idle) ring: warp (rg, kg > 0)
    // publishes, warp (rg, 0) merges in key-group order
    float* scr = reinterpret_cast<float*>(ring);
    const int slot_floats = 16 * D + 32;
    if (active && kg > 0) {
      float* sp = scr + (rg * KG + kg) * slot_floats;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int d = n * 8 + 2 * c;
        sp[g * D + d] = o[n][0];
        sp[g * D + d + 1] = o[n][1];
        sp[(g + 8) * D + d] = o[n][2];
        sp[(g + 8) * D + d + 1] = o[n][3];
      }
      if (c == 0) {
        sp[16 * D + g] = m0;
        sp[16 * D + g + 8] = m1;
        sp[16 * D + 16 + g] = l0;
        sp[16 * D + 16 + g + 8] = l1;
      }
    }
    __syncthreads();
    if (active && kg == 0) {
      float M0 = m0, M1 = m1;
      for (int j = 1; j < KG; ++j) {
        const float* sp = scr + (rg * KG + j) * slot_floats;
        M0 = fmaxf(M0, sp[16 * D + g]);
        M1 = fmaxf(M1, sp[16 * D + g + 8]);
      }
      const float w00 = M0 == -INFINITY ? 0.f : exp2f(m0 - M0);
      const float w10 = M1 == -INFINITY ? 0.f : exp2f(m1 - M1);
      l0 *= w00;
      l1 *= w10;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= w00; o[n][1] *= w00; o[n][2] *= w10; o[n][3] *= w10;
      }
      for (int j = 1; j < KG; ++j) {
        const float* sp = scr + (rg * KG + j) * slot_floats;
        const float mj0 = sp[16 * D + g], mj1 = sp[16 * D + g + 8];
        const float wj0 = mj0 == -INFINITY ? 0.f : exp2f(mj0 - M0);
        const float wj1 = mj1 == -INFINITY ? 0.f : exp2f(mj1 - M1);
        l0 += sp[16 * D + 16 + g] * wj0;
        l1 += sp[16 * D + 16 + g + 8] * wj1;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          const int d = n * 8 + 2 * c;
          o[n][0] += sp[g * D + d] * wj0;
          o[n][1] += sp[g * D + d + 1] * wj0;
          o[n][2] += sp[(g + 8) * D + d] * wj1;
          o[n][3] += sp[(g + 8) * D + d + 1] * wj1;
        }
      }
    }
  }
  if (!active || kg != 0) return;
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int ta0 = r0 / G, ga0 = r0 % G, ta1 = r1 / G, ga1 = r1 % G;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    const int d = n * 8 + 2 * c;
    if (r0 < R)
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t0 + ta0) * Hq + hk * G + ga0) * D +
                                         d) = __floats2bfloat162_rn(o[n][0] * inv0, o[n][1] * inv0);
    if (r1 < R)
      *reinterpret_cast<__nv_bfloat162*>(out + ((size_t)(qs + t0 + ta1) * Hq + hk * G + ga1) * D +
                                         d) = __floats2bfloat162_rn(o[n][2] * inv1, o[n][3] * inv1);
  }
}

// ---- decode attention: every key of a sequence in flight at once -------------
// For draft decode passes (<= 16 query rows per kv head: 1-2 tokens x G heads).
// One CTA per (sequence, kv head) issues the cp.async copies of ALL its key
// tiles at once (up to `cap` tiles per round -- the whole context at the
// BASELINE shapes: one HBM round trip instead of a ring of them); the keys of
// earlier steps are requested before griddepcontrol.wait.  With ROPE the CTA
// rotates its queries from the QKV split-K partials and writes this step's
// K / V rows both to the paged cache (for later steps) and straight into its
// shared-memory tiles, so they are not read back through L2.  Tiles are stored
// unpadded with the 16-byte chunks XOR-swizzled per row (ldmatrix of 8
// consecutive keys hits 8 bank groups).  Math as in attention_kernel (key
// groups of warps, mma.sync m16n8k16, online exp2 softmax, shared-memory merge
// of the key groups).  Measured variants (profiles/r02_attn_dec.txt): a
// cluster split of the keys with a DSMEM merge was 2-5x slower at these
// shapes, 8 warps instead of 4 no faster.
template <int D>
__device__ __forceinline__ uint32_t swz(int r, int c) {
  constexpr int CPR = D / 8;  // 16-byte chunks per key row
  if constexpr (CPR >= 8)
    return (uint32_t)(r * CPR + ((c & ~7) | ((c & 7) ^ (r & 7)))) * 16u;
  else
    return (uint32_t)(r * CPR + (c ^ ((r >> 1) & 3))) * 16u;
}

constexpr int ADEC_KT = 32;  // keys per tile

template <int D, bool ROPE>
__global__ void __launch_bounds__(ATT_THREADS)
attn_dec_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ block_table,
                int max_blocks, const int32_t* __restrict__ seq_slot,
                const int32_t* __restrict__ q_start, const int32_t* __restrict__ q_len,
                const int32_t* __restrict__ q_pos0, const int32_t* __restrict__ kv_len, int Hq,
                int Hkv, int bs, float scale_log2, int cap, __nv_bfloat16* __restrict__ out,
                const RopeSrc rs) {
  constexpr int KT = ADEC_KT;
  constexpr int P = D + 8;                 // sQ row pitch
  constexpr int TB = KT * D * 2;           // bytes of one K (or V) tile
  constexpr int CPR = D / 8;
  constexpr int PER_T = KT * CPR / ATT_THREADS;
  static_assert(KT * CPR % ATT_THREADS == 0, "tile chunks must tile the CTA");
  constexpr int KG = 4;                    // one row group (<= 16 rows), 4 key groups
  const int seq = blockIdx.x, hk = blockIdx.y;
  const int G = Hq / Hkv;
  const int tid = threadIdx.x, lane = tid & 31, kg = tid >> 5;
  const int g = lane >> 2, c = lane & 3;

  const int nt = q_len[seq];
  const int R = nt * G;
  const int kvl = kv_len[seq];
  const int qs = q_start[seq];
  const int first_pos = q_pos0[seq];
  const int last_key = nt > 0 ? min(first_pos + nt - 1, kvl - 1) : -1;
  const int ntl = last_key >= 0 ? last_key / KT + 1 : 0;

  extern __shared__ __align__(128) uint8_t ad_smem[];
  typedef __nv_bfloat16 Row[P];
  Row* sQ = reinterpret_cast<Row*>(ad_smem);
  uint8_t* sKV = ad_smem + ((16 * P * 2 + 127) & ~127);  // cap x (K tile, V tile)
  int* bt = reinterpret_cast<int*>(sKV + (size_t)cap * 2 * TB);
  const int bs_shift = __ffs(bs) - 1;
  const int nblk_used = last_key >= 0 ? min((last_key >> bs_shift) + 1, max_blocks) : 0;
  if (nt > 0) {
    const int* btg = block_table + (size_t)seq_slot[seq] * max_blocks;
    for (int i = tid; i < nblk_used; i += ATT_THREADS) bt[i] = btg[i];
  }
  __syncthreads();
  // per-thread constants of its chunk positions (see attention_kernel)
  uint32_t c_off[PER_T], c_soff[PER_T];
  int c_row[PER_T], c_blk[PER_T];
#pragma unroll
  for (int i = 0; i < PER_T; ++i) {
    const int idx = tid + ATT_THREADS * i;
    const int r = idx / CPR, cc = idx % CPR;
    c_row[i] = r;
    c_blk[i] = r >> bs_shift;
    c_off[i] = (uint32_t)(((r & (bs - 1)) * Hkv + hk) * D + cc * 8);
    c_soff[i] = swz<D>(r, cc);
  }
  const uint32_t blk_elems = (uint32_t)(bs * Hkv * D);
  const uint32_t skv_s = static_cast<uint32_t>(__cvta_generic_to_shared(sKV));
  // tiles [t0, t0 + n) into slots 0..n-1.  direct: rows of this step's keys
  // are not copied (RoPE stores them into the slots); rows past the last key
  // are zero-filled
  auto load_tiles = [&](int t0, int n, bool direct) {
    for (int j = 0; j < n; ++j) {
      const int tile = t0 + j;
      const uint32_t sk = skv_s + (uint32_t)(j * 2 * TB);
      const uint32_t sv = sk + TB;
      const int blk0 = (tile * KT) >> bs_shift;
#pragma unroll
      for (int i = 0; i < PER_T; ++i) {
        const int key = tile * KT + c_row[i];
        const bool ok = key <= last_key;
        if (direct && ok && key >= first_pos) continue;
        const uint64_t o = ok ? (uint64_t)(uint32_t)bt[blk0 + c_blk[i]] * blk_elems + c_off[i] : 0ull;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sk + c_soff[i]),
                     "l"(kc + o), "r"(ok ? 16 : 0));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sv + c_soff[i]),
                     "l"(vc + o), "r"(ok ? 16 : 0));
      }
    }
    cp_async_commit();
  };
  const int n0 = min(ntl, cap);
  // this step's keys go straight into the slots when they lie in round 0
  const bool direct = ROPE && (first_pos / KT) < n0;
  load_tiles(0, n0, direct);
  pdl_wait();
  pdl_trigger();
  if constexpr (ROPE) {
    constexpr int half = D / 2;
    const int NQKV = (Hq + 2 * Hkv) * D;
    // slot address of element i of new key row t (round 0 only)
    auto kv_slot = [&](int t, int i, bool v) -> __nv_bfloat16* {
      const int key = first_pos + t;
      const int j = key / KT, r = key % KT;
      return reinterpret_cast<__nv_bfloat16*>(sKV + (size_t)j * 2 * TB + (v ? TB : 0) +
                                              swz<D>(r, i / 8) + (i % 8) * 2);
    };
    // per token: (G + 1) rotation heads x half pairs, then the D values of
    // the V row -- every index split is by a power of two (no runtime division)
    const int nrot1 = (G + 1) * half;
    for (int t = 0; t < nt; ++t) {
      const int m = qs + t;
      const int sl = rs.slots[m];
      const float pos = (float)rs.positions[m];
      const bool to_smem = direct && first_pos + t <= last_key;
      for (int j = tid; j < nrot1 + D; j += ATT_THREADS) {
        if (j >= nrot1) {
          const int i = j - nrot1;
          if (sl < 0) continue;
          const int col = (Hq + Hkv + hk) * D + i;
          float a = sum_parts(rs, (size_t)m * NQKV + col);
          if (rs.bias) a = a + __bfloat162float(rs.bias[col]);
          vc_w(vc, ((size_t)sl * Hkv + hk) * D + i, a);
          if (to_smem) *kv_slot(t, i, true) = __float2bfloat16(a);
          continue;
        }
        const int hh = j / half, i = j % half;
        if (hh == G && sl < 0) continue;
        const int head = hh < G ? hk * G + hh : Hq + hk;
        const int col = head * D + i;
        float a = sum_parts(rs, (size_t)m * NQKV + col);
        float b = sum_parts(rs, (size_t)m * NQKV + col + half);
        if (rs.bias) {
          a = __bfloat162float(__float2bfloat16(a + __bfloat162float(rs.bias[col])));
          b = __bfloat162float(__float2bfloat16(b + __bfloat162float(rs.bias[col + half])));
        }
        float sn, cs;
        sincosf(pos * rs.inv_freq[i], &sn, &cs);
        const __nv_bfloat16 ra = __float2bfloat16(a * cs - b * sn);
        const __nv_bfloat16 rb = __float2bfloat16(b * cs + a * sn);
        if (hh < G) {
          sQ[t * G + hh][i] = ra;
          sQ[t * G + hh][i + half] = rb;
        } else {
          __nv_bfloat16* dst = const_cast<__nv_bfloat16*>(kc) + ((size_t)sl * Hkv + hk) * D;
          dst[i] = ra;
          dst[i + half] = rb;
          if (to_smem) {
            *kv_slot(t, i, false) = ra;
            *kv_slot(t, i + half, false) = rb;
          }
        }
      }
    }
    for (int idx = tid; idx < (16 - R) * D; idx += ATT_THREADS)
      sQ[R + idx / D][idx % D] = __float2bfloat16(0.f);
    // rows read back through L2 in a later round need the global writes first
    if (!direct) __threadfence();
  } else {
    for (int idx = tid; idx < 16 * (D / 8); idx += ATT_THREADS) {
      const int r = idx / (D / 8), cc = idx % (D / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < R) {
        const int t = r / G, gg = r % G;
        v = *reinterpret_cast<const uint4*>(q + ((size_t)(qs + t) * Hq + hk * G + gg) * D + cc * 8);
      }
      *reinterpret_cast<uint4*>(&sQ[r][cc * 8]) = v;
    }
  }
  __syncthreads();

  const bool active = R > 0;
  const int r0 = g, r1 = g + 8;
  const int lim0 = r0 < R ? min(first_pos + r0 / G, kvl - 1) : -1;
  const int lim1 = r1 < R ? min(first_pos + r1 / G, kvl - 1) : -1;
  uint32_t qf[D / 16][4];
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    qf[kk][0] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 2 * c]);
    qf[kk][1] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 2 * c]);
    qf[kk][2] = *reinterpret_cast<const uint32_t*>(&sQ[r0][kk * 16 + 8 + 2 * c]);
    qf[kk][3] = *reinterpret_cast<const uint32_t*>(&sQ[r1][kk * 16 + 8 + 2 * c]);
  }
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int lrow = lane & 7, lmat = lane >> 3;

  for (int rb = 0; rb < ntl; rb += cap) {
    const int nr = min(cap, ntl - rb);
    if (rb > 0) {
      __syncthreads();  // the previous round's tiles are consumed
      load_tiles(rb, nr, false);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (!active) continue;
    for (int j = kg; j < nr; j += KG) {
      const int kt = rb + j;
      const uint32_t sk = static_cast<uint32_t>(__cvta_generic_to_shared(sKV + (size_t)j * 2 * TB));
      const uint32_t sv = sk + TB;
      float sacc[KT / 8][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < KT / 8; n += 2) {
          uint32_t kb[4];
          const int krow = (n + (lmat >> 1)) * 8 + lrow;
          const uint32_t a = sk + swz<D>(krow, 2 * kk + (lmat & 1));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(kb[0]), "=r"(kb[1]), "=r"(kb[2]), "=r"(kb[3]) : "r"(a));
          mma_bf16_16816(sacc[n], qf[kk], kb[0], kb[1]);
          mma_bf16_16816(sacc[n + 1], qf[kk], kb[2], kb[3]);
        }
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const int key = kt * KT + n * 8 + 2 * c;
        sacc[n][0] = key <= lim0 ? sacc[n][0] * scale_log2 : -INFINITY;
        sacc[n][1] = key + 1 <= lim0 ? sacc[n][1] * scale_log2 : -INFINITY;
        sacc[n][2] = key <= lim1 ? sacc[n][2] * scale_log2 : -INFINITY;
        sacc[n][3] = key + 1 <= lim1 ? sacc[n][3] * scale_log2 : -INFINITY;
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
      uint32_t pf[KT / 16][4];
#pragma unroll
      for (int n = 0; n < KT / 8; ++n) {
        const float p0 = exp2f(sacc[n][0] - base0), p1 = exp2f(sacc[n][1] - base0);
        const float p2 = exp2f(sacc[n][2] - base1), p3 = exp2f(sacc[n][3] - base1);
        ps0 += p0 + p1;
        ps1 += p2 + p3;
        const int kk = n >> 1;
        if ((n & 1) == 0) {
          pf[kk][0] = pack_bf16(p0, p1);
          pf[kk][1] = pack_bf16(p2, p3);
        } else {
          pf[kk][2] = pack_bf16(p0, p1);
          pf[kk][3] = pack_bf16(p2, p3);
        }
      }
      l0 = l0 * al0 + ps0;
      l1 = l1 * al1 + ps1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= al0; o[n][1] *= al0; o[n][2] *= al1; o[n][3] *= al1;
      }
#pragma unroll
      for (int kk = 0; kk < KT / 16; ++kk) {
#pragma unroll
        for (int n = 0; n < D / 8; n += 2) {
          uint32_t vb[4];
          const int krow = kk * 16 + (lmat & 1) * 8 + lrow;
          const uint32_t a = sv + swz<D>(krow, n + (lmat >> 1));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]) : "r"(a));
          mma_bf16_16816(o[n], pf[kk], vb[0], vb[1]);
          mma_bf16_16816(o[n + 1], pf[kk], vb[2], vb[3]);
        }
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  // merge the key groups: warps 1..3 publish in the (now idle) tile region,
  // warp 0 merges in key-group order
  cp_async_wait<0>();
  __syncthreads();
  float* scr = reinterpret_cast<float*>(sKV);
  const int slot_floats = 16 * D + 32;
  if (active && kg > 0) {
    float* sp = scr + kg * slot_floats;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int d = n * 8 + 2 * c;
      sp[g * D + d] = o[n][0];
      sp[g * D + d + 1] = o[n][1];
      sp[(g + 8) * D + d] = o[n][2];
      sp[(g + 8) * D + d + 1] = o[n][3];
    }
    if (c == 0) {
      sp[16 * D + g] = m0;
      sp[16 * D + g + 8] = m1;
      sp[16 * D + 16 + g] = l0;
      sp[16 * D + 16 + g + 8] = l1;
    }
  }
  __syncthreads();
  if (!active || kg != 0) return;
  float M0 = m0, M1 = m1;
  for (int j = 1; j < KG; ++j) {
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
    o[n][0] *= w00; o[n][1] *= w00; o[n][2] *= w10; o[n][3] *= w10;
  }
  for (int j = 1; j < KG; ++j) {
    const float* sp = scr + j * slot_floats;
    const float mj0 = sp[16 * D + g], mj1 = sp[16 * D + g + 8];
    const float wj0 = mj0 == -INFINITY ? 0.f : exp2f(mj0 - M0);
    const float wj1 = mj1 == -INFINITY ? 0.f : exp2f(mj1 - M1);
    l0 += sp[16 * D + 16 + g] * wj0;
    l1 += sp[16 * D + 16 + g + 8] * wj1;
#pragma unroll
    for (int n = 0; n < D / 8; ++n) {
      const int d = n * 8 + 2 * c;
      o[n][0] += sp[g * D + d] * wj0;
      o[n][1] += sp[g * D + d + 1] * wj0;
      o[n][2] += sp[(g + 8) * D + d] * wj1;
      o[n][3] += sp[(g + 8) * D + d + 1] * wj1;
    }
  }
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  __nv_bfloat16* o0 = out + ((size_t)(qs + r0 / G) * Hq + hk * G + r0 % G) * D;
  __nv_bfloat16* o1 = out + ((size_t)(qs + r1 / G) * Hq + hk * G + r1 % G) * D;
#pragma unroll
  for (int n = 0; n < D / 8; ++n) {
    const int d = n * 8 + 2 * c;
    if (r0 < R)
      *reinterpret_cast<__nv_bfloat162*>(o0 + d) = __floats2bfloat162_rn(o[n][0] * inv0, o[n][1] * inv0);
    if (r1 < R)
      *reinterpret_cast<__nv_bfloat162*>(o1 + d) = __floats2bfloat162_rn(o[n][2] * inv1, o[n][3] * inv1);
  }
}

// key splits for split-KV: a decode/verify CTA's latency is its serial chain
// of key tiles, so split until every CTA has <= ~128 keys or the grid holds
// ~4 waves of 148 SMs (>= 32 keys per split)
// PSD_ATT_MAX_SPLITS caps the split-KV factor (A/B runs)
int att_max_splits() {
  static int v = [] {
    const char* e = getenv("PSD_ATT_MAX_SPLITS");
    return e ? atoi(e) : 8;
  }();
  return v;
}

int att_splits(int ctas, int max_kv_len) {
  if (max_kv_len <= 0) return 1;
  int S = 1;
  const int smax = att_max_splits();
  while (S < smax && (ctas * S < 4 * 148 || max_kv_len / S > 128) && max_kv_len / (S * 2) >= 32)
    S *= 2;
  return S;
}

// ---- synthetic-language bias (shared by draft and target) -----------------------
// logits hold vocabulary columns [v0, v1) (a tensor-parallel shard, or the
// whole row with v0 = 0, v1 = V)
__global__ void bigram_bias_kernel(float* __restrict__ logits, int64_t ld,
                                   const int32_t* __restrict__ prev, int M,
                                   const int32_t* __restrict__ succ, int V, float beta, int v0,
                                   int v1) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int t = prev[m];
  if (t < 0 || t >= V) return;
  const int col = succ[t];
  if (col >= v0 && col < v1) logits[m * ld + col - v0] += beta;
}

// ---- Philox4x32-10 uniforms keyed (seed, request, verify index, position) ------
__host__ __device__ inline void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
  c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

__global__ void philox_uniform_kernel(uint64_t seed, const int32_t* __restrict__ rid,
                                      const int32_t* __restrict__ jv, int B, int n, int base,
                                      float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * n) return;
  const int b = idx / n, i = idx % n;
  uint32_t c[4] = {(uint32_t)rid[b], (uint32_t)jv[b], (uint32_t)(base + i), 0u};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[idx] = (float)(c[0] >> 8) * (1.0f / 16777216.0f);
}

// dst[dst_idx[i]] = src[src_idx[i]]  (negative dst index: skip)
__global__ void index_copy_kernel(int32_t* __restrict__ dst, const int32_t* __restrict__ dst_idx,
                                  const int32_t* __restrict__ src,
                                  const int32_t* __restrict__ src_idx, int n) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = dst_idx ? dst_idx[i] : i;
  if (d < 0) return;
  dst[d] = src[src_idx ? src_idx[i] : i];
}

// K5 commit: per verified row append accepted + bonus to the slot's output,
// advance the slot's generated count and its last two tokens.
__global__ void commit_kernel(const int32_t* __restrict__ acc, const int32_t* __restrict__ out_tok,
                              int K, const int32_t* __restrict__ row_slot, int n,
                              int32_t* __restrict__ gen, int32_t* __restrict__ slot_tok, int ldt,
                              int32_t* __restrict__ outputs, int ldo) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int s = row_slot[b];
  if (s < 0) return;
  const int a = acc[b];
  const int g = gen[s];
  const int32_t* o = out_tok + (size_t)b * (K + 1);
  for (int i = 0; i <= a; ++i)
    if (g + i < ldo) outputs[(size_t)s * ldo + g + i] = o[i];
  gen[s] = g + a + 1;
  int32_t* t = slot_tok + (size_t)s * ldt;
  t[0] = a >= 1 ? o[a - 1] : t[1];
  t[1] = o[a];
}

// deterministic weight init: x_i = (u_i - 1/2) * span, u_i = top 24 bits of
// splitmix64(seed, i) / 2^24 (bit-reproducible in numpy, see oracle/model.py)
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  uint64_t x = (i + seed * 0x100000000ull) * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void fill_uniform_kernel(__nv_bfloat16* __restrict__ out, size_t n, uint64_t seed,
                                    float span) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float u = (float)(splitmix_at(seed, i) >> 40) * (1.0f / 16777216.0f);
    out[i] = __float2bfloat16((u - 0.5f) * span);
  }
}

// rows [row0, row0 + rows) x cols [col0, col0 + cols) of a virtual row-major
// tensor with `full_cols` columns, filled as fill_uniform_kernel would fill the
// whole tensor (element index row * full_cols + col) -> a tensor-parallel shard
// is generated in place, identical to the corresponding block of the full tensor
__global__ void fill_uniform_block_kernel(__nv_bfloat16* __restrict__ out, int64_t ld, int rows,
                                          int cols, int64_t full_cols, int64_t row0,
                                          int64_t col0, uint64_t seed, float span) {
  const size_t n = (size_t)rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)(i / cols), c = (int64_t)(i % cols);
    const uint64_t idx = (uint64_t)((row0 + r) * full_cols + col0 + c);
    const float u = (float)(splitmix_at(seed, idx) >> 40) * (1.0f / 16777216.0f);
    out[r * ld + c] = __float2bfloat16((u - 0.5f) * span);
  }
}

// dst[dst_rows[r] * dst_ld + c] = src[r * src_ld + c] (negative row: skip)
__global__ void copy_rows_kernel(float* __restrict__ dst, const int32_t* __restrict__ dst_rows,
                                 int64_t dst_ld, const float* __restrict__ src,
                                 const int32_t* __restrict__ src_rows, int64_t src_ld,
                                 int ncols) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const int dr = dst_rows ? dst_rows[r] : r;
  const int sr = src_rows ? src_rows[r] : r;
  if (dr < 0 || sr < 0) return;
  const float4* s4 = reinterpret_cast<const float4*>(src + sr * src_ld);
  float4* d4 = reinterpret_cast<float4*>(dst + dr * dst_ld);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols / 4; c += gridDim.x * blockDim.x)
    d4[c] = s4[c];
}

}  // namespace

extern "C" {

long long psd_launch_count(void) { return psd::launch_counter().load(); }

int psd_copy_rows_f32(float* dst, const int32_t* dst_rows, int64_t dst_ld, const float* src,
                      int64_t src_ld, int nrows, int ncols, void* stream) {
  if (nrows <= 0) return 0;
  if ((ncols & 3) || (dst_ld & 3) || (src_ld & 3)) return (int)cudaErrorMisalignedAddress;
  dim3 grid(16, nrows);
  return (int)psd::launch(copy_rows_kernel, grid, dim3(256), 0, (cudaStream_t)stream, dst, dst_rows,
                          dst_ld, src, (const int32_t*)nullptr, src_ld, ncols);
}

int psd_gather_rows_f32(float* dst, int64_t dst_ld, const float* src, const int32_t* src_rows,
                        int64_t src_ld, int nrows, int ncols, void* stream) {
  if (nrows <= 0) return 0;
  if ((ncols & 3) || (dst_ld & 3) || (src_ld & 3)) return (int)cudaErrorMisalignedAddress;
  dim3 grid(16, nrows);
  return (int)psd::launch(copy_rows_kernel, grid, dim3(256), 0, (cudaStream_t)stream, dst,
                          (const int32_t*)nullptr, dst_ld, src, src_rows, src_ld, ncols);
}

int psd_index_copy_i32(int32_t* dst, const int32_t* dst_idx, const int32_t* src,
                       const int32_t* src_idx, int n, void* stream) {
  if (n <= 0) return 0;
  return (int)psd::launch(index_copy_kernel, dim3((n + 255) / 256), dim3(256), 0,
                          (cudaStream_t)stream, dst, dst_idx, src, src_idx, n);
}

int psd_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return 0;
  return (int)cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream);
}

int psd_commit(const int32_t* accepted_len, const int32_t* out_tokens, int K,
               const int32_t* row_slot, int n, int32_t* generated, int32_t* slot_tokens,
               int slot_tokens_ld, int32_t* outputs, int outputs_ld, void* stream) {
  if (n <= 0) return 0;
  return (int)psd::launch(commit_kernel, dim3((n + 127) / 128), dim3(128), 0,
                          (cudaStream_t)stream, accepted_len, out_tokens, K, row_slot, n,
                          generated, slot_tokens, slot_tokens_ld, outputs, outputs_ld);
}

int psd_fill_uniform_bf16(void* out, size_t n, uint64_t seed, float span, void* stream) {
  if (n == 0) return 0;
  psd::count_launches();
  fill_uniform_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(static_cast<__nv_bfloat16*>(out),
                                                                n, seed, span);
  return (int)cudaGetLastError();
}

int psd_fill_uniform_bf16_block(void* out, int64_t ld, int rows, int cols, int64_t full_cols,
                                int64_t row0, int64_t col0, uint64_t seed, float span,
                                void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  psd::count_launches();
  fill_uniform_block_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      static_cast<__nv_bfloat16*>(out), ld, rows, cols, full_cols, row0, col0, seed, span);
  return (int)cudaGetLastError();
}

int psd_embed(const int32_t* tokens, int M, const void* table, int H, void* out, void* stream) {
  if (M <= 0) return 0;
  if (H % 8) return (int)cudaErrorInvalidValue;
  return (int)psd::launch(embed_kernel, dim3(M), dim3(128), 0, (cudaStream_t)stream, tokens,
                          static_cast<const __nv_bfloat16*>(table),
                          static_cast<__nv_bfloat16*>(out), H);
}

int psd_add_rmsnorm(void* x, int ldx, const float* partials, int S, size_t slice, int ldp,
                    const int32_t* rows, const void* w, void* y, int ldy, int M, int H, float eps,
                    int write_back, void* stream) {
  if (M <= 0) return 0;
  if (H % 8 || H > 8 * NORM_THREADS * 4) return (int)cudaErrorInvalidValue;
  auto go = [&](auto kern) {
    psd::launch(kern, dim3(M), dim3(NORM_THREADS), 0, (cudaStream_t)stream,
                static_cast<__nv_bfloat16*>(x), ldx, partials, S, slice, ldp, rows,
                static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(y), ldy, H, eps,
                write_back);
  };
  const int nv = (H / 8 + NORM_THREADS - 1) / NORM_THREADS;
  if (nv <= 1) go(add_rmsnorm_kernel<1>);
  else if (nv <= 2) go(add_rmsnorm_kernel<2>);
  else go(add_rmsnorm_kernel<4>);
  return (int)cudaGetLastError();
}

static int rope_launch(const QkvSrc& src, int M, int Hq, int Hkv, int D,
                       const int32_t* positions, const int32_t* slots, const float* inv_freq,
                       const void* qkv_bias, void* q_out, void* k_cache, void* v_cache,
                       void* stream);

int psd_rope_kv_partials(const float* qkv_partials, int S, size_t slice, int M, int Hq, int Hkv,
                         int D, const int32_t* positions, const int32_t* slots,
                         const float* inv_freq, const void* qkv_bias, void* q_out,
                         void* k_cache, void* v_cache, void* stream) {
  QkvSrc src{nullptr, qkv_partials, S, slice};
  return rope_launch(src, M, Hq, Hkv, D, positions, slots, inv_freq, qkv_bias, q_out, k_cache,
                     v_cache, stream);
}

int psd_rope_kv(const void* qkv, int M, int Hq, int Hkv, int D, const int32_t* positions,
                const int32_t* slots, const float* inv_freq, const void* qkv_bias, void* q_out,
                void* k_cache, void* v_cache, void* stream) {
  QkvSrc src{static_cast<const __nv_bfloat16*>(qkv), nullptr, 0, 0};
  return rope_launch(src, M, Hq, Hkv, D, positions, slots, inv_freq, qkv_bias, q_out, k_cache,
                     v_cache, stream);
}

static int rope_launch(const QkvSrc& src, int M, int Hq, int Hkv, int D,
                       const int32_t* positions, const int32_t* slots, const float* inv_freq,
                       const void* qkv_bias, void* q_out, void* k_cache, void* v_cache,
                       void* stream) {
  if (M <= 0) return 0;
  if (D % 16 || D > 256) return (int)cudaErrorInvalidValue;
  return (int)psd::launch(rope_kv_kernel, dim3(M), dim3(256), 0, (cudaStream_t)stream, src, Hq,
                          Hkv, D, positions, slots, inv_freq,
                          static_cast<const __nv_bfloat16*>(qkv_bias),
                          static_cast<__nv_bfloat16*>(q_out),
                          static_cast<__nv_bfloat16*>(k_cache),
                          static_cast<__nv_bfloat16*>(v_cache));
}

size_t psd_attention_workspace_bytes(int num_seqs, int Hkv, int max_q_len, int Hq, int D,
                                     int max_kv_len) {
  const int G = Hq / Hkv;
  // the finer token chunking attention_launch may pick (two key groups per CTA)
  const int tpc = std::max(1, std::min(ATT_MAXR / std::max(1, G), 32 / std::max(1, G)));
  const int chunks = (max_q_len + tpc - 1) / tpc;
  const int S = att_splits(num_seqs * Hkv * chunks, max_kv_len);
  const size_t units = (size_t)num_seqs * Hkv * chunks;
  return 4096 * sizeof(int) + units * S * ATT_MAXR * (D + 2) * sizeof(float);
}

// TMA view of one paged cache tensor [slots][Hkv][D] bf16: box = 64 dims x 1
// head x 16 slots, 128-byte swizzle.  The slot extent is left open (2^24):
// coordinates come from the block table, negative ones zero-fill.
typedef CUresult (*KvEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static KvEncodeFn kv_encode_fn() {
  static KvEncodeFn fn = [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<KvEncodeFn>(p);
    return (KvEncodeFn) nullptr;
  }();
  return fn;
}

static int make_kv_map(CUtensorMap* map, const void* base, int Hkv, int D) {
  KvEncodeFn fn = kv_encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15)) return 1;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)Hkv, (cuuint64_t)1 << 24};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)Hkv * D * 2};
  cuuint32_t box[3] = {64, 1, 16};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

// PSD_ATT_TMA=0 keeps the cp.async kernel for verify / prefill (A/B runs)
static int att_tma() {
  static const int v = [] {
    const char* e = getenv("PSD_ATT_TMA");
    return e ? atoi(e) : 1;
  }();
  return v;
}

static int att_ns() {
  static const int v = [] {
    const char* e = getenv("PSD_ATT_NS");
    return e ? atoi(e) : 2;
  }();
  return v;
}

static int attention_launch(const void* q, const void* k_cache, const void* v_cache,
                            const int32_t* block_table, int max_blocks, const int32_t* seq_slot,
                            const int32_t* q_start, const int32_t* q_len, const int32_t* q_pos0,
                            const int32_t* kv_len, int num_seqs, int max_q_len, int Hq, int Hkv,
                            int D, int block_size, float scale, void* out, int max_kv_len,
                            void* workspace, size_t workspace_bytes, const RopeSrc* rope,
                            void* stream) {
  if (num_seqs <= 0) return 0;
  if (Hq % Hkv) return (int)cudaErrorInvalidValue;
  const int G = Hq / Hkv;
  if (G > ATT_MAXR || max_blocks > ATT_MAX_BLOCKS) return (int)cudaErrorInvalidValue;
  if (block_size <= 0 || (block_size & (block_size - 1))) return (int)cudaErrorInvalidValue;
  int tpc = ATT_MAXR / G;
  // keep two key groups per CTA: when a sequence's rows would fill all four
  // warps as row groups (e.g. Qwen2.5-7B verify: 5 tokens x 7 heads), split
  // its tokens over two CTAs instead (PSD_ATT_KG2=0: the single-chunk split)
  static const int kg2 = [] {
    const char* e = getenv("PSD_ATT_KG2");
    return e ? atoi(e) : 1;
  }();
  // (not with fused RoPE, which needs a sequence's tokens in one CTA, nor
  // with split-KV, whose merge keeps the one-chunk geometry)
  if (kg2 && !rope && att_splits(num_seqs * Hkv * ((max_q_len + tpc - 1) / tpc),
                                 max_kv_len) == 1 &&
      (std::min(max_q_len, tpc) * G + 15) / 16 > 2)
    tpc = std::max(1, 32 / G);
  const int chunks = (max_q_len + tpc - 1) / tpc;
  // rows per CTA -> row groups; the other warps become key groups
  const int rmax = std::min(ATT_MAXR, std::min(max_q_len, tpc) * G);
  int RG = (rmax + 15) / 16;
  if (RG == 3) RG = 4;  // 4 / RG must be an integer number of key groups
  const int KG = 4 / RG;
  int S = rope ? 1 : att_splits(num_seqs * Hkv * chunks, max_kv_len);
  const size_t units = (size_t)num_seqs * Hkv * chunks;
  if (S > 1 && (!workspace || units > 4096 ||
                workspace_bytes < 4096 * sizeof(int) + units * S * ATT_MAXR * (D + 2) * 4))
    S = 1;  // no (or too little) workspace: no split
  // fused RoPE needs every token of a sequence in one CTA
  if (rope && (chunks != 1 || (rope->S > 16))) return (int)cudaErrorInvalidValue;
  int* tickets = static_cast<int*>(workspace);
  float* wsf = workspace ? reinterpret_cast<float*>(static_cast<char*>(workspace) + 4096 * 4)
                         : nullptr;
  dim3 grid(num_seqs, Hkv, chunks * S);
  const float sl2 = scale * 1.44269504088896341f;
  const RopeSrc rs = rope ? *rope : RopeSrc{};
  cudaError_t err = cudaSuccess;
  if (!rope && S == 1 && block_size == 16 && (D == 64 || D == 128) && att_tma()) {
    CUtensorMap mk, mv;
    if (make_kv_map(&mk, k_cache, Hkv, D) == 0 && make_kv_map(&mv, v_cache, Hkv, D) == 0) {
      const int ns = att_ns() >= 3 ? 3 : 2;
      const int tileb = 32 * D * 2;
      const int smem = 1024 + ns * KG * 2 * tileb + RG * 16 * (D + 8) * 2;
      auto go_tma = [&](auto kern) {
        if ((err = psd::ensure_smem_limit((const void*)kern, 200 * 1024, (cudaStream_t)stream)))
          return;
        err = psd::launch(kern, dim3(num_seqs, Hkv, chunks), dim3(ATT_THREADS), smem,
                          (cudaStream_t)stream, mk, mv, static_cast<const __nv_bfloat16*>(q),
                          block_table, max_blocks, seq_slot, q_start, q_len, q_pos0, kv_len, Hq,
                          Hkv, sl2, tpc, RG, static_cast<__nv_bfloat16*>(out));
      };
      if (D == 64) ns == 3 ? go_tma(attention_tma_kernel<64, 3>) : go_tma(attention_tma_kernel<64, 2>);
      else ns == 3 ? go_tma(attention_tma_kernel<128, 3>) : go_tma(attention_tma_kernel<128, 2>);
      return (int)err;
    }
  }
  auto go = [&](auto kern, int kt, int d, int ns = ATT_STAGES) {
    const int smem = (RG * 16 + 2 * ns * KG * kt) * (d + 8) * 2;
    if ((err = psd::ensure_smem_limit((const void*)kern, 200 * 1024, (cudaStream_t)stream)))
      return;
    err = psd::launch(kern, grid, dim3(ATT_THREADS), smem, (cudaStream_t)stream,
                static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k_cache),
                static_cast<const __nv_bfloat16*>(v_cache), block_table, max_blocks, seq_slot,
                q_start, q_len, q_pos0, kv_len, Hq, Hkv, block_size, sl2, tpc, RG, S, wsf,
                tickets, static_cast<__nv_bfloat16*>(out), rs);
  };
  switch (D) {
    case 32:
      if (rope) go(attention_kernel<32, 64, ATT_STAGES, true>, 64, 32);
      else go(attention_kernel<32, 64, ATT_STAGES, false>, 64, 32);
      break;
    case 64:
      if (rope) go(attention_kernel<64, 32, ATT_STAGES, true>, 32, 64);
      else go(attention_kernel<64, 32, ATT_STAGES, false>, 32, 64);
      break;
    case 128:
      // verify passes (k + 1 tokens x G heads): one more ring stage keeps two
      // tile groups in flight per CTA (PSD_ATT_NS=2: the 2-stage ring)
      if (rope) go(attention_kernel<128, 32, ATT_STAGES, true>, 32, 128);
      else if (att_ns() >= 3) go(attention_kernel<128, 32, 3, false>, 32, 128, 3);
      else go(attention_kernel<128, 32, ATT_STAGES, false>, 32, 128);
      break;
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)err;
}

// decode attention (attn_dec_kernel): one CTA per (sequence, kv head), every
// key tile in flight (cap = the block table's tiles, fewer if shared memory
// runs out: several rounds).  PSD_ATT_DEC=0 routes these passes to
// attention_kernel (A/B runs).
static bool attn_dec_eligible(int max_q_len, int G, int D) {
  static const int on = [] {
    const char* e = getenv("PSD_ATT_DEC");
    return e ? atoi(e) : 1;
  }();
  return on && max_q_len * G <= 16 && (D == 32 || D == 64 || D == 128);
}

static int attn_dec_launch(const void* q, const void* k_cache, const void* v_cache,
                           const int32_t* block_table, int max_blocks, const int32_t* seq_slot,
                           const int32_t* q_start, const int32_t* q_len, const int32_t* q_pos0,
                           const int32_t* kv_len, int num_seqs, int Hq, int Hkv, int D,
                           int block_size, float scale, void* out, const RopeSrc* rope,
                           void* stream) {
  int cap = (max_blocks * block_size + ADEC_KT - 1) / ADEC_KT;
  const int TB = ADEC_KT * D * 2;
  const int sq = (16 * (D + 8) * 2 + 127) & ~127;
  const int scratch = 4 * (16 * D + 32) * 4;  // key-group merge slots
  auto bytes = [&](int cp) { return sq + std::max(cp * 2 * TB + max_blocks * 4, scratch); };
  while (cap > 1 && bytes(cap) > 200 * 1024) --cap;
  cap = std::max(cap, 1);
  const int smem = bytes(cap);
  const RopeSrc rs = rope ? *rope : RopeSrc{};
  const float sl2 = scale * 1.44269504088896341f;
  cudaError_t err = cudaSuccess;
  auto go = [&](auto kern) {
    if ((err = psd::ensure_smem_limit((const void*)kern, 200 * 1024 + 1024, (cudaStream_t)stream)))
      return;
    err = psd::launch(kern, dim3(num_seqs, Hkv), dim3(ATT_THREADS), smem, (cudaStream_t)stream,
                      static_cast<const __nv_bfloat16*>(q),
                      static_cast<const __nv_bfloat16*>(k_cache),
                      static_cast<const __nv_bfloat16*>(v_cache), block_table, max_blocks,
                      seq_slot, q_start, q_len, q_pos0, kv_len, Hq, Hkv, block_size, sl2, cap,
                      static_cast<__nv_bfloat16*>(out), rs);
  };
  const bool r = rope != nullptr;
  switch (D) {
    case 32: r ? go(attn_dec_kernel<32, true>) : go(attn_dec_kernel<32, false>); break;
    case 64: r ? go(attn_dec_kernel<64, true>) : go(attn_dec_kernel<64, false>); break;
    case 128: r ? go(attn_dec_kernel<128, true>) : go(attn_dec_kernel<128, false>); break;
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)err;
}

int psd_attention(const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* block_table, int max_blocks, const int32_t* seq_slot,
                  const int32_t* q_start, const int32_t* q_len, const int32_t* q_pos0,
                  const int32_t* kv_len, int num_seqs, int max_q_len, int Hq, int Hkv, int D,
                  int block_size, float scale, void* out, int max_kv_len, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (num_seqs > 0 && Hkv > 0 && Hq % Hkv == 0 && max_blocks <= ATT_MAX_BLOCKS &&
      block_size > 0 && !(block_size & (block_size - 1)) &&
      attn_dec_eligible(max_q_len, Hq / Hkv, D))
    return attn_dec_launch(q, k_cache, v_cache, block_table, max_blocks, seq_slot, q_start, q_len,
                           q_pos0, kv_len, num_seqs, Hq, Hkv, D, block_size, scale, out, nullptr,
                           stream);
  return attention_launch(q, k_cache, v_cache, block_table, max_blocks, seq_slot, q_start, q_len,
                          q_pos0, kv_len, num_seqs, max_q_len, Hq, Hkv, D, block_size, scale, out,
                          max_kv_len, workspace, workspace_bytes, nullptr, stream);
}

int psd_attention_rope(const float* qkv_partials, int S, size_t slice, const int32_t* positions,
                       const int32_t* slots, const float* inv_freq, const void* qkv_bias,
                       void* k_cache, void* v_cache, const int32_t* block_table, int max_blocks,
                       const int32_t* seq_slot, const int32_t* q_start, const int32_t* q_len,
                       const int32_t* q_pos0, const int32_t* kv_len, int num_seqs, int max_q_len,
                       int Hq, int Hkv, int D, int block_size, float scale, void* out,
                       void* stream) {
  if (!qkv_partials || S <= 0 || !positions || !slots || !inv_freq)
    return (int)cudaErrorInvalidValue;
  RopeSrc rs;
  rs.P = qkv_partials;
  rs.S = S;
  rs.slice = slice;
  rs.positions = positions;
  rs.slots = slots;
  rs.inv_freq = inv_freq;
  rs.bias = static_cast<const __nv_bfloat16*>(qkv_bias);
  if (num_seqs > 0 && Hkv > 0 && Hq % Hkv == 0 && S <= 16 && max_blocks <= ATT_MAX_BLOCKS &&
      block_size > 0 && !(block_size & (block_size - 1)) &&
      attn_dec_eligible(max_q_len, Hq / Hkv, D))
    return attn_dec_launch(nullptr, k_cache, v_cache, block_table, max_blocks, seq_slot, q_start,
                           q_len, q_pos0, kv_len, num_seqs, Hq, Hkv, D, block_size, scale, out, &rs,
                           stream);
  return attention_launch(nullptr, k_cache, v_cache, block_table, max_blocks, seq_slot, q_start,
                          q_len, q_pos0, kv_len, num_seqs, max_q_len, Hq, Hkv, D, block_size,
                          scale, out, 0, nullptr, 0, &rs, stream);
}

int psd_bigram_bias(float* logits, int64_t ld, const int32_t* prev_tokens, int M,
                    const int32_t* successor, int V, float beta, void* stream) {
  return psd_bigram_bias_range(logits, ld, prev_tokens, M, successor, V, beta, 0, 1 << 30,
                               stream);
}

int psd_bigram_bias_range(float* logits, int64_t ld, const int32_t* prev_tokens, int M,
                          const int32_t* successor, int V, float beta, int v0, int v1,
                          void* stream) {
  if (M <= 0) return 0;
  return (int)psd::launch(bigram_bias_kernel, dim3((M + 127) / 128), dim3(128), 0,
                          (cudaStream_t)stream, logits, ld, prev_tokens, M, successor, V, beta,
                          v0, v1);
}

int psd_philox_uniforms(uint64_t seed, const int32_t* request_ids, const int32_t* verify_index,
                        int B, int n, int base, float* out, void* stream) {
  if (B * n <= 0) return 0;
  return (int)psd::launch(philox_uniform_kernel, dim3((B * n + 255) / 256), dim3(256), 0,
                          (cudaStream_t)stream, seed, request_ids, verify_index, B, n, base, out);
}

}  // extern "C"
