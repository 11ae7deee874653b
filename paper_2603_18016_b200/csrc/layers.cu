// layers.cu -- the non-GEMM kernels of the draft / target forwards (K3, K3',
// K4) and the small device-side glue of the PSD step (K5, K6 helpers).
//
// Replaces the virtual pass durations of the reference (verify_latency /
// draft_latency .duration, pkg/src/specsim/engine.py:338, 359-360, 378, 402,
// 429) together with gemm.cu.  All of these are HBM / latency bound and run
// on CUDA cores with 128-bit accesses; none is GEMM-shaped enough to pay for
// tensor-core staging at the BASELINE shapes (<= 64 query rows per KV head).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/psd.h"

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
  const int m = blockIdx.x;
  const int t = tok[m];
  const uint4* src = reinterpret_cast<const uint4*>(E + (size_t)(t < 0 ? 0 : t) * H);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)m * H);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x)
    dst[i] = t < 0 ? make_uint4(0, 0, 0, 0) : src[i];
}

// ---- RMSNorm (fp32 statistics) ------------------------------------------------
__global__ void rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, int ldx,
                               const int32_t* __restrict__ rows,
                               const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ y,
                               int ldy, int H, float eps) {
  const int m = blockIdx.x;
  const int src = rows ? rows[m] : m;
  const __nv_bfloat162* xr = reinterpret_cast<const __nv_bfloat162*>(x + (size_t)src * ldx);
  float ss = 0.f;
  for (int i = threadIdx.x; i < H / 2; i += blockDim.x) {
    const float2 v = __bfloat1622float2(xr[i]);
    ss += v.x * v.x + v.y * v.y;
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / H + eps);
  const __nv_bfloat162* wr = reinterpret_cast<const __nv_bfloat162*>(w);
  __nv_bfloat162* yr = reinterpret_cast<__nv_bfloat162*>(y + (size_t)m * ldy);
  for (int i = threadIdx.x; i < H / 2; i += blockDim.x) {
    const float2 v = __bfloat1622float2(xr[i]);
    const float2 g = __bfloat1622float2(wr[i]);
    yr[i] = __floats2bfloat162_rn(v.x * inv * g.x, v.y * inv * g.y);
  }
}

// ---- RoPE + paged KV write ------------------------------------------------------
// qkv [M, (Hq + 2 Hkv) D]; q_out [M, Hq, D]; caches [blocks, bs, Hkv, D].
// rotate-half convention: pairs (i, i + D/2), angle = pos * inv_freq[i].
__global__ void rope_kv_kernel(const __nv_bfloat16* __restrict__ qkv, int Hq, int Hkv, int D,
                               const int32_t* __restrict__ pos, const int32_t* __restrict__ slot,
                               const float* __restrict__ inv_freq,
                               const __nv_bfloat16* __restrict__ bias,
                               __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kc,
                               __nv_bfloat16* __restrict__ vc) {
  const int m = blockIdx.x;
  const int p = pos[m];
  const int s = slot[m];
  const int half = D / 2;
  const int nh = Hq + Hkv;  // heads that get rotated
  const __nv_bfloat16* row = qkv + (size_t)m * (Hq + 2 * Hkv) * D;
  for (int idx = threadIdx.x; idx < nh * half; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    float sn, cs;
    sincosf((float)p * inv_freq[i], &sn, &cs);
    float a = __bfloat162float(row[h * D + i]);
    float b = __bfloat162float(row[h * D + i + half]);
    if (bias) {  // qkv bias (Qwen2), rounded to bf16 like the projection output
      a = __bfloat162float(__float2bfloat16(a + __bfloat162float(bias[h * D + i])));
      b = __bfloat162float(__float2bfloat16(b + __bfloat162float(bias[h * D + i + half])));
    }
    const __nv_bfloat16 r0 = __float2bfloat16(a * cs - b * sn);
    const __nv_bfloat16 r1 = __float2bfloat16(b * cs + a * sn);
    if (h < Hq) {
      q_out[((size_t)m * Hq + h) * D + i] = r0;
      q_out[((size_t)m * Hq + h) * D + i + half] = r1;
    } else if (s >= 0) {
      const size_t o = ((size_t)s * Hkv + (h - Hq)) * D;
      kc[o + i] = r0;
      kc[o + i + half] = r1;
    }
  }
  if (s >= 0) {
    const __nv_bfloat16* vrow = row + (size_t)(Hq + Hkv) * D;
    const __nv_bfloat16* vb = bias ? bias + (size_t)(Hq + Hkv) * D : nullptr;
    for (int idx = threadIdx.x; idx < Hkv * D; idx += blockDim.x)
      vc[(size_t)s * Hkv * D + idx] =
          vb ? __float2bfloat16(__bfloat162float(vrow[idx]) + __bfloat162float(vb[idx])) : vrow[idx];
  }
}

// ---- paged multi-query attention (causal within the query window, GQA) ---------
// One CTA per (sequence, kv head, query chunk).  Query rows of the chunk: the
// chunk's tokens x the G = Hq / Hkv heads sharing this kv head.  KV streamed
// in tiles of 32 keys through shared memory; online softmax in fp32.
constexpr int ATT_THREADS = 128;
constexpr int ATT_KT = 32;        // keys per tile
constexpr int ATT_MAXR = 64;      // query rows per CTA
constexpr int ATT_MAXD = 128;

__global__ void __launch_bounds__(ATT_THREADS)
attention_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                 const __nv_bfloat16* __restrict__ vc, const int32_t* __restrict__ block_table,
                 int max_blocks, const int32_t* __restrict__ seq_slot,
                 const int32_t* __restrict__ q_start, const int32_t* __restrict__ q_len,
                 const int32_t* __restrict__ q_pos0, const int32_t* __restrict__ kv_len, int Hq,
                 int Hkv, int D, int bs, float scale, int tok_per_chunk,
                 __nv_bfloat16* __restrict__ out) {
  const int seq = blockIdx.x, hk = blockIdx.y, chunk = blockIdx.z;
  const int G = Hq / Hkv;
  const int ql = q_len[seq];
  const int t0 = chunk * tok_per_chunk;
  if (t0 >= ql) return;
  const int nt = min(tok_per_chunk, ql - t0);
  const int R = nt * G;
  const int kvl = kv_len[seq];
  const int qs = q_start[seq];
  const int first_pos = q_pos0[seq];  // position of query token 0
  // query t attends keys 0 .. min(first_pos + t, kvl - 1)
  const int last_key = min(first_pos + t0 + nt - 1, kvl - 1);
  const int* bt = block_table + (size_t)seq_slot[seq] * max_blocks;
  const int tid = threadIdx.x;

  __shared__ __nv_bfloat16 sQ[ATT_MAXR][ATT_MAXD + 8];
  __shared__ __nv_bfloat16 sK[ATT_KT][ATT_MAXD + 8];
  __shared__ __nv_bfloat16 sV[ATT_KT][ATT_MAXD + 8];
  __shared__ float sS[ATT_MAXR][ATT_KT + 1];
  __shared__ float sAlpha[ATT_MAXR], sM[ATT_MAXR], sL[ATT_MAXR];

  for (int idx = tid; idx < R * D; idx += ATT_THREADS) {
    const int r = idx / D, d = idx % D;
    const int t = r / G, g = r % G;
    sQ[r][d] = q[((size_t)(qs + t0 + t) * Hq + hk * G + g) * D + d];
  }
  for (int r = tid; r < R; r += ATT_THREADS) { sM[r] = -INFINITY; sL[r] = 0.f; }
  // PV ownership: item = (row, 4-dim group)
  const int dq = D / 4;
  const int nitems = R * dq;
  float acc[ATT_MAXR * ATT_MAXD / 4 / ATT_THREADS][4];
  constexpr int MAXIT = ATT_MAXR * ATT_MAXD / 4 / ATT_THREADS;
#pragma unroll
  for (int i = 0; i < MAXIT; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  __syncthreads();

  for (int k0 = 0; k0 <= last_key; k0 += ATT_KT) {
    // load K / V tile (keys k0 .. k0+31) from the paged cache
    for (int idx = tid; idx < ATT_KT * (D / 8); idx += ATT_THREADS) {
      const int j = idx / (D / 8), c = idx % (D / 8);
      const int key = k0 + j;
      uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = kv4;
      if (key <= last_key) {
        const int blk = bt[key / bs];
        const size_t o = (((size_t)blk * bs + key % bs) * Hkv + hk) * D + c * 8;
        kv4 = *reinterpret_cast<const uint4*>(kc + o);
        vv4 = *reinterpret_cast<const uint4*>(vc + o);
      }
      *reinterpret_cast<uint4*>(&sK[j][c * 8]) = kv4;
      *reinterpret_cast<uint4*>(&sV[j][c * 8]) = vv4;
    }
    __syncthreads();
    // scores
    for (int idx = tid; idx < R * ATT_KT; idx += ATT_THREADS) {
      const int r = idx / ATT_KT, j = idx % ATT_KT;
      const int key = k0 + j;
      const int qpos = min(first_pos + t0 + r / G, kvl - 1);
      float s = -INFINITY;
      if (key <= qpos) {
        s = 0.f;
        const __nv_bfloat162* kr = reinterpret_cast<const __nv_bfloat162*>(&sK[j][0]);
        const __nv_bfloat162* qr = reinterpret_cast<const __nv_bfloat162*>(&sQ[r][0]);
#pragma unroll 8
        for (int d2 = 0; d2 < D / 2; ++d2) {
          const float2 kf = __bfloat1622float2(kr[d2]);
          const float2 qf = __bfloat1622float2(qr[d2]);
          s += qf.x * kf.x + qf.y * kf.y;
        }
        s *= scale;
      }
      sS[r][j] = s;
    }
    __syncthreads();
    // online softmax, one warp per row
    for (int r = tid >> 5; r < R; r += ATT_THREADS / 32) {
      const int lane = tid & 31;
      const float s = sS[r][lane];
      const float mt = warp_max(s);
      const float mo = sM[r];
      const float mn = fmaxf(mo, mt);
      const float pexp = (s == -INFINITY) ? 0.f : __expf(s - mn);
      const float ps = warp_sum(pexp);
      sS[r][lane] = pexp;
      if (lane == 0) {
        const float al = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
        sAlpha[r] = al;
        sL[r] = sL[r] * al + ps;
        sM[r] = mn;
      }
    }
    __syncthreads();
    // O = alpha O + P V
#pragma unroll
    for (int i = 0; i < MAXIT; ++i) {
      const int it = tid + i * ATT_THREADS;
      if (it < nitems) {
        const int r = it / dq, d = (it % dq) * 4;
        const float al = sAlpha[r];
        float a0 = acc[i][0] * al, a1 = acc[i][1] * al, a2 = acc[i][2] * al, a3 = acc[i][3] * al;
#pragma unroll 8
        for (int j = 0; j < ATT_KT; ++j) {
          const float pj = sS[r][j];
          const float2 v01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sV[j][d]));
          const float2 v23 =
              __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sV[j][d + 2]));
          a0 += pj * v01.x; a1 += pj * v01.y; a2 += pj * v23.x; a3 += pj * v23.y;
        }
        acc[i][0] = a0; acc[i][1] = a1; acc[i][2] = a2; acc[i][3] = a3;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MAXIT; ++i) {
    const int it = tid + i * ATT_THREADS;
    if (it < nitems) {
      const int r = it / dq, d = (it % dq) * 4;
      const int t = r / G, g = r % G;
      const float inv = 1.f / sL[r];
      __nv_bfloat16* o = out + ((size_t)(qs + t0 + t) * Hq + hk * G + g) * D + d;
      *reinterpret_cast<__nv_bfloat162*>(o) = __floats2bfloat162_rn(acc[i][0] * inv, acc[i][1] * inv);
      *reinterpret_cast<__nv_bfloat162*>(o + 2) =
          __floats2bfloat162_rn(acc[i][2] * inv, acc[i][3] * inv);
    }
  }
}

// ---- synthetic-language bias (shared by draft and target) -----------------------
__global__ void bigram_bias_kernel(float* __restrict__ logits, int64_t ld,
                                   const int32_t* __restrict__ prev, int M,
                                   const int32_t* __restrict__ succ, int V, float beta) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int t = prev[m];
  if (t < 0 || t >= V) return;
  logits[m * ld + succ[t]] += beta;
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
                                      const int32_t* __restrict__ jv, int B, int n,
                                      float* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * n) return;
  const int b = idx / n, i = idx % n;
  uint32_t c[4] = {(uint32_t)rid[b], (uint32_t)jv[b], (uint32_t)i, 0u};
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

}  // namespace

extern "C" {

int psd_index_copy_i32(int32_t* dst, const int32_t* dst_idx, const int32_t* src,
                       const int32_t* src_idx, int n, void* stream) {
  if (n <= 0) return 0;
  index_copy_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(dst, dst_idx, src, src_idx, n);
  return (int)cudaGetLastError();
}

int psd_commit(const int32_t* accepted_len, const int32_t* out_tokens, int K,
               const int32_t* row_slot, int n, int32_t* generated, int32_t* slot_tokens,
               int slot_tokens_ld, int32_t* outputs, int outputs_ld, void* stream) {
  if (n <= 0) return 0;
  commit_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      accepted_len, out_tokens, K, row_slot, n, generated, slot_tokens, slot_tokens_ld, outputs,
      outputs_ld);
  return (int)cudaGetLastError();
}

int psd_fill_uniform_bf16(void* out, size_t n, uint64_t seed, float span, void* stream) {
  if (n == 0) return 0;
  fill_uniform_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(static_cast<__nv_bfloat16*>(out),
                                                                n, seed, span);
  return (int)cudaGetLastError();
}

int psd_embed(const int32_t* tokens, int M, const void* table, int H, void* out, void* stream) {
  if (M <= 0) return 0;
  if (H % 8) return (int)cudaErrorInvalidValue;
  embed_kernel<<<M, 128, 0, (cudaStream_t)stream>>>(
      tokens, static_cast<const __nv_bfloat16*>(table), static_cast<__nv_bfloat16*>(out), H);
  return (int)cudaGetLastError();
}

int psd_rmsnorm(const void* x, int ldx, const int32_t* rows, const void* w, void* y, int ldy, int M,
                int H, float eps, void* stream) {
  if (M <= 0) return 0;
  if (H % 2) return (int)cudaErrorInvalidValue;
  rmsnorm_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(x), ldx, rows, static_cast<const __nv_bfloat16*>(w),
      static_cast<__nv_bfloat16*>(y), ldy, H, eps);
  return (int)cudaGetLastError();
}

int psd_rope_kv(const void* qkv, int M, int Hq, int Hkv, int D, const int32_t* positions,
                const int32_t* slots, const float* inv_freq, const void* qkv_bias, void* q_out,
                void* k_cache, void* v_cache, void* stream) {
  if (M <= 0) return 0;
  if (D % 2 || D > 256) return (int)cudaErrorInvalidValue;
  rope_kv_kernel<<<M, 128, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(qkv), Hq, Hkv, D, positions, slots, inv_freq,
      static_cast<const __nv_bfloat16*>(qkv_bias), static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_cache),
      static_cast<__nv_bfloat16*>(v_cache));
  return (int)cudaGetLastError();
}

int psd_attention(const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* block_table, int max_blocks, const int32_t* seq_slot,
                  const int32_t* q_start, const int32_t* q_len, const int32_t* q_pos0,
                  const int32_t* kv_len, int num_seqs, int max_q_len, int Hq, int Hkv, int D,
                  int block_size, float scale, void* out, void* stream) {
  if (num_seqs <= 0) return 0;
  if (D > ATT_MAXD || D % 8 || Hq % Hkv) return (int)cudaErrorInvalidValue;
  const int G = Hq / Hkv;
  if (G > ATT_MAXR) return (int)cudaErrorInvalidValue;
  const int tpc = ATT_MAXR / G;
  const int chunks = (max_q_len + tpc - 1) / tpc;
  dim3 grid(num_seqs, Hkv, chunks);
  attention_kernel<<<grid, ATT_THREADS, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k_cache),
      static_cast<const __nv_bfloat16*>(v_cache), block_table, max_blocks, seq_slot, q_start, q_len,
      q_pos0, kv_len, Hq, Hkv, D, block_size, scale, tpc, static_cast<__nv_bfloat16*>(out));
  return (int)cudaGetLastError();
}

int psd_bigram_bias(float* logits, int64_t ld, const int32_t* prev_tokens, int M,
                    const int32_t* successor, int V, float beta, void* stream) {
  if (M <= 0) return 0;
  bigram_bias_kernel<<<(M + 127) / 128, 128, 0, (cudaStream_t)stream>>>(logits, ld, prev_tokens, M,
                                                                      successor, V, beta);
  return (int)cudaGetLastError();
}

int psd_philox_uniforms(uint64_t seed, const int32_t* request_ids, const int32_t* verify_index,
                        int B, int n, float* out, void* stream) {
  if (B * n <= 0) return 0;
  philox_uniform_kernel<<<(B * n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      seed, request_ids, verify_index, B, n, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
