// verify.cu -- K1: fused speculative verification on sm_100a.
//
// Replaces the reference's coin-flip acceptance (pkg/src/specsim/
// acceptance_model.py:82-97, called from engine.py:245-256) with the real
// token-level rule over target / draft logits.  Bit-exact with the CPU oracle
// (oracle/verify_oracle.c) because both evaluate include/psd_canon.h in the
// canonical order documented there.
//
// Two kernels per launch, HBM-bound by design:
//   verify_stats<SAMPLE>  grid (slice, request*row): every active (row, slice)
//       streams 8192 fp32 logits once with 128-bit L1-bypassing loads and
//       produces the canonical (max, sum-exp) [sampling] or (max, argmax)
//       [greedy] partial.
//   greedy:   verify_fold, one CTA per request: folds the slices, tests all k
//       drafts at once (one lane per draft, __ballot_sync finds the first
//       rejection), writes the accepted prefix and the bonus token.
//   sampling: verify_sample, grid (8-block chunk, request): each CTA folds and
//       decides for its request, then sums its chunk's 1024-element blocks of
//       the residual max(0, p - q) (or p for the bonus); the last chunk of a
//       request (atomic ticket) does the normalised prefix search and writes
//       the sampled token.
// Algorithmic bytes: greedy 4V*sum(k_b+1); sampling
// 4V*sum(2k_b+1) (+ small terms).  The sampling pass re-reads one (t, d) row
// pair per request (mostly from L2).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/psd.h"
#include "common.h"
#include "sm100.cuh"
#include "../../include/psd_canon.h"

namespace {
using namespace psd;

constexpr int kThreads = 256;

struct Plan {
  int mode;     // 1 = residual at row `row`, 2 = bonus from p at row `row`
  int row;      // position index a
  float Mt, St, Md, Sd;
  int pad[2];
};

struct Params {
  const float* t; int64_t tsb, tsi; int V;
  const float* d; int64_t dsb, dsi; int Vd;
  const int32_t* d_rows;  // optional: draft rows of request b start at d + d_rows[b] * dsb
  const int32_t* ids; const int32_t* len; const float* u;
  float c; int B, K;  // c = psd_scale(1/T)
  int32_t* acc; int32_t* out;
  int* cnt_b;
  float2* part; float* wblk;
  int NS, NB, R;
  // cached softmax statistics (M, S) of the draft rows: row (b, i) at
  // d_stats[d_rows[b] * d_stats_ld + i].  The draft sampler computed them with
  // the same canonical arithmetic when it drew the token, so the verifier does
  // not stream the draft rows again (null: computed here)
  const float2* d_stats; int64_t d_stats_ld;
  // output: (M, S) of target row 0 of request b to t_stats_out[t_stats_rows[b]]
  // (skipped for a negative row) -- how the draft sampler publishes them
  float2* t_stats_out; const int32_t* t_stats_rows;
  int voff;  // vocabulary offset of this logits shard (greedy partials of a TP rank)
  // replay mode (null: the real test): accept exactly min(forced[b], k_b)
  // drafts, then emit the target's token at that row -- GpuBackend's
  // acceptance="replay" commits the reference's coin-flip counts
  // (acceptance_model.py:82-97) on real logits
  const int32_t* forced;
};

__device__ __forceinline__ float4 ld_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---- packed (f32x2) canonical weights --------------------------------------
// Blackwell's FFMA2 / FADD2 round each half exactly like the scalar IEEE op,
// so two psd_weight() evaluations packed into one 64-bit register are
// bit-identical to two scalar calls (include/psd_canon.h) at half the issue
// slots.  The clamp and the integer exponent add stay scalar.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// (psd_weight(x0, c, bias), psd_weight(x1, c, bias)) -- see psd_exp2.  One
// PTX block on 64-bit register pairs so ptxas keeps the halves paired (no
// pack/unpack moves): FFMA2 argument, scalar clamp (max.f32 maps NaN to -125
// exactly like the canonical t > -125 ? t : -125), FADD2 rounding trick, six
// FFMA2 Horner steps, integer exponent add (bits(r) << 23 == (bits(r) -
// 0x4B400000) << 23 mod 2^32).
__device__ __forceinline__ void psd_weight2(float x0, float x1, unsigned long long c2,
                                            unsigned long long bias2, float& w0, float& w1) {
  asm("{\n\t"
      ".reg .b64 t, r, n, f, p, K, C;\n\t"
      ".reg .f32 a, b;\n\t"
      ".reg .b32 pa, pb, ra, rb;\n\t"
      "mov.b64 t, {%2, %3};\n\t"
      "fma.rn.f32x2 t, t, %4, %5;\n\t"
      "mov.b64 {a, b}, t;\n\t"
      "max.f32 a, a, 0fC2FA0000;\n\t"
      "max.f32 b, b, 0fC2FA0000;\n\t"
      "mov.b64 t, {a, b};\n\t"
      "mov.b64 K, 0x4B4000004B400000;\n\t"
      "add.rn.f32x2 r, t, K;\n\t"
      "sub.rn.f32x2 n, r, K;\n\t"
      "sub.rn.f32x2 f, t, n;\n\t"
      "mov.b64 p, 0x3921848939218489;\n\t"
      "mov.b64 C, 0x3AAEC3FF3AAEC3FF;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 C, 0x3C1D955B3C1D955B;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 C, 0x3D6358473D635847;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 C, 0x3E75FDF03E75FDF0;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 C, 0x3F3172183F317218;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 C, 0x3F8000003F800000;\n\t"
      "fma.rn.f32x2 p, p, f, C;\n\t"
      "mov.b64 {pa, pb}, p;\n\t"
      "mov.b64 {ra, rb}, r;\n\t"
      "shl.b32 ra, ra, 23;\n\t"
      "shl.b32 rb, rb, 23;\n\t"
      "add.u32 %0, pa, ra;\n\t"
      "add.u32 %1, pb, rb;\n\t"
      "}"
      : "=r"(*reinterpret_cast<uint32_t*>(&w0)), "=r"(*reinterpret_cast<uint32_t*>(&w1))
      : "f"(x0), "f"(x1), "l"(c2), "l"(bias2));
}

// three-input max (FMNMX3); the slice max is exact whatever the order
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}



__device__ __forceinline__ float shfl_add_tree(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = psd_add(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;
}


// ---- statistics of one 8192-logit slice held in registers ------------------
// Thread `tid` holds the canonical float4 vectors tid + 256 j (j = 0..7) of
// the slice starting at element `base` of a row of n logits.  Returns, valid on
// thread 0 only, the slice partial: (max, canonical exp2 sum) when SAMPLE, else
// (max, first index attaining it as int bits).  Two __syncthreads; the shared
// scratch may be reused by the next call right after it returns.
template <bool SAMPLE>
__device__ __forceinline__ float2 slice_partial(const float4 (&v)[8], int base, int n, float c) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool full = base + PSD_SLICE <= n;
  // exact slice max: lane -> warp (xor tree) -> block
  float lm = PSD_NEG_INF;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    lm = max3f(max3f(lm, v[j].x, v[j].y), v[j].z, v[j].w);
  float wm = lm;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) wm = psd_max(wm, __shfl_xor_sync(0xffffffffu, wm, off));
  __shared__ float s_max[kThreads / 32];
  __shared__ float s_sum[kThreads / 32];
  __shared__ int s_idx[kThreads / 32];
  if (lane == 0) s_max[warp] = wm;
  __syncthreads();
  float M = s_max[0];
#pragma unroll
  for (int q = 1; q < kThreads / 32; ++q) M = psd_max(M, s_max[q]);
  float2 res = make_float2(M, 0.0f);
  if constexpr (SAMPLE) {
    const float bias = psd_bias(M, c);
    const unsigned long long c2 = f2_pack(c, c), b2 = f2_pack(bias, bias);
    float s = 0.0f;
    auto lane_sum = [&](bool check) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        // elements past the row end (-inf or stale) are not part of it: skip
        const int e = base + 4 * (tid + kThreads * j);
        if (!check || e < n) {
          float wx, wy, wz, ww;
          psd_weight2(v[j].x, v[j].y, c2, b2, wx, wy);
          psd_weight2(v[j].z, v[j].w, c2, b2, wz, ww);
          s = psd_add(s, wx);
          s = psd_add(s, wy);
          s = psd_add(s, wz);
          s = psd_add(s, ww);
        }
      }
    };
    if (full) lane_sum(false);
    else lane_sum(true);
    s = shfl_add_tree(s);
    if (lane == 0) s_sum[warp] = s;
    __syncthreads();
    if (tid == 0) {
      float w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = s_sum[q];
#pragma unroll
      for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
        for (int q = 0; q < off; ++q) w[q] = psd_add(w[q], w[q + off]);
      res.y = w[0];
    }
  } else {
    // first (lowest) index attaining M
    int idx = 0x7fffffff;
    if (lm == M) {
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        const int e = base + 4 * (tid + kThreads * j);
        if (e < n) {
          if (v[j].w == M) idx = e + 3;
          if (v[j].z == M) idx = e + 2;
          if (v[j].y == M) idx = e + 1;
          if (v[j].x == M) idx = e;
        }
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) idx = min(idx, __shfl_xor_sync(0xffffffffu, idx, off));
    if (lane == 0) s_idx[warp] = idx;
    __syncthreads();
    if (tid == 0) {
      int w = s_idx[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) w = min(w, s_idx[q]);
      res.y = __int_as_float(w);
    }
  }
  return res;
}

// ---- fold + decision of request b -------------------------------------------
// Run by every thread of one CTA once all of b's slice partials are published
// (the statistics kernel completed).  Folds each row's slices left to right,
// tests all k_b drafts at once (lane i tests draft i; the first zero bit of the
// ballot is the first rejection) and returns, in shared memory, the plan of
// the sampling pass.  `publish`: this CTA writes accepted_len, the accepted
// tokens (and the greedy bonus token) and the target-row statistics.
template <bool SAMPLE>
__device__ void fold_decide(const Params& p, int b, bool publish, Plan* s_plan) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = p.len[b];
  __shared__ float2 s_part[(2 * PSD_MAX_K + 1) * PSD_MAX_SLICES];
  __shared__ float sMt[PSD_MAX_K + 1], sSt[PSD_MAX_K + 1], sMd[PSD_MAX_K], sSd[PSD_MAX_K];
  __shared__ int sG[PSD_MAX_K + 1];
  const int nst = (p.V + PSD_SLICE - 1) / PSD_SLICE;
  const int nsd = (p.Vd + PSD_SLICE - 1) / PSD_SLICE;
  const int nrows = SAMPLE && !p.d_stats ? 2 * kb + 1 : kb + 1;
  // the drafted tokens' raw logits: requested now so their (random, HBM)
  // loads overlap the partial staging and the fold below
  int x_tok = -1;
  float x_t = 0.0f, x_d = 0.0f;
  if (warp == 0 && lane < kb) {
    x_tok = p.ids[b * p.K + lane];
    if constexpr (SAMPLE) {
      if (x_tok >= 0 && x_tok < p.V) {
        x_t = __ldg(p.t + b * p.tsb + lane * p.tsi + x_tok);
        if (x_tok < p.Vd)
          x_d = __ldg(p.d + (int64_t)(p.d_rows ? p.d_rows[b] : b) * p.dsb + lane * p.dsi + x_tok);
      }
    }
  }
  // stage every partial of request b in shared memory (parallel loads)
  for (int q = tid; q < nrows * p.NS; q += kThreads) {
    const int rowi = q / p.NS, sl = q % p.NS;
    const int rr = rowi > kb ? p.K + 1 + (rowi - (kb + 1)) : rowi;
    s_part[q] = __ldcg(p.part + (b * p.R + rr) * p.NS + sl);
  }
  if constexpr (SAMPLE) {
    if (p.d_stats && tid < kb) {
      const float2 st = __ldcg(p.d_stats + (int64_t)(p.d_rows ? p.d_rows[b] : b) * p.d_stats_ld +
                               tid);
      sMd[tid] = st.x;
      sSd[tid] = st.y;
    }
  }
  __syncthreads();
  if (tid < nrows) {
    const bool dr = tid > kb;
    const int ri = dr ? tid - (kb + 1) : tid;
    const float2* pp = s_part + tid * p.NS;
    const int ns = dr ? nsd : nst;
    if constexpr (SAMPLE) {
      psd_ms a = {pp[0].x, pp[0].y};
      for (int q = 1; q < ns; ++q) a = psd_combine(a, psd_ms{pp[q].x, pp[q].y}, p.c);
      if (dr) { sMd[ri] = a.m; sSd[ri] = a.s; } else { sMt[ri] = a.m; sSt[ri] = a.s; }
    } else {
      psd_vi a = {pp[0].x, __float_as_int(pp[0].y)};
      for (int q = 1; q < ns; ++q) a = psd_argmax2(a, psd_vi{pp[q].x, __float_as_int(pp[q].y)});
      sG[ri] = a.i;
    }
  }
  __syncthreads();
  if (warp == 0) {
    bool ok = false;
    const int x = x_tok;
    if (lane < kb) {
      if constexpr (SAMPLE) {
        if (x >= 0 && x < p.V) {
          const float et = psd_weight(x_t, p.c, psd_bias(sMt[lane], p.c));
          const float ed = x < p.Vd ? psd_weight(x_d, p.c, psd_bias(sMd[lane], p.c)) : 0.0f;
          ok = psd_accept(p.u[b * (p.K + 1) + lane], et, ed, sSt[lane], sSd[lane]);
        }
      } else {
        ok = x == sG[lane];
      }
    }
    const unsigned rej = __ballot_sync(0xffffffffu, !ok) & ((1u << kb) - 1u);
    int a = rej ? __ffs(rej) - 1 : kb;
    if (p.forced) a = min(max(__ldg(p.forced + b), 0), kb);
    if (publish) {
      int32_t* o = p.out + b * (p.K + 1);
      if (lane <= p.K) o[lane] = lane < a ? x : (!SAMPLE && lane == a ? sG[a] : -1);
      if (lane == 0) {
        p.acc[b] = a;
        if constexpr (SAMPLE) {
          if (p.t_stats_out) {
            const int dst = p.t_stats_rows[b];
            if (dst >= 0) p.t_stats_out[dst] = make_float2(sMt[0], sSt[0]);
          }
        }
      }
    }
    if constexpr (SAMPLE) {
      if (lane == 0) {
        Plan pl;
        pl.row = a;
        pl.Mt = sMt[a]; pl.St = sSt[a];
        pl.mode = a < kb ? 1 : 2;
        pl.Md = a < kb ? sMd[a] : 0.0f;
        pl.Sd = a < kb ? sSd[a] : 0.0f;
        pl.pad[0] = pl.pad[1] = 0;
        *s_plan = pl;
      }
    }
  }
  __syncthreads();
}

// ---- statistics pass ----------------------------------------------------------
// One (request b, row r, slice) item per CTA: 8192 logits streamed once with
// 128-bit L1-bypassing loads (all eight vectors of a thread in flight at once),
// the canonical slice partial written to the workspace.  No completion
// tracking: the fold / decision runs in the next kernel (verify_fold, or
// inside verify_sample), which a stream (PDL) dependency orders after this
// one.  Measured against the ticketed variant (the last CTA of a request folds
// and decides) and a persistent TMA-bulk-copy variant: profiles/r02_k1_variants.txt.
template <bool SAMPLE>
__global__ void __launch_bounds__(kThreads)
verify_stats(const Params p) {
  pdl_wait();
  pdl_trigger();
  const int slice = blockIdx.x, b = blockIdx.y / p.R, r = blockIdx.y % p.R;
  const int kb = p.len[b];
  const bool is_draft = r > p.K;
  const int i = is_draft ? r - (p.K + 1) : r;
  const int n = is_draft ? p.Vd : p.V;
  const bool active = (is_draft ? i < kb && !p.d_stats : i <= kb) && slice * PSD_SLICE < n;
  if (!active) return;
  const int db = p.d_rows ? p.d_rows[b] : b;
  const float* row = is_draft ? p.d + db * p.dsb + i * p.dsi : p.t + b * p.tsb + i * p.tsi;
  const int tid = threadIdx.x;
  const int base = slice * PSD_SLICE;
  float4 v[8];
  if (base + PSD_SLICE <= n) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ld_stream(row + base + 4 * (tid + kThreads * j));
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = base + 4 * (tid + kThreads * j);
      v[j] = e < n ? ld_stream(row + e)
                   : make_float4(PSD_NEG_INF, PSD_NEG_INF, PSD_NEG_INF, PSD_NEG_INF);
    }
  }
  float2 part = slice_partial<SAMPLE>(v, base, n, p.c);
  if (!SAMPLE && p.voff && __float_as_int(part.y) != 0x7fffffff)
    part.y = __int_as_float(__float_as_int(part.y) + p.voff);
  if (tid == 0) p.part[(b * p.R + r) * p.NS + slice] = part;
}

// greedy over W vocabulary shards (tensor-parallel LM head):
// partials [W][B][K+1][NS] (max, global argmax index); one CTA per request,
// row r folded by thread r (argmax: any order, ties -> lowest index), then
// the same ballot test as verify_fold.  Every rank runs it on the gathered
// partials and reaches the same decision.
__global__ void __launch_bounds__(kThreads)
verify_fold_sharded(const Params p, int W) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = p.len[b];
  __shared__ int sG[PSD_MAX_K + 1];
  if (tid <= kb) {
    psd_vi a = {PSD_NEG_INF, 0x7fffffff};
    const size_t per_w = (size_t)p.B * p.R * p.NS;
    for (int w = 0; w < W; ++w)
      for (int q = 0; q < p.NS; ++q) {
        const float2 v = __ldcg(p.part + w * per_w + ((size_t)b * p.R + tid) * p.NS + q);
        if (__float_as_int(v.y) != 0x7fffffff) a = psd_argmax2(a, psd_vi{v.x, __float_as_int(v.y)});
      }
    sG[tid] = a.i;
  }
  __syncthreads();
  if (warp == 0) {
    const int x = lane < kb ? p.ids[b * p.K + lane] : -1;
    const bool ok = lane < kb && x == sG[lane];
    const unsigned rej = __ballot_sync(0xffffffffu, !ok) & ((1u << kb) - 1u);
    int a = rej ? __ffs(rej) - 1 : kb;
    if (p.forced) a = min(max(__ldg(p.forced + b), 0), kb);
    int32_t* o = p.out + b * (p.K + 1);
    if (lane <= p.K) o[lane] = lane < a ? x : (lane == a ? sG[a] : -1);
    if (lane == 0) p.acc[b] = a;
  }
}

// greedy from per-row argmax tokens (the target LM head's K6 epilogue +
// argmax fold): one warp per request, the same ballot test and outputs as
// verify_fold / verify_fold_sharded
__global__ void __launch_bounds__(32)
verify_accept_tokens(const int32_t* __restrict__ tok, const Params p) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x, lane = threadIdx.x;
  const int kb = p.len[b];
  const int* g = tok + (size_t)b * (p.K + 1);
  const int x = lane < kb ? p.ids[b * p.K + lane] : -1;
  const bool ok = lane < kb && x == g[lane];
  const unsigned rej = __ballot_sync(0xffffffffu, !ok) & ((1u << kb) - 1u);
  int a = rej ? __ffs(rej) - 1 : kb;
  if (p.forced) a = min(max(__ldg(p.forced + b), 0), kb);
  int32_t* o = p.out + b * (p.K + 1);
  if (lane <= p.K) o[lane] = lane < a ? x : (lane == a ? g[a] : -1);
  if (lane == 0) p.acc[b] = a;
}

// greedy: fold + decide, one CTA per request
__global__ void __launch_bounds__(kThreads)
verify_fold(const Params p) {
  pdl_wait();
  pdl_trigger();
  fold_decide<false>(p, blockIdx.x, true, nullptr);
}

// ---- sampling pass ---------------------------------------------------------
// Grid (chunk of kChunkBlks 1024-element blocks, request).  Each thread owns
// elements 4l..4l+3 of every block of its chunk (the canonical lane layout),
// loads all of them up front (128-bit loads, target and draft rows), evaluates
// the weights with packed f32x2 math (bit-identical to psd_canon.h) and reduces
// every block with the canonical warp tree + 8-warp tree.  The last chunk of a
// request (atomic ticket) runs the canonical prefix search.
constexpr int kChunkBlks = 8;  // 1024-element blocks per sampling item
constexpr int kSubBlks = 4;    // blocks loaded at once (register budget)

struct WeightCtx {
  const float* t; const float* d; int V, Vd; float c, bt, bd, St, Sd; int residual;
};

__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// weights of the 4 elements x0..x0+3 (x0 % 4 == 0; V, Vd multiples of 4)
__device__ __forceinline__ void weights4(const WeightCtx& w, int x0, float4 tv, float4 dv,
                                         float out[4]) {
  if (x0 >= w.V) {
    out[0] = out[1] = out[2] = out[3] = 0.0f;
    return;
  }
  const unsigned long long c2 = f2_pack(w.c, w.c), bt2 = f2_pack(w.bt, w.bt);
  float e[4];
  psd_weight2(tv.x, tv.y, c2, bt2, e[0], e[1]);
  psd_weight2(tv.z, tv.w, c2, bt2, e[2], e[3]);
  if (!w.residual) {
    out[0] = e[0]; out[1] = e[1]; out[2] = e[2]; out[3] = e[3];
    return;
  }
  float q[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  if (x0 < w.Vd) {
    const unsigned long long bd2 = f2_pack(w.bd, w.bd);
    psd_weight2(dv.x, dv.y, c2, bd2, q[0], q[1]);
    psd_weight2(dv.z, dv.w, c2, bd2, q[2], q[3]);
  }
  // psd_residual: max(0, fl(fl(e_t * S_d) - fl(e_d * S_t)))
  const unsigned long long Sd2 = f2_pack(w.Sd, w.Sd), St2 = f2_pack(w.St, w.St);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const unsigned long long r2 = f2_sub(f2_mul(f2_pack(e[2 * h], e[2 * h + 1]), Sd2),
                                         f2_mul(f2_pack(q[2 * h], q[2 * h + 1]), St2));
    float r0, r1;
    f2_unpack(r2, r0, r1);
    out[2 * h] = r0 > 0.0f ? r0 : 0.0f;
    out[2 * h + 1] = r1 > 0.0f ? r1 : 0.0f;
  }
}

__device__ __forceinline__ void load4(const WeightCtx& w, int x0, float4& tv, float4& dv) {
  tv = make_float4(0.f, 0.f, 0.f, 0.f);
  dv = tv;
  if (x0 < w.V) tv = __ldg(reinterpret_cast<const float4*>(w.t + x0));
  if (w.residual && x0 < w.Vd) dv = __ldg(reinterpret_cast<const float4*>(w.d + x0));
}

// canonical block sums of blocks blk0 .. blk0+nb-1 (nb <= kSubBlks); all
// kThreads threads call it; results land in s_blk[0..nb) (valid after return)
__device__ void chunk_block_sums(const WeightCtx& w, int blk0, int nb, float* s_red,
                                 float* s_blk) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float4 tv[kSubBlks], dv[kSubBlks];
#pragma unroll
  for (int k = 0; k < kSubBlks; ++k)
    if (k < nb) load4(w, (blk0 + k) * PSD_SBLK + 4 * tid, tv[k], dv[k]);
#pragma unroll
  for (int k = 0; k < kSubBlks; ++k) {
    if (k < nb) {
      float wv[4];
      weights4(w, (blk0 + k) * PSD_SBLK + 4 * tid, tv[k], dv[k], wv);
      const float ls = psd_add(psd_add(psd_add(wv[0], wv[1]), wv[2]), wv[3]);
      const float ws = shfl_add_tree(ls);
      if (lane == 0) s_red[k * 8 + warp] = ws;
    }
  }
  __syncthreads();
  if (tid < nb) {
    float q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = s_red[tid * 8 + k];
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
      for (int k = 0; k < off; ++k) q[k] = psd_add(q[k], q[k + off]);
    s_blk[tid] = q[0];
  }
  __syncthreads();
}

// last element with positive weight in block blk (all threads return it)
__device__ int last_positive(const WeightCtx& w, int blk, int* s_int) {
  float4 tv, dv;
  const int x0 = blk * PSD_SBLK + 4 * threadIdx.x;
  load4(w, x0, tv, dv);
  float wv[4];
  weights4(w, x0, tv, dv, wv);
  int best = -1;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (wv[c] > 0.0f) best = x0 + c;
  if (threadIdx.x == 0) *s_int = -1;
  __syncthreads();
  if (best >= 0) atomicMax(s_int, best);
  __syncthreads();
  const int r = *s_int;
  __syncthreads();
  return r < 0 ? blk * PSD_SBLK : r;
}

// Sequential left fold of v[0..n) (one thread): prefix[i] = v[0] + ... + v[i-1]
// (prefix[0] = 0, prefix[n] = total) when prefix != nullptr; returns the total.
// Values are pulled from shared memory 32 at a time with 128-bit loads so the
// add chain, not the load latency, sets the pace.
__device__ float seq_fold(const float* v, int n, float* prefix) {
  float C = 0.0f;
  if (prefix) prefix[0] = 0.0f;
  int i = 0;
  for (; i + 32 <= n; i += 32) {
    float4 q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = reinterpret_cast<const float4*>(v + i)[j];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      C = psd_add(C, q[j].x); if (prefix) prefix[i + 4 * j + 1] = C;
      C = psd_add(C, q[j].y); if (prefix) prefix[i + 4 * j + 2] = C;
      C = psd_add(C, q[j].z); if (prefix) prefix[i + 4 * j + 3] = C;
      C = psd_add(C, q[j].w); if (prefix) prefix[i + 4 * j + 4] = C;
    }
  }
  for (; i < n; ++i) {
    C = psd_add(C, v[i]);
    if (prefix) prefix[i + 1] = C;
  }
  return C;
}

// one chunk of request b's sampling pass; the last chunk runs the prefix search
__device__ __forceinline__ void sample_item(const Params& p, int chunk, int b, int nchunks) {
  const int tid = threadIdx.x;
  // every chunk CTA folds request b's statistics and decides (cheap, and no
  // completion tracking in the statistics pass); chunk 0 publishes the result
  __shared__ Plan s_plan;
  fold_decide<true>(p, b, chunk == 0, &s_plan);
  const Plan pl = s_plan;
  WeightCtx w;
  w.V = p.V; w.Vd = p.Vd; w.c = p.c;
  w.t = p.t + b * p.tsb + pl.row * p.tsi;
  w.d = p.d + (int64_t)(p.d_rows ? p.d_rows[b] : b) * p.dsb + pl.row * p.dsi;
  w.bt = psd_bias(pl.Mt, p.c); w.bd = psd_bias(pl.Md, p.c); w.St = pl.St; w.Sd = pl.Sd;
  w.residual = pl.mode == 1;

  __shared__ float s_red[kSubBlks * 8];
  __shared__ float s_blk[kSubBlks];
  __shared__ __align__(16) float s_lane[kThreads];
  __shared__ int s_last, s_int;
  __shared__ float s_T;
  __shared__ int s_chosen;
  __shared__ __align__(16) float wb[PSD_MAX_SBLKS];
  __shared__ __align__(16) float s_pref[PSD_MAX_SBLKS + 1];
  __shared__ __align__(16) float s_lpre[kThreads + 1];

  for (int sub = 0; sub < kChunkBlks; sub += kSubBlks) {
    const int blk0 = chunk * kChunkBlks + sub;
    const int nb = min(kSubBlks, p.NB - blk0);
    if (nb <= 0) break;
    chunk_block_sums(w, blk0, nb, s_red, s_blk);
    if (tid < nb) p.wblk[b * p.NB + blk0 + tid] = s_blk[tid];
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(p.cnt_b + b, 1) == nchunks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int k = tid; k < p.NB; k += kThreads) wb[k] = __ldcg(p.wblk + b * p.NB + k);
  __syncthreads();

  // canonical block prefix P_b (sequential fold, kept in smem), T = u * R;
  // chosen block = first with P_b > T (found in parallel).  A degenerate
  // residual (sums to 0 in fp32) falls back to sampling from p: the block sums
  // of p, then the same fold
  if (tid == 0) {
    const float R = seq_fold(wb, p.NB, s_pref);
    s_int = (w.residual && !(R > 0.0f)) ? 1 : 0;
    s_T = psd_mul(p.u[b * (p.K + 1) + p.K], R);
    s_chosen = 0x7fffffff;
  }
  __syncthreads();
  if (s_int) {
    w.residual = 0;
    for (int k0 = 0; k0 < p.NB; k0 += kSubBlks) {
      const int n = min(kSubBlks, p.NB - k0);
      chunk_block_sums(w, k0, n, s_red, s_blk);
      if (tid < n) wb[k0 + tid] = s_blk[tid];
    }
    __syncthreads();
    if (tid == 0) {
      const float R = seq_fold(wb, p.NB, s_pref);
      s_T = psd_mul(p.u[b * (p.K + 1) + p.K], R);
    }
    __syncthreads();
  }
  for (int k = tid; k < p.NB; k += kThreads)
    if (s_pref[k + 1] > s_T) atomicMin(&s_chosen, k);
  __syncthreads();
  int tok;
  if (s_chosen == 0x7fffffff) {
    // no block hit (rounding): last positive-weight block
    if (tid == 0) {
      int lb = p.NB - 1;
      for (int k = p.NB - 1; k >= 0; --k)
        if (wb[k] > 0.0f) { lb = k; break; }
      s_int = lb;
    }
    __syncthreads();
    tok = last_positive(w, s_int, &s_int);
  } else {
    const int cb = s_chosen;
    const float Pprev = s_pref[cb];
    const int x0 = cb * PSD_SBLK + 4 * tid;
    float4 tv, dv;
    load4(w, x0, tv, dv);
    float wv[4];
    weights4(w, x0, tv, dv, wv);
    s_lane[tid] = psd_add(psd_add(psd_add(wv[0], wv[1]), wv[2]), wv[3]);
    __syncthreads();
    if (tid == 0) {  // exclusive sequential prefix of the lane sums
      seq_fold(s_lane, kThreads, s_lpre);
      s_int = 0x7fffffff;
    }
    __syncthreads();
    float acc = s_lpre[tid];
    int hit = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc = psd_add(acc, wv[c]);
      if (hit == 0x7fffffff && psd_add(Pprev, acc) > s_T) hit = x0 + c;
    }
    if (hit != 0x7fffffff) atomicMin(&s_int, hit);
    __syncthreads();
    tok = s_int;
    __syncthreads();
    if (tok == 0x7fffffff) tok = last_positive(w, cb, &s_int);
  }
  if (tid == 0) {
    p.out[b * (p.K + 1) + pl.row] = tok;
    p.cnt_b[b] = 0;
  }
}

__global__ void __launch_bounds__(kThreads)
verify_sample(const Params p) {
  pdl_wait();
  pdl_trigger();
  sample_item(p, blockIdx.x, blockIdx.y, gridDim.x);
}


size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }


template <bool SAMPLE>
cudaError_t launch_stats(const Params& p, cudaStream_t st) {
  dim3 grid(p.NS, p.B * p.R);
  return psd::launch(verify_stats<SAMPLE>, grid, dim3(kThreads), 0, st, p);
}

cudaError_t launch_greedy(const Params& p, cudaStream_t st) {
  cudaError_t e = launch_stats<false>(p, st);
  if (e != cudaSuccess) return e;
  return psd::launch(verify_fold, dim3(p.B), dim3(kThreads), 0, st, p);
}

cudaError_t launch_sampling(const Params& p, cudaStream_t st) {
  cudaError_t e = launch_stats<true>(p, st);
  if (e != cudaSuccess) return e;
  const int nc = (p.NB + kChunkBlks - 1) / kChunkBlks;
  return psd::launch(verify_sample, dim3(nc, p.B), dim3(kThreads), 0, st, p);
}

struct WsLayout {
  size_t cnt_b, part, wblk, total;
};

WsLayout layout(int B, int K, int V, int Vd, int sampling) {
  const int nmax = V > Vd ? V : Vd;
  const int NS = (nmax + PSD_SLICE - 1) / PSD_SLICE;
  const int NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  const int R = (K + 1) + (sampling ? K : 0);
  WsLayout L;
  size_t off = 0;
  L.cnt_b = off; off = align_up(off + sizeof(int) * B);
  L.part = off; off = align_up(off + sizeof(float2) * (size_t)B * R * NS);
  L.wblk = off; off = align_up(off + sizeof(float) * (size_t)B * NB);
  L.total = off;
  return L;
}

int check_common(const float* t, int64_t tsb, int64_t tsi, int V, int B, int K,
                 const void* ws, size_t ws_bytes, size_t need) {
  if (!t || V <= 0 || B <= 0 || K < 0 || K > PSD_MAX_K) return (int)cudaErrorInvalidValue;
  if (V > PSD_MAX_SLICES * PSD_SLICE) return (int)cudaErrorInvalidValue;
  if ((V & 3) || (tsb & 3) || (tsi & 3) || (reinterpret_cast<uintptr_t>(t) & 15))
    return (int)cudaErrorMisalignedAddress;
  if (!ws || ws_bytes < need) return (int)cudaErrorInvalidValue;
  return 0;
}

}  // namespace

extern "C" {

size_t psd_verify_workspace_bytes(int B, int K, int V, int Vd, int sampling) {
  return layout(B, K, V, sampling ? Vd : 0, sampling).total;
}

int psd_verify_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  return (int)cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream);
}

int psd_verify_greedy(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i, int V,
                      const int32_t* draft_ids, const int32_t* draft_len, int B, int K,
                      int32_t* accepted_len, int32_t* out_tokens, void* ws, size_t ws_bytes,
                      void* stream) {
  return psd_verify_greedy_forced(target_logits, t_stride_b, t_stride_i, V, draft_ids, draft_len,
                                  B, K, nullptr, accepted_len, out_tokens, ws, ws_bytes, stream);
}

size_t psd_verify_partials_count(int B, int K, int V) {
  return (size_t)B * (K + 1) * ((V + PSD_SLICE - 1) / PSD_SLICE) * 2;
}

int psd_verify_greedy_partials(const float* target_logits, int64_t t_stride_b,
                               int64_t t_stride_i, int V, int vocab_offset,
                               const int32_t* draft_len, int B, int K, float* partials,
                               void* stream) {
  if (!partials) return (int)cudaErrorInvalidValue;
  int rc = check_common(target_logits, t_stride_b, t_stride_i, V, B, K, partials, 1, 0);
  if (rc) return rc;
  Params p{};
  p.t = target_logits; p.tsb = t_stride_b; p.tsi = t_stride_i; p.V = V; p.len = draft_len;
  p.c = psd_scale(1.0f); p.B = B; p.K = K; p.voff = vocab_offset;
  p.part = reinterpret_cast<float2*>(partials);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK; p.R = K + 1;
  return (int)launch_stats<false>(p, (cudaStream_t)stream);
}

int psd_verify_greedy_fold(const float* partials, int W, int V_shard, const int32_t* draft_ids,
                           const int32_t* draft_len, int B, int K, const int32_t* forced_len,
                           int32_t* accepted_len, int32_t* out_tokens, void* stream) {
  if (!partials || W < 1 || V_shard <= 0 || B <= 0 || K < 0 || K > PSD_MAX_K)
    return (int)cudaErrorInvalidValue;
  Params p{};
  p.ids = draft_ids; p.len = draft_len; p.B = B; p.K = K; p.forced = forced_len;
  p.acc = accepted_len; p.out = out_tokens;
  p.part = reinterpret_cast<float2*>(const_cast<float*>(partials));
  p.NS = (V_shard + PSD_SLICE - 1) / PSD_SLICE; p.R = K + 1;
  return (int)psd::launch(verify_fold_sharded, dim3(B), dim3(kThreads), 0, (cudaStream_t)stream,
                          p, W);
}

int psd_verify_greedy_tokens(const int32_t* argmax_tokens, const int32_t* draft_ids,
                             const int32_t* draft_len, int B, int K, const int32_t* forced_len,
                             int32_t* accepted_len, int32_t* out_tokens, void* stream) {
  if (!argmax_tokens || B <= 0 || K < 0 || K > PSD_MAX_K || (K > 0 && !draft_ids) ||
      !draft_len || !accepted_len || !out_tokens)
    return (int)cudaErrorInvalidValue;
  Params p{};
  p.ids = draft_ids; p.len = draft_len; p.B = B; p.K = K; p.forced = forced_len;
  p.acc = accepted_len; p.out = out_tokens;
  return (int)psd::launch(verify_accept_tokens, dim3(B), dim3(32), 0, (cudaStream_t)stream,
                          argmax_tokens, p);
}

int psd_verify_greedy_forced(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                             int V, const int32_t* draft_ids, const int32_t* draft_len, int B,
                             int K, const int32_t* forced_len, int32_t* accepted_len,
                             int32_t* out_tokens, void* ws, size_t ws_bytes, void* stream) {
  const WsLayout L = layout(B, K, V, 0, 0);
  int rc = check_common(target_logits, t_stride_b, t_stride_i, V, B, K, ws, ws_bytes, L.total);
  if (rc) return rc;
  Params p{};
  char* w = static_cast<char*>(ws);
  p.t = target_logits; p.tsb = t_stride_b; p.tsi = t_stride_i; p.V = V;
  p.d = nullptr; p.Vd = 0; p.ids = draft_ids; p.len = draft_len; p.u = nullptr;
  p.c = psd_scale(1.0f); p.B = B; p.K = K; p.acc = accepted_len; p.out = out_tokens;
  p.forced = forced_len;
  p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK; p.R = K + 1;
  return (int)launch_greedy(p, (cudaStream_t)stream);
}

int psd_verify_sample(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i, int V,
                      const float* draft_logits, int64_t d_stride_b, int64_t d_stride_i, int Vd,
                      const int32_t* draft_ids, const int32_t* draft_len, const float* uniforms,
                      float temperature, int B, int K, int32_t* accepted_len,
                      int32_t* out_tokens, void* ws, size_t ws_bytes, void* stream) {
  const WsLayout L = layout(B, K, V, Vd, 1);
  int rc = check_common(target_logits, t_stride_b, t_stride_i, V, B, K, ws, ws_bytes, L.total);
  if (rc) return rc;
  if (!draft_logits || Vd <= 0 || Vd > V || !uniforms || !(temperature > 0.0f))
    return (int)cudaErrorInvalidValue;
  if ((Vd & 3) || (d_stride_b & 3) || (d_stride_i & 3) ||
      (reinterpret_cast<uintptr_t>(draft_logits) & 15))
    return (int)cudaErrorMisalignedAddress;
  Params p{};
  char* w = static_cast<char*>(ws);
  p.t = target_logits; p.tsb = t_stride_b; p.tsi = t_stride_i; p.V = V;
  p.d = draft_logits; p.dsb = d_stride_b; p.dsi = d_stride_i; p.Vd = Vd;
  p.ids = draft_ids; p.len = draft_len; p.u = uniforms;
  p.c = psd_scale(1.0f / temperature); p.B = B; p.K = K; p.acc = accepted_len; p.out = out_tokens;
  p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  p.R = 2 * K + 1;
  return (int)launch_sampling(p, (cudaStream_t)stream);
}

int psd_verify_sample_rows(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                           int V, const float* draft_logits, const int32_t* draft_rows,
                           int64_t d_stride_row, int64_t d_stride_i, int Vd,
                      const int32_t* draft_ids, const int32_t* draft_len, const float* uniforms,
                      float temperature, int B, int K, int32_t* accepted_len,
                      int32_t* out_tokens, void* ws, size_t ws_bytes, void* stream) {
  return psd_verify_sample_ext(target_logits, t_stride_b, t_stride_i, V, draft_logits, draft_rows,
                               d_stride_row, d_stride_i, Vd, draft_ids, draft_len, uniforms,
                               temperature, B, K, accepted_len, out_tokens, nullptr, 0, nullptr,
                               nullptr, ws, ws_bytes, stream);
}

int psd_verify_sample_ext(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                          int V, const float* draft_logits, const int32_t* draft_rows,
                          int64_t d_stride_row, int64_t d_stride_i, int Vd,
                          const int32_t* draft_ids, const int32_t* draft_len,
                          const float* uniforms, float temperature, int B, int K,
                          int32_t* accepted_len, int32_t* out_tokens, const void* d_stats,
                          int64_t d_stats_ld, void* t_stats_out, const int32_t* t_stats_rows,
                          void* ws, size_t ws_bytes, void* stream) {
  return psd_verify_sample_forced(target_logits, t_stride_b, t_stride_i, V, draft_logits,
                                  draft_rows, d_stride_row, d_stride_i, Vd, draft_ids, draft_len,
                                  uniforms, temperature, B, K, nullptr, accepted_len, out_tokens,
                                  d_stats, d_stats_ld, t_stats_out, t_stats_rows, ws, ws_bytes,
                                  stream);
}

int psd_verify_sample_forced(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                             int V, const float* draft_logits, const int32_t* draft_rows,
                             int64_t d_stride_row, int64_t d_stride_i, int Vd,
                             const int32_t* draft_ids, const int32_t* draft_len,
                             const float* uniforms, float temperature, int B, int K,
                             const int32_t* forced_len, int32_t* accepted_len,
                             int32_t* out_tokens, const void* d_stats, int64_t d_stats_ld,
                             void* t_stats_out, const int32_t* t_stats_rows, void* ws,
                             size_t ws_bytes, void* stream) {
  if (t_stats_out && !t_stats_rows) return (int)cudaErrorInvalidValue;
  const WsLayout L = layout(B, K, V, Vd, 1);
  int rc = check_common(target_logits, t_stride_b, t_stride_i, V, B, K, ws, ws_bytes, L.total);
  if (rc) return rc;
  if (!draft_logits || Vd <= 0 || Vd > V || !uniforms || !(temperature > 0.0f))
    return (int)cudaErrorInvalidValue;
  if ((Vd & 3) || (d_stride_row & 3) || (d_stride_i & 3) ||
      (reinterpret_cast<uintptr_t>(draft_logits) & 15))
    return (int)cudaErrorMisalignedAddress;
  Params p{};
  char* w = static_cast<char*>(ws);
  p.t = target_logits; p.tsb = t_stride_b; p.tsi = t_stride_i; p.V = V;
  p.d = draft_logits; p.dsb = d_stride_row; p.dsi = d_stride_i; p.Vd = Vd;
  p.d_rows = draft_rows;
  p.d_stats = static_cast<const float2*>(d_stats);
  p.d_stats_ld = d_stats_ld;
  p.t_stats_out = static_cast<float2*>(t_stats_out);
  p.t_stats_rows = t_stats_rows;
  p.forced = forced_len;
  p.ids = draft_ids; p.len = draft_len; p.u = uniforms;
  p.c = psd_scale(1.0f / temperature); p.B = B; p.K = K; p.acc = accepted_len; p.out = out_tokens;
  p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  p.R = 2 * K + 1;
  return (int)launch_sampling(p, (cudaStream_t)stream);
}

}  // extern "C"
