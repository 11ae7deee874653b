// verify.cu -- K1: fused speculative verification on sm_100a.
//
// Replaces the reference's coin-flip acceptance (pkg/src/specsim/
// acceptance_model.py:82-97, called from engine.py:245-256) with the real
// token-level rule over target / draft logits.  Bit-exact with the CPU oracle
// (oracle/verify_oracle.c) because both evaluate include/psd_canon.h in the
// canonical order documented there.
//
// Two kernels, HBM-bound by design:
//   verify_stats<SAMPLE>  grid (slice, request*row): every active (row, slice)
//       streams 8192 fp32 logits once with 128-bit L1-bypassing loads and
//       produces (max, sum-exp) [sampling] or (max, argmax) [greedy] partials;
//       the last CTA of each request (atomic ticket) folds the slices, runs the
//       accept test of all k drafts at once (one lane per draft, __ballot_sync
//       finds the first rejection) and writes the accepted prefix.  Greedy is
//       done after this kernel.
//   verify_sample         grid (1024-block, request): block sums of the
//       residual max(0, p - q) (or p for the bonus), the last CTA per request
//       does the normalised prefix search and writes the final token.
// Algorithmic bytes: greedy 4V*sum(k_b+1); sampling
// 4V*sum(2k_b+1) (+ small terms).  The sampling pass re-reads one (t, d) row
// pair per request (mostly from L2).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/psd.h"
#include "common.h"
#include "../../include/psd_canon.h"

namespace {

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
  int* cnt_a; int* cnt_b;
  float2* part; Plan* plan; float* wblk;
  int NS, NB, R;
};

__device__ __forceinline__ float4 ld_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ psd_ms shfl_ms(psd_ms v, int off) {
  psd_ms o;
  o.m = __shfl_down_sync(0xffffffffu, v.m, off);
  o.s = __shfl_down_sync(0xffffffffu, v.s, off);
  return o;
}

__device__ __forceinline__ psd_vi shfl_vi(psd_vi v, int off) {
  psd_vi o;
  o.v = __shfl_down_sync(0xffffffffu, v.v, off);
  o.i = __shfl_down_sync(0xffffffffu, v.i, off);
  return o;
}

__device__ __forceinline__ float shfl_add_tree(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = psd_add(v, __shfl_down_sync(0xffffffffu, v, off));
  return v;
}

// number of stats CTAs request b launches work in
__device__ __forceinline__ int expected_stats(const Params& p, int kb, bool sample) {
  const int nst = (p.V + PSD_SLICE - 1) / PSD_SLICE;
  const int nsd = (p.Vd + PSD_SLICE - 1) / PSD_SLICE;
  return nst * (kb + 1) + (sample ? nsd * kb : 0);
}

template <bool SAMPLE>
__global__ void __launch_bounds__(kThreads)
verify_stats(const Params p) {
  pdl_wait();
  pdl_trigger();
  const int slice = blockIdx.x;
  const int b = blockIdx.y / p.R;
  const int r = blockIdx.y % p.R;
  const int kb = p.len[b];
  const bool is_draft = r > p.K;
  const int i = is_draft ? r - (p.K + 1) : r;
  const int n = is_draft ? p.Vd : p.V;
  const bool active = (is_draft ? i < kb : i <= kb) && slice * PSD_SLICE < n;
  if (!active) return;
  const int db = p.d_rows ? p.d_rows[b] : b;
  const float* row = is_draft ? p.d + db * p.dsb + i * p.dsi : p.t + b * p.tsb + i * p.tsi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int base = slice * PSD_SLICE;

  float4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int e = base + 4 * (tid + kThreads * j);
    v[j] = e < n ? ld_stream(row + e)
                 : make_float4(PSD_NEG_INF, PSD_NEG_INF, PSD_NEG_INF, PSD_NEG_INF);
  }
  // exact slice max: lane -> warp (xor tree) -> block
  float lm = PSD_NEG_INF;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    lm = psd_max(lm, psd_max(psd_max(v[j].x, v[j].y), psd_max(v[j].z, v[j].w)));
  float wm = lm;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) wm = psd_max(wm, __shfl_xor_sync(0xffffffffu, wm, off));
  __shared__ float s_max[kThreads / 32];
  __shared__ float s_sum[kThreads / 32];
  __shared__ int s_idx[kThreads / 32];
  __shared__ int s_last;
  if (lane == 0) s_max[warp] = wm;
  __syncthreads();
  float M = s_max[0];
#pragma unroll
  for (int q = 1; q < kThreads / 32; ++q) M = psd_max(M, s_max[q]);

  if constexpr (SAMPLE) {
    const float bias = psd_bias(M, p.c);
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // invalid elements (-inf) are not part of the row: skip them
      const int e = base + 4 * (tid + kThreads * j);
      if (e < n) {
        s = psd_add(s, psd_weight(v[j].x, p.c, bias));
        s = psd_add(s, psd_weight(v[j].y, p.c, bias));
        s = psd_add(s, psd_weight(v[j].z, p.c, bias));
        s = psd_add(s, psd_weight(v[j].w, p.c, bias));
      }
    }
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
      p.part[(b * p.R + r) * p.NS + slice] = make_float2(M, w[0]);
    }
  } else {
    // first (lowest) index attaining M
    int idx = 0x7fffffff;
    if (lm == M) {
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        const int e = base + 4 * (tid + kThreads * j);
        if (v[j].w == M) idx = e + 3;
        if (v[j].z == M) idx = e + 2;
        if (v[j].y == M) idx = e + 1;
        if (v[j].x == M) idx = e;
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
      p.part[(b * p.R + r) * p.NS + slice] = make_float2(M, __int_as_float(w));
    }
  }

  // ---- last CTA of request b: fold slices, decide --------------------------
  if (tid == 0) {
    __threadfence();
    const int ticket = atomicAdd(p.cnt_a + b, 1);
    s_last = ticket == expected_stats(p, kb, SAMPLE) - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  __shared__ float2 s_part[(2 * PSD_MAX_K + 1) * PSD_MAX_SLICES];
  __shared__ float sMt[PSD_MAX_K + 1], sSt[PSD_MAX_K + 1], sMd[PSD_MAX_K], sSd[PSD_MAX_K];
  __shared__ int sG[PSD_MAX_K + 1];
  const int nst = (p.V + PSD_SLICE - 1) / PSD_SLICE;
  const int nsd = (p.Vd + PSD_SLICE - 1) / PSD_SLICE;
  const int nrows = SAMPLE ? 2 * kb + 1 : kb + 1;
  // stage every partial of request b in shared memory (parallel loads)
  for (int q = tid; q < nrows * p.NS; q += kThreads) {
    const int rowi = q / p.NS, sl = q % p.NS;
    const int rr = rowi > kb ? p.K + 1 + (rowi - (kb + 1)) : rowi;
    s_part[q] = __ldcg(p.part + (b * p.R + rr) * p.NS + sl);
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
    // lane i tests draft i; first rejection = first zero bit of the ballot
    bool ok = false;
    const int x = lane < kb ? p.ids[b * p.K + lane] : -1;
    if (lane < kb) {
      if constexpr (SAMPLE) {
        if (x >= 0 && x < p.V) {
          const float* tr = p.t + b * p.tsb + lane * p.tsi;
          const float* drw = p.d + (int64_t)(p.d_rows ? p.d_rows[b] : b) * p.dsb + lane * p.dsi;
          const float et = psd_weight(__ldg(tr + x), p.c, psd_bias(sMt[lane], p.c));
          const float ed =
              x < p.Vd ? psd_weight(__ldg(drw + x), p.c, psd_bias(sMd[lane], p.c)) : 0.0f;
          ok = psd_accept(p.u[b * (p.K + 1) + lane], et, ed, sSt[lane], sSd[lane]);
        }
      } else {
        ok = x == sG[lane];
      }
    }
    const unsigned rej = __ballot_sync(0xffffffffu, !ok) & ((1u << kb) - 1u);
    const int a = rej ? __ffs(rej) - 1 : kb;
    int32_t* o = p.out + b * (p.K + 1);
    if (lane <= p.K) o[lane] = lane < a ? x : (!SAMPLE && lane == a ? sG[a] : -1);
    if (lane == 0) {
      p.acc[b] = a;
      if constexpr (SAMPLE) {
        Plan pl;
        pl.row = a;
        pl.Mt = sMt[a]; pl.St = sSt[a];
        pl.mode = a < kb ? 1 : 2;
        pl.Md = a < kb ? sMd[a] : 0.0f;
        pl.Sd = a < kb ? sSd[a] : 0.0f;
        pl.pad[0] = pl.pad[1] = 0;
        p.plan[b] = pl;
      }
      p.cnt_a[b] = 0;  // self-cleaning ticket for the next launch
    }
  }
}

// ---- sampling pass ---------------------------------------------------------
struct WeightCtx {
  const float* t; const float* d; int V, Vd; float c, bt, bd, St, Sd; int residual;
};

__device__ __forceinline__ float weight_of(const WeightCtx& w, float tv, float dv, int x) {
  if (x >= w.V) return 0.0f;
  const float et = psd_weight(tv, w.c, w.bt);
  if (!w.residual) return et;
  const float ed = x < w.Vd ? psd_weight(dv, w.c, w.bd) : 0.0f;
  return psd_residual(et, ed, w.St, w.Sd);
}

// weights of the 4 elements lane `tid` owns in block `blk`
__device__ __forceinline__ void lane_weights(const WeightCtx& w, int blk, int tid, float out[4]) {
  const int x0 = blk * PSD_SBLK + 4 * tid;
  float4 tv = make_float4(0.f, 0.f, 0.f, 0.f), dv = tv;
  if (x0 < w.V) tv = __ldg(reinterpret_cast<const float4*>(w.t + x0));
  if (w.residual && x0 < w.Vd) dv = __ldg(reinterpret_cast<const float4*>(w.d + x0));
  out[0] = weight_of(w, tv.x, dv.x, x0);
  out[1] = weight_of(w, tv.y, dv.y, x0 + 1);
  out[2] = weight_of(w, tv.z, dv.z, x0 + 2);
  out[3] = weight_of(w, tv.w, dv.w, x0 + 3);
}

__device__ float block_weight_sum(const WeightCtx& w, int blk, float* s_lane, float* s_red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float wv[4];
  lane_weights(w, blk, tid, wv);
  const float ls = psd_add(psd_add(psd_add(wv[0], wv[1]), wv[2]), wv[3]);
  if (s_lane) s_lane[tid] = ls;
  const float ws = shfl_add_tree(ls);
  if (lane == 0) s_red[warp] = ws;
  __syncthreads();
  float tot = 0.0f;
  if (tid == 0) {
    float q[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) q[k] = s_red[k];
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
      for (int k = 0; k < off; ++k) q[k] = psd_add(q[k], q[k + off]);
    tot = q[0];
  }
  __syncthreads();
  return tot;  // valid in thread 0
}

// last element with positive weight in block blk (all threads return it)
__device__ int last_positive(const WeightCtx& w, int blk, int* s_int) {
  float wv[4];
  lane_weights(w, blk, threadIdx.x, wv);
  int best = -1;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (wv[c] > 0.0f) best = blk * PSD_SBLK + 4 * threadIdx.x + c;
  if (threadIdx.x == 0) *s_int = -1;
  __syncthreads();
  if (best >= 0) atomicMax(s_int, best);
  __syncthreads();
  const int r = *s_int;
  __syncthreads();
  return r < 0 ? blk * PSD_SBLK : r;
}

__global__ void __launch_bounds__(kThreads)
verify_sample(const Params p) {
  pdl_wait();
  pdl_trigger();
  const int blk = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const Plan pl = p.plan[b];
  WeightCtx w;
  w.V = p.V; w.Vd = p.Vd; w.c = p.c;
  w.t = p.t + b * p.tsb + pl.row * p.tsi;
  w.d = p.d + (int64_t)(p.d_rows ? p.d_rows[b] : b) * p.dsb + pl.row * p.dsi;
  w.bt = psd_bias(pl.Mt, p.c); w.bd = psd_bias(pl.Md, p.c); w.St = pl.St; w.Sd = pl.Sd;
  w.residual = pl.mode == 1;

  __shared__ float s_red[8];
  __shared__ float s_lane[kThreads];
  __shared__ int s_last, s_int;
  __shared__ float s_T, s_Pprev;
  __shared__ int s_chosen;

  const float W = block_weight_sum(w, blk, nullptr, s_red);
  if (tid == 0) {
    p.wblk[b * p.NB + blk] = W;
    __threadfence();
    s_last = atomicAdd(p.cnt_b + b, 1) == p.NB - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ float wb[PSD_MAX_SBLKS];
  for (int k = tid; k < p.NB; k += kThreads) wb[k] = __ldcg(p.wblk + b * p.NB + k);
  __syncthreads();

  // degenerate residual (sums to 0 in fp32): fall back to sampling from p
  if (tid == 0) {
    float R = 0.0f;
    for (int k = 0; k < p.NB; ++k) R = psd_add(R, wb[k]);
    s_int = (w.residual && !(R > 0.0f)) ? 1 : 0;
  }
  __syncthreads();
  if (s_int) {
    w.residual = 0;
    __syncthreads();
    for (int k = 0; k < p.NB; ++k) {
      const float Wk = block_weight_sum(w, k, nullptr, s_red);
      if (tid == 0) wb[k] = Wk;
    }
    __syncthreads();
  }
  if (tid == 0) {
    float R = 0.0f;
    for (int k = 0; k < p.NB; ++k) R = psd_add(R, wb[k]);
    const float T = psd_mul(p.u[b * (p.K + 1) + p.K], R);
    float P = 0.0f;
    int chosen = -1;
    float Pprev = 0.0f;
    for (int k = 0; k < p.NB; ++k) {
      const float Pn = psd_add(P, wb[k]);
      if (Pn > T) { chosen = k; Pprev = P; break; }
      P = Pn;
    }
    if (chosen < 0) {
      chosen = -2 - (p.NB - 1);
      for (int k = p.NB - 1; k >= 0; --k)
        if (wb[k] > 0.0f) { chosen = -2 - k; break; }
    }
    s_chosen = chosen; s_T = T; s_Pprev = Pprev;
  }
  __syncthreads();
  int tok;
  if (s_chosen <= -2) {
    tok = last_positive(w, -2 - s_chosen, &s_int);
  } else {
    const int cb = s_chosen;
    float wv[4];
    lane_weights(w, cb, tid, wv);
    s_lane[tid] = psd_add(psd_add(psd_add(wv[0], wv[1]), wv[2]), wv[3]);
    __syncthreads();
    if (tid == 0) {  // exclusive sequential prefix of lane sums, in place
      float C = 0.0f;
      for (int l = 0; l < kThreads; ++l) { const float s = s_lane[l]; s_lane[l] = C; C = psd_add(C, s); }
      s_int = 0x7fffffff;
    }
    __syncthreads();
    float acc = s_lane[tid];
    int hit = 0x7fffffff;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      acc = psd_add(acc, wv[c]);
      if (hit == 0x7fffffff && psd_add(s_Pprev, acc) > s_T) hit = cb * PSD_SBLK + 4 * tid + c;
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

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

struct WsLayout {
  size_t cnt_a, cnt_b, part, plan, wblk, total;
};

WsLayout layout(int B, int K, int V, int Vd, int sampling) {
  const int nmax = V > Vd ? V : Vd;
  const int NS = (nmax + PSD_SLICE - 1) / PSD_SLICE;
  const int NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  const int R = (K + 1) + (sampling ? K : 0);
  WsLayout L;
  size_t off = 0;
  L.cnt_a = off; off = align_up(off + sizeof(int) * B);
  L.cnt_b = off; off = align_up(off + sizeof(int) * B);
  L.part = off; off = align_up(off + sizeof(float2) * (size_t)B * R * NS);
  L.plan = off; off = align_up(off + sizeof(Plan) * (size_t)B);
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
  const WsLayout L = layout(B, K, V, 0, 0);
  int rc = check_common(target_logits, t_stride_b, t_stride_i, V, B, K, ws, ws_bytes, L.total);
  if (rc) return rc;
  Params p{};
  char* w = static_cast<char*>(ws);
  p.t = target_logits; p.tsb = t_stride_b; p.tsi = t_stride_i; p.V = V;
  p.d = nullptr; p.Vd = 0; p.ids = draft_ids; p.len = draft_len; p.u = nullptr;
  p.c = psd_scale(1.0f); p.B = B; p.K = K; p.acc = accepted_len; p.out = out_tokens;
  p.cnt_a = reinterpret_cast<int*>(w + L.cnt_a); p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part); p.plan = reinterpret_cast<Plan*>(w + L.plan);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK; p.R = K + 1;
  dim3 grid(p.NS, B * p.R);
  return (int)psd::launch(verify_stats<false>, grid, dim3(kThreads), 0, (cudaStream_t)stream, p);
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
  p.cnt_a = reinterpret_cast<int*>(w + L.cnt_a); p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part); p.plan = reinterpret_cast<Plan*>(w + L.plan);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  p.R = 2 * K + 1;
  dim3 grid(p.NS, B * p.R);
  cudaError_t e = psd::launch(verify_stats<true>, grid, dim3(kThreads), 0, (cudaStream_t)stream, p);
  if (e != cudaSuccess) return (int)e;
  dim3 grid2(p.NB, B);
  return (int)psd::launch(verify_sample, grid2, dim3(kThreads), 0, (cudaStream_t)stream, p);
}

int psd_verify_sample_rows(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                           int V, const float* draft_logits, const int32_t* draft_rows,
                           int64_t d_stride_row, int64_t d_stride_i, int Vd,
                      const int32_t* draft_ids, const int32_t* draft_len, const float* uniforms,
                      float temperature, int B, int K, int32_t* accepted_len,
                      int32_t* out_tokens, void* ws, size_t ws_bytes, void* stream) {
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
  p.ids = draft_ids; p.len = draft_len; p.u = uniforms;
  p.c = psd_scale(1.0f / temperature); p.B = B; p.K = K; p.acc = accepted_len; p.out = out_tokens;
  p.cnt_a = reinterpret_cast<int*>(w + L.cnt_a); p.cnt_b = reinterpret_cast<int*>(w + L.cnt_b);
  p.part = reinterpret_cast<float2*>(w + L.part); p.plan = reinterpret_cast<Plan*>(w + L.plan);
  p.wblk = reinterpret_cast<float*>(w + L.wblk);
  p.NS = (V + PSD_SLICE - 1) / PSD_SLICE; p.NB = (V + PSD_SBLK - 1) / PSD_SBLK;
  p.R = 2 * K + 1;
  dim3 grid(p.NS, B * p.R);
  cudaError_t e = psd::launch(verify_stats<true>, grid, dim3(kThreads), 0, (cudaStream_t)stream, p);
  if (e != cudaSuccess) return (int)e;
  dim3 grid2(p.NB, B);
  return (int)psd::launch(verify_sample, grid2, dim3(kThreads), 0, (cudaStream_t)stream, p);
}

}  // extern "C"
