/*
 * verify_oracle.c -- CPU restatement of speculative verification (TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg as the checker; never linked
 * into the product library).
 *
 * Parity status: the reference package has NO token-level verification (it
 * draws coin flips: pkg/src/specsim/acceptance_model.py:82-97), so this file
 * restates the algorithm from its contract, and that part is "parity
 * unpinned" against the reference:
 *   - chain contract: draft i is accepted only if 0..i-1 were, strict "<"
 *     test (acceptance_model.py:91-96);
 *   - commit rule: accepted + exactly one bonus token (engine.py:257-262);
 *   - speculative sampling: accept x_i iff
 *     u_i < p_i(x_i) / q_i(x_i); at the first rejection sample from
 *     norm(max(0, p - q)); if all k accepted sample the bonus from p_{k+1};
 *   - greedy: accept iff x_i == argmax p_i (ties -> lowest id), bonus =
 *     argmax at the first mismatch (or at position k).
 * It is pinned instead (tests/test_verify_oracle.py) against an independent
 * float64 numpy evaluation of the same rule (decisions must agree wherever
 * the exact-math margin exceeds fp32 rounding) and against committed golden
 * vectors tests/golden/verify_golden.json.
 *
 * Arithmetic: every float op goes through include/psd_canon.h, evaluated in the
 * canonical order documented there, written here as plain sequential loops.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/psd_canon.h"

/* ---- softmax statistics in canonical order ------------------------------ */
static psd_ms slice_stats(const float* row, int begin, int n, float c) {
  /* exact slice max */
  float M = PSD_NEG_INF;
  const int end = begin + PSD_SLICE < n ? begin + PSD_SLICE : n;
  for (int e = begin; e < end; ++e) M = psd_max(M, row[e]);
  const float bias = psd_bias(M, c);
  float lane[PSD_SLICE_LANES];
  for (int l = 0; l < PSD_SLICE_LANES; ++l) {
    float s = 0.0f;
    for (int j = 0; j < 8; ++j)
      for (int q = 0; q < 4; ++q) {
        const int e = begin + 4 * (l + PSD_SLICE_LANES * j) + q;
        if (e < n) s = psd_add(s, psd_weight(row[e], c, bias));
      }
    lane[l] = s;
  }
  for (int w = 0; w < PSD_SLICE_LANES / 32; ++w)
    for (int off = 16; off >= 1; off >>= 1)
      for (int l = 0; l < off; ++l) lane[32 * w + l] = psd_add(lane[32 * w + l], lane[32 * w + l + off]);
  float wr[8];
  for (int w = 0; w < 8; ++w) wr[w] = lane[32 * w];
  for (int off = 4; off >= 1; off >>= 1)
    for (int w = 0; w < off; ++w) wr[w] = psd_add(wr[w], wr[w + off]);
  psd_ms out = {M, wr[0]};
  return out;
}

void oracle_row_stats(const float* row, int n, float inv_temp, float* M, float* S) {
  const float c = psd_scale(inv_temp);
  psd_ms acc = {PSD_NEG_INF, 0.0f};
  int first = 1;
  for (int begin = 0; begin < n; begin += PSD_SLICE) {
    psd_ms sl = slice_stats(row, begin, n, c);
    acc = first ? sl : psd_combine(acc, sl, c);
    first = 0;
  }
  *M = acc.m;
  *S = acc.s;
}

float oracle_exp2(float t) { return psd_exp2(t); }

int32_t oracle_row_argmax(const float* row, int n) {
  psd_vi best = {PSD_NEG_INF, 0x7fffffff};
  for (int e = 0; e < n; ++e) {
    psd_vi c = {row[e], e};
    best = psd_argmax2(best, c);
  }
  return best.i;
}

/* ---- prefix-search sampling in canonical order -------------------------- */
typedef struct {
  const float* t; /* target row */
  const float* d; /* draft row or NULL (bonus mode) */
  int V, Vd;
  float c, Mt, St, Md, Sd;
  int residual; /* 1: r = max(0, p - q); 0: w = p */
} weight_src;

static float weight_at(const weight_src* w, int x) {
  if (x >= w->V) return 0.0f;
  const float et = psd_weight(w->t[x], w->c, psd_bias(w->Mt, w->c));
  if (!w->residual) return et;
  const float ed = (x < w->Vd) ? psd_weight(w->d[x], w->c, psd_bias(w->Md, w->c)) : 0.0f;
  return psd_residual(et, ed, w->St, w->Sd);
}

static float block_sum(const weight_src* w, int blk, float lanes[256]) {
  float v[256];
  for (int l = 0; l < 256; ++l) {
    const int base = blk * PSD_SBLK + 4 * l;
    float s = weight_at(w, base);
    s = psd_add(s, weight_at(w, base + 1));
    s = psd_add(s, weight_at(w, base + 2));
    s = psd_add(s, weight_at(w, base + 3));
    v[l] = s;
    if (lanes) lanes[l] = s;
  }
  for (int wp = 0; wp < 8; ++wp)
    for (int off = 16; off >= 1; off >>= 1)
      for (int l = 0; l < off; ++l) v[32 * wp + l] = psd_add(v[32 * wp + l], v[32 * wp + l + off]);
  float wr[8];
  for (int wp = 0; wp < 8; ++wp) wr[wp] = v[32 * wp];
  for (int off = 4; off >= 1; off >>= 1)
    for (int wp = 0; wp < off; ++wp) wr[wp] = psd_add(wr[wp], wr[wp + off]);
  return wr[0];
}

static int last_positive_in_block(const weight_src* w, int blk) {
  for (int x = blk * PSD_SBLK + PSD_SBLK - 1; x >= blk * PSD_SBLK; --x)
    if (weight_at(w, x) > 0.0f) return x;
  return blk * PSD_SBLK;
}

static int32_t prefix_sample(const weight_src* w, float u) {
  const int nb = (w->V + PSD_SBLK - 1) / PSD_SBLK;
  float* W = (float*)malloc(sizeof(float) * nb);
  float R = 0.0f;
  for (int b = 0; b < nb; ++b) {
    W[b] = block_sum(w, b, NULL);
    R = psd_add(R, W[b]);
  }
  const float T = psd_mul(u, R);
  float P = 0.0f;
  int chosen = -1;
  float P_prev = 0.0f;
  for (int b = 0; b < nb; ++b) {
    const float Pn = psd_add(P, W[b]);
    if (Pn > T) { chosen = b; P_prev = P; break; }
    P = Pn;
  }
  int32_t result;
  if (chosen < 0) {
    int lastb = nb - 1;
    for (int b = nb - 1; b >= 0; --b)
      if (W[b] > 0.0f) { lastb = b; break; }
    result = last_positive_in_block(w, lastb);
  } else {
    float lanes[256];
    block_sum(w, chosen, lanes);
    float C = 0.0f;
    result = -1;
    for (int l = 0; l < 256 && result < 0; ++l) {
      float acc = C;
      for (int j = 0; j < 4; ++j) {
        const int x = chosen * PSD_SBLK + 4 * l + j;
        acc = psd_add(acc, weight_at(w, x));
        if (psd_add(P_prev, acc) > T) { result = x; break; }
      }
      C = psd_add(C, lanes[l]);
    }
    if (result < 0) result = last_positive_in_block(w, chosen);
  }
  free(W);
  return result;
}

/* ---- the two verification entry points ----------------------------------- */
/* Layouts: target logits row (b, i) at t + b*tsb + i*tsi, i in 0..K;
 * draft logits row (b, i) at d + b*dsb + i*dsi, i in 0..K-1;
 * draft_ids[b*K + i]; uniforms[b*(K+1) + i] (i < K acceptance, i == K sample);
 * out_tokens[b*(K+1) + i], -1 past the emitted tokens. */
/* forced_len (NULL: the real test): replay mode -- accept exactly
 * min(forced_len[b], k_b) drafts whatever the logits say, then emit the
 * target's token at that row (bonus / residual sample), as the GPU's
 * psd_verify_*_forced do for GpuBackend(acceptance="replay"). */
static int verify_greedy_impl(const float* t, int64_t tsb, int64_t tsi, int V,
                              const int32_t* draft_ids, const int32_t* draft_len, int B, int K,
                              const int32_t* forced_len, int32_t* accepted_len,
                              int32_t* out_tokens) {
  for (int b = 0; b < B; ++b) {
    const int kb = draft_len[b];
    if (kb < 0 || kb > K) return 1;
    int a = 0;
    int32_t g = 0;
    if (forced_len) {
      a = forced_len[b] < 0 ? 0 : (forced_len[b] > kb ? kb : forced_len[b]);
      g = oracle_row_argmax(t + b * tsb + a * tsi, V);
    } else {
      for (int i = 0; i <= kb; ++i) {
        g = oracle_row_argmax(t + b * tsb + i * tsi, V);
        if (i == kb || draft_ids[b * K + i] != g) break;
        ++a;
      }
    }
    accepted_len[b] = a;
    for (int i = 0; i <= K; ++i) out_tokens[b * (K + 1) + i] = -1;
    for (int i = 0; i < a; ++i) out_tokens[b * (K + 1) + i] = draft_ids[b * K + i];
    out_tokens[b * (K + 1) + a] = g;
  }
  return 0;
}

int oracle_verify_greedy(const float* t, int64_t tsb, int64_t tsi, int V,
                         const int32_t* draft_ids, const int32_t* draft_len, int B, int K,
                         int32_t* accepted_len, int32_t* out_tokens) {
  return verify_greedy_impl(t, tsb, tsi, V, draft_ids, draft_len, B, K, NULL, accepted_len,
                            out_tokens);
}

int oracle_verify_greedy_forced(const float* t, int64_t tsb, int64_t tsi, int V,
                                const int32_t* draft_ids, const int32_t* draft_len, int B, int K,
                                const int32_t* forced_len, int32_t* accepted_len,
                                int32_t* out_tokens) {
  return verify_greedy_impl(t, tsb, tsi, V, draft_ids, draft_len, B, K, forced_len, accepted_len,
                            out_tokens);
}

static int verify_sample_impl(const float* t, int64_t tsb, int64_t tsi, int V, const float* d,
                              int64_t dsb, int64_t dsi, int Vd, const int32_t* draft_ids,
                              const int32_t* draft_len, const float* uniforms, float temperature,
                              int B, int K, const int32_t* forced_len, int32_t* accepted_len,
                              int32_t* out_tokens) {
  const float inv_temp = 1.0f / temperature;
  const float c = psd_scale(inv_temp);
  for (int b = 0; b < B; ++b) {
    const int kb = draft_len[b];
    if (kb < 0 || kb > K) return 1;
    int a = 0;
    float Mt = 0, St = 0, Md = 0, Sd = 0;
    if (forced_len) {
      a = forced_len[b] < 0 ? 0 : (forced_len[b] > kb ? kb : forced_len[b]);
      if (a < kb) {
        oracle_row_stats(t + b * tsb + a * tsi, V, inv_temp, &Mt, &St);
        oracle_row_stats(d + b * dsb + a * dsi, Vd, inv_temp, &Md, &Sd);
      }
    } else {
      for (; a < kb; ++a) {
        const float* tr = t + b * tsb + a * tsi;
        const float* dr = d + b * dsb + a * dsi;
        oracle_row_stats(tr, V, inv_temp, &Mt, &St);
        oracle_row_stats(dr, Vd, inv_temp, &Md, &Sd);
        const int32_t x = draft_ids[b * K + a];
        if (x < 0 || x >= V) break;
        const float et = psd_weight(tr[x], c, psd_bias(Mt, c));
        const float ed = x < Vd ? psd_weight(dr[x], c, psd_bias(Md, c)) : 0.0f;
        if (!psd_accept(uniforms[b * (K + 1) + a], et, ed, St, Sd)) break;
      }
    }
    weight_src w;
    w.V = V;
    w.Vd = Vd;
    w.c = c;
    w.t = t + b * tsb + a * tsi;
    if (a < kb) { /* rejected at a: stats of rows a already computed */
      w.d = d + b * dsb + a * dsi;
      w.Mt = Mt; w.St = St; w.Md = Md; w.Sd = Sd;
      w.residual = 1;
      /* degenerate residual (sums to zero in fp32): sample from p */
      const int nb = (V + PSD_SBLK - 1) / PSD_SBLK;
      float R = 0.0f;
      for (int blk = 0; blk < nb; ++blk) R = psd_add(R, block_sum(&w, blk, NULL));
      if (!(R > 0.0f)) w.residual = 0;
    } else {
      oracle_row_stats(w.t, V, inv_temp, &w.Mt, &w.St);
      w.d = NULL;
      w.Md = 0; w.Sd = 0;
      w.residual = 0;
    }
    const int32_t tok = prefix_sample(&w, uniforms[b * (K + 1) + K]);
    accepted_len[b] = a;
    for (int i = 0; i <= K; ++i) out_tokens[b * (K + 1) + i] = -1;
    for (int i = 0; i < a; ++i) out_tokens[b * (K + 1) + i] = draft_ids[b * K + i];
    out_tokens[b * (K + 1) + a] = tok;
  }
  return 0;
}

int oracle_verify_sample(const float* t, int64_t tsb, int64_t tsi, int V, const float* d,
                         int64_t dsb, int64_t dsi, int Vd, const int32_t* draft_ids,
                         const int32_t* draft_len, const float* uniforms, float temperature,
                         int B, int K, int32_t* accepted_len, int32_t* out_tokens) {
  return verify_sample_impl(t, tsb, tsi, V, d, dsb, dsi, Vd, draft_ids, draft_len, uniforms,
                            temperature, B, K, NULL, accepted_len, out_tokens);
}

int oracle_verify_sample_forced(const float* t, int64_t tsb, int64_t tsi, int V, const float* d,
                                int64_t dsb, int64_t dsi, int Vd, const int32_t* draft_ids,
                                const int32_t* draft_len, const float* uniforms,
                                float temperature, int B, int K, const int32_t* forced_len,
                                int32_t* accepted_len, int32_t* out_tokens) {
  return verify_sample_impl(t, tsb, tsi, V, d, dsb, dsi, Vd, draft_ids, draft_len, uniforms,
                            temperature, B, K, forced_len, accepted_len, out_tokens);
}
