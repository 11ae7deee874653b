/*
 * psd_canon.h -- the canonical fp32 arithmetic of speculative verification.
 *
 * Bit-exact acceptance decisions between the sm_100a kernel
 * (paper_2603_18016_b200/csrc/verify.cu) and the CPU oracle
 * (oracle/verify_oracle.c) need (1) one exp implementation whose every
 * operation is a single IEEE-rounded fp32 op (no contraction, no MUFU
 * approximation), and (2) one fixed reduction structure.  This header is (1)
 * and documents (2); both sides include it.  Compile host code with
 * -ffp-contract=off; device code uses the explicit __f*_rn intrinsics below,
 * which nvcc never fuses.
 *
 * Probabilities.  With c = fl(fl(1/T) * log2 e) (psd_scale) and a reference
 * maximum M of the raw logits, the unnormalised weight of logit x is
 *     e(x; M) = E2(fma(x, c, -fl(M * c)))        (= exp((x - M) / T))
 * where E2 is the canonical 2^t below.  p(x) = e(x; M_row) / S_row.
 *
 * Reduction structure ("canonical order"):
 *   softmax statistics (row max M, S = sum_x e(x; M)) of a row of n logits:
 *     - the row is cut into slices of PSD_SLICE = 8192 elements; slice max
 *       M_s is exact;
 *     - inside a slice, lane l (0..255) owns the float4 vectors l + 256 j
 *       (j = 0..7); lane sum s_l = sequential sum over j, then x,y,z,w, of
 *       e(x; M_s);
 *     - slice sum: each warp of 32 lanes adds pairwise with offsets
 *       16,8,4,2,1 (v[l] = v[l] + v[l+off]), then the 8 warp results with
 *       offsets 4,2,1;
 *     - slices fold left to right with psd_combine.
 *   greedy: argmax over the row, ties -> lowest index (order free).
 *   sampling by prefix search over non-negative weights w_x:
 *     - the row is cut into blocks of PSD_SBLK = 1024 elements; lane l owns
 *       elements 4l..4l+3; lane sum = ((w0 + w1) + w2) + w3; block sum W_b is
 *       the warp tree (16..1) then the 8-warp tree (4,2,1) of lane sums;
 *     - block prefix P_b = P_{b-1} + W_b (sequential), total R = P_last;
 *     - threshold T = u * R; the chosen block is the first with P_b > T;
 *       inside it, the lane prefix C_l is the sequential sum of lane sums
 *       0..l-1 and element x = 4l + j is chosen iff it is the first with
 *       P_{b-1} + (((C_l + w_{4l}) + ...) + w_{4l+j}) > T;
 *     - no hit (rounding): last positive-weight element of the chosen block
 *       (or, with no block hit, of the last positive-weight block).
 * Acceptance (speculative sampling, Leviathan et al. / Chen et al.):
 *     accept draft x at position i  iff  (u_i * e_d(x)) * S_t < e_t(x) * S_d
 *     with e_t(x) = e(x; M_t), e_d(x) = e(x; M_d) over the target / draft
 *     rows; this is u_i < p(x) / q(x) without a division.
 * Residual weight: r(x) = max(0, e_t(x) * S_d - e_d(x) * S_t), proportional to
 *     max(0, p(x) - q(x)); e_d(x) = 0 beyond the draft vocabulary.
 */
#ifndef PSD_CANON_H
#define PSD_CANON_H

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define PSD_HD __host__ __device__ __forceinline__
#else
#define PSD_HD static inline
#include <math.h>
#endif

#define PSD_SLICE 8192
#define PSD_SLICE_LANES 256
#define PSD_SBLK 1024

#ifdef __CUDA_ARCH__
PSD_HD float psd_mul(float a, float b) { return __fmul_rn(a, b); }
PSD_HD float psd_add(float a, float b) { return __fadd_rn(a, b); }
PSD_HD float psd_sub(float a, float b) { return __fsub_rn(a, b); }
PSD_HD float psd_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
PSD_HD uint32_t psd_bits(float x) { return __float_as_uint(x); }
PSD_HD float psd_from_bits(uint32_t u) { return __uint_as_float(u); }
#else
/* host: build with -ffp-contract=off (oracle/Makefile) so these stay single
 * rounded operations */
PSD_HD float psd_mul(float a, float b) { return a * b; }
PSD_HD float psd_add(float a, float b) { return a + b; }
PSD_HD float psd_sub(float a, float b) { return a - b; }
PSD_HD float psd_fma(float a, float b, float c) { return fmaf(a, b, c); }
PSD_HD uint32_t psd_bits(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
PSD_HD float psd_from_bits(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }
#endif

PSD_HD float psd_max(float a, float b) { return a > b ? a : b; }

#define PSD_NEG_INF (-__builtin_inff())

/* E2(t) = 2^t for t <= ~0, canonical: t clamped to >= -125 (so results stay
 * normal; -inf and NaN map to 2^-125), n = rint(t) by the 1.5*2^23 trick,
 * f = t - n in [-1/2, 1/2], 2^f by a degree-6 Taylor polynomial (Horner with
 * fused multiply-adds), exponent added as an integer.  E2(0) == 1 exactly. */
PSD_HD float psd_exp2(float t) {
  t = t > -125.0f ? t : -125.0f;
  const float r = psd_add(t, 12582912.0f); /* 1.5 * 2^23 */
  const float n = psd_sub(r, 12582912.0f);
  const float f = psd_sub(t, n);
  float p = 1.54035304e-4f;
  p = psd_fma(p, f, 1.33335581e-3f);
  p = psd_fma(p, f, 9.61812911e-3f);
  p = psd_fma(p, f, 5.55041087e-2f);
  p = psd_fma(p, f, 2.40226507e-1f);
  p = psd_fma(p, f, 6.93147181e-1f);
  p = psd_fma(p, f, 1.0f);
  /* bits(r) = 0x4B400000 + n for |n| < 2^22: no float->int conversion */
  return psd_from_bits(psd_bits(p) + ((psd_bits(r) - 0x4B400000u) << 23));
}

/* c = fl(fl(1/T) * log2(e)) */
PSD_HD float psd_scale(float inv_temp) { return psd_mul(inv_temp, 1.44269504088896341f); }
/* exponent bias for reference max M: -fl(M * c) */
PSD_HD float psd_bias(float M, float c) { return -psd_mul(M, c); }
/* e(x; M) = E2(fma(x, c, bias)) */
PSD_HD float psd_weight(float x, float c, float bias) { return psd_exp2(psd_fma(x, c, bias)); }

/* (m, s) pair: max of the raw logits and sum of e(x; m). */
typedef struct { float m; float s; } psd_ms;

PSD_HD psd_ms psd_combine(psd_ms a, psd_ms b, float c) {
  if (a.m == PSD_NEG_INF) return b;
  if (b.m == PSD_NEG_INF) return a;
  psd_ms o;
  o.m = psd_max(a.m, b.m);
  const float bias = psd_bias(o.m, c);
  o.s = psd_add(psd_mul(a.s, psd_weight(a.m, c, bias)), psd_mul(b.s, psd_weight(b.m, c, bias)));
  return o;
}

/* (value, index) argmax pair; ties -> lowest index. */
typedef struct { float v; int32_t i; } psd_vi;

PSD_HD psd_vi psd_argmax2(psd_vi a, psd_vi b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

/* Acceptance test of one drafted token (see header comment). */
PSD_HD int psd_accept(float u, float e_t, float e_d, float S_t, float S_d) {
  return psd_mul(psd_mul(u, e_d), S_t) < psd_mul(e_t, S_d);
}

/* Residual weight proportional to max(0, p - q). */
PSD_HD float psd_residual(float e_t, float e_d, float S_t, float S_d) {
  const float r = psd_sub(psd_mul(e_t, S_d), psd_mul(e_d, S_t));
  return r > 0.0f ? r : 0.0f;
}

#endif /* PSD_CANON_H */
