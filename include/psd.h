/*
 * psd.h -- C ABI of libpsd.so, the B200-native hot path of batch-parallel
 * speculative decoding (PSD).
 *
 * Plain pointers and sizes only (no torch types); every call is
 * stream-ordered on the `stream` argument (a cudaStream_t passed as void*)
 * and returns a cudaError_t value (0 = success).  Device pointers are raw
 * CUDA allocations; the library owns no persistent memory except what a
 * caller-provided workspace holds.
 *
 * The reference package (specsim, pure Python) has no FFI.  Each entry point
 * names the reference abstraction it replaces so a maintainer can see which
 * seam it plugs into (INTEGRATION.md shows the ctypes binding):
 *
 *   psd_verify_greedy / psd_verify_sample
 *       replace accepted_count(model, k, draft_time, rng) +
 *       acceptance_stream(seed, rid, j)
 *       (pkg/src/specsim/acceptance_model.py:50-52, 82-97), as called by the
 *       verification of a batch (pkg/src/specsim/engine.py:245-256), and the
 *       commit rule accepted + 1 bonus (engine.py:257-262).
 */
#ifndef PSD_H
#define PSD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSD_MAX_K 16 /* largest draft depth a verification row may carry */

/* ---- K1: fused speculative verification --------------------------------
 * Layouts (elements, fp32 logits):
 *   target row (b, i), i = 0..K:   target_logits + b*t_stride_b + i*t_stride_i
 *   draft row (b, i),  i = 0..K-1: draft_logits  + b*d_stride_b + i*d_stride_i
 *   draft_ids[b*K + i], draft_len[b] = k_b in [0, K] (0 = idle pass)
 *   uniforms[b*(K+1) + i]: i < k_b acceptance uniforms, i == K the sampling
 *   uniform, all in [0, 1)
 * Outputs: accepted_len[b] = a_b; out_tokens[b*(K+1) + i] = accepted drafts
 *   (i < a_b), the bonus / residual-sampled token at i == a_b, -1 after.
 * V, Vd, strides must be multiples of 4 and logits 16-byte aligned; Vd <= V
 * (draft probability is 0 past Vd).  The workspace must be zeroed once with
 * psd_verify_workspace_init; the kernels leave it reusable.
 * Arithmetic: include/psd_canon.h (bit-exact with oracle/verify_oracle.c). */
size_t psd_verify_workspace_bytes(int B, int K, int V, int Vd, int sampling);
int psd_verify_workspace_init(void* workspace, size_t workspace_bytes, void* stream);
int psd_verify_greedy(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                      int V, const int32_t* draft_ids, const int32_t* draft_len, int B, int K,
                      int32_t* accepted_len, int32_t* out_tokens, void* workspace,
                      size_t workspace_bytes, void* stream);
int psd_verify_sample(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                      int V, const float* draft_logits, int64_t d_stride_b, int64_t d_stride_i,
                      int Vd, const int32_t* draft_ids, const int32_t* draft_len,
                      const float* uniforms, float temperature, int B, int K,
                      int32_t* accepted_len, int32_t* out_tokens, void* workspace,
                      size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSD_H */
