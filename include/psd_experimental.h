/*
 * psd_experimental.h -- measured-and-parked variants, built only with
 * PSD_EXPERIMENTAL=1 (python -m paper_2603_18016_b200.build_native).  Neither
 * is on the product path: both measured slower than what ships (DESIGN.md §3,
 * profiles/r01_kbench_gemm_variants.txt, profiles/r01b_fused_draft_trace.txt).
 */
#ifndef PSD_EXPERIMENTAL_H
#define PSD_EXPERIMENTAL_H

#include "psd.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Pre-tiled weights: [N/128][ceil(K/64)][128][64] bf16 with the 128-byte
 * swizzle applied, so every (128-row, 64-col) weight tile is one contiguous,
 * already-swizzled 16 KB block loaded with a single 1-D bulk copy (sequential
 * HBM bursts, no tensor-map walk).  psd_gemm_tiled = stream-K GEMM on them. */
size_t psd_tiled_weight_bytes(int N, int K);
int psd_tile_weights(const void* W, int N, int K, int ldw, void* tiled, void* stream);
int psd_gemm_tiled(const void* X, int ldx, int M, int K, const void* W_tiled, int N, void* Y,
                   int ldy, int epi, const void* R, int ldr, void* workspace,
                   size_t workspace_bytes, void* stream);
/* ---- fused k-step greedy draft decode (csrc/decode_mk.cu) -------------------
 * One persistent kernel runs all k draft steps of a batch (embedding, every
 * layer, LM head, argmax, scatter of the draft token into slot_tok).  The
 * model and the forward buffers are bound once; psd_mk_launch enqueues one
 * launch (graph-capturable once a (nb, steps) program was built eagerly).
 * Replaces the per-kernel draft forward of model.py for head_dim 32/64, greedy. */
typedef struct {
  int layers, hidden, heads, kv_heads, head_dim, ffn /* padded to 64 */, vocab;
  float eps, attn_scale, beta;
  int block_size, max_blocks, grid /* 0 = all SMs */, max_tokens;
  /* 9 per layer: wqkv, wo, wgu (packed), wdown, attn_norm, mlp_norm, bqkv|NULL, k cache, v cache */
  const void* const* layer_ptrs;
  const void* embed;
  const void* lm_head;
  const void* final_norm;
  const float* inv_freq;
  const int32_t* successor; /* synthetic-language successor table (beta = 0: unused) */
  const int32_t* block_table;
  void* x; void* xn; void* attn; void* act; void* xf; /* forward buffers, >= 64 rows */
  float* part;   /* split-K partials */
  void* argpart; /* (vocab / 128) * 64 float2 */
  int32_t* slot_tok;
  int32_t* meta; int set_stride; int field_offsets[11];
} psd_mk_model;
size_t psd_mk_smem_bytes(void);
void* psd_mk_create(const psd_mk_model* model);
void psd_mk_destroy(void* handle);
int psd_mk_grid(void* handle);
int psd_mk_launch(void* handle, int nb, int steps, void* stream);
/* Diagnostics: ops of a built (nb, steps) program (-1: not built), and a launch
 * that records per-CTA per-op %globaltimer stamps (entry, inputs ready, done)
 * into trace[grid][n_ops][3] (u64). */
int psd_mk_n_ops(void* handle, int nb, int steps);
int psd_mk_launch_traced(void* handle, int nb, int steps, void* trace, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSD_EXPERIMENTAL_H */
