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
#define PSD_MAX_SLICES 32 /* vocab <= 32 * 8192 = 262144 */
#define PSD_MAX_SBLKS 256 /* vocab / 1024 */

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
/* as psd_verify_sample, but request b's draft rows start at
 * draft_logits + draft_rows[b] * d_stride_row (per-slot draft storage) */
int psd_verify_sample_rows(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                           int V, const float* draft_logits, const int32_t* draft_rows,
                           int64_t d_stride_row, int64_t d_stride_i, int Vd,
                           const int32_t* draft_ids, const int32_t* draft_len,
                           const float* uniforms, float temperature, int B, int K,
                           int32_t* accepted_len, int32_t* out_tokens, void* workspace,
                           size_t workspace_bytes, void* stream);
/* psd_verify_sample_rows with cached draft-row statistics: d_stats (float2
 * (M, S) per draft row, row (b, i) at d_stats[draft_rows[b] * d_stats_ld + i];
 * NULL: computed from the draft rows) skips re-reading the draft rows, and
 * t_stats_out[t_stats_rows[b]] (NULL: not written; negative row: skipped)
 * receives the (M, S) of target row 0 -- the draft sampler (K = 0) publishes
 * the statistics of the distribution it sampled from.  Same canonical
 * arithmetic either way, so results are bit-identical. */
int psd_verify_sample_ext(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                          int V, const float* draft_logits, const int32_t* draft_rows,
                          int64_t d_stride_row, int64_t d_stride_i, int Vd,
                          const int32_t* draft_ids, const int32_t* draft_len,
                          const float* uniforms, float temperature, int B, int K,
                          int32_t* accepted_len, int32_t* out_tokens, const void* d_stats,
                          int64_t d_stats_ld, void* t_stats_out, const int32_t* t_stats_rows,
                          void* ws, size_t ws_bytes, void* stream);
/* Replay mode (GpuBackend(acceptance="replay")): as psd_verify_greedy /
 * psd_verify_sample_ext, but request b accepts exactly min(forced_len[b], k_b)
 * drafts whatever the logits say, then emits the target's token at that row
 * (greedy: its argmax; sampling: the residual sample, or the bonus from p when
 * every draft is kept).  Replaces the accepted count of a verified row with
 * the reference's own draw, accepted_count(model, k, draft_time,
 * acceptance_stream(seed, rid, j)) (pkg/src/specsim/acceptance_model.py:82-97,
 * engine.py:250-256), so a GPU run's step log equals specsim's byte for byte
 * while every pass runs on real logits. */
int psd_verify_greedy_forced(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                             int V, const int32_t* draft_ids, const int32_t* draft_len, int B,
                             int K, const int32_t* forced_len, int32_t* accepted_len,
                             int32_t* out_tokens, void* workspace, size_t workspace_bytes,
                             void* stream);
int psd_verify_sample_forced(const float* target_logits, int64_t t_stride_b, int64_t t_stride_i,
                             int V, const float* draft_logits, const int32_t* draft_rows,
                             int64_t d_stride_row, int64_t d_stride_i, int Vd,
                             const int32_t* draft_ids, const int32_t* draft_len,
                             const float* uniforms, float temperature, int B, int K,
                             const int32_t* forced_len, int32_t* accepted_len,
                             int32_t* out_tokens, const void* d_stats, int64_t d_stats_ld,
                             void* t_stats_out, const int32_t* t_stats_rows, void* ws,
                             size_t ws_bytes, void* stream);

/* Vocabulary-parallel greedy K1 (tensor-parallel LM head):
 * each rank reduces its logits shard (columns vocab_offset .. + V of the full
 * row) to canonical slice partials (max, global argmax index) -- floats
 * (psd_verify_partials_count) -- the ranks exchange them (e.g.
 * psd_tp_allgather_f32: W x count floats, rank order) and every rank folds
 * all W shards and decides (same accepted_len / out_tokens as psd_verify_greedy
 * on the gathered rows, without gathering M x V logits). */
size_t psd_verify_partials_count(int B, int K, int V);
int psd_verify_greedy_partials(const float* target_logits, int64_t t_stride_b,
                               int64_t t_stride_i, int V, int vocab_offset,
                               const int32_t* draft_len, int B, int K, float* partials,
                               void* stream);
int psd_verify_greedy_fold(const float* partials, int W, int V_shard, const int32_t* draft_ids,
                           const int32_t* draft_len, int B, int K, const int32_t* forced_len,
                           int32_t* accepted_len, int32_t* out_tokens, void* stream);

/* Greedy K1 fused into the target LM head: argmax_tokens[b * (K + 1) + j] is
 * the argmax (ties -> lowest index) of row j of request b's target logits
 * with the synthetic-language bias, produced by psd_gemm_argmax (K6 epilogue)
 * + psd_argmax_fold without storing logits; accepted_len / out_tokens as
 * psd_verify_greedy(_forced) on those logits. */
int psd_verify_greedy_tokens(const int32_t* argmax_tokens, const int32_t* draft_ids,
                             const int32_t* draft_len, int B, int K, const int32_t* forced_len,
                             int32_t* accepted_len, int32_t* out_tokens, void* stream);

/* ---- K2: bf16 GEMM on tcgen05 (TMEM accumulators, TMA, mbarrier ring) -----
 *   Y[m, n] = epi( sum_k X[m*ldx + k] * W[n*ldw + k] )   X [M,K], W [N,K] bf16
 * Replaces the virtual pass durations verify_latency / draft_latency
 * .duration(...) (pkg/src/specsim/engine.py:338, 359-360, 378, 402, 429;
 * request_model.py:112-117) with the real contractions of the forwards.
 * epi: PSD_EPI_BF16 (Y bf16), PSD_EPI_F32 (Y fp32), PSD_EPI_RESID (Y bf16 =
 * acc + R, Y may alias R), PSD_EPI_SILU (W rows packed per 128-row tile: for
 * q = 0..3, rows 32q..32q+15 are gate features tile*64+16q+0..15 and rows
 * 32q+16..32q+31 the matching up features; Y [M, N/2] bf16 = silu(g) * u).
 * N must be a multiple of 128, K and the leading dims multiples of 8.
 * splits_hint 0 (default) = stream-K persistent kernel: one CTA per SM,
 * balanced weight k-blocks per SM, cut tiles finished by their last-arriving
 * contributor; `workspace` (psd_gemm_plan bytes) must be ZEROED once at
 * allocation and not shared by concurrently running GEMMs (it is left zeroed).
 * splits_hint >= 1 = legacy grid split-K (fp32 partials + reduction). */
#define PSD_EPI_BF16 0
#define PSD_EPI_F32 1
#define PSD_EPI_RESID 2
#define PSD_EPI_SILU 3
#define PSD_EPI_PARTIAL 4 /* internal: split-K partials */
#define PSD_EPI_ARGMAX 5 /* internal: per-(128-row tile, token) (max, first argmax) partials (K6) */
/* Cap the CTAs of subsequently enqueued (or captured) GEMM grids (0 = all SMs):
 * the verify forward runs beside the draft loop on one GPU. */
void psd_gemm_set_max_ctas(int n);
/* Whole-K geometry for subsequently enqueued GEMMs (1 = on): no k-splitting
 * (one split for the grid split-K GEMMs, whole tiles only for stream-K), so
 * every output element is summed over K in the same order for any M -- the
 * prefill passes use it, making a prompt's KV cache independent of which
 * prompts share its prefill chunk. */
void psd_gemm_set_whole_k(int on);
/* Diagnostics: a device buffer of [CTAs][16] u64 that subsequent stream-K GEMMs
 * fill with %globaltimer stamps per CTA (entry, first operands, last MMA
 * issued, last accumulator ready, epilogue done, segments, fast finishes, rounds);
 * NULL turns it off (default). */
void psd_gemm_set_trace(void* trace);
int psd_gemm_plan(int M, int N, int K, int epi, int splits_hint, int* splits_out,
                  size_t* workspace_bytes);
int psd_gemm_bf16(const void* X, int ldx, int M, int K, const void* W, int ldw, int N, void* Y,
                  int ldy, int epi, const void* R, int ldr, int splits_hint, void* workspace,
                  size_t workspace_bytes, void* stream);
/* fp32 split-K partials P[z][m][n] (z < *splits_used, row pitch N); the
 * consumer kernel (psd_add_rmsnorm, psd_rope_kv) reduces them in z order, so
 * no separate reduction launch is needed.  Fewer splits are used when
 * p_bytes cannot hold splits*M*N floats. */
int psd_gemm_partials(const void* X, int ldx, int M, int K, const void* W, int ldw, int N,
                      float* P, size_t p_bytes, int splits_hint, int* splits_used, void* stream);

/* K6, the draft's greedy sampler fused into its LM head (replaces the logits
 * store + psd_bigram_bias + psd_verify_greedy(k = 0) of a draft step; seam
 * engine.py:355-364, 376-380): the stream-K LM-head GEMM's epilogue reduces
 * every finished (128-row vocabulary tile, token) to (max, lowest argmax
 * index) -- after adding `beta` to token m's logit at column
 * successor[tokens[rows ? rows[m] : m]] when successor and beta != 0 -- into
 * `partials` (psd_argmax_partials_bytes); psd_argmax_fold reduces the tiles
 * (ties -> lowest index, K1's canonical argmax) into out_tokens[m] and/or
 * dst[dst_idx[m]] (skipped when negative).  M <= 512, N % 128 == 0; the
 * workspace is psd_gemm_bf16's stream-K workspace. */
size_t psd_argmax_partials_bytes(int M, int N);
int psd_gemm_argmax(const void* X, int ldx, int M, int K, const void* W, int ldw, int N,
                    const int32_t* tokens, const int32_t* rows, const int32_t* successor,
                    float beta, void* partials, void* workspace, size_t workspace_bytes,
                    void* stream);
int psd_argmax_fold(const void* partials, int M, int N, int32_t* out_tokens, int32_t* dst,
                    const int32_t* dst_idx, void* stream);

/* ---- K3/K3'/K4: forward-pass building blocks (bf16 storage, fp32 math) ----
 * Same seam as K2 (the virtual pass durations).  Row-major activations. */
int psd_embed(const int32_t* tokens, int M, const void* table, int H, void* out, void* stream);
/* as psd_rope_kv, reading qkv = bf16(sum_z qkv_partials[z*slice + ...]) (the
 * QKV GEMM's split-K reduction fused into the RoPE pass) */
int psd_rope_kv_partials(const float* qkv_partials, int S, size_t slice, int M, int Hq, int Hkv,
                         int D, const int32_t* positions, const int32_t* slots,
                         const float* inv_freq, const void* qkv_bias, void* q_out,
                         void* k_cache, void* v_cache, void* stream);
/* src = rows ? rows[m] : m; v = bf16(x[src] + sum_z partials[z*slice + src*ldp])
 * (no add when partials == NULL; v written back to x when write_back);
 * y[m] = v * rsqrt(mean(v^2) + eps) * w.  H <= 8192. */
int psd_add_rmsnorm(void* x, int ldx, const float* partials, int S, size_t slice, int ldp,
                    const int32_t* rows, const void* w, void* y, int ldy, int M, int H, float eps,
                    int write_back, void* stream);
/* qkv [M, (Hq+2Hkv) D] bf16 (+ optional bias) -> rotate-half RoPE on q, k;
 * q -> q_out [M, Hq, D]; k, v -> caches [blocks*block_size, Hkv, D] at slot
 * slots[m] (negative: not written). */
int psd_rope_kv(const void* qkv, int M, int Hq, int Hkv, int D, const int32_t* positions,
                const int32_t* slots, const float* inv_freq, const void* qkv_bias, void* q_out,
                void* k_cache, void* v_cache, void* stream);
/* Paged multi-query attention, GQA.  Sequence s: query tokens q_start[s] ..
 * +q_len[s]-1 at positions q_pos0[s] + t; token t attends keys
 * 0 .. min(q_pos0[s] + t, kv_len[s] - 1) read through
 * block_table[seq_slot[s] * max_blocks + key / block_size].
 * max_kv_len (host hint, >= every kv_len) enables split-KV: the keys of a
 * (sequence, kv head) are cut across CTAs whose partial softmax states the
 * last-arriving CTA merges (workspace: psd_attention_workspace_bytes, zeroed
 * once; NULL or 0 disables splitting). */
size_t psd_attention_workspace_bytes(int num_seqs, int Hkv, int max_q_len, int Hq, int D,
                                     int max_kv_len);
int psd_attention(const void* q, const void* k_cache, const void* v_cache,
                  const int32_t* block_table, int max_blocks, const int32_t* seq_slot,
                  const int32_t* q_start, const int32_t* q_len, const int32_t* q_pos0,
                  const int32_t* kv_len, int num_seqs, int max_q_len, int Hq, int Hkv, int D,
                  int block_size, float scale, void* out, int max_kv_len, void* workspace,
                  size_t workspace_bytes, void* stream);
/* psd_attention with the RoPE + paged-KV write fused in (decode / verify passes:
 * max_q_len <= 64 / (Hq / Hkv)): reads the QKV split-K partials (S slices of
 * `slice` floats) instead of q, rotates Q / K per token position, writes this
 * pass's K / V rows into the caches and attends.  cudaErrorInvalidValue when the
 * pass needs several query chunks per sequence (use psd_rope_kv_partials +
 * psd_attention). */
int psd_attention_rope(const float* qkv_partials, int S, size_t slice, const int32_t* positions,
                       const int32_t* slots, const float* inv_freq, const void* qkv_bias,
                       void* k_cache, void* v_cache, const int32_t* block_table, int max_blocks,
                       const int32_t* seq_slot, const int32_t* q_start, const int32_t* q_len,
                       const int32_t* q_pos0, const int32_t* kv_len, int num_seqs, int max_q_len,
                       int Hq, int Hkv, int D, int block_size, float scale, void* out,
                       void* stream);
/* synthetic-language logit bias: logits[m, successor[prev_tokens[m]]] += beta */
int psd_bigram_bias(float* logits, int64_t ld, const int32_t* prev_tokens, int M,
                    const int32_t* successor, int V, float beta, void* stream);
/* the same on a vocabulary shard: logits hold columns [v0, v1) */
int psd_bigram_bias_range(float* logits, int64_t ld, const int32_t* prev_tokens, int M,
                          const int32_t* successor, int V, float beta, int v0, int v1,
                          void* stream);
/* out[b*n + i] = Philox4x32-10(key seed, counter (request_ids[b], verify_index[b],
 * base + i, 0)), top 24 bits / 2^24, in [0, 1) */
int psd_philox_uniforms(uint64_t seed, const int32_t* request_ids, const int32_t* verify_index,
                        int B, int n, int base, float* out, void* stream);
/* dst[dst_rows[r] * dst_ld + c] = src[r * src_ld + c], c < ncols (negative row: skip) */
int psd_copy_rows_f32(float* dst, const int32_t* dst_rows, int64_t dst_ld, const float* src,
                      int64_t src_ld, int nrows, int ncols, void* stream);
/* dst[r * dst_ld + c] = src[src_rows[r] * src_ld + c] (negative row: skip): packs the
 * draft distributions q of drafted rows for the hand-off to a target GPU */
int psd_gather_rows_f32(float* dst, int64_t dst_ld, const float* src, const int32_t* src_rows,
                        int64_t src_ld, int nrows, int ncols, void* stream);

/* ---- C1 / C2: peer-memory communicator (NVLink / NVSwitch load-stores) ---
 * Replaces the scalar `comm_overhead` the reference adds to a PSD step
 * (pkg/src/specsim/request_model.py:128; engine.py:435-442) with the real
 * exchanges: the row-parallel all-reduce of a tensor-parallel target (C2) and
 * the draft-id hand-off between a draft GPU and its target GPU (C1).
 * One process per GPU.  psd_comm_create allocates this rank's region and
 * writes its IPC handle (psd_comm_handle_bytes bytes) to handle_out; the
 * caller exchanges the handles (any host transport) and passes all `world`
 * of them, in rank order, to psd_comm_open.  Every rank must issue the same
 * sequence of all-reduce calls; kernels wait on peers with a 10 s watchdog
 * (trap) instead of hanging.  Kernels may be captured in CUDA graphs. */
#define PSD_COMM_MAX_WORLD 16
size_t psd_comm_handle_bytes(void);
int psd_comm_create(int rank, int world, size_t buf_bytes, size_t mbox_bytes, void** comm,
                    void* handle_out);
int psd_comm_open(void* comm, const void* handles);
/* One process driving `world` ranks (devices[r], ranks may share a device):
 * comms[r] ready to use, no IPC (peer access enabled between distinct
 * devices).  Rank r's calls must run on devices[r], concurrently with the
 * other ranks' (separate streams). */
int psd_comm_create_local(int world, const int* devices, size_t buf_bytes, size_t mbox_bytes,
                          void** comms);
int psd_comm_destroy(void* comm);
/* out[i] = sum over ranks r = 0..world-1 (in that order) of
 * sum over s = 0..S-1 (in that order) of partials_r[s * stride + i]:
 * the split-K reduction of a row-parallel GEMM fused with the cross-rank sum;
 * bit-identical on every rank.  n, stride multiples of 4, 16-byte aligned,
 * 4 n <= buf_bytes. */
int psd_tp_allreduce_partials(void* comm, const float* partials, int S, size_t stride, size_t n,
                              float* out, void* stream);
int psd_tp_allreduce_f32(void* comm, float* data, size_t n, void* stream);
/* out[r * n + i] = src_r[i] for every rank r (out must not alias src) */
int psd_tp_allgather_f32(void* comm, const float* src, size_t n, float* out, void* stream);
/* mailbox (depth 1 per peer pair): put copies n int32 into this rank's slot
 * of `peer`'s mailbox once the peer consumed the previous message; get waits
 * for the next message from `peer` and copies it to dst.  4 n <= mbox_bytes. */
int psd_p2p_put_i32(void* comm, int peer, const int32_t* src, int n, void* stream);
int psd_p2p_get_i32(void* comm, int peer, int32_t* dst, int n, void* stream);

/* ---- K5 / glue: KV commit of accepted tokens, token routing ---------------
 * psd_commit replaces the commit rule + KV write accounting of a verified row
 * (pkg/src/specsim/engine.py:257-262; kv_manager.py:130-144): per row b
 * (slot row_slot[b]), append out_tokens[b, 0..a_b] to outputs[slot], advance
 * generated[slot] by a_b + 1 and the slot's last two tokens.  The rejected
 * tail needs no device work: KV validity is positional, so rolling back is the
 * host shrinking the sequence length / block list (KVBlockTable.trim_to_written). */
int psd_commit(const int32_t* accepted_len, const int32_t* out_tokens, int K,
               const int32_t* row_slot, int n, int32_t* generated, int32_t* slot_tokens,
               int slot_tokens_ld, int32_t* outputs, int outputs_ld, void* stream);
/* dst[dst_idx ? dst_idx[i] : i] = src[src_idx ? src_idx[i] : i], negative dst skipped */
int psd_index_copy_i32(int32_t* dst, const int32_t* dst_idx, const int32_t* src,
                       const int32_t* src_idx, int n, void* stream);
/* ---- host-side staging of the draft / verify pass metadata ---------------
 * (no reference counterpart: the reference's passes are virtual durations,
 * SURVEY §8a a16, request_model.py:92-117 called at engine.py:338, 359-360,
 * 378, 402, 429).  Pure host code: fills the pinned metadata set(s) of a
 * forward (field order tokens, positions, slots, seq_slot, q_start, q_len,
 * q_pos0, kv_len, logit_rows, gather_src, scatter_dst; `fields` = 11
 * offset / capacity pairs in int32 units) for n real rows padded to nb with
 * the scratch slot.  KV write slots come from the block table
 * (block_table[slot * bt_ld + pos / block_size] * block_size + pos % block_size);
 * a position past nblk[slot] blocks is PSD_STAGE_KV_OVERRUN unless `replay`
 * (then that row writes nowhere, -1).
 * psd_stage_draft: kmax decode sets (set_stride int32 apart); set 0 feeds the
 *   last two committed tokens (positions L-2, L-1), set i >= 1 the draft at
 *   L-1+i for rows with i < k[r]; scatter targets slot * ldt + 2 + i.
 * psd_stage_verify: one set of nb * (kmax + 1) query tokens (row r token j
 *   at position L-1+j; KV written for j <= k[r]). */
#define PSD_STAGE_BAD_ARGS 1001
#define PSD_STAGE_CAPACITY 1002
#define PSD_STAGE_KV_OVERRUN 1003
int psd_stage_draft(int32_t* sets, int64_t set_stride, const int32_t* fields,
                    const int32_t* block_table, int bt_ld, const int32_t* nblk, int block_size,
                    int replay, int ldt, int scratch_slot, const int32_t* slot, const int32_t* L,
                    const int32_t* k, int n, int nb, int kmax);
int psd_stage_verify(int32_t* set, const int32_t* fields, const int32_t* block_table, int bt_ld,
                     const int32_t* nblk, int block_size, int replay, int ldt, int scratch_slot,
                     const int32_t* slot, const int32_t* L, const int32_t* k, int n, int nb,
                     int kmax);
/* stream-ordered copy (cudaMemcpyAsync, direction from the pointers): the
 * per-step metadata uploads from pinned staging, without a kernel */
int psd_copy_async(void* dst, const void* src, size_t bytes, void* stream);
/* kernels enqueued by this library so far (host-side counter; a captured
 * CUDA graph's launches are counted once, at capture) */
long long psd_launch_count(void);
/* deterministic random init: (u - 1/2) * span, u = splitmix64(seed, i) >> 40 / 2^24 */
int psd_fill_uniform_bf16(void* out, size_t n, uint64_t seed, float span, void* stream);
/* The [rows x cols] block at (row0, col0) of the virtual [* x full_cols] tensor
 * psd_fill_uniform_bf16 would produce with `seed` (row pitch ld): the weights of
 * a tensor-parallel shard, generated in place. */
int psd_fill_uniform_bf16_block(void* out, int64_t ld, int rows, int cols, int64_t full_cols,
                                int64_t row0, int64_t col0, uint64_t seed, float span,
                                void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSD_H */
