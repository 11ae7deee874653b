// Host-side metadata staging of the draft and verify passes (native runtime).
//
// The reference has no forward pass: its draft and verify steps are virtual
// durations (request_model.py:92-117, called at
// engine.py:338, 359-360, 378, 402, 429).  Their B200 replacements run real
// forwards whose per-token metadata -- gather sources, RoPE positions, paged
// KV write slots, per-sequence query / key extents, LM-head rows, draft
// scatter targets -- the host computes every step from the committed lengths
// and the block table.  Doing it here (one pass over the rows, straight into
// the pinned staging buffer) instead of numpy takes the staging off the
// critical path at the start of each step (the GPU is idle until the draft
// graph is launched).
//
// Field order of a metadata set (offset / capacity pairs in `fields`) follows
// model.META_FIELDS: tokens, positions, slots, seq_slot, q_start, q_len,
// q_pos0, kv_len, logit_rows, gather_src, scatter_dst.
#include <cstdint>
#include <initializer_list>

#include "psd.h"

namespace {

enum Field { TOKENS, POSITIONS, SLOTS, SEQ_SLOT, Q_START, Q_LEN, Q_POS0, KV_LEN, LOGIT_ROWS,
             GATHER_SRC, SCATTER_DST, NFIELDS };

struct Table {
  const int32_t* bt;
  int ld;
  const int32_t* nblk;
  int bs;
  int replay;
  // paged KV slot of (slot, pos); -1 past the allocation in replay mode
  // (rows beyond the replayed commit write nowhere), error otherwise
  bool at(int s, int pos, int32_t* out) const {
    int bi = pos / bs;
    if (bi >= nblk[s]) {
      if (!replay) return false;
      *out = -1;
      return true;
    }
    *out = bt[(int64_t)s * ld + bi] * bs + pos % bs;
    return true;
  }
};

struct Set {
  int32_t* base;
  const int32_t* fields;
  int32_t* f(Field x) const { return base + fields[2 * x]; }
  bool fits(Field x, int n) const { return n <= fields[2 * x + 1]; }
};

}  // namespace

extern "C" int psd_stage_draft(int32_t* sets, int64_t set_stride, const int32_t* fields,
                               const int32_t* block_table, int bt_ld, const int32_t* nblk,
                               int block_size, int replay, int ldt, int scratch_slot,
                               const int32_t* slot, const int32_t* L, const int32_t* k, int n,
                               int nb, int kmax) {
  if (n < 0 || nb < n || kmax < 1 || block_size <= 0) return PSD_STAGE_BAD_ARGS;
  Table t{block_table, bt_ld, nblk, block_size, replay};
  Set s0{sets, fields};
  for (Field x : {POSITIONS, SLOTS, GATHER_SRC})
    if (!s0.fits(x, 2 * nb)) return PSD_STAGE_CAPACITY;
  for (Field x : {SEQ_SLOT, Q_START, Q_LEN, Q_POS0, KV_LEN, LOGIT_ROWS, SCATTER_DST})
    if (!s0.fits(x, nb)) return PSD_STAGE_CAPACITY;
  // set 0: the last two committed tokens of every row (the one before the
  // bonus token may lack draft KV); padding rows use the scratch slot
  for (int r = 0; r < nb; ++r) {
    const bool real = r < n;
    const int sl = real ? slot[r] : scratch_slot;
    const int Lr = real ? L[r] : 2;
    for (int j = 0; j < 2; ++j) {
      const int i = 2 * r + j, pos = Lr - 2 + j;
      int32_t kv;
      if (!t.at(sl, pos > 0 ? pos : 0, &kv)) return PSD_STAGE_KV_OVERRUN;
      s0.f(GATHER_SRC)[i] = sl * ldt + j;
      s0.f(POSITIONS)[i] = real ? pos : 0;
      s0.f(SLOTS)[i] = real ? kv : -1;
    }
    s0.f(SEQ_SLOT)[r] = sl;
    s0.f(Q_START)[r] = 2 * r;
    s0.f(Q_LEN)[r] = 2;
    s0.f(Q_POS0)[r] = real ? Lr - 2 : 0;
    s0.f(KV_LEN)[r] = real ? Lr : 1;
    s0.f(LOGIT_ROWS)[r] = 2 * r + 1;
    s0.f(SCATTER_DST)[r] = real ? sl * ldt + 2 : -1;
  }
  // sets 1 .. kmax-1: step i feeds the previous draft at position L - 1 + i
  for (int i = 1; i < kmax; ++i) {
    Set si{sets + i * set_stride, fields};
    for (int r = 0; r < nb; ++r) {
      const bool real = r < n;
      const int sl = real ? slot[r] : scratch_slot;
      const bool act = real && i < k[r];
      const int pos = act ? L[r] - 1 + i : 0;
      int32_t kv;
      if (!t.at(sl, pos, &kv)) return PSD_STAGE_KV_OVERRUN;
      si.f(GATHER_SRC)[r] = sl * ldt + 1 + i;
      si.f(POSITIONS)[r] = pos;
      si.f(SLOTS)[r] = act ? kv : -1;
      si.f(SEQ_SLOT)[r] = sl;
      si.f(Q_START)[r] = r;
      si.f(Q_LEN)[r] = 1;
      si.f(Q_POS0)[r] = pos;
      si.f(KV_LEN)[r] = act ? L[r] + i : 1;
      si.f(LOGIT_ROWS)[r] = r;
      si.f(SCATTER_DST)[r] = act ? sl * ldt + 2 + i : -1;
    }
  }
  return 0;
}

extern "C" int psd_stage_verify(int32_t* set, const int32_t* fields, const int32_t* block_table,
                                int bt_ld, const int32_t* nblk, int block_size, int replay,
                                int ldt, int scratch_slot, const int32_t* slot, const int32_t* L,
                                const int32_t* k, int n, int nb, int kmax) {
  if (n < 0 || nb < n || kmax < 0 || block_size <= 0) return PSD_STAGE_BAD_ARGS;
  const int K1 = kmax + 1;
  Table t{block_table, bt_ld, nblk, block_size, replay};
  Set s{set, fields};
  for (Field x : {POSITIONS, SLOTS, GATHER_SRC, LOGIT_ROWS})
    if (!s.fits(x, nb * K1)) return PSD_STAGE_CAPACITY;
  for (Field x : {SEQ_SLOT, Q_START, Q_LEN, Q_POS0, KV_LEN})
    if (!s.fits(x, nb)) return PSD_STAGE_CAPACITY;
  // K1 = k_max + 1 query tokens per row whatever the row's k_i (the
  // batch-invariant geometry); token j > k_i re-reads the bonus token and
  // writes no KV
  for (int r = 0; r < nb; ++r) {
    const bool real = r < n;
    const int sl = real ? slot[r] : scratch_slot;
    const int Lr = real ? L[r] : 1;
    const int kr = real ? k[r] : 0;
    for (int j = 0; j < K1; ++j) {
      const int i = r * K1 + j, pos = Lr - 1 + j;
      const bool wr = real && j <= kr;
      int32_t kv;
      if (!t.at(sl, wr ? pos : 0, &kv)) return PSD_STAGE_KV_OVERRUN;
      s.f(GATHER_SRC)[i] = sl * ldt + ((j == 0 || j > kr) ? 1 : 1 + j);
      s.f(POSITIONS)[i] = real ? pos : 0;
      s.f(SLOTS)[i] = wr ? kv : -1;
      s.f(LOGIT_ROWS)[i] = i;
    }
    s.f(SEQ_SLOT)[r] = sl;
    s.f(Q_START)[r] = r * K1;
    s.f(Q_LEN)[r] = K1;
    s.f(Q_POS0)[r] = real ? Lr - 1 : 0;
    s.f(KV_LEN)[r] = real ? Lr + kr : 1;
  }
  return 0;
}
