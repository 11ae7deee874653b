"""GpuBackend: the scheduler's passes as real sm_100a work.

Replaces the reference's two abstractions:
  * pass durations ``draft_latency`` / ``verify_latency .duration`` (engine.py:
    338, 359-360, 378, 402, 429) -> the draft model's k-step decode loop and the
    target model's verify forward over k+1 tokens per request (model.py),
    timed with CUDA events;
  * ``accepted_count(acceptance_stream(seed, rid, j))`` (engine.py:245-256)
    -> the fused verification kernel K1 (ops.verify_greedy / verify_sample)
    over the real logits.

Batch parallelism: the skip batch's draft loop runs on the *draft stream*
while the target batch is verified on the *target stream* (one GPU; a
dedicated draft GPU is the pair layout of pair.py, which runs one GpuBackend
per role on two ranks).  The only host sync per
step is the D2H of the verified rows' accepted lengths.

Per-request device state lives in "slots" (one per running request):
  slot_tok[s, 0..1]   last two committed tokens (inputs of the next draft)
  slot_tok[s, 2+i]    draft i of the pending draft
  generated[s], outputs[s, :]   committed output tokens
  block_table[s, :]   physical KV blocks (shared by target and draft caches)
KV sizing: a GPU cannot peek the next acceptance (the reference does,
engine.py:162-175), so grants reserve k_i + 1 positions and the rejected
tail is given back after the commit (KVBlockTable.trim_to_written).
"""

from __future__ import annotations

import gc
import time

import numpy as np
import torch

from . import native, ops
from .errors import ConfigError, KVError, ProtocolError
from .kvtable import BlockPool
from .model import PRESETS, Forward, ModelShape, Transformer, successor_table
from .scheduler import EngineState, StepPlan, StepResult, VerifyRow
from .workload import attach_prompt_ids

__all__ = ["GpuBackend"]


def _shape(x) -> ModelShape:
    if isinstance(x, ModelShape):
        return x
    if x not in PRESETS:
        raise ConfigError(f"unknown model preset {x!r}; known: {sorted(PRESETS)}")
    return PRESETS[x]


class GpuBackend:
    """Real draft / verify passes on a B200 (sm_100a)."""

    def __init__(self, target="llama-3.1-8b", draft="llama-3.2-1b", *, max_requests: int = 64,
                 max_batch: int = 64, k_max: int = 8, max_seq_len: int = 1024,
                 mode: str = "greedy", temperature: float = 1.0, seed: int = 0,
                 beta_target: float = 6.0, beta_draft: float = 12.0,
                 device: str | torch.device = "cuda:0", dual_stream: bool = True,
                 block_size: int = 16, num_blocks: int | None = None,
                 prefill_chunk_tokens: int = 4096, use_graphs: bool = True,
                 roles: tuple = ("target", "draft"), fused_draft: bool | None = None,
                 mk_grid: int = 0, tp=None, acceptance: str = "kernel") -> None:
        if not torch.cuda.is_available():
            raise native.NativeError("GpuBackend needs a CUDA device (no CPU fallback)")
        native.load()
        if mode not in ("greedy", "sample"):
            raise ConfigError(f"mode must be greedy or sample, got {mode!r}")
        if acceptance not in ("kernel", "replay"):
            raise ConfigError(f"acceptance must be kernel or replay, got {acceptance!r}")
        # replay: real draft / verify passes on real logits, but every verified
        # row accepts the reference's own coin-flip count accepted_count(model,
        # k, draft_time, acceptance_stream(seed, rid, j)) (acceptance_model.py:
        # 50-52, 82-97; engine.py:250-256) through K1's forced mode, KV grants
        # are sized exactly like the reference's (engine.py:162-175) and the
        # scheduler sees the latency models' virtual durations -- so the step
        # log, KV log and metrics equal specsim's byte for byte while the
        # measured CUDA-event durations go to ``measured_log``
        self.replay = acceptance == "replay"
        self.measured_log: list = []
        if self.replay:
            from .sim import SimBackend
            self._sim = SimBackend()
        if k_max > 16:
            raise ConfigError("k_max must be <= 16 (PSD_MAX_K)")
        self.tshape, self.dshape = _shape(target), _shape(draft)
        if self.dshape.vocab > self.tshape.vocab:
            raise ConfigError("draft vocabulary must not exceed the target vocabulary")
        self.device = torch.device(device)
        self.mode = mode
        self.temperature = float(temperature)
        self.seed = seed
        self.k_max = k_max
        self.max_requests = max_requests
        self.max_batch = max_batch
        self.block_size = block_size
        self.max_blocks = (max_seq_len + block_size - 1) // block_size + 1
        if num_blocks is None:
            num_blocks = max_requests * self.max_blocks + 1
        # block 0 is a reserved scratch block: unused slots point at it
        self.block_pool = BlockPool(num_blocks)
        self.block_pool.take(1)
        self.prefill_chunk = prefill_chunk_tokens
        self.beta_target, self.beta_draft = beta_target, beta_draft
        dev = self.device
        self.roles = set(roles)
        has_t, has_d = "target" in self.roles, "draft" in self.roles
        with torch.cuda.device(dev):
            # tp = (rank, size, process group): the target is a tensor-parallel
            # shard (model.py); every TP rank runs the same scheduler (SPMD), the
            # draft is replicated and K1 runs on the all-gathered logits
            self.tp = tp
            self.target = Transformer(self.tshape, dev, seed * 2 + 1, num_blocks, block_size,
                                      self.max_blocks, tp=tp) if has_t else None
            self.draft = Transformer(self.dshape, dev, seed * 2 + 2, num_blocks, block_size,
                                     self.max_blocks) if has_d else None
            i32 = torch.int32
            # one extra scratch slot (index max_requests) backs the padding
            # rows of bucketed batches; its block-table row is block 0
            self.scratch_slot = max_requests
            nslot = max_requests + 1
            self.block_table = torch.zeros(nslot, self.max_blocks, dtype=i32, device=dev)
            self.block_table_host = torch.zeros(nslot, self.max_blocks, dtype=i32).pin_memory()
            self.bt_np = self.block_table_host.numpy()
            self.bt_ptr = self.block_table_host.data_ptr()
            self.nblk = np.zeros(nslot, np.int32)
            self.nblk[self.scratch_slot] = 1
            # per-pass row arrays (slot, committed length, k) for the stagers
            self._rows_np = np.zeros((3, max_batch), np.int32)
            self.ldt = k_max + 2
            self.slot_tok = torch.zeros(nslot, self.ldt, dtype=i32, device=dev)
            self.generated = torch.zeros(max_requests, dtype=i32, device=dev)
            self.max_out = max_seq_len
            self.outputs = torch.full((max_requests, self.max_out), -1, dtype=i32, device=dev)
            succ = successor_table(self.tshape.vocab, self.dshape.vocab, seed)
            self.succ_t = torch.from_numpy(succ).to(dev)
            self.succ_d = torch.from_numpy(succ[:self.dshape.vocab].copy()).to(dev)
            B, K = max_batch, k_max
            # a prompt longer than a chunk is prefilled alone
            vt_tokens = max(B * (K + 1), prefill_chunk_tokens, max_seq_len)
            vd_tokens = max(2 * B, prefill_chunk_tokens, max_seq_len)
            self.tfwd = Forward(self.target, vt_tokens, max(B, 256), B * (K + 1),
                                self.block_table, sets=1, max_kv_len=0) if has_t else None
            self.dfwd = Forward(self.draft, vd_tokens, max(B, 256), B, self.block_table,
                                sets=K + 1, max_kv_len=0) if has_d else None
            self.tlogits = torch.empty(B * (K + 1), self.tshape.vocab, dtype=torch.float32,
                                       device=dev) if has_t else None
            self.dlogits = torch.empty(B, self.dshape.vocab, dtype=torch.float32,
                                       device=dev) if has_d else None
            if mode == "sample":
                # with a dedicated draft GPU (pair.py) the draft rank ships the q
                # rows of every drafted token to the target rank's qbuf
                # per-slot draft distributions q (fp32 logits after the bias);
                # K1 reads request b's rows at qbuf[slot_b] (verify_sample_rows)
                self.qbuf = torch.empty(nslot * K, self.dshape.vocab, dtype=torch.float32,
                                        device=dev)
                # their canonical (max, sum): written by the draft sampler, read by
                # K1 instead of re-streaming the q rows (psd_verify_sample_ext)
                self.qstats = torch.zeros(nslot * K, 2, dtype=torch.float32, device=dev)
                self.d_u = torch.empty(K, B, dtype=torch.float32, device=dev)
                self.v_u = torch.empty(B, K + 1, dtype=torch.float32, device=dev)
                # per-row (request id, committed length) keys of the uniforms
                # a ring of pinned staging rows: an async H2D copy reads its row
                # when it executes, so a row is rewritten only after the event
                # recorded behind its copy has completed (two draft loops may be
                # enqueued back to back without a host sync, e.g. startup steps)
                self.d_key_ring = 4
                self.d_key_host = torch.zeros(self.d_key_ring, 2 * B + K * B,
                                              dtype=i32).pin_memory()
                self.d_key_events = [None] * self.d_key_ring
                self.d_key_cur = 0
                self.d_key = torch.zeros(2 * B + K * B, dtype=i32, device=dev)
                self.v_key_host = torch.zeros(2 * B, dtype=i32).pin_memory()
                self.v_key = torch.zeros(2 * B, dtype=i32, device=dev)
                self.d_dummy = torch.zeros(B, 1, 4, dtype=torch.float32, device=dev)
            self.v_ids = torch.empty(B, K, dtype=i32, device=dev)
            self.v_acc = torch.empty(B, dtype=i32, device=dev)
            self.v_out = torch.empty(B * (K + 1), dtype=i32, device=dev)
            self.v_tok = torch.empty(B * (K + 1), dtype=i32, device=dev)  # argmax per row
            self.v_len = torch.empty(B, dtype=i32, device=dev)
            self.v_slot = torch.empty(B, dtype=i32, device=dev)
            # v_meta: [0, B) draft depths, [B, 2B) slots, [2B, 3B) replay counts,
            # [3B, 3B + BK) slot_tok indices of the drafts
            self.v_meta_host = torch.zeros(3 * B + B * K, dtype=i32).pin_memory()
            self.v_meta = torch.zeros(3 * B + B * K, dtype=i32, device=dev)
            self.acc_host = torch.zeros(B, dtype=i32).pin_memory()
            self.out_host = torch.zeros(B * (K + 1), dtype=i32).pin_memory()
            self.d_out = torch.empty(B, 1, dtype=i32, device=dev)
            self.d_acc = torch.empty(B, dtype=i32, device=dev)
            self.d_len0 = torch.zeros(B, dtype=i32, device=dev)
            self.d_ids0 = torch.zeros(B, 0, dtype=i32, device=dev)
            # stream priorities (PSD_STREAM_PRIO=none|draft|target) measured no
            # gain for the overlapped step (profiles/r01b_stream_priority.txt)
            import os
            prio = os.environ.get("PSD_STREAM_PRIO", "none")
            hi, lo = -1, 0
            self.s_target = torch.cuda.Stream(dev, priority=hi if prio == "target" else lo)
            self.s_draft = (torch.cuda.Stream(dev, priority=hi if prio == "draft" else lo)
                            if dual_stream else self.s_target)
            torch.cuda.synchronize(dev)
        # fused k-step greedy draft decode (csrc/decode_mk.cu, experimental
        # build only): one persistent kernel per draft loop instead of ~130
        # launches per step; measured 35 % slower, off by default
        import os
        self.mk = None
        want_mk = fused_draft if fused_draft is not None else \
            os.environ.get("PSD_FUSED_DRAFT", "0") == "1"
        if want_mk and not native.has("psd_mk_create"):
            raise ConfigError("fused_draft needs the experimental build (PSD_EXPERIMENTAL=1 "
                              "python -m paper_2603_18016_b200.build_native)")
        if want_mk and has_d and mode == "greedy":
            grid = mk_grid or int(os.environ.get("PSD_MK_GRID", "0"))
            with torch.cuda.device(dev):
                self.mk = self._make_mk(grid)
        self._step_events = None
        self._bt_sig = {}  # slot -> (request, block-list version) on the host table
        self.draft_first = os.environ.get("PSD_DRAFT_FIRST", "0") == "1"
        # greedy verification through the target LM head's argmax epilogue
        # (PSD_K1_EPI=0: stored logits + K1, for A/B runs)
        self.k1_epi = os.environ.get("PSD_K1_EPI", "1") == "1"
        # K6: the greedy draft's argmax (+ bias) in its LM-head epilogue
        # (PSD_K6=0: logits + bigram + K1(k = 0) + scatter, for A/B runs)
        self.k6 = (os.environ.get("PSD_K6", "1") == "1" and has_d
                   and self.dshape.vocab % 128 == 0 and max_batch <= 128)
        # verify GEMM grids capped below the SM count when the draft loop runs
        # beside them (dual stream): PSD_VERIFY_CTAS (0 = all SMs)
        # Default from the drafting / verify weight-volume ratio r = k x draft
        # weights / target weights (measured optima, profiles/r01b_verify_cta_cap.txt):
        # r >= 1/2 (cfg2, r = 0.82): 92; 1/4 <= r < 1/2 (cfg3, r = 0.28): 104;
        # r < 1/4 (cfg4, r = 0.07): no cap -- the verify is the critical path
        env_cap = os.environ.get("PSD_VERIFY_CTAS")
        if not dual_stream or not (has_t and has_d):
            self.verify_ctas = 0
        elif env_cap is not None:
            self.verify_ctas = int(env_cap)
        else:
            wb = lambda m: sum(t.numel() for L in m.layers for t in L.values()  # noqa: E731
                               if isinstance(t, torch.Tensor)) + m.lm_head.numel()
            r = k_max * wb(self.draft) / max(1, wb(self.target))
            self.verify_ctas = 92 if r >= 0.5 else 104 if r >= 0.25 else 0
        # and the draft GEMM grids (persistent stream-K grids sized to the SMs
        # the verify leaves free): PSD_DRAFT_CTAS (0 = all SMs)
        self.draft_ctas = int(os.environ.get("PSD_DRAFT_CTAS", "0")) if dual_stream else 0
        # PSD_QSTATS_CACHE=0 makes K1 re-read the draft rows (A/B runs)
        self.qstats_cache = os.environ.get("PSD_QSTATS_CACHE", "1") == "1"
        # set when a dedicated draft GPU ships the q statistics with the q rows
        self.qstats_remote = False
        self.c3_part = self.c3_all = None  # TP greedy: K1 partials of this shard / all
        self.seed_draft = (seed * 0x9E3779B1 + 0xD7A7) & 0xFFFFFFFFFFFF
        self.seed_verify = (seed * 0x85EBCA77 + 0x7E51) & 0xFFFFFFFFFFFF
        self.capture_verify = None  # set to a list to record K1 inputs (tests)
        self.use_graphs = use_graphs
        self.graphs: dict[tuple, torch.cuda.CUDAGraph] = {}
        self.graph_streams: list = []
        self.graph_launches: dict[tuple, int] = {}
        self.launches = 0  # kernels of libpsd.so executed (graph replays included)
        # bytes this backend copied host -> device / device -> host (e2e accounting)
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.slots: dict[int, int] = {}
        self.free_slots = list(range(max_requests - 1, -1, -1))
        self.pending_k: dict[int, int] = {}
        self.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0}
        self._state: EngineState | None = None

    def _make_mk(self, grid: int):
        """Bind the draft model and its forward buffers to the fused decode
        kernel; None when the shape is outside its envelope (head_dim 32/64,
        hidden <= 4096, <= 16 query rows per kv head)."""
        import ctypes
        lib = native.load()
        m, f, s = self.draft, self.dfwd, self.dshape
        ptrs = []
        for li, L in enumerate(m.layers):
            ptrs += [L["wqkv"].data_ptr(), L["wo"].data_ptr(), L["wgu"].data_ptr(),
                     L["wdown"].data_ptr(), L["attn_norm"].data_ptr(), L["mlp_norm"].data_ptr(),
                     L["bqkv"].data_ptr() if L["bqkv"] is not None else 0,
                     m.kv[li, 0].data_ptr(), m.kv[li, 1].data_ptr()]
        self._mk_ptrs = (ctypes.c_void_p * len(ptrs))(*ptrs)
        self._mk_argpart = torch.empty(s.vocab // 128 * 64 * 2, dtype=torch.float32,
                                       device=self.device)
        mm = native.MkModel()
        mm.layers, mm.hidden, mm.heads, mm.kv_heads = s.layers, s.hidden, s.heads, s.kv_heads
        mm.head_dim, mm.ffn, mm.vocab = s.head_dim, s.ffn_padded, s.vocab
        mm.eps, mm.attn_scale, mm.beta = s.rms_eps, 1.0 / (s.head_dim ** 0.5), self.beta_draft
        mm.block_size, mm.max_blocks, mm.grid = self.block_size, self.max_blocks, grid
        mm.max_tokens = f.max_tokens
        mm.layer_ptrs = ctypes.cast(self._mk_ptrs, ctypes.c_void_p)
        mm.embed, mm.lm_head = m.embed.data_ptr(), m.lm_head.data_ptr()
        mm.final_norm, mm.inv_freq = m.final_norm.data_ptr(), m.inv_freq.data_ptr()
        mm.successor, mm.block_table = self.succ_d.data_ptr(), self.block_table.data_ptr()
        mm.x, mm.xn, mm.attn = f.x.data_ptr(), f.xn.data_ptr(), f.attn.data_ptr()
        mm.act, mm.xf, mm.part = f.act.data_ptr(), f.xf.data_ptr(), f.part.data_ptr()
        mm.argpart, mm.slot_tok = self._mk_argpart.data_ptr(), self.slot_tok.data_ptr()
        mm.meta, mm.set_stride = f.meta.data_ptr(), f.set_size
        from .model import META_FIELDS
        for i, name in enumerate(META_FIELDS):
            mm.field_offsets[i] = f._offsets[name][0]
        h = lib.psd_mk_create(ctypes.byref(mm))
        return h or None

    def close(self) -> None:
        if getattr(self, "mk", None):
            native.load().psd_mk_destroy(self.mk)
            self.mk = None

    # ------------------------------------------------------------------
    # Backend protocol
    # ------------------------------------------------------------------
    def bind(self, state: EngineState) -> None:
        if state.config.block_size != self.block_size:
            raise ConfigError(f"SimConfig.block_size {state.config.block_size} != KV cache "
                              f"block size {self.block_size}")
        if state.config.k > self.k_max or any(k > self.k_max for k in state.config.k_overrides):
            raise ConfigError(f"draft depth exceeds k_max={self.k_max}")
        cfg = state.config
        width = cfg.m * (max(1, cfg.sd_batch_factor) if cfg.mode == "standard-sd" else 1)
        if width > self.max_batch:
            raise ConfigError(f"batch width {width} (m={cfg.m}, mode {cfg.mode}) exceeds "
                              f"max_batch={self.max_batch}")
        running = cfg.m * (max(1, cfg.sd_batch_factor) if cfg.mode == "standard-sd" else 2)
        if min(running, len(state.requests)) > self.max_requests:
            raise ConfigError(f"up to {min(running, len(state.requests))} concurrent requests "
                              f"need slots, max_requests={self.max_requests}")
        need = [r for r in state.requests.values() if r.prompt_ids is None]
        if need:
            attach_prompt_ids(need, self.dshape.vocab, self.seed)
        for r in state.requests.values():
            if r.prompt_len < 2:
                raise ConfigError(f"request {r.id}: GPU backend needs prompt_len >= 2")
            if len(r.prompt_ids) != r.prompt_len:
                raise ConfigError(f"request {r.id}: prompt_ids length != prompt_len")
            if r.prompt_len + r.target_output_len + self.k_max + 1 > self.max_out:
                raise ConfigError(f"request {r.id} exceeds max_seq_len={self.max_out}")
        self._state = state
        if self.replay:
            self._sim.bind(state)

    def estimate(self, state, plan):
        if self.replay:  # the draft_time the reference's acceptance law sees
            return self._sim.estimate(state, plan)
        return 0.0, 0.0, 0.0

    def planned_commit(self, state, rid, k_i, draft_time):
        if self.replay:  # exact sizing: peek the row's acceptance stream
            return self._sim.planned_commit(state, rid, k_i, draft_time)
        return min(k_i + 1, state.requests[rid].remaining)

    def commit(self, state, rid, tokens):
        if self.replay:
            return  # grants were exact (or eager k_i + 1, kept as the reference does)
        # roll back the reserved-but-rejected tail: keep blocks for the
        # committed tokens only (the reference's exact-size invariant)
        state.kv.trim_to_written(rid)

    def retire(self, state, rid):
        s = self.slots.pop(rid, None)
        if s is None:
            return
        req = state.requests[rid]
        n = req.generated
        req.output_ids = self.outputs[s, :n].cpu().tolist()
        self.d2h_bytes += 4 * n
        self._bt_sig.pop(s, None)
        self.free_slots.append(s)
        self.pending_k.pop(rid, None)

    # ------------------------------------------------------------------
    # helpers
    # ------------------------------------------------------------------
    def _kv_slot(self, state, rid: int, pos: int) -> int:
        blocks = state.kv.blocks_of(rid)
        bi = pos // self.block_size
        if bi >= len(blocks):
            raise KVError(f"request {rid}: KV position {pos} beyond its {len(blocks)} blocks")
        return blocks[bi] * self.block_size + pos % self.block_size

    def _h2d(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        """Stream-ordered copy of pinned host staging into a same-sized device
        buffer on the current stream (psd_copy_async: no torch dispatch)."""
        native.check(native.load().psd_copy_async(
            dst.data_ptr(), src.data_ptr(), src.numel() * src.element_size(),
            torch.cuda.current_stream(self.device).cuda_stream), "h2d copy")

    def _upload_block_table(self, state) -> None:
        """Host block table -> device.  Rows are rewritten only for slots whose
        (request, block-list version) changed; rows of free slots are never
        read (no batch references them)."""
        bt = self.bt_np
        sig = self._bt_sig
        kv = state.kv
        for rid, s in self.slots.items():
            key = (rid, kv.list_version(rid))
            if sig.get(s) == key:
                continue
            blocks = kv.blocks_of(rid)
            n = len(blocks)
            if n > self.max_blocks:
                raise KVError(f"request {rid}: {n} blocks > max {self.max_blocks}")
            bt[s, :n] = blocks
            bt[s, n:] = 0
            self.nblk[s] = n
            sig[s] = key
        self._h2d(self.block_table, self.block_table_host)
        self.h2d_bytes += self.block_table_host.numel() * 4

    def _admit(self, state, ids) -> None:
        """Assign slots and initialise slot tokens for new requests."""
        triples = []
        for rid in ids:
            if not self.free_slots:
                raise ProtocolError("GpuBackend: out of request slots")
            s = self.free_slots.pop()
            self.slots[rid] = s
            p = state.requests[rid].prompt_ids
            triples.append((s, p[-2], p[-1]))
        self._init_slots(triples, reset_generated=True)

    def _init_slots(self, triples, reset_generated: bool = False) -> None:
        """slot_tok[s, 0:2] = (tok_prev, tok_last) for (s, tok_prev, tok_last)."""
        n = len(triples)
        if n == 0:
            return
        idx = np.empty(2 * n, dtype=np.int32)
        val = np.empty(2 * n, dtype=np.int32)
        for i, (s, tp, tl) in enumerate(triples):
            idx[2 * i:2 * i + 2] = (s * self.ldt, s * self.ldt + 1)
            val[2 * i:2 * i + 2] = (tp, tl)
        dev = self.device
        stage = torch.from_numpy(np.concatenate([idx, val])).pin_memory().to(dev,
                                                                            non_blocking=True)
        self.h2d_bytes += stage.numel() * 4
        st = torch.cuda.current_stream(dev).cuda_stream
        lib = native.load()
        native.check(lib.psd_index_copy_i32(self.slot_tok.data_ptr(), stage.data_ptr(),
                                            stage[2 * n:].data_ptr(), None, 2 * n, st),
                     "slot init")
        self.launches += 1
        if reset_generated:
            sl = torch.tensor([t[0] for t in triples], dtype=torch.int64)
            self.generated[sl.to(dev)] = 0
            self.h2d_bytes += 8 * len(triples)

    def _set_slot_values(self, pairs) -> None:
        """slot_tok.view(-1)[flat] = value for (flat, value) pairs (draft ids
        arriving from a dedicated draft GPU)."""
        n = len(pairs)
        if n == 0:
            return
        arr = np.asarray(pairs, dtype=np.int32).T.reshape(-1)
        stage = torch.from_numpy(arr).pin_memory().to(self.device, non_blocking=True)
        self.h2d_bytes += stage.numel() * 4
        st = torch.cuda.current_stream(self.device).cuda_stream
        native.check(native.load().psd_index_copy_i32(
            self.slot_tok.data_ptr(), stage.data_ptr(), stage[n:].data_ptr(), None, n, st),
            "slot values")
        self.launches += 1

    def _prefill(self, state, ids, fwd: Forward, logits_model: str) -> None:
        self._prefill_rows([(self.slots[rid], state.requests[rid].prompt_ids) for rid in ids],
                           fwd)

    def _prefill_rows(self, rows, fwd: Forward) -> None:
        """Prompt tokens 0..p-2 of each (slot, prompt_ids) through one model."""
        chunks, cur, cur_tok = [], [], 0
        for row in rows:
            n = len(row[1]) - 1
            if cur and cur_tok + n > self.prefill_chunk:
                chunks.append(cur)
                cur, cur_tok = [], 0
            cur.append(row)
            cur_tok += n
        if cur:
            chunks.append(cur)
        for chunk in chunks:
            toks, pos, slots = [], [], []
            seq_slot, q_start, q_len, q_pos0, kv_len = [], [], [], [], []
            for slot, prompt in chunk:
                n = len(prompt) - 1
                q_start.append(len(toks))
                toks.extend(prompt[:n])
                pos.extend(range(n))
                slots.extend(self._slots_at(np.full(n, slot), np.arange(n)).tolist())
                seq_slot.append(slot)
                q_len.append(n)
                q_pos0.append(0)
                kv_len.append(n)
            if len(toks) > fwd.max_tokens:
                raise ConfigError("prompt longer than the prefill chunk")
            fwd.begin()
            fwd.stage(0, {"tokens": np.asarray(toks, np.int32),
                          "positions": np.asarray(pos, np.int32),
                          "slots": np.asarray(slots, np.int32),
                          "seq_slot": np.asarray(seq_slot, np.int32),
                          "q_start": np.asarray(q_start, np.int32),
                          "q_len": np.asarray(q_len, np.int32),
                          "q_pos0": np.asarray(q_pos0, np.int32),
                          "kv_len": np.asarray(kv_len, np.int32)})
            fwd.upload(1)
            lib = native.load()
            c0 = lib.psd_launch_count()
            # whole-K GEMM geometry: a prompt's KV cache is the same whatever
            # else shares its chunk (requests are admitted in different groups
            # by PSD, SD(m) and SD(2m) -- continuous batching)
            lib.psd_gemm_set_whole_k(1)
            try:
                fwd.run(len(toks), len(chunk), max(q_len), 0, None)
            finally:
                lib.psd_gemm_set_whole_k(0)
            self.launches += lib.psd_launch_count() - c0

    # ---- bucketed, graph-captured device passes ------------------------
    def _bucket(self, n: int) -> int:
        return min(self.max_batch, max(8, (n + 7) // 8 * 8))

    def _slots_at(self, slot_rows: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """KV write slots of (slot, position) pairs from the host block table.
        Replay mode grants exactly the next commit, so draft / verify rows past
        it (beyond the replayed acceptance, never committed) write nowhere (-1)."""
        bi = pos // self.block_size
        beyond = bi >= self.nblk[slot_rows]
        if beyond.any():
            if not self.replay:
                raise KVError("KV position beyond the request's allocated blocks")
            bi = np.where(beyond, 0, bi)
            return np.where(beyond, -1,
                            self.bt_np[slot_rows, bi] * self.block_size + pos % self.block_size)
        return self.bt_np[slot_rows, bi] * self.block_size + pos % self.block_size

    def _run_graph(self, key, launch) -> None:
        """Replay the CUDA graph for ``key`` on the current stream, capturing
        it from ``launch`` on first use (the first use also runs eagerly)."""
        lib = native.load()
        g = self.graphs.get(key)
        if g is not None:
            g.replay()
            self.launches += self.graph_launches[key]
            return
        c0 = lib.psd_launch_count()
        launch()  # eager: correct results now, warms every kernel / workspace
        self.launches += lib.psd_launch_count() - c0
        if not self.use_graphs:
            return
        cur = torch.cuda.current_stream(self.device)
        # captured kernel nodes keep the capture stream's priority
        cs = torch.cuda.Stream(self.device, priority=cur.priority)
        self.graph_streams.append(cs)  # keep handles unique (per-stream K1 workspaces)
        cs.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        c0 = lib.psd_launch_count()
        # a dead reference cycle holding an old CUDAGraph, collected while
        # this stream captures, would destroy that graph mid-capture (an
        # unsafe call that invalidates the capture): collect first, and keep
        # the cyclic collector off until the capture ends
        gc.collect()
        gc_was_enabled = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                launch()
        finally:
            if gc_was_enabled:
                gc.enable()
        self.graph_launches[key] = lib.psd_launch_count() - c0
        cur.wait_stream(cs)
        self.graphs[key] = g

    def _draft_loop(self, state, ids, quotas) -> None:
        """k-step draft decode for the rows in ``ids`` (k_i = quotas[rid])."""
        for rid in ids:
            self.pending_k[rid] = quotas[rid]
        self._draft_rows([(rid, self.slots[rid],
                           state.requests[rid].prompt_len + state.requests[rid].generated,
                           quotas[rid]) for rid in ids if quotas[rid] > 0])

    def _stage_rows(self, n: int, nb: int, L_pad: int):
        """(slot, L, k) row arrays padded to nb (scratch slot, L_pad, 0)."""
        a = self._rows_np
        sl, L, k = a[0, :nb], a[1, :nb], a[2, :nb]
        sl[n:] = self.scratch_slot
        L[n:] = L_pad
        k[n:] = 0
        return sl, L, k

    def _stage_check(self, rc: int, what: str) -> None:
        if rc == 0:
            return
        if rc == native.STAGE_KV_OVERRUN:
            raise KVError(f"{what}: KV position beyond the request's allocated blocks")
        raise ConfigError(f"{what}: metadata staging failed ({rc})")

    def _draft_rows(self, draft_rows) -> None:
        """k-step draft decode of (rid, slot, committed length L, k) rows; the
        drafts land in slot_tok[slot, 2..2+k).  The forward metadata of all
        k steps is staged natively (psd_stage_draft)."""
        if not draft_rows:
            return
        n = len(draft_rows)
        nb = self._bucket(n)
        sl, L, k = self._stage_rows(n, nb, 2)
        sl[:n] = [r[1] for r in draft_rows]
        L[:n] = [r[2] for r in draft_rows]
        k[:n] = [r[3] for r in draft_rows]
        kmax = int(k[:n].max())
        fwd = self.dfwd
        fwd.begin()
        self._stage_check(native.load().psd_stage_draft(
            fwd.host_set_ptr(0), fwd.set_size, fwd.fields_ptr, self.bt_ptr, self.max_blocks,
            self.nblk.ctypes.data, self.block_size, int(self.replay), self.ldt, self.scratch_slot,
            sl.ctypes.data, L.ctypes.data, k.ctypes.data, n, nb, kmax), "draft staging")
        fwd.upload(kmax)
        if self.mode == "sample":
            self.d_key_cur = (self.d_key_cur + 1) % self.d_key_ring
            ev = self.d_key_events[self.d_key_cur]
            if ev is not None:
                ev.synchronize()
            kh = self.d_key_host[self.d_key_cur].numpy()
            B = self.max_batch
            real = np.arange(nb) < n
            kh[:nb] = [r[0] for r in draft_rows] + [0] * (nb - n)
            kh[B:B + nb] = L
            # q storage row of (row r, step i): slot * k_max + i (scratch slot for padding)
            K = self.k_max
            for i in range(kmax):
                kh[2 * B + i * B:2 * B + i * B + nb] = np.where(real & (i < k), sl * K + i, -1)
            self._h2d(self.d_key, self.d_key_host[self.d_key_cur])
            self.h2d_bytes += self.d_key.numel() * 4
            ev = torch.cuda.Event()
            ev.record()
            self.d_key_events[self.d_key_cur] = ev
        self._run_graph(("draft", nb, kmax), lambda: self._draft_launch_capped(nb, kmax))

    def _draft_launch_capped(self, nb: int, kmax: int) -> None:
        lib = native.load()
        lib.psd_gemm_set_max_ctas(self.draft_ctas)
        try:
            self._draft_launch(nb, kmax)
        finally:
            lib.psd_gemm_set_max_ctas(0)

    def _draft_launch(self, nb: int, kmax: int) -> None:
        fwd = self.dfwd
        lib = native.load()
        st = torch.cuda.current_stream(self.device).cuda_stream
        if self.mk is not None and 2 * nb <= 64:
            native.check(lib.psd_mk_launch(self.mk, nb, kmax, st), "fused draft decode")
            return
        for i in range(kmax):
            M = 2 * nb if i == 0 else nb
            native.check(lib.psd_index_copy_i32(fwd.view("tokens", i).data_ptr(), None,
                                                self.slot_tok.data_ptr(),
                                                fwd.view("gather_src", i).data_ptr(), M, st),
                         "draft gather")
            if self.mode == "greedy" and self.k6:
                # K6: argmax (+ bias) in the LM head's epilogue, the fold
                # scatters the token into its slot -- no logits, no K1 launch
                fwd.run(M, nb, 2 if i == 0 else 1, nb, None, self.dshape.vocab,
                        bigram=(self.succ_d, self.beta_draft), set_index=i,
                        argmax_into=(self.d_out[:nb], self.slot_tok,
                                     fwd.view("scatter_dst", i)))
                continue
            fwd.run(M, nb, 2 if i == 0 else 1, nb, self.dlogits, self.dshape.vocab,
                    bigram=(self.succ_d, self.beta_draft), set_index=i)
            if self.mode == "greedy":
                ops.verify_greedy(self.dlogits[:nb].view(nb, 1, -1), self.d_ids0[:nb],
                                  self.d_len0[:nb], self.d_acc[:nb], self.d_out[:nb])
            else:
                B = self.max_batch
                V = self.dshape.vocab
                # keep q for the verifier, then sample the draft token from q
                native.check(lib.psd_copy_rows_f32(
                    self.qbuf.data_ptr(), self.d_key[2 * B + i * B:].data_ptr(), V,
                    self.dlogits.data_ptr(), V, nb, V, st), "q rows")
                u = self.d_u[i, :nb]
                native.check(lib.psd_philox_uniforms(
                    self.seed_draft, self.d_key.data_ptr(), self.d_key[B:].data_ptr(), nb, 1, i,
                    u.data_ptr(), st), "draft uniforms")
                ops.verify_sample(self.dlogits[:nb].view(nb, 1, -1), self.d_dummy[:nb, :0],
                                  self.d_ids0[:nb], self.d_len0[:nb], u.view(nb, 1),
                                  self.temperature, self.d_acc[:nb], self.d_out[:nb],
                                  t_stats_out=self.qstats,
                                  t_stats_rows=self.d_key[2 * B + i * B:2 * B + i * B + nb])
            native.check(lib.psd_index_copy_i32(self.slot_tok.data_ptr(),
                                                fwd.view("scatter_dst", i).data_ptr(),
                                                self.d_out.data_ptr(), None, nb, st),
                         "draft scatter")

    def _verify(self, state, rows: list[VerifyRow], beside_draft: bool = False) -> int:
        """Stage and launch the verify pass; returns the number of real rows
        whose accepted lengths land in ``acc_host``."""
        n = len(rows)
        nb = self._bucket(n)
        # every verify pass has k_max + 1 query tokens per row, whatever this
        # batch's deepest draft: a token's attention then runs with the same
        # warp / key-group split in every pass (batch-invariant numerics, so
        # greedy PSD, SD(m) and SD(2m) emit identical tokens); rows with k_i <
        # k_max neither write KV past their drafts nor accept beyond k_i
        kmax = self.k_max
        K1 = kmax + 1
        ldt = self.ldt
        sl, L, k = self._stage_rows(n, nb, 1)
        for r, row in enumerate(rows):
            rid = row.request_id
            if row.k != self.pending_k.get(rid, 0):
                raise ProtocolError(f"request {rid}: verifying {row.k} drafts, device holds "
                                    f"{self.pending_k.get(rid, 0)}")
            sl[r] = self.slots[rid]
            req = state.requests[rid]
            L[r] = req.prompt_len + req.generated
            k[r] = row.k
        real = np.arange(nb) < n
        fwd = self.tfwd
        fwd.begin()
        self._stage_check(native.load().psd_stage_verify(
            fwd.host_set_ptr(0), fwd.fields_ptr, self.bt_ptr, self.max_blocks,
            self.nblk.ctypes.data, self.block_size, int(self.replay), ldt, self.scratch_slot,
            sl.ctypes.data, L.ctypes.data, k.ctypes.data, n, nb, kmax), "verify staging")
        fwd.upload(1)
        vm = self.v_meta_host.numpy()
        B = self.max_batch
        vm[:nb] = k
        vm[B:B + nb] = np.where(real, sl, -1)
        if self.replay:
            from .acceptance import acceptance_stream, accepted_count
            cfg = state.config
            forced = [accepted_count(cfg.acceptance, r.k, r.draft_time,
                                     acceptance_stream(cfg.seed, r.request_id, r.j))
                      if r.k > 0 else 0 for r in rows]
            vm[2 * B:2 * B + nb] = forced + [0] * (nb - n)
        if kmax:
            vm[3 * B:3 * B + nb * kmax] = (sl[:, None] * ldt + 2 + np.arange(kmax)[None, :]
                                           ).reshape(-1)
        self._h2d(self.v_meta, self.v_meta_host)
        self.h2d_bytes += self.v_meta_host.numel() * 4
        if self.mode == "sample":
            kh = self.v_key_host.numpy()
            kh[:nb] = [r.request_id for r in rows] + [0] * (nb - n)
            kh[B:B + nb] = L
            self._h2d(self.v_key, self.v_key_host)
            self.h2d_bytes += self.v_key_host.numel() * 4
        capped = beside_draft and self.verify_ctas > 0
        self._run_graph(("verify", nb, kmax, capped, self.replay),
                        lambda: self._verify_launch(nb, kmax, capped))
        if self.capture_verify is not None:
            torch.cuda.current_stream(self.device).synchronize()
            V = self.tshape.vocab
            rec = {"forced": vm[2 * B:2 * B + n].copy() if self.replay else None,
                   "target": self.tlogits[:nb * K1].view(nb, K1, V)[:n].cpu().numpy(),
                   "ids": self.v_ids.view(-1)[:nb * kmax].view(nb, kmax)[:n].cpu().numpy(),
                   "len": k[:n].astype(np.int32), "acc": self.v_acc[:n].cpu().numpy(),
                   "out": self.v_out[:nb * K1].view(nb, K1)[:n].cpu().numpy()}
            if self.mode == "sample":
                Vd = self.dshape.vocab
                q = self.qbuf.view(-1, self.k_max, Vd)
                rec["draft"] = q[torch.as_tensor(sl[:n])][:, :kmax].cpu().numpy()
                rec["uniforms"] = self.v_u.view(-1)[:nb * K1].view(nb, K1)[:n].cpu().numpy()
            self.capture_verify.append(rec)
        return n

    def _verify_launch(self, nb: int, kmax: int, capped: bool = False) -> None:
        lib = native.load()
        lib.psd_gemm_set_max_ctas(self.verify_ctas if capped else 0)
        try:
            self._verify_launch_inner(nb, kmax)
        finally:
            lib.psd_gemm_set_max_ctas(0)

    def _verify_launch_inner(self, nb: int, kmax: int) -> None:
        K1 = kmax + 1
        B = self.max_batch
        lib = native.load()
        st = torch.cuda.current_stream(self.device).cuda_stream
        fwd = self.tfwd
        M = nb * K1
        native.check(lib.psd_index_copy_i32(fwd.view("tokens").data_ptr(), None,
                                            self.slot_tok.data_ptr(),
                                            fwd.view("gather_src").data_ptr(), M, st),
                     "verify gather")
        # tensor-parallel greedy target over peer memory: each rank reduces its
        # LM-head vocabulary shard to K1 partials, the ranks all-gather the
        # partials (KBs instead of M x V logits) and fold them identically
        c3 = (self.mode == "greedy" and fwd.comm is not None and self.capture_verify is None)
        # greedy K1 fused into the LM head: the K6 epilogue reduces each logit
        # row to (max, argmax) per vocabulary tile, a fold gives the argmax
        # token per row, one warp per request decides -- no M x V logits are
        # stored or re-read (same decisions as K1 on the stored logits)
        tp = self.target.tp
        k1_epi = (self.mode == "greedy" and self.k1_epi and (tp is None or tp[1] <= 1)
                  and self.capture_verify is None and M <= fwd.amax_rows)
        if k1_epi:
            fwd.run(M, nb, K1, M, None, self.tshape.vocab,
                    bigram=(self.succ_t, self.beta_target),
                    argmax_into=(self.v_tok[:M], None, None))
        else:
            fwd.run(M, nb, K1, M, self.tlogits, self.tshape.vocab,
                    bigram=(self.succ_t, self.beta_target), shard_out=c3)
        v_len = self.v_meta[:nb]
        v_slot = self.v_meta[B:B + nb]
        forced = self.v_meta[2 * B:2 * B + nb] if self.replay else None
        if kmax:
            native.check(lib.psd_index_copy_i32(self.v_ids.data_ptr(), None,
                                                self.slot_tok.data_ptr(),
                                                self.v_meta[3 * B:].data_ptr(), nb * kmax, st),
                         "verify ids")
            v_ids = self.v_ids.view(-1)[:nb * kmax].view(nb, kmax)
        else:
            v_ids = self.v_ids[:nb, :0]
        logits = self.tlogits[:M].view(nb, K1, -1)
        out = self.v_out[:nb * K1].view(nb, K1)
        if c3:
            tm = self.target
            vs, vp = tm.vocab_shard, tm.shape.vocab
            cnt = lib.psd_verify_partials_count(nb, kmax, vs)
            if self.c3_part is None:
                full = lib.psd_verify_partials_count(B, self.k_max, vs)
                self.c3_part = torch.empty(full, dtype=torch.float32, device=self.device)
                self.c3_all = torch.empty(tm.tp[1] * full, dtype=torch.float32,
                                          device=self.device)
            native.check(lib.psd_verify_greedy_partials(
                fwd.lshard.data_ptr(), K1 * vp, vp, vs, tm.tp[0] * vs, v_len.data_ptr(), nb,
                kmax, self.c3_part.data_ptr(), st), "verify partials (shard)")
            fwd.comm.allgather(self.c3_part[:cnt], self.c3_all)
            native.check(lib.psd_verify_greedy_fold(
                self.c3_all.data_ptr(), tm.tp[1], vs, v_ids.data_ptr(), v_len.data_ptr(), nb,
                kmax, forced.data_ptr() if forced is not None else None, self.v_acc.data_ptr(),
                out.data_ptr(), st), "verify fold (shards)")
        elif k1_epi:
            native.check(lib.psd_verify_greedy_tokens(
                self.v_tok.data_ptr(), v_ids.data_ptr(), v_len.data_ptr(), nb, kmax,
                forced.data_ptr() if forced is not None else None, self.v_acc.data_ptr(),
                out.data_ptr(), st), "verify (argmax tokens)")
        elif self.mode == "greedy":
            ops.verify_greedy(logits, v_ids, v_len, self.v_acc[:nb], out, forced_len=forced)
        else:
            native.check(lib.psd_philox_uniforms(
                self.seed_verify, self.v_key.data_ptr(), self.v_key[B:].data_ptr(), nb, K1, 0,
                self.v_u.data_ptr(), st), "verify uniforms")
            Vd = self.dshape.vocab
            ws = ops._verify_workspace(self.device, nb, kmax, self.tshape.vocab, Vd, True)
            # the q statistics are cached when this process drew the drafts, or
            # shipped with the q rows by a dedicated draft GPU (pair.py)
            cached = ("draft" in self.roles or self.qstats_remote) and self.qstats_cache
            native.check(lib.psd_verify_sample_forced(
                logits.data_ptr(), K1 * self.tshape.vocab, self.tshape.vocab,
                self.tshape.vocab, self.qbuf.data_ptr(), v_slot.data_ptr(), self.k_max * Vd, Vd,
                Vd, v_ids.data_ptr(), v_len.data_ptr(), self.v_u.data_ptr(), self.temperature, nb,
                kmax, forced.data_ptr() if forced is not None else None, self.v_acc.data_ptr(),
                out.data_ptr(), self.qstats.data_ptr() if cached else None, self.k_max, None,
                None, ws.data_ptr(), ws.numel(), st), "verify_sample")
        native.check(lib.psd_commit(self.v_acc.data_ptr(), out.data_ptr(), kmax,
                                    v_slot.data_ptr(), nb, self.generated.data_ptr(),
                                    self.slot_tok.data_ptr(), self.ldt, self.outputs.data_ptr(),
                                    self.max_out, st), "commit")
        self.acc_host[:nb].copy_(self.v_acc[:nb], non_blocking=True)
        self.out_host[:nb * K1].copy_(self.v_out[:nb * K1], non_blocking=True)
        self.d2h_bytes += 4 * nb * (K1 + 1)

    def transfer_bytes(self) -> tuple[int, int]:
        """(host -> device, device -> host) bytes copied so far, the forwards'
        metadata uploads included."""
        h2d = self.h2d_bytes
        for f in (getattr(self, "tfwd", None), getattr(self, "dfwd", None)):
            if f is not None:
                h2d += f.h2d_bytes
        return h2d, self.d2h_bytes

    # ------------------------------------------------------------------
    def execute(self, state: EngineState, plan: StepPlan, rows: list[VerifyRow]) -> StepResult:
        dev = self.device
        ts, ds = self.s_target, self.s_draft
        # the step's timing events, created once (every step ends synchronised)
        if self._step_events is None:
            self._step_events = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        e_start, e_pf_t, e_pf_d, e_sd, e_ov, e_v0, e_v1 = self._step_events
        t_host = time.perf_counter()
        cur = torch.cuda.current_stream(dev)
        cur.synchronize()
        with torch.cuda.stream(ts):
            e_start.record(ts)
            if plan.prefill_ids:
                self._admit(state, plan.prefill_ids)
            self._upload_block_table(state)
        ds.wait_stream(ts)
        # prefill: target model on the target stream, draft model on the draft stream
        with torch.cuda.stream(ts):
            if plan.prefill_ids:
                self._prefill(state, plan.prefill_ids, self.tfwd, "target")
            e_pf_t.record(ts)
        with torch.cuda.stream(ds):
            if plan.prefill_ids:
                self._prefill(state, plan.prefill_ids, self.dfwd, "draft")
            e_pf_d.record(ds)
            # serial drafts (startup target batch / fallback / SD batch)
            self._draft_loop(state, plan.serial_draft_ids, plan.quotas)
            e_sd.record(ds)
        ts.wait_event(e_sd)
        # the verify is enqueued first: with the draft loop shortened it is the
        # longer of the two overlapped passes, so it gets the earlier start
        # (PSD_DRAFT_FIRST=1: the previous order)
        def verify():
            with torch.cuda.stream(ts):
                e_v0.record(ts)
                if rows:
                    # capped GEMM grids only while drafts run beside the verify
                    self._verify(state, rows, beside_draft=any(
                        plan.quotas.get(rid, 0) > 0 for rid in plan.overlap_draft_ids))
                e_v1.record(ts)
        if not self.draft_first:
            verify()
        with torch.cuda.stream(ds):
            # overlapped drafts of the skip batch
            self._draft_loop(state, plan.overlap_draft_ids, plan.quotas)
            e_ov.record(ds)
        if self.draft_first:
            verify()
        e_v1.synchronize()
        e_ov.synchronize()
        accepted = {}
        if rows:
            a = self.acc_host.numpy()[:len(rows)]
            for r, row in enumerate(rows):
                if row.k > 0:
                    accepted[row.request_id] = int(a[r])
        for row in rows:
            self.pending_k.pop(row.request_id, None)
        prefill_ms = max(e_start.elapsed_time(e_pf_t), e_start.elapsed_time(e_pf_d))
        serial_ms = e_pf_d.elapsed_time(e_sd)
        overlap_ms = e_sd.elapsed_time(e_ov)
        verify_ms = e_v0.elapsed_time(e_v1)
        step_ms = max(e_start.elapsed_time(e_v1), e_start.elapsed_time(e_ov))
        self.stats["steps"] += 1
        self.stats["draft_ms"] += serial_ms + overlap_ms
        self.stats["verify_ms"] += verify_ms
        self.stats["prefill_ms"] += prefill_ms
        self.stats["host_s"] = self.stats.get("host_s", 0.0) + (time.perf_counter() - t_host)
        measured = StepResult(prefill_ms, serial_ms, overlap_ms, verify_ms, step_ms, accepted)
        if self.replay:
            # the scheduler advances on the reference's virtual durations (so
            # arrivals and preemptions fire at the same steps as in specsim);
            # the device really committed the replayed counts
            virt = self._sim.execute(state, plan, rows)
            if virt.accepted != accepted:
                raise ProtocolError(f"replay: device accepted {accepted} != reference "
                                    f"{virt.accepted}")
            self.measured_log.append(measured)
            return virt
        return measured
