"""Llama / Qwen2-shaped decoder-only transformers on the C ABI (target verify
forward and draft decode forward).

The reference simulates these passes as virtual durations
(``LatencyModel.duration``, pkg/src/specsim/request_model.py:92-117, charged
at engine.py:338, 359-360, 378, 402, 429).  Here they are real: embedding ->
L x [RMSNorm -> QKV GEMM -> RoPE + paged-KV write -> paged attention ->
O GEMM (+residual) -> RMSNorm -> gate/up GEMM (+SiLU*up) -> down GEMM
(+residual)] -> final RMSNorm on the logit rows -> LM-head GEMM (fp32 logits)
-> synthetic-language bias.  Every step is one of our sm_100a kernels
(include/psd.h); torch only allocates memory.

Weights are random-init (no checkpoints offline): every matrix is
``(u - 1/2) * span`` with u from splitmix64(seed_t, i) (uniform, std 0.02),
norms are 1.  ``oracle/model.py`` regenerates the identical bf16 weights in
numpy for the CPU reference forward.

Synthetic language: random-init models agree on the next token with
probability ~1/V, which would make speculative decoding degenerate.  Both
models therefore add ``beta * onehot(successor[prev_token])`` to their logits
(SURVEY.md §7 hard part 4, option (a)); ``beta_target`` sets how often the
target's argmax follows the shared successor table, i.e. the acceptance rate.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import native
from .errors import ConfigError

__all__ = ["ModelShape", "PRESETS", "Transformer", "Forward", "pack_gate_up", "successor_table",
           "tensor_seed", "rope_inv_freq"]

INIT_STD = 0.02
INIT_SPAN = INIT_STD * math.sqrt(12.0)  # uniform(-span/2, span/2) has std 0.02


@dataclass(frozen=True)
class ModelShape:
    name: str
    vocab: int
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    rope_theta: float
    rope_scaling: tuple | None = None  # llama3: (factor, low, high, original_max)
    tie_embeddings: bool = False
    qkv_bias: bool = False
    rms_eps: float = 1e-5

    @property
    def ffn_padded(self) -> int:
        """FFN width padded to 64 (gate/up are packed per 64-row half tiles);
        padded features have zero weights and contribute exactly 0."""
        return (self.ffn + 63) // 64 * 64

    @property
    def qkv_out(self) -> int:
        return (self.heads + 2 * self.kv_heads) * self.head_dim

    def param_count(self) -> int:
        h = self.hidden
        per = h * self.qkv_out + self.heads * self.head_dim * h + 3 * h * self.ffn + 2 * h
        emb = self.vocab * h * (1 if self.tie_embeddings else 2)
        return self.layers * per + emb + h


_L31 = (8.0, 1.0, 4.0, 8192)
_L32 = (32.0, 1.0, 4.0, 8192)
PRESETS: dict[str, ModelShape] = {
    "llama-3.1-8b": ModelShape("llama-3.1-8b", 128256, 4096, 32, 32, 8, 128, 14336, 500000.0,
                               _L31),
    "llama-3.2-1b": ModelShape("llama-3.2-1b", 128256, 2048, 16, 32, 8, 64, 8192, 500000.0,
                               _L32, tie_embeddings=True),
    "llama-3.1-70b": ModelShape("llama-3.1-70b", 128256, 8192, 80, 64, 8, 128, 28672, 500000.0,
                                _L31),
    "qwen2.5-7b": ModelShape("qwen2.5-7b", 152064, 3584, 28, 28, 4, 128, 18944, 1000000.0,
                             None, qkv_bias=True, rms_eps=1e-6),
    "qwen2.5-0.5b": ModelShape("qwen2.5-0.5b", 151936, 896, 24, 14, 2, 64, 4864, 1000000.0,
                               None, tie_embeddings=True, qkv_bias=True, rms_eps=1e-6),
    # BASELINE config 1: tiny random-init pair
    "tiny-target": ModelShape("tiny-target", 1024, 256, 4, 8, 2, 32, 688, 10000.0),
    # tiny Qwen2-style model (qkv bias, tied embeddings): the bias paths in tests
    "tiny-qwen": ModelShape("tiny-qwen", 1024, 128, 2, 4, 2, 32, 344, 1000000.0, None,
                            tie_embeddings=True, qkv_bias=True, rms_eps=1e-6),
    # tiny target whose QKV shards stay 128-row aligned at TP = 2 (tests)
    "tiny-target-tp": ModelShape("tiny-target-tp", 1024, 256, 4, 8, 4, 32, 688, 10000.0),
    "tiny-draft": ModelShape("tiny-draft", 1024, 128, 2, 4, 2, 32, 344, 10000.0),
}


def rope_inv_freq(shape: ModelShape) -> np.ndarray:
    """Rotary inverse frequencies (Llama-3 scaled where configured), float32."""
    d = shape.head_dim
    inv = 1.0 / (shape.rope_theta ** (np.arange(0, d, 2, dtype=np.float64) / d))
    if shape.rope_scaling is not None:
        factor, low, high, orig = shape.rope_scaling
        wavelen = 2.0 * math.pi / inv
        low_wl, high_wl = orig / low, orig / high
        scaled = np.where(wavelen > low_wl, inv / factor, inv)
        smooth = (orig / wavelen - low) / (high - low)
        smoothed = (1.0 - smooth) * scaled / factor + smooth * scaled
        medium = (wavelen >= high_wl) & (wavelen <= low_wl)
        inv = np.where(medium, smoothed, scaled)
    return inv.astype(np.float32)


def pack_gate_up(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    """[F, H] gate and up -> [2F, H] in the PSD_EPI_SILU order: per 128-row
    tile and per 32-row quarter q, 16 gate rows then the 16 matching up rows
    (so one warp shuffle pairs them in the GEMM epilogue)."""
    F, H = gate.shape
    g = gate.view(F // 64, 4, 16, H)
    u = up.view(F // 64, 4, 16, H)
    return torch.stack([g, u], dim=2).reshape(2 * F, H).contiguous()


def tensor_seed(model_seed: int, layer: int, which: int) -> int:
    """Per-tensor init seed (also used by oracle/model.py)."""
    return (model_seed * 1_000_003 + (layer + 1) * 101 + which) & 0x7FFFFFFF


def successor_table(vocab: int, draft_vocab: int, seed: int) -> np.ndarray:
    """The synthetic language: next token = successor[prev] (a permutation of
    the shared vocabulary; ids past it wrap)."""
    v = min(vocab, draft_vocab)
    perm = np.random.Generator(np.random.Philox(key=[seed, 0x5EC])).permutation(v)
    succ = np.empty(vocab, dtype=np.int32)
    succ[:v] = perm
    succ[v:] = perm[np.arange(v, vocab) % v]
    return succ


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _chk(rc: int, what: str) -> None:
    if rc != 0:
        native.check(rc, what)


class Transformer:
    """Device weights + paged KV cache of one model."""

    # which-ids for tensor_seed
    W_QKV, W_O, W_GATE, W_UP, W_DOWN, W_EMB, W_LM, B_QKV = range(8)

    def __init__(self, shape: ModelShape, device: torch.device, seed: int, num_blocks: int,
                 block_size: int = 16, max_blocks_per_seq: int = 64, tp=None) -> None:
        self.tp = tp  # (rank, size, process group) or None
        self.full_vocab = shape.vocab
        if tp is not None and tp[1] > 1:
            self._init_tp_shard(shape, device, seed, num_blocks, block_size, max_blocks_per_seq)
            return
        if shape.qkv_out % 128 or shape.hidden % 128 or shape.vocab % 128:
            raise ConfigError(f"{shape.name}: GEMM output dims must be multiples of 128")
        self.shape = shape
        self.device = device
        self.seed = seed
        self.block_size = block_size
        self.num_blocks = num_blocks
        self.max_blocks = max_blocks_per_seq
        lib = native.load()
        self._lib = lib
        s = shape
        H, F, Fp = s.hidden, s.ffn, s.ffn_padded
        bf = torch.bfloat16
        dev = device

        def fill(t: torch.Tensor, tseed: int) -> torch.Tensor:
            _chk(lib.psd_fill_uniform_bf16(t.data_ptr(), t.numel(), tseed, INIT_SPAN,
                                           _stream_ptr(dev)), "psd_fill_uniform_bf16")
            return t

        self.layers = []
        for li in range(s.layers):
            wqkv = fill(torch.empty(s.qkv_out, H, dtype=bf, device=dev),
                        tensor_seed(seed, li, self.W_QKV))
            wo = fill(torch.empty(H, s.heads * s.head_dim, dtype=bf, device=dev),
                      tensor_seed(seed, li, self.W_O))
            gate = torch.zeros(Fp, H, dtype=bf, device=dev)
            up = torch.zeros(Fp, H, dtype=bf, device=dev)
            fill(gate[:F], tensor_seed(seed, li, self.W_GATE))
            fill(up[:F], tensor_seed(seed, li, self.W_UP))
            wgu = pack_gate_up(gate, up)
            del gate, up
            down = torch.zeros(H, Fp, dtype=bf, device=dev)
            dtmp = fill(torch.empty(H, F, dtype=bf, device=dev), tensor_seed(seed, li, self.W_DOWN))
            down[:, :F] = dtmp
            del dtmp
            bias = None
            if s.qkv_bias:
                bias = fill(torch.empty(s.qkv_out, dtype=bf, device=dev),
                            tensor_seed(seed, li, self.B_QKV))
            self.layers.append({
                "attn_norm": torch.ones(H, dtype=bf, device=dev),
                "wqkv": wqkv, "wo": wo,
                "mlp_norm": torch.ones(H, dtype=bf, device=dev),
                "wgu": wgu, "wdown": down, "bqkv": bias,
            })
        self.embed = fill(torch.empty(s.vocab, H, dtype=bf, device=dev),
                          tensor_seed(seed, -1, self.W_EMB))
        self.lm_head = self.embed if s.tie_embeddings else fill(
            torch.empty(s.vocab, H, dtype=bf, device=dev), tensor_seed(seed, -1, self.W_LM))
        self.final_norm = torch.ones(H, dtype=bf, device=dev)
        self.inv_freq = torch.from_numpy(rope_inv_freq(s)).to(dev)
        # paged KV cache: [layers, 2, blocks * block_size, Hkv, D]
        self.kv = torch.zeros(s.layers, 2, num_blocks * block_size, s.kv_heads, s.head_dim,
                              dtype=bf, device=dev)
        self.block_table = torch.zeros(0, dtype=torch.int32, device=dev)

    def _init_tp_shard(self, full: ModelShape, device, seed, num_blocks, block_size,
                       max_blocks) -> None:
        """Megatron-style tensor-parallel shard of the target:
        column-parallel QKV (this rank's query / kv heads) and gate/up (an FFN
        slice), row-parallel O and down (their input columns; outputs are
        partial sums, all-reduced in Forward.run), vocab-parallel LM head (a
        vocab slice, all-gathered into full logit rows).  Every shard is the
        exact block of the full random-init tensor (psd_fill_uniform_bf16_block),
        so a TP forward computes the same function as the unsharded model."""
        r, T, _ = self.tp
        s = full
        if s.heads % T or s.kv_heads % T or s.vocab % T:
            raise ConfigError(f"{s.name}: heads / kv heads / vocab must divide by TP={T}")
        D, H = s.head_dim, s.hidden
        hq, hkv = s.heads // T, s.kv_heads // T
        f_tp = -(-s.ffn // (64 * T)) * 64 * T
        fl = f_tp // T
        vs = s.vocab // T
        vs_pad = -(-vs // 128) * 128
        local = ModelShape(f"{s.name}-tp{r}of{T}", vs_pad, H, s.layers, hq, hkv, D, fl,
                           s.rope_theta, s.rope_scaling, False, s.qkv_bias, s.rms_eps)
        if local.qkv_out % 128 or H % 128:
            raise ConfigError(f"{s.name}: TP={T} shard QKV rows {local.qkv_out} not 128-aligned")
        self.shape = local
        self.vocab_shard = vs
        self.device = device
        self.seed = seed
        self.block_size = block_size
        self.num_blocks = num_blocks
        self.max_blocks = max_blocks
        lib = native.load()
        self._lib = lib
        bf = torch.bfloat16
        dev = device
        st = _stream_ptr(dev)

        def block(dst, rows, cols, full_cols, row0, col0, tseed):
            _chk(lib.psd_fill_uniform_bf16_block(dst.data_ptr(), dst.stride(0), rows, cols,
                                                 full_cols, row0, col0, tseed, INIT_SPAN, st),
                 "psd_fill_uniform_bf16_block")

        q0, k0, v0 = r * hq * D, s.heads * D + r * hkv * D, (s.heads + s.kv_heads) * D + r * hkv * D
        self.layers = []
        for li in range(s.layers):
            tq = tensor_seed(seed, li, self.W_QKV)
            wqkv = torch.empty(local.qkv_out, H, dtype=bf, device=dev)
            block(wqkv[:hq * D], hq * D, H, H, q0, 0, tq)
            block(wqkv[hq * D:(hq + hkv) * D], hkv * D, H, H, k0, 0, tq)
            block(wqkv[(hq + hkv) * D:], hkv * D, H, H, v0, 0, tq)
            wo = torch.empty(H, hq * D, dtype=bf, device=dev)
            block(wo, H, hq * D, s.heads * D, 0, r * hq * D, tensor_seed(seed, li, self.W_O))
            gate = torch.zeros(fl, H, dtype=bf, device=dev)
            up = torch.zeros(fl, H, dtype=bf, device=dev)
            real = max(0, min(s.ffn, (r + 1) * fl) - r * fl)
            if real:
                block(gate, real, H, H, r * fl, 0, tensor_seed(seed, li, self.W_GATE))
                block(up, real, H, H, r * fl, 0, tensor_seed(seed, li, self.W_UP))
            wgu = pack_gate_up(gate, up)
            del gate, up
            down = torch.zeros(H, fl, dtype=bf, device=dev)
            if real:
                block(down, H, real, s.ffn, 0, r * fl, tensor_seed(seed, li, self.W_DOWN))
            bias = None
            if s.qkv_bias:
                tb = tensor_seed(seed, li, self.B_QKV)
                bias = torch.empty(local.qkv_out, 1, dtype=bf, device=dev)
                block(bias[:hq * D], hq * D, 1, 1, q0, 0, tb)
                block(bias[hq * D:(hq + hkv) * D], hkv * D, 1, 1, k0, 0, tb)
                block(bias[(hq + hkv) * D:], hkv * D, 1, 1, v0, 0, tb)
                bias = bias.view(-1)
            self.layers.append({
                "attn_norm": torch.ones(H, dtype=bf, device=dev),
                "wqkv": wqkv, "wo": wo,
                "mlp_norm": torch.ones(H, dtype=bf, device=dev),
                "wgu": wgu, "wdown": down, "bqkv": bias,
            })
        # embedding replicated (every token id is looked up on every rank)
        self.embed = torch.empty(s.vocab, H, dtype=bf, device=dev)
        block(self.embed, s.vocab, H, H, 0, 0, tensor_seed(seed, -1, self.W_EMB))
        self.lm_head = torch.zeros(vs_pad, H, dtype=bf, device=dev)
        lm_seed = tensor_seed(seed, -1, self.W_EMB if s.tie_embeddings else self.W_LM)
        block(self.lm_head, vs, H, H, r * vs, 0, lm_seed)
        self.final_norm = torch.ones(H, dtype=bf, device=dev)
        self.inv_freq = torch.from_numpy(rope_inv_freq(s)).to(dev)
        self.kv = torch.zeros(s.layers, 2, num_blocks * block_size, hkv, D, dtype=bf, device=dev)
        self.block_table = torch.zeros(0, dtype=torch.int32, device=dev)

    def kv_bytes_per_block(self) -> int:
        s = self.shape
        return s.layers * 2 * self.block_size * s.kv_heads * s.head_dim * 2


META_FIELDS = ("tokens", "positions", "slots", "seq_slot", "q_start", "q_len", "q_pos0",
               "kv_len", "logit_rows", "gather_src", "scatter_dst")


class Forward:
    """One model's forward over a batch described by device metadata.

    Per token: tokens, positions, slots (KV write slot, -1 = none).  Per
    sequence: seq_slot (block-table row), q_start, q_len, q_pos0, kv_len.
    logit_rows: hidden-state rows that get logits.  gather_src / scatter_dst:
    device token routing for the draft loop (see GpuBackend).  ``sets``
    independent metadata sets live in one packed int32 buffer, uploaded with a
    single copy, so a k-step draft loop needs one host->device transfer.
    """

    def __init__(self, model: Transformer, max_tokens: int, max_seqs: int,
                 max_logit_rows: int, block_table: torch.Tensor, sets: int = 1,
                 workspace_bytes: int = 64 << 20, max_kv_len: int = 0) -> None:
        s = model.shape
        dev = model.device
        self.model = model
        self.block_table = block_table  # [slots, max_blocks] int32, shared with the backend
        self.max_tokens, self.max_seqs, self.max_logit_rows = max_tokens, max_seqs, max_logit_rows
        bf = torch.bfloat16
        T = max_tokens
        self.x = torch.empty(T, s.hidden, dtype=bf, device=dev)
        self.xn = torch.empty(T, s.hidden, dtype=bf, device=dev)
        self.qkv = torch.empty(T, s.qkv_out, dtype=bf, device=dev)
        self.q = torch.empty(T, s.heads * s.head_dim, dtype=bf, device=dev)
        self.attn = torch.empty(T, s.heads * s.head_dim, dtype=bf, device=dev)
        self.act = torch.empty(T, s.ffn_padded, dtype=bf, device=dev)
        self.xf = torch.empty(max_logit_rows, s.hidden, dtype=bf, device=dev)
        self.prev = torch.empty(max_logit_rows, dtype=torch.int32, device=dev)
        # K6 argmax partials for up to 512 logit rows (the draft's LM head, and
        # the target's when its greedy verification folds argmax tokens);
        # allocated here: never inside a graph capture
        self.amax_rows = min(max_logit_rows, 512) if s.vocab % 128 == 0 else 0
        self.amax = (torch.empty(native.load().psd_argmax_partials_bytes(self.amax_rows,
                                                                         s.vocab),
                                 dtype=torch.uint8, device=dev) if self.amax_rows else None)
        self.comm = None
        if model.tp is not None and model.tp[1] > 1:
            import os
            if os.environ.get("PSD_TP_COMM", "peer") == "peer":
                # C2 over NVLink peer memory: the split-K reduction of the
                # row-parallel O / down GEMMs fused with the cross-rank sum
                # (csrc/comm.cu); PSD_TP_COMM=dist keeps torch.distributed
                from .comm import PeerComm
                self.comm = PeerComm(model.tp[2], buf_bytes=T * s.hidden * 4, device=dev)
            self.lshard = torch.empty(max_logit_rows * s.vocab, dtype=torch.float32, device=dev)
            self.lgather = torch.empty(model.tp[1] * max_logit_rows * s.vocab,
                                       dtype=torch.float32, device=dev)
        # stream-K GEMM workspace (partials + tickets): zeroed once, left zeroed
        import ctypes
        lib = native.load()
        need = 0
        for mm in sorted({T, max_logit_rows, min(T, 64), min(T, 320), 32, 2 * max_seqs}):
            for (n_out, k_in) in ((s.qkv_out, s.hidden), (s.hidden, s.heads * s.head_dim),
                                  (2 * s.ffn_padded, s.hidden), (s.hidden, s.ffn_padded),
                                  (s.vocab, s.hidden)):
                wb = ctypes.c_size_t()
                lib.psd_gemm_plan(mm, n_out, k_in, native.EPI_BF16, 0, None, ctypes.byref(wb))
                need = max(need, wb.value)
        self.ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
        # split-KV attention workspace (tickets + partial softmax states), zeroed
        self.max_kv_len = max_kv_len
        aw = lib.psd_attention_workspace_bytes(max_seqs, s.kv_heads, 16, s.heads, s.head_dim,
                                               max_kv_len) if max_kv_len else 0
        self.att_ws = torch.zeros(max(aw, 16384), dtype=torch.uint8, device=dev)
        # fp32 split-K partials of the QKV / O / down GEMMs (one buffer, reused
        # in sequence: each is consumed before the next GEMM overwrites it)
        self._nsplit = ctypes.byref(ctypes.c_int(1))
        pneed = 0
        for mm in sorted({T, max_logit_rows, min(T, 64), min(T, 320), 32, 2 * max_seqs}):
            for (n_out, k_in) in ((s.qkv_out, s.hidden), (s.hidden, s.heads * s.head_dim),
                                  (s.hidden, s.ffn_padded)):
                sp = ctypes.c_int()
                lib.psd_gemm_plan(mm, n_out, k_in, native.EPI_PARTIAL, 0, ctypes.byref(sp), None)
                pneed = max(pneed, sp.value * mm * n_out)
        self.part = torch.empty(pneed, dtype=torch.float32, device=dev)
        sizes = {"tokens": T, "positions": T, "slots": T, "seq_slot": max_seqs,
                 "q_start": max_seqs, "q_len": max_seqs, "q_pos0": max_seqs, "kv_len": max_seqs,
                 "logit_rows": max_logit_rows, "gather_src": T, "scatter_dst": max_logit_rows}
        self._offsets = {}
        o = 0
        for name in META_FIELDS:
            self._offsets[name] = (o, sizes[name])
            o += sizes[name]
        self.set_size = o
        self.sets = sets
        import os
        self.fuse_rope = os.environ.get("PSD_FUSED_ROPE", "1") == "1"
        # split count of the QKV / O / down split-K GEMMs (0 = the shape's
        # default); tests use it to measure the forward's reordering noise floor
        self.splits_hint = int(os.environ.get("PSD_SPLITS_HINT", "0"))
        # widest per-sequence query count that takes the fused path
        self.fuse_rope_max_q = int(os.environ.get("PSD_FUSED_ROPE_MAXQ", "2"))
        self.meta = torch.zeros(sets, o, dtype=torch.int32, device=dev)
        self.h2d_bytes = 0  # metadata bytes uploaded (GpuBackend.transfer_bytes)
        # ring of pinned staging buffers: an async H2D copy reads its buffer
        # when it executes, so a buffer is rewritten only after its copy ran
        self.ring = 4
        self.meta_host = torch.zeros(self.ring, sets, o, dtype=torch.int32).pin_memory()
        self._host_np = self.meta_host.numpy()
        self._events = [None] * self.ring
        self._event_pool = [torch.cuda.Event() for _ in range(self.ring)]
        self._cur = 0
        # (offset, capacity) per META_FIELDS entry, for the native stagers
        self.fields_np = np.array([v for name in META_FIELDS for v in self._offsets[name]],
                                  np.int32)
        self.fields_ptr = self.fields_np.ctypes.data

    # ---- tensor parallelism (target TP) ---------------------
    def _tp_reduce(self, S: int, n: int) -> int:
        """Sum the ranks' row-parallel partial outputs (S fp32 split-K slices of
        n = M * H floats); returns the slice count the consumer reduces.

        Peer memory (default): one kernel sums the local splits and the ranks'
        sums in fixed (rank, split) order into slice 0 -- n floats cross
        NVLink per rank instead of S * n, and every rank holds identical bits
        (consumer: 1 slice).  torch.distributed fallback: all-reduce of all S
        slices (linear, so the consumer's split reduction is unchanged)."""
        if self.comm is not None:
            self.comm.allreduce_partials(self.part, S, n, n, self.part)
            return 1
        import torch.distributed as dist
        dist.all_reduce(self.part[:S * n], group=self.model.tp[2])
        return S

    def _gather_logits(self, logits: torch.Tensor, ld: int, R: int) -> None:
        import torch.distributed as dist
        m = self.model
        T = m.tp[1]
        vp, vs = m.shape.vocab, m.vocab_shard
        parts = list(self.lgather[:T * R * vp].view(T, R * vp).unbind(0))
        dist.all_gather(parts, self.lshard[:R * vp], group=m.tp[2])
        full = logits.view(-1)[:R * ld].view(R, ld)[:, :T * vs].view(R, T, vs)
        full.copy_(self.lgather[:T * R * vp].view(T, R, vp)[:, :, :vs].permute(1, 0, 2))

    def view(self, name: str, set_index: int = 0) -> torch.Tensor:
        o, n = self._offsets[name]
        return self.meta[set_index, o:o + n]

    def begin(self) -> None:
        """Start staging a new upload (advances the staging ring)."""
        self._cur = (self._cur + 1) % self.ring
        ev = self._events[self._cur]
        if ev is not None:
            ev.synchronize()

    def host_set_ptr(self, set_index: int = 0) -> int:
        """Address of a metadata set in the current pinned staging buffer."""
        return self.meta_host.data_ptr() + 4 * (self._cur * self.sets + set_index) * self.set_size

    def stage(self, set_index: int, arrays: dict[str, np.ndarray]) -> None:
        """Write host metadata (int32) for one set into pinned staging."""
        host = self._host_np[self._cur, set_index]
        for name, arr in arrays.items():
            o, n = self._offsets[name]
            if len(arr) > n:
                raise ConfigError(f"forward metadata {name}: {len(arr)} > capacity {n}")
            host[o:o + len(arr)] = arr

    def stage_many(self, first_set: int, arrays: dict[str, np.ndarray]) -> None:
        """Write metadata of sets first_set .. first_set + n - 1 at once:
        each array is [n, len] (one row per set)."""
        host = self._host_np[self._cur]
        for name, arr in arrays.items():
            o, n = self._offsets[name]
            if arr.shape[1] > n:
                raise ConfigError(f"forward metadata {name}: {arr.shape[1]} > capacity {n}")
            host[first_set:first_set + arr.shape[0], o:o + arr.shape[1]] = arr

    def upload(self, n_sets: int = 1) -> None:
        """Copy staged sets 0..n_sets-1 to the device on the current stream."""
        nbytes = n_sets * self.set_size * 4
        _chk(self.model._lib.psd_copy_async(self.meta.data_ptr(), self.host_set_ptr(0), nbytes,
                                            _stream_ptr(self.model.device)), "metadata upload")
        self.h2d_bytes += nbytes
        ev = self._event_pool[self._cur]
        ev.record()
        self._events[self._cur] = ev

    def run(self, n_tokens: int, n_seqs: int, max_q_len: int, n_logit_rows: int,
            logits: torch.Tensor | None, logits_ld: int = 0, bigram=None,
            set_index: int = 0, shard_out: bool = False, argmax_into=None) -> None:
        """Enqueue the forward on the current stream.  ``tokens`` may be
        filled on device beforehand (draft loop); ``logits`` (fp32, row pitch
        ``logits_ld``) receives the LM-head output of ``logit_rows``.
        shard_out (tensor-parallel target): keep this rank's vocabulary shard
        in ``lshard`` ([rows, vocab shard padded], bigram bias applied to the
        shard's columns) instead of all-gathering full rows -- the greedy
        verifier reduces shards to partials.
        argmax_into (greedy draft step, K6): (out_tokens, dst, dst_idx) -- the
        LM head's epilogue reduces the (biased) logits to per-tile argmax
        partials and one fold writes each row's token to out_tokens[m] and
        dst[dst_idx[m]]; no logits are stored."""
        m = self.model
        s = m.shape
        lib = m._lib
        dev = m.device
        st = _stream_ptr(dev)
        M = n_tokens
        v = {name: self.view(name, set_index) for name in META_FIELDS}
        H = s.hidden
        _chk(lib.psd_embed(v["tokens"].data_ptr(), M, m.embed.data_ptr(), H, self.x.data_ptr(),
                           st), "psd_embed")
        scale = 1.0 / math.sqrt(s.head_dim)
        ws, wsn = self.ws.data_ptr(), self.ws.numel()
        part, partn = self.part.data_ptr(), self.part.numel() * 4
        nsp = self._nsplit
        Dq = s.heads * s.head_dim
        Fp = s.ffn_padded
        X = self.x.data_ptr()
        # QKV / O / down: grid split-K GEMMs (few weight tiles) whose fp32
        # partials are reduced inside the consumer kernel (RoPE, add+RMSNorm);
        # gate/up and the LM head: stream-K persistent GEMMs
        tp = m.tp if (m.tp is not None and m.tp[1] > 1) else None
        prev_S = 0  # splits of the pending down-proj partials (0 = none)
        # draft decode (<= 2 query tokens per sequence): RoPE fused into the
        # attention kernel (-3 % per draft step); at verify widths (k + 1 tokens)
        # the separate RoPE kernel's parallelism wins (+3 % when fused)
        fuse_rope = self.fuse_rope and max_q_len <= self.fuse_rope_max_q
        for li, L in enumerate(m.layers):
            kc = m.kv[li, 0]
            vc = m.kv[li, 1]
            _chk(lib.psd_add_rmsnorm(X, H, part if prev_S else None, prev_S, M * H, H, None,
                                     L["attn_norm"].data_ptr(), self.xn.data_ptr(), H, M, H,
                                     s.rms_eps, 1, st), "add+attn norm")
            _chk(lib.psd_gemm_partials(self.xn.data_ptr(), H, M, H, L["wqkv"].data_ptr(), H,
                                       s.qkv_out, part, partn, self.splits_hint, nsp, st),
                 "gemm qkv")
            if fuse_rope:
                # decode / verify: RoPE + KV write inside the attention kernel
                _chk(lib.psd_attention_rope(
                    part, nsp._obj.value, M * s.qkv_out, v["positions"].data_ptr(),
                    v["slots"].data_ptr(), m.inv_freq.data_ptr(),
                    L["bqkv"].data_ptr() if L["bqkv"] is not None else None, kc.data_ptr(),
                    vc.data_ptr(), self.block_table.data_ptr(), self.block_table.shape[1],
                    v["seq_slot"].data_ptr(), v["q_start"].data_ptr(), v["q_len"].data_ptr(),
                    v["q_pos0"].data_ptr(), v["kv_len"].data_ptr(), n_seqs, max_q_len, s.heads,
                    s.kv_heads, s.head_dim, m.block_size, scale, self.attn.data_ptr(), st),
                    "attention+rope")
            else:
                _chk(lib.psd_rope_kv_partials(part, nsp._obj.value, M * s.qkv_out, M, s.heads,
                                              s.kv_heads, s.head_dim, v["positions"].data_ptr(),
                                              v["slots"].data_ptr(), m.inv_freq.data_ptr(),
                                              L["bqkv"].data_ptr() if L["bqkv"] is not None else None,
                                              self.q.data_ptr(), kc.data_ptr(), vc.data_ptr(), st),
                     "rope_kv")
                _chk(lib.psd_attention(self.q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                                       self.block_table.data_ptr(), self.block_table.shape[1],
                                       v["seq_slot"].data_ptr(), v["q_start"].data_ptr(),
                                       v["q_len"].data_ptr(), v["q_pos0"].data_ptr(),
                                       v["kv_len"].data_ptr(), n_seqs, max_q_len, s.heads,
                                       s.kv_heads, s.head_dim, m.block_size, scale,
                                       self.attn.data_ptr(), self.max_kv_len if M <= 4 * n_seqs * 4
                                       else 0, self.att_ws.data_ptr(), self.att_ws.numel(), st),
                     "attention")
            _chk(lib.psd_gemm_partials(self.attn.data_ptr(), Dq, M, Dq, L["wo"].data_ptr(), Dq, H,
                                       part, partn, self.splits_hint, nsp, st), "gemm o")
            S_o = nsp._obj.value
            if tp:  # row-parallel O: sum the ranks' partial outputs
                S_o = self._tp_reduce(S_o, M * H)
            _chk(lib.psd_add_rmsnorm(X, H, part, S_o, M * H, H, None,
                                     L["mlp_norm"].data_ptr(), self.xn.data_ptr(), H, M, H,
                                     s.rms_eps, 1, st), "add+mlp norm")
            _chk(lib.psd_gemm_bf16(self.xn.data_ptr(), H, M, H, L["wgu"].data_ptr(), H, 2 * Fp,
                                   self.act.data_ptr(), Fp, native.EPI_SILU, None, 0, 0, ws, wsn,
                                   st), "gemm gate/up")
            _chk(lib.psd_gemm_partials(self.act.data_ptr(), Fp, M, Fp, L["wdown"].data_ptr(), Fp,
                                       H, part, partn, self.splits_hint, nsp, st), "gemm down")
            prev_S = nsp._obj.value
            if tp:  # row-parallel down
                prev_S = self._tp_reduce(prev_S, M * H)
        if n_logit_rows == 0 or (logits is None and argmax_into is None):
            return  # prefill: only the KV cache is needed
        R = n_logit_rows
        _chk(lib.psd_add_rmsnorm(X, H, part, prev_S, M * H, H, v["logit_rows"].data_ptr(),
                                 m.final_norm.data_ptr(), self.xf.data_ptr(), H, R, H, s.rms_eps,
                                 0, st), "final norm")
        V = m.full_vocab
        ld = logits_ld or V
        if argmax_into is not None and not tp:
            out_tok, dst, dst_idx = argmax_into
            if self.amax is None or R > self.amax_rows:
                raise ValueError("argmax LM head needs vocab % 128 == 0 and <= 512 logit rows")
            succ, beta = bigram if bigram is not None else (None, 0.0)
            _chk(lib.psd_gemm_argmax(self.xf.data_ptr(), H, R, H, m.lm_head.data_ptr(), H, s.vocab,
                                     v["tokens"].data_ptr(), v["logit_rows"].data_ptr(),
                                     succ.data_ptr() if succ is not None else None, float(beta),
                                     self.amax.data_ptr(), ws, wsn, st), "gemm lm_head argmax")
            _chk(lib.psd_argmax_fold(self.amax.data_ptr(), R, s.vocab,
                                     out_tok.data_ptr() if out_tok is not None else None,
                                     dst.data_ptr() if dst is not None else None,
                                     dst_idx.data_ptr() if dst_idx is not None else None, st),
                 "argmax fold")
            return
        if tp:
            # vocab-parallel LM head: this rank's slice (all-gathered into full
            # rows unless the caller consumes the shard)
            _chk(lib.psd_gemm_bf16(self.xf.data_ptr(), H, R, H, m.lm_head.data_ptr(), H, s.vocab,
                                   self.lshard.data_ptr(), s.vocab, native.EPI_F32, None, 0, 0,
                                   ws, wsn, st), "gemm lm_head shard")
            if shard_out:
                if bigram is not None and bigram[1] != 0.0:
                    v0 = tp[0] * m.vocab_shard
                    _chk(lib.psd_index_copy_i32(self.prev.data_ptr(), None,
                                                v["tokens"].data_ptr(),
                                                v["logit_rows"].data_ptr(), R, st), "prev tokens")
                    _chk(lib.psd_bigram_bias_range(self.lshard.data_ptr(), s.vocab,
                                                   self.prev.data_ptr(), R, bigram[0].data_ptr(),
                                                   V, float(bigram[1]), v0, v0 + m.vocab_shard,
                                                   st), "bigram shard")
                return
            self._gather_logits(logits, ld, R)
        else:
            _chk(lib.psd_gemm_bf16(self.xf.data_ptr(), H, R, H, m.lm_head.data_ptr(), H, s.vocab,
                                   logits.data_ptr(), ld, native.EPI_F32, None, 0, 0, ws, wsn, st),
                 "gemm lm_head")
        if bigram is not None:
            succ, beta = bigram
            if beta != 0.0:
                # the token that produced each logit row is its predecessor
                _chk(lib.psd_index_copy_i32(self.prev.data_ptr(), None, v["tokens"].data_ptr(),
                                            v["logit_rows"].data_ptr(), R, st), "prev tokens")
                _chk(lib.psd_bigram_bias(logits.data_ptr(), ld, self.prev.data_ptr(), R,
                                         succ.data_ptr(), V, float(beta), st), "bigram")
