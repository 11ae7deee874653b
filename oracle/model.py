"""numpy restatement of the draft / target forward (TEST INFRASTRUCTURE ONLY).

Same random-init weights as the device (bit-identical bf16 values regenerated
by liboracle_model.so), fp32 math, and bf16 rounding at exactly the points
where the GPU stores bf16 (norm outputs, projections, RoPE output, attention
output, residual stream, SiLU*up).  Differences to the GPU are fp32 summation
order and the GPU's fast exp in attention -> logits agree to ~1e-3 relative
(the tests use rtol 1e-2, the north-star tolerance).

Semantics mirrored from paper_2603_18016_b200/model.py (itself the real
counterpart of the reference's virtual pass durations, pkg/src/specsim/
request_model.py:92-117).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

from paper_2603_18016_b200.model import (INIT_SPAN, ModelShape, Transformer, rope_inv_freq,
                                         tensor_seed)

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


def _clib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle_model.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(path)
        L.oracle_fill_uniform.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                          ctypes.c_float]
        L.oracle_round_bf16.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        _lib = L
    return _lib


def rand_weight(shape, seed: int) -> np.ndarray:
    out = np.empty(shape, dtype=np.float32)
    _clib().oracle_fill_uniform(out.ctypes.data, out.size, seed, ctypes.c_float(INIT_SPAN))
    return out


def bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (RNE), kept as float32.  Returns a new array."""
    x = np.array(x, dtype=np.float32, copy=True, order="C")
    _clib().oracle_round_bf16(x.ctypes.data, x.size)
    return x


def _rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    ss = (x * x).sum(axis=1, dtype=np.float32) / np.float32(x.shape[1])
    inv = (np.float32(1.0) / np.sqrt(ss + np.float32(eps))).astype(np.float32)
    return bf16(x * inv[:, None] * g[None, :])


class OracleModel:
    """CPU forward with per-request contiguous KV caches."""

    def __init__(self, shape: ModelShape, seed: int) -> None:
        s = shape
        self.shape = s
        H, F = s.hidden, s.ffn
        self.layers = []
        for li in range(s.layers):
            L = {
                "wqkv": rand_weight((s.qkv_out, H), tensor_seed(seed, li, Transformer.W_QKV)),
                "wo": rand_weight((H, s.heads * s.head_dim), tensor_seed(seed, li, Transformer.W_O)),
                "gate": rand_weight((F, H), tensor_seed(seed, li, Transformer.W_GATE)),
                "up": rand_weight((F, H), tensor_seed(seed, li, Transformer.W_UP)),
                "down": rand_weight((H, F), tensor_seed(seed, li, Transformer.W_DOWN)),
                "bqkv": (rand_weight((s.qkv_out,), tensor_seed(seed, li, Transformer.B_QKV))
                         if s.qkv_bias else None),
            }
            self.layers.append(L)
        self.embed = rand_weight((s.vocab, H), tensor_seed(seed, -1, Transformer.W_EMB))
        self.lm_head = self.embed if s.tie_embeddings else rand_weight(
            (s.vocab, H), tensor_seed(seed, -1, Transformer.W_LM))
        self.ones = np.ones(H, np.float32)
        self.inv_freq = rope_inv_freq(s)

    def new_cache(self, max_len: int):
        s = self.shape
        return [(np.zeros((max_len, s.kv_heads, s.head_dim), np.float32),
                 np.zeros((max_len, s.kv_heads, s.head_dim), np.float32))
                for _ in range(s.layers)]

    def _rope(self, x: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """x [M, nh, D] fp32 (bf16 values) -> rotated, bf16."""
        D = x.shape[2]
        half = D // 2
        ang = pos.astype(np.float32)[:, None] * self.inv_freq[None, :]
        cs = np.cos(ang).astype(np.float32)[:, None, :]
        sn = np.sin(ang).astype(np.float32)[:, None, :]
        a, b = x[..., :half], x[..., half:]
        return bf16(np.concatenate([a * cs - b * sn, b * cs + a * sn], axis=2))

    def forward(self, seqs, caches):
        """seqs: list of (tokens list, first position); caches: matching list
        of per-request caches.  Writes K/V at the token positions, returns the
        final residual stream [sum n, H] (bf16 values)."""
        s = self.shape
        toks = np.concatenate([np.asarray(t, np.int64) for t, _ in seqs])
        pos = np.concatenate([np.arange(p0, p0 + len(t)) for t, p0 in seqs])
        bounds = np.cumsum([0] + [len(t) for t, _ in seqs])
        x = self.embed[toks].copy()
        Hq, Hkv, D = s.heads, s.kv_heads, s.head_dim
        G = Hq // Hkv
        scale = np.float32(1.0 / math.sqrt(D))
        for li, L in enumerate(self.layers):
            xn = _rmsnorm(x, self.ones, s.rms_eps)
            qkv = bf16(xn @ L["wqkv"].T)
            if L["bqkv"] is not None:
                qkv = bf16(qkv + L["bqkv"][None, :])
            q = self._rope(qkv[:, :Hq * D].reshape(-1, Hq, D), pos)
            k = self._rope(qkv[:, Hq * D:(Hq + Hkv) * D].reshape(-1, Hkv, D), pos)
            v = qkv[:, (Hq + Hkv) * D:].reshape(-1, Hkv, D)
            attn = np.empty((x.shape[0], Hq, D), np.float32)
            for si, ((t, p0), cache) in enumerate(zip(seqs, caches)):
                a, b = bounds[si], bounds[si + 1]
                Kc, Vc = cache[li]
                Kc[p0:p0 + len(t)] = k[a:b]
                Vc[p0:p0 + len(t)] = v[a:b]
                n = len(t)
                kv = p0 + n
                Ks = Kc[:kv]  # [kv, Hkv, D]
                Vs = Vc[:kv]
                for g in range(Hkv):
                    qg = q[a:b, g * G:(g + 1) * G, :].reshape(n * G, D)
                    sc = (qg @ Ks[:, g, :].T) * scale  # [n*G, kv]
                    qp = (p0 + np.arange(n)).repeat(G)
                    mask = np.arange(kv)[None, :] > qp[:, None]
                    sc = np.where(mask, -np.inf, sc).astype(np.float32)
                    sc = sc - sc.max(axis=1, keepdims=True)
                    p = np.exp(sc).astype(np.float32)
                    o = (p @ Vs[:, g, :]) / p.sum(axis=1, keepdims=True)
                    attn[a:b, g * G:(g + 1) * G, :] = o.reshape(n, G, D)
            attn = bf16(attn.reshape(x.shape[0], Hq * D))
            x = bf16(attn @ L["wo"].T + x)
            xn = _rmsnorm(x, self.ones, s.rms_eps)
            gt = xn @ L["gate"].T
            up = xn @ L["up"].T
            act = bf16(gt / (np.float32(1.0) + np.exp(-gt)) * up)
            x = bf16(act @ L["down"].T + x)
        return x

    def logits(self, hidden_rows: np.ndarray, prev_tokens: np.ndarray, succ=None,
               beta: float = 0.0) -> np.ndarray:
        xf = _rmsnorm(hidden_rows, self.ones, self.shape.rms_eps)
        lg = (xf @ self.lm_head.T).astype(np.float32)
        if succ is not None and beta != 0.0:
            lg[np.arange(lg.shape[0]), succ[prev_tokens]] += np.float32(beta)
        return lg
