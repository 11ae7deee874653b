"""Deterministic, numpy-version-independent test inputs (splitmix64 in numpy)."""

from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)


def splitmix(seed: int, n: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (np.arange(n, dtype=np.uint64) + np.uint64(seed & 0xFFFFFFFF) * np.uint64(1 << 32)
             ) * _G + _G
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
        return x ^ (x >> np.uint64(31))


def uniform(seed: int, shape) -> np.ndarray:
    """float32 in [0, 1): top 24 bits of splitmix64."""
    n = int(np.prod(shape))
    return ((splitmix(seed, n) >> np.uint64(40)).astype(np.float32) *
            np.float32(2.0 ** -24)).reshape(shape)


def normalish(seed: int, shape, scale: float = 2.0) -> np.ndarray:
    """Approximately N(0, scale^2) float32 (Irwin-Hall of 4 uniforms)."""
    u = uniform(seed, (4,) + tuple(shape))
    return ((u.sum(axis=0) - np.float32(2.0)) * np.float32(scale * np.sqrt(3.0))).astype(
        np.float32)


def verify_case(seed: int, B: int, K: int, V: int, Vd: int | None = None, tau: float = 0.5,
                greedy: bool = False, ragged: bool = True):
    """Target logits, draft logits (= target + noise), draft ids, lengths, uniforms."""
    Vd = V if Vd is None else Vd
    t = normalish(seed, (B, K + 1, V))
    d = (t[:, :K, :Vd] + normalish(seed + 1, (B, K, Vd), tau)).astype(np.float32)
    if greedy:
        ids = d.argmax(axis=2).astype(np.int32) if K else np.zeros((B, 0), np.int32)
    else:
        # sample ids from q by inverse CDF (float64)
        ids = np.zeros((B, K), np.int32)
        uu = uniform(seed + 2, (B, max(K, 1)))
        for b in range(B):
            for i in range(K):
                q = np.exp(d[b, i].astype(np.float64) - d[b, i].max())
                c = np.cumsum(q / q.sum())
                ids[b, i] = min(int(np.searchsorted(c, uu[b, i], side="right")), Vd - 1)
    if ragged:
        ln = (splitmix(seed + 3, B) % np.uint64(K + 1)).astype(np.int32)
        ln[0] = K
    else:
        ln = np.full(B, K, np.int32)
    u = uniform(seed + 4, (B, K + 1))
    return t, d, ids, ln, u
