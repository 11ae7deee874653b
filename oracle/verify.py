"""ctypes binding of oracle/liboracle_verify.so (see verify_oracle.c).

Test infrastructure only (see oracle/__init__.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_verify.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_exp2.restype = ctypes.c_float
        L.oracle_exp2.argtypes = [ctypes.c_float]
        L.oracle_row_stats.restype = None
        L.oracle_row_stats.argtypes = [_f32p, ctypes.c_int, ctypes.c_float, _f32p, _f32p]
        L.oracle_row_argmax.restype = ctypes.c_int32
        L.oracle_row_argmax.argtypes = [_f32p, ctypes.c_int]
        L.oracle_verify_greedy.restype = ctypes.c_int
        L.oracle_verify_greedy.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                           _i32p, _i32p, ctypes.c_int, ctypes.c_int, _i32p, _i32p]
        L.oracle_verify_sample.restype = ctypes.c_int
        L.oracle_verify_sample.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                           _f32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                           _i32p, _i32p, _f32p, ctypes.c_float, ctypes.c_int,
                                           ctypes.c_int, _i32p, _i32p]
        L.oracle_verify_greedy_forced.restype = ctypes.c_int
        L.oracle_verify_greedy_forced.argtypes = (L.oracle_verify_greedy.argtypes[:8] + [_i32p]
                                                  + L.oracle_verify_greedy.argtypes[8:])
        L.oracle_verify_sample_forced.restype = ctypes.c_int
        L.oracle_verify_sample_forced.argtypes = (L.oracle_verify_sample.argtypes[:14] + [_i32p]
                                                  + L.oracle_verify_sample.argtypes[14:])
        _lib = L
    return _lib


def _fp(a):
    return a.ctypes.data_as(_f32p)


def _ip(a):
    return a.ctypes.data_as(_i32p)


def exp2(x: float) -> float:
    return lib().oracle_exp2(float(x))


def row_stats(row: np.ndarray, temperature: float = 1.0) -> tuple[float, float]:
    row = np.ascontiguousarray(row, dtype=np.float32)
    M, S = ctypes.c_float(), ctypes.c_float()
    lib().oracle_row_stats(_fp(row), row.size, ctypes.c_float(np.float32(1.0) /
                                                              np.float32(temperature)),
                           ctypes.byref(M), ctypes.byref(S))
    return M.value, S.value


def verify_greedy(target: np.ndarray, draft_ids: np.ndarray, draft_len: np.ndarray,
                  forced_len: np.ndarray | None = None):
    """target [B, K+1, V] f32, draft_ids [B, K] i32, draft_len [B] i32;
    forced_len [B] i32: replay mode (accept exactly min(forced, k_b))."""
    t = np.ascontiguousarray(target, dtype=np.float32)
    B, K1, V = t.shape
    K = K1 - 1
    ids = np.ascontiguousarray(draft_ids, dtype=np.int32).reshape(B, K)
    ln = np.ascontiguousarray(draft_len, dtype=np.int32)
    acc = np.zeros(B, np.int32)
    out = np.zeros((B, K + 1), np.int32)
    if forced_len is not None:
        fl = np.ascontiguousarray(forced_len, dtype=np.int32)
        rc = lib().oracle_verify_greedy_forced(_fp(t), K1 * V, V, V, _ip(ids), _ip(ln), B, K,
                                               _ip(fl), _ip(acc), _ip(out))
    else:
        rc = lib().oracle_verify_greedy(_fp(t), K1 * V, V, V, _ip(ids), _ip(ln), B, K,
                                        _ip(acc), _ip(out))
    if rc:
        raise ValueError("oracle_verify_greedy: bad arguments")
    return acc, out


def verify_sample(target: np.ndarray, draft: np.ndarray, draft_ids: np.ndarray,
                  draft_len: np.ndarray, uniforms: np.ndarray, temperature: float = 1.0,
                  forced_len: np.ndarray | None = None):
    """target [B, K+1, V], draft [B, K, Vd] f32; uniforms [B, K+1] f32."""
    t = np.ascontiguousarray(target, dtype=np.float32)
    d = np.ascontiguousarray(draft, dtype=np.float32)
    B, K1, V = t.shape
    K = K1 - 1
    Vd = d.shape[2]
    if K == 0:
        d = np.zeros((B, 1, Vd), np.float32)
    ids = np.ascontiguousarray(draft_ids, dtype=np.int32).reshape(B, K)
    ln = np.ascontiguousarray(draft_len, dtype=np.int32)
    u = np.ascontiguousarray(uniforms, dtype=np.float32).reshape(B, K + 1)
    acc = np.zeros(B, np.int32)
    out = np.zeros((B, K + 1), np.int32)
    args = (_fp(t), K1 * V, V, V, _fp(d), max(K, 1) * Vd, Vd, Vd, _ip(ids), _ip(ln), _fp(u),
            ctypes.c_float(temperature), B, K)
    if forced_len is not None:
        fl = np.ascontiguousarray(forced_len, dtype=np.int32)
        rc = lib().oracle_verify_sample_forced(*args, _ip(fl), _ip(acc), _ip(out))
    else:
        rc = lib().oracle_verify_sample(*args, _ip(acc), _ip(out))
    if rc:
        raise ValueError("oracle_verify_sample: bad arguments")
    return acc, out
