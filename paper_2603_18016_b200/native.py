"""ctypes binding of libpsd.so -- the C ABI declared in include/psd.h.

The product path has no CPU fallback: if the library is missing, every entry
point raises ``NativeError`` (on a GPU host this is loud by design).
"""

from __future__ import annotations

import ctypes
import os
import re

from .errors import NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
# PSD_LIB: an alternative build of the same ABI (experiments / bisection)
LIB_PATH = os.path.abspath(os.environ["PSD_LIB"]) if os.environ.get("PSD_LIB") else \
    os.path.join(_HERE, "libpsd.so")
HEADER = os.path.join(_HERE, "..", "include", "psd.h")

_c = ctypes
_p = _c.c_void_p
_i = _c.c_int
_i64 = _c.c_int64
_sz = _c.c_size_t
_f = _c.c_float

# name -> (restype, argtypes); must match include/psd.h exactly
SIGNATURES: dict[str, tuple] = {
    "psd_verify_workspace_bytes": (_sz, [_i, _i, _i, _i, _i]),
    "psd_verify_workspace_init": (_i, [_p, _sz, _p]),
    "psd_verify_greedy": (_i, [_p, _i64, _i64, _i, _p, _p, _i, _i, _p, _p, _p, _sz, _p]),
    "psd_verify_sample": (_i, [_p, _i64, _i64, _i, _p, _i64, _i64, _i, _p, _p, _p, _f, _i, _i,
                               _p, _p, _p, _sz, _p]),
    "psd_gemm_plan": (_i, [_i, _i, _i, _i, _i, _c.POINTER(_i), _c.POINTER(_sz)]),
    "psd_gemm_bf16": (_i, [_p, _i, _i, _i, _p, _i, _i, _p, _i, _i, _p, _i, _i, _p, _sz, _p]),
    "psd_argmax_partials_bytes": (_sz, [_i, _i]),
    "psd_gemm_argmax": (_i, [_p, _i, _i, _i, _p, _i, _i, _p, _p, _p, _f, _p, _p, _sz, _p]),
    "psd_argmax_fold": (_i, [_p, _i, _i, _p, _p, _p, _p]),
    "psd_embed": (_i, [_p, _i, _p, _i, _p, _p]),
    "psd_add_rmsnorm": (_i, [_p, _i, _p, _i, _sz, _i, _p, _p, _p, _i, _i, _i, _f, _i, _p]),
    "psd_rope_kv": (_i, [_p, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "psd_tiled_weight_bytes": (_sz, [_i, _i]),
    "psd_tile_weights": (_i, [_p, _i, _i, _i, _p, _p]),
    "psd_gemm_tiled": (_i, [_p, _i, _i, _i, _p, _i, _p, _i, _i, _p, _i, _p, _sz, _p]),
    "psd_gemm_partials": (_i, [_p, _i, _i, _i, _p, _i, _i, _p, _sz, _i, _c.POINTER(_i), _p]),
    "psd_attention": (_i, [_p, _p, _p, _p, _i, _p, _p, _p, _p, _p, _i, _i, _i, _i, _i, _i, _f,
                           _p, _i, _p, _sz, _p]),
    "psd_attention_workspace_bytes": (_sz, [_i, _i, _i, _i, _i, _i]),
    "psd_attention_rope": (_i, [_p, _i, _sz, _p, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _p,
                                _i, _i, _i, _i, _i, _i, _f, _p, _p]),
    "psd_bigram_bias": (_i, [_p, _i64, _p, _i, _p, _i, _f, _p]),
    "psd_bigram_bias_range": (_i, [_p, _i64, _p, _i, _p, _i, _f, _i, _i, _p]),
    "psd_philox_uniforms": (_i, [_c.c_uint64, _p, _p, _i, _i, _i, _p, _p]),
    "psd_rope_kv_partials": (_i, [_p, _i, _sz, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p]),
    "psd_copy_rows_f32": (_i, [_p, _p, _i64, _p, _i64, _i, _i, _p]),
    "psd_gather_rows_f32": (_i, [_p, _i64, _p, _p, _i64, _i, _i, _p]),
    "psd_verify_sample_rows": (_i, [_p, _i64, _i64, _i, _p, _p, _i64, _i64, _i, _p, _p, _p, _f,
                                    _i, _i, _p, _p, _p, _sz, _p]),
    "psd_verify_sample_ext": (_i, [_p, _i64, _i64, _i, _p, _p, _i64, _i64, _i, _p, _p, _p, _f,
                                   _i, _i, _p, _p, _p, _i64, _p, _p, _p, _sz, _p]),
    "psd_verify_greedy_forced": (_i, [_p, _i64, _i64, _i, _p, _p, _i, _i, _p, _p, _p, _p, _sz,
                                      _p]),
    "psd_verify_sample_forced": (_i, [_p, _i64, _i64, _i, _p, _p, _i64, _i64, _i, _p, _p, _p,
                                      _f, _i, _i, _p, _p, _p, _p, _i64, _p, _p, _p, _sz, _p]),
    "psd_verify_partials_count": (_sz, [_i, _i, _i]),
    "psd_verify_greedy_partials": (_i, [_p, _i64, _i64, _i, _i, _p, _i, _i, _p, _p]),
    "psd_verify_greedy_fold": (_i, [_p, _i, _i, _p, _p, _i, _i, _p, _p, _p, _p]),
    "psd_commit": (_i, [_p, _p, _i, _p, _i, _p, _p, _i, _p, _i, _p]),
    "psd_index_copy_i32": (_i, [_p, _p, _p, _p, _i, _p]),
    "psd_verify_greedy_tokens": (_i, [_p, _p, _p, _i, _i, _p, _p, _p, _p]),
    "psd_copy_async": (_i, [_p, _p, _sz, _p]),
    "psd_stage_draft": (_i, [_p, _i64, _p, _p, _i, _p, _i, _i, _i, _i, _p, _p, _p, _i, _i, _i]),
    "psd_stage_verify": (_i, [_p, _p, _p, _i, _p, _i, _i, _i, _i, _p, _p, _p, _i, _i, _i]),
    "psd_fill_uniform_bf16": (_i, [_p, _sz, _c.c_uint64, _f, _p]),
    "psd_fill_uniform_bf16_block": (_i, [_p, _i64, _i, _i, _i64, _i64, _i64, _c.c_uint64, _f,
                                         _p]),
    "psd_launch_count": (_c.c_longlong, []),
    "psd_gemm_set_max_ctas": (None, [_i]),
    "psd_gemm_set_whole_k": (None, [_i]),
    "psd_gemm_set_trace": (None, [_p]),
    "psd_comm_handle_bytes": (_sz, []),
    "psd_comm_create": (_i, [_i, _i, _sz, _sz, _c.POINTER(_p), _p]),
    "psd_comm_open": (_i, [_p, _p]),
    "psd_comm_create_local": (_i, [_i, _p, _sz, _sz, _p]),
    "psd_comm_destroy": (_i, [_p]),
    "psd_tp_allreduce_partials": (_i, [_p, _p, _i, _sz, _sz, _p, _p]),
    "psd_tp_allreduce_f32": (_i, [_p, _p, _sz, _p]),
    "psd_tp_allgather_f32": (_i, [_p, _p, _sz, _p, _p]),
    "psd_p2p_put_i32": (_i, [_p, _i, _p, _i, _p]),
    "psd_p2p_get_i32": (_i, [_p, _i, _p, _i, _p]),
    "psd_mk_smem_bytes": (_sz, []),
    "psd_mk_create": (_p, [_p]),
    "psd_mk_destroy": (None, [_p]),
    "psd_mk_grid": (_i, [_p]),
    "psd_mk_launch": (_i, [_p, _i, _i, _p]),
    "psd_mk_n_ops": (_i, [_p, _i, _i]),
    "psd_mk_launch_traced": (_i, [_p, _i, _i, _p, _p]),
}


class MkModel(_c.Structure):
    """psd_mk_model (include/psd.h): the draft model + forward buffers bound to
    the fused k-step decode kernel."""

    _fields_ = [(n, _i) for n in ("layers", "hidden", "heads", "kv_heads", "head_dim", "ffn",
                                  "vocab")] + \
        [(n, _f) for n in ("eps", "attn_scale", "beta")] + \
        [(n, _i) for n in ("block_size", "max_blocks", "grid", "max_tokens")] + \
        [(n, _p) for n in ("layer_ptrs", "embed", "lm_head", "final_norm", "inv_freq",
                           "successor", "block_table", "x", "xn", "attn", "act", "xf", "part",
                           "argpart", "slot_tok", "meta")] + \
        [("set_stride", _i), ("field_offsets", _i * 11)]

EPI_BF16, EPI_F32, EPI_RESID, EPI_SILU, EPI_PARTIAL = 0, 1, 2, 3, 4

_lib = None


# include/psd_experimental.h (PSD_EXPERIMENTAL=1 builds only)
EXPERIMENTAL = ("psd_tiled_weight_bytes", "psd_tile_weights", "psd_gemm_tiled",
                "psd_mk_smem_bytes", "psd_mk_create", "psd_mk_destroy", "psd_mk_grid",
                "psd_mk_launch", "psd_mk_n_ops", "psd_mk_launch_traced")


def has(name: str) -> bool:
    """Whether the loaded library exports `name` (experimental symbols)."""
    return getattr(load(), name, None) is not None


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function declared in include/psd.h (or `path`)."""
    with open(path) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|void|float|long long)\s*\**\s*(psd_\w+)\s*\(",
                                 text, re.M)))


def load():
    """Load libpsd.so once and attach the signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: run `python -m "
                          "paper_2603_18016_b200.build_native` (there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            if name in EXPERIMENTAL:
                continue  # built only with PSD_EXPERIMENTAL=1
            raise NativeError(f"{LIB_PATH} does not export {name}")
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


# psd_stage_* return codes (include/psd.h)
STAGE_BAD_ARGS = 1001
STAGE_CAPACITY = 1002
STAGE_KV_OVERRUN = 1003


def check(rc: int, what: str) -> None:
    if rc != 0:
        raise NativeError(f"{what} failed: cudaError {rc}")
