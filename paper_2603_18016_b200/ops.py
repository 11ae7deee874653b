"""Torch-facing wrappers over the C ABI (include/psd.h).

Torch is plumbing here: device memory, streams, dtype/shape checks.  Every
function launches on the *current* torch CUDA stream and returns without
synchronising.  No CPU fallback: a CPU tensor or a missing library raises.
"""

from __future__ import annotations

import torch

from . import native
from .errors import ConfigError

__all__ = ["gemm", "gemm_plan", "verify_greedy", "verify_sample"]

_workspaces: dict[tuple, torch.Tensor] = {}


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check(t: torch.Tensor, name: str, dtype: torch.dtype, ndim: int) -> None:
    if not t.is_cuda:
        raise ConfigError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ConfigError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != ndim:
        raise ConfigError(f"{name} must have {ndim} dims, got {tuple(t.shape)}")


def _verify_workspace(device, B, K, V, Vd, sampling) -> torch.Tensor:
    lib = native.load()
    stream = _stream_ptr(device)
    key = (device.index, stream, B, K, V, Vd, sampling)
    buf = _workspaces.get(key)
    if buf is None:
        nbytes = lib.psd_verify_workspace_bytes(B, K, V, Vd, int(sampling))
        buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        native.check(lib.psd_verify_workspace_init(buf.data_ptr(), nbytes, stream),
                     "psd_verify_workspace_init")
        _workspaces[key] = buf
    return buf


def _rows_view(x: torch.Tensor, name: str):
    """Strides (batch, position) in elements of a [B, P, V] logits view."""
    if x.stride(2) != 1:
        raise ConfigError(f"{name}: vocabulary dimension must be contiguous")
    return x.stride(0), x.stride(1)


def verify_greedy(target_logits: torch.Tensor, draft_ids: torch.Tensor,
                  draft_len: torch.Tensor, accepted_len: torch.Tensor | None = None,
                  out_tokens: torch.Tensor | None = None,
                  forced_len: torch.Tensor | None = None):
    """Greedy speculative verification (K1).

    target_logits [B, K+1, V] fp32; draft_ids [B, K] int32; draft_len [B]
    int32.  Returns (accepted_len [B] int32, out_tokens [B, K+1] int32).
    forced_len [B] int32: replay mode (psd_verify_greedy_forced).
    """
    _check(target_logits, "target_logits", torch.float32, 3)
    B, K1, V = target_logits.shape
    K = K1 - 1
    _check(draft_ids, "draft_ids", torch.int32, 2)
    _check(draft_len, "draft_len", torch.int32, 1)
    if tuple(draft_ids.shape) != (B, K) or draft_len.shape[0] != B:
        raise ConfigError("draft_ids must be [B, K] and draft_len [B]")
    dev = target_logits.device
    if accepted_len is None:
        accepted_len = torch.empty(B, dtype=torch.int32, device=dev)
    if out_tokens is None:
        out_tokens = torch.empty(B, K1, dtype=torch.int32, device=dev)
    ws = _verify_workspace(dev, B, K, V, 0, False)
    sb, si = _rows_view(target_logits, "target_logits")
    lib = native.load()
    if forced_len is not None:
        _check(forced_len, "forced_len", torch.int32, 1)
        native.check(lib.psd_verify_greedy_forced(
            target_logits.data_ptr(), sb, si, V, draft_ids.contiguous().data_ptr(),
            draft_len.contiguous().data_ptr(), B, K, forced_len.contiguous().data_ptr(),
            accepted_len.data_ptr(), out_tokens.data_ptr(), ws.data_ptr(), ws.numel(),
            _stream_ptr(dev)), "psd_verify_greedy_forced")
        return accepted_len, out_tokens
    native.check(lib.psd_verify_greedy(
        target_logits.data_ptr(), sb, si, V, draft_ids.contiguous().data_ptr(),
        draft_len.contiguous().data_ptr(), B, K, accepted_len.data_ptr(),
        out_tokens.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dev)),
        "psd_verify_greedy")
    return accepted_len, out_tokens


def verify_sample(target_logits: torch.Tensor, draft_logits: torch.Tensor,
                  draft_ids: torch.Tensor, draft_len: torch.Tensor, uniforms: torch.Tensor,
                  temperature: float = 1.0, accepted_len: torch.Tensor | None = None,
                  out_tokens: torch.Tensor | None = None, d_stats: torch.Tensor | None = None,
                  t_stats_out: torch.Tensor | None = None,
                  t_stats_rows: torch.Tensor | None = None,
                  forced_len: torch.Tensor | None = None):
    """Speculative rejection sampling (K1).

    target_logits [B, K+1, V], draft_logits [B, K, Vd] fp32 (Vd <= V);
    uniforms [B, K+1] fp32 in [0, 1).  Returns (accepted_len, out_tokens).
    d_stats [B, K, 2] fp32: cached (max, sum) of the draft rows (not re-read);
    t_stats_out [*, 2] + t_stats_rows [B] int32: receive the (max, sum) of
    target row 0 (psd_verify_sample_ext).  forced_len [B] int32: replay mode
    (psd_verify_sample_forced).
    """
    _check(target_logits, "target_logits", torch.float32, 3)
    _check(draft_logits, "draft_logits", torch.float32, 3)
    B, K1, V = target_logits.shape
    K = K1 - 1
    Vd = draft_logits.shape[2]
    if draft_logits.shape[0] != B or draft_logits.shape[1] < max(K, 1) and K > 0:
        raise ConfigError("draft_logits must be [B, K, Vd]")
    _check(draft_ids, "draft_ids", torch.int32, 2)
    _check(draft_len, "draft_len", torch.int32, 1)
    _check(uniforms, "uniforms", torch.float32, 2)
    if tuple(uniforms.shape) != (B, K1):
        raise ConfigError("uniforms must be [B, K+1]")
    dev = target_logits.device
    if accepted_len is None:
        accepted_len = torch.empty(B, dtype=torch.int32, device=dev)
    if out_tokens is None:
        out_tokens = torch.empty(B, K1, dtype=torch.int32, device=dev)
    ws = _verify_workspace(dev, B, K, V, Vd, True)
    sb, si = _rows_view(target_logits, "target_logits")
    if draft_logits.numel() == 0:  # K == 0: idle passes only, draft rows never read
        draft_logits, Vd = target_logits, V
    db, di = _rows_view(draft_logits, "draft_logits")
    lib = native.load()
    if d_stats is not None or t_stats_out is not None or forced_len is not None:
        if d_stats is not None:
            _check(d_stats, "d_stats", torch.float32, 3)
        if forced_len is not None:
            _check(forced_len, "forced_len", torch.int32, 1)
        native.check(lib.psd_verify_sample_forced(
            target_logits.data_ptr(), sb, si, V, draft_logits.data_ptr(), None, db, di, Vd,
            draft_ids.contiguous().data_ptr(), draft_len.contiguous().data_ptr(),
            uniforms.contiguous().data_ptr(), float(temperature), B, K,
            forced_len.contiguous().data_ptr() if forced_len is not None else None,
            accepted_len.data_ptr(),
            out_tokens.data_ptr(), d_stats.data_ptr() if d_stats is not None else None,
            d_stats.stride(0) // 2 if d_stats is not None else 0,
            t_stats_out.data_ptr() if t_stats_out is not None else None,
            t_stats_rows.data_ptr() if t_stats_rows is not None else None,
            ws.data_ptr(), ws.numel(), _stream_ptr(dev)), "psd_verify_sample_forced")
        return accepted_len, out_tokens
    native.check(lib.psd_verify_sample(
        target_logits.data_ptr(), sb, si, V, draft_logits.data_ptr(), db, di, Vd,
        draft_ids.contiguous().data_ptr(), draft_len.contiguous().data_ptr(),
        uniforms.contiguous().data_ptr(), float(temperature), B, K, accepted_len.data_ptr(),
        out_tokens.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dev)),
        "psd_verify_sample")
    return accepted_len, out_tokens


# ---------------------------------------------------------------------------
# K2: tcgen05 GEMM
# ---------------------------------------------------------------------------
def gemm_plan(M: int, N: int, K: int, epi: int = 0, splits: int = 0) -> tuple[int, int]:
    """(splits, workspace bytes) the GEMM will use for this shape."""
    import ctypes
    lib = native.load()
    s = ctypes.c_int()
    w = ctypes.c_size_t()
    native.check(lib.psd_gemm_plan(M, N, K, epi, splits, ctypes.byref(s), ctypes.byref(w)),
                 "psd_gemm_plan")
    return s.value, w.value


def gemm(x: torch.Tensor, w: torch.Tensor, out: torch.Tensor | None = None,
         epi: int = 0, residual: torch.Tensor | None = None, splits: int = 0,
         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """out = epi(x @ w.T) on tcgen05.  x [M, K] bf16, w [N, K] bf16 (row-major).

    epi: native.EPI_BF16 / EPI_F32 / EPI_RESID (out = acc + residual) /
    EPI_SILU (w packed gate/up per 128-row tile, out [M, N/2]).
    """
    _check(x, "x", torch.bfloat16, 2)
    _check(w, "w", torch.bfloat16, 2)
    M, K = x.shape
    N = w.shape[0]
    if w.shape[1] != K or x.stride(1) != 1 or w.stride(1) != 1:
        raise ConfigError("gemm: x [M, K], w [N, K] with unit inner stride")
    n_out = N // 2 if epi == native.EPI_SILU else N
    odt = torch.float32 if epi == native.EPI_F32 else torch.bfloat16
    if out is None:
        out = torch.empty(M, n_out, dtype=odt, device=x.device)
    if out.dtype != odt or out.shape[0] != M or out.shape[1] != n_out or out.stride(1) != 1:
        raise ConfigError(f"gemm: out must be [{M}, {n_out}] {odt}")
    if epi == native.EPI_RESID:
        if residual is None or residual.dtype != torch.bfloat16 or residual.stride(1) != 1:
            raise ConfigError("gemm: EPI_RESID needs a bf16 residual [M, N]")
    if splits < 0:  # legacy split-K with automatic split count
        splits, _ = gemm_plan(M, N, K, native.EPI_PARTIAL, 0)
    nsplit, need = gemm_plan(M, N, K, epi, splits)
    if need and (workspace is None or workspace.numel() * workspace.element_size() < need):
        workspace = torch.zeros(need, dtype=torch.uint8, device=x.device)
    lib = native.load()
    native.check(lib.psd_gemm_bf16(
        x.data_ptr(), x.stride(0), M, K, w.data_ptr(), w.stride(0), N, out.data_ptr(),
        out.stride(0), epi, residual.data_ptr() if residual is not None else None,
        residual.stride(0) if residual is not None else 0, splits,
        workspace.data_ptr() if workspace is not None else None,
        (workspace.numel() * workspace.element_size()) if workspace is not None else 0,
        _stream_ptr(x.device)), "psd_gemm_bf16")
    return out
