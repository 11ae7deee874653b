"""Torch-facing wrappers over the C ABI (include/psd.h).

Torch is plumbing here: device memory, streams, dtype/shape checks.  Every
function launches on the *current* torch CUDA stream and returns without
synchronising.  No CPU fallback: a CPU tensor or a missing library raises.
"""

from __future__ import annotations

import torch

from . import native
from .errors import ConfigError

__all__ = ["verify_greedy", "verify_sample"]

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
                  out_tokens: torch.Tensor | None = None):
    """Greedy speculative verification (K1).

    target_logits [B, K+1, V] fp32; draft_ids [B, K] int32; draft_len [B]
    int32.  Returns (accepted_len [B] int32, out_tokens [B, K+1] int32).
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
    native.check(lib.psd_verify_greedy(
        target_logits.data_ptr(), sb, si, V, draft_ids.contiguous().data_ptr(),
        draft_len.contiguous().data_ptr(), B, K, accepted_len.data_ptr(),
        out_tokens.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dev)),
        "psd_verify_greedy")
    return accepted_len, out_tokens


def verify_sample(target_logits: torch.Tensor, draft_logits: torch.Tensor,
                  draft_ids: torch.Tensor, draft_len: torch.Tensor, uniforms: torch.Tensor,
                  temperature: float = 1.0, accepted_len: torch.Tensor | None = None,
                  out_tokens: torch.Tensor | None = None):
    """Speculative rejection sampling (K1).

    target_logits [B, K+1, V], draft_logits [B, K, Vd] fp32 (Vd <= V);
    uniforms [B, K+1] fp32 in [0, 1).  Returns (accepted_len, out_tokens).
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
    native.check(lib.psd_verify_sample(
        target_logits.data_ptr(), sb, si, V, draft_logits.data_ptr(), db, di, Vd,
        draft_ids.contiguous().data_ptr(), draft_len.contiguous().data_ptr(),
        uniforms.contiguous().data_ptr(), float(temperature), B, K, accepted_len.data_ptr(),
        out_tokens.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dev)),
        "psd_verify_sample")
    return accepted_len, out_tokens
