"""K4 building blocks vs torch fp32 references: fused add+RMSNorm, RoPE + KV
write, embedding, and the GEMM shapes of the tiny model (stream-K edge cases
with many contributors per tile)."""

import math

import numpy as np
import pytest
import torch

from paper_2603_18016_b200 import native, ops

pytestmark = pytest.mark.gpu
bf = torch.bfloat16


@pytest.mark.parametrize("M,H,S", [(63, 256, 0), (32, 2048, 6), (192, 4096, 4), (5, 896, 2)])
def test_add_rmsnorm(cuda_device, M, H, S):
    dev = cuda_device
    x = torch.randn(M, H, device=dev).to(bf)
    P = torch.randn(max(S, 1), M, H, device=dev)
    w = (torch.rand(H, device=dev) + 0.5).to(bf)
    y = torch.empty_like(x)
    x0 = x.clone()
    lib = native.load()
    rc = lib.psd_add_rmsnorm(x.data_ptr(), H, P.data_ptr() if S else None, S, M * H, H, None,
                             w.data_ptr(), y.data_ptr(), H, M, H, 1e-5, 1,
                             torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    acc = torch.zeros(M, H, device=dev)
    for z in range(S):  # the kernel's summation order
        acc = acc + P[z]
    v = (acc + x0.float()).to(bf).float() if S else x0.float()
    ref = v * torch.rsqrt((v * v).mean(1, keepdim=True) + 1e-5) * w.float()
    assert (y.float() - ref).abs().max().item() < 2e-2 * ref.abs().max().item()
    if S:
        assert torch.equal(x, v.to(bf))


@pytest.mark.parametrize("Hq,Hkv,D", [(8, 2, 32), (32, 8, 64), (32, 8, 128), (28, 4, 128)])
def test_rope_kv(cuda_device, Hq, Hkv, D):
    dev = cuda_device
    M = 19
    qkv = torch.randn(M, (Hq + 2 * Hkv) * D, device=dev).to(bf)
    pos = torch.arange(M, dtype=torch.int32, device=dev) * 7 + 3
    slots = torch.arange(M, dtype=torch.int32, device=dev) * 2
    slots[5] = -1
    inv = (1.0 / (10000.0 ** (torch.arange(0, D, 2, device=dev).float() / D))).contiguous()
    q = torch.zeros(M, Hq, D, dtype=bf, device=dev)
    kc = torch.zeros(2 * M, Hkv, D, dtype=bf, device=dev)
    vc = torch.zeros(2 * M, Hkv, D, dtype=bf, device=dev)
    lib = native.load()
    rc = lib.psd_rope_kv(qkv.data_ptr(), M, Hq, Hkv, D, pos.data_ptr(), slots.data_ptr(),
                         inv.data_ptr(), None, q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    x = qkv.float().view(M, Hq + 2 * Hkv, D)
    ang = pos.float()[:, None] * inv[None, :]
    cs, sn = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    a, b = x[..., :D // 2], x[..., D // 2:]
    rot = torch.cat([a * cs - b * sn, b * cs + a * sn], dim=2)
    assert (q.float() - rot[:, :Hq]).abs().max().item() < 3e-2
    for m in range(M):
        s = slots[m].item()
        if s < 0:
            continue
        assert (kc[s].float() - rot[m, Hq:Hq + Hkv]).abs().max().item() < 3e-2
        assert torch.equal(vc[s], qkv[m].view(Hq + 2 * Hkv, D)[Hq + Hkv:])


_WS = {}


def _shared_ws(dev):
    if "ws" not in _WS:
        _WS["ws"] = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    return _WS["ws"]


@pytest.mark.parametrize("M,N,K,epi", [(63, 1024, 256, "f32"), (63, 384, 256, "bf16"),
                                       (63, 256, 704, "bf16"), (63, 1408, 256, "silu"),
                                       (16, 256, 128, "bf16"), (128, 1024, 256, "f32")])
def test_tiny_model_gemm_shapes(cuda_device, M, N, K, epi):
    dev = cuda_device
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    x = torch.randn(M, K, device=dev, generator=g).to(bf)
    w = (torch.randn(N, K, device=dev, generator=g) * 0.05).to(bf)
    e = {"bf16": native.EPI_BF16, "silu": native.EPI_SILU, "f32": native.EPI_F32}[epi]
    ws = _shared_ws(dev)
    # interleave with a GEMM of another shape on the same workspace: the
    # stream-K tickets must stay valid across shapes
    other_x = torch.randn(192, 512, device=dev).to(bf)
    other_w = (torch.randn(4096, 512, device=dev) * 0.05).to(bf)
    for _ in range(2):
        y = ops.gemm(x, w, epi=e, workspace=ws)
        ops.gemm(other_x, other_w, workspace=ws)
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    if epi == "silu":
        F = N // 2
        gt = ref.view(M, F // 64, 4, 2, 16)[:, :, :, 0].reshape(M, F)
        up = ref.view(M, F // 64, 4, 2, 16)[:, :, :, 1].reshape(M, F)
        ref = torch.nn.functional.silu(gt) * up
    err = (y.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K,epi", [(192, 1024, 4096, "bf16"), (32, 2048, 1000, "silu"),
                                       (63, 1024, 256, "f32"), (300, 512, 704, "bf16")])
def test_gemm_pretiled_weights(cuda_device, M, N, K, epi):
    if not native.has("psd_gemm_tiled"):
        pytest.skip("experimental build only (PSD_EXPERIMENTAL=1)")
    dev = cuda_device
    g = torch.Generator(device=dev).manual_seed(M * 3 + N + K)
    x = torch.randn(M, K, device=dev, generator=g).to(bf)
    w = (torch.randn(N, K, device=dev, generator=g) * 0.05).to(bf)
    lib = native.load()
    st = torch.cuda.current_stream().cuda_stream
    t = torch.empty(lib.psd_tiled_weight_bytes(N, K) // 2, dtype=bf, device=dev)
    assert lib.psd_tile_weights(w.data_ptr(), N, K, K, t.data_ptr(), st) == 0
    e = {"bf16": native.EPI_BF16, "silu": native.EPI_SILU, "f32": native.EPI_F32}[epi]
    n_out = N // 2 if epi == "silu" else N
    y = torch.empty(M, n_out, dtype=torch.float32 if epi == "f32" else bf, device=dev)
    ws = _shared_ws(dev)
    assert lib.psd_gemm_tiled(x.data_ptr(), K, M, K, t.data_ptr(), N, y.data_ptr(), n_out, e,
                              None, 0, ws.data_ptr(), ws.numel(), st) == 0
    torch.cuda.synchronize()
    ref = x.float() @ w.float().T
    if epi == "silu":
        F = N // 2
        gt = ref.view(M, F // 64, 4, 2, 16)[:, :, :, 0].reshape(M, F)
        up = ref.view(M, F // 64, 4, 2, 16)[:, :, :, 1].reshape(M, F)
        ref = torch.nn.functional.silu(gt) * up
    err = (y.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-3, err
