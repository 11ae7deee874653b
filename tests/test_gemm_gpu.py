"""K2 (tcgen05 GEMM) vs a torch fp32 reference of the same op.

Shapes cover the verify (M = B(k+1)) and draft (M = B) token counts of the
BASELINE configs, split-K and no split, every epilogue.  Tolerance: bf16
output rounding + fp32 accumulation-order differences (rtol 1e-2 on values
of O(1), atol scaled by sqrt(K)).
"""

import pytest
import torch

from paper_2603_18016_b200 import native, ops

pytestmark = pytest.mark.gpu


def _ref(x, w):
    return x.float() @ w.float().T


def _close(got, ref, K):
    err = (got.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-2 * scale + 1e-3, (err, scale)


@pytest.mark.parametrize("M,N,K", [(32, 3072, 2048), (192, 6144, 4096), (160, 4608, 3584),
                                   (1, 128, 64), (37, 256, 192), (320, 2560, 8192),
                                   (64, 1024, 1000), (700, 512, 512), (192, 8192, 4096), (32, 128256, 2048),
                                   (384, 4096, 4096), (300, 1024, 2048), (512, 2048, 1024)])
@pytest.mark.parametrize("splits", [0, 1])
def test_gemm_bf16(cuda_device, M, N, K, splits):
    g = torch.Generator(device=cuda_device).manual_seed(M * 7 + N + K)
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    y = ops.gemm(x, w, splits=splits)
    torch.cuda.synchronize()
    _close(y, _ref(x, w), K)


@pytest.mark.parametrize("splits", [0, 1])
def test_gemm_f32_and_resid(cuda_device, splits):
    g = torch.Generator(device=cuda_device).manual_seed(5)
    M, N, K = 96, 2048, 2048
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    y = ops.gemm(x, w, epi=native.EPI_F32, splits=splits)
    torch.cuda.synchronize()
    _close(y, _ref(x, w), K)
    r = torch.randn(M, N, device=cuda_device, generator=g).to(torch.bfloat16)
    r0 = r.clone()
    ops.gemm(x, w, out=r, epi=native.EPI_RESID, residual=r, splits=splits)  # in place
    torch.cuda.synchronize()
    _close(r, _ref(x, w) + r0.float(), K)


@pytest.mark.parametrize("M,splits", [(32, 0), (192, 1), (192, 0), (384, 0), (320, 1), (300, 2)])
def test_gemm_silu_mul(cuda_device, M, splits):
    g = torch.Generator(device=cuda_device).manual_seed(9)
    F, K = 1024, 2048
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    wg = (torch.randn(F, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    wu = (torch.randn(F, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    from paper_2603_18016_b200.model import pack_gate_up
    packed = pack_gate_up(wg, wu)
    y = ops.gemm(x, packed, epi=native.EPI_SILU, splits=splits)
    torch.cuda.synchronize()
    gt = _ref(x, wg)
    ref = torch.nn.functional.silu(gt) * _ref(x, wu)
    _close(y, ref, K)


@pytest.mark.parametrize("M,N,K", [(192, 6144, 4096), (192, 4096, 14336), (32, 3072, 2048),
                                   (32, 2048, 8192), (320, 2560, 8192), (384, 6144, 4096)])
def test_gemm_partials_sum(cuda_device, M, N, K):
    """psd_gemm_partials: the sum of the returned split slices equals x @ w.T
    (split-K reduced through DSMEM inside a (1, 1, S) cluster when S <= 8)."""
    import ctypes
    g = torch.Generator(device=cuda_device).manual_seed(M + N + K)
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    part = torch.full((16 * M * N,), float("nan"), device=cuda_device)
    sp = ctypes.c_int()
    lib = native.load()
    native.check(lib.psd_gemm_partials(x.data_ptr(), K, M, K, w.data_ptr(), K, N,
                                       part.data_ptr(), part.numel() * 4, 0, ctypes.byref(sp),
                                       torch.cuda.current_stream().cuda_stream), "partials")
    torch.cuda.synchronize()
    got = part[:sp.value * M * N].view(sp.value, M, N).sum(0)
    _close(got, _ref(x, w), K)


@pytest.mark.parametrize("epi", [native.EPI_BF16, native.EPI_F32, native.EPI_SILU])
@pytest.mark.parametrize("pad", [8, 1])
@pytest.mark.parametrize("M", [37, 192])
def test_gemm_strided_out(cuda_device, epi, pad, M):
    """Stream-K output into a column slice of a wider buffer: a 16-byte aligned
    row stride leaves through TMA stores (rows m >= M clipped by the tensor
    map), an odd stride through per-thread stores; the padding is untouched."""
    g = torch.Generator(device=cuda_device).manual_seed(M + pad + epi)
    N, K = 2048, 1024
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    n_out = N // 2 if epi == native.EPI_SILU else N
    odt = torch.float32 if epi == native.EPI_F32 else torch.bfloat16
    big = torch.full((M + 3, n_out + pad), 7.0, dtype=odt, device=cuda_device)
    out = big[:M, :n_out]
    ops.gemm(x, w, out=out, epi=epi, splits=0)
    torch.cuda.synchronize()
    if epi == native.EPI_SILU:
        wg = torch.cat([w[t * 128 + q * 32: t * 128 + q * 32 + 16] for t in range(N // 128)
                        for q in range(4)])
        wu = torch.cat([w[t * 128 + q * 32 + 16: t * 128 + q * 32 + 32] for t in range(N // 128)
                        for q in range(4)])
        ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
    else:
        ref = _ref(x, w)
    _close(out, ref, K)
    assert (big[:, n_out:] == 7.0).all() and (big[M:] == 7.0).all()


@pytest.mark.parametrize("N,epi", [(28672, native.EPI_SILU), (19200, native.EPI_BF16),
                                   (37888, native.EPI_BF16), (18944, native.EPI_F32)])
def test_gemm_stream_k_schedules(cuda_device, N, epi):
    """Stream-K tile schedules on 148 SMs: 224 tiles (148 whole tiles + a
    stream-K share of 76), 150 (a 2-tile remainder: all tiles stream-K), 296
    (whole tiles only, no stream-K units), 148 (one wave: the grid kernel)."""
    g = torch.Generator(device=cuda_device).manual_seed(N + epi)
    M, K = 192, 512
    x = torch.randn(M, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    y = ops.gemm(x, w, epi=epi, splits=0)
    torch.cuda.synchronize()
    if epi == native.EPI_SILU:
        wg = w.view(N // 128, 4, 2, 16, K)[:, :, 0].reshape(N // 2, K)
        wu = w.view(N // 128, 4, 2, 16, K)[:, :, 1].reshape(N // 2, K)
        ref = torch.nn.functional.silu(_ref(x, wg)) * _ref(x, wu)
    else:
        ref = _ref(x, w)
    _close(y, ref, K)


def test_gemm_trace_timeline(cuda_device):
    """psd_gemm_set_trace: every stream-K CTA stamps entry <= first operands <=
    last MMA issued <= epilogue done, and its segment count; off again after."""
    lib = native.load()
    M, N, K = 192, 28672, 512
    x = torch.randn(M, K, device=cuda_device).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device) * 0.05).to(torch.bfloat16)
    tr = torch.zeros(1024, 16, dtype=torch.int64, device=cuda_device)
    lib.psd_gemm_set_trace(tr.data_ptr())
    try:
        ops.gemm(x, w, epi=native.EPI_SILU, splits=0)
        torch.cuda.synchronize()
    finally:
        lib.psd_gemm_set_trace(None)
    rows = [r for r in tr.cpu().tolist() if r[0]]
    assert len(rows) == torch.cuda.get_device_properties(cuda_device).multi_processor_count
    for r in rows:
        assert r[0] <= r[1] <= r[2] <= r[4] and r[5] >= 1
    tr.zero_()
    ops.gemm(x, w, epi=native.EPI_SILU, splits=0)
    torch.cuda.synchronize()
    assert int(tr.abs().sum()) == 0


@pytest.mark.parametrize("M,N,K", [(32, 128256, 2048), (1, 1024, 256), (8, 151936, 896),
                                   (64, 128256, 2048), (100, 2048, 512), (192, 128256, 4096),
                                   (256, 4096, 1024), (384, 128256, 4096), (512, 4096, 1024)])
@pytest.mark.parametrize("bias", [False, True])
def test_lm_head_argmax_epilogue(cuda_device, M, N, K, bias):
    """K6: argmax (+ the synthetic-language bias) in the stream-K LM head's
    epilogue + the tile fold == argmax of the same GEMM's stored fp32 logits
    after psd_bigram_bias (bit-identical values, lowest index on ties), and
    the fold's scatter into dst."""
    dev = cuda_device
    g = torch.Generator(device=dev).manual_seed(M + N + K)
    x = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    w[N // 2] = w[N // 3]       # exact ties: the lower index must win
    w[N - 1] = w[5]
    lib = native.load()
    st = torch.cuda.current_stream().cuda_stream
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    tokens = torch.randint(0, N, (M + 3,), device=dev, dtype=torch.int32, generator=g)
    rows = torch.arange(M, device=dev, dtype=torch.int32) + 3
    succ = torch.randint(0, N, (N,), device=dev, dtype=torch.int32, generator=g)
    beta = 7.0 if bias else 0.0
    logits = torch.empty(M, N, device=dev)
    assert lib.psd_gemm_bf16(x.data_ptr(), K, M, K, w.data_ptr(), K, N, logits.data_ptr(), N,
                             native.EPI_F32, None, 0, 0, ws.data_ptr(), ws.numel(), st) == 0
    if bias:
        prev = tokens[rows.long()].contiguous()
        assert lib.psd_bigram_bias(logits.data_ptr(), N, prev.data_ptr(), M, succ.data_ptr(), N,
                                   beta, st) == 0
    part = torch.empty(lib.psd_argmax_partials_bytes(M, N), dtype=torch.uint8, device=dev)
    out = torch.full((M,), -1, dtype=torch.int32, device=dev)
    dst = torch.full((2 * M,), -7, dtype=torch.int32, device=dev)
    dst_idx = (torch.arange(M, device=dev, dtype=torch.int32) * 2)
    dst_idx[0] = -1  # skipped
    assert lib.psd_gemm_argmax(x.data_ptr(), K, M, K, w.data_ptr(), K, N, tokens.data_ptr(),
                               rows.data_ptr(), succ.data_ptr() if bias else None, beta,
                               part.data_ptr(), ws.data_ptr(), ws.numel(), st) == 0
    assert lib.psd_argmax_fold(part.data_ptr(), M, N, out.data_ptr(), dst.data_ptr(),
                               dst_idx.data_ptr(), st) == 0
    torch.cuda.synchronize()
    ref = logits.argmax(dim=1).to(torch.int32)
    assert torch.equal(out, ref)
    assert dst[0].item() == -7 and torch.equal(dst[2::2], ref[1:])


@pytest.mark.parametrize("N,K,epi", [(4096, 4096, native.EPI_F32), (2048, 8192, native.EPI_F32),
                                     (8192, 4096, native.EPI_SILU),
                                     (128256, 4096, native.EPI_F32),
                                     (9728, 896, native.EPI_SILU)])
def test_stream_k_batch_invariant_any_m(cuda_device, N, K, epi):
    """Stream-K: a token's output bits do not depend on how many tokens share
    the launch -- M = 24 .. 1100 (one, two and up to five token tiles per
    weight tile), with and without a CTA cap -- so greedy PSD and SD(2m)
    agree at any verify width (cfg4's SD(2m) pass is 640 tokens)."""
    g = torch.Generator(device=cuda_device).manual_seed(N + K)
    Mmax = 1100
    x = torch.randn(Mmax, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    lib = native.load()
    ref = ops.gemm(x[:24], w, epi=epi)
    for M, cap in ((24, 74), (192, 0), (320, 0), (512, 0), (640, 0), (640, 74), (1100, 0)):
        lib.psd_gemm_set_max_ctas(cap)
        try:
            y = ops.gemm(x[:M], w, epi=epi)
        finally:
            lib.psd_gemm_set_max_ctas(0)
        torch.cuda.synchronize()
        assert torch.equal(y[:24], ref), (M, cap)
    _close(y, _ref(x, w) if epi != native.EPI_SILU else y.float(), K)


@pytest.mark.parametrize("N,K", [(4096, 4096), (6144, 4096), (8192, 8192), (2048, 8192)])
def test_split_k_partials_batch_invariant_any_m(cuda_device, N, K):
    """Grid split-K: the split count and every slice's bits for a token are
    the same at M = 32 and M = 640 / 1024 (the consumer then sums the same
    slices in the same order)."""
    import ctypes
    g = torch.Generator(device=cuda_device).manual_seed(N * 3 + K)
    Mmax = 1024
    x = torch.randn(Mmax, K, device=cuda_device, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda_device, generator=g) * 0.05).to(torch.bfloat16)
    lib = native.load()
    part = torch.empty(16 * Mmax * N, device=cuda_device)
    out = {}
    for M in (32, 320, 640, 1024):
        sp = ctypes.c_int()
        native.check(lib.psd_gemm_partials(x.data_ptr(), K, M, K, w.data_ptr(), K, N,
                                           part.data_ptr(), part.numel() * 4, 0,
                                           ctypes.byref(sp),
                                           torch.cuda.current_stream().cuda_stream), "partials")
        torch.cuda.synchronize()
        out[M] = (sp.value, part[:sp.value * M * N].view(sp.value, M, N)[:, :32].clone())
    s0, p0 = out[32]
    for M, (s, p) in out.items():
        assert s == s0, (M, s, s0)
        assert torch.equal(p, p0), M
    _close(p0.sum(0), _ref(x[:32], w), K)


@pytest.mark.parametrize("B,K", [(32, 5), (7, 8), (40, 1), (3, 0), (64, 5)])
@pytest.mark.parametrize("forced", [False, True])
def test_verify_greedy_from_argmax_epilogue(cuda_device, B, K, forced):
    """Greedy K1 fused into the target LM head (the verify path at <= 256 rows):
    psd_gemm_argmax + psd_argmax_fold + psd_verify_greedy_tokens give the same
    accepted lengths and output tokens as K1 (psd_verify_greedy) on the stored,
    biased fp32 logits -- drafts agreeing with the target for a random prefix."""
    dev = cuda_device
    N, H = 32000, 1024
    R = B * (K + 1)
    g = torch.Generator(device=dev).manual_seed(B * 31 + K + forced)
    x = torch.randn(R, H, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, H, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    lib = native.load()
    st = torch.cuda.current_stream().cuda_stream
    ws = torch.zeros(128 << 20, dtype=torch.uint8, device=dev)
    tokens = torch.randint(0, N, (R,), device=dev, dtype=torch.int32, generator=g)
    succ = torch.randint(0, N, (N,), device=dev, dtype=torch.int32, generator=g)
    beta = 7.0
    logits = torch.empty(R, N, device=dev)
    assert lib.psd_gemm_bf16(x.data_ptr(), H, R, H, w.data_ptr(), H, N, logits.data_ptr(), N,
                             native.EPI_F32, None, 0, 0, ws.data_ptr(), ws.numel(), st) == 0
    assert lib.psd_bigram_bias(logits.data_ptr(), N, tokens.data_ptr(), R, succ.data_ptr(), N,
                               beta, st) == 0
    torch.cuda.synchronize()
    am = logits.argmax(dim=1).view(B, K + 1)
    # drafts: the target's choice for a random prefix, then a miss
    ids = torch.randint(0, N, (B, max(K, 1)), device=dev, dtype=torch.int32, generator=g)[:, :K]
    for b in range(B):
        keep = int(torch.randint(0, K + 1, (1,), generator=torch.Generator().manual_seed(b)))
        ids[b, :keep] = am[b, :keep].to(torch.int32)
    ids = ids.contiguous()
    ln = torch.randint(0, K + 1, (B,), device=dev, dtype=torch.int32, generator=g)
    fl = torch.randint(0, K + 1, (B,), device=dev, dtype=torch.int32, generator=g) if forced else None
    acc_ref = torch.empty(B, dtype=torch.int32, device=dev)
    out_ref = torch.empty(B, K + 1, dtype=torch.int32, device=dev)
    ops.verify_greedy(logits.view(B, K + 1, N), ids, ln, acc_ref, out_ref, forced_len=fl)
    part = torch.empty(lib.psd_argmax_partials_bytes(R, N), dtype=torch.uint8, device=dev)
    tok = torch.empty(R, dtype=torch.int32, device=dev)
    assert lib.psd_gemm_argmax(x.data_ptr(), H, R, H, w.data_ptr(), H, N, tokens.data_ptr(),
                               None, succ.data_ptr(), beta, part.data_ptr(), ws.data_ptr(),
                               ws.numel(), st) == 0
    assert lib.psd_argmax_fold(part.data_ptr(), R, N, tok.data_ptr(), None, None, st) == 0
    acc = torch.full((B,), -9, dtype=torch.int32, device=dev)
    out = torch.full((B, K + 1), -9, dtype=torch.int32, device=dev)
    assert lib.psd_verify_greedy_tokens(tok.data_ptr(), ids.data_ptr(), ln.data_ptr(), B, K,
                                        fl.data_ptr() if fl is not None else None,
                                        acc.data_ptr(), out.data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert torch.equal(tok.view(B, K + 1), am.to(torch.int32))
    assert torch.equal(acc, acc_ref)
    assert torch.equal(out, out_ref)
