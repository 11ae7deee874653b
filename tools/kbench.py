"""Per-kernel microbenchmarks at the cfg2 shapes (CUDA events, L2-cold weights).

    python tools/kbench.py [--json out.json]

Each line: kernel, shape, us/launch, algorithmic bytes, GB/s, fraction of the
measured HBM peak.  Weight-streaming kernels rotate over several copies so
every launch reads its weights from HBM, as in the real forward (each layer
has its own weights).
"""
import argparse
import ctypes
import json
import math
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18016_b200 import native, ops  # noqa: E402
from paper_2603_18016_b200.verify_bench import algorithmic_bytes, make_inputs  # noqa: E402

try:
    PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
except OSError:
    PEAK = 6461.2
dev = torch.device("cuda:0")
lib = native.load()
bf = torch.bfloat16
rows = []


def timeit(fn, iters=40):
    """Device time per call: the calls are captured in a CUDA graph so the
    host's launch rate does not pace the GPU (as in the real forward)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def report(name, shape, us, nbytes, flops=0):
    gbs = nbytes / (us * 1e-6) / 1e9
    r = {"kernel": name, "shape": shape, "us": round(us, 2), "bytes": nbytes,
         "GBps": round(gbs, 1), "frac_hbm": round(gbs / PEAK, 3)}
    if flops:
        r["TFLOPs"] = round(flops / (us * 1e-6) / 1e12, 1)
    rows.append(r)
    print(f"{name:28s} {shape:34s} {us:9.2f} us {gbs:8.0f} GB/s {100 * gbs / PEAK:5.1f}%"
          + (f" {r['TFLOPs']:7.1f} TF/s" if flops else ""), flush=True)


def gemm_case(tag, M, N, K, epi, copies=6, legacy=False, tiled=False, splits=None):
    x = torch.randn(M, K, device=dev).to(bf)
    if tiled and not hasattr(lib, "psd_tile_weights"):
        print(f"{tag}: pre-tiled GEMM not built (PSD_EXPERIMENTAL=1)")
        return
    ws = [(torch.randn(N, K, device=dev) * 0.02).to(bf) for _ in range(copies)]
    if tiled:
        tws = []
        for w in ws:
            t = torch.empty(lib.psd_tiled_weight_bytes(N, K) // 2, dtype=bf, device=dev)
            assert lib.psd_tile_weights(w.data_ptr(), N, K, K, t.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream) == 0
            tws.append(t)
        e = {"bf16": native.EPI_BF16, "silu": native.EPI_SILU, "f32": native.EPI_F32}[epi]
        n_out = N // 2 if epi == "silu" else N
        out = torch.empty(M, n_out, dtype=torch.float32 if epi == "f32" else bf, device=dev)
        wsp = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
        it = [0]

        def fn():
            st = torch.cuda.current_stream().cuda_stream
            rc = lib.psd_gemm_tiled(x.data_ptr(), K, M, K, tws[it[0] % copies].data_ptr(), N,
                                    out.data_ptr(), n_out, e, None, 0, wsp.data_ptr(),
                                    wsp.numel(), st)
            assert rc == 0
            it[0] += 1
        us = timeit(fn)
        nbytes = N * K * 2 + M * K * 2 + out.numel() * out.element_size()
        report(f"gemm {tag} tiled", f"M={M} N={N} K={K}", us, nbytes, 2 * M * N * K)
        return
    if epi == "partial":
        part = torch.empty(16 * M * N, dtype=torch.float32, device=dev)
        sp = ctypes.c_int()
        it = [0]
        hint = splits or 0

        def fn():
            st = torch.cuda.current_stream().cuda_stream
            w = ws[it[0] % copies]
            it[0] += 1
            rc = lib.psd_gemm_partials(x.data_ptr(), K, M, K, w.data_ptr(), K, N, part.data_ptr(),
                                       part.numel() * 4, hint, ctypes.byref(sp), st)
            assert rc == 0
        us = timeit(fn)
        out_bytes = sp.value * M * N * 4
        tag = f"{tag} (S={sp.value})"
    else:
        e = {"bf16": native.EPI_BF16, "silu": native.EPI_SILU, "f32": native.EPI_F32}[epi]
        n_out = N // 2 if epi == "silu" else N
        out = torch.empty(M, n_out, dtype=torch.float32 if epi == "f32" else bf, device=dev)
        wsp = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
        it = [0]

        sp_arg = splits if splits is not None else (-1 if legacy else 0)

        def fn():
            ops.gemm(x, ws[it[0] % copies], out=out, epi=e, workspace=wsp, splits=sp_arg)
            it[0] += 1
        us = timeit(fn)
        out_bytes = out.numel() * out.element_size()
    nbytes = N * K * 2 + M * K * 2 + out_bytes
    report(f"gemm {tag}", f"M={M} N={N} K={K}", us, nbytes, 2 * M * N * K)


def attn_case(tag, nseq, ql, ctx, Hq, Hkv, D):
    bs = 16
    nblk_seq = (ctx + ql + bs) // bs + 1
    nb = nseq * nblk_seq + 1
    kc = torch.randn(nb * bs, Hkv, D, device=dev).to(bf)
    vc = torch.randn(nb * bs, Hkv, D, device=dev).to(bf)
    bt = torch.arange(1, 1 + nseq * nblk_seq, dtype=torch.int32, device=dev).view(nseq, nblk_seq)
    q = torch.randn(nseq * ql, Hq, D, device=dev).to(bf)
    out = torch.empty_like(q)
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
    seq_slot = i32(list(range(nseq)))
    q_start = i32([i * ql for i in range(nseq)])
    q_len = i32([ql] * nseq)
    q_pos0 = i32([ctx] * nseq)
    kv_len = i32([ctx + ql] * nseq)
    aws = torch.zeros(lib.psd_attention_workspace_bytes(nseq, Hkv, ql, Hq, D, 400) + 16384,
                      dtype=torch.uint8, device=dev)
    kvh = [0]

    def fn():
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.psd_attention(q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(),
                               nblk_seq, seq_slot.data_ptr(), q_start.data_ptr(), q_len.data_ptr(),
                               q_pos0.data_ptr(), kv_len.data_ptr(), nseq, ql, Hq, Hkv, D, bs,
                               1 / math.sqrt(D), out.data_ptr(), kvh[0], aws.data_ptr(),
                               aws.numel(), st)
        assert rc == 0
    us = timeit(fn)
    report(f"attention {tag} nosplit", f"seqs={nseq} q={ql} ctx={ctx} D={D}", us,
           nseq * (ctx + ql) * Hkv * D * 2 * 2 + q.numel() * 2 * 2)
    kvh[0] = 400
    us = timeit(fn)
    nbytes = nseq * (ctx + ql) * Hkv * D * 2 * 2 + q.numel() * 2 * 2
    report(f"attention {tag}", f"seqs={nseq} q={ql} ctx={ctx} D={D}", us, nbytes)


def attn_rope_case(tag, nseq, ql, ctx, Hq, Hkv, D, S):
    """Decode attention with RoPE + KV write fused (psd_attention_rope), fed by
    S fp32 split-K partials of the QKV projection, as in the draft loop."""
    bs = 16
    nblk_seq = (ctx + ql + bs) // bs + 1
    nb = nseq * nblk_seq + 1
    kc = torch.randn(nb * bs, Hkv, D, device=dev).to(bf)
    vc = torch.randn(nb * bs, Hkv, D, device=dev).to(bf)
    bt = torch.arange(1, 1 + nseq * nblk_seq, dtype=torch.int32, device=dev).view(nseq, nblk_seq)
    M = nseq * ql
    nqkv = (Hq + 2 * Hkv) * D
    part = torch.randn(S * M * nqkv, device=dev) * 0.1
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
    positions = i32([ctx + t for _ in range(nseq) for t in range(ql)])
    slots = i32([int(bt[s_, (ctx + t) // bs]) * bs + (ctx + t) % bs
                 for s_ in range(nseq) for t in range(ql)])
    inv_freq = (10000.0 ** (-torch.arange(0, D, 2, device=dev).float() / D)).contiguous()
    out = torch.empty(M, Hq, D, device=dev).to(bf)
    seq_slot = i32(list(range(nseq)))
    q_start = i32([i * ql for i in range(nseq)])
    q_len = i32([ql] * nseq)
    q_pos0 = i32([ctx] * nseq)
    kv_len = i32([ctx + ql] * nseq)

    def fn():
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.psd_attention_rope(part.data_ptr(), S, M * nqkv, positions.data_ptr(),
                                    slots.data_ptr(), inv_freq.data_ptr(), None, kc.data_ptr(),
                                    vc.data_ptr(), bt.data_ptr(), nblk_seq, seq_slot.data_ptr(),
                                    q_start.data_ptr(), q_len.data_ptr(), q_pos0.data_ptr(),
                                    kv_len.data_ptr(), nseq, ql, Hq, Hkv, D, bs,
                                    1 / math.sqrt(D), out.data_ptr(), st)
        assert rc == 0
    us = timeit(fn)
    report(f"attention+rope {tag}", f"seqs={nseq} q={ql} ctx={ctx} D={D} S={S}", us,
           nseq * (ctx + ql) * Hkv * D * 2 * 2 + S * M * nqkv * 4)


def norm_case(tag, M, H, S):
    x = torch.randn(M, H, device=dev).to(bf)
    P = torch.randn(S * M * H, device=dev)
    w = torch.ones(H, device=dev).to(bf)
    y = torch.empty_like(x)
    def fn():
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.psd_add_rmsnorm(x.data_ptr(), H, P.data_ptr(), S, M * H, H, None, w.data_ptr(),
                                 y.data_ptr(), H, M, H, 1e-5, 1, st)
        assert rc == 0
    us = timeit(fn)
    report(f"add_rmsnorm {tag}", f"M={M} H={H} S={S}", us, M * H * (2 + 2 + 2 + 4 * S))


def rope_case(tag, M, Hq, Hkv, D, S):
    N = (Hq + 2 * Hkv) * D
    P = torch.randn(S * M * N, device=dev)
    q = torch.empty(M, Hq, D, dtype=bf, device=dev)
    kc = torch.empty(M + 16, Hkv, D, dtype=bf, device=dev)
    vc = torch.empty_like(kc)
    pos = torch.arange(M, dtype=torch.int32, device=dev) + 100
    slots = torch.arange(M, dtype=torch.int32, device=dev)
    inv = torch.rand(D // 2, device=dev) * 0.5
    def fn():
        st = torch.cuda.current_stream().cuda_stream
        rc = lib.psd_rope_kv_partials(P.data_ptr(), S, M * N, M, Hq, Hkv, D, pos.data_ptr(),
                             slots.data_ptr(), inv.data_ptr(), None, q.data_ptr(), kc.data_ptr(),
                             vc.data_ptr(), st)
        assert rc == 0
    us = timeit(fn)
    report(f"rope_kv {tag}", f"M={M} S={S}", us, M * N * 4 * S + M * N * 2)


def verify_case(tag, B, K, V, sampling, cached=False):
    sets = [make_inputs(B, K, V, sampling, dev, seed=i) for i in range(3)]
    stats = []
    if cached:  # the draft sampler's (max, sum) of every q row (psd_verify_sample_ext)
        for t, d, ids, ln, u in sets:
            st = torch.empty(B, K, 2, device=dev)
            rows = d.reshape(B * K, 1, -1)
            ops.verify_sample(rows, rows[:, :0], torch.zeros(B * K, 0, dtype=torch.int32,
                                                             device=dev),
                              torch.zeros(B * K, dtype=torch.int32, device=dev),
                              torch.rand(B * K, 1, device=dev), t_stats_out=st.view(B * K, 2),
                              t_stats_rows=torch.arange(B * K, dtype=torch.int32, device=dev))
            stats.append(st)
    it = [0]

    def fn():
        t, d, ids, ln, u = sets[it[0] % 3]
        if sampling:
            ops.verify_sample(t, d, ids, ln, u, d_stats=stats[it[0] % 3] if cached else None)
        else:
            ops.verify_greedy(t, ids, ln)
        it[0] += 1
    us = timeit(fn)
    report(f"K1 {tag}", f"B={B} k={K} V={V}", us, algorithmic_bytes(B, K, V, sampling))


def lm_argmax_case(tag, M, N, K, copies=2):
    """K6: the draft's greedy LM head + sampler, fused (argmax epilogue + fold)
    vs stored logits + bigram bias + K1 (k = 0)"""
    x = torch.randn(M, K, device=dev).to(bf)
    ws = [(torch.randn(N, K, device=dev) * 0.02).to(bf) for _ in range(copies)]
    wsp = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    logits = torch.empty(M, N, device=dev)
    tok = torch.randint(0, N, (M,), dtype=torch.int32, device=dev)
    succ = torch.randint(0, N, (N,), dtype=torch.int32, device=dev)
    part = torch.empty(lib.psd_argmax_partials_bytes(M, N), dtype=torch.uint8, device=dev)
    out = torch.empty(M, dtype=torch.int32, device=dev)
    ids0 = torch.zeros(M, 0, dtype=torch.int32, device=dev)
    len0 = torch.zeros(M, dtype=torch.int32, device=dev)
    acc = torch.empty(M, dtype=torch.int32, device=dev)
    o1 = torch.empty(M, 1, dtype=torch.int32, device=dev)
    it = [0]

    def fused():
        st = torch.cuda.current_stream().cuda_stream
        w = ws[it[0] % copies]
        it[0] += 1
        assert lib.psd_gemm_argmax(x.data_ptr(), K, M, K, w.data_ptr(), K, N, tok.data_ptr(), None,
                                   succ.data_ptr(), 16.0, part.data_ptr(), wsp.data_ptr(),
                                   wsp.numel(), st) == 0
        assert lib.psd_argmax_fold(part.data_ptr(), M, N, out.data_ptr(), None, None, st) == 0

    def unfused():
        st = torch.cuda.current_stream().cuda_stream
        w = ws[it[0] % copies]
        it[0] += 1
        assert lib.psd_gemm_bf16(x.data_ptr(), K, M, K, w.data_ptr(), K, N, logits.data_ptr(), N,
                                 native.EPI_F32, None, 0, 0, wsp.data_ptr(), wsp.numel(), st) == 0
        assert lib.psd_bigram_bias(logits.data_ptr(), N, tok.data_ptr(), M, succ.data_ptr(), N,
                                   16.0, st) == 0
        ops.verify_greedy(logits.view(M, 1, N), ids0, len0, acc, o1)
    nbytes = N * K * 2 + M * K * 2
    report(f"lm head+argmax {tag} fused", f"M={M} N={N} K={K}", timeit(fused), nbytes)
    report(f"lm head+argmax {tag} unfused", f"M={M} N={N} K={K}", timeit(unfused), nbytes)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    sel = a.only.split(",") if a.only else None

    def want(k):
        return sel is None or k in sel
    if want("gemmx"):
        gemm_case("8B gu as f32", 192, 28672, 4096, "f32")
        gemm_case("8B gu as bf16", 192, 28672, 4096, "bf16")
        gemm_case("8B gu silu", 192, 28672, 4096, "silu")
        gemm_case("8B N57344 bf16", 192, 57344, 4096, "bf16", copies=3)
        gemm_case("8B N114688 bf16", 192, 114688, 4096, "bf16", copies=2)
        gemm_case("1B gu as f32", 32, 16384, 2048, "f32")
        gemm_case("1B gu silu", 32, 16384, 2048, "silu")
        gemm_case("1B N65536 f32", 32, 65536, 2048, "f32", copies=3)
        gemm_case("M128 gu bf16", 128, 28672, 4096, "bf16")
        gemm_case("M64 gu bf16", 64, 28672, 4096, "bf16")
        gemm_case("M256 gu bf16", 256, 28672, 4096, "bf16")
    if want("gemm"):
        # 8B verify (M = 32 x 6)
        gemm_case("8B qkv", 192, 6144, 4096, "bf16")
        gemm_case("8B o", 192, 4096, 4096, "bf16")
        gemm_case("8B gate/up", 192, 28672, 4096, "silu")
        gemm_case("8B down", 192, 4096, 14336, "bf16")
        gemm_case("8B gate/up legacy", 192, 28672, 4096, "silu", legacy=True)
        gemm_case("8B qkv", 192, 6144, 4096, "bf16", tiled=True)
        gemm_case("8B o", 192, 4096, 4096, "bf16", tiled=True)
        gemm_case("8B gate/up", 192, 28672, 4096, "silu", tiled=True)
        gemm_case("8B down", 192, 4096, 14336, "bf16", tiled=True)
        gemm_case("8B lm_head", 192, 128256, 4096, "f32", copies=2, tiled=True)
        gemm_case("8B lm_head", 192, 128256, 4096, "f32", copies=2)
        # 1B draft (M = 32, first step 64)
        gemm_case("1B qkv", 32, 3072, 2048, "bf16")
        gemm_case("1B o", 32, 2048, 2048, "bf16")
        gemm_case("1B gate/up", 32, 16384, 2048, "silu")
        gemm_case("1B down", 32, 2048, 8192, "bf16")
        gemm_case("1B down legacy", 32, 2048, 8192, "bf16", legacy=True)
        gemm_case("1B qkv", 32, 3072, 2048, "bf16", tiled=True)
        gemm_case("1B o", 32, 2048, 2048, "bf16", tiled=True)
        gemm_case("1B gate/up", 32, 16384, 2048, "silu", tiled=True)
        gemm_case("1B down", 32, 2048, 8192, "bf16", tiled=True)
        gemm_case("1B lm_head", 32, 128256, 2048, "f32", copies=2, tiled=True)
        gemm_case("1B lm_head", 32, 128256, 2048, "f32", copies=2)
        gemm_case("1B gate/up M64", 64, 16384, 2048, "silu")
        # the split-K partial GEMMs the forward uses for QKV / O / down
        gemm_case("8B qkv part", 192, 6144, 4096, "partial")
        gemm_case("8B o part", 192, 4096, 4096, "partial")
        gemm_case("8B down part", 192, 4096, 14336, "partial")
        gemm_case("1B qkv part", 32, 3072, 2048, "partial")
        gemm_case("1B o part", 32, 2048, 2048, "partial")
        gemm_case("1B down part", 32, 2048, 8192, "partial")
    if want("gemm1b"):
        gemm_case("1B qkv part", 32, 3072, 2048, "partial")
        gemm_case("1B gate/up", 32, 16384, 2048, "silu")
    if want("gemmpf"):
        gemm_case("8B gate/up", 192, 28672, 4096, "silu")
        gemm_case("8B lm_head", 192, 128256, 4096, "f32", copies=2)
        gemm_case("8B qkv part", 192, 6144, 4096, "partial")
        gemm_case("8B o part", 192, 4096, 4096, "partial")
        gemm_case("8B down part", 192, 4096, 14336, "partial")
        gemm_case("1B gate/up", 32, 16384, 2048, "silu")
        gemm_case("1B down part", 32, 2048, 8192, "partial")
        gemm_case("1B lm_head", 32, 128256, 2048, "f32", copies=2)
    if want("gemmsp"):
        for sp in (None, 1, 2):
            gemm_case(f"1B gate/up sp{sp}", 32, 16384, 2048, "silu", splits=sp)
            gemm_case(f"1B gate/up M64 sp{sp}", 64, 16384, 2048, "silu", splits=sp)
            gemm_case(f"8B gate/up sp{sp}", 192, 28672, 4096, "silu", splits=sp)
            gemm_case(f"1B lm sp{sp}", 32, 128256, 2048, "f32", copies=2, splits=sp)
    if want("gemmpart"):
        for (tag, M, N, K) in (("1B qkv", 32, 3072, 2048), ("1B o", 32, 2048, 2048),
                               ("1B down", 32, 2048, 8192), ("8B qkv", 192, 6144, 4096),
                               ("8B o", 192, 4096, 4096), ("8B down", 192, 4096, 14336)):
            for sp in ((None,) if os.environ.get("KB_AUTO_ONLY") else (None, 2, 3, 4, 6, 8, 12, 16)):
                gemm_case(f"{tag} part", M, N, K, "partial", splits=sp)
    if want("gemmnt"):
        gemm_case("8B gate/up M384", 384, 28672, 4096, "silu")
        gemm_case("8B qkv part M384", 384, 6144, 4096, "partial")
        gemm_case("8B down part M384", 384, 4096, 14336, "partial")
        gemm_case("8B lm M384", 384, 128256, 4096, "f32", copies=2)
        gemm_case("70B gate/up M320", 320, 57344, 8192, "silu", copies=2)
        gemm_case("70B down part M320", 320, 8192, 28672, "partial", copies=2)
    if want("gemmmw"):
        gemm_case("8B gate/up", 192, 28672, 4096, "silu")
        gemm_case("8B lm", 192, 128256, 4096, "f32", copies=2)
        gemm_case("8B gate/up M96", 96, 28672, 4096, "silu")
        gemm_case("8B gate/up M256", 256, 28672, 4096, "silu")
        gemm_case("Qwen7B gate/up M160", 160, 37888, 3584, "silu")
    if want("gemmskp"):
        # the split-K shapes through stream-K with an fp32 output (one slice)
        for (tag, M, N, K) in (("8B qkv", 192, 6144, 4096), ("8B o", 192, 4096, 4096),
                               ("8B down", 192, 4096, 14336), ("1B qkv", 32, 3072, 2048),
                               ("1B o", 32, 2048, 2048), ("1B down", 32, 2048, 8192)):
            gemm_case(f"{tag} part", M, N, K, "partial")
            gemm_case(f"{tag} sk f32", M, N, K, "f32", splits=0)
    if want("gemmgu"):
        gemm_case("8B gate/up", 192, 28672, 4096, "silu")
    if want("gemmguM"):
        # gate/up vs M: B (token) traffic through L2 grows with M, weights do not
        for mm in (32, 64, 96, 128, 160, 192, 256):
            gemm_case(f"8B gate/up M{mm}", mm, 28672, 4096, "silu")
    if want("attnrope"):
        attn_rope_case("1B draft", 32, 1, 300, 32, 8, 64, 6)
        attn_rope_case("1B draft step0", 32, 2, 300, 32, 8, 64, 6)
    if want("attn1b"):
        attn_case("1B draft", 32, 1, 300, 32, 8, 64)
    if want("attn8b"):
        attn_case("8B verify", 32, 6, 300, 32, 8, 128)
    if want("attn"):
        attn_case("8B verify", 32, 6, 300, 32, 8, 128)
        attn_case("1B draft", 32, 1, 300, 32, 8, 64)
        attn_case("1B draft step0", 32, 2, 300, 32, 8, 64)
    if want("norm"):
        norm_case("8B", 192, 4096, 4)
        norm_case("1B", 32, 2048, 6)
        rope_case("8B", 192, 32, 8, 128, 3)
        rope_case("1B", 32, 32, 8, 64, 6)
    if want("lmargmax"):
        lm_argmax_case("1B", 32, 128256, 2048)
        lm_argmax_case("1B M64", 64, 128256, 2048)
        lm_argmax_case("8B verify M192", 192, 128256, 4096)
        lm_argmax_case("8B SD(2m) M384", 384, 128256, 4096)
    if want("k1"):
        verify_case("greedy cfg2", 32, 5, 128256, False)
        verify_case("sample cfg2", 32, 5, 128256, True)
        verify_case("sample cfg2 cachedq", 32, 5, 128256, True, cached=True)
        verify_case("draft argmax", 32, 0, 128256, False)
    if a.json:
        json.dump({"peak_gbps": PEAK, "rows": rows}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
