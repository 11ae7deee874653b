"""Per-CTA timeline of the stream-K GEMM (psd_gemm_set_trace, %globaltimer ns).

    python tools/sk_trace.py

For each shape: one isolated launch (synchronised before and after) and the
last launch of a graph of back-to-back launches over rotating weight copies.
Prints percentiles over CTAs of: entry skew, first operands ready after entry,
last MMA issued, last accumulator ready, epilogue done (all relative to the
earliest CTA entry), plus segments per CTA and fast (no-publish) finishes.
"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_18016_b200 import native, ops  # noqa: E402

if os.environ.get("PSD_LIB"):  # a variant build (experiments)
    native.LIB_PATH = os.path.abspath(os.environ["PSD_LIB"])
dev = torch.device("cuda:0")
lib = native.load()
bf = torch.bfloat16


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * (len(v) - 1) + 0.5))]


def summarize(tag, tr):
    rows = [r for r in tr.tolist() if r[0] != 0]
    t0 = min(r[0] for r in rows)
    cols = {"entry": [(r[0] - t0) / 1e3 for r in rows],
            "first_ops-entry": [(r[1] - r[0]) / 1e3 for r in rows],
            "mma_end": [(r[2] - t0) / 1e3 for r in rows],
            "last_acc": [(r[3] - t0) / 1e3 for r in rows],
            "epi_end": [(r[4] - t0) / 1e3 for r in rows],
            "epi_tail": [(r[4] - r[3]) / 1e3 for r in rows],
            "epi_pre_rounds": [(r[7] - r[3]) / 1e3 for r in rows]}
    for k in range(4):
        if all(r[8 + 2 * k] and r[9 + 2 * k] for r in rows):
            cols[f"round{k}"] = [(r[9 + 2 * k] - r[8 + 2 * k]) / 1e3 for r in rows]
            cols[f"gap_before_r{k}"] = [(r[8 + 2 * k] - (r[7] if k == 0 else r[7 + 2 * k])) / 1e3
                                        for r in rows]
    print(f"{tag}: {len(rows)} CTAs, span {max(cols['epi_end']):.2f} us, segments "
          f"{min(r[5] for r in rows)}-{max(r[5] for r in rows)}, fast finishes "
          f"{sum(r[6] for r in rows)}")
    for k, v in cols.items():
        print(f"   {k:16s} min {min(v):7.2f}  p10 {pct(v, .1):7.2f}  p50 {pct(v, .5):7.2f}  "
              f"p90 {pct(v, .9):7.2f}  max {max(v):7.2f}")


def case(tag, M, N, K, epi, copies=4):
    x = torch.randn(M, K, device=dev).to(bf)
    ws = [(torch.randn(N, K, device=dev) * 0.02).to(bf) for _ in range(copies)]
    n_out = N // 2 if epi == native.EPI_SILU else N
    out = torch.empty(M, n_out, dtype=torch.float32 if epi == native.EPI_F32 else bf, device=dev)
    wsp = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    tr = torch.zeros(1024, 16, dtype=torch.int64, device=dev)
    for i in range(4):
        ops.gemm(x, ws[i % copies], out=out, epi=epi, workspace=wsp)
    torch.cuda.synchronize()
    lib.psd_gemm_set_trace(tr.data_ptr())
    ops.gemm(x, ws[0], out=out, epi=epi, workspace=wsp)
    torch.cuda.synchronize()
    summarize(f"{tag} isolated", tr.cpu())
    tr.zero_()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for i in range(8):
            ops.gemm(x, ws[i % copies], out=out, epi=epi, workspace=wsp)
    lib.psd_gemm_set_trace(None)
    g.replay()
    torch.cuda.synchronize()
    tr.zero_()
    g.replay()
    torch.cuda.synchronize()
    summarize(f"{tag} graph (last of 8)", tr.cpu())


case("8B gate/up silu", 192, 28672, 4096, native.EPI_SILU)
case("8B lm_head f32", 192, 128256, 4096, native.EPI_F32, copies=2)
case("1B lm_head f32", 32, 128256, 2048, native.EPI_F32, copies=2)
case("8B gate/up bf16", 192, 28672, 4096, native.EPI_BF16)
case("8B gate/up M128 bf16", 128, 28672, 4096, native.EPI_BF16)
