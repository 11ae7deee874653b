"""Verification-kernel sweep (BASELINE config 5): achieved HBM GB/s of K1.

    python -m paper_2603_18016_b200.verify_bench [--quick] [--json]

Algorithmic bytes per launch:
  greedy   4 V sum_b(k_b+1) + 4 B k + 4 B (k+2)
  sampling 4 V sum_b(2 k_b+1) + 4 B (k+1) + 4 B k + 4 B (k+2)
Timing: CUDA events on the launching stream, median of N launches, L2 flushed
(a 256 MiB write) before every timed launch.
"""

from __future__ import annotations

import argparse
import json
import statistics

import torch

from . import ops

PEAK_FALLBACK = 6461.2


def algorithmic_bytes(B: int, K: int, V: int, sampling: bool, klen=None) -> int:
    ks = [K] * B if klen is None else list(klen)
    if sampling:
        return 4 * V * sum(2 * k + 1 for k in ks) + 4 * B * (K + 1) + 4 * B * K + 4 * B * (K + 2)
    return 4 * V * sum(k + 1 for k in ks) + 4 * B * K + 4 * B * (K + 2)


def make_inputs(B, K, V, sampling, device, seed=0):
    g = torch.Generator(device=device).manual_seed(seed)
    t = torch.randn(B, K + 1, V, device=device, generator=g) * 2.0
    d = (t[:, :K] + 0.5 * torch.randn(B, K, V, device=device, generator=g)).contiguous()
    ids = d.argmax(dim=2).to(torch.int32) if K else torch.zeros(B, 0, dtype=torch.int32,
                                                                 device=device)
    if sampling and K:
        q = torch.softmax(d, dim=2).reshape(B * K, V)
        ids = torch.multinomial(q, 1, generator=g).reshape(B, K).to(torch.int32)
    ln = torch.full((B,), K, dtype=torch.int32, device=device)
    u = torch.rand(B, K + 1, device=device, generator=g)
    return t, d, ids, ln, u


def time_verify(B, K, V, sampling, iters=30, device="cuda", flush=True):
    dev = torch.device(device)
    t, d, ids, ln, u = make_inputs(B, K, V, sampling, dev)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    def launch():
        if sampling:
            ops.verify_sample(t, d, ids, ln, u)
        else:
            ops.verify_greedy(t, ids, ln)

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush:
            scratch.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        launch()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    nbytes = algorithmic_bytes(B, K, V, sampling)
    return {"B": B, "k": K, "V": V, "mode": "sampling" if sampling else "greedy",
            "us": ms * 1e3, "bytes": nbytes, "GBps": nbytes / (ms * 1e-3) / 1e9}


def sweep(quick: bool):
    if quick:
        pts = [(32, 5, 128256), (64, 4, 128256), (32, 4, 152064), (512, 8, 262144),
               (1, 1, 32000), (8, 5, 128256), (128, 5, 128256)]
    else:
        pts = [(B, K, V) for V in (32000, 65536, 128256, 152064, 262144)
               for K in (1, 2, 4, 5, 8) for B in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512)
               if B * (2 * K + 1) * V * 4 <= 12 << 30]
    out = []
    for B, K, V in pts:
        for sampling in (False, True):
            out.append(time_verify(B, K, V, sampling))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    try:
        with open("MEASURED_PEAKS.json") as fh:
            peak = json.load(fh)["hbm_gbs"]
    except OSError:
        peak = PEAK_FALLBACK
    res = sweep(a.quick)
    for r in res:
        r["frac"] = r["GBps"] / peak
        print(f"{r['mode']:8s} B={r['B']:4d} k={r['k']} V={r['V']:6d}  {r['us']:9.1f} us  "
              f"{r['GBps']:7.0f} GB/s  {100 * r['frac']:5.1f}% of {peak}")
    if a.json:
        with open(a.json, "w") as fh:
            json.dump({"peak_gbps": peak, "points": res}, fh, indent=1)


if __name__ == "__main__":
    main()
