"""Verification-kernel sweep (BASELINE config 5): achieved HBM GB/s of K1.

    python -m paper_2603_18016_b200.verify_bench [--quick] [--json]

Algorithmic bytes per launch:
  greedy   4 V sum_b(k_b+1) + 4 B k + 4 B (k+2)
  sampling 4 V sum_b(2 k_b+1) + 4 B (k+1) + 4 B k + 4 B (k+2)
Timing: K1 behind an L2 flush (a 256 MiB write), ten of each captured in a
CUDA graph; K1 time = (graph time - flush-only graph time) / 10, CUDA events,
median of several replays.
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


def time_verify(B, K, V, sampling, iters=30, device="cuda", flush=True, cached=False):
    """Median device time of one K1 launch (both kernels when sampling).

    Ten (L2 flush, K1) pairs are captured in one CUDA graph and ten flushes
    in another; K1's time is the difference of the two replays / 10 (median
    of several), so it excludes host launch latency and includes the
    in-graph launch gap, as in the PSD loop.  cached: the draft rows'
    (max, sum) come from the draft sampler (psd_verify_sample_ext), so K1
    streams the target rows only."""
    dev = torch.device(device)
    t, d, ids, ln, u = make_inputs(B, K, V, sampling, dev)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    stats = None
    if cached and sampling and K:
        stats = torch.empty(B, K, 2, device=dev)
        rows = d.reshape(B * K, 1, V)
        ops.verify_sample(rows, rows[:, :0], torch.zeros(B * K, 0, dtype=torch.int32,
                                                         device=dev),
                          torch.zeros(B * K, dtype=torch.int32, device=dev),
                          torch.rand(B * K, 1, device=dev), t_stats_out=stats.view(B * K, 2),
                          t_stats_rows=torch.arange(B * K, dtype=torch.int32, device=dev))

    def launch():
        if sampling:
            ops.verify_sample(t, d, ids, ln, u, d_stats=stats)
        else:
            ops.verify_greedy(t, ids, ln)

    # warm up on the capture stream: the workspace (keyed by stream) exists
    # before capture, so the graphs hold the kernels only
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for _ in range(3):
            launch()
    torch.cuda.synchronize()
    reps = 10

    def capture(with_k1):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
            for _ in range(reps):
                if flush:
                    scratch.fill_(1)
                if with_k1:
                    launch()
        return g

    g_k1, g_flush = capture(True), capture(False)

    def timed(g):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    times = []
    for _ in range(max(3, iters // reps)):
        times.append((timed(g_k1) - timed(g_flush)) / reps)
    ms = statistics.median(times)
    nbytes = algorithmic_bytes(B, K, V, sampling)
    r = {"B": B, "k": K, "V": V, "mode": "sampling" if sampling else "greedy",
         "us": ms * 1e3, "bytes": nbytes, "GBps": nbytes / (ms * 1e-3) / 1e9}
    if stats is not None:
        r["mode"] = "sampling_cached_q"
        r["bytes_streamed"] = algorithmic_bytes(B, K, V, False)
        r["GBps_streamed"] = r["bytes_streamed"] / (ms * 1e-3) / 1e9
    return r


# where the PSD loop runs K1 with the draft sampler's cached q statistics (cfg2,
# cfg3 shapes)
CACHED_POINTS = {(32, 5, 128256), (32, 4, 152064)}


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
        if K and (B, K, V) in CACHED_POINTS:
            out.append(time_verify(B, K, V, True, cached=True))
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
