#!/usr/bin/env python
"""PSD output tokens/s vs sequential SD on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Workload (BASELINE config 2): Llama-3.2-1B draft / Llama-3.1-8B target shapes,
random-init bf16 weights (no checkpoints offline), synthetic prompts, two
batches of 32 requests (m=32), k=5, prompt 128, output 256, greedy, one GPU
per replica with draft and verify on separate CUDA streams.  One bench *step*
is one complete pass of the hot path over the workload: all 64 requests from
admission to their last token through the public API ``run(config,
workload, backend=GpuBackend)``.

Multi-GPU: one process per GPU, each an independent PSD replica on its own
64 requests (requests shard with no data-path collective) -> "scaling":
"weak"; time is the max over ranks.

Keys beyond the base contract: ``sd`` (same workload, mode standard-sd with
sd_batch_factor 2 = one batch of 64), ``psd_vs_sd``, ``mean_accepted_len``,
``draft_hidden_frac``, ``verify_kernel`` (K1 at the workload shape),
``roofline`` (dominant kernel: the verify gate/up GEMM), ``cpu_baseline``
(CPU oracle PSD on a bounded sample, rank 0, N=1).
``--impl reference`` times the CPU oracle (the reference has no CPU
implementation of token-level PSD; oracle/ is its restatement) on the same
workload shapes, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(target="llama-3.1-8b", draft="llama-3.2-1b", m=32, n_requests=64, k=5,
           prompt=128, output=256)
# BASELINE config 4 (--layout tp): Llama-3.1-70B target tensor-parallel over all
# ranks, Llama-3.2-1B draft replicated on each, 2 x 64 requests, k = 4
CFG4 = dict(target="llama-3.1-70b", draft="llama-3.2-1b", m=64, n_requests=128, k=4,
            prompt=128, output=256)
# the 70B's random logits spread ~sqrt(8192 / 4096) wider than the 8B's, so its
# synthetic-language bias scales with it (same acceptance regime as cfg2)
BETA_TARGET_CFG4 = 10.0
# BASELINE config 3 (--workload cfg3): Qwen2.5-7B target / Qwen2.5-0.5B draft,
# temperature-1.0 rejection sampling over the 152k vocabulary (V_draft 151936 <
# V_target 152064), 2 x 32 requests, k = 4; both models on one GPU here
CFG3 = dict(target="qwen2.5-7b", draft="qwen2.5-0.5b", m=32, n_requests=64, k=4,
            prompt=128, output=256)
BETAS_CFG3 = (14.0, 14.0)  # sampling at T = 1: bias e^14 dominates 152k near-uniform logits
BETA_TARGET = 7.0
BETA_DRAFT = 16.0
METRIC = "PSD output tok/s vs sequential SD, mean accepted len; verify-kernel HBM GB/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p.get("bf16_tflops", 1682.3), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _workload(seed: int):
    from paper_2603_18016_b200 import make_requests
    return make_requests([CFG["output"]] * CFG["n_requests"], prompt_len=CFG["prompt"])


def _config(mode: str):
    """psd | standard-sd (one batch of 2m = all 64) | sd-m (batches of m = 32)."""
    from paper_2603_18016_b200 import SimConfig
    if mode == "sd-m":
        return SimConfig(mode="standard-sd", m=CFG["m"], k=CFG["k"], sd_batch_factor=1)
    return SimConfig(mode=mode, m=CFG["m"], k=CFG["k"],
                     sd_batch_factor=2 if mode == "standard-sd" else 1)


def _time_graph(fn, n: int = 32, replays: int = 5) -> float:
    """Average device time (ms) of fn() captured n times back to back in one
    CUDA graph (as the PSD loop launches its kernels), median over replays."""
    import statistics as stt
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(replays):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / n)
    return stt.median(times)


TRAFFIC_FILE = os.path.join("profiles", "r02_ncu_traffic.json")


def _ncu_traffic(key: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of the
    roofline kernel, from this round's ncu --set full capture of the same
    kernel at the same shape (TRAFFIC_FILE, written by tools/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, TRAFFIC_FILE)) as fh:
            t = json.load(fh)[key]
        return t["dram_read"] + t["dram_write"]
    except (OSError, KeyError, ValueError):
        return None


def _sk_physical(dev, cap: int) -> int:
    """CTAs a stream-K GEMM runs on under a CTA cap (gemm.cu sk_physical): the
    work is split over one virtual CTA per SM whatever the cap, and each
    physical CTA takes the same number of virtual ones."""
    import torch
    G = torch.cuda.get_device_properties(dev).multi_processor_count
    if cap <= 0 or cap >= G:
        return G
    per = -(-G // cap)
    return -(-G // per)


def kernel_rooflines(backend, hbm_peak: float, bf16_peak: float) -> tuple[dict, dict]:
    """Dominant kernel (verify-forward gate/up GEMM) and K1 at the workload shapes."""
    import torch
    from paper_2603_18016_b200 import native, ops
    from paper_2603_18016_b200.verify_bench import time_verify
    dev = backend.device
    s = backend.tshape
    M = CFG["m"] * (CFG["k"] + 1)
    w = backend.target.layers[0]["wgu"]
    x = torch.randn(M, s.hidden, device=dev).to(torch.bfloat16)
    out = torch.empty(M, w.shape[0] // 2, dtype=torch.bfloat16, device=dev)  # SiLU: N / 2 (a TP shard under --tp)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    # rotate over all layers' weights so every launch streams from HBM
    ws_list = [L["wgu"] for L in backend.target.layers]
    it = [0]

    def gemm():
        ops.gemm(x, ws_list[it[0] % len(ws_list)], out=out, epi=native.EPI_SILU, workspace=ws)
        it[0] += 1

    lib = native.load()
    ms = _time_graph(gemm, 64)
    # the same GEMM under the CTA cap it runs with inside an overlapped PSD step
    # (the draft's kernels take the other SMs there); timed alone here
    cap = backend.verify_ctas
    ms_cap = None
    if cap:
        lib.psd_gemm_set_max_ctas(cap)
        try:
            ms_cap = _time_graph(gemm, 64)
        finally:
            lib.psd_gemm_set_max_ctas(0)
    N, Kd = w.shape[0], s.hidden
    nbytes = w.numel() * 2 + x.numel() * 2 + out.numel() * 2
    flops = 2 * M * N * Kd
    # roofline class from arithmetic intensity vs the ridge point of the
    # measured peaks (M = 192 is below the ridge, M = 320 above)
    intensity = flops / nbytes
    ridge = bf16_peak * 1e12 / (hbm_peak * 1e9)
    bound = "tensor" if intensity >= ridge else "hbm"
    if bound == "hbm":
        achieved, peak, unit = nbytes / (ms * 1e-3) / 1e9, hbm_peak, "GB/s"
    else:
        achieved, peak, unit = flops / (ms * 1e-3) / 1e12, bf16_peak, "TFLOP/s"
    roof = {"kernel": f"gemm_sk_kernel<SILU> (verify gate/up, M={M} N={N} K={Kd})",
            "bound": bound, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
            "frac": round(achieved / peak, 4),
            "traffic": _ncu_traffic(f"gate_up_M{M}_N{N}_K{Kd}"),
            "traffic_source": TRAFFIC_FILE,
            "intensity_flop_per_byte": round(intensity, 1), "ridge_flop_per_byte": round(ridge, 1),
            "bytes_per_launch": nbytes, "us_per_launch": round(ms * 1e3, 2),
            "tflops": round(flops / (ms * 1e-3) / 1e12, 1),
            "timing": "alone, all SMs, 64 launches back to back in a CUDA graph rotating over "
                      "every layer's weights (inputs > L2)",
            "psd_step_config": ({"cta_cap": cap, "ctas": _sk_physical(dev, cap),
                                 "us_per_launch": round(ms_cap * 1e3, 2),
                                 "GBps": round(nbytes / (ms_cap * 1e-3) / 1e9, 1),
                                 "frac": round(nbytes / (ms_cap * 1e-3) / 1e9 / hbm_peak, 4),
                                 "note": "CTA cap of the verify GEMMs in overlapped PSD steps, "
                                         "timed alone (beside the draft the SMs are shared)"}
                                if ms_cap else None)}
    # K1 as the PSD loop runs it: inside CUDA graphs, behind an L2 flush
    # (verify_bench.time_verify: graph of (flush, K1) pairs minus a graph of
    # flushes), so the number is the kernels' device time, not host launch rate
    B, K, V = CFG["m"], CFG["k"], s.vocab
    rg = time_verify(B, K, V, False, iters=60, device=dev)
    rs = time_verify(B, K, V, True, iters=30, device=dev)
    # the PSD loop's sampling K1: q-row statistics cached by the draft sampler
    # (psd_verify_sample_ext), so the draft rows are not streamed again
    rc = time_verify(B, K, V, True, iters=30, device=dev, cached=True)
    vb, vbs = rg["bytes"], rs["bytes"]
    read_c = rc["bytes_streamed"]
    ms1, ms2, ms3 = rg["us"] * 1e-3, rs["us"] * 1e-3, rc["us"] * 1e-3
    timing = "CUDA graph, L2 flushed before every launch (verify_bench.time_verify)"
    vk = {"greedy": {"B": B, "k": K, "V": V, "us": round(ms1 * 1e3, 2), "bytes": vb,
                     "GBps": round(vb / (ms1 * 1e-3) / 1e9, 1),
                     "frac": round(vb / (ms1 * 1e-3) / 1e9 / hbm_peak, 4), "timing": timing},
          "sampling": {"B": B, "k": K, "V": V, "us": round(ms2 * 1e3, 2), "bytes": vbs,
                       "GBps": round(vbs / (ms2 * 1e-3) / 1e9, 1),
                       "frac": round(vbs / (ms2 * 1e-3) / 1e9 / hbm_peak, 4), "timing": timing},
          "sampling_cached_q": {
              "B": B, "k": K, "V": V, "us": round(ms3 * 1e3, 2),
              "note": "q-row (max, sum) cached by the draft sampler; streams the k+1 target "
                      "rows only",
              "algorithmic_bytes": vbs,
              "GBps_algorithmic": round(vbs / (ms3 * 1e-3) / 1e9, 1),
              "bytes_streamed": read_c,
              "GBps_streamed": round(read_c / (ms3 * 1e-3) / 1e9, 1),
              "frac_streamed": round(read_c / (ms3 * 1e-3) / 1e9 / hbm_peak, 4),
              "timing": timing}}
    return roof, vk


def verify_sweep_summary(hbm_peak: float) -> dict:
    """K1 over a grid of BASELINE config 5 (batch x k x vocab, greedy and
    sampling; verify_bench.time_verify: L2 flushed, inside CUDA graphs):
    min / median fraction of the HBM peak.  The full 500-point sweep is
    profiles/r02_verify_sweep.txt."""
    import statistics as stt
    from paper_2603_18016_b200.verify_bench import time_verify
    pts = [(B, K, V) for B in (8, 64, 512) for K in (1, 4, 8) for V in (32000, 262144)]
    rows = {"greedy": [], "sampling": []}
    for B, K, V in pts:
        for sampling in (False, True):
            r = time_verify(B, K, V, sampling, iters=20)
            rows[r["mode"]].append((B, K, V, round(r["GBps"] / hbm_peak, 4)))
    out = {"grid": "B {8, 64, 512} x k {1, 4, 8} x V {32000, 262144}", "peak_GBps": hbm_peak}
    for mode, rs in rows.items():
        fr = [x[3] for x in rs]
        out[mode] = {"min_frac": min(fr), "median_frac": round(stt.median(fr), 4),
                     "max_frac": max(fr), "points": rs}
    return out


def draft_hiding(states) -> dict:
    """Exposed drafting: per overlapped PSD step, exposed =
    max(0, t_step - t_prefill - t_verify); hidden fraction = 1 - sum(exposed) /
    sum(t_draft).  Durations are CUDA-event ms from GpuBackend.execute."""
    exposed = drafted = step = 0.0
    n = 0
    for state in states:
        for rec in state.step_log:
            if rec.fallback or rec.target_batch is None or rec.draft_duration <= 0.0:
                continue
            e = max(0.0, rec.step_duration - rec.prefill_duration - rec.verify_duration)
            exposed += e
            drafted += rec.draft_duration
            step += rec.step_duration
            n += 1
    if n == 0 or drafted <= 0.0:
        return {"draft_hidden_frac": None, "exposed_draft_frac_of_step": None, "steps": 0}
    return {"draft_hidden_frac": round(1.0 - exposed / drafted, 4),
            "exposed_draft_frac_of_step": round(exposed / step, 4), "steps": n}


def cpu_sample(steps: int = 1, n_req: int = 2, out_len: int = 6):
    """The CPU oracle PSD (numpy + C verify) on a bounded sample of the
    workload: same model shapes, k, prompt length; n_req requests of out_len
    tokens.  Returns (tok/s, seconds, tokens, cores)."""
    import numpy as np  # noqa: F401
    from oracle.psd_cpu import CpuBackend
    from paper_2603_18016_b200 import SimConfig, make_requests, run
    be = CpuBackend(CFG["target"], CFG["draft"], seed=0, beta_target=BETA_TARGET,
                    beta_draft=BETA_DRAFT, max_seq_len=CFG["prompt"] + out_len + 16)
    cfg = SimConfig(mode="psd", m=max(1, n_req // 2), k=CFG["k"])
    total_tok, total_s = 0, 0.0
    for _ in range(steps):
        reqs = make_requests([out_len] * n_req, prompt_len=CFG["prompt"])
        t0 = time.perf_counter()
        st, rep = run(cfg, reqs, backend=be)
        total_s += time.perf_counter() - t0
        total_tok += rep.total_generated
    return total_tok / total_s, total_s, total_tok, os.cpu_count()


def cpu_plan_baselines(vocab: int) -> dict:
    """BASELINE.md §2, timed on this host: (1) the reference's scheduler
    algorithm (the byte-identical port with the reference's latency / coin-flip
    models, SimBackend; one Python thread) on the workload's PSD and SD
    configs, p = 0.8; (2) the CPU verification oracle (oracle/verify_oracle.c,
    one thread) at the workload's verify shape, GB/s over the same algorithmic
    bytes as K1; (3) the CPU oracle end to end on config 1 (tiny pair, 2 x 8
    requests, k = 4, greedy): PSD and sequential SD tok/s, mean accepted length."""
    import numpy as np
    from oracle import verify as ov
    from oracle.psd_cpu import CpuBackend
    from paper_2603_18016_b200 import SimConfig, make_requests, mean_accepted_length, run
    from paper_2603_18016_b200.sim import SimBackend
    from paper_2603_18016_b200.verify_bench import algorithmic_bytes
    out = {"cores_host": os.cpu_count()}
    # (1) scheduler wall clock (virtual-time backend)
    sched = {}
    for mode, fac in (("psd", 1), ("standard-sd", 2)):
        reqs = make_requests([CFG["output"]] * CFG["n_requests"], prompt_len=CFG["prompt"])
        t0 = time.perf_counter()
        run(SimConfig(mode=mode, m=CFG["m"], k=CFG["k"], sd_batch_factor=fac), reqs,
            backend=SimBackend())
        sched[mode] = round((time.perf_counter() - t0) * 1e3, 1)
    out["scheduler_wall_ms"] = dict(sched, threads=1,
                                    note="reference scheduler semantics (port, byte-identical "
                                         "step logs) with its latency and coin-flip acceptance "
                                         "models, p = 0.8")
    # (2) CPU verification oracle at the verify shape
    B, K = CFG["m"], CFG["k"]
    rng = np.random.default_rng(0)
    t = (rng.standard_normal((B, K + 1, vocab), dtype=np.float32) * 2.0)
    ids = t[:, :K].argmax(axis=2).astype(np.int32)
    ln = np.full(B, K, np.int32)
    t0 = time.perf_counter()
    ov.verify_greedy(t, ids, ln)
    dt = time.perf_counter() - t0
    d = (t[:, :K] + rng.standard_normal((B, K, vocab), dtype=np.float32) * 0.5)
    u = rng.random((B, K + 1), dtype=np.float32)
    t0 = time.perf_counter()
    ov.verify_sample(t, d, ids, ln, u)
    dts = time.perf_counter() - t0
    gb, gbs = algorithmic_bytes(B, K, vocab, False), algorithmic_bytes(B, K, vocab, True)
    out["verify_oracle"] = {"shape": f"B={B} k={K} V={vocab}", "threads": 1,
                            "greedy_GBps": round(gb / dt / 1e9, 3),
                            "sampling_GBps": round(gbs / dts / 1e9, 3)}
    del t, d
    # (3) config 1 on the CPU oracle: PSD vs sequential SD
    c1 = {}
    be = CpuBackend("tiny-target", "tiny-draft", seed=0, beta_target=3.0, beta_draft=12.0,
                    max_seq_len=64)
    for mode, fac in (("psd", 1), ("standard-sd", 2)):
        reqs = make_requests([32] * 16, prompt_len=16)
        t0 = time.perf_counter()
        _, rep = run(SimConfig(mode=mode, m=8, k=4, sd_batch_factor=fac), reqs, backend=be)
        dt = time.perf_counter() - t0
        c1[mode] = {"tok_s": round(rep.total_generated / dt, 1),
                    "mean_accepted_len": round(mean_accepted_length(rep), 4)}
    out["cfg1_cpu_oracle"] = dict(c1, workload="tiny pair, 2 x 8 requests, prompt 16, "
                                               "output 32, k = 4, greedy", threads=1)
    return out


def run_reference(args) -> None:
    world, rank, _ = _dist()
    if rank != 0:
        return
    from oracle.psd_cpu import CpuBackend  # noqa: F401
    sample = dict(n_req=2, out_len=6)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    vals = []
    t_all = 0.0
    tok_all = 0
    # model construction happens once inside cpu_sample's backend; warm-up
    # steps are not timed
    import oracle.psd_cpu as pc
    from paper_2603_18016_b200 import SimConfig, make_requests, run
    be = pc.CpuBackend(CFG["target"], CFG["draft"], seed=0, beta_target=BETA_TARGET,
                       beta_draft=BETA_DRAFT, max_seq_len=CFG["prompt"] + 32)
    cfg = SimConfig(mode="psd", m=1, k=CFG["k"])
    for i in range(args.warmup + args.steps):
        reqs = make_requests([sample["out_len"]] * sample["n_req"], prompt_len=CFG["prompt"])
        t0 = time.perf_counter()
        st, rep = run(cfg, reqs, backend=be)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(rep.total_generated / dt)
            t_all += dt
            tok_all += rep.total_generated
    v = tok_all / t_all
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "tok/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t_all / args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg2 (8B target / 1B draft, k=5, prompt 128) bounded CPU "
                                   f"sample: {sample['n_req']} requests x {sample['out_len']} "
                                   "tokens per step",
                       "impl": "CPU oracle (oracle/: numpy forward + C canonical verify)"},
            "cpu_baseline": {"value": round(v, 4), "unit": "tok/s", "cores": os.cpu_count(),
                             "kind": "port",
                             "sample": f"{sample['n_req']} req x {sample['out_len']} tok, "
                                       "prompt 128, k=5, 8B/1B shapes"},
            "e2e": {"value": round(v, 4), "unit": "tok/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def replica_sd(args, rank, world, dev, barrier) -> dict:
    """SD(2m) with every rank an independent target + draft replica, timed
    like the main modes (warm-up, barrier, CUDA events, max over ranks)."""
    import torch

    from paper_2603_18016_b200 import dist as pd
    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.gpu import GpuBackend
    be = GpuBackend(CFG["target"], CFG["draft"], max_requests=CFG["n_requests"],
                    max_batch=CFG["n_requests"], k_max=CFG["k"],
                    max_seq_len=CFG["prompt"] + CFG["output"] + 16, seed=rank // 2,
                    beta_target=BETA_TARGET, beta_draft=BETA_DRAFT, device=dev,
                    mode="sample" if args.workload == "cfg3" else "greedy", temperature=1.0)
    for _ in range(args.warmup):
        run(_config("standard-sd"), _workload(rank), backend=be)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tok = 0
    for _ in range(args.steps):
        _, rep = run(_config("standard-sd"), _workload(rank), backend=be)
        tok += rep.total_generated
    e1.record()
    barrier()
    tokens, ms = pd.aggregate(tok, e0.elapsed_time(e1), dev)
    del be
    torch.cuda.empty_cache()
    return {"value": round(tokens / (ms * 1e-3), 1), "unit": "tok/s",
            "mode": f"standard-sd (sd_batch_factor 2), {world} independent replicas, target "
                    "+ draft on every GPU"}


def pair_model(psd: dict, sdm: dict, sd: dict, steps: int) -> dict:
    """One-GPU model of the dedicated-draft-GPU pair (SURVEY §7 hard part 1),
    from this run's isolated phase timings: SD(m) steps draft then verify one
    batch of m alone on the GPU, so its per-step draft and verify times are
    what each GPU of a pair would spend.  A pair's PSD step = max(draft,
    verify) (+ the id hand-off, ~0.1 ms over NVLink, neglected); the baselines
    on the same two GPUs are SD with the draft on its own GPU (draft + verify
    per step) and two SD(2m) replicas."""
    if not sdm["steps"]:
        return {}
    d = sdm["draft_ms"] / sdm["steps"]
    v = sdm["verify_ms"] / sdm["steps"]
    tok_pass = psd["tokens"] / steps
    psd_steps = psd["steps"] / steps
    sdm_steps = sdm["steps"] / steps
    t_psd = psd_steps * max(d, v) * 1e-3
    t_sdd = sdm_steps * (d + v) * 1e-3
    rep2 = 2 * sd["tokens"] / (sd["ms"] * 1e-3)
    return {"draft_ms_per_step": round(d, 3), "verify_ms_per_step": round(v, 3),
            "psd_pair_tok_s": round(tok_pass / t_psd, 1),
            "sd_dedicated_draft_tok_s": round(tok_pass / t_sdd, 1),
            "sd2m_two_replicas_tok_s": round(rep2, 1),
            "psd_pair_vs_sd_dedicated_draft": round(t_sdd / t_psd, 4),
            "psd_pair_vs_sd2m_two_replicas": round(tok_pass / t_psd / rep2, 4),
            "note": "model from isolated one-GPU phase times (SD(m) steps), not a 2-GPU "
                    "measurement"}


def run_ours(args) -> None:
    import torch

    from paper_2603_18016_b200 import dist as pd
    world, rank, local = pd.init(args.dist_backend)
    # --dist-backend gloo with more ranks than GPUs (a smoke run of the pair
    # protocol on one GPU) shares the devices round-robin
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2603_18016_b200 import mean_accepted_length, run
    from paper_2603_18016_b200.gpu import GpuBackend

    hbm_peak, bf16_peak, peak_kind = _peaks()
    if args.layout == "auto":
        # PSD's structural gain needs the draft on its own GPU:
        # even N runs N/2 (target GPU, draft GPU) pairs; N = 1 (or odd) runs
        # target + draft on each GPU, two streams
        args.layout = "pairs" if world >= 2 and world % 2 == 0 else "replicas"
    pairs = args.layout == "pairs"
    # tp-draft: the paper's cfg4 deployment -- a tensor-parallel target over
    # --tp ranks plus one dedicated draft rank per replica (world % (tp + 1) == 0)
    tp_draft = args.layout == "tp-draft"
    tp_layout = args.layout == "tp" or tp_draft
    global BETA_TARGET, BETA_DRAFT
    if tp_layout:
        CFG.update(CFG4)
        BETA_TARGET = BETA_TARGET_CFG4
    sampling = args.workload == "cfg3"
    if sampling:
        CFG.update(CFG3)
        BETA_TARGET, BETA_DRAFT = BETAS_CFG3
    if args.models:  # smoke runs of a layout at smaller shapes (not a bench number)
        CFG["target"], CFG["draft"] = args.models.split(",")
    if pairs and world % 2:
        raise SystemExit("--layout pairs needs an even number of GPUs")
    # replicas: every rank = target + draft on one GPU (two streams)
    # pairs: even rank = target GPU (scheduler), odd rank = dedicated draft GPU
    roles = ("target", "draft") if not pairs else (("target",) if rank % 2 == 0 else ("draft",))
    replica = rank // 2 if pairs else rank
    tp = None
    tp_size = 1
    group_size = 1  # ranks per replica
    if tp_draft:
        tp_size = args.tp or max(1, world - 1)
        group_size = tp_size + 1
        if world % group_size:
            raise SystemExit("--layout tp-draft needs a multiple of (--tp + 1) GPUs")
        replica, li = rank // group_size, rank % group_size
        roles = ("draft",) if li == tp_size else ("target",)
        groups = [torch.distributed.new_group(list(range(r * group_size,
                                                         r * group_size + tp_size)))
                  for r in range(world // group_size)]
        if tp_size > 1 and li < tp_size:
            tp = (li, tp_size, groups[replica])
    elif tp_layout:
        # world // tp_size replicas, each a tensor-parallel target over tp_size
        # ranks (SPMD scheduler) with the draft on a second stream of every TP
        # rank: the 8-GPU cfg4 layout "two TP4 replicas" (SURVEY §7 hard part 8)
        tp_size = args.tp or world
        if world % tp_size:
            raise SystemExit("--tp must divide the number of GPUs")
        replica = rank // tp_size
        groups = [torch.distributed.new_group(list(range(r * tp_size, (r + 1) * tp_size)))
                  for r in range(world // tp_size)] if world > 1 else []
        if tp_size > 1:
            tp = (rank % tp_size, tp_size, groups[replica])
    be = GpuBackend(CFG["target"], CFG["draft"], max_requests=CFG["n_requests"],
                    max_batch=CFG["n_requests"], k_max=CFG["k"], tp=tp,
                    max_seq_len=CFG["prompt"] + CFG["output"] + 16, seed=replica,
                    beta_target=BETA_TARGET, beta_draft=BETA_DRAFT, device=dev, roles=roles,
                    mode="sample" if sampling else "greedy", temperature=1.0)
    is_draft_rank = (pairs and rank % 2 == 1) or (tp_draft and "target" not in roles)
    backend = be
    if tp_draft:
        from paper_2603_18016_b200.pair import (DraftServer, GpuDraftEngine, GpuTargetEngine,
                                                PairLink, PairTarget)
        base = replica * group_size
        draft_rank = base + tp_size
        rep_groups = [torch.distributed.new_group(list(range(r * group_size,
                                                             (r + 1) * group_size)))
                      for r in range(world // group_size)]
        comm = None
        if os.environ.get("PSD_PAIR_LINK", "peer") == "peer":
            from paper_2603_18016_b200.comm import PeerComm
            comm = PeerComm(rep_groups[replica], buf_bytes=1 << 12, mbox_bytes=1 << 20,
                            device=dev)
        nccl = dev if args.dist_backend == "nccl" else None
        if is_draft_rank:
            link = PairLink(base, nccl, comm=comm, comm_peer=0)
            followers = tuple(PairLink(base + j, nccl, comm=comm, comm_peer=j)
                              for j in range(1, tp_size))
        else:
            link = PairLink(draft_rank, nccl, comm=comm, comm_peer=tp_size)
            backend = PairTarget(GpuTargetEngine(be), link, leader=rank == base)
    if pairs:
        from paper_2603_18016_b200.pair import (DraftServer, GpuDraftEngine, GpuTargetEngine,
                                                PairLink, PairTarget)
        peer = rank + 1 if rank % 2 == 0 else rank - 1
        # drafted ids through a 2-rank peer-memory mailbox (csrc/comm.cu) by
        # default; PSD_PAIR_LINK=dist keeps them on dist.send / recv
        pair_groups = [torch.distributed.new_group([2 * t, 2 * t + 1])
                       for t in range(world // 2)]
        comm = None
        if os.environ.get("PSD_PAIR_LINK", "peer") == "peer":
            from paper_2603_18016_b200.comm import PeerComm
            comm = PeerComm(pair_groups[rank // 2], buf_bytes=1 << 12, mbox_bytes=1 << 20,
                            device=dev)
        link = PairLink(peer, dev if args.dist_backend == "nccl" else None, comm=comm)
        if not is_draft_rank:
            backend = PairTarget(GpuTargetEngine(be), link)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    launches = {}

    tuners = []

    def one(mode):
        if mode == "psd-ktune":  # online draft depth
            from paper_2603_18016_b200 import KTuner
            t = KTuner(k_max=CFG["k"], mode="psd", warmup=3)
            tuners.append(t)
            return run(_config("psd"), _workload(rank), backend=backend, k_tuner=t)
        return run(_config(mode), _workload(rank), backend=backend)

    results = {}
    modes = ("psd", "standard-sd", "sd-m") + (("psd-ktune",) if args.ktune else ())
    for mode in modes:
        if is_draft_rank:
            # serve warm-up + timed passes of this mode, then join the timing reduction
            fol = followers if tp_draft else ()
            DraftServer(GpuDraftEngine(be), link, fol).serve()
            barrier()
            DraftServer(GpuDraftEngine(be), link, fol).serve()
            barrier()
            pd.aggregate(0, 0.0, dev)
            results[mode] = None
            continue
        for _ in range(args.warmup):
            one(mode)
        if pairs or tp_draft:
            backend.stop()
        barrier()
        clocks = Clocks(local) if mode == "psd" else None
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        reps, states = [], []
        stats0 = dict(backend.stats)
        l0 = be.launches
        for _ in range(args.steps):
            st_, rep_ = one(mode)
            reps.append(rep_)
            states.append(st_)
        e1.record()
        if pairs or tp_draft:
            backend.stop()
        barrier()
        launches[mode] = be.launches - l0
        ms_local = e0.elapsed_time(e1)
        tokens, ms = pd.aggregate(sum(r.total_generated for r in reps), ms_local, dev)
        if tp_layout:
            tokens //= tp_size  # every TP rank of a replica emits the same tokens
        results[mode] = {"ms": ms, "tokens": tokens, "reps": reps, "states": states,
                         "clocks": clocks.stop() if clocks else None,
                         "draft_ms": backend.stats["draft_ms"] - stats0["draft_ms"],
                         "verify_ms": backend.stats["verify_ms"] - stats0["verify_ms"],
                         "steps": backend.stats["steps"] - stats0["steps"]}
    # end to end through the public API with host prompts / host outputs
    barrier()
    if is_draft_rank:
        DraftServer(GpuDraftEngine(be), link, followers if tp_draft else ()).serve()
    else:
        x0 = be.transfer_bytes()
        t0 = time.perf_counter()
        st, rep_e2e = one("psd")
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        x1 = be.transfer_bytes()
        if pairs or tp_draft:
            backend.stop()
    # the other baseline on the same GPUs: every GPU an independent SD(2m)
    # replica (target + draft on one GPU, its own 64 requests)
    sd_rep = replica_sd(args, rank, world, dev, barrier) if pairs else None
    if is_draft_rank:
        pd.finalize()
        return
    roof, vk = kernel_rooflines(be, hbm_peak, bf16_peak)
    vsweep = verify_sweep_summary(hbm_peak) if rank == 0 and not args.no_sweep else None
    cpu = None
    # the CPU sample is quoted on the 8B / 1B shapes: cfg2 / cfg3 runs only
    # (the 70B layouts skip it)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.layout not in ("tp",
                                                                                   "tp-draft"):
        try:
            v, secs, toks, cores = cpu_sample()
            cpu = {"value": round(v, 4), "unit": "tok/s", "cores": cores, "kind": "port",
                   "sample": f"CPU oracle PSD (numpy / BLAS forward on the host cores, C "
                             f"verify), 2 "
                             f"requests x 6 tokens, prompt 128, k=5, 8B/1B shapes "
                             f"({toks} tokens in {secs:.1f} s)",
                   "plan": cpu_plan_baselines(be.tshape.vocab)}
        except MemoryError as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "tok/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"skipped: {exc}"}
    if rank != 0:
        pd.finalize()
        return
    psd, sd, sdm = results["psd"], results["standard-sd"], results["sd-m"]

    def outputs(res):
        return [r.output_ids for st_ in res["states"] for r in st_.request_list()]
    # greedy output is schedule independent: PSD, SD(2m) and SD(m) must emit
    # the same tokens for every request of every timed pass (north star:
    # identical greedy sequences); sampling compares the same way (uniforms
    # are keyed by request and position, not by schedule)
    po = outputs(psd)
    ident = {"psd_vs_sd": po == outputs(sd), "psd_vs_sd_m": po == outputs(sdm),
             "requests": len(po), "tokens": sum(len(x) for x in po),
             "mismatched_requests": sum(a != b for a, b in zip(po, outputs(sd)))}
    value = psd["tokens"] / (psd["ms"] * 1e-3)  # tokens summed over ranks / max time
    sd_value = sd["tokens"] / (sd["ms"] * 1e-3)
    r0 = psd["reps"][0]
    steps_sd = sd["steps"] / max(1, args.steps)
    steps_psd = psd["steps"] / max(1, args.steps)
    # counted at every host <-> device copy the backend issued during the e2e pass
    h2d, d2h = x1[0] - x0[0], x1[1] - x0[1]
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tok/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(psd["ms"] / args.steps, 2), "higher_is_better": True,
        "scaling": ("strong" if tp_layout and tp_size == world else "weak"), "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": ("cfg3: Qwen2.5-7B target / Qwen2.5-0.5B draft shapes, "
                                "random-init bf16, 2x32 requests, k=4, prompt 128, output 256, "
                                "T=1.0 rejection sampling, both models on one GPU"
                                if sampling else
                                ("cfg4: Llama-3.1-70B target (tensor-parallel over --tp ranks "
                                 "+ a dedicated draft rank per replica) / " if tp_draft else
                                 "cfg4: Llama-3.1-70B target (tensor-parallel replicas, --tp "
                                 "ranks each, draft on a second stream of every TP rank) / ") +
                                "Llama-3.2-1B draft shapes, random-init bf16, 2x64 requests, "
                                "k=4, prompt 128, output 256, greedy" if tp_layout else
                                "cfg2: Llama-3.1-8B target / Llama-3.2-1B draft shapes, "
                                "random-init bf16, 2x32 requests, k=5, prompt 128, output 256, "
                                "greedy, 1 GPU per replica (draft / verify on separate streams)"),
                   "global_batch": (world // group_size if tp_draft else
                                    world // tp_size if tp_layout else
                                    world // 2 if pairs else world)
                   * CFG["n_requests"],
                   "seq_len": CFG["prompt"] + CFG["output"],
                   "models": f"{CFG['target']} / {CFG['draft']}" + (" (--models smoke override)"
                                                                    if args.models else ""),
                   "parallelism": (f"tp{tp_size}+draft x{world // group_size}" if tp_draft else
                                   f"tp{tp_size}x{world // tp_size}" if tp_layout else
                                   f"pairs{world // 2}" if pairs else f"replicas{world}"),
                   "l2": "inputs > L2 (weights 18.5 GB streamed per step)",
                   "synthetic_language_beta": [BETA_TARGET, BETA_DRAFT]},
        "sd": {"value": round(sd_value, 1), "unit": "tok/s",
               "mode": ("standard-sd with the draft on its own GPU (the paper's baseline), "
                        if pairs else "standard-sd, ") + "one batch of 64 (sd_batch_factor 2)",
               "steps_per_pass": steps_sd,
               "draft_ms_per_pass": round(sd["draft_ms"] / args.steps, 2),
               "verify_ms_per_pass": round(sd["verify_ms"] / args.steps, 2),
               "gpu_launches": launches.get("standard-sd")},
        "sd_m": {"value": round(sdm["tokens"] / (sdm["ms"] * 1e-3), 1), "unit": "tok/s",
                 "mode": ("standard-sd with the draft on its own GPU, " if pairs else
                          "standard-sd, ") + "batches of m (sd_batch_factor 1), the PSD batch "
                                             "size"},
        "psd_ktune": ({"value": round(results["psd-ktune"]["tokens"]
                                      / (results["psd-ktune"]["ms"] * 1e-3), 1),
                       "unit": "tok/s", "final_k": tuners[-1].k if tuners else None,
                       "p_est": round(tuners[-1].p, 4) if tuners and tuners[-1].p else None}
                      if "psd-ktune" in results and results["psd-ktune"] else None),
        "psd_vs_sd": round(value / sd_value, 4),
        "sd_replicas": sd_rep,
        "psd_vs_sd_replicas": (round(value / sd_rep["value"], 4) if sd_rep else None),
        "pair_model": (pair_model(psd, sdm, sd, args.steps) if world == 1 else None),
        "psd_vs_sd_m": round(value / (sdm["tokens"] / (sdm["ms"] * 1e-3)), 4),
        "greedy_identical": ident,
        "mean_accepted_len": round(mean_accepted_length(r0), 4),
        "accepted_per_verify": round(r0.total_accepted / max(1, r0.total_bonus), 4),
        "psd_steps_per_pass": steps_psd,
        "draft_hiding": draft_hiding(psd["states"]),
        # CUDA-event time inside PSD steps vs the timed wall time: the rest is
        # host scheduling between steps (the GPU idles there)
        "device_step_ms_per_pass": round(sum(rec.step_duration for st in psd["states"]
                                             for rec in st.step_log) / max(1, len(psd["states"])),
                                         2),
        "draft_ms_per_pass": round(psd["draft_ms"] / args.steps, 2),
        "verify_ms_per_pass": round(psd["verify_ms"] / args.steps, 2),
        "e2e": {"value": round(rep_e2e.total_generated / e2e_s, 1), "unit": "tok/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches.get("psd"),
        "clocks": psd["clocks"],
        "roofline": dict(roof, peak_kind=peak_kind),
        "verify_kernel": vk,
        "verify_sweep": vsweep,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    pd.finalize()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend (gloo: host transport, for a smoke run "
                         "of the multi-rank layouts on one GPU)")
    ap.add_argument("--tp", type=int, default=0,
                    help="--layout tp: ranks per tensor-parallel replica (default: all)")
    ap.add_argument("--models", default="",
                    help="TARGET,DRAFT preset override for smoke runs of a layout (e.g. "
                         "tp-draft with 8B / 1B shapes on one GPU); not a bench number")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the config-5 verify-kernel grid (verify_sweep)")
    ap.add_argument("--ktune", action="store_true",
                    help="also run PSD with the online draft-depth tuner (ktune.KTuner)")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "cfg3"],
                    help="cfg2: 8B / 1B greedy (the headline); cfg3: Qwen2.5-7B / 0.5B, "
                         "T = 1.0 rejection sampling over the 152k vocabulary")
    ap.add_argument("--layout", default="auto",
                    choices=["auto", "replicas", "pairs", "tp", "tp-draft"],
                    help="auto: pairs for an even number of GPUs, else replicas; "
                         "replicas: each GPU runs target+draft (two streams); pairs: "
                         "dedicated draft GPU per target GPU (NCCL hand-off, pair.py); tp: "
                         "BASELINE config 4, 70B target tensor-parallel over all GPUs; "
                         "tp-draft: config 4 as deployed in the paper, a --tp-way "
                         "tensor-parallel target + a dedicated draft GPU per replica")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
