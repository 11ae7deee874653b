"""Replay acceptance mode on the GPU vs the REFERENCE's own outputs.

``GpuBackend(acceptance="replay")`` runs the real draft loop and target verify
forward on the B200 (tcgen05 GEMMs, paged attention, K1 in forced mode, KV
commit), but every verified row accepts the reference's coin-flip count
``accepted_count(model, k, draft_time, acceptance_stream(seed, rid, j))``
(pkg/src/specsim/acceptance_model.py:50-52, 82-97; engine.py:250-256), KV
grants are sized exactly like the reference's (engine.py:162-175) and the
scheduler advances on the latency models' virtual durations.  The step log,
metrics, KV log, finish log and request states must then equal the fixtures
produced by the unmodified specsim (tests/golden/scheduler_golden.json)
byte for byte -- the GPU path is pinned to the reference itself, not to a
restatement.
"""

import json
import os

import numpy as np
import pytest
import torch

from paper_2603_18016_b200 import (AcceptanceModel, LatencyModel, Preemption, Request,
                                   SimConfig, render_metrics, render_step_log, run)
from paper_2603_18016_b200.gpu import GpuBackend

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "scheduler_golden.json")
with open(GOLDEN) as fh:
    SCENARIOS = json.load(fh)


def _eligible(sc):
    c, w = sc["config"], sc["workload"]
    return ("error" not in sc and c["block_size"] == 16 and min(x[2] for x in w) >= 2
            and max([c["k"]] + list(c["k_overrides"])) <= 8)


ELIGIBLE = [s for s in SCENARIOS if _eligible(s)]


def _cfg(d):
    return SimConfig(
        mode=d["mode"], m=d["m"], k=d["k"], capacity=d["capacity"],
        draft_latency=LatencyModel(*d["draft_latency"]),
        verify_latency=LatencyModel(*d["verify_latency"]),
        comm_overhead=d["comm_overhead"], acceptance=AcceptanceModel(*d["acceptance"]),
        block_size=d["block_size"], seed=d["seed"], assign_policy=d["assign_policy"],
        kv_policy=d["kv_policy"], sd_batch_factor=d["sd_batch_factor"],
        k_overrides=tuple(d["k_overrides"]))


def _backend(sc, **kw):
    c, w = sc["config"], sc["workload"]
    k_max = max([c["k"]] + list(c["k_overrides"]))
    width = c["m"] * (c["sd_batch_factor"] if c["mode"] == "standard-sd" else 1)
    running = c["m"] * (c["sd_batch_factor"] if c["mode"] == "standard-sd" else 2)
    return GpuBackend("tiny-target", "tiny-draft", max_requests=min(len(w), running),
                      max_batch=width, k_max=k_max,
                      max_seq_len=max(x[2] + x[3] for x in w) + k_max + 16, seed=1,
                      beta_target=3.0, beta_draft=12.0, prefill_chunk_tokens=2048,
                      acceptance="replay", **kw)


def _run(sc, backend):
    reqs = [Request(id=a, arrival_time=b, prompt_len=c, target_output_len=d)
            for a, b, c, d in sc["workload"]]
    pres = [Preemption(a, b) for a, b in sc["preemptions"]] or None
    return run(_cfg(sc["config"]), reqs, pres, backend=backend)


def test_eligible_scenarios_cover_the_knobs():
    names = {s["name"] for s in ELIGIBLE}
    assert {"c08", "readme", "cfg1-psd", "cfg2-psd", "cfg2-standard-sd"} <= names
    kinds = {s["config"]["acceptance"][0] for s in ELIGIBLE}
    assert kinds == {"bernoulli-chain", "frontier-coupled", "deterministic-accept-all"}
    assert {s["config"]["kv_policy"] for s in ELIGIBLE} == {"deferred", "eager"}
    assert len(ELIGIBLE) >= 15


@pytest.mark.parametrize("sc", ELIGIBLE, ids=[s["name"] for s in ELIGIBLE])
def test_gpu_replay_matches_reference_byte_for_byte(cuda_device, sc):
    be = _backend(sc)
    state, report = _run(sc, be)
    assert render_step_log(state.step_log) == sc["step_log"]
    assert render_metrics(report) == sc["metrics"]
    assert [[k.step_index, list(k.allocated_ids), list(k.skipped_ids), k.blocks_in_use]
            for k in state.kv_log] == sc["kv_log"]
    assert [[f.request_id, f.finish_time, f.blocks_at_finish, f.prompt_len, f.total_len]
            for f in state.finish_log] == sc["finish_log"]
    assert [[r.id, r.generated, r.state.value, r.batch_id, r.finish_time]
            for r in state.request_list()] == sc["requests"]
    # the device really ran every step and produced every committed token
    assert len(be.measured_log) == len(state.step_log)
    assert all(m.verify_duration > 0.0 for m in be.measured_log)
    for r in state.request_list():
        if r.state.value == "finished":
            assert len(r.output_ids) == r.target_output_len
            assert all(0 <= t < 1024 for t in r.output_ids)


@pytest.mark.parametrize("mode", ["greedy", "sample"])
def test_replay_k1_forced_mode_matches_oracle_on_live_logits(cuda_device, mode):
    """Every forced K1 launch inside a replayed run, re-run through the CPU
    oracle's forced mode on the same (GPU-produced) logits / uniforms:
    identical accepted lengths and tokens."""
    from oracle import verify as ov
    sc = next(s for s in ELIGIBLE if s["name"] == "readme")
    be = _backend(sc, mode=mode, temperature=0.8)
    be.capture_verify = []
    state, _ = _run(sc, be)
    assert render_step_log(state.step_log) == sc["step_log"]
    assert len(be.capture_verify) >= 5
    for rec in be.capture_verify:
        if mode == "greedy":
            acc, out = ov.verify_greedy(rec["target"], rec["ids"], rec["len"],
                                        forced_len=rec["forced"])
        else:
            acc, out = ov.verify_sample(rec["target"], rec["draft"], rec["ids"], rec["len"],
                                        rec["uniforms"], 0.8, forced_len=rec["forced"])
        np.testing.assert_array_equal(acc, np.minimum(rec["forced"], rec["len"]))
        np.testing.assert_array_equal(acc, rec["acc"])
        np.testing.assert_array_equal(out, rec["out"])


def test_forced_kernel_accepts_exactly_the_replayed_count(cuda_device):
    """psd_verify_greedy_forced / psd_verify_sample_forced at sweep sizes."""
    from oracle import verify as ov
    from paper_2603_18016_b200 import ops
    from tests import _gen
    dev = cuda_device
    for greedy in (True, False):
        t, d, ids, ln, u = _gen.verify_case(33, 37, 6, 32000, tau=0.5, greedy=greedy)
        rng = np.random.default_rng(5)
        forced = rng.integers(-1, 8, size=37).astype(np.int32)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        if greedy:
            ea, eo = ov.verify_greedy(t, ids, ln, forced_len=forced)
            ga, go = ops.verify_greedy(T(t), T(ids), T(ln), forced_len=T(forced))
        else:
            ea, eo = ov.verify_sample(t, d, ids, ln, u, forced_len=forced)
            ga, go = ops.verify_sample(T(t), T(d), T(ids), T(ln), T(u), forced_len=T(forced))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ea, np.clip(forced, 0, ln))
        np.testing.assert_array_equal(ga.cpu().numpy(), ea)
        np.testing.assert_array_equal(go.cpu().numpy(), eo)
