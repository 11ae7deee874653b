"""Scheduler parity against the reference ``specsim`` (golden fixtures).

Each scenario in tests/golden/scheduler_golden.json was produced by running the
unmodified reference (tests/golden/make_scheduler_golden.py).  Here the same
config / workload / preemptions run through this package's scheduler with the
SimBackend and every artefact must match byte-for-byte: rendered step log,
rendered metrics, KV log, finish log, final request states -- or the same
exception type.  Covers c08 (pkg/tests/test_acceptance.py:315-393), the
README example (pkg/README.md:79-82), the BASELINE-shaped configs and 60
randomized configs over every knob (modes, policies, latency kinds,
acceptance laws, k overrides, poisson arrivals, preemptions).
"""

import json
import os

import pytest

from paper_2603_18016_b200 import (AcceptanceModel, LatencyModel, Preemption, Request,
                                   SimConfig, SpecsimError, render_metrics,
                                   render_step_log, run)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "scheduler_golden.json")
with open(GOLDEN) as fh:
    SCENARIOS = json.load(fh)


def _cfg(d):
    return SimConfig(
        mode=d["mode"], m=d["m"], k=d["k"], capacity=d["capacity"],
        draft_latency=LatencyModel(*d["draft_latency"]),
        verify_latency=LatencyModel(*d["verify_latency"]),
        comm_overhead=d["comm_overhead"], acceptance=AcceptanceModel(*d["acceptance"]),
        block_size=d["block_size"], seed=d["seed"], assign_policy=d["assign_policy"],
        kv_policy=d["kv_policy"], sd_batch_factor=d["sd_batch_factor"],
        k_overrides=tuple(d["k_overrides"]))


@pytest.mark.parametrize("sc", SCENARIOS, ids=[s["name"] for s in SCENARIOS])
def test_replay_matches_reference(sc):
    reqs = [Request(id=a, arrival_time=b, prompt_len=c, target_output_len=d)
            for a, b, c, d in sc["workload"]]
    pres = [Preemption(a, b) for a, b in sc["preemptions"]] or None
    if "error" in sc:
        with pytest.raises(SpecsimError) as info:
            run(_cfg(sc["config"]), reqs, pres)
        assert type(info.value).__name__ == sc["error"]
        return
    state, report = run(_cfg(sc["config"]), reqs, pres)
    assert render_step_log(state.step_log) == sc["step_log"]
    assert render_metrics(report) == sc["metrics"]
    assert [[k.step_index, list(k.allocated_ids), list(k.skipped_ids), k.blocks_in_use]
            for k in state.kv_log] == sc["kv_log"]
    assert [[f.request_id, f.finish_time, f.blocks_at_finish, f.prompt_len, f.total_len]
            for f in state.finish_log] == sc["finish_log"]
    assert [[r.id, r.generated, r.state.value, r.batch_id, r.finish_time]
            for r in state.request_list()] == sc["requests"]


def test_readme_example_numbers():
    sc = next(s for s in SCENARIOS if s["name"] == "readme")
    assert "throughput = 6.85714286" in sc["metrics"]
    assert "vsr = 0.696296296" in sc["metrics"]
