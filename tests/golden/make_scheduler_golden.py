"""Generate scheduler golden fixtures by running the REFERENCE ``specsim``.

Run in the build container only (needs /root/reference):

    python tests/golden/make_scheduler_golden.py

Writes tests/golden/scheduler_golden.json: for every scenario the config,
the workload, the preemptions and the reference's outputs -- rendered step
log, KV log, finish log, rendered metrics -- or the exception type it raised.
tests/test_scheduler_parity.py replays each scenario through this package's
scheduler + SimBackend and demands byte equality.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

import specsim  # noqa: E402
from specsim import (AcceptanceModel, LatencyModel, Preemption, Request,  # noqa: E402
                     SimConfig, run)
from specsim.metrics import render_metrics, render_step_log  # noqa: E402
from specsim.workload import LengthSpec, WorkloadSpec, generate_requests  # noqa: E402

OUT = Path(__file__).with_name("scheduler_golden.json")


def cfg_to_dict(c: SimConfig) -> dict:
    return {
        "mode": c.mode, "m": c.m, "k": c.k, "capacity": c.capacity,
        "draft_latency": [c.draft_latency.kind, c.draft_latency.base,
                          c.draft_latency.per_token, c.draft_latency.per_request],
        "verify_latency": [c.verify_latency.kind, c.verify_latency.base,
                           c.verify_latency.per_token, c.verify_latency.per_request],
        "comm_overhead": c.comm_overhead,
        "acceptance": [c.acceptance.kind, c.acceptance.p, c.acceptance.alpha],
        "block_size": c.block_size, "seed": c.seed,
        "assign_policy": c.assign_policy, "kv_policy": c.kv_policy,
        "sd_batch_factor": c.sd_batch_factor, "k_overrides": list(c.k_overrides),
    }


def dict_to_cfg(d: dict) -> SimConfig:
    return SimConfig(
        mode=d["mode"], m=d["m"], k=d["k"], capacity=d["capacity"],
        draft_latency=LatencyModel(*d["draft_latency"]),
        verify_latency=LatencyModel(*d["verify_latency"]),
        comm_overhead=d["comm_overhead"],
        acceptance=AcceptanceModel(*d["acceptance"]),
        block_size=d["block_size"], seed=d["seed"],
        assign_policy=d["assign_policy"], kv_policy=d["kv_policy"],
        sd_batch_factor=d["sd_batch_factor"], k_overrides=tuple(d["k_overrides"]))


def scenario(name, config, workload, preemptions=()):
    wl = [[r.id, r.arrival_time, r.prompt_len, r.target_output_len] for r in workload]
    pre = [[p.request_index, p.time] for p in preemptions]
    reqs = [Request(id=a, arrival_time=b, prompt_len=c, target_output_len=d)
            for a, b, c, d in wl]
    pres = [Preemption(a, b) for a, b in pre] or None
    entry = {"name": name, "config": cfg_to_dict(config), "workload": wl,
             "preemptions": pre}
    try:
        state, report = run(config, reqs, pres)
    except specsim.SpecsimError as exc:
        entry["error"] = type(exc).__name__
        return entry
    entry["step_log"] = render_step_log(state.step_log)
    entry["metrics"] = render_metrics(report)
    entry["kv_log"] = [[k.step_index, list(k.allocated_ids), list(k.skipped_ids),
                        k.blocks_in_use] for k in state.kv_log]
    entry["finish_log"] = [[f.request_id, f.finish_time, f.blocks_at_finish,
                            f.prompt_len, f.total_len] for f in state.finish_log]
    entry["requests"] = [[r.id, r.generated, r.state.value, r.batch_id, r.finish_time]
                         for r in state.request_list()]
    return entry


def const(x):
    return LatencyModel("constant", x)


def main() -> None:
    out = []
    # criterion c08 (pkg/tests/test_acceptance.py:315-393)
    c8 = SimConfig(mode="psd", m=4, k=3, draft_latency=const(1.0),
                   verify_latency=const(1.0), comm_overhead=0.0,
                   acceptance=AcceptanceModel("deterministic-accept-all"),
                   block_size=16, seed=7)
    lens = [4, 16, 8, 16, 12, 16, 16, 16, 20, 20, 20, 20]
    out.append(scenario("c08", c8, [Request(i, 0.0, 8, n) for i, n in enumerate(lens)]))
    # README simulate example (pkg/README.md:79-82): CLI defaults, seed 1234
    readme = SimConfig(seed=1234)
    wl = generate_requests(WorkloadSpec(count=6, prompt_len=LengthSpec("constant", value=8),
                                        output_len=LengthSpec("constant", value=24)), 1234)
    out.append(scenario("readme", readme, wl))
    # the BASELINE-shaped scheduler configs (p = 0.8, output 256, prompt 128)
    for name, m, k, n in (("cfg1", 8, 4, 16), ("cfg2", 32, 5, 64), ("cfg4", 64, 4, 128)):
        for mode in ("psd", "standard-sd"):
            cfg = SimConfig(mode=mode, m=m, k=k, seed=0, sd_batch_factor=2 if mode ==
                            "standard-sd" else 1,
                            acceptance=AcceptanceModel("bernoulli-chain", p=0.8))
            out.append(scenario(f"{name}-{mode}", cfg,
                                [Request(i, 0.0, 128, 256) for i in range(n)]))
    # randomized sweep over every knob
    master = random.Random(20260317)
    for idx in range(60):
        m = master.choice([1, 2, 3, 4, 6])
        k = master.choice([1, 2, 3, 4, 5])
        mode = master.choice(["psd", "psd", "psd", "standard-sd", "psd-fallback-disabled"])
        kind = master.choice(["bernoulli-chain", "frontier-coupled",
                              "deterministic-accept-all"])
        acc = AcceptanceModel(kind, p=master.choice([0.3, 0.6, 0.8, 0.95]),
                              alpha=master.choice([0.5, 1.0, 2.0]))
        lat = lambda: (const(master.choice([0.5, 1.0, 2.0])) if master.random() < 0.5
                       else LatencyModel("affine", master.choice([0.1, 0.5]),
                                         master.choice([0.0, 0.01, 0.05]),
                                         master.choice([0.0, 0.02])))
        koverrides = ()
        if master.random() < 0.2:
            koverrides = tuple(master.randint(1, 6) for _ in range(master.randint(1, 5)))
        cfg = SimConfig(
            mode=mode, m=m, k=k, draft_latency=lat(), verify_latency=lat(),
            comm_overhead=master.choice([0.0, 0.0, 0.1, 0.25]), acceptance=acc,
            block_size=master.choice([4, 8, 16]), seed=master.randint(0, 2**31),
            assign_policy=master.choice(["skip-batch", "skip-batch", "always-balance"]),
            kv_policy=master.choice(["deferred", "deferred", "eager"]),
            sd_batch_factor=master.choice([1, 1, 2]), k_overrides=koverrides)
        count = master.randint(1, 3 * m + 2)
        if master.random() < 0.4:
            spec = WorkloadSpec(arrival="poisson", rate=master.choice([0.5, 1.0, 3.0]),
                                count=count,
                                prompt_len=LengthSpec("uniform", lo=0, hi=24),
                                output_len=LengthSpec("uniform", lo=1, hi=40))
        else:
            spec = WorkloadSpec(count=count, prompt_len=LengthSpec("uniform", lo=1, hi=20),
                                output_len=LengthSpec("uniform", lo=1, hi=48))
        wl = generate_requests(spec, master.randint(0, 1000))
        pre = ()
        if master.random() < 0.3:
            pre = tuple(Preemption(master.randrange(count), master.uniform(0.0, 12.0))
                        for _ in range(master.randint(1, 3)))
        out.append(scenario(f"rand{idx:02d}", cfg, wl, pre))
    OUT.write_text(json.dumps(out, indent=0))
    print(f"wrote {len(out)} scenarios to {OUT} "
          f"({sum(1 for e in out if 'error' in e)} raise)")


if __name__ == "__main__":
    main()
