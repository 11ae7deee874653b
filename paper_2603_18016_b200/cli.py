"""Command line: ``python -m paper_2603_18016_b200 simulate|sweep``.

Mirrors the reference CLI's simulate / sweep subcommands
(pkg/src/specsim/cli.py:1-14, 60-85, 105-150, 284-330): the same flat
``key = value`` config files and ``--set KEY=VALUE`` overrides over the same
keys (config.py:31-67), the same output artefacts (``step_log.csv`` in the
``# step-log v1`` format, ``metrics.txt`` in ``# metrics v1``,
``resolved_config.txt``; ``sweep.csv`` in ``# sweep v1``) and the same exit
codes (0 ok, 2 configuration / workload error, 3 protocol / KV / numeric
failure).  SPECSIM_SEED overrides engine.seed.

What is added is the backend: ``gpu.backend = gpu`` runs every pass on the B200
(GpuBackend: real draft / target forwards, K1 verification), with the models
and sampling set by the ``gpu.*`` keys; the step log then carries CUDA-event
milliseconds.  ``gpu.backend = sim`` (default) is the reference's virtual-time
simulation, byte-identical to specsim.  The theory subcommands (analyze,
verify-theory) are out of scope.
"""

from __future__ import annotations

import argparse
import itertools
import os
import sys
from pathlib import Path

from .acceptance import AcceptanceModel
from .errors import ConfigError, KVError, NumericError, ProtocolError, WorkloadError
from .metrics import MetricsReport, render_metrics, render_step_log
from .records import LatencyModel, SimConfig, validate_config
from .scheduler import run
from .workload import LengthSpec, WorkloadSpec, generate_requests, parse_preemptions

__all__ = ["DEFAULTS", "main", "resolve", "build"]

CONFIG_VERSION = "# config v1"

# the reference's keys (config.py:31-67, theory.* omitted) + the gpu.* backend keys
DEFAULTS: dict[str, str] = {
    "engine.mode": "psd", "engine.m": "4", "engine.k": "3", "engine.capacity": "",
    "engine.comm_overhead": "0.0", "engine.seed": "1234", "engine.assign_policy": "skip-batch",
    "engine.sd_batch_factor": "1", "engine.k_per_request": "",
    "engine.draft_selection": "all",
    "draft.kind": "constant", "draft.base": "1.0", "draft.per_token": "0.0",
    "draft.per_request": "0.0",
    "verify.kind": "constant", "verify.base": "1.0", "verify.per_token": "0.0",
    "verify.per_request": "0.0",
    "acceptance.kind": "bernoulli-chain", "acceptance.p": "0.8", "acceptance.alpha": "1.0",
    "kv.block_size": "16", "kv.policy": "deferred",
    "workload.arrival": "all-at-once", "workload.rate": "0.0", "workload.count": "",
    "workload.prompt_len": "32", "workload.output_len": "128", "workload.preemptions": "",
    "gpu.backend": "sim", "gpu.target": "tiny-target", "gpu.draft": "tiny-draft",
    "gpu.sampling": "greedy", "gpu.temperature": "1.0", "gpu.beta_target": "6.0",
    "gpu.beta_draft": "12.0", "gpu.max_seq_len": "",
}

SWEEP_COLUMNS = tuple(MetricsReport.__dataclass_fields__)


def _parse(text: str, source: str) -> dict[str, str]:
    out = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        key, sep, value = line.partition("=")
        if not sep:
            raise ConfigError(f"{source}:{lineno}: expected KEY = VALUE, got {raw!r}")
        if key.strip() not in DEFAULTS:
            raise ConfigError(f"{source}:{lineno}: unknown config key {key.strip()!r}")
        out[key.strip()] = value.strip()
    return out


def resolve(config_path: str | None, overrides: list[str], seed_env: str | None) -> dict:
    """defaults < config file < --set overrides < SPECSIM_SEED."""
    cfg = dict(DEFAULTS)
    if config_path:
        try:
            cfg.update(_parse(Path(config_path).read_text(encoding="utf-8"), config_path))
        except OSError as exc:
            raise ConfigError(f"cannot read config {config_path}: {exc}") from exc
    for item in overrides:
        key, sep, value = item.partition("=")
        if not sep or key.strip() not in DEFAULTS:
            raise ConfigError(f"override {item!r}: expected a known KEY=VALUE")
        cfg[key.strip()] = value.strip()
    if seed_env is not None and seed_env.strip():
        cfg["engine.seed"] = seed_env.strip()
    return cfg


def _num(cfg, key, cast):
    try:
        return cast(cfg[key])
    except ValueError as exc:
        raise ConfigError(f"{key}: cannot parse {cfg[key]!r}") from exc


def _latency(cfg, prefix):
    return LatencyModel(cfg[f"{prefix}.kind"], _num(cfg, f"{prefix}.base", float),
                        _num(cfg, f"{prefix}.per_token", float),
                        _num(cfg, f"{prefix}.per_request", float))


def build(cfg: dict) -> tuple[SimConfig, WorkloadSpec]:
    k_text = cfg["engine.k_per_request"].strip()
    try:
        k_over = tuple(int(x) for x in k_text.split(",")) if k_text else ()
    except ValueError as exc:
        raise ConfigError(f"engine.k_per_request: bad integer in {k_text!r}") from exc
    try:
        acc = AcceptanceModel(cfg["acceptance.kind"], p=_num(cfg, "acceptance.p", float),
                              alpha=_num(cfg, "acceptance.alpha", float))
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    cap = cfg["engine.capacity"].strip()
    sim = validate_config(SimConfig(
        mode=cfg["engine.mode"], m=_num(cfg, "engine.m", int), k=_num(cfg, "engine.k", int),
        capacity=int(cap) if cap else None, draft_latency=_latency(cfg, "draft"),
        verify_latency=_latency(cfg, "verify"),
        comm_overhead=_num(cfg, "engine.comm_overhead", float), acceptance=acc,
        block_size=_num(cfg, "kv.block_size", int), seed=_num(cfg, "engine.seed", int),
        assign_policy=cfg["engine.assign_policy"], kv_policy=cfg["kv.policy"],
        sd_batch_factor=_num(cfg, "engine.sd_batch_factor", int), k_overrides=k_over,
        draft_selection=cfg["engine.draft_selection"].strip()))
    count = cfg["workload.count"].strip()
    spec = WorkloadSpec(
        arrival=cfg["workload.arrival"], rate=_num(cfg, "workload.rate", float),
        count=int(count) if count else None,
        prompt_len=LengthSpec.parse(cfg["workload.prompt_len"], "workload.prompt_len", 0),
        output_len=LengthSpec.parse(cfg["workload.output_len"], "workload.output_len", 1),
        preemptions=parse_preemptions(cfg["workload.preemptions"]))
    return sim, spec


def _backend(cfg: dict, sim: SimConfig, requests):
    kind = cfg["gpu.backend"]
    if kind == "sim":
        return None
    if kind != "gpu":
        raise ConfigError(f"gpu.backend must be sim or gpu, got {kind!r}")
    from .gpu import GpuBackend
    longest = max(r.prompt_len + r.target_output_len for r in requests)
    msl = cfg["gpu.max_seq_len"].strip()
    k_max = max((sim.k,) + sim.k_overrides)
    # slots for the requests that can run at once (two PSD batches of m, or one
    # SD batch of m * sd_batch_factor), not for the whole workload
    width = sim.m * max(1, sim.sd_batch_factor)
    concurrent = min(len(requests), max(2 * sim.m, width))
    return GpuBackend(cfg["gpu.target"], cfg["gpu.draft"], max_requests=concurrent,
                      max_batch=sim.m * max(1, sim.sd_batch_factor), k_max=k_max,
                      max_seq_len=int(msl) if msl else longest + k_max + 16,
                      mode=cfg["gpu.sampling"], temperature=_num(cfg, "gpu.temperature", float),
                      seed=sim.seed, beta_target=_num(cfg, "gpu.beta_target", float),
                      beta_draft=_num(cfg, "gpu.beta_draft", float),
                      block_size=sim.block_size)


def simulate_once(cfg: dict):
    sim, spec = build(cfg)
    requests = generate_requests(spec, sim.seed)
    return run(sim, requests, list(spec.preemptions),
               backend=_backend(cfg, sim, requests))


def render_resolved(cfg: dict) -> str:
    return "\n".join([CONFIG_VERSION] + [f"{k} = {cfg[k]}" for k in sorted(cfg)]) + "\n"


def cmd_simulate(args) -> int:
    cfg = resolve(args.config, args.set or [], os.environ.get("SPECSIM_SEED"))
    state, report = simulate_once(cfg)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    (out / "step_log.csv").write_text(render_step_log(state.step_log), encoding="utf-8")
    (out / "metrics.txt").write_text(render_metrics(report), encoding="utf-8")
    (out / "resolved_config.txt").write_text(render_resolved(cfg), encoding="utf-8")
    print(f"simulate: {report.finished}/{report.num_requests} finished in {report.total_steps} "
          f"steps ({report.fallback_steps} fallback), makespan {report.makespan:.9g}, "
          f"throughput {report.throughput:.9g}, vsr {report.vsr:.9g}")
    print(f"simulate: wrote {out / 'step_log.csv'}")
    return 0


def _cell(v) -> str:
    if v is None:
        return ""
    return f"{v:.9g}" if isinstance(v, float) else str(v)


def cmd_sweep(args) -> int:
    base = resolve(args.config, args.set or [], os.environ.get("SPECSIM_SEED"))
    if not args.grid:
        raise ConfigError("empty sweep: at least one --grid axis is required")
    axes = []
    for item in args.grid:
        key, sep, vals = item.partition("=")
        values = [v.strip() for v in vals.split(",") if v.strip()]
        if not sep or not values:
            raise ConfigError(f"--grid {item!r}: expected KEY=V1,V2,...")
        if key.strip() not in DEFAULTS:
            raise ConfigError(f"--grid: unknown config key {key.strip()!r}")
        axes.append((key.strip(), values))
    keys = [k for k, _ in axes]
    lines = ["# sweep v1", ",".join(keys + list(SWEEP_COLUMNS) + ["error"])]
    failed = 0
    for combo in itertools.product(*(v for _, v in axes)):
        cfg = dict(base)
        cfg.update(dict(zip(keys, combo)))
        try:
            _, rep = simulate_once(cfg)
            row = [_cell(getattr(rep, c)) for c in SWEEP_COLUMNS] + [""]
        except (ConfigError, WorkloadError, ProtocolError, KVError, NumericError) as exc:
            failed += 1
            row = [""] * len(SWEEP_COLUMNS) + [str(exc).replace(",", ";").replace("\n", " ")]
        lines.append(",".join(list(combo) + row))
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    (out / "sweep.csv").write_text("\n".join(lines) + "\n", encoding="utf-8")
    print(f"sweep: {len(lines) - 2} configurations ({failed} failed), wrote {out / 'sweep.csv'}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2603_18016_b200",
                                description="batch-parallel speculative decoding on B200")
    sub = p.add_subparsers(dest="command", required=True)
    for name, fn in (("simulate", cmd_simulate), ("sweep", cmd_sweep)):
        sp = sub.add_parser(name)
        sp.add_argument("--config", default=None, help="key = value config file")
        sp.add_argument("--set", action="append", metavar="KEY=VALUE", help="override a key")
        sp.add_argument("--out", required=True, help="output directory")
        if name == "sweep":
            sp.add_argument("--grid", action="append", default=[], metavar="KEY=V1,V2,...")
        sp.set_defaults(func=fn)
    return p


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ConfigError, WorkloadError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except (ProtocolError, KVError, NumericError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
