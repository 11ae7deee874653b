"""CLI parity: `python -m paper_2603_18016_b200
simulate` with the sim backend writes the same step_log.csv / metrics.txt
bytes as the reference CLI on the same --set overrides
(tests/golden/cli, tests/golden/make_cli_golden.py), and the exit codes of
the reference (2: configuration / workload error)."""

import json
import os

import pytest

from paper_2603_18016_b200.cli import main

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")
CASES = json.load(open(os.path.join(GOLD, "cases.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_simulate_matches_reference_cli(name, tmp_path):
    argv = ["simulate", "--out", str(tmp_path)]
    for s in CASES[name]:
        argv += ["--set", s]
    assert main(argv) == 0
    for f in ("step_log.csv", "metrics.txt"):
        got = (tmp_path / f).read_text()
        want = open(os.path.join(GOLD, name, f)).read()
        assert got == want, f


def test_sweep_and_errors(tmp_path, capsys):
    rc = main(["sweep", "--out", str(tmp_path), "--set", "workload.count=6",
               "--grid", "engine.k=1,3", "--grid", "engine.mode=psd,standard-sd"])
    assert rc == 0
    lines = (tmp_path / "sweep.csv").read_text().splitlines()
    assert lines[0] == "# sweep v1" and len(lines) == 2 + 4
    assert main(["simulate", "--out", str(tmp_path), "--set", "engine.k=0"]) == 2
    assert main(["simulate", "--out", str(tmp_path), "--set", "nope.key=1"]) == 2


@pytest.mark.gpu
def test_simulate_on_the_gpu_backend(tmp_path, cuda_device):
    """gpu.backend = gpu: the same artefacts from real B200 passes (CUDA-event
    ms in the step log), every request finished with its full output."""
    rc = main(["simulate", "--out", str(tmp_path), "--set", "gpu.backend=gpu",
               "--set", "workload.count=8", "--set", "workload.prompt_len=12",
               "--set", "workload.output_len=20", "--set", "engine.m=4", "--set", "engine.k=3",
               "--set", "gpu.beta_target=3", "--set", "gpu.beta_draft=12"])
    assert rc == 0
    metrics = dict(line.split(" = ") for line in
                   (tmp_path / "metrics.txt").read_text().splitlines()[1:])
    assert metrics["finished"] == "8"
    log = (tmp_path / "step_log.csv").read_text().splitlines()
    assert log[0] == "# step-log v1" and len(log) > 3
