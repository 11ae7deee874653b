"""Regenerate tests/golden/cli/*: the reference CLI's simulate artefacts.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

Runs the unmodified reference (`specsim.cli.main`, pkg/src/specsim/cli.py)
on a few configurations; tests/test_cli.py checks that
`python -m paper_2603_18016_b200 simulate` with the same --set overrides writes
byte-identical step_log.csv and metrics.txt.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {
    "psd_default": ["workload.count=12", "engine.m=4", "engine.k=3"],
    "sd_affine": ["engine.mode=standard-sd", "workload.count=10", "engine.m=3", "engine.k=4",
                  "draft.kind=affine", "draft.base=0.5", "draft.per_token=0.25",
                  "verify.kind=affine", "verify.base=2", "verify.per_request=0.1",
                  "engine.sd_batch_factor=2"],
    "psd_poisson_preempt": ["workload.count=16", "workload.arrival=poisson",
                            "workload.rate=0.5", "workload.prompt_len=uniform:4:20",
                            "workload.output_len=uniform:8:40", "workload.preemptions=0@2 5@9",
                            "engine.m=4", "engine.k=4", "engine.k_per_request=1,2,3,4",
                            "acceptance.kind=frontier-coupled", "acceptance.alpha=0.7",
                            "engine.comm_overhead=0.05", "kv.policy=deferred"],
}


def main():
    from specsim.cli import main as ref_main
    for name, sets in CASES.items():
        out = os.path.join(HERE, "cli", name)
        argv = ["simulate", "--out", out]
        for s in sets:
            argv += ["--set", s]
        rc = ref_main(argv)
        assert rc == 0, (name, rc)
        os.remove(os.path.join(out, "resolved_config.txt"))  # key sets differ (gpu.*, theory.*)
    with open(os.path.join(HERE, "cli", "cases.json"), "w") as fh:
        json.dump(CASES, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
