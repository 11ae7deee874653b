"""Host-side measurement logic of bench.py (no GPU): the exposed-drafting
statistic and the JSON-line contract keys it feeds."""

import types

import bench
from paper_2603_18016_b200.records import StepRecord


def _rec(i, tb, draft, verify, prefill, step, fallback=False):
    return StepRecord(step_index=i, target_batch=tb, draft_batch=1 - tb if tb is not None else None,
                      drafted_tokens=10, accepted_tokens=5, bonus_tokens=2, draft_duration=draft,
                      verify_duration=verify, prefill_duration=prefill, step_duration=step,
                      fallback=fallback)


def test_draft_hiding_counts_only_overlapped_steps():
    log = [
        _rec(1, 0, 4.0, 5.0, 2.0, 11.0),          # startup: exposed = 11 - 2 - 5 = 4
        _rec(2, 1, 4.0, 5.0, 0.0, 5.5),           # overlap: exposed 0.5
        _rec(3, 0, 4.0, 5.0, 0.0, 5.0),           # fully hidden
        _rec(4, 1, 3.0, 2.0, 0.0, 5.0, True),     # fallback: not an overlapped step
        _rec(5, None, 0.0, 1.0, 0.0, 1.0),        # no drafting
    ]
    state = types.SimpleNamespace(step_log=log)
    h = bench.draft_hiding([state])
    assert h["steps"] == 3
    assert abs(h["draft_hidden_frac"] - (1 - 4.5 / 12.0)) < 1e-4
    assert abs(h["exposed_draft_frac_of_step"] - 4.5 / 21.5) < 1e-4


def test_draft_hiding_empty():
    h = bench.draft_hiding([types.SimpleNamespace(step_log=[])])
    assert h["draft_hidden_frac"] is None and h["steps"] == 0
