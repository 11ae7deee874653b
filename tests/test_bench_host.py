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


def test_pair_model_from_isolated_phases():
    # SD(m): 10 steps per pass, draft 4 ms + verify 6 ms per step; PSD: 20
    # steps per pass; 1000 tokens per pass; SD(2m): 1000 tokens in 50 ms
    sdm = {"steps": 10, "draft_ms": 40.0, "verify_ms": 60.0}
    psd = {"steps": 20, "tokens": 1000}
    sd = {"tokens": 1000, "ms": 50.0}
    m = bench.pair_model(psd, sdm, sd, steps=1)
    assert m["draft_ms_per_step"] == 4.0 and m["verify_ms_per_step"] == 6.0
    # PSD pair: 20 steps x max(4, 6) ms = 120 ms -> 8333.3 tok/s
    assert abs(m["psd_pair_tok_s"] - 1000 / 0.12) < 0.1
    # SD with a dedicated draft GPU: 10 x (4 + 6) = 100 ms
    assert abs(m["psd_pair_vs_sd_dedicated_draft"] - 100 / 120) < 1e-4
    assert m["sd2m_two_replicas_tok_s"] == 40000.0


def test_sk_physical_matches_gemm_cu():
    class P:
        multi_processor_count = 148
    import torch
    orig = torch.cuda.get_device_properties
    torch.cuda.get_device_properties = lambda dev: P
    try:
        assert bench._sk_physical(None, 0) == 148
        assert bench._sk_physical(None, 92) == 74    # 2 virtual CTAs each
        assert bench._sk_physical(None, 104) == 74
        assert bench._sk_physical(None, 148) == 148
        assert bench._sk_physical(None, 50) == 50    # 3 each: 148 / 3 -> 50
    finally:
        torch.cuda.get_device_properties = orig
