"""Capacity-bound draft selection (D_s; selection.py).

CPU: the selection rule itself, the scheduler with a binding capacity
(every verify pass within capacity, where the reference's "send everything"
policy raises ProtocolError), byte-identical step logs when the capacity does
not bind, and greedy tokens unchanged on the CPU oracle (greedy output does
not depend on draft depth).  GPU: the same token identity on the device path.
"""

import pytest

from oracle.psd_cpu import CpuBackend
from paper_2603_18016_b200 import (AcceptanceModel, ConfigError, ProtocolError, SimConfig,
                                   make_requests, run)
from paper_2603_18016_b200.selection import AcceptanceTracker, select_depths


def test_under_capacity_unchanged():
    q = {0: 3, 1: 2, 2: 4}
    assert select_depths(q, 9, {0: 0.5, 1: 0.5, 2: 0.5}) == q
    assert select_depths(q, 100, {0: 0.1, 1: 0.9, 2: 0.5}) == q


def test_uniform_p_fills_levels():
    q = {0: 4, 1: 4, 2: 4, 3: 4}
    # 10 positions: every request gets depth 2, then the two lowest ids a third
    assert select_depths(q, 10, dict.fromkeys(q, 0.8)) == {0: 3, 1: 3, 2: 2, 3: 2}
    assert select_depths(q, 0, dict.fromkeys(q, 0.8)) == dict.fromkeys(q, 0)


def test_high_acceptance_gets_deeper_drafts():
    q = {0: 5, 1: 5}
    got = select_depths(q, 6, {0: 0.95, 1: 0.3})
    assert sum(got.values()) == 6 and got[0] > got[1]
    # 0.95^j > 0.3 for j <= 23: request 1 keeps only what is worth more than
    # request 0's remaining positions
    assert got == {0: 5, 1: 1}


@pytest.mark.parametrize("seed", range(20))
def test_selection_properties(seed):
    import random
    rng = random.Random(seed)
    q = {i: rng.randint(0, 8) for i in range(rng.randint(1, 12))}
    p = {i: rng.uniform(0.05, 1.0) for i in q}
    cap = rng.randint(0, sum(q.values()) + 3)
    got = select_depths(q, cap, p)
    assert set(got) == set(q)
    assert sum(got.values()) == min(cap, sum(q.values()))
    assert all(0 <= got[i] <= q[i] for i in q)
    # optimality: the kept positions' values dominate every dropped one
    kept = [p[i] ** j for i in q for j in range(1, got[i] + 1)]
    dropped = [p[i] ** j for i in q for j in range(got[i] + 1, q[i] + 1)]
    if kept and dropped:
        assert min(kept) >= max(dropped) - 1e-12


def test_tracker_estimates_chain_probability():
    tr = AcceptanceTracker(0.8)
    assert tr.p(7) == pytest.approx(0.8)
    for _ in range(50):
        tr.observe(7, 4, 1)  # one accepted then a rejection: p ~ 0.5
    assert tr.p(7) == pytest.approx((50 + 3.2) / (100 + 4))
    tr.observe(8, 4, 4)      # full acceptance: no failed trial
    assert tr.p(8) > 0.8


def _cfg(**kw):
    base = dict(mode="psd", m=4, k=4, acceptance=AcceptanceModel("bernoulli-chain", p=0.7),
                seed=5)
    base.update(kw)
    return SimConfig(**base)


def test_capacity_must_match_without_selection():
    with pytest.raises(ConfigError):
        run(_cfg(capacity=10), make_requests([20] * 8))


def test_reference_policy_raises_where_tetris_fits():
    over = (4,) * 8
    with pytest.raises(ProtocolError):
        run(_cfg(capacity=10, k_overrides=over), make_requests([20] * 8))
    st, rep = run(_cfg(capacity=10, k_overrides=over, draft_selection="tetris"),
                  make_requests([20] * 8))
    assert rep.finished == 8


@pytest.mark.parametrize("mode,factor", [("psd", 1), ("standard-sd", 1), ("standard-sd", 2)])
def test_binding_capacity_every_pass_fits(mode, factor):
    cap = 7
    st, rep = run(_cfg(mode=mode, capacity=cap, draft_selection="tetris", sd_batch_factor=factor),
                  make_requests([5, 9, 17, 30, 12, 25, 8, 40, 3, 22]))
    assert rep.finished == 10
    for rec in st.step_log:
        if mode == "psd":
            # startup drafts both batches (each verified on its own)
            lim = 2 * cap if rec.step_index == 1 else cap
        else:
            lim = cap * factor
        assert rec.drafted_tokens <= lim
    assert rep.total_accepted > 0


def test_non_binding_capacity_is_byte_identical():
    reqs = lambda: make_requests([5, 9, 17, 30, 12, 25, 8, 40])  # noqa: E731
    a, _ = run(_cfg(), reqs())
    b, _ = run(_cfg(draft_selection="tetris"), reqs())
    assert a.step_log == b.step_log and a.kv_log == b.kv_log


def test_tetris_keeps_greedy_tokens_on_cpu_oracle():
    kw = dict(seed=0, beta_target=3.0, beta_draft=12.0)
    reqs = lambda: make_requests([10] * 6, prompt_len=12)  # noqa: E731
    ref, _ = run(SimConfig(mode="psd", m=3, k=3), reqs(),
                 backend=CpuBackend("tiny-target", "tiny-draft", **kw))
    st, rep = run(SimConfig(mode="psd", m=3, k=3, capacity=5, draft_selection="tetris"),
                  reqs(), backend=CpuBackend("tiny-target", "tiny-draft", **kw))
    assert [r.output_ids for r in st.request_list()] == [r.output_ids for r in ref.request_list()]
    assert max(s.drafted_tokens for s in st.step_log[1:]) <= 5


@pytest.mark.gpu
def test_tetris_keeps_greedy_tokens_on_gpu(cuda_device):
    from paper_2603_18016_b200.gpu import GpuBackend
    kw = dict(max_requests=16, max_batch=16, k_max=4, max_seq_len=128, seed=0, beta_target=3.0,
              beta_draft=12.0, prefill_chunk_tokens=512)
    reqs = lambda: make_requests([24] * 16, prompt_len=16)  # noqa: E731
    ref, _ = run(SimConfig(mode="psd", m=8, k=4), reqs(),
                 backend=GpuBackend("tiny-target", "tiny-draft", **kw))
    st, rep = run(SimConfig(mode="psd", m=8, k=4, capacity=12, draft_selection="tetris"),
                  reqs(), backend=GpuBackend("tiny-target", "tiny-draft", **kw))
    assert [r.output_ids for r in st.request_list()] == [r.output_ids for r in ref.request_list()]
    assert max(s.drafted_tokens for s in st.step_log[1:]) <= 12
    assert rep.total_accepted > 0
