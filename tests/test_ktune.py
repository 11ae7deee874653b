"""Online draft-depth tuner on the simulation backend.

The reference's frontier model (pkg/src/specsim/analytic.py) says the
batch-parallel optimum drafts as long as verification takes; with a
bernoulli-chain acceptance p, a per-token draft cost and a constant verify
time, the best integer depth is known in closed form and the tuner must find
it from the step log alone.
"""

import pytest

from paper_2603_18016_b200 import KTuner, SimConfig, make_requests, run
from paper_2603_18016_b200.acceptance import AcceptanceModel
from paper_2603_18016_b200.ktune import expected_chain_accepts, invert_chain_accepts
from paper_2603_18016_b200.records import LatencyModel


@pytest.mark.parametrize("p", [0.3, 0.6, 0.85, 0.97])
@pytest.mark.parametrize("k", [1, 3, 5, 8])
def test_chain_inversion(p, k):
    a = expected_chain_accepts(p, k)
    assert abs(invert_chain_accepts(a, k) - p) < 1e-6


def _cfg(mode, k, p, draft_per_token, verify):
    return SimConfig(mode=mode, m=4, k=k,
                     draft_latency=LatencyModel("affine", 0.0, per_token=draft_per_token),
                     verify_latency=LatencyModel("constant", verify),
                     acceptance=AcceptanceModel("bernoulli-chain", p=p), seed=7)


@pytest.mark.parametrize("mode,p,cost,verify", [
    ("psd", 0.8, 0.625, 10.0),     # d = 2.5 per draft step of 4 rows: PSD optimum k = 4
    ("psd", 0.95, 0.25, 10.0),     # cheap drafts, high acceptance: deep
    ("standard-sd", 0.8, 0.625, 10.0),
    ("standard-sd", 0.5, 2.0, 4.0),  # expensive drafts, low acceptance: shallow
])
def test_tuner_converges_to_the_model_optimum(mode, p, cost, verify):
    tuner = KTuner(k_max=8, mode=mode, warmup=2, ema=0.2)
    cfg = _cfg(mode, 8, p, cost, verify)
    # many requests so batches stay full (4 rows) over the measured window
    st, rep = run(cfg, make_requests([400] * 32, prompt_len=8), k_tuner=tuner)
    assert rep.finished == 32
    d = cost * 4  # one draft step of a full batch (4 rows)
    want = tuner.best_k(p, d, verify)
    # steady state: the middle half of the run (batches full); the estimate of
    # p is noisy, so the chosen depth is the optimum or within 3 % of its rate
    hist = tuner.history[len(tuner.history) // 4: 3 * len(tuner.history) // 4]
    ks = [h[1] for h in hist]
    got = max(set(ks), key=ks.count)
    assert got == want or tuner.rate(got, p, d, verify) >= 0.97 * tuner.rate(want, p, d, verify)
    assert abs(sum(h[2] for h in hist) / len(hist) - p) < 0.05
    assert abs(sum(h[3] for h in hist) / len(hist) - d) < 0.05 * d


def test_without_tuner_the_run_is_unchanged():
    cfg = _cfg("psd", 5, 0.8, 0.5, 10.0)
    a, _ = run(cfg, make_requests([40] * 8, prompt_len=8))
    b, _ = run(cfg, make_requests([40] * 8, prompt_len=8), k_tuner=None)
    assert [(s.drafted_tokens, s.accepted_tokens) for s in a.step_log] == \
        [(s.drafted_tokens, s.accepted_tokens) for s in b.step_log]


def test_rows_inversion_with_mixed_depths():
    from paper_2603_18016_b200.ktune import invert_chain_accepts_rows
    p = 0.7
    pairs = [(1, 0), (3, 0), (5, 0), (8, 0)]
    total = sum(expected_chain_accepts(p, k) for k, _ in pairs)
    # spread the expected total over the rows (only the sum matters)
    pairs = [(k, total / len(pairs)) for k, _ in pairs]
    assert abs(invert_chain_accepts_rows(pairs) - p) < 1e-6


def test_tuner_estimates_p_from_verified_rows_with_unequal_batches():
    """Batches of different sizes (odd request count, arrivals ramping up and
    draining): the skip batch's drafted count and the verified batch's
    accepted count come from different rows, so p must come from the
    verified rows alone."""
    p = 0.8
    tuner = KTuner(k_max=5, mode="psd", warmup=10_000, ema=0.05, k0=5)
    cfg = _cfg("psd", 5, p, 0.5, 10.0)
    lens = [60, 300, 45, 200, 90, 150, 30]  # 7 requests: batches of 4 and 3, uneven drain
    st, rep = run(cfg, make_requests(lens, prompt_len=8), k_tuner=tuner)
    assert rep.finished == 7
    tail = tuner.history[len(tuner.history) // 3:]
    est = sum(h[2] for h in tail) / len(tail)
    assert abs(est - p) < 0.06, est
