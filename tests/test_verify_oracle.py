"""The CPU verification oracle (oracle/verify_oracle.c), pinned without a GPU.

The reference has no token-level verification, so the oracle is pinned
against (a) an independent float64 numpy evaluation of the same rule,
(b) the distributional identity of speculative sampling (the emitted token is
distributed as p), and (c) committed regression vectors
tests/golden/verify_golden.json (tests/golden/make_verify_golden.py).
"""

import json
import math
import os

import numpy as np
import pytest

from oracle import verify as ov
from tests import _gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "verify_golden.json")


def test_canonical_exp2_accuracy_and_edges():
    assert ov.exp2(0.0) == 1.0
    assert ov.exp2(-1.0) == 0.5
    assert ov.exp2(float("-inf")) == ov.exp2(-125.0) == 2.0 ** -125
    ts = np.linspace(-125.0, 0.0, 20001, dtype=np.float32)
    got = np.array([ov.exp2(float(t)) for t in ts], dtype=np.float64)
    ref = np.exp2(ts.astype(np.float64))
    assert (np.abs(got - ref) / ref).max() < 5e-7


@pytest.mark.parametrize("n", [1, 4, 1000, 8192, 8196, 128256])
def test_row_stats_vs_float64(n):
    row = _gen.normalish(n, (n,), 3.0)
    M, S = ov.row_stats(row)
    assert M == float(row.max())
    S64 = np.exp(row.astype(np.float64) - row.max()).sum()
    assert abs(S - S64) / S64 < 1e-5


def test_greedy_matches_numpy_argmax():
    t, d, ids, ln, _ = _gen.verify_case(11, 16, 5, 3000, greedy=True)
    # force some ties at the max: lowest index must win
    t[0, 0, 7] = t[0, 0, 9] = 50.0
    acc, out = ov.verify_greedy(t, ids, ln)
    g = t.argmax(axis=2)
    for b in range(16):
        a = 0
        while a < ln[b] and ids[b, a] == g[b, a]:
            a += 1
        assert acc[b] == a
        assert list(out[b, :a]) == list(ids[b, :a])
        assert out[b, a] == g[b, a]
        assert all(x == -1 for x in out[b, a + 1:])
    assert out[0, 0] == 7 or acc[0] > 0


def test_sampling_decisions_match_float64_away_from_ties():
    B, K, V = 64, 4, 2000
    t, d, ids, ln, u = _gen.verify_case(5, B, K, V, tau=0.7)
    acc, out = ov.verify_sample(t, d, ids, ln, u)
    mism = 0
    for b in range(B):
        a = 0
        margin_ok = True
        while a < ln[b]:
            p = np.exp(t[b, a].astype(np.float64) - t[b, a].max())
            p /= p.sum()
            q = np.exp(d[b, a].astype(np.float64) - d[b, a].max())
            q /= q.sum()
            ratio = p[ids[b, a]] / q[ids[b, a]]
            if abs(u[b, a] - ratio) < 1e-4 * max(1.0, ratio):
                margin_ok = False
            if not u[b, a] < ratio:
                break
            a += 1
        if margin_ok:
            mism += int(acc[b] != a)
    assert mism == 0
    assert 0 < acc.mean() < K  # the case mixes accepts and rejects


def test_sampling_emits_target_distribution():
    """Speculative sampling is exact: the first emitted token ~ p_0."""
    N, K, V = 40000, 2, 12
    rng = np.random.default_rng(0)
    t1 = rng.normal(0, 1.0, V).astype(np.float32)
    d1 = (t1 + rng.normal(0, 1.0, V)).astype(np.float32)
    t = np.broadcast_to(t1, (N, K + 1, V)).copy()
    d = np.broadcast_to(d1, (N, K, V)).copy()
    q = np.exp(d1.astype(np.float64) - d1.max())
    q /= q.sum()
    ids = rng.choice(V, size=(N, K), p=q).astype(np.int32)
    ln = np.full(N, K, np.int32)
    u = rng.random((N, K + 1)).astype(np.float32)
    acc, out = ov.verify_sample(t, d, ids, ln, u)
    p = np.exp(t1.astype(np.float64) - t1.max())
    p /= p.sum()
    counts = np.bincount(out[:, 0], minlength=V)
    chi2 = ((counts - N * p) ** 2 / (N * p)).sum()
    # dof = 11; P(chi2 > 40) ~ 3e-5
    assert chi2 < 40.0, (chi2, counts, N * p)


def test_idle_rows_and_bonus():
    t, d, ids, ln, u = _gen.verify_case(3, 4, 3, 1000)
    ln[:] = 0
    acc, out = ov.verify_greedy(t, ids, ln)
    assert (acc == 0).all()
    assert (out[:, 0] == t[:, 0].argmax(axis=1)).all()
    assert (out[:, 1:] == -1).all()


def test_golden_vectors():
    with open(GOLDEN) as fh:
        cases = json.load(fh)
    for c in cases:
        t, d, ids, ln, u = _gen.verify_case(c["seed"], c["B"], c["K"], c["V"], c["Vd"],
                                            c["tau"], greedy=c["greedy"])
        if c["greedy"]:
            acc, out = ov.verify_greedy(t, ids, ln)
        else:
            acc, out = ov.verify_sample(t, d, ids, ln, u, c["temperature"])
        assert acc.tolist() == c["accepted_len"], c["name"]
        assert out.tolist() == c["out_tokens"], c["name"]
