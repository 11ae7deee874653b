"""Capacity-bound draft selection (the set D_s of PAPER §3, TETRIS-style).

The reference always sends every drafted token and raises ``ProtocolError``
when a verify pass would exceed the verifier capacity
(engine.py:316-322, ``_check_verify_capacity``); its SPEC.md:160 names the
selection policy for a binding capacity as open.  With
``SimConfig(draft_selection="tetris")`` the scheduler instead trims each
drafted batch's per-request depths k_i so that the batch fits the capacity,
keeping the draft positions most likely to be accepted:

* position j of request i is accepted only if positions 1..j all are, so its
  value is P_i(j) = p_i ** j under a per-token acceptance probability p_i;
* the ``capacity`` positions with the largest P_i(j) are kept (ties: the
  shallower position, then the lower request id).  P_i(j) decreases in j, so
  the kept set is a prefix of every request's draft: it defines new k_i.

p_i is a Beta-smoothed running estimate from the request's own verified rows
(accepted drafts / Bernoulli trials, a rejection being one failed trial), with
the acceptance model's per-token probability as the prior mean -- requests
that have been accepting well get deeper drafts when capacity binds.
"""

from __future__ import annotations

import math

PRIOR_WEIGHT = 4.0  # pseudo-trials of the prior


class AcceptanceTracker:
    """Per-request Bernoulli-chain statistics from verified rows."""

    def __init__(self, prior: float):
        self.prior = min(max(prior, 0.05), 0.99)
        self.acc: dict[int, int] = {}
        self.trials: dict[int, int] = {}

    def observe(self, rid: int, k: int, accepted: int) -> None:
        """A verified row: ``accepted`` of ``k`` drafts (a chain stops at the
        first rejection, so trials = accepted + (accepted < k))."""
        if k <= 0:
            return
        self.acc[rid] = self.acc.get(rid, 0) + accepted
        self.trials[rid] = self.trials.get(rid, 0) + accepted + (1 if accepted < k else 0)

    def p(self, rid: int) -> float:
        a = self.acc.get(rid, 0)
        n = self.trials.get(rid, 0)
        return (a + PRIOR_WEIGHT * self.prior) / (n + PRIOR_WEIGHT)

    def forget(self, rid: int) -> None:
        self.acc.pop(rid, None)
        self.trials.pop(rid, None)


def select_depths(quotas: dict[int, int], capacity: int,
                  p: dict[int, float]) -> dict[int, int]:
    """Trim ``quotas`` (request id -> k_i) to at most ``capacity`` positions
    in total, keeping the positions with the largest p_i ** j."""
    total = sum(quotas.values())
    if total <= capacity:
        return dict(quotas)
    cand = []
    for rid, k in quotas.items():
        lp = math.log(min(max(p[rid], 1e-12), 1.0))
        for j in range(1, k + 1):
            cand.append((-j * lp, j, rid))
    cand.sort()
    kept = dict.fromkeys(quotas, 0)
    for _, j, rid in cand[:max(capacity, 0)]:
        kept[rid] = max(kept[rid], j)
    # prefix-closed by construction (scores increase with j for a request)
    return kept
