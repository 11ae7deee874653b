"""Online draft-depth tuner.

The reference models the draft depth trade-off in closed form
(pkg/src/specsim/analytic.py:1-20, 181-216): drafting time t buys acceptance
f(t); serial SD pays draft + verify per round, batch-parallel SD hides drafting
up to the verification time, so its optimum sits at drafting time ==
verify_time.  The reference evaluates that model offline; the paper shows the
best k is workload dependent and non-monotone.

``KTuner`` closes the loop at run time, from the step log the scheduler
already produces (``StepRecord``, request_model.py:185-199):

* per-token acceptance p: the mean accepted count per verified row a at depth k
  inverts the chain law of acceptance_model.py:82-97,
  E[a | k] = p (1 - p^k) / (1 - p);
* per-draft-step time d = draft_ms / k and verification time V = verify_ms, as
  exponential moving averages of the measured (CUDA-event) durations;
* the next depth maximises expected committed tokens per row per unit time
  over the integers 1..k_max (the discrete form of the reference's frontier
  optimum):  psd: (E[a|k] + 1) / max(V, k d);  standard-sd: (E[a|k] + 1) /
  (k d + V).

It only sets the depth the scheduler drafts (``_quota``); acceptance, KV
accounting and the step protocol are unchanged, so a run without a tuner is
byte-identical to the reference.
"""

from __future__ import annotations

from .records import StepRecord

__all__ = ["KTuner", "expected_chain_accepts", "invert_chain_accepts", "invert_chain_accepts_rows"]


def expected_chain_accepts(p: float, k: int) -> float:
    """E[accepted | depth k] under a per-token acceptance probability p."""
    if k <= 0:
        return 0.0
    if p >= 1.0:
        return float(k)
    return p * (1.0 - p ** k) / (1.0 - p)


def invert_chain_accepts(a: float, k: float) -> float:
    """p in [0, 1] with expected_chain_accepts(p, k) == a (bisection; the
    expectation is increasing in p)."""
    if k <= 0 or a <= 0.0:
        return 0.0
    if a >= k:
        return 1.0
    lo, hi = 0.0, 1.0
    kk = max(1, int(round(k)))
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if expected_chain_accepts(mid, kk) < a:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def invert_chain_accepts_rows(pairs) -> float:
    """p with sum_i E[a | k_i, p] == sum_i a_i over verified rows (k_i, a_i),
    k_i > 0 (bisection; every term is increasing in p)."""
    total = sum(a for _, a in pairs)
    if total <= 0:
        return 0.0
    if total >= sum(k for k, _ in pairs):
        return 1.0
    lo, hi = 0.0, 1.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if sum(expected_chain_accepts(mid, k) for k, _ in pairs) < total:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


class KTuner:
    """Chooses the draft depth between steps from measured acceptance and
    timings.  ``k`` is the depth to draft next; ``history`` records (step,
    k, p, d, V) after every update."""

    def __init__(self, k_max: int, mode: str = "psd", k_min: int = 1, warmup: int = 3,
                 ema: float = 0.25, k0: int | None = None) -> None:
        if k_max < k_min or k_min < 1:
            raise ValueError("need 1 <= k_min <= k_max")
        if mode not in ("psd", "standard-sd"):
            raise ValueError(f"unknown mode {mode!r}")
        self.k_max, self.k_min, self.mode = k_max, k_min, mode
        self.warmup, self.ema = warmup, ema
        self.k = k0 if k0 is not None else k_max
        self.p = self.d = self.v = None
        self.seen = 0
        self.history: list[tuple[int, int, float, float, float]] = []

    def _avg(self, old, new):
        return new if old is None else (1.0 - self.ema) * old + self.ema * new

    def observe(self, rec: StepRecord, verified=None, draft_steps: int | None = None) -> None:
        """``verified``: the step's verified rows as (k_i, accepted) -- in PSD
        they were drafted one step earlier, possibly at another depth and batch
        size than this step's drafts, so acceptance is estimated from them
        alone (rows with k_i = 0 are idle passes and carry no information).
        ``draft_steps``: sequential draft steps behind ``rec.draft_duration``
        (a startup step drafts two batches).  Without them (a bare StepRecord)
        the record's aggregate counts are used."""
        steps = draft_steps if draft_steps else self.k
        if rec.draft_duration > 0.0 and steps > 0:
            self.d = self._avg(self.d, rec.draft_duration / steps)
        if verified is not None:
            pairs = [(k, a) for k, a in verified if k > 0]
            if not pairs:
                return
            p = invert_chain_accepts_rows(pairs)
        else:
            rows = rec.bonus_tokens  # exactly one bonus per verified row
            if rows <= 0 or rec.drafted_tokens <= 0:
                return
            p = invert_chain_accepts(rec.accepted_tokens / rows, rec.drafted_tokens / rows)
        self.p = self._avg(self.p, p)
        if rec.verify_duration > 0.0:
            self.v = self._avg(self.v, rec.verify_duration)
        self.seen += 1
        if self.seen >= self.warmup and self.d and self.v:
            self.k = self.best_k(self.p, self.d, self.v)
        self.history.append((rec.step_index, self.k, self.p,
                             self.d or 0.0, self.v or 0.0))

    def rate(self, k: int, p: float, d: float, v: float) -> float:
        """Expected committed tokens per row per unit time at depth k."""
        tokens = expected_chain_accepts(p, k) + 1.0
        t = max(v, k * d) if self.mode == "psd" else k * d + v
        return tokens / t if t > 0.0 else 0.0

    def best_k(self, p: float, d: float, v: float) -> int:
        best, best_rate = self.k_min, -1.0
        for k in range(self.k_min, self.k_max + 1):
            r = self.rate(k, p, d, v)
            if r > best_rate * (1.0 + 1e-12):
                best, best_rate = k, r
        return best
