"""Virtual-time backend: the reference's latency and acceptance models.

With this backend the scheduler reproduces ``specsim`` exactly -- the parity
harness (tests/test_scheduler_parity.py) checks step logs, KV logs, finish logs
and metrics byte-for-byte against fixtures produced by the reference.

Reference behaviour restated here:
  * prefill charged as ``verify_latency(prompt_tokens, n)`` (engine.py:335-338)
  * draft durations per batch (engine.py:359-360, 378, 402, 496)
  * verify duration from the drafted tokens (engine.py:429, 518)
  * step time: startup = prefill + d_target + comm + max(v, d_skip) + comm;
    overlap = prefill + max(v, d_skip) + comm; fallback / SD = prefill + d + v
    (engine.py:435-442, 522)
  * exact-commit KV sizing by peeking the acceptance stream; ``eager``
    reserves k_i + 1 (engine.py:162-175)
  * acceptance = leading run of ``u < q`` on stream (seed, rid, j)
    (engine.py:250-256; acceptance_model.py:82-97)
"""

from __future__ import annotations

from .acceptance import acceptance_stream, accepted_count
from .scheduler import EngineState, StepPlan, StepResult, VerifyRow

__all__ = ["SimBackend"]


class SimBackend:
    """Latency-model timing + coin-flip acceptance (no device work)."""

    block_pool = None

    def bind(self, state: EngineState) -> None:
        self._state = state

    def _draft_time(self, state: EngineState, ids: tuple[int, ...],
                    quotas: dict[int, int]) -> float:
        return state.config.draft_latency.duration(sum(quotas[r] for r in ids), len(ids))

    def estimate(self, state: EngineState, plan: StepPlan) -> tuple[float, float, float]:
        prompt = sum(state.requests[r].prompt_len for r in plan.prefill_ids)
        prefill = state.config.verify_latency.duration(prompt, len(plan.prefill_ids))
        return (prefill, self._draft_time(state, plan.serial_draft_ids, plan.quotas),
                self._draft_time(state, plan.overlap_draft_ids, plan.quotas))

    def planned_commit(self, state: EngineState, rid: int, k_i: int,
                       draft_time: float) -> int:
        cfg = state.config
        left = state.requests[rid].remaining
        if cfg.kv_policy == "eager":
            return min(k_i + 1, left)
        a = 0
        if k_i > 0:
            j = state.verify_counts.get(rid, 0) + 1
            a = accepted_count(cfg.acceptance, k_i, draft_time,
                               acceptance_stream(cfg.seed, rid, j))
        return min(a + 1, left)

    def execute(self, state: EngineState, plan: StepPlan,
                rows: list[VerifyRow]) -> StepResult:
        cfg = state.config
        prefill, serial, overlap = self.estimate(state, plan)
        verify = cfg.verify_latency.duration(sum(r.k for r in rows), len(rows))
        accepted = {
            r.request_id: accepted_count(cfg.acceptance, r.k, r.draft_time,
                                         acceptance_stream(cfg.seed, r.request_id, r.j))
            for r in rows if r.k > 0
        }
        comm = plan.comm_overhead
        if plan.branch in ("fallback", "sd"):
            step = prefill + serial + verify
        elif plan.branch == "startup":
            step = prefill + serial + comm + max(verify, overlap) + comm
        else:
            step = prefill + max(verify, overlap) + comm
        return StepResult(prefill, serial, overlap, verify, step, accepted)

    def commit(self, state: EngineState, rid: int, tokens: int) -> None:
        pass

    def retire(self, state: EngineState, rid: int) -> None:
        pass
