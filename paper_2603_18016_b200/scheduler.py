"""The two-batch PSD scheduler and the sequential-SD baseline.

This is the host side of the hot path.  It keeps the reference engine's
semantics and entry points (pkg/src/specsim/engine.py) and replaces the two
abstractions the reference simulates -- pass durations and coin-flip
acceptance -- with a pluggable :class:`Backend`:

* :class:`~.sim.SimBackend` evaluates the reference's latency models and
  acceptance streams, so a run is byte-identical to ``specsim``
  (tests/test_scheduler_parity.py).
* :class:`~.gpu.GpuBackend` runs the draft model's k-step decode loop on one
  CUDA stream while the target model verifies the other batch on another
  (or on a dedicated draft GPU), and takes accepted lengths from the fused
  verification kernel.

Reference map (engine.py):
  ``PendingDraft`` :51-57, ``KvStepRecord`` :60-68, ``FinishRecord`` :71-79,
  ``EngineState`` :82-103, admission :118-152, draft quota :155-159,
  planned commit :162-175, allocations :178-217, prefill commit :220-224,
  verification :227-265, finish :268-289, preemption :292-313, capacity
  :316-322, PSD step :325-477 (startup / overlap / fallback branches at
  350/374/388, timing 435-442, sync-point order 451-463), SD step :480-548,
  ``step_once`` :551-559, ``new_state`` :562-581, ``run`` :584-604.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Protocol

from .batches import BatchManager
from .errors import CapacityError, ProtocolError
from .kvtable import ALLOCATE, AllocationContext, KVBlockTable
from .metrics import MetricsReport, compute_metrics
from .selection import AcceptanceTracker, select_depths
from .records import (TERMINAL_STATES, Request, RequestState, SimConfig, StepRecord,
                      validate_config)

__all__ = [
    "Backend",
    "EngineState",
    "FinishRecord",
    "KvStepRecord",
    "PendingDraft",
    "Preemption",
    "StepPlan",
    "StepResult",
    "VerifyRow",
    "new_state",
    "run",
    "step_once",
]


# ---------------------------------------------------------------------------
# records
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Preemption:
    """Evict ``request_index`` at the first sync point at or after ``time``."""

    request_index: int
    time: float


@dataclass(frozen=True)
class PendingDraft:
    """Drafted tokens awaiting verification and the time spent drafting."""

    tokens: int
    draft_time: float


@dataclass(frozen=True)
class KvStepRecord:
    step_index: int
    allocated_ids: tuple[int, ...]
    skipped_ids: tuple[int, ...]
    blocks_in_use: int


@dataclass(frozen=True)
class FinishRecord:
    request_id: int
    finish_time: float
    blocks_at_finish: int
    prompt_len: int
    total_len: int


@dataclass(frozen=True)
class VerifyRow:
    """One row of a verification pass: ``k`` drafted tokens (0 = idle pass),
    verification index ``j`` (1-based, per request)."""

    request_id: int
    k: int
    draft_time: float
    j: int


@dataclass
class StepPlan:
    """Everything a backend must execute for one step.

    ``branch`` is "startup", "overlap", "fallback" or "sd".
    ``serial_draft_ids`` are drafted before verification starts (the startup
    target batch, the fallback batch, the SD batch); ``overlap_draft_ids`` are
    drafted concurrently with verification (the skip batch).  ``quotas`` maps
    every drafted request to its k_i.
    """

    step_index: int
    branch: str
    prefill_ids: tuple[int, ...]
    serial_draft_ids: tuple[int, ...]
    overlap_draft_ids: tuple[int, ...]
    verify_ids: tuple[int, ...]
    quotas: dict[int, int]
    comm_overhead: float = 0.0


@dataclass
class StepResult:
    """What a backend reports back: durations and accepted counts per
    verified row (requests with ``k == 0`` need no entry)."""

    prefill_duration: float
    serial_draft_duration: float
    overlap_draft_duration: float
    verify_duration: float
    step_duration: float
    accepted: dict[int, int]


class Backend(Protocol):
    """The seam between the scheduler and whatever executes the passes."""

    def bind(self, state: "EngineState") -> None: ...

    def estimate(self, state: "EngineState", plan: StepPlan) -> tuple[float, float, float]:
        """(prefill, serial draft, overlap draft) durations known *before*
        execution; they become the ``draft_time`` of this step's drafts."""

    def planned_commit(self, state: "EngineState", rid: int, k_i: int,
                       draft_time: float) -> int:
        """Tokens to reserve KV room for ahead of the next commit."""

    def execute(self, state: "EngineState", plan: StepPlan,
                rows: list[VerifyRow]) -> StepResult: ...

    def commit(self, state: "EngineState", rid: int, tokens: int) -> None:
        """Called after ``tokens`` were committed for ``rid``."""

    def retire(self, state: "EngineState", rid: int) -> None:
        """A request left the engine (finished or preempted)."""


# ---------------------------------------------------------------------------
# state
# ---------------------------------------------------------------------------
@dataclass
class EngineState:
    config: SimConfig
    requests: dict[int, Request]
    waiting: list[int]
    bm: BatchManager
    kv: KVBlockTable
    clock: float = 0.0
    step_index: int = 0
    pending: dict[int, dict[int, PendingDraft]] = field(
        default_factory=lambda: {0: {}, 1: {}})
    verify_counts: dict[int, int] = field(default_factory=dict)
    newly_admitted: list[int] = field(default_factory=list)
    preemptions: list[Preemption] = field(default_factory=list)
    step_log: list[StepRecord] = field(default_factory=list)
    kv_log: list[KvStepRecord] = field(default_factory=list)
    finish_log: list[FinishRecord] = field(default_factory=list)
    sd_members: dict[int, None] = field(default_factory=dict)
    backend: Backend | None = None
    k_tuner: object | None = None  # ktune.KTuner: online draft depth (None = config.k)
    # the last step's verified rows as (k_i, accepted) and its sequential draft
    # steps (sum over its draft loops of max k_i): what the tuner observes
    last_verified: list[tuple[int, int]] = field(default_factory=list)
    last_draft_steps: int = 0
    # selection.AcceptanceTracker when config.draft_selection == "tetris"
    acceptance_tracker: object | None = None

    def request_list(self) -> list[Request]:
        return [self.requests[rid] for rid in sorted(self.requests)]


def _live(state: EngineState) -> bool:
    return any(r.state not in TERMINAL_STATES for r in state.requests.values())


# ---------------------------------------------------------------------------
# admission
# ---------------------------------------------------------------------------
def _arrivals(state: EngineState) -> list[int]:
    now = state.clock
    return [rid for rid in state.waiting if state.requests[rid].arrival_time <= now]


def _enter(state: EngineState, rid: int, batch_id: int) -> None:
    req = state.requests[rid]
    req.batch_id = batch_id
    req.transition(RequestState.PREFILL)
    state.waiting.remove(rid)
    state.newly_admitted.append(rid)


def _admit(state: EngineState, psd: bool) -> None:
    """FIFO admission; stops at the first request that does not fit."""
    cap = state.config.m * state.config.sd_batch_factor
    for rid in _arrivals(state):
        if psd:
            try:
                batch_id = state.bm.assign(rid)
            except CapacityError:
                break
        else:
            if len(state.sd_members) >= cap:
                break
            state.sd_members[rid] = None
            batch_id = 0
        _enter(state, rid, batch_id)


def _ensure_admission(state: EngineState, running: int, psd: bool) -> None:
    if running or state.newly_admitted:
        return
    if not state.waiting:
        raise ProtocolError("engine stepped with no runnable requests")
    first = min(state.requests[rid].arrival_time for rid in state.waiting)
    state.clock = max(state.clock, first)
    _admit(state, psd)
    if not state.newly_admitted:
        raise ProtocolError("no request could be admitted to an empty engine")


# ---------------------------------------------------------------------------
# per-request helpers
# ---------------------------------------------------------------------------
def _quota(state: EngineState, rid: int) -> int:
    """k_i = min(configured depth, remaining - 1): the commit (accepted + one
    bonus) can never overshoot the output budget."""
    left = state.requests[rid].remaining - 1
    depth = state.config.draft_len(rid)
    if state.k_tuner is not None and not state.config.k_overrides:
        depth = min(depth, state.k_tuner.k)
    return min(depth, left if left > 0 else 0)


def _select(state: EngineState, quotas: dict[int, int], groups, capacity: int) -> dict[int, int]:
    """draft_selection "tetris": trim each group's depths to ``capacity``
    (selection.select_depths); "all" keeps them (over-capacity then fails in
    _check_capacity as in the reference)."""
    if state.config.draft_selection != "tetris":
        return quotas
    tr = state.acceptance_tracker
    if tr is None:
        tr = state.acceptance_tracker = AcceptanceTracker(
            state.config.acceptance.token_probability(0.0))
    out = dict(quotas)
    for g in groups:
        if g:
            sub = {rid: quotas[rid] for rid in g}
            out.update(select_depths(sub, capacity, {rid: tr.p(rid) for rid in g}))
    return out


def _grow(state: EngineState, ctx: AllocationContext,
          sizing: dict[int, tuple[int, float]],
          decisions: dict[int, str] | None = None) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """Apply the growth decisions; each grant covers the next commit."""
    cfg = state.config
    backend = state.backend
    if decisions is None:
        decisions = state.kv.schedule_allocation(ctx)
    granted: list[int] = []
    skipped: list[int] = []
    for rid, what in decisions.items():
        if what != ALLOCATE:
            skipped.append(rid)
            continue
        granted.append(rid)
        if cfg.kv_policy == "eager":
            k_i, dt = sizing.get(rid, (_quota(state, rid), 0.0))
        elif rid in sizing:
            k_i, dt = sizing[rid]
        elif rid in ctx.prefill_ids:
            k_i, dt = 0, 0.0  # admitted straight into the verified batch
        else:
            raise ProtocolError(
                f"request {rid} granted block growth outside any draft/verify role")
        req = state.requests[rid]
        need = backend.planned_commit(state, rid, k_i, dt)
        state.kv.ensure_capacity(rid, req.prompt_len + req.generated + need)
    return tuple(granted), tuple(skipped)


def _write_prompts(state: EngineState, prefill_ids: tuple[int, ...]) -> None:
    for rid in prefill_ids:
        req = state.requests[rid]
        state.kv.commit_write(rid, req.prompt_len)
        req.transition(RequestState.DECODING)


def _verify_rows(state: EngineState, ids: list[int],
                 drafts: dict[int, PendingDraft]) -> list[VerifyRow]:
    """Pop each row's pending draft and assign its verification index."""
    rows = []
    for rid in ids:
        pend = drafts.pop(rid, None)
        j = state.verify_counts.get(rid, 0) + 1
        state.verify_counts[rid] = j
        rows.append(VerifyRow(rid, pend.tokens if pend else 0,
                              pend.draft_time if pend else 0.0, j))
    return rows


def _commit_rows(state: EngineState, rows: list[VerifyRow],
                 accepted: dict[int, int]) -> tuple[int, int, list[int]]:
    """Commit accepted + bonus per row; returns (accepted, bonus, finished)."""
    acc_total = bonus_total = 0
    finished: list[int] = []
    state.last_verified = []
    for row in rows:
        req = state.requests[row.request_id]
        a = accepted.get(row.request_id, 0) if row.k > 0 else 0
        state.last_verified.append((row.k, a))
        if state.acceptance_tracker is not None:
            state.acceptance_tracker.observe(row.request_id, row.k, a)
        commit = min(a + 1, req.remaining)
        req.generated += commit
        state.kv.commit_write(row.request_id, commit)
        state.backend.commit(state, row.request_id, commit)
        kept = min(a, commit)
        acc_total += kept
        bonus_total += commit - kept
        if req.remaining == 0:
            finished.append(row.request_id)
    return acc_total, bonus_total, finished


def _finish(state: EngineState, finished: list[int], psd: bool) -> None:
    for rid in finished:
        req = state.requests[rid]
        state.finish_log.append(FinishRecord(
            request_id=rid, finish_time=state.clock,
            blocks_at_finish=state.kv.allocated_of(rid), prompt_len=req.prompt_len,
            total_len=req.prompt_len + req.target_output_len))
        req.finish_time = state.clock
        req.transition(RequestState.FINISHED)
        if psd:
            state.pending[state.bm.recycle(rid)].pop(rid, None)
        else:
            del state.sd_members[rid]
        state.kv.release(rid)
        state.backend.retire(state, rid)


def _preempt(state: EngineState, psd: bool) -> int:
    """Apply due injections to DECODING requests; others are dropped."""
    due = [p for p in state.preemptions if p.time <= state.clock]
    state.preemptions = [p for p in state.preemptions if p.time > state.clock]
    applied = 0
    for pre in due:
        req = state.requests.get(pre.request_index)
        if req is None or req.state is not RequestState.DECODING:
            continue
        if psd:
            state.pending[state.bm.recycle(req.id)].pop(req.id, None)
        else:
            state.sd_members.pop(req.id, None)
        req.batch_id = None
        req.transition(RequestState.PREEMPTED)
        state.kv.release(req.id)
        state.backend.retire(state, req.id)
        applied += 1
    return applied


def _check_capacity(cfg: SimConfig, tokens: int, scale: int = 1) -> None:
    cap = cfg.effective_capacity * scale
    if tokens > cap:
        raise ProtocolError(f"verifier capacity exceeded: {tokens} drafted tokens in "
                            f"one pass, capacity {cap}")


# ---------------------------------------------------------------------------
# the steps
# ---------------------------------------------------------------------------
def _psd_step(state: EngineState) -> StepRecord:
    cfg = state.config
    bm = state.bm
    backend = state.backend
    _ensure_admission(state, bm.size_of(0) + bm.size_of(1), psd=True)

    step_index = state.step_index + 1
    prefill_ids = tuple(state.newly_admitted)
    state.newly_admitted = []
    target, skip = bm.target_batch, bm.skip_batch
    target_ids, skip_ids = bm.members_of(target), bm.members_of(skip)

    if not bm.first_step_done and target_ids and skip_ids:
        # bootstrap: draft the target batch serially, then verify it while
        # the skip batch drafts for the first time
        branch = "startup"
        serial, overlap = tuple(target_ids), tuple(skip_ids)
        verify_ids = target_ids
    elif state.pending[target]:
        branch = "overlap"
        serial, overlap = (), tuple(skip_ids)
        verify_ids = target_ids
    else:
        if cfg.mode == "psd-fallback-disabled":
            raise ProtocolError(f"step {step_index}: target batch {target} has no "
                                "pre-drafted tokens and fallback is disabled")
        if state.pending[0] or state.pending[1]:
            raise ProtocolError("stale pending drafts at fallback entry")
        branch = "fallback"
        eff = target_ids if target_ids else skip_ids
        serial, overlap = tuple(eff), ()
        verify_ids = eff
    record_target = target if (branch != "fallback" or target_ids) else skip

    quotas = {rid: _quota(state, rid) for rid in serial + overlap}
    # each drafted group is verified as one pass: fit it to the capacity
    quotas = _select(state, quotas, (serial, overlap), cfg.effective_capacity)
    state.last_draft_steps = (max((quotas[r] for r in serial), default=0)
                              + max((quotas[r] for r in overlap), default=0))
    plan = StepPlan(step_index, branch, prefill_ids, serial, overlap,
                    tuple(verify_ids), quotas, cfg.comm_overhead)
    prefill_est, serial_est, overlap_est = backend.estimate(state, plan)

    draft_info = {rid: (quotas[rid], serial_est) for rid in serial}
    draft_info.update({rid: (quotas[rid], overlap_est) for rid in overlap})
    if branch == "overlap":
        verify_drafts = state.pending[target]
    else:
        verify_drafts = {rid: PendingDraft(*draft_info[rid]) for rid in verify_ids}

    ctx = AllocationContext(
        prefill_ids=prefill_ids,
        decode_ids=tuple(bm.members_of(0) + bm.members_of(1)),
        draft_batch_ids=frozenset(draft_info),
        batch_sizes=(bm.size_of(0), bm.size_of(1)))
    sizing = dict(draft_info)
    for rid, pend in verify_drafts.items():
        sizing.setdefault(rid, (pend.tokens, pend.draft_time))
    granted, skipped = _grow(state, ctx, sizing)
    _write_prompts(state, prefill_ids)

    _check_capacity(cfg, sum(d.tokens for d in verify_drafts.values()))
    rows = _verify_rows(state, verify_ids, verify_drafts)
    result = backend.execute(state, plan, rows)
    accepted, bonus, finished = _commit_rows(state, rows, result.accepted)

    if branch != "fallback":
        # only the skip batch's fresh drafts pend (startup: the target
        # batch's drafts were just consumed)
        for rid in skip_ids:
            if rid not in finished:
                state.pending[skip][rid] = PendingDraft(quotas[rid],
                                                        result.overlap_draft_duration)

    state.clock += result.step_duration
    state.kv_log.append(KvStepRecord(step_index, granted, skipped,
                                     state.kv.total_blocks_in_use))
    _finish(state, finished, psd=True)
    _preempt(state, psd=True)
    bm.alternate_skip()
    _admit(state, psd=True)

    return StepRecord(
        step_index=step_index,
        target_batch=record_target,
        draft_batch=skip if branch != "fallback" else record_target,
        drafted_tokens=sum(quotas.values()),
        accepted_tokens=accepted,
        bonus_tokens=bonus,
        draft_duration=result.serial_draft_duration + result.overlap_draft_duration,
        verify_duration=result.verify_duration,
        prefill_duration=result.prefill_duration,
        step_duration=result.step_duration,
        fallback=branch == "fallback")


def _sd_step(state: EngineState) -> StepRecord:
    cfg = state.config
    backend = state.backend
    _ensure_admission(state, len(state.sd_members), psd=False)

    step_index = state.step_index + 1
    prefill_ids = tuple(state.newly_admitted)
    state.newly_admitted = []
    ids = list(state.sd_members)
    quotas = {rid: _quota(state, rid) for rid in ids}
    quotas = _select(state, quotas, (tuple(ids),),
                     cfg.effective_capacity * cfg.sd_batch_factor)
    state.last_draft_steps = max(quotas.values(), default=0)
    plan = StepPlan(step_index, "sd", prefill_ids, tuple(ids), (), tuple(ids), quotas)
    _, serial_est, _ = backend.estimate(state, plan)

    drafts = {rid: PendingDraft(quotas[rid], serial_est) for rid in ids}
    ctx = AllocationContext(prefill_ids=prefill_ids, decode_ids=tuple(ids),
                            draft_batch_ids=frozenset(ids), batch_sizes=(len(ids), 0))
    decisions = dict.fromkeys(prefill_ids + tuple(ids), ALLOCATE)
    sizing = {rid: (d.tokens, d.draft_time) for rid, d in drafts.items()}
    # SD sizes every grant from this step's own drafts (prefill-only rows: 0)
    for rid in decisions:
        sizing.setdefault(rid, (0, 0.0))
    granted, _ = _grow(state, ctx, sizing, decisions)
    _write_prompts(state, prefill_ids)

    tokens = sum(quotas.values())
    _check_capacity(cfg, tokens, scale=cfg.sd_batch_factor)
    rows = _verify_rows(state, ids, drafts)
    result = backend.execute(state, plan, rows)
    accepted, bonus, finished = _commit_rows(state, rows, result.accepted)

    state.clock += result.step_duration
    state.kv_log.append(KvStepRecord(step_index, granted, (),
                                     state.kv.total_blocks_in_use))
    _finish(state, finished, psd=False)
    _preempt(state, psd=False)
    _admit(state, psd=False)

    return StepRecord(
        step_index=step_index, target_batch=None, draft_batch=None,
        drafted_tokens=tokens, accepted_tokens=accepted, bonus_tokens=bonus,
        draft_duration=result.serial_draft_duration,
        verify_duration=result.verify_duration,
        prefill_duration=result.prefill_duration,
        step_duration=result.step_duration, fallback=False)


# ---------------------------------------------------------------------------
# public entry points
# ---------------------------------------------------------------------------
def step_once(state: EngineState, config: SimConfig | None = None) -> StepRecord:
    """Advance one step and append it to the step log."""
    if config is not None and config is not state.config:
        state.config = validate_config(config)
    rec = _sd_step(state) if state.config.mode == "standard-sd" else _psd_step(state)
    state.step_log.append(rec)
    state.step_index = rec.step_index
    if state.k_tuner is not None:
        state.k_tuner.observe(rec, verified=state.last_verified,
                              draft_steps=state.last_draft_steps)
    return rec


def new_state(config: SimConfig, workload: list[Request],
              backend: Backend | None = None) -> EngineState:
    """Fresh engine state over ``workload`` (every request WAITING)."""
    config = validate_config(config)
    requests: dict[int, Request] = {}
    for req in workload:
        if req.id in requests:
            raise ProtocolError(f"duplicate request id {req.id}")
        if req.state is not RequestState.WAITING:
            raise ProtocolError(f"request {req.id} must start in the waiting state")
        requests[req.id] = req
    if not requests:
        raise ProtocolError("workload is empty")
    if backend is None:
        from .sim import SimBackend
        backend = SimBackend()
    order = sorted(requests, key=lambda rid: (requests[rid].arrival_time, rid))
    state = EngineState(
        config=config, requests=requests, waiting=order,
        bm=BatchManager(config.m, config.assign_policy),
        kv=KVBlockTable(config.block_size, config.kv_policy,
                        pool=getattr(backend, "block_pool", None)),
        backend=backend)
    backend.bind(state)
    return state


def run(config: SimConfig, workload: list[Request],
        preemptions: list[Preemption] | None = None, max_steps: int = 5_000_000,
        backend: Backend | None = None, k_tuner=None) -> tuple[EngineState, MetricsReport]:
    """Run to completion; returns the final state and its metrics.  ``k_tuner``
    (ktune.KTuner) picks the draft depth online (<= config.k) from the step log."""
    state = new_state(config, workload, backend)
    state.k_tuner = k_tuner
    if preemptions:
        for pre in preemptions:
            if pre.request_index not in state.requests:
                raise ProtocolError(
                    f"preemption targets unknown request {pre.request_index}")
        state.preemptions = sorted(preemptions, key=lambda p: (p.time, p.request_index))
    while _live(state):
        step_once(state)
        if state.step_index >= max_steps:
            raise ProtocolError(f"exceeded {max_steps} steps without finishing")
    return state, compute_metrics(state.step_log, state.request_list(), state.kv_log)
