"""The PSD hot path on the CPU (TEST INFRASTRUCTURE + CPU baseline arm).

``CpuBackend`` plugs the numpy forward (oracle/model.py) and the canonical
verification oracle (oracle/verify_oracle.c) into the same scheduler seam as
``GpuBackend``, with the same token routing (draft step 0 re-reads the last
two committed tokens, verify over [last, d_1..d_k]) and the same KV grant /
trim accounting, so GPU and CPU runs are comparable step for step.

Used by tests (greedy end-to-end identity), ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg, never by the product.
"""

from __future__ import annotations

import time

import numpy as np

from oracle import verify as ov
from oracle.model import OracleModel
from paper_2603_18016_b200.model import PRESETS, successor_table
from paper_2603_18016_b200.scheduler import EngineState, StepPlan, StepResult, VerifyRow
from paper_2603_18016_b200.workload import attach_prompt_ids


class CpuBackend:
    block_pool = None

    def __init__(self, target="tiny-target", draft="tiny-draft", *, seed: int = 0,
                 beta_target: float = 6.0, beta_draft: float = 12.0, max_seq_len: int = 1024,
                 mode: str = "greedy") -> None:
        if mode != "greedy":
            raise NotImplementedError("CPU oracle backend: greedy mode")
        self.tshape = PRESETS[target] if isinstance(target, str) else target
        self.dshape = PRESETS[draft] if isinstance(draft, str) else draft
        self.seed = seed
        self.t = OracleModel(self.tshape, seed * 2 + 1)
        self.d = OracleModel(self.dshape, seed * 2 + 2)
        self.succ = successor_table(self.tshape.vocab, self.dshape.vocab, seed)
        self.beta_t, self.beta_d = beta_target, beta_draft
        self.max_len = max_seq_len
        self.seq: dict[int, list[int]] = {}
        self.tc: dict[int, list] = {}
        self.dc: dict[int, list] = {}
        self.pending: dict[int, list[int]] = {}
        self.stats = {"draft_s": 0.0, "verify_s": 0.0, "prefill_s": 0.0, "steps": 0}

    def bind(self, state: EngineState) -> None:
        need = [r for r in state.requests.values() if r.prompt_ids is None]
        if need:
            attach_prompt_ids(need, self.dshape.vocab, self.seed)

    def estimate(self, state, plan):
        return 0.0, 0.0, 0.0

    def planned_commit(self, state, rid, k_i, draft_time):
        return min(k_i + 1, state.requests[rid].remaining)

    def commit(self, state, rid, tokens):
        state.kv.trim_to_written(rid)

    def retire(self, state, rid):
        req = state.requests[rid]
        seq = self.seq.pop(rid, None)
        if seq is not None:
            req.output_ids = seq[req.prompt_len:]
        self.tc.pop(rid, None)
        self.dc.pop(rid, None)
        self.pending.pop(rid, None)

    def _argmax_rows(self, logits: np.ndarray) -> np.ndarray:
        n = logits.shape[0]
        acc, out = ov.verify_greedy(logits.reshape(n, 1, -1), np.zeros((n, 0), np.int32),
                                    np.zeros(n, np.int32))
        return out[:, 0]

    def _prefill(self, state, ids):
        for rid in ids:
            p = state.requests[rid].prompt_ids
            self.seq[rid] = list(p)
            self.tc[rid] = self.t.new_cache(self.max_len)
            self.dc[rid] = self.d.new_cache(self.max_len)
        seqs = [(state.requests[rid].prompt_ids[:-1], 0) for rid in ids]
        self.t.forward(seqs, [self.tc[r] for r in ids])
        self.d.forward(seqs, [self.dc[r] for r in ids])

    def _draft(self, state, ids, quotas):
        rows = [rid for rid in ids if quotas[rid] > 0]
        for rid in ids:
            self.pending[rid] = []
        if not rows:
            return
        kmax = max(quotas[r] for r in rows)
        cur = {}
        for i in range(kmax):
            act = [r for r in rows if i < quotas[r]]
            if i == 0:
                seqs = [(self.seq[r][-2:], len(self.seq[r]) - 2) for r in act]
                h = self.d.forward(seqs, [self.dc[r] for r in act])
                last = h[1::2]
                prev = np.asarray([self.seq[r][-1] for r in act], np.int64)
            else:
                seqs = [([cur[r]], len(self.seq[r]) - 1 + i) for r in act]
                last = self.d.forward(seqs, [self.dc[r] for r in act])
                prev = np.asarray([cur[r] for r in act], np.int64)
            lg = self.d.logits(last, prev, self.succ[:self.dshape.vocab], self.beta_d)
            nxt = self._argmax_rows(lg)
            for r, t in zip(act, nxt):
                cur[r] = int(t)
                self.pending[r].append(int(t))

    def _verify(self, state, rows: list[VerifyRow]) -> dict[int, int]:
        kmax = max((r.k for r in rows), default=0)
        seqs, caches, prevs = [], [], []
        for row in rows:
            rid = row.request_id
            d = self.pending.get(rid, [])
            if len(d) != row.k:
                raise RuntimeError(f"request {rid}: {len(d)} pending drafts, verifying {row.k}")
            toks = [self.seq[rid][-1]] + d
            seqs.append((toks, len(self.seq[rid]) - 1))
            caches.append(self.tc[rid])
        h = self.t.forward(seqs, caches)
        n = len(rows)
        V = self.tshape.vocab
        logits = np.full((n, kmax + 1, V), -np.inf, np.float32)
        ids = np.zeros((n, kmax), np.int32)
        ln = np.zeros(n, np.int32)
        o = 0
        for r, (row, (toks, _)) in enumerate(zip(rows, seqs)):
            m = len(toks)
            lg = self.t.logits(h[o:o + m], np.asarray(toks, np.int64), self.succ, self.beta_t)
            logits[r, :m] = lg
            logits[r, m:] = lg[-1]  # padding rows are never read (k_b < kmax)
            ids[r, :row.k] = toks[1:]
            ln[r] = row.k
            o += m
        acc, out = ov.verify_greedy(logits, ids, ln)
        accepted = {}
        for r, row in enumerate(rows):
            a = int(acc[r])
            self.seq[row.request_id].extend(int(t) for t in out[r, :a + 1])
            self.pending.pop(row.request_id, None)
            if row.k > 0:
                accepted[row.request_id] = a
        return accepted

    def execute(self, state: EngineState, plan: StepPlan, rows: list[VerifyRow]) -> StepResult:
        t0 = time.perf_counter()
        if plan.prefill_ids:
            self._prefill(state, plan.prefill_ids)
        t1 = time.perf_counter()
        self._draft(state, plan.serial_draft_ids, plan.quotas)
        t2 = time.perf_counter()
        self._draft(state, plan.overlap_draft_ids, plan.quotas)
        t3 = time.perf_counter()
        accepted = self._verify(state, rows) if rows else {}
        t4 = time.perf_counter()
        self.stats["steps"] += 1
        self.stats["prefill_s"] += t1 - t0
        self.stats["draft_s"] += t3 - t1
        self.stats["verify_s"] += t4 - t3
        ms = lambda a, b: (b - a) * 1e3  # noqa: E731
        return StepResult(ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t0, t4), accepted)
