"""CPU engines for the dedicated-draft-GPU protocol (TEST INFRASTRUCTURE ONLY).

They plug the numpy oracle models (oracle/psd_cpu.py) into
paper_2603_18016_b200.pair.PairTarget / DraftServer so the two-rank protocol
is exercised end to end on CPU over gloo (tests/test_pair_gloo.py).
"""

from __future__ import annotations

import time

import numpy as np

from oracle.psd_cpu import CpuBackend
from paper_2603_18016_b200.scheduler import VerifyRow


class CpuTargetEngine:
    block_pool = None

    def __init__(self, **kw) -> None:
        self.cb = CpuBackend(**kw)
        self.slots: dict[int, int] = {}

    def bind(self, state):
        self.cb.bind(state)

    def slot_of(self, rid):
        return self.slots[rid]

    def admit(self, state, ids):
        out = []
        for rid in ids:
            self.slots[rid] = len(self.slots)
            out.append((rid, self.slots[rid], list(state.requests[rid].prompt_ids)))
        return out

    def tables(self, state):
        return np.zeros((1, 1), np.int32)

    def expect_drafts(self, rid, k):
        self.cb.pending[rid] = []

    def prefill(self, state, ids):
        if ids:
            cb = self.cb
            for rid in ids:
                p = state.requests[rid].prompt_ids
                cb.seq[rid] = list(p)
                cb.tc[rid] = cb.t.new_cache(cb.max_len)
            cb.t.forward([(state.requests[rid].prompt_ids[:-1], 0) for rid in ids],
                         [cb.tc[r] for r in ids])

    def inject_ids(self, rows, ids):
        """Flat drafted ids in row order (rows: (rid, slot, L, k))."""
        ids = [int(x) for x in ids]
        i = 0
        for rid, _, _, k in rows:
            self.cb.pending[rid] = ids[i:i + k]
            i += k

    def verify(self, state, rows: list[VerifyRow]):
        t0 = time.perf_counter()
        before = {r.request_id: len(self.cb.seq[r.request_id]) for r in rows}
        accepted = self.cb._verify(state, rows)
        committed = {rid: self.cb.seq[rid][n:] for rid, n in before.items()}
        return accepted, committed, (time.perf_counter() - t0) * 1e3

    def retire(self, state, rid):
        self.cb.retire(state, rid)


class CpuDraftEngine:
    def __init__(self, **kw) -> None:
        self.cb = CpuBackend(**kw)

    def set_tables(self, table):
        pass

    def commit(self, rows):
        for rid, _, toks in rows:
            if rid in self.cb.seq:
                self.cb.seq[rid].extend(toks)

    def admit(self, rows):
        for rid, _, prompt in rows:
            self.cb.seq[rid] = list(prompt)
            self.cb.dc[rid] = self.cb.d.new_cache(self.cb.max_len)

    def prefill(self, rows):
        if rows:
            self.cb.d.forward([(p[:-1], 0) for _, _, p in rows], [self.cb.dc[r] for r, _, _ in rows])

    def draft(self, rows, prev_us: int):
        """(flat ids in row order + prev_us, (start, end) host times)."""
        for rid, _, L, _ in rows:
            assert len(self.cb.seq[rid]) == L, (rid, len(self.cb.seq[rid]), L)
        t0 = time.perf_counter()
        self.cb._draft(None, [r[0] for r in rows], {r[0]: r[3] for r in rows})
        flat = [t for r in rows for t in self.cb.pending[r[0]]]
        return np.asarray(flat + [prev_us], np.int32), (t0, time.perf_counter())
