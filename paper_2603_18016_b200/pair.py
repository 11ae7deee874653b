"""PSD with a dedicated draft GPU: target rank + draft rank over torch.distributed.

The paper's deployment: the drafter runs on its own
GPU, the verifier on another; drafts cross to the verifier and sampler
outputs flow back, "one exchange step per PSD step".  The
reference only charges this hand-off as ``comm_overhead`` (engine.py:439, 442).

Rank ``t`` (even) runs the scheduler and the target model; rank ``t+1`` runs
the draft model and serves commands.  Per PSD step, one message goes
target -> draft (new admissions with prompts, KV block tables, the tokens
committed by the previous verification, the rows to draft serially / overlapped)
and one or two replies come back (draft ids).  The overlapped batch is
drafted on the draft GPU *while* the target GPU verifies the other batch --
the overlap the reference only models as max(verify, draft).

The protocol is engine-agnostic: ``GpuTargetEngine`` / ``GpuDraftEngine``
wrap :class:`~.gpu.GpuBackend` (roles "target" / "draft"); the CPU tests
(tests/test_pair_gloo.py) plug the numpy oracle engines into the same classes
over gloo.  Transport = ``dist.send``/``recv``.  The command message is a
small int32 array the draft rank's host decodes; the drafted ids (and, when
sampling, the q rows) stay on the devices under NCCL: the draft rank gathers
them into one int32 buffer on its GPU and sends it without a host sync; the
target rank receives into a device buffer and scatters it into its slot
table with a kernel (``psd_index_copy_i32``), stream-ordered before the
verification that reads them.  Each id message carries, in its last element,
the draft rank's CUDA-event time of its previous draft phase (µs), so no host
ever waits for a draft to finish just to time it.  Under gloo the same
buffers travel through host memory.
"""

from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist

from .scheduler import EngineState, StepPlan, StepResult, VerifyRow
from .workload import attach_prompt_ids

__all__ = ["PairLink", "PairTarget", "DraftServer", "GpuTargetEngine", "GpuDraftEngine"]

MAGIC = 0x50534450  # "PSDP"
K_STEP, K_STOP = 0, 1


class PairLink:
    """Length-prefixed int32 messages to / from one peer rank."""

    def __init__(self, peer: int, device=None, comm=None, comm_peer: int | None = None) -> None:
        self.peer = peer
        self.device = device  # CUDA device for NCCL, None for gloo
        # comm (a comm.PeerComm over the pair, or over a target group + its
        # draft rank): drafted ids go through its device mailbox over NVLink
        # peer memory (psd_p2p_put/get_i32) instead of dist.send / recv;
        # commands and q rows still use dist.  comm_peer: the peer's rank in
        # the comm (default: the other rank of a 2-rank comm)
        self.comm = comm
        self.comm_peer = (1 - comm.rank if comm is not None and comm_peer is None else comm_peer)
        self.bytes_sent = 0
        self.bytes_recv = 0

    def _t(self, arr: np.ndarray) -> torch.Tensor:
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32))
        return t.to(self.device) if self.device is not None else t

    def send(self, arr: np.ndarray) -> None:
        arr = np.asarray(arr, dtype=np.int32)
        dist.send(self._t(np.asarray([arr.size], np.int32)), self.peer)
        if arr.size:
            dist.send(self._t(arr), self.peer)
        self.bytes_sent += 4 * (arr.size + 1)

    def send_rows(self, rows: torch.Tensor) -> None:
        """fp32 [n, V] rows (the draft distributions q), device to device on
        NCCL, through the host on gloo."""
        t = rows if self.device is not None else rows.cpu()
        dist.send(t.contiguous(), self.peer)
        self.bytes_sent += t.numel() * 4

    def recv_rows(self, n: int, v: int, device) -> torch.Tensor:
        buf = torch.empty(n, v, dtype=torch.float32,
                          device=self.device if self.device is not None else "cpu")
        dist.recv(buf, self.peer)
        self.bytes_recv += buf.numel() * 4
        return buf if device is None else buf.to(device, non_blocking=True)

    def send_ids(self, ids) -> None:
        """Flat int32 ids (device tensor under NCCL, else host) as one message."""
        t = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(ids, dtype=np.int32))
        if self.comm is not None:
            self.comm.put(self.comm_peer, t.to(self.comm.device).contiguous())
            self.bytes_sent += 4 * t.numel()
            return
        if self.device is None:
            t = t.cpu()
        elif not t.is_cuda:
            t = t.to(self.device)
        dist.send(t.contiguous(), self.peer)
        self.bytes_sent += 4 * t.numel()

    def recv_ids(self, n: int) -> torch.Tensor:
        """n int32 (device tensor under NCCL / the peer mailbox, host under
        gloo); no host sync."""
        if self.comm is not None:
            buf = torch.empty(n, dtype=torch.int32, device=self.comm.device)
            self.comm.get(self.comm_peer, buf)
            self.bytes_recv += 4 * n
            return buf
        buf = torch.empty(n, dtype=torch.int32,
                          device=self.device if self.device is not None else "cpu")
        dist.recv(buf, self.peer)
        self.bytes_recv += 4 * n
        return buf

    def recv(self) -> np.ndarray:
        hdr = self._t(np.zeros(1, np.int32))
        dist.recv(hdr, self.peer)
        n = int(hdr.cpu()[0])
        if n == 0:
            return np.zeros(0, np.int32)
        buf = self._t(np.zeros(n, np.int32))
        dist.recv(buf, self.peer)
        self.bytes_recv += 4 * (n + 1)
        return buf.cpu().numpy()


# ---------------------------------------------------------------------------
# message codec
# ---------------------------------------------------------------------------
def encode_step(admit, commits, serial, overlap, table) -> np.ndarray:
    """admit: [(rid, slot, prompt)]; commits: [(rid, slot, tokens)];
    serial / overlap: [(rid, slot, L, k)]; table: int32 [slots, max_blocks]."""
    out = [MAGIC, K_STEP, len(admit), len(commits), len(serial), len(overlap),
           table.shape[0], table.shape[1]]
    for rid, slot, prompt in admit:
        out += [rid, slot, len(prompt)] + list(prompt)
    for rid, slot, toks in commits:
        out += [rid, slot, len(toks)] + list(toks)
    for rows in (serial, overlap):
        for r in rows:
            out += list(r)
    return np.concatenate([np.asarray(out, np.int32), table.reshape(-1).astype(np.int32)])


def decode_step(msg: np.ndarray) -> dict:
    if msg[0] != MAGIC:
        raise RuntimeError("PSD pair protocol: bad message")
    kind = int(msg[1])
    if kind == K_STOP:
        return {"stop": True}
    na, nc, ns, no, tr, tc = (int(x) for x in msg[2:8])
    i = 8
    admit, commits = [], []
    for _ in range(na):
        rid, slot, n = (int(x) for x in msg[i:i + 3])
        admit.append((rid, slot, msg[i + 3:i + 3 + n].tolist()))
        i += 3 + n
    for _ in range(nc):
        rid, slot, n = (int(x) for x in msg[i:i + 3])
        commits.append((rid, slot, msg[i + 3:i + 3 + n].tolist()))
        i += 3 + n
    serial = [tuple(int(x) for x in msg[i + 4 * j:i + 4 * j + 4]) for j in range(ns)]
    i += 4 * ns
    overlap = [tuple(int(x) for x in msg[i + 4 * j:i + 4 * j + 4]) for j in range(no)]
    i += 4 * no
    table = msg[i:i + tr * tc].reshape(tr, tc)
    return {"stop": False, "admit": admit, "commits": commits, "serial": serial,
            "overlap": overlap, "table": table}


def split_ids(rows, flat) -> dict:
    """{rid: [ids]} from a flat id array in row order (rows: (rid, slot, L, k))."""
    out, i = {}, 0
    for rid, _, _, k in rows:
        out[rid] = [int(x) for x in flat[i:i + k]]
        i += k
    return out


# ---------------------------------------------------------------------------
# protocol roles
# ---------------------------------------------------------------------------
class PairTarget:
    """Scheduler backend on the target rank (Backend protocol).

    A tensor-parallel target (the paper's TP target + a dedicated
    draft GPU) runs one PairTarget per TP rank, all driving the same SPMD
    scheduler: the leader (TP rank 0) sends the commands, every rank receives
    the drafted ids (and q rows) -- each verifies with them."""

    def __init__(self, engine, link: PairLink, leader: bool = True) -> None:
        self.engine = engine
        self.link = link
        self.leader = leader
        self.block_pool = getattr(engine, "block_pool", None)
        self.pending_commits: list = []
        self.stats = {"draft_ms": 0.0, "verify_ms": 0.0, "prefill_ms": 0.0, "steps": 0,
                      "wait_ms": 0.0}

    def bind(self, state: EngineState) -> None:
        # commits of a previous run target slots / request ids of that run
        self.pending_commits = []
        self.engine.bind(state)

    def estimate(self, state, plan):
        return 0.0, 0.0, 0.0

    def planned_commit(self, state, rid, k_i, draft_time):
        return min(k_i + 1, state.requests[rid].remaining)

    def commit(self, state, rid, tokens):
        state.kv.trim_to_written(rid)

    def retire(self, state, rid):
        self.engine.retire(state, rid)

    def execute(self, state: EngineState, plan: StepPlan, rows: list[VerifyRow]) -> StepResult:
        eng = self.engine
        t0 = time.perf_counter()
        admit = eng.admit(state, plan.prefill_ids)
        table = eng.tables(state)

        def draft_rows(ids):
            out = []
            for rid in ids:
                k = plan.quotas[rid]
                eng.expect_drafts(rid, k)
                if k > 0:
                    req = state.requests[rid]
                    out.append((rid, eng.slot_of(rid), req.prompt_len + req.generated, k))
            return out

        serial = draft_rows(plan.serial_draft_ids)
        overlap = draft_rows(plan.overlap_draft_ids)
        if self.leader:
            self.link.send(encode_step(admit, self.pending_commits, serial, overlap, table))
        self.pending_commits = []
        eng.prefill(state, plan.prefill_ids)
        t1 = time.perf_counter()
        serial_ms = self._take_drafts(serial)
        t2 = time.perf_counter()
        accepted, committed, verify_ms = eng.verify(state, rows) if rows else ({}, {}, 0.0)
        t3 = time.perf_counter()
        overlap_ms = self._take_drafts(overlap)
        t4 = time.perf_counter()
        for rid, toks in committed.items():
            self.pending_commits.append((rid, eng.slot_of(rid), toks))
        ms = lambda a, b: (b - a) * 1e3  # noqa: E731
        self.stats["steps"] += 1
        self.stats["draft_ms"] += serial_ms + overlap_ms
        self.stats["verify_ms"] += verify_ms
        self.stats["prefill_ms"] += ms(t0, t1)
        self.stats["wait_ms"] += ms(t1, t2) + ms(t3, t4)
        return StepResult(ms(t0, t1), serial_ms, overlap_ms, verify_ms, ms(t0, t4), accepted)

    def _take_drafts(self, rows) -> float:
        """Receive one phase's drafted ids (+ q rows when sampling) and hand
        them to the engine; returns the draft time that message reports (the
        draft rank's previous phase, CUDA events, ms).  Nothing here waits on
        the host: the ids land in a device buffer the engine scatters from."""
        if not rows:
            return 0.0
        n = sum(r[3] for r in rows)
        msg = self.link.recv_ids(n + 1)
        self.engine.inject_ids(rows, msg[:n])
        self._recv_q(rows)
        ms = 0.0
        prev = getattr(self, "_prev_msg", None)
        if prev is not None:  # long complete: read without stalling
            ms = int(prev[-1]) / 1000.0
        self._prev_msg = msg
        return ms

    def _recv_q(self, rows) -> None:
        """Sampling mode: the draft distributions of the drafted tokens follow
        the draft ids (one [sum k, V_draft + 4] fp32 message, rows in draft
        order, each row's canonical (max, sum) in columns V, V + 1)."""
        vq = getattr(self.engine, "q_vocab", 0)
        if not vq:
            return
        n = sum(r[3] for r in rows)
        if n:
            # each row carries its canonical (max, sum) in two extra columns
            self.engine.inject_q(rows, self.link.recv_rows(n, vq + 4, self.engine.device))

    def stop(self) -> None:
        """End of a run: the draft rank answers with the time of its last
        draft phase (the one no id message reported)."""
        self.pending_commits = []
        if self.leader:
            self.link.send(np.asarray([MAGIC, K_STOP], np.int32))
        last = self.link.recv()
        self.stats["draft_ms"] += int(last[0]) / 1000.0 if last.size else 0.0
        self._prev_msg = None


class DraftServer:
    """Command loop on the draft rank.  ``link`` reaches the target rank that
    sends the commands; ``followers`` (the other ranks of a tensor-parallel
    target) receive the same drafted ids / q rows and the stop reply."""

    def __init__(self, engine, link: PairLink, followers: tuple = ()) -> None:
        self.engine = engine
        self.link = link
        self.followers = tuple(followers)
        self.steps = 0

    def serve(self) -> int:
        eng = self.engine
        prev_us = 0  # CUDA-event time of the previous draft phase
        pending = None  # (start, end) events of the phase in flight
        while True:
            cmd = decode_step(self.link.recv())
            if pending is not None:
                prev_us = _elapsed_us(*pending)
                pending = None
            if cmd["stop"]:
                for lk in (self.link,) + self.followers:
                    lk.send(np.asarray([prev_us], np.int32))
                return self.steps
            eng.set_tables(cmd["table"])
            eng.commit(cmd["commits"])  # before admissions: a freed slot may be reused
            eng.admit(cmd["admit"])
            eng.prefill(cmd["admit"])
            for rows in (cmd["serial"], cmd["overlap"]):
                if rows:
                    if pending is not None:
                        prev_us = _elapsed_us(*pending)
                    ids, pending = eng.draft(rows, prev_us)
                    q = eng.q_rows(rows) if getattr(eng, "q_vocab", 0) else None
                    for lk in (self.link,) + self.followers:
                        lk.send_ids(ids)
                        if q is not None and q.shape[0]:
                            lk.send_rows(q)
            self.steps += 1


def _elapsed_us(e0, e1) -> int:
    """Microseconds between two recorded events (CUDA events, or host
    perf_counter floats for the CPU engines)."""
    if isinstance(e0, float):
        return int((e1 - e0) * 1e6)
    e1.synchronize()
    return int(e0.elapsed_time(e1) * 1000)


# ---------------------------------------------------------------------------
# GPU engines (GpuBackend with one role each)
# ---------------------------------------------------------------------------
class GpuTargetEngine:
    """Target half of :class:`~.gpu.GpuBackend` behind the pair protocol."""

    def __init__(self, backend) -> None:
        self.be = backend
        self.block_pool = backend.block_pool
        self.last2: dict[int, tuple[int, int]] = {}

    def bind(self, state):
        self.be.bind(state)

    def slot_of(self, rid):
        return self.be.slots[rid]

    def admit(self, state, ids):
        be = self.be
        with torch.cuda.stream(be.s_target):
            be._admit(state, ids)
        out = []
        for rid in ids:
            p = state.requests[rid].prompt_ids
            self.last2[rid] = (p[-2], p[-1])
            out.append((rid, be.slots[rid], list(p)))
        return out

    def tables(self, state):
        be = self.be
        with torch.cuda.stream(be.s_target):
            be._upload_block_table(state)
        return be.bt_np.copy()

    def expect_drafts(self, rid, k):
        self.be.pending_k[rid] = k

    def prefill(self, state, ids):
        be = self.be
        if ids:
            with torch.cuda.stream(be.s_target):
                be._prefill(state, ids, be.tfwd, "target")

    def inject_ids(self, rows, ids: torch.Tensor) -> None:
        """Drafted ids (flat, row order; device buffer under NCCL) ->
        slot_tok[slot, 2 + i] by one scatter kernel on the target stream."""
        be = self.be
        dst = []
        for rid, slot, _, k in rows:
            dst += [slot * be.ldt + 2 + i for i in range(k)]
        if not dst:
            return
        idx = torch.from_numpy(np.asarray(dst, np.int32)).pin_memory()
        # the ids arrived in the current stream's order (NCCL recv / host)
        be.s_target.wait_stream(torch.cuda.current_stream(be.device))
        with torch.cuda.stream(be.s_target):
            idx_d = idx.to(be.device, non_blocking=True)
            src = ids.to(be.device, non_blocking=True) if not ids.is_cuda else ids
            from . import native
            native.check(native.load().psd_index_copy_i32(
                be.slot_tok.data_ptr(), idx_d.data_ptr(), src.data_ptr(), None, len(dst),
                torch.cuda.current_stream(be.device).cuda_stream), "draft ids in")
            be.launches += 1
            be.h2d_bytes += 4 * len(dst) * (1 if ids.is_cuda else 2)
            src.record_stream(be.s_target)
            idx_d.record_stream(be.s_target)

    @property
    def q_vocab(self) -> int:
        return self.be.dshape.vocab if self.be.mode == "sample" else 0

    @property
    def device(self):
        return self.be.device

    def inject_q(self, rows, q: torch.Tensor) -> None:
        """q rows in draft order -> qbuf[slot * k_max + i] (what K1 reads);
        their canonical (max, sum), the last two columns -> qstats, so K1
        takes the cached-statistics path as in a single process."""
        be = self.be
        dst = []
        for rid, slot, _, k in rows:
            dst += [slot * be.k_max + i for i in range(k)]
        idx = torch.from_numpy(np.asarray(dst, np.int32)).pin_memory()
        # q arrived in the current stream's order (NCCL recv / host copy)
        be.s_target.wait_stream(torch.cuda.current_stream(be.device))
        with torch.cuda.stream(be.s_target):
            idx_d = idx.to(be.device, non_blocking=True)
            from . import native
            V = be.dshape.vocab
            native.check(native.load().psd_copy_rows_f32(
                be.qbuf.data_ptr(), idx_d.data_ptr(), V, q.data_ptr(), V + 4, len(dst), V,
                torch.cuda.current_stream(be.device).cuda_stream), "q rows in")
            be.qstats.index_copy_(0, idx_d.long(), q[:, V:V + 2])
            be.qstats_remote = True
            q.record_stream(be.s_target)

    def verify(self, state, rows):
        be = self.be
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(be.s_target):
            ev0.record()
            n = be._verify(state, rows)
            ev1.record()
        ev1.synchronize()
        acc = be.acc_host.numpy()[:n]
        out = be.out_host.numpy()
        K1 = be.k_max + 1  # every verify pass is k_max + 1 tokens wide (GpuBackend._verify)
        accepted, committed = {}, {}
        for r, row in enumerate(rows):
            a = int(acc[r])
            toks = out[r * K1:r * K1 + a + 1].tolist()
            committed[row.request_id] = toks
            if row.k > 0:
                accepted[row.request_id] = a
            be.pending_k.pop(row.request_id, None)
        return accepted, committed, ev0.elapsed_time(ev1)

    def retire(self, state, rid):
        self.be.retire(state, rid)
        self.last2.pop(rid, None)


class GpuDraftEngine:
    """Draft half of :class:`~.gpu.GpuBackend` behind the pair protocol."""

    def __init__(self, backend) -> None:
        self.be = backend
        self.last2: dict[int, tuple[int, int]] = {}

    def set_tables(self, table):
        be = self.be
        be.bt_np[:] = table
        be.nblk[:] = (table != 0).sum(axis=1)
        be.nblk[be.scratch_slot] = 1
        be.block_table.copy_(be.block_table_host, non_blocking=True)

    def admit(self, rows):
        for rid, slot, prompt in rows:
            self.last2[rid] = (prompt[-2], prompt[-1])
        self.be._init_slots([(slot, p[-2], p[-1]) for _, slot, p in rows])

    def commit(self, rows):
        triples = []
        for rid, slot, toks in rows:
            prev = self.last2.get(rid, (0, 0))
            seq = [prev[1]] + list(toks)
            self.last2[rid] = (seq[-2], seq[-1])
            triples.append((slot, seq[-2], seq[-1]))
        self.be._init_slots(triples)

    def prefill(self, rows):
        if rows:
            self.be._prefill_rows([(slot, p) for _, slot, p in rows], self.be.dfwd)

    def draft(self, rows, prev_us: int):
        """Draft `rows` on this GPU; returns (message, events): the drafted
        ids gathered from slot_tok in row order plus `prev_us` as the last
        element, one device int32 buffer ready to send, and the CUDA events
        bracketing this phase.  No host synchronisation."""
        be = self.be
        dev = be.device
        src = []
        for rid, slot, _, k in rows:
            src += [slot * be.ldt + 2 + i for i in range(k)]
        n = len(src)
        host = torch.from_numpy(np.asarray(src + [prev_us], np.int32)).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        be._draft_rows(rows)
        e1.record()
        hd = host.to(dev, non_blocking=True)
        be.h2d_bytes += 4 * (n + 1)
        msg = torch.empty(n + 1, dtype=torch.int32, device=dev)
        from . import native
        st = torch.cuda.current_stream(dev).cuda_stream
        native.check(native.load().psd_index_copy_i32(msg.data_ptr(), None, be.slot_tok.data_ptr(),
                                                      hd.data_ptr(), n, st), "draft ids out")
        be.launches += 1
        msg[n:].copy_(hd[n:])
        return msg, (e0, e1)

    @property
    def q_vocab(self) -> int:
        return self.be.dshape.vocab if self.be.mode == "sample" else 0

    def q_rows(self, rows) -> torch.Tensor:
        """Sampling mode: the q rows of the drafted tokens, packed in draft
        order ([sum k, V_draft + 4] fp32 on the draft GPU, statistics after the row)."""
        be = self.be
        src = []
        for _, slot, _, k in rows:
            src += [slot * be.k_max + i for i in range(k)]
        V = be.dshape.vocab
        # [sum k, V + 4]: the q row, its canonical (max, sum) from the sampler,
        # two pad columns (rows stay 16-byte aligned for the vector copies)
        out = torch.zeros(len(src), V + 4, dtype=torch.float32, device=be.device)
        if src:
            from . import native
            idx = torch.from_numpy(np.asarray(src, np.int32)).to(be.device)
            native.check(native.load().psd_gather_rows_f32(
                out.data_ptr(), V + 4, be.qbuf.data_ptr(), idx.data_ptr(), V, len(src), V,
                torch.cuda.current_stream(be.device).cuda_stream), "q rows out")
            out[:, V:V + 2] = be.qstats.index_select(0, idx.long())
            torch.cuda.current_stream(be.device).synchronize()
        return out
