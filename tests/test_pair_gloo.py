"""Dedicated-draft-GPU PSD protocol (pair.py) on CPU over gloo.

Rank 0 runs the scheduler + target model, rank 1 the draft model; the numpy
oracle engines stand in for the GPU engines.  The two-rank run must produce
exactly the token sequences and step log of the single-process CPU PSD.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

KW = dict(target="tiny-target", draft="tiny-draft", seed=0, beta_target=1.0, beta_draft=12.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg_reqs():
    from paper_2603_18016_b200 import SimConfig, make_requests
    return SimConfig(mode="psd", m=3, k=4), make_requests([9, 14, 20, 7, 12, 16, 5], prompt_len=6)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from oracle.pair_cpu import CpuDraftEngine, CpuTargetEngine
    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.pair import DraftServer, PairLink, PairTarget
    dist.init_process_group("gloo", init_method="env://")
    if rank == 0:
        be = PairTarget(CpuTargetEngine(**KW), PairLink(1))
        cfg, reqs = _cfg_reqs()
        st, rep = run(cfg, reqs, backend=be)
        be.stop()
        q.put(("out", [r.output_ids for r in st.request_list()],
               [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in st.step_log],
               be.link.bytes_sent, be.link.bytes_recv))
    else:
        steps = DraftServer(CpuDraftEngine(**KW), PairLink(0)).serve()
        q.put(("steps", steps))
    dist.destroy_process_group()


def test_pair_protocol_matches_single_process():
    from oracle.psd_cpu import CpuBackend
    from paper_2603_18016_b200 import run
    cfg, reqs = _cfg_reqs()
    st, rep = run(cfg, reqs, backend=CpuBackend(**KW))
    ref_out = [r.output_ids for r in st.request_list()]
    ref_log = [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in st.step_log]

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out, log, sent, recvd = got["out"]
    assert out == ref_out
    assert log == ref_log
    assert got["steps"][0] == len(ref_log)
    assert sent > 0 and recvd > 0


def _worker_group(rank, port, q, world):
    """ranks 0..world-2: one target group (SPMD scheduler; rank 0 leads), the
    last rank: the dedicated draft rank serving all of them"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from oracle.pair_cpu import CpuDraftEngine, CpuTargetEngine
    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.pair import DraftServer, PairLink, PairTarget
    dist.init_process_group("gloo", init_method="env://")
    d = world - 1
    if rank < d:
        be = PairTarget(CpuTargetEngine(**KW), PairLink(d), leader=rank == 0)
        cfg, reqs = _cfg_reqs()
        st, rep = run(cfg, reqs, backend=be)
        be.stop()
        q.put((f"out{rank}", [r.output_ids for r in st.request_list()],
               [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in st.step_log]))
    else:
        steps = DraftServer(CpuDraftEngine(**KW), PairLink(0),
                            followers=tuple(PairLink(r) for r in range(1, d))).serve()
        q.put(("steps", steps))
    dist.destroy_process_group()


def test_target_group_with_dedicated_draft_rank():
    """The tensor-parallel target + dedicated draft GPU layout's protocol (2
    target ranks, one draft rank): every target rank gets the same drafts and
    emits the single-process tokens and step log."""
    from oracle.psd_cpu import CpuBackend
    from paper_2603_18016_b200 import run
    cfg, reqs = _cfg_reqs()
    st, rep = run(cfg, reqs, backend=CpuBackend(**KW))
    ref_out = [r.output_ids for r in st.request_list()]
    ref_log = [(s.drafted_tokens, s.accepted_tokens, s.bonus_tokens) for s in st.step_log]
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_group, args=(r, port, q, world)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world - 1):
        out, log = got[f"out{r}"]
        assert out == ref_out and log == ref_log
    assert got["steps"][0] == len(ref_log)
