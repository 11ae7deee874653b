"""Dedicated-draft-GPU PSD with the real GPU engines, two processes on one GPU.

The driver's boxes have one GPU, so both ranks share cuda:0 and talk over gloo
(host tensors); on a multi-GPU node bench.py --layout pairs uses NCCL between
two devices with the same engines.  Output tokens must equal the
single-process GpuBackend run.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(max_requests=16, max_batch=16, k_max=4, max_seq_len=128, seed=0, beta_target=2.0,
          beta_draft=12.0, prefill_chunk_tokens=512)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg_reqs():
    from paper_2603_18016_b200 import SimConfig, make_requests
    return SimConfig(mode="psd", m=4, k=4), make_requests([9, 14, 20, 7, 12, 16, 5, 30],
                                                         prompt_len=10)


def _worker(rank, port, q, extra=None, mailbox=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.gpu import GpuBackend
    from paper_2603_18016_b200.pair import (DraftServer, GpuDraftEngine, GpuTargetEngine,
                                            PairLink, PairTarget)
    dist.init_process_group("gloo", init_method="env://")
    comm = None
    if mailbox:  # drafted ids through the peer-memory mailbox (csrc/comm.cu)
        import torch

        from paper_2603_18016_b200.comm import PeerComm
        comm = PeerComm(mbox_bytes=1 << 16, buf_bytes=1 << 12, device=torch.device("cuda:0"))
    if rank == 0:
        gb = GpuBackend("tiny-target", "tiny-draft", roles=("target",), **KW, **(extra or {}))
        be = PairTarget(GpuTargetEngine(gb), PairLink(1, comm=comm))
        cfg, reqs = _cfg_reqs()
        st, rep = run(cfg, reqs, backend=be)
        be.stop()
        q.put(("out", [r.output_ids for r in st.request_list()], rep.finished))
    else:
        gb = GpuBackend("tiny-target", "tiny-draft", roles=("draft",), **KW, **(extra or {}))
        q.put(("steps", DraftServer(GpuDraftEngine(gb), PairLink(0, comm=comm)).serve()))
    dist.destroy_process_group()


@pytest.mark.parametrize("mailbox", [False, True], ids=["dist", "peer-mailbox"])
def test_pair_gpu_engines_match_single_process(cuda_device, mailbox):
    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.gpu import GpuBackend
    cfg, reqs = _cfg_reqs()
    st, rep = run(cfg, reqs, backend=GpuBackend("tiny-target", "tiny-draft", **KW))
    ref = [r.output_ids for r in st.request_list()]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, None, mailbox)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got["out"][1] == 8
    assert got["out"][0] == ref
    assert got["steps"][0] > 0


def test_pair_gpu_sampling_ships_q_rows(cuda_device):
    """Sampling mode across the pair: the draft rank sends the draft
    distributions q of every drafted token after the ids; the target's K1
    reads them from its qbuf.  Same weights, logits and Philox uniforms on both
    sides -> token-for-token identical to the single-process sampling run."""
    from paper_2603_18016_b200 import run
    from paper_2603_18016_b200.gpu import GpuBackend
    extra = dict(mode="sample", temperature=1.0)
    cfg, reqs = _cfg_reqs()
    kw = dict(KW, beta_target=1.0, beta_draft=1.0)
    st, rep = run(cfg, reqs, backend=GpuBackend("tiny-target", "tiny-draft", **kw, **extra))
    ref = [r.output_ids for r in st.request_list()]
    assert 0 < rep.total_accepted < rep.total_drafted
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    extra_kw = dict(extra, beta_target=1.0, beta_draft=1.0)
    procs = [ctx.Process(target=_worker_kw, args=(r, port, q, extra_kw)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got["out"][1] == 8
    assert got["out"][0] == ref


def _worker_kw(rank, port, q, extra):
    """_worker with KW entries overridden by ``extra``."""
    global KW
    KW = {k: v for k, v in KW.items() if k not in extra}
    _worker(rank, port, q, extra)


def _worker_tp(rank, port, q):
    """ranks 0, 1: a tensor-parallel (TP = 2) target; rank 2: its dedicated
    draft rank -- three processes sharing cuda:0 over gloo"""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="3",
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    from paper_2603_18016_b200 import SimConfig, make_requests, run
    from paper_2603_18016_b200.gpu import GpuBackend
    from paper_2603_18016_b200.pair import (DraftServer, GpuDraftEngine, GpuTargetEngine,
                                            PairLink, PairTarget)
    dist.init_process_group("gloo", init_method="env://")
    tpg = dist.new_group([0, 1])
    kw = dict(KW, beta_target=6.0)
    cfg = SimConfig(mode="psd", m=8, k=4)
    reqs = make_requests([24] * 16, prompt_len=16)
    if rank < 2:
        gb = GpuBackend("tiny-target-tp", "tiny-draft", roles=("target",), tp=(rank, 2, tpg), **kw)
        be = PairTarget(GpuTargetEngine(gb), PairLink(2), leader=rank == 0)
        st, rep = run(cfg, reqs, backend=be)
        be.stop()
        q.put((f"out{rank}", [r.output_ids for r in st.request_list()], rep.finished,
               rep.total_accepted))
    else:
        gb = GpuBackend("tiny-target-tp", "tiny-draft", roles=("draft",), **kw)
        q.put(("steps", DraftServer(GpuDraftEngine(gb), PairLink(0),
                                    followers=(PairLink(1),)).serve()))
    dist.destroy_process_group()


def test_tp_target_with_dedicated_draft_rank(cuda_device):
    """The paper's cfg4 deployment shape: a tensor-parallel target with the
    draft on its own rank (here TP = 2 + 1 on one GPU).  Both TP ranks emit
    the tokens of the single-process unsharded run (greedy, clear margins)."""
    from paper_2603_18016_b200 import SimConfig, make_requests, run
    from paper_2603_18016_b200.gpu import GpuBackend
    st, rep = run(SimConfig(mode="psd", m=8, k=4), make_requests([24] * 16, prompt_len=16),
                  backend=GpuBackend("tiny-target-tp", "tiny-draft", **dict(KW, beta_target=6.0)))
    ref = [r.output_ids for r in st.request_list()]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tp, args=(r, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in (0, 1):
        outs, finished, accepted = got[f"out{r}"]
        assert finished == 16 and outs == ref and accepted > 0
    assert got["steps"][0] > 0
