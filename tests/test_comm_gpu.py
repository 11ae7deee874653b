"""Peer-memory communicator (csrc/comm.cu) with two processes sharing cuda:0.

CUDA IPC maps each rank's region into the other process, as across the GPUs
of an NVLink node.  The fused split-K + cross-rank all-reduce must equal the
same fp32 sums done in (rank, split) order, on every call (the epoch advances
on the device; CUDA-graph replays included), and the mailbox must deliver
messages in order both ways.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(rank, call, S, n):
    import torch
    g = torch.Generator().manual_seed(1000 * call + 10 * rank + S)
    return torch.randn(S, n, generator=g)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
                      RANK=str(rank), LOCAL_RANK="0")
    import torch
    import torch.distributed as dist

    from paper_2603_18016_b200.comm import PeerComm
    dist.init_process_group("gloo", init_method="env://")
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    comm = PeerComm(buf_bytes=8 << 20, mbox_bytes=1 << 16, device=dev)
    errs = []
    S, n = 3, 4096 * 12
    for call in range(6):  # both staging parities, several epochs, varying grids
        nc = n if call % 2 == 0 else 1024 + 4 * call
        mine = _data(rank, call, S, nc)
        part = mine.to(dev).contiguous()
        out = torch.empty(nc, device=dev)
        comm.allreduce_partials(part.view(-1), S, nc, nc, out)
        torch.cuda.synchronize()
        ref = None
        for r in range(2):  # ranks in order, each its splits in order
            d = _data(r, call, S, nc)
            acc = d[0].clone()
            for s in range(1, S):
                acc = acc + d[s]
            ref = acc if ref is None else ref + acc
        errs.append(bool(torch.equal(out.cpu(), ref)))
    # in place (out aliases partials), captured in a CUDA graph, replayed
    buf = torch.empty(S * n, device=dev)
    st = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        comm.allreduce_partials(buf, S, n, n, buf)
    for call in range(6, 9):
        buf.copy_(_data(rank, call, S, n).view(-1).to(dev))
        g.replay()
        torch.cuda.synchronize()
        ref = None
        for r in range(2):
            d = _data(r, call, S, n)
            acc = d[0] + d[1] + d[2]
            ref = acc if ref is None else ref + acc
        errs.append(bool(torch.equal(buf[:n].cpu(), ref)))
    # mailbox: 4 rounds each way, depth-1 flow control
    peer = 1 - rank
    got = []
    for i in range(4):
        msg = torch.arange(100, dtype=torch.int32, device=dev) + 1000 * i + 100000 * rank
        dst = torch.empty(100, dtype=torch.int32, device=dev)
        if rank == 0:
            comm.put(peer, msg)
            comm.get(peer, dst)
        else:
            comm.get(peer, dst)
            comm.put(peer, msg)
        torch.cuda.synchronize()
        exp = torch.arange(100, dtype=torch.int32) + 1000 * i + 100000 * peer
        got.append(bool(torch.equal(dst.cpu(), exp)))
    dist.barrier()
    comm.close()
    dist.destroy_process_group()
    q.put((rank, errs, got))


def test_peer_allreduce_and_mailbox(cuda_device):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, errs, got in res:
        assert all(errs), (rank, errs)
        assert all(got), (rank, got)


def test_local_group_allreduce_gather_mailbox(cuda_device):
    """Two ranks driven by one process on one GPU (psd_comm_create_local), each
    on its own stream so their kernels run concurrently: the same protocol as
    across GPUs, without relying on time slicing between processes."""
    import torch

    from paper_2603_18016_b200.comm import PeerComm
    dev = cuda_device
    comms = PeerComm.local_group([dev, dev], buf_bytes=4 << 20, mbox_bytes=1 << 16)
    streams = [torch.cuda.Stream(dev) for _ in comms]
    S, n = 3, 4096 * 10

    def both(fn):
        torch.cuda.synchronize()
        for r, (c, st) in enumerate(zip(comms, streams)):
            with torch.cuda.stream(st):
                fn(r, c)
        torch.cuda.synchronize()

    for call in range(6):  # varying sizes: the per-call grid changes
        nc = n if call % 2 == 0 else 1024 + 4 * call
        parts = [_data(r, call, S, nc).to(dev) for r in range(2)]
        outs = [torch.empty(nc, device=dev) for _ in range(2)]
        both(lambda r, c: c.allreduce_partials(parts[r].view(-1), S, nc, nc, outs[r]))
        ref = None
        for r in range(2):
            d = _data(r, call, S, nc)
            acc = d[0] + d[1] + d[2]
            ref = acc if ref is None else ref + acc
        for r in range(2):
            assert torch.equal(outs[r].cpu(), ref), (call, r)
    # all-gather
    src = [torch.randn(n, device=dev) for _ in range(2)]
    gat = [torch.empty(2 * n, device=dev) for _ in range(2)]
    both(lambda r, c: c.allgather(src[r], gat[r]))
    for r in range(2):
        assert torch.equal(gat[r].view(2, n)[0], src[0]) and torch.equal(gat[r].view(2, n)[1],
                                                                         src[1])
    # mailbox, both directions, several rounds
    for i in range(3):
        msg = [torch.arange(64, dtype=torch.int32, device=dev) + 1000 * i + 7 * r
               for r in range(2)]
        dst = [torch.empty(64, dtype=torch.int32, device=dev) for _ in range(2)]

        def xchg(r, c):
            c.put(1 - r, msg[r])
            c.get(1 - r, dst[r])
        both(xchg)
        for r in range(2):
            assert torch.equal(dst[r], msg[1 - r])
    for c in comms:
        c.close()
