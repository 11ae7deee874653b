"""The N>1 bench path on CPU: two gloo ranks, each an independent PSD replica
(SimBackend) on its own request shard; tokens add up, time is the max."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    from paper_2603_18016_b200 import LatencyModel, SimConfig, make_requests, run
    from paper_2603_18016_b200 import dist as pd
    pd.init("gloo")
    ids = pd.shard_requests(10, world, rank)
    reqs = make_requests([20 + 3 * i for i in ids], prompt_len=8)
    for r, i in zip(reqs, ids):
        r.id = i
    cfg = SimConfig(mode="psd", m=2, k=3, seed=5,
                    verify_latency=LatencyModel("constant", 1.0 + rank))
    st, rep = run(cfg, reqs)
    tokens, ms = pd.aggregate(rep.total_generated, float(rep.makespan))
    q.put((rank, list(ids), rep.total_generated, rep.makespan, tokens, ms))
    pd.finalize()


def test_two_gloo_replicas_shard_and_aggregate():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ids0, tok0, ms0, agg_t0, agg_m0), (r1, ids1, tok1, ms1, agg_t1, agg_m1) = out
    assert set(ids0).isdisjoint(ids1) and len(ids0) + len(ids1) == 10
    assert agg_t0 == agg_t1 == tok0 + tok1 == sum(20 + 3 * i for i in range(10))
    assert agg_m0 == agg_m1 == max(ms0, ms1)
    assert ms1 > ms0  # rank 1's slower verify shows up in the max
