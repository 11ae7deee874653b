"""Tensor-parallel target (SURVEY.md §8e, cfg4's TP=4) at TP = 2 on one GPU.

Two processes share cuda:0 over gloo (the driver's boxes have one GPU; on a
node the same code runs one rank per GPU over NCCL).  Column-parallel QKV and
gate/up, row-parallel O and down with an all-reduce, vocab-parallel LM head
with an all-gather:
* the sharded verify forward's logits equal the unsharded model's within the
  north-star tolerance (rtol 1e-2 on logits);
* greedy PSD through GpuBackend(tp=...) emits the same tokens as the
  single-process run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(max_requests=16, max_batch=16, k_max=4, max_seq_len=128, seed=0, beta_target=4.0,
          beta_draft=12.0, prefill_chunk_tokens=512, use_graphs=False, fused_draft=False)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _logits(model_tp, seed=3, splits_hint=0):
    """One prefill + logits of every prompt token through Forward."""
    from paper_2603_18016_b200.model import PRESETS, Forward, Transformer
    dev = torch.device("cuda:0")
    shape = PRESETS["tiny-target-tp"]
    m = Transformer(shape, dev, seed=seed, num_blocks=16, block_size=16, max_blocks_per_seq=8,
                    tp=model_tp)
    bt = torch.zeros(4, 8, dtype=torch.int32, device=dev)
    bt[0, :4] = torch.tensor([1, 2, 3, 4])
    bt[1, :4] = torch.tensor([5, 6, 7, 8])
    fwd = Forward(m, 128, 8, 64, bt)
    fwd.splits_hint = splits_hint
    rng = np.random.default_rng(0)
    lens = [23, 40]
    toks = [rng.integers(0, shape.vocab, n).tolist() for n in lens]
    flat = np.concatenate(toks).astype(np.int32)
    pos = np.concatenate([np.arange(n) for n in lens]).astype(np.int32)
    slots = np.concatenate([
        np.asarray([bt[s, p // 16].item() * 16 + p % 16 for p in range(n)])
        for s, n in enumerate(lens)]).astype(np.int32)
    fwd.begin()
    fwd.stage(0, {"tokens": flat, "positions": pos, "slots": slots,
                  "seq_slot": np.asarray([0, 1], np.int32),
                  "q_start": np.asarray([0, lens[0]], np.int32),
                  "q_len": np.asarray(lens, np.int32), "q_pos0": np.zeros(2, np.int32),
                  "kv_len": np.asarray(lens, np.int32),
                  "logit_rows": np.arange(sum(lens), dtype=np.int32)})
    fwd.upload(1)
    logits = torch.empty(sum(lens), shape.vocab, dtype=torch.float32, device=dev)
    fwd.run(sum(lens), 2, max(lens), sum(lens), logits, shape.vocab)
    torch.cuda.synchronize()
    return logits.cpu().numpy()


def _worker(rank, port, q, transport="peer", graphs=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2",
                      RANK=str(rank), LOCAL_RANK=str(rank), PSD_TP_COMM=transport)
    import torch.distributed as dist

    from paper_2603_18016_b200 import SimConfig, make_requests, run
    from paper_2603_18016_b200.gpu import GpuBackend
    dist.init_process_group("gloo", init_method="env://")
    group = dist.group.WORLD
    lg = _logits((rank, 2, group))
    gb = GpuBackend("tiny-target-tp", "tiny-draft", tp=(rank, 2, group),
                    **dict(KW, use_graphs=graphs))
    cfg = SimConfig(mode="psd", m=8, k=4)
    st, rep = run(cfg, make_requests([24] * 16, prompt_len=16), backend=gb)
    q.put((rank, lg, [r.output_ids for r in st.request_list()], rep.finished))
    dist.destroy_process_group()


@pytest.mark.parametrize("transport,graphs", [("peer", False), ("peer", True), ("dist", False)],
                         ids=["peer", "peer-graphs", "torch-dist"])
def test_tp2_target_matches_unsharded(cuda_device, transport, graphs):
    """peer: C2 all-reduce and the C3 greedy shard partials over CUDA-IPC peer
    memory (csrc/comm.cu), also inside CUDA graphs; torch-dist: all-reduce /
    all-gather through torch.distributed."""
    from tests._parity import noise_floor_ok
    from paper_2603_18016_b200 import SimConfig, make_requests, run
    from paper_2603_18016_b200.gpu import GpuBackend
    ref_logits = _logits(None)
    # the unsharded model's own reordering noise: another valid split-K count
    alt_logits = _logits(None, splits_hint=1)
    st, rep = run(SimConfig(mode="psd", m=8, k=4), make_requests([24] * 16, prompt_len=16),
                  backend=GpuBackend("tiny-target-tp", "tiny-draft", **KW))
    ref = [r.output_ids for r in st.request_list()]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, transport, graphs))
             for r in range(2)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in (0, 1):
        lg, outs, finished = got[r]
        # the sharded forward sums in another order (rank slices, then ranks);
        # it must sit within the unsharded model's own reordering noise floor
        ok, info = noise_floor_ok(lg, ref_logits, alt_logits)
        assert ok, info
        assert finished == 16
        assert outs == ref
