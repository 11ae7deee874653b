"""Multi-GPU plumbing: one process per GPU, independent PSD replicas.

PSD shards by request: each rank serves its own requests with
its own draft + target models, so the data path has no collective.  The only
cross-rank traffic is timing / accounting after the measured region (max of
the per-rank device times, sum of tokens) -- done here so the same code runs
on NCCL (GPU ranks) and on gloo (CPU tests, tests/test_dist_gloo.py).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist

__all__ = ["env", "init", "shard_requests", "aggregate", "finalize"]


def env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str = "nccl") -> tuple[int, int, int]:
    world, rank, local = env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, init_method="env://")
    return world, rank, local


def shard_requests(n_total: int, world: int, rank: int) -> range:
    """Contiguous request-id range of a rank (ids stay globally unique)."""
    per = (n_total + world - 1) // world
    return range(rank * per, min(n_total, (rank + 1) * per))


def aggregate(tokens: int, ms: float, device=None) -> tuple[int, float]:
    """(sum of tokens, max of device ms) over ranks; identity when world == 1."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return tokens, ms
    if dist.get_backend() == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(tokens), ms], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    tok = t[:1].clone()
    tm = t[1:].clone()
    dist.all_reduce(tok, op=dist.ReduceOp.SUM)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    return int(tok.item()), float(tm.item())


def finalize() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()
