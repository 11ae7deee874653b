"""Paged KV-cache accounting, deferred-growth policy and the physical block pool.

The accounting and the policy follow pkg/src/specsim/kv_manager.py:
  * ``blocks_needed`` = ceil(tokens / block_size) ........... :31-37
  * ``AllocationContext`` .................................... :40-54
  * deferred decision rule (``has_deferred``, ``empty_batch_seen``,
    degradation on the second empty-batch sighting) ......... :80-112
  * ``ensure_capacity`` never shrinks ........................ :114-128
  * ``commit_write`` overrun check ........................... :130-144
  * ``release`` .............................................. :146-153

B200 additions (not in the reference):
  * an optional :class:`BlockPool` of physical block ids.  When attached, every
    request owns an ordered list of physical blocks that mirrors its allocated
    block count; the GPU backend uploads these lists as the device block table
    read by the paged attention / KV-append kernels.
  * :meth:`KVBlockTable.trim_to_written`: a real GPU cannot peek the next
    acceptance, so it grants the worst case (k_i + 1 positions) before verify
    and gives back the blocks past the committed length afterwards.  That
    keeps the reference invariant "blocks at finish = ceil(total / B)".
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import KVError

__all__ = ["ALLOCATE", "SKIP", "AllocationContext", "BlockPool", "KVBlockTable",
           "blocks_needed"]

ALLOCATE = "allocate"
SKIP = "skip"


def blocks_needed(tokens: int, block_size: int) -> int:
    """Number of ``block_size``-token blocks that hold ``tokens`` tokens."""
    if tokens < 0:
        raise ValueError(f"tokens must be nonnegative, got {tokens}")
    if block_size <= 0:
        raise ValueError(f"block size must be positive, got {block_size}")
    return (tokens + block_size - 1) // block_size


@dataclass(frozen=True)
class AllocationContext:
    """What the growth scheduler sees at the start of a step.

    ``prefill_ids``: prompts written this step; ``decode_ids``: running
    requests of both batches (new admissions appear in both tuples);
    ``draft_batch_ids``: requests drafted for this step; ``batch_sizes``:
    current sizes of batches 0 and 1.
    """

    prefill_ids: tuple[int, ...]
    decode_ids: tuple[int, ...]
    draft_batch_ids: frozenset[int]
    batch_sizes: tuple[int, int]


class BlockPool:
    """LIFO free list of physical KV block ids ``0 .. num_blocks-1``."""

    def __init__(self, num_blocks: int) -> None:
        if num_blocks <= 0:
            raise KVError(f"block pool needs at least one block, got {num_blocks}")
        self.num_blocks = num_blocks
        self._free = list(range(num_blocks - 1, -1, -1))

    @property
    def free_count(self) -> int:
        return len(self._free)

    def take(self, n: int) -> list[int]:
        if n > len(self._free):
            raise KVError(f"KV block pool exhausted: need {n}, {len(self._free)} free "
                          f"of {self.num_blocks}")
        out = self._free[len(self._free) - n:][::-1]
        del self._free[len(self._free) - n:]
        return out

    def give(self, blocks: list[int]) -> None:
        self._free.extend(reversed(blocks))


class KVBlockTable:
    def __init__(self, block_size: int, policy: str = "deferred",
                 pool: BlockPool | None = None) -> None:
        if block_size <= 0:
            raise KVError(f"block size must be positive, got {block_size}")
        if policy not in ("deferred", "eager"):
            raise KVError(f"unknown kv policy {policy!r}")
        self.block_size = block_size
        self.policy = policy
        self.pool = pool
        self.has_deferred: set[int] = set()
        self.empty_batch_seen = False
        self._written: dict[int, int] = {}
        self._allocated: dict[int, int] = {}
        self._blocks: dict[int, list[int]] = {}
        self.version = 0  # bumped whenever a physical block list changes
        self._list_version: dict[int, int] = {}  # per request, same rule

    # -- queries --------------------------------------------------------
    def written_of(self, request_id: int) -> int:
        return self._written.get(request_id, 0)

    def allocated_of(self, request_id: int) -> int:
        return self._allocated.get(request_id, 0)

    def blocks_of(self, request_id: int) -> list[int]:
        return self._blocks.get(request_id, [])

    def list_version(self, request_id: int) -> int:
        """Changes whenever ``blocks_of(request_id)`` does (device-table caching)."""
        return self._list_version.get(request_id, 0)

    @property
    def total_blocks_in_use(self) -> int:
        return sum(self._allocated.values())

    # -- growth policy --------------------------------------------------
    def schedule_allocation(self, ctx: AllocationContext) -> dict[int, str]:
        """Per request, grow this step ("allocate") or not ("skip").

        Insertion ordered: prefill ids first, then the remaining decode ids.
        """
        decisions: dict[int, str] = dict.fromkeys(ctx.prefill_ids, ALLOCATE)
        if self.policy == "eager":
            for rid in ctx.decode_ids:
                decisions.setdefault(rid, ALLOCATE)
            return decisions

        degraded = False
        if 0 in ctx.batch_sizes:
            # first sighting of an empty batch only arms the flag; from the
            # second on the alternation is considered broken
            degraded = self.empty_batch_seen
            self.empty_batch_seen = True
        for rid in ctx.decode_ids:
            if rid in decisions:
                continue
            grow = (degraded or rid not in self.has_deferred
                    or rid in ctx.draft_batch_ids)
            decisions[rid] = ALLOCATE if grow else SKIP
        self.has_deferred.update(ctx.decode_ids)
        return decisions

    # -- accounting -----------------------------------------------------
    def _resize(self, request_id: int, target: int) -> None:
        current = self._allocated[request_id]
        self._allocated[request_id] = target
        if self.pool is None or target == current:
            return
        blocks = self._blocks.setdefault(request_id, [])
        if target > current:
            blocks.extend(self.pool.take(target - current))
        else:
            self.pool.give(blocks[target:])
            del blocks[target:]
        self.version += 1
        self._list_version[request_id] = self.version

    def ensure_capacity(self, request_id: int, total_tokens: int) -> int:
        """Grow the allocation to cover ``total_tokens``; returns blocks added."""
        target = blocks_needed(total_tokens, self.block_size)
        if request_id not in self._allocated:
            self._written.setdefault(request_id, 0)
            self._allocated[request_id] = 0
            if self.pool is not None:
                self._blocks[request_id] = []
        current = self._allocated[request_id]
        if target <= current:
            return 0
        self._resize(request_id, target)
        return target - current

    def commit_write(self, request_id: int, tokens: int) -> None:
        """Record ``tokens`` written; a write past the allocation is a KVError."""
        if tokens < 0:
            raise KVError(f"cannot commit a negative token count ({tokens})")
        if request_id not in self._allocated:
            raise KVError(f"request {request_id} has no block-table entry")
        written = self._written[request_id]
        limit = self._allocated[request_id] * self.block_size
        if written + tokens > limit:
            raise KVError(f"request {request_id}: write of {tokens} tokens overruns "
                          f"allocation ({written} written, {limit} token capacity)")
        self._written[request_id] = written + tokens

    def trim_to_written(self, request_id: int, keep_tokens: int | None = None) -> int:
        """Give back blocks beyond ``keep_tokens`` (default: tokens written).

        Used after a worst-case grant once the accepted length is known (the
        rollback of the rejected draft tail).  Returns blocks freed.
        """
        if request_id not in self._allocated:
            raise KVError(f"request {request_id} has no block-table entry")
        keep = self._written[request_id] if keep_tokens is None else keep_tokens
        if keep < self._written[request_id]:
            raise KVError(f"request {request_id}: cannot trim below written tokens")
        target = blocks_needed(keep, self.block_size)
        current = self._allocated[request_id]
        if target >= current:
            return 0
        self._resize(request_id, target)
        return current - target

    def release(self, request_id: int) -> int:
        """Free a departing request's blocks; returns the count freed."""
        if request_id not in self._allocated:
            raise KVError(f"request {request_id} has no block-table entry")
        freed = self._allocated.pop(request_id)
        del self._written[request_id]
        self.has_deferred.discard(request_id)
        blocks = self._blocks.pop(request_id, None)
        self._list_version.pop(request_id, None)
        if blocks:
            self.pool.give(blocks)
            self.version += 1
        return freed
