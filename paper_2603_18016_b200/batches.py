"""Two-batch membership for batch-parallel speculative decoding.

Every step one batch is *drafted* (the "skip" batch) while the other one is
*verified* (the target batch); the roles swap at each sync point.  Semantics
follow pkg/src/specsim/batch_manager.py:
  * start with ``skip_batch = 1``, ``balance = 0`` (:31-33)
  * ``balance = |B1| - |B0|``; a balanced pick goes to batch 0 iff
    ``balance >= 0`` (:62-64)
  * the first admission wave (and every admission under ``always-balance``)
    is balanced; later ones land in the current skip batch (:66-77)
  * ``recycle`` removes a departing request and fixes the balance (:79-88)
  * ``alternate_skip`` swaps roles and ends the startup phase (:90-94)

Membership is insertion ordered (dict keys), which fixes the row order of
every batch the GPU backend launches.
"""

from __future__ import annotations

from .errors import CapacityError, ProtocolError

__all__ = ["BatchManager"]

_POLICIES = ("skip-batch", "always-balance")


class BatchManager:
    def __init__(self, batch_capacity: int, policy: str = "skip-batch") -> None:
        if batch_capacity <= 0:
            raise ValueError(f"batch_capacity must be positive, got {batch_capacity}")
        if policy not in _POLICIES:
            raise ValueError(f"unknown assignment policy {policy!r}")
        self.batch_capacity = batch_capacity
        self.policy = policy
        self.balance = 0
        self.skip_batch = 1
        self.first_step_done = False
        self._batches: tuple[dict[int, None], dict[int, None]] = ({}, {})

    # -- queries --------------------------------------------------------
    def members_of(self, batch_id: int) -> list[int]:
        return list(self._batches[batch_id])

    def size_of(self, batch_id: int) -> int:
        return len(self._batches[batch_id])

    def _find(self, request_id: int) -> int | None:
        if request_id in self._batches[0]:
            return 0
        if request_id in self._batches[1]:
            return 1
        return None

    def batch_of(self, request_id: int) -> int:
        where = self._find(request_id)
        if where is None:
            raise ProtocolError(f"request {request_id} is not in any batch")
        return where

    @property
    def target_batch(self) -> int:
        return 1 - self.skip_batch

    # -- mutations ------------------------------------------------------
    def assign(self, request_id: int) -> int:
        """Admit a new request; returns the batch it joined."""
        if self._find(request_id) is not None:
            raise ProtocolError(f"request {request_id} is already assigned")
        balanced = self.policy == "always-balance" or not self.first_step_done
        if balanced:
            dest = 0 if self.balance >= 0 else 1
        else:
            dest = self.skip_batch
        members = self._batches[dest]
        if len(members) >= self.batch_capacity:
            raise CapacityError(f"batch {dest} is full ({self.batch_capacity} slots)")
        members[request_id] = None
        self.balance += 1 if dest == 1 else -1
        return dest

    def recycle(self, request_id: int) -> int:
        """Remove a departing request; returns the batch it left."""
        where = self._find(request_id)
        if where is None:
            raise ProtocolError(f"request {request_id} is not in any batch")
        del self._batches[where][request_id]
        self.balance += 1 if where == 0 else -1
        return where

    def alternate_skip(self) -> int:
        """Swap drafting / verifying roles at a sync point."""
        self.skip_batch ^= 1
        self.first_step_done = True
        return self.skip_batch
