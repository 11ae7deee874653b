"""Synthetic workloads: request lengths, arrivals, prompt token ids, preemptions.

``generate_requests`` restates the reference draw order so a seeded workload
is identical to ``specsim``'s (pkg/src/specsim/workload.py:184-249): one
stream ``Random(mix_stream_key(seed, 0x776B6C64))``; per request draw prompt
length, output length, then (poisson) the inter-arrival gap.  Trace files are
out of scope; ``parse_preemptions`` keeps the ``IDX@TIME``
syntax (workload.py:166-181).

``attach_prompt_ids`` is the B200 addition: uniform token ids in [0, vocab)
per request from a torch-free, seeded numpy generator, used by the GPU backend
and by the CPU oracle alike.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from .acceptance import mix_stream_key
from .errors import WorkloadError
from .records import Request
from .scheduler import Preemption

__all__ = ["LengthSpec", "WorkloadSpec", "attach_prompt_ids", "generate_requests",
           "make_requests", "parse_preemptions"]

_WORKLOAD_TAG = 0x776B6C64


@dataclass(frozen=True)
class LengthSpec:
    """A constant length or ``uniform:LO:HI`` (inclusive)."""

    kind: str
    value: int = 0
    lo: int = 0
    hi: int = 0

    @staticmethod
    def parse(text: str, name: str, minimum: int) -> "LengthSpec":
        text = text.strip()
        if text.startswith("uniform:"):
            parts = text.split(":")
            if len(parts) != 3:
                raise WorkloadError(f"{name}: expected uniform:LO:HI, got {text!r}")
            try:
                lo, hi = int(parts[1]), int(parts[2])
            except ValueError as exc:
                raise WorkloadError(f"{name}: non-integer bound in {text!r}") from exc
            if lo < minimum or hi < lo:
                raise WorkloadError(
                    f"{name}: bounds must satisfy {minimum} <= LO <= HI, got {text!r}")
            return LengthSpec("uniform", lo=lo, hi=hi)
        try:
            value = int(text)
        except ValueError as exc:
            raise WorkloadError(f"{name}: expected an integer or uniform:LO:HI, "
                                f"got {text!r}") from exc
        if value < minimum:
            raise WorkloadError(f"{name}: must be at least {minimum}, got {value}")
        return LengthSpec("constant", value=value)

    def draw(self, rng: random.Random) -> int:
        if self.kind == "constant":
            return self.value
        if self.kind == "uniform":
            return rng.randint(self.lo, self.hi)
        raise WorkloadError(f"unsupported length kind {self.kind!r}")


@dataclass(frozen=True)
class WorkloadSpec:
    arrival: str = "all-at-once"
    rate: float = 0.0
    count: int | None = None
    prompt_len: LengthSpec = LengthSpec("constant", value=32)
    output_len: LengthSpec = LengthSpec("constant", value=128)
    preemptions: tuple[Preemption, ...] = ()


def parse_preemptions(text: str) -> tuple[Preemption, ...]:
    out = []
    for token in text.split():
        idx_s, sep, time_s = token.partition("@")
        if not sep:
            raise WorkloadError(f"preemption {token!r}: expected IDX@TIME")
        try:
            idx, when = int(idx_s), float(time_s)
        except ValueError as exc:
            raise WorkloadError(f"preemption {token!r}: expected IDX@TIME") from exc
        if idx < 0 or when < 0.0:
            raise WorkloadError(f"preemption {token!r}: index and time must be >= 0")
        out.append(Preemption(idx, when))
    return tuple(out)


def generate_requests(spec: WorkloadSpec, seed: int) -> list[Request]:
    if spec.arrival not in ("all-at-once", "poisson"):
        raise WorkloadError(f"unknown arrival kind {spec.arrival!r}")
    if spec.count is None:
        raise WorkloadError("workload count is required")
    if spec.count <= 0:
        raise WorkloadError(f"workload count must be positive, got {spec.count}")
    if spec.arrival == "poisson" and not spec.rate > 0.0:
        raise WorkloadError(f"poisson arrivals need a positive rate, got {spec.rate}")
    for pre in spec.preemptions:
        if pre.request_index >= spec.count:
            raise WorkloadError(f"preemption targets request {pre.request_index} "
                                f"but only {spec.count} requests exist")
    rng = random.Random(mix_stream_key(seed, _WORKLOAD_TAG))
    clock = 0.0
    out = []
    for i in range(spec.count):
        prompt = spec.prompt_len.draw(rng)
        output = spec.output_len.draw(rng)
        if spec.arrival == "poisson":
            clock += rng.expovariate(spec.rate)
        out.append(Request(id=i, arrival_time=clock, prompt_len=prompt,
                           target_output_len=output))
    return out


def make_requests(output_lens: list[int], prompt_len: int | list[int] = 8,
                  arrivals: list[float] | None = None) -> list[Request]:
    """Convenience builder: one request per output length."""
    prompts = ([prompt_len] * len(output_lens) if isinstance(prompt_len, int)
               else list(prompt_len))
    return [Request(id=i, arrival_time=0.0 if arrivals is None else arrivals[i],
                    prompt_len=prompts[i], target_output_len=n)
            for i, n in enumerate(output_lens)]


def attach_prompt_ids(requests: list[Request], vocab: int, seed: int) -> list[Request]:
    """Give every request uniform synthetic prompt token ids in [0, vocab)."""
    for req in requests:
        gen = np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF,
                                                        req.id]))
        req.prompt_ids = gen.integers(0, vocab, size=req.prompt_len).tolist()
    return requests
