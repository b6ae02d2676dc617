"""Reduction plans and the device reducer.

API mirror of /root/reference/pkg/src/mptaylor/reduction.py. In the
reference a reducer evaluates the order-i convolution sums on CPU worker
processes over a fixed chunk partition, so that the rounded result depends
only on the chunk count (reduction.py:1-22). On the device every Cauchy sum is
accumulated exactly in integer column accumulators and rounded once, so the
result does not depend on chunking, thread count or scheduling at all -- the
reference's determinism contract holds trivially and more strongly.

``ReducePlan``, ``partition`` and ``chunk_bounds`` keep their reference
signatures and validation (they describe the reference's rounding structure
and are used by the CPU baseline); ``make_reducer`` returns a DeviceReducer
that carries the device options used by taylor.integrate / compute_jet.
"""

from __future__ import annotations

from dataclasses import dataclass

from .fixed import DEFAULT_GUARD_BITS

DEFAULT_NUM_CHUNKS = 64
DEFAULT_SERIAL_THRESHOLD = 256


@dataclass(frozen=True)
class ReducePlan:
    """Same fields and validation as reduction.py:40 ReducePlan."""

    num_chunks: int = DEFAULT_NUM_CHUNKS
    workers: int = 1
    serial_threshold: int = DEFAULT_SERIAL_THRESHOLD
    chunks_follow_workers: bool = False

    def __post_init__(self):
        for name in ("num_chunks", "workers", "serial_threshold"):
            value = getattr(self, name)
            if value < 1:
                raise ValueError(f"{name} must be >= 1, got {value}")

    def effective_chunks(self) -> int:
        return self.workers if self.chunks_follow_workers else self.num_chunks


def chunk_bounds(i: int, num_chunks: int, c: int) -> tuple:
    """Inclusive (lo, hi) of chunk c of [0, i] (reduction.py:84)."""
    base, rem = divmod(i + 1, num_chunks)
    lo = c * base + min(c, rem)
    return lo, lo + base + (1 if c < rem else 0) - 1


def partition(i: int, num_chunks: int) -> list:
    """[0, i] in num_chunks contiguous near-equal ranges, larger first (reduction.py:70)."""
    if i < 0:
        raise ValueError(f"order index must be >= 0, got {i}")
    if num_chunks < 1:
        raise ValueError(f"num_chunks must be >= 1, got {num_chunks}")
    return [chunk_bounds(i, num_chunks, c) for c in range(num_chunks)]


class DeviceReducer:
    """Device options for the Taylor engine; a context manager like the
    reference reducers (reduction.py:187 SerialReducer)."""

    def __init__(self, plan: ReducePlan | None = None, device: int = 0,
                 guard_bits: int = DEFAULT_GUARD_BITS):
        self.plan = plan if plan is not None else ReducePlan()
        self.device = device
        self.guard_bits = guard_bits

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


# The reference's reducer class names, kept so existing call sites import
# unchanged; both run the device engine.
SerialReducer = DeviceReducer
ProcessReducer = DeviceReducer


def make_reducer(plan: ReducePlan | None = None) -> DeviceReducer:
    return DeviceReducer(plan)
