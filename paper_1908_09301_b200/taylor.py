"""High-order Taylor stepping on the B200 engine -- drop-in for the
reference's integrator entry points (/root/reference/pkg/src/mptaylor/taylor.py):
same names, signatures, recording policy, observer protocol and errors.

What changes underneath:
  * numbers are device fixed-point digit rows with F >= P + guard bits;
  * the coefficient recurrence (taylor.py:117) runs tau-scaled,
    a~_{i+1} = tau/(i+1) * (...), in one persistent CUDA kernel per launch;
    the Cauchy sums are exact integer column sums rounded once;
  * the Horner evaluation (taylor.py:168) becomes the exact sum of the
    scaled rows, fused into the same kernel, and the state is rounded to the
    context precision P (round-to-nearest-even) after every step, so every
    recorded state is a P-bit MPValue like the reference's.
Results agree with the reference to a relative tolerance of 10^-(K-d) over
short horizons (tests/test_gpu.py states the guard digits d(t) per run).
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict
from contextlib import contextmanager
from dataclasses import dataclass, field
from decimal import Decimal, localcontext
from fractions import Fraction

import numpy as np

from ._native import MPT_ERANGE, NativeError
from .engine import DevicePlan, SystemTables
from .fixed import FixedFormat
from .mp import MPValue, PrecisionContext, RangeError, mp_from_decimal
from .reduction import DeviceReducer
from .systems import QuadraticODESystem

DEFAULT_RECORD_STRIDE = 100


@dataclass(frozen=True)
class Jet:
    """coeffs[m][i] = i-th normalized derivative of variable m (taylor.py:37)."""

    dim: int
    order: int
    coeffs: tuple

    def __post_init__(self):
        if len(self.coeffs) != self.dim:
            raise ValueError("coeffs must have dim rows")
        if any(len(row) != self.order + 1 for row in self.coeffs):
            raise ValueError("each coefficient row must have order+1 entries")


@dataclass(frozen=True)
class StepConfig:
    """Step size as exact decimal text, method order, workers (taylor.py:57)."""

    tau_text: str
    order_n: int
    workers: int = 1

    def __post_init__(self):
        try:
            tau = Decimal(self.tau_text)
        except ArithmeticError as exc:
            raise ValueError(f"step size is not a decimal: {self.tau_text!r}") from exc
        if tau == 0:
            raise ValueError("step size must be nonzero")
        if self.order_n < 1:
            raise ValueError(f"order_n must be >= 1, got {self.order_n}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")

    def tau(self, ctx: PrecisionContext) -> MPValue:
        return mp_from_decimal(self.tau_text, ctx)


@dataclass(frozen=True)
class TrajectoryPoint:
    step: int
    state: tuple


@dataclass
class Trajectory:
    """Recorded states sampled on a fixed step stride (taylor.py:92)."""

    dim: int
    tau_text: str
    points: list = field(default_factory=list)

    def time_of(self, step: int) -> Decimal:
        return exact_time(step, self.tau_text)

    def steps(self) -> list:
        return [p.step for p in self.points]

    def final_state(self) -> tuple:
        return self.points[-1].state


def exact_time(step: int, tau_text: str) -> Decimal:
    """step * tau as an exact decimal (taylor.py:109)."""
    tau = Decimal(tau_text)
    with localcontext() as dctx:
        dctx.prec = len(tau.as_tuple().digits) + len(str(step)) + 4
        return +(tau * step)


def _device_options(reducer):
    if isinstance(reducer, DeviceReducer):
        return reducer.device, reducer.guard_bits
    return 0, FixedFormat(64).guard_bits


def _to_values(fmt: FixedFormat, rows, prec: int) -> tuple:
    return tuple(MPValue.from_fraction(f, prec) for f in fmt.digits_to_fractions(rows))


def _check_state(system: QuadraticODESystem, state):
    if len(state) != system.dim:
        raise ValueError(f"state has {len(state)} components, system dim {system.dim}")


def compute_jet(system: QuadraticODESystem, state, order_n: int, ctx: PrecisionContext, reducer=None) -> Jet:
    """Taylor coefficients through `state` up to order_n (taylor.py:139).

    The device computes the jet scaled by s^i with s = 2^-k (exact power of
    two, so unscaling is exact); k grows until no coefficient leaves the
    fixed-point range. Each coefficient is then rounded to ctx precision.
    """
    _check_state(system, state)
    if order_n < 1:
        raise ValueError(f"order_n must be >= 1, got {order_n}")
    device, guard = _device_options(reducer)
    fmt = FixedFormat(ctx.precision_bits, guard)
    st = fmt.to_digits(state)
    last = None
    for k in (7, 10, 14, 20, 28):
        try:
            with checked_out_plan(system, order_n, Fraction(1, 1 << k), ctx, reducer) as (_, plan):
                coef = plan.compute_jet(st)[0]
        except NativeError as exc:
            if exc.code == MPT_ERANGE:  # a coefficient left the range: retry with a smaller scale
                last = exc
                continue
            raise
        rows = []
        for m in range(system.dim):
            fr = fmt.digits_to_fractions(coef[m])
            row = [state[m]] + [
                MPValue.from_fraction(f * (1 << (k * i)), ctx.precision_bits) for i, f in enumerate(fr) if i > 0
            ]
            rows.append(tuple(row))
        return Jet(dim=system.dim, order=order_n, coeffs=tuple(rows))
    raise RangeError(f"jet coefficients exceed the device range: {last}")


def horner_eval(jet_row, tau: MPValue, ctx: PrecisionContext) -> MPValue:
    """a[0] + tau*(a[1] + tau*(a[2] + ...)) (taylor.py:168).

    A host utility on MPValues for API completeness; the stepping path never
    calls it (its evaluation is fused into the device kernel)."""
    if len(jet_row) < 1:
        raise ValueError("jet row must have at least one coefficient")
    if tau.is_zero():
        return jet_row[0]
    acc = jet_row[-1]
    for idx in range(len(jet_row) - 2, -1, -1):
        acc = ctx.add(jet_row[idx], ctx.mul(tau, acc))
    return acc


# Device plans of integrate() / step() / compute_jet(), keyed by everything
# that defines them (the digit tables byte for byte, format, order, device, the
# kernel-selection environment and the process id): repeated calls on one
# system skip allocation and constant upload. A plan owns one set of device
# buffers, so an entry is used by one caller at a time (per-entry lock; other
# keys run concurrently, as the reference's reentrant integrate() does).
# Least-recently-used entries beyond the limit are destroyed once idle.
_PLAN_CACHE: "OrderedDict[tuple, _PlanEntry]" = OrderedDict()
_PLAN_CACHE_SIZE = 8
_PLAN_CACHE_LOCK = threading.Lock()


class _PlanEntry:
    def __init__(self, fmt, plan):
        self.fmt, self.plan = fmt, plan
        self.lock = threading.Lock()
        self.users = 0
        self.evicted = False


def _forget_plans_in_child():
    # a forked child inherits handles of the parent's CUDA context: never free them there
    for entry in _PLAN_CACHE.values():
        entry.plan.h = None
    _PLAN_CACHE.clear()


os.register_at_fork(after_in_child=_forget_plans_in_child)


def _plan_key(tables: SystemTables, guard: int, prec_bits: int, order: int, device: int, n_traj: int) -> tuple:
    return (os.getpid(), device, n_traj, guard, prec_bits, order, tables.dim, tables.c_shift,
            tuple(os.environ.get(v) for v in ("MPT_KERNEL", "MPT_CLUSTER", "MPT_TEAM_MB")),
            *(np.ascontiguousarray(a).tobytes() for a in
              (tables.teq, tables.tj, tables.tk, tables.cst, tables.lin, tables.q, tables.ctab)))


@contextmanager
def checked_out_plan(system, order_n: int, scale: Fraction, ctx: PrecisionContext, reducer, n_traj: int = 1,
                     device=None):
    """(fmt, plan) of n_traj trajectories for (system, order, step scale),
    exclusively held for the duration of the with-block."""
    dev, guard = _device_options(reducer)
    device = dev if device is None else device
    fmt = FixedFormat(ctx.precision_bits, guard)
    tables = SystemTables.build(system, fmt, order_n, scale)
    key = _plan_key(tables, guard, ctx.precision_bits, order_n, device, n_traj)
    stale = []
    with _PLAN_CACHE_LOCK:
        entry = _PLAN_CACHE.get(key)
        if entry is None:
            entry = _PLAN_CACHE[key] = _PlanEntry(fmt, DevicePlan(tables, fmt, order_n, n_traj, device))
        _PLAN_CACHE.move_to_end(key)
        entry.users += 1
        while len(_PLAN_CACHE) > _PLAN_CACHE_SIZE:
            _, old = _PLAN_CACHE.popitem(last=False)
            old.evicted = True
            if old.users == 0:
                stale.append(old)
    for old in stale:
        old.plan.close()
    try:
        with entry.lock:
            yield entry.fmt, entry.plan
    finally:
        with _PLAN_CACHE_LOCK:
            entry.users -= 1
            close_now = entry.evicted and entry.users == 0
        if close_now:
            entry.plan.close()


def clear_plan_cache() -> None:
    """Destroy every idle cached device plan (tests; before a device reset)."""
    with _PLAN_CACHE_LOCK:
        entries = list(_PLAN_CACHE.values())
        _PLAN_CACHE.clear()
        for e in entries:
            e.evicted = True
        idle = [e for e in entries if e.users == 0]
    for e in idle:
        e.plan.close()


def step(system: QuadraticODESystem, state, cfg: StepConfig, ctx: PrecisionContext, reducer=None) -> tuple:
    """Advance the state by one Taylor step of size cfg.tau (taylor.py:182)."""
    _check_state(system, state)
    with checked_out_plan(system, cfg.order_n, cfg.tau(ctx).as_fraction(), ctx, reducer) as (fmt, plan):
        out, status = plan.step(fmt.to_digits(state))
    if status.any():
        raise RangeError("state left the device fixed-point range (|x| >= 2^27) in step")
    out = out[0]
    return _to_values(fmt, out, ctx.precision_bits)


def integrate(
    system: QuadraticODESystem,
    state0,
    cfg: StepConfig,
    n_steps: int,
    ctx: PrecisionContext,
    reducer=None,
    observer=None,
    record_stride: int = DEFAULT_RECORD_STRIDE,
    start_step: int = 0,
) -> Trajectory:
    """Apply `step` n_steps times on the device (taylor.py:202).

    Records step start_step, every multiple of record_stride and n_steps; an
    observer, when given, is called once per step with (n, exact time,
    state) after the launch, in step order (it cannot influence the run).
    """
    if n_steps < 0:
        raise ValueError(f"n_steps must be >= 0, got {n_steps}")
    if not 0 <= start_step <= n_steps:
        raise ValueError(f"start_step must be in [0, {n_steps}], got {start_step}")
    if record_stride < 1:
        raise ValueError(f"record_stride must be >= 1, got {record_stride}")
    _check_state(system, state0)
    traj = Trajectory(dim=system.dim, tau_text=cfg.tau_text)
    traj.points.append(TrajectoryPoint(step=start_step, state=tuple(state0)))
    if n_steps == start_step:
        return traj
    dev_stride = 1 if observer is not None else record_stride
    with checked_out_plan(system, cfg.order_n, cfg.tau(ctx).as_fraction(), ctx, reducer) as (fmt, plan):
        steps, recs, status = plan.integrate(fmt.to_digits(state0), n_steps, start_step, dev_stride)
    if status.any():
        raise RangeError("state left the device fixed-point range (|x| >= 2^27) during integrate")
    prec = ctx.precision_bits
    for r in range(1, len(steps)):
        n = int(steps[r])
        state = _to_values(fmt, recs[r, 0], prec)
        if n % record_stride == 0 or n == n_steps:
            traj.points.append(TrajectoryPoint(step=n, state=state))
        if observer is not None:
            observer(n, exact_time(n, cfg.tau_text), state)
    return traj
