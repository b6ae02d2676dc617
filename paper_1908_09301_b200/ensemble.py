"""Ensembles of trajectories and their divergence times (BASELINE configs[4]).

M trajectories whose initial conditions are the canonical Lorenz point plus
seeded uniform perturbations are integrated at a base budget (K, N) and at a
verify budget (K + 50, N + 30); each member's divergence time is the
reference's critical time t_c (cns.py:202 estimate_tc semantics) of its own
base/verify pair. One DevicePlan integrates a whole shard of members in one
launch (team kernel: one CTA per trajectory, rows in HBM/L2).

Multi-GPU: members are split into contiguous shards, one per rank
(`shard_bounds`); there is no collective on the data path. The results are
collected at the end with `gather_rows` (torch.distributed all_gather over
NCCL on GPUs, gloo in the CPU tests).

The agreement metric is the reference's (cns.py:52), computed exactly on the
fixed-point integers of the two runs (both states carry exactly P bits).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from decimal import Decimal, localcontext
from fractions import Fraction

import numpy as np

from .cns import AGREEMENT_EXACT, tc_from_series
from .engine import DevicePlan, SystemTables
from .fixed import FixedFormat
from .mp import PrecisionContext, bits_for_digits, mp_from_decimal
from .systems import builtin_system
from .taylor import exact_time

CANON_INIT = ("-15.8", "-17.48", "35.64")
EXACT_CODE = 1 << 30  # AGREEMENT_EXACT in integer matrices


def perturbed_inits(n_members: int, seed: int = 0, amplitude: str = "1e-20", base=CANON_INIT,
                    resolution_digits: int = 12) -> list:
    """Decimal initial conditions base + u, u ~ uniform on [-amplitude, amplitude]
    (grid of amplitude * 10^-resolution_digits), seeded; one tuple per member."""
    rng = np.random.default_rng(seed)
    lim = 10**resolution_digits
    draws = rng.integers(-lim, lim, size=(n_members, len(base)), endpoint=True)
    unit = Decimal(amplitude).scaleb(-resolution_digits)
    out = []
    with localcontext() as dctx:
        dctx.prec = 200
        for row in draws:
            out.append(tuple(str(Decimal(b) + int(n) * unit) for b, n in zip(base, row)))
    return out


def shard_bounds(n_members: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced shard [lo, hi) of rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, rem = divmod(n_members, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass
class EnsembleRun:
    """Recorded states of a shard of members at one (bits, order)."""

    bits: int
    order: int
    tau_text: str
    fmt: FixedFormat
    steps: np.ndarray  # [nrec]
    records: np.ndarray  # [nrec, members, dim, W] int32 digits
    status: np.ndarray  # [members]
    kernel_ms: float = 0.0

    def ints(self, rec: int) -> list:
        """Fixed-point numerators of record `rec`: [members][dim] Python ints."""
        r = self.records[rec]
        flat = self.fmt.digits_to_ints(r.reshape(-1, r.shape[-1]))
        d = r.shape[1]
        return [flat[i * d:(i + 1) * d] for i in range(r.shape[0])]


def run_members(system_name: str, inits, bits: int, order: int, tau_text: str, n_steps: int, stride: int,
                device: int = 0, kernel: str = "auto") -> EnsembleRun:
    """Integrate every member of `inits` (decimal texts, parsed at `bits`) on one GPU."""
    ctx = PrecisionContext(bits)
    system = builtin_system(system_name, ctx) if isinstance(system_name, str) else system_name(ctx)
    fmt = FixedFormat(bits)
    tau = mp_from_decimal(tau_text, ctx)
    tables = SystemTables.build(system, fmt, order, tau.as_fraction())
    states = np.stack([fmt.to_digits([mp_from_decimal(t, ctx) for t in row]) for row in inits])
    with DevicePlan(tables, fmt, order, len(inits), device) as plan:
        if kernel != "auto":
            plan.configure(kernel, 1)
        steps, recs, status = plan.integrate(states, n_steps, 0, stride)
        ms = plan.last_kernel_ms()
    return EnsembleRun(bits, order, tau_text, fmt, steps, recs, status, ms)


def _floor_neg_log10(num: int, den: int, pow10: list) -> int:
    if num > den:
        return 0
    d = max(0, int((den.bit_length() - num.bit_length() - 1) * 0.30102999566398120))
    while d > 0 and num * pow10[d] > den:
        d -= 1
    while num * pow10[d + 1] <= den:
        d += 1
    return d


def agreement_matrix(a: EnsembleRun, b: EnsembleRun) -> np.ndarray:
    """[nrec, members] agreement digits (cns.py:52; EXACT_CODE for identical
    samples), exact integer arithmetic on the aligned fixed-point numerators."""
    if not np.array_equal(a.steps, b.steps) or a.records.shape[1] != b.records.shape[1]:
        raise ValueError("runs are not sampled on the same grid / members")
    fa, fb = a.fmt.frac_bits, b.fmt.frac_bits
    F = max(fa, fb)
    sa, sb = F - fa, F - fb
    one = 1 << F
    cap = (max(a.bits, b.bits) * 30103) // 100000 + 8
    pow10 = [10**k for k in range(cap + 2)]
    nrec, members = a.records.shape[0], a.records.shape[1]
    out = np.zeros((nrec, members), np.int64)
    for r in range(nrec):
        ia, ib = a.ints(r), b.ints(r)
        for m in range(members):
            worst = EXACT_CODE
            for x, y in zip(ia[m], ib[m]):
                x <<= sa
                y <<= sb
                if x == y:
                    continue
                g = max(abs(x), abs(y), one)
                worst = min(worst, _floor_neg_log10(abs(x - y), g, pow10))
            out[r, m] = worst
    return out


def divergence_times(steps, tau_text: str, agreement: np.ndarray, d: int) -> list:
    """Per member: t_c = time of the last sample before the first one with
    fewer than d digits (cns.py:137 semantics), as Decimal."""
    times = [exact_time(int(s), tau_text) for s in steps]
    out = []
    for m in range(agreement.shape[1]):
        series = [(int(s), t, (AGREEMENT_EXACT if v == EXACT_CODE else int(v)))
                  for s, t, v in zip(steps, times, agreement[:, m])]
        out.append(tc_from_series(series, d))
    return out


@dataclass
class EnsembleReport:
    base: tuple  # (bits, order)
    verify: tuple
    tau_text: str
    steps: np.ndarray
    agreement: np.ndarray  # [nrec, members]
    t_c: list  # Decimal per member
    final_base: np.ndarray  # [members, dim, W_base] digits
    kernel_ms: dict = field(default_factory=dict)

    def tc_seconds(self) -> np.ndarray:
        return np.array([float(t) for t in self.t_c])


def ensemble_tc(inits, K: int, N: int, tau_text: str, t_end_text: str, d: int = 10, stride: int = 100,
                verify_margin=(50, 30), system_name: str = "lorenz", device: int = 0) -> EnsembleReport:
    """Divergence times of every member against its own (K+50, N+30) run."""
    ratio = Decimal(t_end_text) / Decimal(tau_text)
    if ratio != ratio.to_integral_value():
        raise ValueError(f"t_end {t_end_text} is not an integer multiple of tau {tau_text}")
    n_steps = int(ratio)
    bb, vb = bits_for_digits(K), bits_for_digits(K + verify_margin[0])
    base = run_members(system_name, inits, bb, N, tau_text, n_steps, stride, device)
    ver = run_members(system_name, inits, vb, N + verify_margin[1], tau_text, n_steps, stride, device)
    if base.status.any() or ver.status.any():
        raise ArithmeticError("a member left the device fixed-point range")
    agr = agreement_matrix(base, ver)
    return EnsembleReport((bb, N), (vb, N + verify_margin[1]), tau_text, base.steps, agr,
                          divergence_times(base.steps, tau_text, agr, d), base.records[-1],
                          {"base": base.kernel_ms, "verify": ver.kernel_ms})


# ------------------------------------------------------------------ gather
def gather_rows(local: np.ndarray, n_total: int, world: int, rank: int, device=None) -> np.ndarray:
    """Concatenate every rank's shard (rows [lo, hi) of shard_bounds) in rank
    order with torch.distributed all_gather; NCCL needs CUDA tensors (pass
    `device`), gloo works on CPU. Returns the full [n_total, ...] array on every rank."""
    import torch
    import torch.distributed as dist

    lo, hi = shard_bounds(n_total, world, rank)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, shard is {hi - lo}")
    per = -(-n_total // world)
    tail = local.shape[1:]
    buf = np.zeros((per,) + tail, dtype=local.dtype)
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    rows = []
    for r, p in enumerate(parts):
        a, b = shard_bounds(n_total, world, r)
        rows.append(p[: b - a].cpu().numpy())
    return np.concatenate(rows, axis=0)
