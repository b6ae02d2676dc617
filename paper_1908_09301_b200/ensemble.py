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
from .fixed import MAX_INT_BITS, RADIX, RADIX_BITS, FixedFormat
from .mp import _DECIMAL_RE, PrecisionContext, RangeError, _round_scaled, bits_for_digits, mp_from_decimal
from .systems import builtin_system
from .taylor import checked_out_plan, exact_time

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


def decimal_to_fixed_int(text: str, bits: int, fmt: FixedFormat) -> int:
    """fmt.to_int(mp_from_decimal(text, ctx)) on plain integers: the decimal is
    rounded to `bits` significant bits (ties to even, mp.py:122) and then placed
    on the fixed-point grid; no MPValue / Fraction objects (ensemble uploads
    convert 3 M values per call)."""
    stripped = text.strip()
    if not _DECIMAL_RE.match(stripped):
        raise ValueError(f"not a valid decimal literal: {text!r}")
    neg = stripped[0] == "-"
    mant_txt, _, exp_txt = stripped.lstrip("+-").replace("E", "e").partition("e")
    whole, _, frac = mant_txt.partition(".")
    digits = int((whole or "0") + frac)
    e10 = (int(exp_txt) if exp_txt else 0) - len(frac)
    if digits == 0:
        return 0
    if abs(len(str(digits)) + e10) > 10**6:
        raise RangeError(f"decimal exponent out of range: {text!r}")
    num, den = (digits * 10**e10, 1) if e10 >= 0 else (digits, 10**(-e10))
    mant, exp = _round_scaled(1, num, den, bits)
    sh = exp + fmt.frac_bits
    if sh >= 0:
        x = mant << sh
    else:
        q, r = divmod(mant, 1 << -sh)
        half = 1 << (-sh - 1)
        x = q + (1 if r > half or (r == half and q & 1) else 0)
    if x >> (fmt.frac_bits + MAX_INT_BITS):
        raise RangeError(f"|value| >= 2^{MAX_INT_BITS} does not fit the device format")
    return -x if neg else x


def states_from_decimals(inits, bits: int, fmt: FixedFormat) -> np.ndarray:
    """[members, dim, W] digit rows of decimal initial conditions parsed at `bits`."""
    dim = len(inits[0])
    flat = [decimal_to_fixed_int(t, bits, fmt) for row in inits for t in row]
    return fmt.ints_to_digits(flat).reshape(len(inits), dim, fmt.width)


def run_members(system_name: str, inits, bits: int, order: int, tau_text: str, n_steps: int, stride: int,
                device: int = 0, kernel: str = "auto") -> EnsembleRun:
    """Integrate every member of `inits` (decimal texts, parsed at `bits`) on one GPU.
    The device plan (buffers, constant tables) is cached across calls."""
    ctx = PrecisionContext(bits)
    system = builtin_system(system_name, ctx) if isinstance(system_name, str) else system_name(ctx)
    tau = mp_from_decimal(tau_text, ctx)
    fmt = FixedFormat(bits)
    states = states_from_decimals(inits, bits, fmt)
    with checked_out_plan(system, order, tau.as_fraction(), ctx, None, n_traj=len(inits), device=device) as (_, plan):
        plan.configure(kernel, 16 if len(inits) == 1 else 1)
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


def _agreement_exact(x: int, y: int, one: int, pow10: list) -> int:
    if x == y:
        return EXACT_CODE
    return _floor_neg_log10(abs(x - y), max(abs(x), abs(y), one), pow10)


def _top3(dig: np.ndarray):
    """(mantissa, digit exponent) of the values of signed digit rows [n, W]:
    value ~= mantissa * B^exponent from the three leading nonzero digits
    (relative error < 2^-25); zero rows give mantissa 0."""
    n, W = dig.shape
    nz = dig != 0
    top = np.where(nz.any(axis=1), W - 1 - np.argmax(nz[:, ::-1], axis=1), 2)
    top = np.maximum(top, 2)
    idx = np.arange(n)
    B = float(RADIX)
    mant = (dig[idx, top].astype(np.float64) * B + dig[idx, top - 1]) * B + dig[idx, top - 2]
    return mant, top - 2


def agreement_matrix(a: EnsembleRun, b: EnsembleRun) -> np.ndarray:
    """[nrec, members] agreement digits (cns.py:52; EXACT_CODE for identical
    samples). The digit count floor(-log10(|x-y| / max(|x|, |y|, 1))) is
    evaluated in floating point on the three leading digits of the aligned
    fixed-point rows (both formats are whole radix-2^28 digits apart), and
    recomputed in exact integer arithmetic wherever the estimate is within 1e-6
    of an integer boundary, so the result is the exact one."""
    if not np.array_equal(a.steps, b.steps) or a.records.shape[1] != b.records.shape[1]:
        raise ValueError("runs are not sampled on the same grid / members")
    la, lb = a.fmt.frac_digits, b.fmt.frac_digits
    Lf = max(la, lb)
    F = RADIX_BITS * Lf
    one = 1 << F
    cap = (max(a.bits, b.bits) * 30103) // 100000 + 8
    pow10 = [10**k for k in range(cap + 2)]
    nrec, members, dim = a.records.shape[0], a.records.shape[1], a.records.shape[2]
    out = np.zeros((nrec, members), np.int64)
    log10B = RADIX_BITS * np.log10(2.0)

    def aligned(run, lf, r):  # digit rows on the common grid, [members*dim, Lf + 1]
        rows = run.records[r].reshape(members * dim, -1).astype(np.int64)
        return np.pad(rows, ((0, 0), (Lf - lf, 0)))

    for r in range(nrec):
        da, db = aligned(a, la, r), aligned(b, lb, r)
        md, ed = _top3(da - db)
        ma, ea = _top3(da)
        mb, eb = _top3(db)
        with np.errstate(divide="ignore", invalid="ignore"):
            lg_d = np.log10(np.abs(md)) + ed * log10B
            lg_g = np.maximum(np.maximum(np.log10(np.abs(ma)) + ea * log10B, np.log10(np.abs(mb)) + eb * log10B), Lf * log10B)
            est = lg_g - lg_d  # log10(max(|x|, |y|, 1) / |x - y|)
        same = md == 0
        est = np.where(same, 0.5, est)
        digits = np.floor(est)
        risky = ~same & (np.abs(est - np.round(est)) < 1e-6)
        digits = np.where(est < 0, 0, digits).astype(np.int64)
        digits[same] = EXACT_CODE
        if risky.any():
            ia = a.fmt.digits_to_ints(a.records[r].reshape(members * dim, -1)[risky])
            ib = b.fmt.digits_to_ints(b.records[r].reshape(members * dim, -1)[risky])
            sa, sb = RADIX_BITS * (Lf - la), RADIX_BITS * (Lf - lb)
            digits[risky] = [_agreement_exact(x << sa, y << sb, one, pow10) for x, y in zip(ia, ib)]
        out[r] = digits.reshape(members, dim).min(axis=1)
    return out


def agreement_matrix_exact(a: EnsembleRun, b: EnsembleRun) -> np.ndarray:
    """agreement_matrix in exact integer arithmetic throughout (the checker of the fast path)."""
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
            out[r, m] = min(_agreement_exact(x << sa, y << sb, one, pow10) for x, y in zip(ia[m], ib[m]))
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


def tc_steps(steps, agreement_by_member: np.ndarray, d: int) -> np.ndarray:
    """divergence_times as step indices, vectorised: [members] step of the last
    sample before the first one with fewer than d digits (the last sample when
    none fails, 0 when the first one fails); t_c = step * tau exactly."""
    steps = np.asarray(steps, np.int64)
    fails = np.asarray(agreement_by_member) < d
    first = np.where(fails.any(axis=1), fails.argmax(axis=1), len(steps))
    return np.where(first == 0, 0, steps[np.maximum(first, 1) - 1]).astype(np.int64)


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


# ------------------------------------------------------------------ T_c-K sweep
@dataclass
class SweepReport:
    """One (K, N) point of the T_c-K diagram over the whole ensemble (every rank
    holds the gathered arrays; member order = perturbed_inits order)."""

    K: int
    N: int
    base: tuple  # (bits, order)
    verify: tuple
    tau_text: str
    steps: np.ndarray  # [nrec] sampled step indices
    agreement: np.ndarray  # [members, nrec] digits (EXACT_CODE = identical)
    tc_step: np.ndarray  # [members] step index of t_c (t_c = tc_step * tau, exact)
    final_xyz: np.ndarray  # [members, dim] float64 view of the base run's final state
    final_digits: np.ndarray  # [members, dim, W_base] its exact digits
    world: int = 1
    kernel_ms: dict = field(default_factory=dict)

    def t_c(self) -> list:
        return [exact_time(int(s), self.tau_text) for s in self.tc_step]

    def tc_mean(self) -> float:
        return float(np.mean([float(t) for t in self.t_c()]))


def _device_run_fn(system_name, device):
    def run(inits, bits, order, tau_text, n_steps, stride):
        return run_members(system_name, inits, bits, order, tau_text, n_steps, stride, device)

    return run


def tc_sweep(K: int, N: int, n_members: int, n_steps: int, rank: int = 0, world: int = 1, device: int = 0,
             tau_text: str = "0.01", d: int = 10, stride: int = 100, seed: int = 0, amplitude: str = "1e-20",
             verify_margin=(50, 30), system_name: str = "lorenz", run_fn=None, gather: bool = True,
             gather_device=None) -> SweepReport:
    """BASELINE configs[4] at one (K, N): this rank's shard of the M seeded members
    is integrated at (K, N) and at the verify budget (K+50, N+30) on `device`, each
    member's divergence time t_c is taken against its own verify run (reference
    cns.py:202 estimate_tc / :254 cns_run semantics, as scripts/tc_sweep.py does
    per sweep point through cns.py:290 tc_diagram), and x, y, z and t_c of all M
    members are all-gathered (torch.distributed; NCCL when `gather_device` is a
    CUDA device, gloo on CPU). No collective touches the integration itself.

    run_fn(inits, bits, order, tau_text, n_steps, stride) -> EnsembleRun replaces
    the device run in the host-logic tests."""
    if n_steps % stride:
        raise ValueError(f"n_steps {n_steps} is not a multiple of the sampling stride {stride}")
    lo, hi = shard_bounds(n_members, world, rank)
    inits = perturbed_inits(n_members, seed=seed, amplitude=amplitude)[lo:hi]
    run = run_fn or _device_run_fn(system_name, device)
    bb, vb = bits_for_digits(K), bits_for_digits(K + verify_margin[0])
    vn = N + verify_margin[1]
    if hi > lo:
        base = run(inits, bb, N, tau_text, n_steps, stride)
        ver = run(inits, vb, vn, tau_text, n_steps, stride)
        if base.status.any() or ver.status.any():
            raise ArithmeticError("a member left the device fixed-point range")
        steps = np.asarray(base.steps, np.int64)
        agr = agreement_matrix(base, ver).T.copy()  # [members, nrec]
        tc_step = tc_steps(steps, agr, d)
        final_digits = np.ascontiguousarray(base.records[-1])
        one = 1 << base.fmt.frac_bits  # int / int: correctly rounded, no float overflow at large F
        final_xyz = np.array([[x / one for x in row] for row in base.ints(base.records.shape[0] - 1)], np.float64)
        kms = {"base": base.kernel_ms, "verify": ver.kernel_ms}
    else:  # more ranks than members: an empty shard still takes part in the gather
        fmt = FixedFormat(bb)
        nrec = n_steps // stride + 1
        steps = np.arange(nrec, dtype=np.int64) * stride
        agr = np.zeros((0, nrec), np.int64)
        tc_step = np.zeros(0, np.int64)
        final_digits = np.zeros((0, len(CANON_INIT), fmt.width), np.int32)
        final_xyz = np.zeros((0, len(CANON_INIT)), np.float64)
        kms = {"base": 0.0, "verify": 0.0}
    if gather and world > 1:
        agr = gather_rows(agr, n_members, world, rank, gather_device)
        tc_step = gather_rows(tc_step, n_members, world, rank, gather_device)
        final_digits = gather_rows(final_digits, n_members, world, rank, gather_device)
        final_xyz = gather_rows(final_xyz, n_members, world, rank, gather_device)
    return SweepReport(K, N, (bb, N), (vb, vn), tau_text, steps, agr, tc_step, final_xyz, final_digits, world, kms)


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
