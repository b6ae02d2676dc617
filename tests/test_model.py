"""The device arithmetic (as restated by oracle/fixmodel.c) against the
reference's frozen outputs: agreement to relative 10^-(K-d) with the
reference's own metric, d(t) guard digits as derived in tests/helpers.py
(accumulated rounding of N orders over 1/(lambda tau) steps plus the Lorenz
system's largest Lyapunov exponent, 0.906 / ln 10 digits per time unit).

These run on the CPU; the GPU is checked bit for bit against the same model
in tests/test_gpu.py, so together they carry the parity claim."""

import math
from fractions import Fraction

import numpy as np
import pytest

import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

from .helpers import agreement_digits, frac, guard_digits, system_from_json


def _small_int_q(tables):
    Lf = tables.q.shape[1] - 1 if len(tables.q) else 0
    return [not r[:Lf].any() and abs(int(r[Lf])) <= 4096 for r in tables.q]


VARIANTS = [0, 1, 2, 3]  # 0: per-order C-product recurrence, 1: matrix recurrence (mx kernel), 2: value-exact matrix
# recurrence (lx kernel), 3: value-exact per-order recurrence (warp kernel)


def run_model(case, guard_bits=32, variant=0):
    P = case["prec_bits"]
    ctx = M.PrecisionContext(P)
    system = system_from_json(case["system"], ctx)
    fmt = FixedFormat(P, guard_bits)
    tau = M.mp_from_decimal(case["tau"], ctx)
    tables = SystemTables.build(system, fmt, case["order"], tau.as_fraction())
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in case["init"]])
    steps, recs = FX.integrate(tables, fmt.frac_digits, case["order"], P, st, case["n_steps"], 0, case["stride"],
                                variant=variant)
    return fmt, steps, recs


@pytest.mark.parametrize(
    "name", ["config0_k50_n40", "cns_pair_128_n20", "cns_pair_256_n30", "config1_k500_n200_3steps",
             "backward_256_n30"]
)
@pytest.mark.parametrize("variant", VARIANTS)
def test_model_matches_reference_within_tolerance(golden, name, variant):
    c = golden[name]
    fmt, steps, recs = run_model(c, variant=variant)
    K = M.decimal_digits(c["prec_bits"])
    tau = float(Fraction(c["tau"]))
    assert [int(s) for s in steps] == [r["step"] for r in c["records"]]
    for r, rec in zip(recs, c["records"]):
        got = fmt.digits_to_fractions(r)
        ref = [frac(h) for h in rec["state"]]
        t = abs(rec["step"] * tau)
        assert agreement_digits(got, ref) >= K - guard_digits(t, c["order"], tau), (name, rec["step"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_model_states_are_reference_precision_values(golden, variant):
    """The device rounds the state to P bits each step: every recorded state
    is a P-bit binary float, like the reference's."""
    c = golden["config0_k50_n40"]
    fmt, _, recs = run_model(c, variant=variant)
    for r in recs[1:]:
        for f in fmt.digits_to_fractions(r):
            v = M.MPValue.from_fraction(f, c["prec_bits"])
            assert v.as_fraction() == f


@pytest.mark.parametrize("variant", VARIANTS)
def test_zero_state_is_a_fixed_point(golden, variant):
    c = golden["zero_state_256_n8"]
    fmt, _, recs = run_model(c, variant=variant)
    assert not recs.any()


@pytest.mark.parametrize("variant", VARIANTS)
def test_jets_match_reference_jets(golden, variant):
    """Model jets (tau-scaled by 2^-7, unscaled exactly) vs the reference's
    jets: each coefficient agrees to the absolute accuracy of the scaled row."""
    for name, c in golden.items():
        if c["kind"] != "jet" or c["prec_bits"] > 300:
            continue
        P, N = c["prec_bits"], c["order"]
        ctx = M.PrecisionContext(P)
        system = system_from_json(c["system"], ctx)
        fmt = FixedFormat(P)
        k = 7
        tables = SystemTables.build(system, fmt, N, Fraction(1, 1 << k))
        st = fmt.to_digits([frac(h) for h in c["state"]])
        if variant >= 1 and not all(_small_int_q(tables)):
            continue
        coef = FX.compute_jet(tables, fmt.frac_digits, N, st, variant=variant)
        for m in range(system.dim):
            fr = fmt.digits_to_fractions(coef[m])
            for i in range(N + 1):
                ref = frac(c["coeffs"][m][i])
                got = fr[i] * (1 << (k * i))
                tol = max(abs(ref), Fraction(1)) * Fraction(1, 2 ** (P - 12)) + Fraction(1 << (k * i), 2 ** (P + 20))
                assert abs(got - ref) <= tol, (name, m, i)


def test_guard_bits_change_nothing_beyond_tolerance(golden):
    c = golden["config0_k50_n40"]
    f32, _, r32 = run_model(c, 32)
    f64, _, r64 = run_model(c, 64)
    for a, b in zip(r32, r64):
        assert agreement_digits(f32.digits_to_fractions(a), f64.digits_to_fractions(b)) >= 40


# ------------------------------------------------------------ error budget
def _oracle_fixture(name):
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", f"oracle_{name}.json")) as fh:
        return json.load(fh)


def test_reference_error_budget_against_p64_oracle():
    """How much of d(t) is the reference's own rounding: the oracle at P bits
    against the same oracle at P + 64 bits (same inputs, same order, so the
    truncation error is shared). The declared d(t) keeps >= 2 digits of margin
    over the reference's measured loss on configs[1], configs[2] and configs[3]."""
    for name in ("config1_k500_n200_10000", "config2_k2200_n1000_500", "config3_k4200_n3500_100"):
        ref, truth = _oracle_fixture(name), _oracle_fixture(name + "_p64")
        assert truth["work_prec_bits"] == ref["prec_bits"] + 64 and truth["order"] == ref["order"]
        K, tau = ref["K"], float(ref["tau"])
        for ra, rb in zip(ref["records"][1:], truth["records"][1:]):
            assert ra["step"] == rb["step"]
            lost = K - agreement_digits([frac(h) for h in ra["state"]], [frac(h) for h in rb["state"]])
            assert 0 <= lost <= guard_digits(ra["step"] * tau, ref["order"], tau) - 2, (name, ra["step"], lost)


@pytest.mark.parametrize("variant", [1, 3])  # the arithmetic of the kernels that run configs[1]-like shapes (mx, warp/block)
def test_model_is_at_least_as_accurate_as_the_reference(variant):
    """configs[1], first 1000 steps (t = 10): the device arithmetic's distance
    from the P + 64-bit oracle equals the reference's own to within one digit
    (the state is rounded to the reference precision P after every step, as the
    reference's is, and that rounding dominates both)."""
    ref = _oracle_fixture("config1_k500_n200_10000")
    truth = _oracle_fixture("config1_k500_n200_10000_p64")
    case = dict(prec_bits=ref["prec_bits"], system=None, tau=ref["tau"], order=ref["order"], init=ref["init"],
                n_steps=1000, stride=1000)
    P = case["prec_bits"]
    ctx = M.PrecisionContext(P)
    fmt = FixedFormat(P)
    tables = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, case["order"],
                                M.mp_from_decimal(case["tau"], ctx).as_fraction())
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in case["init"]])
    _, recs = FX.integrate(tables, fmt.frac_digits, case["order"], P, st, 1000, 0, 1000, variant=variant)
    got = fmt.digits_to_fractions(recs[-1])
    tr = [frac(h) for h in truth["records"][1]["state"]]
    rf = [frac(h) for h in ref["records"][1]["state"]]
    assert truth["records"][1]["step"] == 1000
    e_model, e_ref = agreement_digits(got, tr), agreement_digits(rf, tr)
    assert e_model >= e_ref - 1, (e_model, e_ref)
    assert agreement_digits(got, rf) >= min(e_model, e_ref) - 1
