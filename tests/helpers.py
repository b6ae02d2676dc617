"""Shared helpers for the test-suite (exact arithmetic only)."""

from __future__ import annotations

import math
from fractions import Fraction

from oracle import ref as R

EXACT = math.inf

# ---------------------------------------------------------------------------
# Declared tolerance. Two correct integrations of the same chaotic system that
# round differently (the reference rounds every multiply and add to P bits;
# the device carries 32 more bits and rounds once per sum) separate as
#     e(t) ~ u * c * sum_s exp(lambda (t - s tau)) ~ u * c * exp(lambda t) / (lambda tau),
# u = 10^-K, lambda = the largest Lyapunov exponent (0.906 for the Lorenz
# attractor), c <= N the rounding error of one step in ulps (N accumulated
# orders). In decimal digits:
#     d(t) = ceil(log10(N / (lambda |tau|))) + ceil(1.05 * lambda t / ln 10)
# (5 % on the slope for the finite-time fluctuation of the exponent). Measured
# against the oracle re-run at P + 64 bits (tests/golden/*_p64.json,
# profiles/r02_error_budget.json) the REFERENCE ITSELF loses 42 of its 500
# digits by t = 100 and d(100) = 47; the test bound is this d(t) everywhere.
LYAPUNOV = 0.906


def guard_digits(t: float, order: int, tau: float = 0.01) -> int:
    return math.ceil(math.log10(order / (LYAPUNOV * abs(tau)))) + math.ceil(1.05 * LYAPUNOV / math.log(10) * abs(t))


def frac(hexval: str) -> Fraction:
    return R.dy_to_fraction(R.dy_from_hex(hexval))


def floor_neg_log10(rel: Fraction) -> int:
    """Largest d >= 0 with rel <= 10^-d (exact)."""
    if rel >= 1:
        return 0
    d = 0
    while rel * 10 ** (d + 1) <= 1:
        d += 1
    return d


def agreement_digits(a, b) -> float:
    """The reference's coincidence metric (cns.py:52 agreement_digits):
    min over components of floor(-log10(|a-b| / max(|a|, |b|, 1))), EXACT
    when all components are identical."""
    worst = None
    for x, y in zip(a, b):
        x, y = Fraction(x), Fraction(y)
        if x == y:
            continue
        d = floor_neg_log10(abs(x - y) / max(abs(x), abs(y), Fraction(1)))
        worst = d if worst is None else min(worst, d)
    return EXACT if worst is None else worst


def system_from_json(js, ctx):
    """Reference-fixture system description -> product QuadraticODESystem (exact values)."""
    import paper_1908_09301_b200 as M

    P = ctx.precision_bits

    def mv(h):
        d = R.dy_from_hex(h)
        return M.MPValue(d.sign, d.mant, d.exp, P)

    dim = js["dim"]
    bil = [[] for _ in range(dim)]
    for m, j, k, h in js["terms"]:
        bil[m].append(M.BilinearTerm(j, k, mv(h)))
    return M.QuadraticODESystem(
        dim=dim,
        constant=tuple(mv(h) for h in js["constant"]),
        linear=tuple(tuple(mv(h) for h in row) for row in js["linear"]),
        bilinear=tuple(tuple(t) for t in bil),
    )


def mp_of_hex(h, prec):
    import paper_1908_09301_b200 as M

    d = R.dy_from_hex(h)
    return M.MPValue(d.sign, d.mant, d.exp, prec)
