"""Shared helpers for the test-suite (exact arithmetic only)."""

from __future__ import annotations

import math
from fractions import Fraction

from oracle import ref as R

EXACT = math.inf


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
