"""Host MP values: correctly rounded arithmetic checked against MPFR, and the
reference's examples for decimal conversion and digit/bit counts
(/root/reference/pkg/tests/test_mp.py contract)."""

import random
from fractions import Fraction

import pytest

import paper_1908_09301_b200 as M
from oracle import ref as R


def _same(v: M.MPValue, d: R.Dy):
    return v.as_fraction() == R.dy_to_fraction(d)


@pytest.mark.parametrize("bits", [64, 100, 167, 256, 1661])
def test_decimal_parse_matches_mpfr(bits):
    ctx = M.PrecisionContext(bits)
    for text in ("-15.8", "-17.48", "35.64", "0.01", "-0.01", "1e-300", "2.5e-3", "+7", ".5", "123.",
                 "99999999999999999999999.999999999999999999999"):
        assert _same(M.mp_from_decimal(text, ctx), R.from_decimal(text, bits)), text


@pytest.mark.parametrize("bits", [64, 128, 256, 800])
def test_arithmetic_single_rounding_matches_mpfr(bits):
    rnd = random.Random(bits)
    ctx = M.PrecisionContext(bits)
    for _ in range(200):
        a = M.MPValue.from_fraction(Fraction(rnd.randrange(-10**40, 10**40), rnd.randrange(1, 10**25)), bits + 40)
        b = M.MPValue.from_fraction(Fraction(rnd.randrange(-10**40, 10**40), rnd.randrange(1, 10**25)), bits + 40)
        da, db = R.dy_from_fraction(a.as_fraction()), R.dy_from_fraction(b.as_fraction())
        for op in ("add", "sub", "mul"):
            assert _same(getattr(ctx, op)(a, b), R.binop(op, da, db, bits))
        if not b.is_zero():
            assert _same(ctx.div(a, b), R.div(da, db, bits))


def test_eight_thirds_and_digit_counts():
    ctx = M.PrecisionContext(256)
    assert M.mp_to_decimal(ctx.div(ctx.from_int(8), ctx.from_int(3)), 10) == "2.666666667"
    assert M.decimal_digits(8000) == 2408
    assert M.decimal_digits(1) == 0
    assert M.bits_for_digits(800) == 2658
    assert M.bits_for_digits(50) == 167
    assert M.bits_for_digits(500) == 1661


def test_decimal_output_formats():
    ctx = M.PrecisionContext(256)
    assert M.mp_to_decimal(ctx.from_int(2), 5) == "2.0000"
    assert M.mp_to_decimal(ctx.zero, 4) == "0.000"
    assert M.mp_to_decimal(M.mp_from_decimal("-15.8", M.PrecisionContext(8000)), 3) == "-15.8"
    assert M.mp_to_decimal(M.mp_from_decimal("0.001", ctx), 2) == "0.0010"
    assert "e" in M.mp_to_decimal(M.mp_from_decimal("1e-30", ctx), 3)


def test_round_trip_decimal_bit_exact():
    rnd = random.Random(3)
    for bits in (64, 256, 1000):
        ctx = M.PrecisionContext(bits)
        for _ in range(30):
            v = M.MPValue.from_fraction(Fraction(rnd.randrange(-10**30, 10**30), rnd.randrange(1, 10**9)), bits)
            text = M.mp_to_decimal(v, M.decimal_digits(bits) + 2)
            assert M.mp_bits_equal(M.mp_from_decimal(text, ctx), v)


def test_errors():
    ctx = M.PrecisionContext(128)
    with pytest.raises(ValueError):
        M.PrecisionContext(63)
    with pytest.raises(ValueError):
        M.mp_from_decimal("1.2.3", ctx)
    with pytest.raises(ZeroDivisionError):
        ctx.div(ctx.one, ctx.zero)
    with pytest.raises(ValueError):
        M.arith("pow", ctx.one, ctx.one, ctx)
    with pytest.raises(M.RangeError):
        M.mp_from_decimal("1e999999999", ctx)


def test_signed_zero_and_bits_equal():
    ctx = M.PrecisionContext(128)
    nz = ctx.mul(ctx.from_int(-1), ctx.zero)
    assert nz.is_zero() and nz.is_signed()
    assert not M.mp_bits_equal(nz, ctx.zero)
    assert M.mp_to_decimal(nz, 3) == "-0.00"


@pytest.mark.parametrize("K", [50, 500, 4200])
def test_digit_rows_round_trip(K):
    """Batched int -> radix-2^28 digit rows (the H2D format) and back, with the
    width edges; values past the width raise like the reference's range errors."""
    import numpy as np

    from paper_1908_09301_b200.fixed import FixedFormat

    fmt = FixedFormat(M.bits_for_digits(K))
    top = (1 << (28 * fmt.width)) - 1
    rng = random.Random(K)
    xs = [rng.randint(-(1 << (fmt.frac_bits + 20)), 1 << (fmt.frac_bits + 20)) for _ in range(200)]
    xs += [0, 1, -1, top, -top, 1 << 27, -(1 << 28)]
    d = fmt.ints_to_digits(xs)
    assert d.dtype == np.int32 and d.shape == (len(xs), fmt.width) and d.flags.c_contiguous
    assert (np.abs(d) < (1 << 28)).all()
    assert fmt.digits_to_ints(d) == xs
    for r, x in zip(d[:20], xs[:20]):  # digit-by-digit definition
        assert sum(int(v) << (28 * j) for j, v in enumerate(r)) == x
    assert fmt.ints_to_digits([]).shape == (0, fmt.width)
    with pytest.raises(M.RangeError):
        fmt.ints_to_digits([top + 1])
