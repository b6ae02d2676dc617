"""Host-side multiple-precision values: contexts, creation, arithmetic, conversion.

Mirror of the reference module /root/reference/pkg/src/mptaylor/mp.py (same
names, argument meaning and errors). The reference wraps MPFR through gmpy2;
this image has no gmpy2, and the host side only needs MP arithmetic for
plumbing (parsing decimal initial data, building system coefficients such as
b = 8/3, formatting output), so the value type here is a small exact-dyadic
class with correctly rounded (round-to-nearest-even) operations written on
Python integers. The hot path never touches it: it runs on the device in the
fixed-point digit format of paper_1908_09301_b200.fixed.

Rounding is to nearest, ties to even, exactly once per operation -- the MPFR
contract the reference relies on (mp.py:1 module docstring). Tests check
these operations bit for bit against the system MPFR library.
"""

from __future__ import annotations

import re
from fractions import Fraction

MIN_PRECISION_BITS = 64
_EMAX = 2**30 - 1
_EMIN = -(2**30 - 1)
_DECIMAL_RE = re.compile(r"^[+-]?(\d+(\.\d*)?|\.\d+)([eE][+-]?\d+)?$")


class RangeError(ArithmeticError):
    """A value fell outside the supported binary exponent range."""


def _round_scaled(sign: int, num: int, den: int, prec: int):
    """RN-even of sign*num/den (num, den > 0) to `prec` bits -> (mant, exp)."""
    # binade: 2^(e-1) <= num/den < 2^e
    def ge_pow2(k):  # num/den >= 2^k
        return (num << max(0, -k)) >= (den << max(0, k))

    e = num.bit_length() - den.bit_length() + 1
    while not ge_pow2(e - 1):
        e -= 1
    while ge_pow2(e):
        e += 1
    # scaled = num/den * 2^(prec - e) in [2^(prec-1), 2^prec)
    shift = prec - e
    if shift >= 0:
        q, r = divmod(num << shift, den)
    else:
        q, r = divmod(num, den << (-shift))
    half = 2 * r
    dd = den if shift >= 0 else den << (-shift)
    if half > dd or (half == dd and (q & 1)):
        q += 1
    exp = -shift
    if q.bit_length() > prec:  # carried into a new binade
        q >>= 1
        exp += 1
    return q, exp


class MPValue:
    """Immutable binary floating-point value: sign * mant * 2**exp at `precision` bits.

    `mant` is stored reduced (odd, or 0). Zeros keep their sign, like MPFR.
    """

    __slots__ = ("sign", "mant", "exp", "precision")

    def __init__(self, sign: int, mant: int, exp: int, precision: int):
        if mant < 0:
            raise ValueError("mantissa must be non-negative")
        if mant:
            tz = (mant & -mant).bit_length() - 1
            mant >>= tz
            exp += tz
            if mant.bit_length() > precision:
                raise ValueError("mantissa exceeds precision")
            top = exp + mant.bit_length()
            if top > _EMAX or top < _EMIN:
                raise RangeError(f"binary exponent {top} out of range")
        else:
            exp = 0
        object.__setattr__(self, "sign", -1 if sign < 0 else 1)
        object.__setattr__(self, "mant", mant)
        object.__setattr__(self, "exp", exp)
        object.__setattr__(self, "precision", int(precision))

    def __setattr__(self, *_):
        raise AttributeError("MPValue is immutable")

    # --- constructors -------------------------------------------------------
    @classmethod
    def from_fraction(cls, f: Fraction, prec: int) -> "MPValue":
        f = Fraction(f)
        if f == 0:
            return cls(1, 0, 0, prec)
        sign = 1 if f > 0 else -1
        mant, exp = _round_scaled(sign, abs(f.numerator), f.denominator, prec)
        return cls(sign, mant, exp, prec)

    @classmethod
    def from_dyadic(cls, sign: int, mant: int, exp: int, prec: int) -> "MPValue":
        """RN-even of sign*mant*2^exp to prec bits (exact when it fits)."""
        if mant == 0:
            return cls(sign, 0, 0, prec)
        if mant.bit_length() <= prec:
            return cls(sign, mant, exp, prec)
        m, e = _round_scaled(sign, mant, 1, prec)
        return cls(sign, m, e + exp, prec)

    # --- exact views ---------------------------------------------------------
    def is_zero(self) -> bool:
        return self.mant == 0

    def is_signed(self) -> bool:
        return self.sign < 0

    def as_fraction(self) -> Fraction:
        if self.mant == 0:
            return Fraction(0)
        if self.exp >= 0:
            return Fraction(self.sign * (self.mant << self.exp))
        return Fraction(self.sign * self.mant, 1 << (-self.exp))

    def as_integer_ratio(self):
        f = self.as_fraction()
        return f.numerator, f.denominator

    def as_mantissa_exp(self):
        """(significand with exactly `precision` bits, exponent), like gmpy2/MPFR."""
        if self.mant == 0:
            return 0, 0
        s = self.precision - self.mant.bit_length()
        return self.sign * (self.mant << s), self.exp - s

    def __float__(self) -> float:
        return float(self.as_fraction())

    def __eq__(self, other):
        if isinstance(other, MPValue):
            return self.as_fraction() == other.as_fraction()
        if isinstance(other, (int, Fraction)):
            return self.as_fraction() == other
        return NotImplemented

    def __lt__(self, other):
        o = other.as_fraction() if isinstance(other, MPValue) else Fraction(other)
        return self.as_fraction() < o

    def __hash__(self):
        return hash(self.as_fraction())

    def __repr__(self):
        return f"MPValue({mp_to_decimal(self, 20)!r}, {self.precision})"

    def __str__(self):
        return mp_to_decimal(self, max(1, decimal_digits(self.precision)))


class PrecisionContext:
    """A fixed working precision (bits of significand), rounding to nearest-even.

    Mirrors mptaylor.mp.PrecisionContext (mp.py:44): contexts are immutable,
    compare by bit count, and every operation rounds exactly once.
    """

    __slots__ = ("precision_bits", "zero", "one")

    def __init__(self, precision_bits: int):
        if not isinstance(precision_bits, int) or isinstance(precision_bits, bool):
            raise TypeError(f"precision_bits must be an int, got {precision_bits!r}")
        if precision_bits < MIN_PRECISION_BITS:
            raise ValueError(
                f"precision_bits must be >= {MIN_PRECISION_BITS}, got {precision_bits}"
            )
        object.__setattr__(self, "precision_bits", precision_bits)
        object.__setattr__(self, "zero", MPValue(1, 0, 0, precision_bits))
        object.__setattr__(self, "one", MPValue(1, 1, 0, precision_bits))

    def __setattr__(self, *_):
        raise AttributeError("PrecisionContext is immutable")

    def _coerce(self, x) -> Fraction:
        if isinstance(x, MPValue):
            return x.as_fraction()
        if isinstance(x, (int, Fraction)):
            return Fraction(x)
        raise TypeError(f"unsupported operand {x!r}")

    def _signed_zero(self, a, b, op) -> MPValue:
        sa = a.sign if isinstance(a, MPValue) else (1 if a >= 0 else -1)
        sb = b.sign if isinstance(b, MPValue) else (1 if b >= 0 else -1)
        if op == "mul" or op == "div":
            return MPValue(sa * sb, 0, 0, self.precision_bits)
        if op == "sub":
            sb = -sb
        return MPValue(sa if sa == sb else 1, 0, 0, self.precision_bits)

    def _result(self, f: Fraction, a, b, op) -> MPValue:
        if f == 0:
            return self._signed_zero(a, b, op)
        return MPValue.from_fraction(f, self.precision_bits)

    def add(self, a, b) -> MPValue:
        return self._result(self._coerce(a) + self._coerce(b), a, b, "add")

    def sub(self, a, b) -> MPValue:
        return self._result(self._coerce(a) - self._coerce(b), a, b, "sub")

    def mul(self, a, b) -> MPValue:
        return self._result(self._coerce(a) * self._coerce(b), a, b, "mul")

    def div(self, a, b) -> MPValue:
        fb = self._coerce(b)
        if fb == 0:
            raise ZeroDivisionError("division by zero")
        return self._result(self._coerce(a) / fb, a, b, "div")

    def neg(self, a) -> MPValue:
        if isinstance(a, MPValue):
            return MPValue.from_dyadic(-a.sign, a.mant, a.exp, self.precision_bits)
        return self.from_int(-a)

    def mul_2exp(self, a, e: int) -> MPValue:
        return MPValue.from_dyadic(a.sign, a.mant, a.exp + e, self.precision_bits)

    def from_int(self, n: int) -> MPValue:
        if n == 0:
            return self.zero
        return MPValue.from_dyadic(1 if n > 0 else -1, abs(n), 0, self.precision_bits)

    def parse(self, text: str) -> MPValue:
        return mp_from_decimal(text, self)

    def __eq__(self, other) -> bool:
        return isinstance(other, PrecisionContext) and other.precision_bits == self.precision_bits

    def __hash__(self) -> int:
        return hash(("PrecisionContext", self.precision_bits))

    def __repr__(self) -> str:
        return f"PrecisionContext({self.precision_bits})"


def mp_from_decimal(text: str, ctx: PrecisionContext) -> MPValue:
    """Parse a decimal string to the nearest representable value (mp.py:122)."""
    if not isinstance(text, str):
        raise ValueError(f"decimal text must be a string, got {type(text).__name__}")
    stripped = text.strip()
    if not _DECIMAL_RE.match(stripped):
        raise ValueError(f"not a valid decimal literal: {text!r}")
    neg = stripped.startswith("-")
    body = stripped.lstrip("+-")
    mant_txt, _, exp_txt = body.replace("E", "e").partition("e")
    e10 = int(exp_txt) if exp_txt else 0
    whole, _, frac = mant_txt.partition(".")
    digits = int((whole or "0") + frac) if (whole or frac) else 0
    e10 -= len(frac)
    if digits == 0:
        return MPValue(-1 if neg else 1, 0, 0, ctx.precision_bits)
    # decimal magnitude ~ 10^(len(digits) + e10): reject before building huge powers
    approx_bits = (len(str(digits)) + e10) * 3.3219280948873626
    if approx_bits > _EMAX + 8 or approx_bits < _EMIN - 8:
        raise RangeError(f"decimal exponent out of range: {text!r}")
    f = Fraction(digits) * (Fraction(10) ** e10)
    if neg:
        f = -f
    try:
        return MPValue.from_fraction(f, ctx.precision_bits)
    except RangeError as exc:
        raise RangeError(f"decimal exponent out of range: {text!r}") from exc


def _decimal_digits_of(f: Fraction, n: int):
    """Correctly rounded (ties-to-even) n significant digits of f > 0.

    Returns (digit string, exp10) with f ~= 0.<digits> * 10**exp10.
    """
    num, den = f.numerator, f.denominator
    # exp10 such that 10^(exp10-1) <= f < 10^exp10
    exp10 = len(str(num)) - len(str(den))
    while True:
        lo = Fraction(10) ** (exp10 - 1)
        if f < lo:
            exp10 -= 1
        elif f >= lo * 10:
            exp10 += 1
        else:
            break
    scaled = f * (Fraction(10) ** (n - exp10))
    q, r = divmod(scaled.numerator, scaled.denominator)
    if 2 * r > scaled.denominator or (2 * r == scaled.denominator and q % 2 == 1):
        q += 1
    text = str(q)
    if len(text) > n:
        exp10 += 1
        text = text[:n]
    return text, exp10


def mp_to_decimal(v: MPValue, digits: int) -> str:
    """Correctly rounded decimal with `digits` significant digits (mp.py:146)."""
    if not isinstance(digits, int) or isinstance(digits, bool) or digits < 1:
        raise ValueError(f"digits must be a positive integer, got {digits!r}")
    if v.is_zero():
        sign = "-" if v.is_signed() else ""
        if digits == 1:
            return sign + "0"
        return sign + "0." + "0" * (digits - 1)
    f = v.as_fraction()
    sign = "-" if f < 0 else ""
    mant, exp10 = _decimal_digits_of(abs(f), digits)
    if 0 < exp10 <= len(mant):
        whole, frac = mant[:exp10], mant[exp10:]
        return sign + (whole + "." + frac if frac else whole)
    if -4 < exp10 <= 0:
        return sign + "0." + "0" * (-exp10) + mant
    if len(mant) == 1:
        return f"{sign}{mant}e{exp10 - 1}"
    return f"{sign}{mant[0]}.{mant[1:]}e{exp10 - 1}"


_ARITH_OPS = ("add", "sub", "mul", "div")


def arith(op: str, a: MPValue, b: MPValue, ctx: PrecisionContext) -> MPValue:
    """One of add/sub/mul/div with a single rounding (mp.py:178)."""
    if op not in _ARITH_OPS:
        raise ValueError(f"unknown operation {op!r}, expected one of {_ARITH_OPS}")
    return getattr(ctx, op)(a, b)


def decimal_digits(precision_bits: int) -> int:
    """floor(precision_bits * log10 2), exactly (mp.py:189)."""
    if not isinstance(precision_bits, int) or isinstance(precision_bits, bool):
        raise TypeError(f"precision_bits must be an int, got {precision_bits!r}")
    if precision_bits < 1:
        raise ValueError(f"precision_bits must be >= 1, got {precision_bits}")
    d = int(precision_bits * 0.30102999566398114)
    target = 1 << precision_bits
    while 10 ** (d + 1) <= target:
        d += 1
    while d > 0 and 10**d > target:
        d -= 1
    return d


def bits_for_digits(digits: int) -> int:
    """Smallest p with 2**p >= 10**digits (mp.py:209)."""
    if not isinstance(digits, int) or isinstance(digits, bool):
        raise TypeError(f"digits must be an int, got {digits!r}")
    if digits < 1:
        raise ValueError(f"digits must be >= 1, got {digits}")
    p = int(digits * 3.321928094887362)
    target = 10**digits
    while (1 << p) < target:
        p += 1
    while p > 1 and (1 << (p - 1)) >= target:
        p -= 1
    return p


def mp_bits_equal(a: MPValue, b: MPValue) -> bool:
    """Identical bit patterns, -0 != +0, precision must match (mp.py:229)."""
    if a.precision != b.precision:
        return False
    if a.is_zero() or b.is_zero():
        return a.is_zero() and b.is_zero() and a.is_signed() == b.is_signed()
    return (a.sign, a.mant, a.exp) == (b.sign, b.mant, b.exp)
