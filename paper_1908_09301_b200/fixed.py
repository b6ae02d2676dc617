"""The device number format: fixed-point digit rows of radix 2^28.

A value is X * 2^-F with F = 28 * Lf fractional bits and X = sum_j d_j 2^(28 j)
over W = Lf + 1 signed digits |d_j| < 2^28 that all carry the sign of X
(DESIGN.md §3). Lf is chosen so that F >= P + guard_bits, P being the
reference precision (mp.py:44 PrecisionContext.precision_bits): every P-bit
value the reference produces with magnitude >= 2^-guard_bits is exact in this
format, and the absolute resolution is 2^-guard_bits finer than the
reference's ulp at magnitude 1 -- the scale of the reference's own agreement
metric (cns.py agreement_digits uses max(|a|, |b|, 1)).

Conversions here run on the host once per launch (inputs, constant tables,
outputs); the per-order arithmetic never leaves the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .mp import MPValue, RangeError

RADIX_BITS = 28
RADIX = 1 << RADIX_BITS
DEFAULT_GUARD_BITS = 32
# |value| < 2^MAX_INT_BITS keeps every column sum far from int64 overflow
MAX_INT_BITS = 27


def _round_div(num: int, den: int) -> int:
    """round-half-even(num / den), den > 0."""
    q, r = divmod(num, den)
    twice = 2 * r
    if twice > den or (twice == den and q & 1):
        q += 1
    return q


_CTAB_CACHE: dict = {}  # (frac_bits, width, step, order) -> read-only digit table


@dataclass(frozen=True)
class FixedFormat:
    prec_bits: int
    guard_bits: int = DEFAULT_GUARD_BITS

    @property
    def frac_digits(self) -> int:
        return -(-(self.prec_bits + self.guard_bits) // RADIX_BITS)

    @property
    def frac_bits(self) -> int:
        return RADIX_BITS * self.frac_digits

    @property
    def width(self) -> int:
        return self.frac_digits + 1

    # ------------------------------------------------------------ scalars
    def to_int(self, v) -> int:
        """Nearest X (ties to even) with X * 2^-F ~= v; v MPValue or Fraction."""
        f = v.as_fraction() if isinstance(v, MPValue) else Fraction(v)
        x = _round_div(f.numerator << self.frac_bits, f.denominator)
        if abs(x) >> (self.frac_bits + MAX_INT_BITS):
            raise RangeError(f"|value| >= 2^{MAX_INT_BITS} does not fit the device format")
        return x

    def is_exact(self, v) -> bool:
        f = v.as_fraction() if isinstance(v, MPValue) else Fraction(v)
        return Fraction(self.to_int(f), 1 << self.frac_bits) == f

    def int_to_fraction(self, x: int) -> Fraction:
        return Fraction(x, 1 << self.frac_bits)

    # ------------------------------------------------------------- digits
    def ints_to_digits(self, xs) -> np.ndarray:
        """Signed integers -> int32 digit rows (len(xs) x W)."""
        W = self.width
        xs = [int(x) for x in xs]
        if not xs:
            return np.zeros((0, W), dtype=np.int32)
        nbytes = (RADIX_BITS * W + 7) // 8 + 1
        mags = [abs(x) for x in xs]
        if any(m >> (RADIX_BITS * W) for m in mags):
            raise RangeError("value exceeds the digit width")
        # all rows at once: little-endian bytes -> bits -> radix-2^28 digits
        raw = np.frombuffer(b"".join(m.to_bytes(nbytes + 4, "little") for m in mags), dtype=np.uint8)
        raw = raw.reshape(len(xs), nbytes + 4).astype(np.int64)
        off = RADIX_BITS * np.arange(W)
        b0, sh = off // 8, off % 8  # digit j = 4 bytes from byte b0, shifted right by sh
        word = raw[:, b0] | (raw[:, b0 + 1] << 8) | (raw[:, b0 + 2] << 16) | (raw[:, b0 + 3] << 24) | (
            raw[:, b0 + 4] << 32)
        d = (word >> sh) & ((1 << RADIX_BITS) - 1)
        neg = np.fromiter((x < 0 for x in xs), dtype=bool, count=len(xs))
        return np.ascontiguousarray(np.where(neg[:, None], -d, d), dtype=np.int32)

    def digits_to_ints(self, rows) -> list:
        """Digit rows -> integers. Canonical rows (every digit carries the
        value's sign) are packed through their bit patterns (vectorised);
        other rows take the exact digit-by-digit path."""
        rows = np.asarray(rows, dtype=np.int64).reshape(-1, self.width)
        if rows.shape[0] == 0:
            return []
        neg = (rows < 0).any(axis=1)
        canon = ~(neg & (rows > 0).any(axis=1)) & (np.abs(rows) < (1 << RADIX_BITS)).all(axis=1)
        mags = np.abs(rows).astype("<u4")
        bits = np.unpackbits(mags.view(np.uint8).reshape(rows.shape[0], self.width, 4), axis=2,
                             bitorder="little")[:, :, :RADIX_BITS].reshape(rows.shape[0], -1)
        packed = np.packbits(bits, axis=1, bitorder="little")
        out = []
        for r in range(rows.shape[0]):
            if canon[r]:
                x = int.from_bytes(packed[r].tobytes(), "little")
                out.append(-x if neg[r] else x)
            else:
                x = 0
                for d in reversed(rows[r].tolist()):
                    x = (x << RADIX_BITS) + d
                out.append(x)
        return out

    def to_digits(self, values) -> np.ndarray:
        return self.ints_to_digits([self.to_int(v) for v in values])

    def digits_to_fractions(self, rows) -> list:
        return [self.int_to_fraction(x) for x in self.digits_to_ints(rows)]

    # --------------------------------------------------------- tau tables
    @staticmethod
    def c_shift(scale: Fraction) -> int:
        a = abs(Fraction(scale))
        if a == 0:
            raise ValueError("step size must be nonzero")
        if a >= Fraction(1 << (MAX_INT_BITS - 1)):
            raise RangeError("step size too large for the device format")
        return 1 if a < Fraction(1, 4) else 0

    def ctab_ints(self, scale: Fraction, order: int) -> list:
        """round(scale * 2^(F + 28 sc) / (i+1)), i = 0..order-1 (ties to even)."""
        scale = Fraction(scale)
        sc = self.c_shift(scale)
        num = scale.numerator << (self.frac_bits + RADIX_BITS * sc)
        den = scale.denominator
        return [_round_div(num, den * (i + 1)) for i in range(order)]

    def ctab(self, scale: Fraction, order: int) -> np.ndarray:
        """The tau/(i+1) digit table; memoised per (format, step, order): at K = 4200,
        N = 3500 it is 3500 divisions of 14 000-bit integers, repeated by every
        integrate() call on the same step size otherwise."""
        key = (self.frac_bits, self.width, Fraction(scale), order)
        hit = _CTAB_CACHE.get(key)
        if hit is None:
            hit = self.ints_to_digits(self.ctab_ints(scale, order))
            hit.setflags(write=False)
            if len(_CTAB_CACHE) >= 16:
                _CTAB_CACHE.pop(next(iter(_CTAB_CACHE)))
            _CTAB_CACHE[key] = hit
        return hit
