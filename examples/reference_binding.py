"""Reference-side binding of the B200 engine: a ctypes stub over the C ABI
(include/mptaylor_b200.h) that a maintainer of the reference package would add
as `mptaylor/_b200.py` to swap the stepping loop of taylor.py:202 integrate
while keeping the reference's own objects.

It depends on nothing from this repository but `libmptaylor_b200.so`: systems
are the reference's QuadraticODESystem (constant / linear / bilinear with
.j, .k, .coeff), values are anything with `as_integer_ratio()` (gmpy2.mpfr has
it), and the result is a list of (step, [(numerator, denominator_log2), ...])
that the caller turns back into its value type (exact: every state already has
at most P significant bits).

    records = integrate_b200(lib_path, system, state0, "0.01", order, n_steps, prec_bits)
"""

from __future__ import annotations

import ctypes
from fractions import Fraction

RADIX_BITS = 28
GUARD_BITS = 32
MPT_ERANGE = -5


def _round_div(num: int, den: int) -> int:
    q, r = divmod(num, den)
    return q + (1 if 2 * r > den or (2 * r == den and q & 1) else 0)


def _to_fixed(value, frac_bits: int) -> int:
    n, d = value.as_integer_ratio() if hasattr(value, "as_integer_ratio") else (Fraction(value).numerator, Fraction(value).denominator)
    return _round_div(int(n) << frac_bits, int(d))


def _round_to_bits(fr: Fraction, bits: int) -> Fraction:
    """fr rounded to `bits` significant bits, ties to even (what mpfr(text, precision) does)."""
    if fr == 0:
        return fr
    n, d = abs(fr.numerator), fr.denominator
    s = bits + d.bit_length() - n.bit_length() + 1
    for _ in range(3):
        q = _round_div(n << s, d) if s >= 0 else _round_div(n, d << -s)
        if q.bit_length() <= bits:
            break
        s -= 1
    val = Fraction(q, 1 << s) if s >= 0 else Fraction(q << -s)
    return -val if fr < 0 else val


def _digits(x: int, width: int) -> list:
    sign, mag = (-1, -x) if x < 0 else (1, x)
    return [sign * ((mag >> (RADIX_BITS * j)) & ((1 << RADIX_BITS) - 1)) for j in range(width)]


def _from_digits(row) -> int:
    x = 0
    for d in reversed(row):
        x = (x << RADIX_BITS) + d
    return x


def integrate_b200(lib_path, system, state0, tau_text, order, n_steps, prec_bits, record_stride=100, start_step=0, device=0):
    lib = ctypes.CDLL(lib_path)
    lib.mpt_last_error.restype = ctypes.c_char_p
    i32p = ctypes.POINTER(ctypes.c_int32)

    def arr(values):
        return (ctypes.c_int32 * len(values))(*values)

    def check(rc):
        if rc < 0:
            msg = lib.mpt_last_error().decode()
            raise (ArithmeticError if rc == MPT_ERANGE else RuntimeError)(f"mptaylor_b200 error {rc}: {msg}")
        return rc

    # 1. fixed-point format: Lf fractional radix-2^28 digits with F = 28 Lf >= P + 32, W = Lf + 1
    lf = -(-(prec_bits + GUARD_BITS) // RADIX_BITS)
    width, frac_bits = lf + 1, RADIX_BITS * lf
    # 2. the system's constants and the tau/(i+1) table as digit rows (round to nearest even)
    terms = [(m, t.j, t.k, t.coeff) for m, row in enumerate(system.bilinear) for t in row]
    flat = lambda values: [d for v in values for d in _digits(_to_fixed(v, frac_bits), width)]
    cst = arr(flat(system.constant))
    lin = arr(flat([v for row in system.linear for v in row]))
    q = arr(flat([t[3] for t in terms]) or [0] * width)
    tau = _round_to_bits(Fraction(tau_text), prec_bits)  # the reference steps with tau rounded to P bits (taylor.py:234)
    c_shift = 1 if abs(tau) < Fraction(1, 4) else 0
    num = tau.numerator << (frac_bits + RADIX_BITS * c_shift)
    ctab = arr([d for i in range(order) for d in _digits(_round_div(num, tau.denominator * (i + 1)), width)])
    # 3. plan: taylor.py:234-239 (tau, product pairs) and the reducer session
    plan = ctypes.c_void_p()
    teq, tj, tk = (arr([t[c] for t in terms] or [0]) for c in range(3))
    check(lib.mpt_plan_create(ctypes.byref(plan), system.dim, len(terms), teq, tj, tk, lf, c_shift, order,
                              prec_bits, 1, device))
    try:
        check(lib.mpt_plan_set_constants(plan, cst, lin, q, ctab))
        # 4. the stepping loop: taylor.py:242-253
        nrec = check(lib.mpt_record_count(n_steps, start_step, record_stride))
        st = arr(flat(state0))
        rec_steps = (ctypes.c_int32 * nrec)()
        records = (ctypes.c_int32 * (nrec * system.dim * width))()
        status = (ctypes.c_int32 * 1)()
        check(lib.mpt_integrate(plan, st, n_steps, start_step, record_stride, rec_steps, records, status))
    finally:
        lib.mpt_plan_destroy(plan)
    # 5. digit rows -> exact dyadic values numerator * 2^-frac_bits
    out = []
    for r in range(nrec):
        row = []
        for m in range(system.dim):
            base = (r * system.dim + m) * width
            row.append((_from_digits(records[base:base + width]), frac_bits))
        out.append((int(rec_steps[r]), row))
    return out
