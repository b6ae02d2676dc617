"""ctypes front end of the CPU oracle (reference semantics on MPFR).

TEST INFRASTRUCTURE ONLY. Importable from tests/, __graft_entry__.smoke()
and bench.py (cpu_baseline and --impl reference legs) -- never from the
product package. The product path fails loudly without its CUDA library and
has no route into this module.

Values are exact dyadics ``Dy(sign, mant, exp)`` = sign * mant * 2**exp,
sign in {+1, -1} (kept for zeros so -0 survives), mant >= 0. The system
description mirrors the reference's QuadraticODESystem
(/root/reference/pkg/src/mptaylor/systems.py:32): dense constant vector,
dense linear matrix, bilinear terms per equation in stored order.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from collections import namedtuple
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_mpfr.so")

Dy = namedtuple("Dy", "sign mant exp")

_lib = None


def build():
    """Compile the oracle libraries with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.ref_mpfr_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def mpfr_version() -> str:
    return lib().ref_mpfr_version().decode()


# ---------------------------------------------------------------- values
def dy_from_fraction(f: Fraction) -> Dy:
    """Exact dyadic of a dyadic rational (raises if the denominator is not 2^k)."""
    f = Fraction(f)
    if f == 0:
        return Dy(1, 0, 0)
    den = f.denominator
    if den & (den - 1):
        raise ValueError(f"{f} is not dyadic")
    e = -(den.bit_length() - 1)
    m = abs(f.numerator)
    tz = (m & -m).bit_length() - 1
    return Dy(1 if f > 0 else -1, m >> tz, e + tz)


def dy_to_fraction(v: Dy) -> Fraction:
    return v.sign * Fraction(v.mant) * (Fraction(2) ** v.exp)


def dy_normal(v: Dy) -> Dy:
    """Canonical form: odd mantissa (or zero with exp 0)."""
    if v.mant == 0:
        return Dy(v.sign, 0, 0)
    tz = (v.mant & -v.mant).bit_length() - 1
    return Dy(v.sign, v.mant >> tz, v.exp + tz)


def dy_hex(v: Dy) -> str:
    """Stable text form used by the golden fixtures: [-]hexmant p exp (odd mant)."""
    v = dy_normal(v)
    s = "-" if v.sign < 0 else ""
    return f"{s}{v.mant:x}p{v.exp}"


def dy_from_hex(text: str) -> Dy:
    neg = text.startswith("-")
    body = text[1:] if neg else text
    m, e = body.split("p")
    return Dy(-1 if neg else 1, int(m, 16), int(e))


def _nlimbs(values) -> int:
    return max([1] + [(v.mant.bit_length() + 63) // 64 for v in values])


def _pack(values, nl=None):
    values = list(values)
    nl = nl or _nlimbs(values)
    n = len(values)
    sgn = (ctypes.c_int32 * max(n, 1))()
    ex = (ctypes.c_int64 * max(n, 1))()
    limbs = (ctypes.c_uint64 * max(n * nl, 1))()
    mask = (1 << 64) - 1
    for i, v in enumerate(values):
        if v.mant == 0:
            sgn[i] = 0 if v.sign > 0 else -2
            ex[i] = 0
            continue
        sgn[i] = 1 if v.sign > 0 else -1
        ex[i] = v.exp
        m = v.mant
        for j in range(nl):
            limbs[i * nl + j] = m & mask
            m >>= 64
        if m:
            raise ValueError("mantissa exceeds limb budget")
    return sgn, ex, limbs, nl


def _out(n, nl):
    return (
        (ctypes.c_int32 * max(n, 1))(),
        (ctypes.c_int64 * max(n, 1))(),
        (ctypes.c_uint64 * max(n * nl, 1))(),
    )


def _unpack(sgn, ex, limbs, n, nl):
    out = []
    for i in range(n):
        s = sgn[i]
        if s in (0, -2):
            out.append(Dy(1 if s == 0 else -1, 0, 0))
            continue
        m = 0
        for j in reversed(range(nl)):
            m = (m << 64) | limbs[i * nl + j]
        out.append(Dy(1 if s > 0 else -1, m, ex[i]))
    return out


def _onl(prec):
    return (prec + 63) // 64 + 1


# ------------------------------------------------------------ conversions
def from_decimal(text: str, prec: int) -> Dy:
    """RN_prec of a decimal literal (mp.py:122 mp_from_decimal on MPFR)."""
    onl = _onl(prec)
    s, e, l = _out(1, onl)
    rc = lib().ref_from_decimal(prec, text.strip().encode(), s, e, l, onl)
    if rc:
        raise ValueError(f"not a decimal: {text!r}")
    return _unpack(s, e, l, 1, onl)[0]


def from_int(n: int, prec: int) -> Dy:
    return from_decimal(str(n), prec)


def div(a: Dy, b: Dy, prec: int) -> Dy:
    sgn, ex, limbs, nl = _pack([a, b])
    onl = _onl(prec)
    s, e, l = _out(1, onl)
    if lib().ref_div(prec, sgn, ex, limbs, nl, s, e, l, onl):
        raise ArithmeticError("division failed")
    return _unpack(s, e, l, 1, onl)[0]


def binop(op: str, a: Dy, b: Dy, prec: int) -> Dy:
    code = {"add": 0, "sub": 1, "mul": 2}[op]
    sgn, ex, limbs, nl = _pack([a, b])
    onl = _onl(prec)
    s, e, l = _out(1, onl)
    if lib().ref_binop(prec, code, sgn, ex, limbs, nl, s, e, l, onl):
        raise ArithmeticError("binop failed")
    return _unpack(s, e, l, 1, onl)[0]


def neg(v: Dy) -> Dy:
    return Dy(-v.sign, v.mant, v.exp)


# ---------------------------------------------------------------- systems
def lorenz(prec: int, sigma=10, r=28, b_num=8, b_den=3):
    """systems.py:94 lorenz_system with LorenzParams.default (systems.py:84)."""
    zero = Dy(1, 0, 0)
    one = from_int(1, prec)
    s = from_int(sigma, prec)
    big_r = from_int(r, prec)
    b = div(from_int(b_num, prec), from_int(b_den, prec), prec)
    return {
        "dim": 3,
        "constant": [zero, zero, zero],
        "linear": [[neg(s), s, zero], [big_r, neg(one), zero], [zero, zero, neg(b)]],
        "terms": [(1, 0, 2, neg(one)), (2, 0, 1, one)],
    }


def _sys_pack(system, extra):
    dim = system["dim"]
    terms = sorted(enumerate(system["terms"]), key=lambda it: (it[1][0], it[0]))
    terms = [t for _, t in terms]
    vals = list(system["constant"]) + [v for row in system["linear"] for v in row]
    vals += [t[3] for t in terms] + list(extra)
    nt = len(terms)
    teq = (ctypes.c_int32 * max(nt, 1))(*[t[0] for t in terms])
    tj = (ctypes.c_int32 * max(nt, 1))(*[t[1] for t in terms])
    tk = (ctypes.c_int32 * max(nt, 1))(*[t[2] for t in terms])
    sgn, ex, limbs, nl = _pack(vals)
    return dim, nt, teq, tj, tk, sgn, ex, limbs, nl


def compute_jet(system, state, order, prec, chunks=64, threshold=256, threads=1):
    """taylor.py:139 compute_jet -> coeffs[m][i] as Dy."""
    dim, nt, teq, tj, tk, sgn, ex, limbs, nl = _sys_pack(system, state)
    onl = _onl(prec)
    n = dim * (order + 1)
    s, e, l = _out(n, onl)
    rc = lib().ref_compute_jet(
        prec, dim, nt, teq, tj, tk, sgn, ex, limbs, nl, order, chunks, threshold, threads,
        s, e, l, onl,
    )
    if rc:
        raise ArithmeticError(f"ref_compute_jet failed ({rc})")
    flat = _unpack(s, e, l, n, onl)
    return [flat[m * (order + 1):(m + 1) * (order + 1)] for m in range(dim)]


def integrate(system, state0, tau, order, n_steps, prec, stride=100, start_step=0,
              chunks=64, threshold=256, threads=1):
    """taylor.py:202 integrate -> [(step, [Dy]*dim)] on the reference's record grid."""
    dim, nt, teq, tj, tk, sgn, ex, limbs, nl = _sys_pack(system, list(state0) + [tau])
    onl = _onl(prec)
    max_rec = (n_steps - start_step) // stride + 3
    steps = (ctypes.c_int32 * max_rec)()
    s, e, l = _out(max_rec * dim, onl)
    nrec = lib().ref_integrate(
        prec, dim, nt, teq, tj, tk, sgn, ex, limbs, nl, order, n_steps, start_step, stride,
        chunks, threshold, threads, max_rec, steps, s, e, l, onl,
    )
    if nrec < 0:
        raise ArithmeticError(f"ref_integrate failed ({nrec})")
    flat = _unpack(s, e, l, nrec * dim, onl)
    return [(steps[r], flat[r * dim:(r + 1) * dim]) for r in range(nrec)]


def convolve(arrays, i, prec, chunks=64, threshold=256, threads=1):
    """reduction.py:149 convolve (2 arrays) / convolve_pair (4 arrays)."""
    npairs = len(arrays) // 2
    length = len(arrays[0])
    vals = [v for arr in arrays for v in arr]
    sgn, ex, limbs, nl = _pack(vals)
    onl = _onl(prec) + 1
    s, e, l = _out(npairs, onl)
    rc = lib().ref_convolve(prec, npairs, length, sgn, ex, limbs, nl, i, chunks, threshold,
                            threads, s, e, l, onl)
    if rc:
        raise ArithmeticError("ref_convolve failed")
    return _unpack(s, e, l, npairs, onl)
