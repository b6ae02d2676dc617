"""Minimal ``gmpy2`` stand-in over the system MPFR library (ctypes).

TEST INFRASTRUCTURE ONLY -- used by tests/golden/make_golden.py, in the
build container, to run the UNMODIFIED reference package
(/root/reference/pkg/src/mptaylor) and freeze its outputs as fixtures.
gmpy2 is not installed in this image, but the library gmpy2 wraps is:
libmpfr.so.6 (MPFR 4.2.1). Every arithmetic call below is the same MPFR
function gmpy2 would make (round-to-nearest-even at the context
precision), so the reference runs here with its real rounding behaviour.

Only the API surface the reference touches is provided.
"""

from __future__ import annotations

import ctypes
import pickle
from fractions import Fraction

_mpfr = ctypes.CDLL("libmpfr.so.6")
_gmp = ctypes.CDLL("libgmp.so.10")


class _MpfrStruct(ctypes.Structure):
    _fields_ = [
        ("prec", ctypes.c_long),
        ("sign", ctypes.c_int),
        ("exp", ctypes.c_long),
        ("d", ctypes.c_void_p),
    ]


class _MpzStruct(ctypes.Structure):
    _fields_ = [("alloc", ctypes.c_int), ("size", ctypes.c_int), ("d", ctypes.c_void_p)]


_P = ctypes.POINTER(_MpfrStruct)
_Z = ctypes.POINTER(_MpzStruct)
_RNDN = 0


def _sig(name, res, *args, lib=_mpfr):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_init2 = _sig("mpfr_init2", None, _P, ctypes.c_long)
_clear = _sig("mpfr_clear", None, _P)
_set4 = _sig("mpfr_set4", ctypes.c_int, _P, _P, ctypes.c_int, ctypes.c_int)
_set_str = _sig("mpfr_set_str", ctypes.c_int, _P, ctypes.c_char_p, ctypes.c_int, ctypes.c_int)
_add = _sig("mpfr_add", ctypes.c_int, _P, _P, _P, ctypes.c_int)
_sub = _sig("mpfr_sub", ctypes.c_int, _P, _P, _P, ctypes.c_int)
_mul = _sig("mpfr_mul", ctypes.c_int, _P, _P, _P, ctypes.c_int)
_div = _sig("mpfr_div", ctypes.c_int, _P, _P, _P, ctypes.c_int)
_neg = _sig("mpfr_neg", ctypes.c_int, _P, _P, ctypes.c_int)
_mul_2si = _sig("mpfr_mul_2si", ctypes.c_int, _P, _P, ctypes.c_long, ctypes.c_int)
_zero_p = _sig("mpfr_zero_p", ctypes.c_int, _P)
_nan_p = _sig("mpfr_nan_p", ctypes.c_int, _P)
_inf_p = _sig("mpfr_inf_p", ctypes.c_int, _P)
_signbit = _sig("mpfr_signbit", ctypes.c_int, _P)
_get_z_2exp = _sig("mpfr_get_z_2exp", ctypes.c_long, _Z, _P)
_get_str = _sig(
    "mpfr_get_str",
    ctypes.c_void_p,
    ctypes.c_char_p,
    ctypes.POINTER(ctypes.c_long),
    ctypes.c_int,
    ctypes.c_size_t,
    _P,
    ctypes.c_int,
)
_free_str = _sig("mpfr_free_str", None, ctypes.c_void_p)
_z_init = _sig("__gmpz_init", None, _Z, lib=_gmp)
_z_clear = _sig("__gmpz_clear", None, _Z, lib=_gmp)
_z_get_str = _sig("__gmpz_get_str", ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, _Z, lib=_gmp)
_libc = ctypes.CDLL(None)
_libc.free.argtypes = [ctypes.c_void_p]

RoundToNearest = 0
_DEFAULT_PREC = 53


class context:
    def __init__(self, precision=_DEFAULT_PREC, round=RoundToNearest, **_traps):
        if round != RoundToNearest:
            raise NotImplementedError("shim supports round-to-nearest only")
        self.precision = precision

    def _coerce(self, x):
        if isinstance(x, mpfr):
            return x
        if isinstance(x, int):
            return mpfr(x, max(64, abs(x).bit_length() + 1))
        raise TypeError(f"unsupported operand {x!r}")

    def _bin(self, fn, a, b):
        a, b = self._coerce(a), self._coerce(b)
        r = mpfr._blank(self.precision)
        fn(r._p, a._p, b._p, _RNDN)
        return r

    def add(self, a, b):
        return self._bin(_add, a, b)

    def sub(self, a, b):
        return self._bin(_sub, a, b)

    def mul(self, a, b):
        return self._bin(_mul, a, b)

    def div(self, a, b):
        b = self._coerce(b)
        if _zero_p(b._p):
            raise ZeroDivisionError("division by zero")
        return self._bin(_div, a, b)

    def minus(self, a):
        r = mpfr._blank(self.precision)
        _neg(r._p, self._coerce(a)._p, _RNDN)
        return r

    def mul_2exp(self, a, e):
        r = mpfr._blank(self.precision)
        _mul_2si(r._p, self._coerce(a)._p, int(e), _RNDN)
        return r


_current = context()


def get_context():
    return _current


def set_context(ctx):
    global _current
    _current = ctx


class mpfr:
    __slots__ = ("_s", "_p", "precision")

    @classmethod
    def _blank(cls, prec):
        self = object.__new__(cls)
        self._s = _MpfrStruct()
        self._p = ctypes.pointer(self._s)
        self.precision = int(prec)
        _init2(self._p, self.precision)
        return self

    def __new__(cls, x=0, precision=0):
        prec = precision or _current.precision
        self = cls._blank(prec)
        if isinstance(x, mpfr):
            _set4(self._p, x._p, _RNDN, x._s.sign)
        elif isinstance(x, (int, str)):
            text = str(x).strip()
            if _set_str(self._p, text.encode(), 10, _RNDN) != 0:
                raise ValueError(f"invalid digits {x!r}")
        else:
            raise TypeError(f"unsupported mpfr source {x!r}")
        return self

    def __del__(self):
        try:
            _clear(self._p)
        except Exception:
            pass

    # --- exact views --------------------------------------------------
    def as_mantissa_exp(self):
        if _zero_p(self._p):
            return 0, 0
        z = _MpzStruct()
        _z_init(ctypes.byref(z))
        e = _get_z_2exp(ctypes.byref(z), self._p)
        s = _z_get_str(None, 16, ctypes.byref(z))
        text = ctypes.cast(s, ctypes.c_char_p).value.decode()
        _libc.free(s)
        _z_clear(ctypes.byref(z))
        return int(text, 16), int(e)

    def as_integer_ratio(self):
        m, e = self.as_mantissa_exp()
        f = Fraction(m) * (Fraction(2) ** e)
        return f.numerator, f.denominator

    def digits(self, base=10, n=0):
        e = ctypes.c_long(0)
        s = _get_str(None, ctypes.byref(e), base, n, self._p, _RNDN)
        text = ctypes.cast(s, ctypes.c_char_p).value.decode()
        _free_str(s)
        return text, int(e.value), self.precision

    def __float__(self):
        n, d = self.as_integer_ratio()
        return n / d

    def _frac(self):
        return Fraction(*self.as_integer_ratio())

    def __eq__(self, other):
        if isinstance(other, (mpfr, int, Fraction)):
            o = other._frac() if isinstance(other, mpfr) else Fraction(other)
            return self._frac() == o
        return NotImplemented

    def __hash__(self):
        return hash(self._frac())

    def __repr__(self):
        return f"mpfr({self.digits(10, 0)[0]!r}e{self.digits(10, 0)[1]}, {self.precision})"


def is_zero(x):
    return bool(_zero_p(x._p))


def is_signed(x):
    return bool(_signbit(x._p))


def is_finite(x):
    return not (_nan_p(x._p) or _inf_p(x._p))


def to_binary(x):
    m, e = x.as_mantissa_exp()
    return pickle.dumps((m, e, x.precision, is_signed(x)))


def from_binary(b):
    m, e, prec, neg = pickle.loads(b)
    ctx = context(precision=prec)
    v = ctx.mul_2exp(mpfr(m, prec), e) if m else mpfr(0, prec)
    if m == 0 and neg:
        v = ctx.minus(v)
    return v
