"""ctypes front end of oracle/fixmodel.c, the bit-exact CPU model of the
device arithmetic. TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench checks).

Inputs are the same int32 digit tables the product hands to the C ABI
(paper_1908_09301_b200.engine.SystemTables), so a GPU result and a model
result can be compared element for element.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import ref as _ref

LIB_PATH = os.path.join(_ref.HERE, "liboracle_fix.so")
_lib = None
_i32p = ctypes.POINTER(ctypes.c_int32)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            _ref.build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return np.ascontiguousarray(a, dtype=np.int32).ctypes.data_as(_i32p)


def _tables(t):
    nt = len(t.teq)
    dummy = np.zeros(1, np.int32)
    keep = [np.ascontiguousarray(x, dtype=np.int32) for x in
            (t.teq if nt else dummy, t.tj if nt else dummy, t.tk if nt else dummy,
             t.cst, t.lin, t.q if nt else np.zeros((1, t.cst.shape[1]), np.int32), t.ctab)]
    return nt, keep


def _bulk(bulk):
    if bulk is not None:
        lib().fix_set_bulk(int(bulk))


def compute_jet(tables, frac_digits: int, order: int, state: np.ndarray, variant: int = 0,
                bulk: int | None = None) -> np.ndarray:
    """-> coef[dim, order+1, W] (digits), exactly as the kernel computes them.

    variant 0: per-order C-product recurrence (team and grid kernels);
    variant 1: matrix recurrence (mx kernel) with `bulk` bulk CTAs (the partition
    of the Cauchy sums enters its rounding); variant 2: value-exact matrix
    recurrence; variant 3: value-exact per-order recurrence (warp kernel)."""
    _bulk(bulk)
    W = frac_digits + 1
    nt, k = _tables(tables)
    st = np.ascontiguousarray(state, dtype=np.int32).reshape(tables.dim, W)
    out = np.zeros((tables.dim, order + 1, W), np.int32)
    rc = lib().fix_compute_jet_v(variant, tables.dim, nt, _p(k[0]), _p(k[1]), _p(k[2]), frac_digits,
                               tables.c_shift, order, _p(k[3]), _p(k[4]), _p(k[5]), _p(k[6]),
                               _p(st), out.ctypes.data_as(_i32p))
    if rc:
        raise ArithmeticError(f"fix_compute_jet failed ({rc})")
    return out


def integrate(tables, frac_digits: int, order: int, prec_bits: int, state0: np.ndarray,
              n_steps: int, start_step: int = 0, stride: int = 1, variant: int = 0, bulk: int | None = None):
    """-> (steps, records[nrec, dim, W]) on the reference's record grid."""
    _bulk(bulk)
    W = frac_digits + 1
    nt, k = _tables(tables)
    st = np.ascontiguousarray(state0, dtype=np.int32).reshape(tables.dim, W)
    max_rec = (n_steps - start_step) // stride + 3
    steps = np.zeros(max_rec, np.int32)
    recs = np.zeros((max_rec, tables.dim, W), np.int32)
    nrec = lib().fix_integrate_v(variant, tables.dim, nt, _p(k[0]), _p(k[1]), _p(k[2]), frac_digits,
                               tables.c_shift, order, prec_bits, _p(k[3]), _p(k[4]), _p(k[5]),
                               _p(k[6]), _p(st), n_steps, start_step, stride, max_rec,
                               steps.ctypes.data_as(_i32p), recs.ctypes.data_as(_i32p))
    if nrec < 0:
        raise ArithmeticError(f"fix_integrate failed ({nrec})")
    return steps[:nrec], recs[:nrec]
