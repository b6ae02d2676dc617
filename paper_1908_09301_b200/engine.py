"""Device plans: a quadratic system, an order, a precision and a step scale
bound to device buffers through the C ABI (include/mptaylor_b200.h).

A plan replaces, for one (system, precision, order, tau) tuple, everything
the reference builds per call of taylor.py:202 integrate / :139 compute_jet:
the product-pair list (systems.py:65), the reducer session
(reduction.py:187/:279) and the per-order 1/(i+1) factors (taylor.py:125),
which here become the tau/(i+1) table of the tau-scaled recurrence.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native
from .fixed import FixedFormat


@dataclass(frozen=True)
class SystemTables:
    """Digit tables of one system in one format (host side, int32)."""

    dim: int
    teq: np.ndarray
    tj: np.ndarray
    tk: np.ndarray
    cst: np.ndarray  # dim x W
    lin: np.ndarray  # dim*dim x W
    q: np.ndarray  # nterms x W
    ctab: np.ndarray  # order x W
    c_shift: int

    @classmethod
    def build(cls, system, fmt: FixedFormat, order: int, scale: Fraction) -> "SystemTables":
        terms = system.terms_in_order()
        W = fmt.width
        q = fmt.to_digits([t[3] for t in terms]) if terms else np.zeros((0, W), np.int32)
        return cls(
            dim=system.dim,
            teq=np.array([t[0] for t in terms], dtype=np.int32),
            tj=np.array([t[1] for t in terms], dtype=np.int32),
            tk=np.array([t[2] for t in terms], dtype=np.int32),
            cst=fmt.to_digits(system.constant),
            lin=fmt.to_digits([v for row in system.linear for v in row]),
            q=q,
            ctab=fmt.ctab(scale, order),
            c_shift=fmt.c_shift(scale),
        )


KERNEL_NAMES = {1: "team", 4: "grid", 6: "mx", 7: "warp", 8: "block", 9: "cblock"}  # include/mptaylor_b200.h mpt_plan_configure


def _p(a: np.ndarray):
    return a.ctypes.data_as(_native.i32p)


class DevicePlan:
    """n_traj trajectories of one system on one GPU."""

    def __init__(self, tables: SystemTables, fmt: FixedFormat, order: int, n_traj: int = 1, device: int = 0):
        self.lib = _native.load()
        self.fmt = fmt
        self.order = order
        self.dim = tables.dim
        self.n_traj = n_traj
        self.W = fmt.width
        self.tables = tables
        h = ctypes.c_void_p()
        nt = len(tables.teq)
        dummy = np.zeros(1, np.int32)
        _native.check(
            self.lib.mpt_plan_create(
                ctypes.byref(h), tables.dim, nt,
                _p(tables.teq if nt else dummy), _p(tables.tj if nt else dummy), _p(tables.tk if nt else dummy),
                fmt.frac_digits, tables.c_shift, order, fmt.prec_bits, n_traj, device,
            )
        )
        self.h = h
        self._keep = [np.ascontiguousarray(a, dtype=np.int32) for a in
                      (tables.cst, tables.lin, tables.q if nt else np.zeros((1, self.W), np.int32), tables.ctab)]
        _native.check(self.lib.mpt_plan_set_constants(h, *[_p(a) for a in self._keep]))

    # ------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.mpt_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def info(self) -> dict:
        s, k, t = (ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32())
        _native.check(self.lib.mpt_plan_info(self.h, ctypes.byref(s), ctypes.byref(k), ctypes.byref(t)))
        kern, cl = ctypes.c_int32(), ctypes.c_int32()
        _native.check(self.lib.mpt_plan_kernel(self.h, ctypes.byref(kern), ctypes.byref(cl)))
        return {"smem_bytes": s.value, "k_chunk": k.value, "threads": t.value,
                "kernel": KERNEL_NAMES.get(kern.value, "?"), "cluster": cl.value}

    @property
    def variant(self) -> int:
        """Arithmetic variant of the selected kernel (oracle/fixmodel.c): 1 for the
        matrix-recurrence kernel, 3 for the warp kernel (value-exact roundings), 0
        for the per-order C-product kernels (team, grid)."""
        return self.model_kwargs()["variant"]

    def model_kwargs(self) -> dict:
        """Arguments that make oracle/fixmodel.c reproduce this plan's kernel bit for
        bit (test infrastructure): the arithmetic variant and, for the matrix
        recurrence, the number of bulk CTAs (their partition of the Cauchy sums
        enters the rounding)."""
        kern, cl = ctypes.c_int32(), ctypes.c_int32()
        _native.check(self.lib.mpt_plan_kernel(self.h, ctypes.byref(kern), ctypes.byref(cl)))
        if kern.value == 6:
            return {"variant": 1, "bulk": cl.value - 1}
        if kern.value in (7, 8, 9):
            return {"variant": 3}
        return {"variant": 0}

    def configure(self, kernel: str = "auto", cluster: int = 8):
        code = {"auto": 0, **{v: k for k, v in KERNEL_NAMES.items()}}[kernel]
        _native.check(self.lib.mpt_plan_configure(self.h, code, cluster))

    def _state(self, state: np.ndarray) -> np.ndarray:
        st = np.ascontiguousarray(state, dtype=np.int32).reshape(self.n_traj, self.dim, self.W)
        return st

    # ------------------------------------------------------------------
    def integrate(self, state0, n_steps: int, start_step: int = 0, stride: int = 1):
        """-> (steps[nrec], records[nrec, n_traj, dim, W], status[n_traj])."""
        st = self._state(state0)
        nrec = self.lib.mpt_record_count(n_steps, start_step, stride)
        _native.check(nrec)
        steps = np.zeros(nrec, np.int32)
        recs = np.zeros((nrec, self.n_traj, self.dim, self.W), np.int32)
        status = np.zeros(self.n_traj, np.int32)
        got = self.lib.mpt_integrate(self.h, _p(st), n_steps, start_step, stride, _p(steps), _p(recs), _p(status))
        _native.check(got)
        return steps, recs, status

    def compute_jet(self, state):
        st = self._state(state)
        coef = np.zeros((self.n_traj, self.dim, self.order + 1, self.W), np.int32)
        status = np.zeros(self.n_traj, np.int32)
        _native.check(self.lib.mpt_compute_jet(self.h, _p(st), _p(coef), _p(status)))
        return coef

    def step(self, state):
        st = self._state(state)
        out = np.zeros_like(st)
        status = np.zeros(self.n_traj, np.int32)
        _native.check(self.lib.mpt_step(self.h, _p(st), _p(out), _p(status)))
        return out, status

    # device-resident throughput path ------------------------------------
    def upload(self, state):
        st = self._state(state)
        _native.check(self.lib.mpt_state_upload(self.h, _p(st)))

    def download(self):
        out = np.zeros((self.n_traj, self.dim, self.W), np.int32)
        _native.check(self.lib.mpt_state_download(self.h, _p(out)))
        return out

    def run_device(self, n_steps: int, stream: int = 0):
        _native.check(self.lib.mpt_integrate_device(self.h, n_steps, ctypes.c_void_p(stream)))

    def last_kernel_ms(self) -> float:
        return float(self.lib.mpt_last_kernel_ms(self.h))

    def count_macs(self, enable: bool = True):
        _native.check(self.lib.mpt_count_macs(self.h, 1 if enable else 0))

    def read_macs(self):
        u, x = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        _native.check(self.lib.mpt_read_macs(self.h, ctypes.byref(u), ctypes.byref(x)))
        return u.value, x.value
