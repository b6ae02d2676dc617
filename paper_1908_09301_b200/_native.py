"""Loader of the CUDA engine (libmptaylor_b200.so) through its C ABI.

The library is built in-tree (paper_1908_09301_b200/_lib) by
``__graft_entry__.build()`` / ``python -m paper_1908_09301_b200._build``.
There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every engine call raises NativeUnavailable.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libmptaylor_b200.so")

# every symbol declared in include/mptaylor_b200.h
EXPORTS = (
    "mpt_version",
    "mpt_last_error",
    "mpt_device_count",
    "mpt_plan_create",
    "mpt_plan_destroy",
    "mpt_plan_width",
    "mpt_plan_set_constants",
    "mpt_record_count",
    "mpt_integrate",
    "mpt_state_upload",
    "mpt_state_download",
    "mpt_integrate_device",
    "mpt_compute_jet",
    "mpt_step",
    "mpt_last_kernel_ms",
    "mpt_plan_info",
    "mpt_plan_configure",
    "mpt_plan_kernel",
    "mpt_count_macs",
    "mpt_read_macs",
    "mpt_imad_probe",
    "mpt_l2_flush",
)


# error codes of include/mptaylor_b200.h
MPT_EINVAL, MPT_ENODEV, MPT_ECUDA, MPT_EUNSUP, MPT_ERANGE = -1, -2, -3, -4, -5


class NativeUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"mptaylor_b200 error {code}: {msg}")
        self.code = code


_lib = None

i32p = ctypes.POINTER(ctypes.c_int32)


def _declare(L):
    vp = ctypes.c_void_p
    L.mpt_version.restype = ctypes.c_int
    L.mpt_last_error.restype = ctypes.c_char_p
    L.mpt_device_count.restype = ctypes.c_int
    L.mpt_plan_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, i32p, i32p, i32p,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int]
    L.mpt_plan_destroy.argtypes = [vp]
    L.mpt_plan_width.argtypes = [vp]
    L.mpt_plan_set_constants.argtypes = [vp, i32p, i32p, i32p, i32p]
    L.mpt_record_count.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.mpt_integrate.argtypes = [vp, i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, i32p, i32p]
    L.mpt_state_upload.argtypes = [vp, i32p]
    L.mpt_state_download.argtypes = [vp, i32p]
    L.mpt_integrate_device.argtypes = [vp, ctypes.c_int, vp]
    L.mpt_compute_jet.argtypes = [vp, i32p, i32p, i32p]
    L.mpt_step.argtypes = [vp, i32p, i32p, i32p]
    L.mpt_last_kernel_ms.argtypes = [vp]
    L.mpt_last_kernel_ms.restype = ctypes.c_float
    L.mpt_plan_info.argtypes = [vp, i32p, i32p, i32p]
    L.mpt_plan_configure.argtypes = [vp, ctypes.c_int, ctypes.c_int]
    L.mpt_plan_kernel.argtypes = [vp, i32p, i32p]
    u64p = ctypes.POINTER(ctypes.c_ulonglong)
    L.mpt_count_macs.argtypes = [vp, ctypes.c_int]
    L.mpt_read_macs.argtypes = [vp, u64p, u64p]
    L.mpt_imad_probe.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float)]
    L.mpt_l2_flush.argtypes = [ctypes.c_int, ctypes.c_size_t]


def load(require_device: bool = True):
    """The ctypes handle; raises NativeUnavailable when the engine cannot run."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"CUDA engine not built ({LIB_PATH} missing); run __graft_entry__.build()"
            )
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    if require_device and _lib.mpt_device_count() <= 0:
        raise NativeUnavailable("no CUDA device visible: the engine has no CPU fallback")
    return _lib


def check(rc: int) -> int:
    if rc < 0:
        raise NativeError(rc, load(require_device=False).mpt_last_error().decode())
    return rc
