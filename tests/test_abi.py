"""The C ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/mptaylor_b200.h declares, and fails loudly (no CPU fallback)
when no device is present."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1908_09301_b200 import _native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "mptaylor_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mpt_[a-z0-9_]+)\s*\(", text)))


def test_library_exists_and_exports_header_symbols():
    assert os.path.exists(_native.LIB_PATH), "run __graft_entry__.build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mpt_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    assert set(_native.EXPORTS) == set(header_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_loads_without_device_and_pure_functions_work():
    L = _native.load(require_device=False)
    assert L.mpt_version() >= 1
    assert L.mpt_record_count(1000, 0, 100) == 11
    assert L.mpt_record_count(250, 0, 100) == 4
    assert L.mpt_record_count(60, 20, 20) == 3
    assert L.mpt_record_count(5, 0, 0) < 0
    # n_steps == start_step: the initial record only, also off the stride grid
    assert L.mpt_record_count(250, 250, 100) == 1
    assert L.mpt_record_count(200, 200, 100) == 1
    assert L.mpt_record_count(0, 0, 7) == 1
    assert L.mpt_record_count(251, 250, 100) == 2
    assert L.mpt_record_count(10, 20, 5) < 0


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and
                    _native.load(require_device=False).mpt_device_count() > 0,
                    reason="a GPU is present")
def test_no_device_fails_loudly():
    L = _native.load(require_device=False)
    assert L.mpt_device_count() == 0
    h = ctypes.c_void_p()
    z = np.zeros(4, np.int32)
    p = z.ctypes.data_as(_native.i32p)
    rc = L.mpt_plan_create(ctypes.byref(h), 3, 2, p, p, p, 8, 1, 10, 200, 1, 0)
    assert rc == -2  # MPT_ENODEV
    assert b"no CUDA device" in L.mpt_last_error()
    with pytest.raises(_native.NativeUnavailable):
        _native.load()
    import paper_1908_09301_b200 as M

    ctx = M.PrecisionContext(128)
    system = M.builtin_system("lorenz", ctx)
    state = tuple(M.mp_from_decimal(t, ctx) for t in ("-15.8", "-17.48", "35.64"))
    with pytest.raises(_native.NativeUnavailable):
        M.integrate(system, state, M.StepConfig("0.01", 10), 5, ctx)
