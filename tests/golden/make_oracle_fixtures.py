#!/usr/bin/env python3
"""Long-run fixtures from the C oracle (reference semantics on MPFR).

The oracle is pinned bit-for-bit to the unmodified reference by
make_golden.py; running the reference itself (Python + ctypes MPFR shim)
at these sizes would take days, so the long configurations of
BASELINE.json are frozen from the oracle instead, with the reference's
default reduction plan (64 chunks, serial threshold 256 -- the chunked
rounding applies for orders >= 255, exactly as in the reference).

    python tests/golden/make_oracle_fixtures.py [name ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref as R  # noqa: E402

INIT = ("-15.8", "-17.48", "35.64")

# name: (K digits, N, tau, n_steps, stride)
CASES = {
    "config1_k500_n200_10000": (500, 200, "0.01", 10000, 1000),
    "config2_k2200_n1000_500": (2200, 1000, "0.01", 500, 100),
    "config3_k4200_n3500_4": (4200, 3500, "0.01", 4, 1),
    "config3_k4200_n3500_100": (4200, 3500, "0.01", 100, 10),
}

# Error-budget companions: the same inputs (initial condition, tau and the
# system constants rounded to the reference precision P, exactly as the
# reference and the device see them), integrated by the same oracle at
# working precision P + EXTRA_BITS with the same order N. Both the device and
# the reference are compared against these runs (tests/test_gpu.py
# test_error_budget_*): the distance of each from the P+64 run is its own
# rounding error, since the truncation error is shared.
EXTRA_BITS = 64
HIPREC = {
    "config1_k500_n200_10000_p64": "config1_k500_n200_10000",
    "config2_k2200_n1000_500_p64": "config2_k2200_n1000_500",
    "config3_k4200_n3500_100_p64": "config3_k4200_n3500_100",
}


def bits_for_digits(d: int) -> int:
    p = int(d * 3.321928094887362)
    while (1 << p) < 10**d:
        p += 1
    while p > 1 and (1 << (p - 1)) >= 10**d:
        p -= 1
    return p


def run(name):
    base = HIPREC.get(name, name)
    K, N, tau, n_steps, stride = CASES[base]
    P = bits_for_digits(K)
    work = P + EXTRA_BITS if name in HIPREC else P
    t0 = time.time()
    rows = R.integrate(R.lorenz(P), [R.from_decimal(t, P) for t in INIT], R.from_decimal(tau, P), N, n_steps, work,
                       stride=stride, threads=os.cpu_count() or 1)
    dt = time.time() - t0
    print(f"{name}: P={P} {dt:.1f}s", flush=True)
    return {
        "name": name, "K": K, "prec_bits": P, "work_prec_bits": work, "order": N, "tau": tau, "init": list(INIT),
        "n_steps": n_steps, "stride": stride, "oracle_seconds": dt, "threads": os.cpu_count(),
        "records": [{"step": s, "state": [R.dy_hex(v) for v in st]} for s, st in rows],
    }


def main():
    names = sys.argv[1:] or list(CASES) + list(HIPREC)
    for name in names:
        out = os.path.join(HERE, f"oracle_{name}.json")
        case = run(name)
        with open(out, "w") as fh:
            json.dump(case, fh, indent=0)
        print(f"wrote {out}", flush=True)


if __name__ == "__main__":
    main()
