#!/usr/bin/env python3
"""Freeze golden vectors from the UNMODIFIED reference package.

Run in the build container (it needs /root/reference, which does not exist
on the GPU box):

    python tests/golden/make_golden.py

The reference (/root/reference/pkg/src/mptaylor) is imported as-is; its
arithmetic backend gmpy2 is absent from this image, so tests/golden/_shim
provides the few gmpy2 entry points it uses on top of the same MPFR library
gmpy2 wraps. Every case is also recomputed with the C oracle
(oracle/mpfr_ref.c) and the script refuses to write a fixture unless the two
agree bit for bit -- that is the pin of the oracle.

Fixture values are stored as exact dyadics "[-]<odd hex mantissa>p<exp>".
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(HERE, "_shim"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import mptaylor as M  # noqa: E402  (the reference, via the shim)
from mptaylor.systems import BilinearTerm  # noqa: E402

from oracle import ref as R  # noqa: E402

INIT = ("-15.8", "-17.48", "35.64")


def hx(v) -> str:
    """reference MPValue -> fixture text (exact)."""
    m, e = v.as_mantissa_exp()
    neg = m < 0 or (m == 0 and v._s.sign < 0)
    return R.dy_hex(R.Dy(-1 if neg else 1, abs(m), e))


def dy(v) -> R.Dy:
    return R.dy_from_hex(hx(v))


def sys_to_oracle(system):
    return {
        "dim": system.dim,
        "constant": [dy(v) for v in system.constant],
        "linear": [[dy(v) for v in row] for row in system.linear],
        "terms": [
            (m, t.j, t.k, dy(t.coeff)) for m, terms in enumerate(system.bilinear) for t in terms
        ],
    }


def sys_to_json(system):
    return {
        "dim": system.dim,
        "constant": [hx(v) for v in system.constant],
        "linear": [[hx(v) for v in row] for row in system.linear],
        "terms": [
            [m, t.j, t.k, hx(t.coeff)] for m, terms in enumerate(system.bilinear) for t in terms
        ],
    }


def same(a, b):
    return R.dy_hex(a) == R.dy_hex(b) and (a.mant != 0 or a.sign == b.sign)


def check_traj(name, traj, oracle_rows):
    ref_rows = [(p.step, [dy(v) for v in p.state]) for p in traj.points]
    assert [s for s, _ in ref_rows] == [s for s, _ in oracle_rows], name
    for (s, ra), (_, oa) in zip(ref_rows, oracle_rows):
        for a, b in zip(ra, oa):
            assert same(a, b), f"{name}: oracle differs from reference at step {s}"


def integrate_case(name, bits, order, tau, n_steps, stride, init=INIT, system_name="lorenz",
                   chunks=None, threshold=None):
    """chunks/threshold: a non-default ReducePlan (reduction.py:40), passed to
    the reference as SerialReducer(plan) and to the oracle as its chunk plan."""
    t0 = time.time()
    ctx = M.PrecisionContext(bits)
    system = M.builtin_system(system_name, ctx)
    state0 = tuple(M.mp_from_decimal(t, ctx) for t in init)
    cfg = M.StepConfig(tau_text=tau, order_n=order)
    plan_kw = {}
    reducer = None
    if chunks is not None or threshold is not None:
        plan = M.ReducePlan(num_chunks=chunks or 64, serial_threshold=threshold or 256)
        reducer = M.SerialReducer(plan)
        plan_kw = {"chunks": plan.num_chunks, "threshold": plan.serial_threshold}
    traj = M.integrate(system, state0, cfg, n_steps, ctx, reducer=reducer, record_stride=stride)
    t_ref = time.time() - t0
    t0 = time.time()
    rows = R.integrate(
        sys_to_oracle(system), [dy(v) for v in state0], dy(cfg.tau(ctx)), order, n_steps, bits,
        stride=stride, **plan_kw,
    )
    t_orc = time.time() - t0
    check_traj(name, traj, rows)
    print(f"{name}: reference {t_ref:.1f}s oracle {t_orc:.2f}s -- bit-identical")
    return {
        "kind": "integrate",
        "name": name,
        "prec_bits": bits,
        "order": order,
        "tau": tau,
        "tau_value": hx(cfg.tau(ctx)),
        "init": list(init),
        "init_values": [hx(v) for v in state0],
        "n_steps": n_steps,
        "stride": stride,
        **({"plan": plan_kw} if plan_kw else {}),
        "system": sys_to_json(system),
        "records": [{"step": p.step, "state": [hx(v) for v in p.state]} for p in traj.points],
    }


def jet_case(name, system, state, bits, order):
    ctx = M.PrecisionContext(bits)
    jet = M.compute_jet(system, state, order, ctx)
    ojet = R.compute_jet(sys_to_oracle(system), [dy(v) for v in state], order, bits)
    for m in range(system.dim):
        for i in range(order + 1):
            assert same(dy(jet.coeffs[m][i]), ojet[m][i]), (name, m, i)
    print(f"{name}: jet bit-identical")
    return {
        "kind": "jet",
        "name": name,
        "prec_bits": bits,
        "order": order,
        "system": sys_to_json(system),
        "state": [hx(v) for v in state],
        "coeffs": [[hx(v) for v in row] for row in jet.coeffs],
    }


def random_systems(n, seed=20260807):
    """Mirrors the generator of the reference's own random-system test
    (tests/test_taylor.py:103) so the fixtures cover the same class."""
    ctx = M.PrecisionContext(256)
    rnd = random.Random(seed)
    out = []
    for _ in range(n):
        dim = rnd.randrange(1, 4)
        order = rnd.randrange(1, 7)
        const = tuple(ctx.div(ctx.from_int(rnd.randrange(-8, 9)), ctx.from_int(4)) for _ in range(dim))
        linear = tuple(
            tuple(ctx.div(ctx.from_int(rnd.randrange(-8, 9)), ctx.from_int(3)) for _ in range(dim))
            for _ in range(dim)
        )
        bil = []
        for _ in range(dim):
            terms = []
            for j in range(dim):
                for k in range(j, dim):
                    if rnd.random() < 0.4:
                        q = ctx.div(ctx.from_int(rnd.randrange(-4, 5)), ctx.from_int(2))
                        terms.append(BilinearTerm(j, k, q))
            bil.append(tuple(terms))
        system = M.QuadraticODESystem(dim=dim, constant=const, linear=linear, bilinear=tuple(bil))
        state = tuple(ctx.div(ctx.from_int(rnd.randrange(-6, 7)), ctx.from_int(5)) for _ in range(dim))
        out.append((system, state, order))
    return out


def main():
    cases = []
    # hand-value jet at the canonical state (test_acceptance.py criterion 1)
    ctx = M.PrecisionContext(256)
    lor = M.builtin_system("lorenz", ctx)
    st = tuple(M.mp_from_decimal(t, ctx) for t in INIT)
    cases.append(jet_case("lorenz_jet_256_n6", lor, st, 256, 6))
    ctx2 = M.PrecisionContext(1661)
    lor2 = M.builtin_system("lorenz", ctx2)
    st2 = tuple(M.mp_from_decimal(t, ctx2) for t in INIT)
    cases.append(jet_case("lorenz_jet_1661_n200", lor2, st2, 1661, 200))
    for idx, (system, state, order) in enumerate(random_systems(12)):
        cases.append(jet_case(f"random_jet_{idx}", system, state, 256, order))
    # exponential system (criterion 2): dx/dt = x, tau = 1, N = 30
    ctxe = M.PrecisionContext(256)
    exp_sys = M.QuadraticODESystem(dim=1, constant=(ctxe.zero,), linear=((ctxe.one,),), bilinear=((),))
    ex = M.step(exp_sys, (ctxe.one,), M.StepConfig(tau_text="1", order_n=30), ctxe)
    cases.append({"kind": "step", "name": "exp_tau1_n30_256", "prec_bits": 256, "order": 30,
                  "tau": "1", "system": sys_to_json(exp_sys), "state": [hx(ctxe.one)],
                  "result": [hx(v) for v in ex]})
    # BASELINE.json configs[0]: K=50 digits, N=40, tau=0.01, 1000 steps, every 100
    k50 = M.bits_for_digits(50)
    cases.append(integrate_case("config0_k50_n40", k50, 40, "0.01", 1000, 100))
    # the reference's own regression pair (tests/test_cns.py:97): 128/N=20 vs 256/N=30, t in [0,25]
    cases.append(integrate_case("cns_pair_128_n20", 128, 20, "0.01", 2500, 100))
    cases.append(integrate_case("cns_pair_256_n30", 256, 30, "0.01", 2500, 100))
    # configs[1] shape, shortened: K=500 digits, N=200, 3 steps recorded every step
    k500 = M.bits_for_digits(500)
    cases.append(integrate_case("config1_k500_n200_3steps", k500, 200, "0.01", 3, 1))
    # zero state is a fixed point (signed-zero handling)
    cases.append(integrate_case("zero_state_256_n8", 256, 8, "0.01", 5, 1, init=("0", "0", "0")))
    # negative step (forward-backward, test_taylor.py:270)
    cases.append(integrate_case("backward_256_n30", 256, 30, "-0.01", 50, 10))
    # the chunked branch of the reference reduction (reduction.py:136-146):
    # orders with i + 1 >= 256 round per chunk of the default 64-chunk plan
    cases.append(integrate_case("chunked_256_n300_3steps", 256, 300, "0.01", 3, 1))
    # the plan the timed reference arm runs (serial threshold 32, 64 chunks)
    cases.append(integrate_case("plan_t32_k500_n200_2steps", k500, 200, "0.01", 2, 1, threshold=32))
    out = os.path.join(HERE, "reference_golden.json")
    with open(out, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "mpfr": R.mpfr_version(),
                   "cases": cases}, fh, indent=0)
    print(f"wrote {out} ({os.path.getsize(out)} bytes, {len(cases)} cases)")


if __name__ == "__main__":
    main()
