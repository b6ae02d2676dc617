"""GPU parity tests (B200): the CUDA path through the C ABI against
  (1) the bit-exact model of the device arithmetic (oracle/fixmodel.c), and
  (2) the reference's frozen outputs (tests/golden, pinned to the unmodified
      reference) within relative 10^-(K-d(t)), d(t) from tests/helpers.py guard_digits
      (derived there; both arms are also measured against a P+64-bit oracle run).
Edge cases follow the reference's tests: zero state, zero steps, backward
step, single-dimension system, random quadratic systems, resume, observer,
determinism."""

import math
from fractions import Fraction

import numpy as np
import pytest

import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

from .conftest import CANON_INIT
from .helpers import EXACT, agreement_digits, frac, guard_digits, system_from_json

pytestmark = pytest.mark.gpu


def lorenz_tables(P, N, tau="0.01", guard=32, scale=None):
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    fmt = FixedFormat(P, guard)
    s = scale if scale is not None else M.mp_from_decimal(tau, ctx).as_fraction()
    return ctx, system, fmt, SystemTables.build(system, fmt, N, s)


# ---------------------------------------------------------------- bit-exact
@pytest.mark.parametrize("P,N,steps,stride", [(128, 20, 30, 10), (167, 40, 40, 10), (256, 30, 25, 5),
                                               (1661, 200, 3, 1), (2658, 240, 2, 1)])
def test_integrate_bit_exact_vs_model(gpu, P, N, steps, stride):
    ctx, system, fmt, tables = lorenz_tables(P, N)
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in CANON_INIT])
    with DevicePlan(tables, fmt, N, 1) as plan:
        s_gpu, r_gpu, status = plan.integrate(st, steps, 0, stride)
        kw = plan.model_kwargs()
    s_cpu, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, st, steps, 0, stride, **kw)
    assert status.tolist() == [0]
    assert list(s_gpu) == list(s_cpu)
    assert np.array_equal(r_gpu[:, 0], r_cpu)


@pytest.mark.parametrize("kernel,cluster", [("team", 1), ("warp", 1), ("grid", 1), ("mx", 2), ("mx", 3), ("mx", 5), ("mx", 8),
                                            ("mx", 16)])
@pytest.mark.parametrize("P,N,steps", [(167, 40, 12), (1661, 200, 2)])
def test_every_kernel_bit_exact_vs_model(gpu, kernel, cluster, P, N, steps):
    ctx, system, fmt, tables = lorenz_tables(P, N)
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in CANON_INIT])
    with DevicePlan(tables, fmt, N, 1) as plan:
        try:
            plan.configure(kernel, cluster)
        except Exception as exc:  # rows do not fit this cluster size's shared memory
            assert "shared memory" in str(exc) or "does not support" in str(exc)
            pytest.skip(str(exc))
        info = plan.info()
        assert info["kernel"] == kernel
        s_gpu, r_gpu, status = plan.integrate(st, steps, 0, 1)
        kw = plan.model_kwargs()
    s_cpu, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, st, steps, 0, 1, **kw)
    assert np.array_equal(r_gpu[:, 0], r_cpu), info


@pytest.mark.parametrize("K,N,steps", [(2200, 40, 2), (4200, 12, 1)])
def test_grid_kernel_large_precision_bit_exact(gpu, K, N, steps):
    P = M.bits_for_digits(K)
    ctx, system, fmt, tables = lorenz_tables(P, N)
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in CANON_INIT])
    with DevicePlan(tables, fmt, N, 1) as plan:
        plan.configure("grid", 1)
        assert plan.info()["kernel"] == "grid"
        _, r_gpu, status = plan.integrate(st, steps, 0, 1)
        jet = plan.compute_jet(st)[0]
    _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, st, steps, 0, 1)
    assert np.array_equal(r_gpu[:, 0], r_cpu)
    assert np.array_equal(jet, FX.compute_jet(tables, fmt.frac_digits, N, st))


def test_jet_bit_exact_vs_model_large_order(gpu):
    P, N = 1661, 200
    ctx, system, fmt, tables = lorenz_tables(P, N)
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in CANON_INIT])
    with DevicePlan(tables, fmt, N, 1) as plan:
        g = plan.compute_jet(st)[0]
        kw = plan.model_kwargs()
    c = FX.compute_jet(tables, fmt.frac_digits, N, st, **kw)
    assert np.array_equal(g, c)


def test_ensemble_of_trajectories_bit_exact(gpu):
    P, N, n_traj = 256, 30, 5
    ctx, system, fmt, tables = lorenz_tables(P, N)
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in CANON_INIT]
    states = np.stack([fmt.to_digits([b + Fraction(j, 10**20) for b in base]) for j in range(n_traj)])
    with DevicePlan(tables, fmt, N, n_traj) as plan:
        _, r_gpu, status = plan.integrate(states, 12, 0, 4)
        kw = plan.model_kwargs()
    assert not status.any()
    for j in range(n_traj):
        _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, states[j], 12, 0, 4, **kw)
        assert np.array_equal(r_gpu[:, j], r_cpu), j


@pytest.mark.parametrize("mb", ["1", "2", "4", "8"])
@pytest.mark.parametrize("K,N,steps", [(100, 60, 6), (400, 240, 2)])
def test_team_kernel_two_ctas_per_sm_bit_exact(gpu, monkeypatch, mb, K, N, steps):
    """Ensemble team kernel at one and two resident CTAs per SM (the k-chunk
    shrinks to fit two CTAs' shared memory): every member bit-exact vs the model."""
    monkeypatch.setenv("MPT_TEAM_MB", mb)
    P = M.bits_for_digits(K)
    n_traj = 7
    ctx, system, fmt, tables = lorenz_tables(P, N)
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in CANON_INIT]
    states = np.stack([fmt.to_digits([b + Fraction(3 * j - 9, 10**20) for b in base]) for j in range(n_traj)])
    with DevicePlan(tables, fmt, N, n_traj) as plan:
        plan.configure("team", 1)
        assert plan.info()["kernel"] == "team"
        _, r_gpu, status = plan.integrate(states, steps, 0, 1)
        kw = plan.model_kwargs()
    assert not status.any()
    for j in (0, 3, n_traj - 1):
        _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, states[j], steps, 0, 1, **kw)
        assert np.array_equal(r_gpu[:, j], r_cpu), j


@pytest.mark.parametrize("K,N,steps,n_traj", [(20, 14, 40, 2), (50, 40, 30, 1), (100, 60, 8, 9), (150, 90, 4, 5),
                                              (200, 120, 3, 37), (250, 150, 2, 3), (260, 20, 3, 2)])
def test_warp_kernel_bit_exact(gpu, K, N, steps, n_traj):
    """One warp per trajectory (W <= 34 digits; one or two columns per lane, every
    product-window width): records and the jet bit-exact vs the value-exact model."""
    P = M.bits_for_digits(K)
    ctx, system, fmt, tables = lorenz_tables(P, N)
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in CANON_INIT]
    states = np.stack([fmt.to_digits([b + Fraction(5 * j - 7, 10**18) for b in base]) for j in range(n_traj)])
    with DevicePlan(tables, fmt, N, n_traj) as plan:
        plan.configure("warp", 1)
        assert plan.info()["kernel"] == "warp"
        _, r_gpu, status = plan.integrate(states, steps, 0, 1)
        jets = plan.compute_jet(states)
        kw = plan.model_kwargs()
    assert kw == {"variant": 3} and not status.any()
    for j in sorted({0, n_traj // 2, n_traj - 1}):
        _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, states[j], steps, 0, 1, **kw)
        assert np.array_equal(r_gpu[:, j], r_cpu), j
        assert np.array_equal(jets[j], FX.compute_jet(tables, fmt.frac_digits, N, states[j], **kw)), j


@pytest.mark.parametrize("K,N,steps,n_traj", [(100, 60, 3, 3), (300, 40, 3, 2), (400, 240, 1, 3), (450, 270, 1, 2),
                                              (470, 30, 2, 1)])
def test_block_kernel_bit_exact(gpu, K, N, steps, n_traj):
    """One CTA per trajectory, rows in shared memory (W <= 58 digits, every product
    window width up to 60): records and the jet bit-exact vs the value-exact model."""
    P = M.bits_for_digits(K)
    ctx, system, fmt, tables = lorenz_tables(P, N)
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in CANON_INIT]
    states = np.stack([fmt.to_digits([b + Fraction(3 * j - 2, 10**18) for b in base]) for j in range(n_traj)])
    with DevicePlan(tables, fmt, N, n_traj) as plan:
        plan.configure("block", 1)
        assert plan.info()["kernel"] == "block"
        _, r_gpu, status = plan.integrate(states, steps, 0, 1)
        jets = plan.compute_jet(states)
        kw = plan.model_kwargs()
    assert kw == {"variant": 3} and not status.any()
    for j in sorted({0, n_traj - 1}):
        _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, states[j], steps, 0, 1, **kw)
        assert np.array_equal(r_gpu[:, j], r_cpu), j
        assert np.array_equal(jets[j], FX.compute_jet(tables, fmt.frac_digits, N, states[j], **kw)), j


@pytest.mark.parametrize("K,N,steps,n_traj,G", [(50, 40, 6, 1, 2), (100, 60, 4, 2, 4), (300, 100, 3, 1, 8), (500, 200, 2, 1, 16),
                                                (500, 200, 1, 1, 8), (500, 200, 1, 1, 3), (700, 120, 2, 1, 16),
                                                (500, 37, 3, 3, 5)])
def test_cblock_kernel_bit_exact(gpu, K, N, steps, n_traj, G):
    """One cluster of G CTAs per trajectory, rows in every CTA's shared memory, the
    Cauchy sums split over CTAs, warps and lanes and all-gathered through DSMEM
    (W <= 93 digits): records and the jet bit-exact vs the value-exact model,
    whatever the cluster size (the partition cannot change a bit)."""
    P = M.bits_for_digits(K)
    ctx, system, fmt, tables = lorenz_tables(P, N)
    base = [M.mp_from_decimal(t, ctx).as_fraction() for t in CANON_INIT]
    states = np.stack([fmt.to_digits([b + Fraction(5 * j - 7, 10**18) for b in base]) for j in range(n_traj)])
    with DevicePlan(tables, fmt, N, n_traj) as plan:
        plan.configure("cblock", G)
        assert plan.info()["kernel"] == "cblock"
        _, r_gpu, status = plan.integrate(states, steps, 0, 1)
        jets = plan.compute_jet(states)
        kw = plan.model_kwargs()
    assert kw == {"variant": 3} and not status.any()
    for j in sorted({0, n_traj - 1}):
        _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, states[j], steps, 0, 1, **kw)
        assert np.array_equal(r_gpu[:, j], r_cpu), j
        assert np.array_equal(jets[j], FX.compute_jet(tables, fmt.frac_digits, N, states[j], **kw)), j


def _mixed_system(ctx):
    """dx/dt = 1/3 + 10.5 (y - x) + 0.7 z,  dy/dt = 28 x - 1.25 y - x z,  dz/dt = -1/7 + 0.3 x - 8/3 z + x y:
    two integer-coefficient pairs, a non-integer linear coefficient in every equation (two in the
    first and the last), non-zero constants."""
    def v(t):
        return M.mp_from_decimal(t, ctx) if "/" not in t else ctx.div(M.mp_from_decimal(t.split("/")[0], ctx),
                                                                       M.mp_from_decimal(t.split("/")[1], ctx))
    z = M.mp_from_decimal("0", ctx)
    return M.QuadraticODESystem(
        dim=3,
        constant=(v("1/3"), z, v("-1/7")),
        linear=((v("-10.5"), v("10.5"), v("0.7")), (v("28"), v("-1.25"), z), (v("0.3"), z, v("-8/3"))),
        bilinear=((), (M.BilinearTerm(0, 2, M.mp_from_decimal("-1", ctx)),), (M.BilinearTerm(0, 1, M.mp_from_decimal("1", ctx)),)),
    )


@pytest.mark.parametrize("kernel,cluster,K,N,steps", [("warp", 1, 100, 40, 5), ("warp", 1, 250, 60, 2), ("block", 1, 300, 60, 3),
                                                       ("block", 1, 450, 50, 2), ("cblock", 4, 300, 60, 3),
                                                       ("cblock", 16, 500, 70, 2), ("cblock", 1, 120, 30, 3)])
def test_value_exact_kernels_general_linear_terms(gpu, kernel, cluster, K, N, steps):
    """The chunked / side-warp products of the non-integer linear coefficients (several per
    system, in every equation) in the warp, block and cblock kernels: records and jet bit-exact
    vs the value-exact model."""
    P = M.bits_for_digits(K)
    ctx = M.PrecisionContext(P)
    system = _mixed_system(ctx)
    fmt = FixedFormat(P)
    tables = SystemTables.build(system, fmt, N, Fraction(1, 128))
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in ("1.5", "-2.25", "3.125")])
    with DevicePlan(tables, fmt, N, 1) as plan:
        plan.configure(kernel, cluster)
        assert plan.info()["kernel"] == kernel
        _, r_gpu, status = plan.integrate(st, steps, 0, 1)
        jet = plan.compute_jet(st)[0]
        kw = plan.model_kwargs()
    assert kw == {"variant": 3} and not status.any()
    _, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, st, steps, 0, 1, **kw)
    assert np.array_equal(r_gpu[:, 0], r_cpu)
    assert np.array_equal(jet, FX.compute_jet(tables, fmt.frac_digits, N, st, **kw))


def test_random_quadratic_systems_jets_bit_exact(golden, gpu):
    for name, c in golden.items():
        if not name.startswith("random_jet"):
            continue
        P, N = c["prec_bits"], c["order"]
        ctx = M.PrecisionContext(P)
        system = system_from_json(c["system"], ctx)
        fmt = FixedFormat(P)
        tables = SystemTables.build(system, fmt, N, Fraction(1, 128))
        st = fmt.to_digits([frac(h) for h in c["state"]])
        with DevicePlan(tables, fmt, N, 1) as plan:
            g = plan.compute_jet(st)[0]
            kw = plan.model_kwargs()
        assert np.array_equal(g, FX.compute_jet(tables, fmt.frac_digits, N, st, **kw)), name


# ---------------------------------------------------- parity vs reference
@pytest.mark.parametrize("name", ["config0_k50_n40", "cns_pair_128_n20", "cns_pair_256_n30",
                                  "config1_k500_n200_3steps", "backward_256_n30", "zero_state_256_n8"])
def test_dropin_integrate_matches_reference(golden, gpu, name):
    c = golden[name]
    P = c["prec_bits"]
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    state0 = tuple(M.mp_from_decimal(t, ctx) for t in c["init"])
    traj = M.integrate(system, state0, M.StepConfig(c["tau"], c["order"]), c["n_steps"], ctx,
                       record_stride=c["stride"])
    assert traj.steps() == [r["step"] for r in c["records"]]
    K = M.decimal_digits(P)
    tau = abs(float(Fraction(c["tau"])))
    for pt, rec in zip(traj.points, c["records"]):
        assert all(v.precision == P for v in pt.state)
        got = [v.as_fraction() for v in pt.state]
        ref = [frac(h) for h in rec["state"]]
        d = agreement_digits(got, ref)
        assert d == EXACT or d >= K - guard_digits(pt.step * tau, c["order"], tau), (name, pt.step, d)


LONG_RUNS = ("config1_k500_n200_10000", "config2_k2200_n1000_500", "config3_k4200_n3500_4",
             "config3_k4200_n3500_100")
ERROR_BUDGET_RUNS = ("config1_k500_n200_10000", "config2_k2200_n1000_500", "config3_k4200_n3500_100")


@pytest.mark.parametrize("name", LONG_RUNS)
def test_long_run_agreement_vs_oracle(gpu, name):
    """BASELINE.json configs 1-3 at full size, through the drop-in entry point,
    against the oracle's frozen trajectories (tests/golden/oracle_*.json: the
    reference algorithm on MPFR, bit-pinned to the reference by
    make_golden.py).  Every recorded output time must agree to 10^-(K-d(t));
    the agreement per record is written to gpurun_out/parity_<name>.json."""
    import json
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_{name}.json")
    with open(path) as fh:
        c = json.load(fh)
    P = c["prec_bits"]
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    state0 = tuple(M.mp_from_decimal(t, ctx) for t in c["init"])
    traj = M.integrate(system, state0, M.StepConfig(c["tau"], c["order"]), c["n_steps"], ctx,
                       record_stride=c["stride"])
    assert traj.steps() == [r["step"] for r in c["records"]]
    K = c["K"]
    tau = abs(float(Fraction(c["tau"])))
    report = []
    for pt, rec in zip(traj.points, c["records"]):
        got = [v.as_fraction() for v in pt.state]
        ref = [frac(h) for h in rec["state"]]
        d = agreement_digits(got, ref)
        need = K - guard_digits(pt.step * tau, c["order"], tau)
        report.append({"step": pt.step, "t": pt.step * tau, "agree_digits": None if d == EXACT else d,
                       "required": need})
        assert d == EXACT or d >= need, (name, pt.step, d, need)
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"parity_{name}.json"), "w") as fh:
        json.dump({"name": name, "K": K, "prec_bits": P, "order": c["order"], "records": report}, fh, indent=1)


@pytest.mark.parametrize("name", ERROR_BUDGET_RUNS)
def test_error_budget_vs_p64_oracle(gpu, name):
    """Both arms against the oracle re-run at P + 64 bits (same inputs and order:
    the truncation error is shared, so each arm's distance from that run is its
    own rounding error). The device rounds its state to the reference precision
    P after every step, as the reference does, and that rounding dominates both:
    the device must be as close to the P + 64 run as the reference is, to within
    one digit, at every record; device-vs-reference agreement then follows from
    the triangle inequality and keeps >= 2 digits of margin over the declared d(t). The table goes to gpurun_out/error_budget_<name>.json."""
    import json
    import os

    gdir = os.path.join(os.path.dirname(__file__), "golden")
    with open(os.path.join(gdir, f"oracle_{name}.json")) as fh:
        c = json.load(fh)
    with open(os.path.join(gdir, f"oracle_{name}_p64.json")) as fh:
        truth = json.load(fh)
    P = c["prec_bits"]
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    state0 = tuple(M.mp_from_decimal(t, ctx) for t in c["init"])
    traj = M.integrate(system, state0, M.StepConfig(c["tau"], c["order"]), c["n_steps"], ctx,
                       record_stride=c["stride"])
    K, tau = c["K"], abs(float(Fraction(c["tau"])))
    rows = []
    for pt, rec, tr in zip(traj.points[1:], c["records"][1:], truth["records"][1:]):
        assert pt.step == rec["step"] == tr["step"]
        got = [v.as_fraction() for v in pt.state]
        ref, tru = [frac(h) for h in rec["state"]], [frac(h) for h in tr["state"]]
        e_dev, e_ref, d = agreement_digits(got, tru), agreement_digits(ref, tru), agreement_digits(got, ref)
        need = K - guard_digits(pt.step * tau, c["order"], tau)
        rows.append({"step": pt.step, "t": pt.step * tau, "device_vs_p64": e_dev, "reference_vs_p64": e_ref,
                     "device_vs_reference": d, "required": need, "margin": d - need})
        assert e_dev >= e_ref - 1, rows[-1]
        assert d >= min(e_dev, e_ref) - 1 and d >= need + 2, rows[-1]
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"error_budget_{name}.json"), "w") as fh:
        json.dump({"name": name, "K": K, "prec_bits": P, "order": c["order"], "records": rows}, fh, indent=1)


def test_reference_regression_pair_on_gpu(gpu):
    """The reference's frozen agreement series (tests/test_cns.py:119), from GPU runs."""
    runs = {}
    for P, N in ((128, 20), (256, 30)):
        ctx = M.PrecisionContext(P)
        system = M.builtin_system("lorenz", ctx)
        state0 = tuple(M.mp_from_decimal(t, ctx) for t in CANON_INIT)
        runs[P] = M.integrate(system, state0, M.StepConfig("0.01", N), 2500, ctx, record_stride=100)
    series = {a.step: agreement_digits([v.as_fraction() for v in a.state], [v.as_fraction() for v in b.state])
              for a, b in zip(runs[128].points, runs[256].points)}
    assert series[0] == 38
    assert 22 <= series[100] <= 24  # reference: 23
    assert 12 <= series[2500] <= 14  # reference: 13
    assert min(series.values()) >= 6  # t_c = 25 at d = 6, as in the reference


# -------------------------------------------------------- drop-in behaviour
def _lorenz(P=256):
    ctx = M.PrecisionContext(P)
    return ctx, M.builtin_system("lorenz", ctx), tuple(M.mp_from_decimal(t, ctx) for t in CANON_INIT)


def test_recording_policy_and_zero_steps(gpu):
    ctx, system, state = _lorenz()
    traj = M.integrate(system, state, M.StepConfig("0.01", 4), 250, ctx, record_stride=100)
    assert traj.steps() == [0, 100, 200, 250]
    assert str(traj.time_of(250)) == "2.50"
    zero = M.integrate(system, state, M.StepConfig("0.01", 4), 0, ctx)
    assert zero.steps() == [0] and all(M.mp_bits_equal(a, b) for a, b in zip(zero.points[0].state, state))


def test_resume_is_bit_exact_and_runs_are_deterministic(gpu):
    ctx, system, state = _lorenz()
    cfg = M.StepConfig("0.01", 10)
    straight = M.integrate(system, state, cfg, 60, ctx, record_stride=20)
    again = M.integrate(system, state, cfg, 60, ctx, record_stride=20)
    head = M.integrate(system, state, cfg, 20, ctx, record_stride=20)
    resumed = M.integrate(system, head.final_state(), cfg, 60, ctx, record_stride=20, start_step=20)
    assert resumed.steps() == [20, 40, 60]
    by_step = {p.step: p.state for p in straight.points}
    for p in resumed.points:
        assert all(M.mp_bits_equal(a, b) for a, b in zip(p.state, by_step[p.step]))
    for a, b in zip(straight.points, again.points):
        assert all(M.mp_bits_equal(x, y) for x, y in zip(a.state, b.state))


def test_observer_sees_every_step(gpu):
    ctx, system, state = _lorenz()
    calls = []
    M.integrate(system, state, M.StepConfig("0.01", 4), 7, ctx,
                observer=lambda n, t, s: calls.append((n, str(t), type(s))))
    assert [c[0] for c in calls] == [1, 2, 3, 4, 5, 6, 7]
    assert calls[0][1] == "0.01" and all(c[2] is tuple for c in calls)


def test_compute_jet_hand_values_criterion_1(gpu):
    ctx, system, state = _lorenz()
    jet = M.compute_jet(system, state, 2, ctx)
    ulp = Fraction(1, 2**250)
    for (m, i), text in {(0, 1): "-16.8", (1, 1): "138.192", (2, 1): "181.144", (0, 2): "774.96"}.items():
        ref = M.mp_from_decimal(text, ctx).as_fraction()
        assert abs(jet.coeffs[m][i].as_fraction() - ref) <= ulp * abs(ref)
    assert all(M.mp_bits_equal(jet.coeffs[m][0], state[m]) for m in range(3))


def test_exponential_step_criterion_2(gpu):
    ctx = M.PrecisionContext(256)
    system = M.QuadraticODESystem(dim=1, constant=(ctx.zero,), linear=((ctx.one,),), bilinear=((),))
    (result,) = M.step(system, (ctx.one,), M.StepConfig("1", 30), ctx)
    e = sum((Fraction(1, math.factorial(n)) for n in range(80)), Fraction(0))
    assert abs(result.as_fraction() - e) < Fraction(1, 10**32)


def test_convergence_order_criterion_3(gpu):
    ctx = M.PrecisionContext(256)
    system = M.QuadraticODESystem(dim=1, constant=(ctx.zero,), linear=((ctx.one,),), bilinear=((),))
    for n in (4, 8):
        errs = []
        for tau in ("0.25", "0.125", "0.0625"):
            (r,) = M.step(system, (ctx.one,), M.StepConfig(tau, n), ctx)
            x = Fraction(tau)
            exact = sum((x**k / math.factorial(k) for k in range(90)), Fraction(0))
            errs.append(abs(r.as_fraction() - exact))
        for a, b in zip(errs, errs[1:]):
            assert 2 ** (n + 1) / 4 <= a / b <= 2 ** (n + 1) * 4


def test_short_horizon_vs_double_precision_rk_criterion_4(gpu):
    scipy_integrate = pytest.importorskip("scipy.integrate")
    ctx, system, state = _lorenz()
    traj = M.integrate(system, state, M.StepConfig("0.01", 30), 200, ctx)
    final = [float(v) for v in traj.final_state()]

    def rhs(_t, s):
        x, y, z = s
        return [-10.0 * x + 10.0 * y, 28.0 * x - y - x * z, x * y - 8.0 / 3.0 * z]

    sol = scipy_integrate.solve_ivp(rhs, (0.0, 2.0), [float(v) for v in state], method="DOP853",
                                    rtol=1e-10, atol=1e-12, t_eval=[2.0])
    for got, ref in zip(final, sol.y[:, -1]):
        assert abs(got - ref) / abs(ref) < 1e-6


def test_overflow_is_reported_not_silent(gpu):
    ctx = M.PrecisionContext(128)
    system = M.QuadraticODESystem(dim=1, constant=(ctx.zero,), linear=((ctx.from_int(1000),),), bilinear=((),))
    with pytest.raises(Exception) as info:
        M.integrate(system, (ctx.from_int(10**5),), M.StepConfig("1", 20), 3, ctx)
    assert "range" in str(info.value).lower()


def test_reference_side_binding_stub(gpu):
    """examples/reference_binding.py (the ctypes stub INTEGRATION.md shows for the
    reference package) drives the C ABI on its own and returns the records of
    the drop-in integrate() bit for bit."""
    import importlib.util
    import os

    from paper_1908_09301_b200 import _native

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "reference_binding.py")
    spec = importlib.util.spec_from_file_location("reference_binding", path)
    stub = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(stub)
    ctx, system, state = _lorenz(200)
    recs = stub.integrate_b200(_native.LIB_PATH, system, state, "0.01", 24, 250, 200, record_stride=100)
    traj = M.integrate(system, state, M.StepConfig("0.01", 24), 250, ctx, record_stride=100)
    assert [s for s, _ in recs] == traj.steps() == [0, 100, 200, 250]
    for (_, row), pt in zip(recs, traj.points):
        for (num, fb), v in zip(row, pt.state):
            assert Fraction(num, 1 << fb) == v.as_fraction()
