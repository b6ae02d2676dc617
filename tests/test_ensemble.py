"""Host logic of the verification layer and of ensembles (CPU only).

* cns.py mirrors the reference's cns.py; the hand cases follow the
  reference's tests/test_cns.py (TestAgreementDigits, CnsConfig validation,
  estimate_tc on fabricated trajectories).
* ensemble.py: seeded perturbations, shard bounds, the exact agreement
  matrix against cns.agreement_digits, divergence times, and the N>1 gather
  path with world_size 2 over gloo.
"""

import math
import os
import socket
import warnings
from decimal import Decimal
from fractions import Fraction

import numpy as np
import pytest

import paper_1908_09301_b200 as M
from paper_1908_09301_b200 import cns, ensemble as E
from paper_1908_09301_b200.fixed import FixedFormat
from paper_1908_09301_b200.taylor import Trajectory, TrajectoryPoint

from .helpers import floor_neg_log10


# ------------------------------------------------------------------ cns
@pytest.fixture
def ctx256():
    return M.PrecisionContext(256)


def test_agreement_hand_cases(ctx256):
    one = ctx256.one
    s = (one, one, one)
    assert cns.agreement_digits(s, s) == cns.AGREEMENT_EXACT == math.inf
    assert cns.agreement_digits((ctx256.from_int(3),), (M.PrecisionContext(64).from_int(3),)) == math.inf
    b = (M.mp_from_decimal("1.00000001", ctx256), one, one)
    rel = abs(b[0].as_fraction() - 1) / b[0].as_fraction()
    assert cns.agreement_digits(s, b) == floor_neg_log10(rel) == 8
    z = (ctx256.zero,) * 3
    zb = (M.mp_from_decimal("0.001", ctx256), ctx256.zero, ctx256.zero)
    assert cns.agreement_digits(z, zb) == floor_neg_log10(abs(zb[0].as_fraction())) == 3
    assert cns.agreement_digits((ctx256.from_int(5),), (ctx256.from_int(-5),)) == 0
    two = (M.mp_from_decimal("1.001", ctx256), M.mp_from_decimal("1.000001", ctx256))
    assert cns.agreement_digits((one, one), two) == 3
    with pytest.raises(ValueError):
        cns.agreement_digits((one,), (one, one))


@pytest.mark.parametrize("num,den", [(1, 10), (1, 11), (1, 9), (7, 10**40), (10**5, 10**5), (3, 2)])
def test_floor_neg_log10_ratio(num, den):
    assert cns.floor_neg_log10_ratio(num, den) == floor_neg_log10(Fraction(num, den))


def test_cns_config_validation():
    ok = cns.CnsConfig(128, 20, 256, 30, "0.01", "25")
    assert ok.n_steps() == 2500
    with pytest.raises(cns.ConfigError) as e:
        cns.CnsConfig(128, 20, 128, 20, "0.01", "25")
    assert len(e.value.problems) == 2
    cns.CnsConfig(128, 20, 128, 20, "0.01", "25", allow_equal_verify=True)
    with pytest.raises(cns.ConfigError):
        cns.CnsConfig(128, 20, 256, 30, "0.01", "-1")
    with pytest.raises(cns.ConfigError):
        cns.CnsConfig(128, 20, 256, 30, "0.01", "25", agreement_digits=0)
    with pytest.raises(cns.ConfigError):
        cns.CnsConfig(128, 20, 256, 30, "0.03", "1").n_steps()
    assert cns.default_verify_margins(300, 30) == (399, 40)


def _traj(vals, prec, tau="0.5"):
    tr = Trajectory(dim=1, tau_text=tau)
    for s, v in vals:
        tr.points.append(TrajectoryPoint(step=s, state=(M.MPValue.from_fraction(Fraction(v), prec),)))
    return tr


def test_estimate_tc_series_and_reports():
    a = _traj([(0, "1"), (1, "1"), (2, "1"), (3, "1")], 128)
    b = _traj([(0, "1"), (1, "1.0000000000001"), (2, "1.00001"), (3, "2")], 128)
    rep = cns.estimate_tc(a, b, 10)
    assert [d for _, _, d in rep.agreement] == [math.inf, 13, 5, 0]
    assert rep.t_c == Decimal("0.5") and rep.t_end == Decimal("1.5")
    assert rep.tc_for(5) == Decimal("1.0") and rep.tc_for(20) == Decimal(0)
    assert "t_c=0.5" in rep.to_kv() and "inf" in rep.agreement_tsv()
    assert "reliable up to t_c = 0.5" in rep.to_text()
    with pytest.raises(ValueError):
        cns.estimate_tc(a, b, 0)
    with pytest.raises(cns.ConfigError):
        cns.estimate_tc(a, _traj([(0, "1")], 128), 3)
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        rep = cns.estimate_tc(a, b, 100)
    assert rep.t_c == 0 and w
    assert cns.diagram_tsv([(38, Decimal("25.00"), None)]) == "# param\tt_c\n38\t25.00\n"


# ------------------------------------------------------------- ensemble
def test_perturbed_inits_seeded_and_bounded():
    a = E.perturbed_inits(64, seed=0)
    assert a == E.perturbed_inits(64, seed=0) and a != E.perturbed_inits(64, seed=1)
    assert len(set(a)) == 64
    for row in a:
        for t, base in zip(row, E.CANON_INIT):
            assert abs(Decimal(t) - Decimal(base)) <= Decimal("1e-20")


@pytest.mark.parametrize("n,world", [(4096, 1), (4096, 2), (4096, 8), (7, 3), (3, 8), (0, 2)])
def test_shard_bounds_partition(n, world):
    got = [E.shard_bounds(n, world, r) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    assert all(got[r][1] == got[r + 1][0] for r in range(world - 1))
    sizes = [h - l for l, h in got]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        E.shard_bounds(n, world, world)


def _fake_run(bits, vals, steps, tau="0.01"):
    fmt = FixedFormat(bits)
    recs = np.stack([np.stack([fmt.to_digits([M.MPValue.from_fraction(Fraction(x), bits) for x in st])
                               for st in member]) for member in vals])
    return E.EnsembleRun(bits, 10, tau, fmt, np.array(steps, np.int32), recs, np.zeros(recs.shape[1], np.int32))


def test_agreement_matrix_matches_cns_metric():
    rng = np.random.default_rng(3)
    steps = [0, 100, 200]
    base, ver = [], []
    for r in range(len(steps)):
        rb, rv = [], []
        for m in range(5):
            x = [Fraction(int(rng.integers(-10**9, 10**9)), 10**7) for _ in range(3)]
            eps = Fraction(1, 10 ** int(rng.integers(3, 60)))
            y = [x[0] + eps * (m % 2), x[1], x[2] - eps * (r % 2)]
            rb.append(x)
            rv.append(y)
        base.append(rb)
        ver.append(rv)
    a, b = _fake_run(256, base, steps), _fake_run(420, ver, steps)
    mat = E.agreement_matrix(a, b)
    for r in range(len(steps)):
        for m in range(5):
            va = [M.MPValue.from_fraction(Fraction(v), 256) for v in base[r][m]]
            vb = [M.MPValue.from_fraction(Fraction(v), 420) for v in ver[r][m]]
            want = cns.agreement_digits(va, vb)
            assert mat[r, m] == (E.EXACT_CODE if want == math.inf else want)
    tc = E.divergence_times(a.steps, "0.01", mat, 10)
    for m in range(5):
        series = [(s, M.exact_time(s, "0.01"), math.inf if v == E.EXACT_CODE else v)
                  for s, v in zip(steps, mat[:, m])]
        assert tc[m] == cns.tc_from_series(series, 10)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, n_total, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = E.shard_bounds(n_total, world, rank)
    local = np.arange(lo * 6, hi * 6, dtype=np.int32).reshape(hi - lo, 2, 3)
    full = E.gather_rows(local, n_total, world, rank)
    q.put((rank, full.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [7, 8])
def test_gather_rows_world2_gloo(n_total):
    import torch.multiprocessing as mp

    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_gather_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(n_total * 6, dtype=np.int32).reshape(n_total, 2, 3).tolist()
    assert got[0] == want and got[1] == want


# ------------------------------------------------------- T_c-K sweep (host logic)
def _model_run(inits, bits, order, tau_text, n_steps, stride):
    """run_fn for tc_sweep on the CPU: every member through the bit-exact model of
    the device arithmetic (oracle/fixmodel.c) -- same digit tables, same records."""
    from oracle import fix as FX
    from paper_1908_09301_b200.engine import SystemTables

    ctx = M.PrecisionContext(bits)
    fmt = FixedFormat(bits)
    system = M.builtin_system("lorenz", ctx)
    tables = SystemTables.build(system, fmt, order, M.mp_from_decimal(tau_text, ctx).as_fraction())
    states = E.states_from_decimals(inits, bits, fmt)
    recs, steps = [], None
    for st in states:
        steps, r = FX.integrate(tables, fmt.frac_digits, order, bits, st, n_steps, 0, stride)
        recs.append(r)
    return E.EnsembleRun(bits, order, tau_text, fmt, steps, np.stack(recs, axis=1),
                         np.zeros(len(inits), np.int32))


SWEEP = dict(K=20, N=14, n_members=5, n_steps=2400, stride=100, d=10)


def _sweep_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep = E.tc_sweep(rank=rank, world=world, run_fn=_model_run, **SWEEP)
    q.put((rank, rep.agreement.tolist(), rep.tc_step.tolist(), rep.final_digits.tolist(), rep.final_xyz.tolist()))
    dist.destroy_process_group()


def test_tc_sweep_world2_gloo_matches_world1():
    """Shard -> base + verify runs -> agreement -> t_c -> gather, world 2 over
    gloo, against the unsharded result: identical for every member (the
    reference's cross-worker-count bit-identity check, bench.py:62 run_benchmark)."""
    import torch.multiprocessing as mp

    one = E.tc_sweep(run_fn=_model_run, **SWEEP)
    assert one.agreement.shape == (5, 25) and one.final_digits.shape[:2] == (5, 3)
    # K=20 digits, d=10: the pair separates inside the run (a real divergence time)
    assert (one.tc_step > 0).all() and (one.tc_step < SWEEP["n_steps"]).any()
    tcs = E.divergence_times(one.steps, "0.01", one.agreement.T, SWEEP["d"])
    assert [E.exact_time(int(s), "0.01") for s in one.tc_step] == tcs == one.t_c()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {r: rest for r, *rest in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [one.agreement.tolist(), one.tc_step.tolist(), one.final_digits.tolist(), one.final_xyz.tolist()]
    assert got[0] == want and got[1] == want


def test_tc_steps_edge_cases():
    steps = np.array([0, 100, 200, 300])
    agr = np.array([[E.EXACT_CODE, 30, 20, 12], [E.EXACT_CODE, 30, 9, 12], [5, 30, 20, 12], [E.EXACT_CODE, 9, 20, 3]])
    assert E.tc_steps(steps, agr, 10).tolist() == [300, 100, 0, 0]
    assert E.tc_steps(steps, np.zeros((0, 4), np.int64), 10).tolist() == []
    with pytest.raises(ValueError):
        E.tc_sweep(20, 14, 4, 150, stride=100, run_fn=_model_run)


def test_decimal_to_fixed_int_matches_mp_path():
    import random

    rnd = random.Random(5)
    for bits in (64, 167, 499, 2658):
        ctx, fmt = M.PrecisionContext(bits), FixedFormat(bits)
        texts = ["0", "-0.0", "1", "-15.8", "35.64", "1e-20", "-17.48000000000000000000731", "134217727.9999", ".5", "2.5e-1"]
        texts += [f"{rnd.choice(['', '-'])}{rnd.randint(0, 10**rnd.randint(1, 8))}.{rnd.randint(0, 10**50):050d}e{rnd.randint(-30, 0)}"
                  for _ in range(100)]
        for t in texts:
            assert E.decimal_to_fixed_int(t, bits, fmt) == fmt.to_int(M.mp_from_decimal(t, ctx)), (bits, t)
        with pytest.raises(M.RangeError):
            E.decimal_to_fixed_int("134217728", bits, fmt)
        with pytest.raises(ValueError):
            E.decimal_to_fixed_int("1,5", bits, fmt)


def test_agreement_matrix_fast_path_equals_exact():
    """The vectorised digit count (three leading digits in floating point, exact
    fallback near integer boundaries) against the all-integer computation, on
    random differences of every size and on exact powers of ten."""
    rng = np.random.default_rng(11)
    steps = list(range(6))
    base, ver = [], []
    for r in steps:
        rb, rv = [], []
        for m in range(40):
            x = [Fraction(int(rng.integers(-10**12, 10**12)), 10 ** int(rng.integers(5, 14))) for _ in range(3)]
            k = int(rng.integers(1, 70))
            eps = Fraction(int(rng.integers(1, 10)) if m % 3 else 1, 10**k)  # m % 3 == 0: exactly 10^-k
            rb.append(x)
            rv.append([x[0] + eps * (m % 2), x[1] - eps, x[2] if m % 5 else x[2] * 0])
        base.append(rb)
        ver.append(rv)
    a, b = _fake_run(300, base, steps), _fake_run(470, ver, steps)
    assert np.array_equal(E.agreement_matrix(a, b), E.agreement_matrix_exact(a, b))
    assert (E.agreement_matrix(a, a) == E.EXACT_CODE).all()
