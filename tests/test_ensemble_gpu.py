"""Verification layer and ensembles on the B200 engine (GPU).

* cns_run through the device reproduces the reference's frozen paired-run
  outcome (reference tests/test_cns.py:119: t_c = 25 at d = 6);
* a batched ensemble gives, member by member, the same agreement series and
  divergence time as the single-trajectory drop-in path, and its states
  agree with the MPFR oracle (the reference algorithm) within 10^-(K-d(t)).
"""

import math
from decimal import Decimal
from fractions import Fraction

import numpy as np
import pytest

import paper_1908_09301_b200 as M
from oracle import ref as R
from paper_1908_09301_b200 import cns, ensemble as E

from .conftest import CANON_INIT
from .helpers import EXACT, agreement_digits, guard_digits

pytestmark = pytest.mark.gpu


def test_cns_run_reference_regression_pair(gpu):
    cfg = cns.CnsConfig(128, 20, 256, 30, "0.01", "25", agreement_digits=6)
    base, rep = cns.cns_run("lorenz", CANON_INIT, cfg)
    assert rep.t_c == Decimal("25.00")
    by_t = {str(t): d for _, t, d in rep.agreement}
    assert by_t["0.00"] == 38
    assert 22 <= by_t["1.00"] <= 24 and 12 <= by_t["25.00"] <= 14
    assert base.points[-1].step == 2500


def test_ensemble_matches_single_trajectory_cns(gpu):
    K, N, tau, t_end, stride, d = 40, 24, "0.01", "8", 100, 10
    inits = E.perturbed_inits(6, seed=0)
    rep = E.ensemble_tc(inits, K, N, tau, t_end, d=d, stride=stride)
    (bb, _), (vb, vn) = rep.base, rep.verify
    assert (bb, vb, vn) == (M.bits_for_digits(K), M.bits_for_digits(K + 50), N + 30)
    for m in (0, 3, 5):
        cfg = cns.CnsConfig(bb, N, vb, vn, tau, t_end, agreement_digits=d, stride=stride)
        _, single = cns.cns_run("lorenz", inits[m], cfg)
        want = [E.EXACT_CODE if v == math.inf else v for _, _, v in single.agreement]
        assert rep.agreement[:, m].tolist() == want
        assert rep.t_c[m] == single.t_c


def test_ensemble_members_vs_oracle(gpu):
    K, N, tau, n_steps = 60, 30, "0.01", 300
    P = M.bits_for_digits(K)
    inits = E.perturbed_inits(5, seed=7)
    run = E.run_members("lorenz", inits, P, N, tau, n_steps, n_steps)
    assert not run.status.any()
    final = run.ints(run.records.shape[0] - 1)
    F = run.fmt.frac_bits
    for m, row in enumerate(inits):
        rows = R.integrate(R.lorenz(P), [R.from_decimal(t, P) for t in row], R.from_decimal(tau, P), N, n_steps, P,
                           stride=n_steps)
        ref = [R.dy_to_fraction(v) for v in rows[-1][1]]
        got = [Fraction(x, 1 << F) for x in final[m]]
        dg = agreement_digits(got, ref)
        assert dg == EXACT or dg >= K - guard_digits(n_steps * 0.01, N), (m, dg)


def test_ensemble_perturbations_diverge_from_each_other(gpu):
    """Members start 1e-20 apart; chaos separates them (the ensemble is a
    real sweep, not copies of one trajectory)."""
    inits = E.perturbed_inits(4, seed=0)
    run = E.run_members("lorenz", inits, M.bits_for_digits(40), 24, "0.01", 5000, 5000)
    fin = run.ints(run.records.shape[0] - 1)
    F = run.fmt.frac_bits
    x = [Fraction(fin[m][0], 1 << F) for m in range(4)]
    assert len(set(x)) == 4
    assert max(abs(a - b) for a in x for b in x) > Fraction(1, 10**5)


# ------------------------------------------------- configs[4] sweep point on the device
def _oracle_series(init, K, N, tau, n_steps, stride):
    """Base and verify runs of one member by the reference-semantics oracle and
    their agreement series (the reference's cns.py:254 cns_run on the CPU)."""
    runs = []
    for k, n in ((K, N), (K + 50, N + 30)):
        P = M.bits_for_digits(k)
        rows = R.integrate(R.lorenz(P), [R.from_decimal(t, P) for t in init], R.from_decimal(tau, P), n, n_steps, P,
                           stride=stride)
        runs.append([[R.dy_to_fraction(v) for v in st] for _, st in rows])
    return [agreement_digits(a, b) for a, b in zip(*runs)]


def test_tc_sweep_real_pair_vs_single_trajectory_and_oracle(gpu):
    """(K, N) = (100, 60), 16 members x 5000 steps (t = 50), each against its own
    (150, 90) verify run: the sharded sweep entry point reproduces, member by
    member, the single-trajectory cns_run of the drop-in path (same agreement
    series, same t_c), shards concatenate to the unsharded result, and the
    divergence time agrees with the reference-semantics oracle's."""
    K, N, Mtot, n_steps, stride, d = 100, 60, 16, 5000, 100, 10
    rep = E.tc_sweep(K, N, Mtot, n_steps, d=d, stride=stride)
    assert rep.agreement.shape == (Mtot, 51) and rep.final_digits.shape[0] == Mtot
    bb, vb = M.bits_for_digits(K), M.bits_for_digits(K + 50)
    inits = E.perturbed_inits(Mtot, seed=0)
    for m in (0, 9, 15):
        cfg = cns.CnsConfig(bb, N, vb, N + 30, "0.01", "50", agreement_digits=d, stride=stride)
        _, single = cns.cns_run("lorenz", inits[m], cfg)
        want = [E.EXACT_CODE if v == math.inf else v for _, _, v in single.agreement]
        assert rep.agreement[m].tolist() == want
        assert rep.t_c()[m] == single.t_c
    # two shards (ranks 0 and 1 of a world of 2, no gather) concatenate to the full result
    parts = [E.tc_sweep(K, N, Mtot, n_steps, rank=r, world=2, d=d, stride=stride, gather=False) for r in range(2)]
    assert np.array_equal(np.concatenate([p.agreement for p in parts]), rep.agreement)
    assert np.array_equal(np.concatenate([p.tc_step for p in parts]), rep.tc_step)
    assert np.array_equal(np.concatenate([p.final_digits for p in parts]), rep.final_digits)
    # the oracle's own base/verify pair for one member: K = 100 digits minus the
    # Lyapunov loss crosses d = 10 well after t = 50, so both report t_c = t_end and
    # agreement series that differ by at most 2 digits sample by sample
    ser = _oracle_series(inits[9], K, N, "0.01", n_steps, stride)
    got = rep.agreement[9].tolist()
    assert rep.tc_step[9] == n_steps and all(v >= d for v in ser)
    for a, b in zip(got[1:], ser[1:]):
        assert abs(a - b) <= 2, (got, ser)
