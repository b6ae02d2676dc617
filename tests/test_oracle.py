"""The CPU oracle, pinned against the reference's own outputs.

tests/golden/reference_golden.json was produced by running the UNMODIFIED
reference package (tests/golden/make_golden.py) and is cross-checked there
against the C oracle. These tests re-establish the pin on every run (no
/root/reference needed) and check the reference's own known answers:
hand-derived coefficients (test_acceptance.py criterion 1), e within 1e-32
(criterion 2) and the frozen agreement series of the 128/256-bit pair
(test_cns.py:119: 38 digits at t=0, 23 at t=1, 13 at t=25, t_c = 25).
"""

from fractions import Fraction

import pytest

from oracle import ref as R

from .helpers import agreement_digits, frac


def _sys(case):
    js = case["system"]
    return {
        "dim": js["dim"],
        "constant": [R.dy_from_hex(h) for h in js["constant"]],
        "linear": [[R.dy_from_hex(h) for h in row] for row in js["linear"]],
        "terms": [(m, j, k, R.dy_from_hex(h)) for m, j, k, h in js["terms"]],
    }


def _same(a: R.Dy, hexval: str) -> bool:
    return R.dy_hex(a) == R.dy_hex(R.dy_from_hex(hexval))


@pytest.mark.parametrize(
    "name", ["config0_k50_n40", "cns_pair_128_n20", "config1_k500_n200_3steps", "zero_state_256_n8",
             "backward_256_n30",
             # N = 300 >= the serial threshold 256: the chunked branch of the
             # reference reduction (reduction.py:136-146) is pinned here
             "chunked_256_n300_3steps",
             # the reduction plan the timed reference arm runs (threshold 32)
             "plan_t32_k500_n200_2steps"]
)
def test_oracle_integrate_bit_identical_to_reference(golden, name):
    c = golden[name]
    P = c["prec_bits"]
    plan = c.get("plan", {})
    rows = R.integrate(_sys(c), [R.dy_from_hex(h) for h in c["init_values"]], R.dy_from_hex(c["tau_value"]),
                       c["order"], c["n_steps"], P, stride=c["stride"], **plan)
    assert [s for s, _ in rows] == [r["step"] for r in c["records"]]
    for (s, state), rec in zip(rows, c["records"]):
        for v, h in zip(state, rec["state"]):
            assert _same(v, h), (name, s)


def test_oracle_jets_bit_identical_to_reference(golden):
    for name, c in golden.items():
        if c["kind"] != "jet":
            continue
        jet = R.compute_jet(_sys(c), [R.dy_from_hex(h) for h in c["state"]], c["order"], c["prec_bits"])
        for m, row in enumerate(c["coeffs"]):
            for i, h in enumerate(row):
                assert _same(jet[m][i], h), (name, m, i)


def test_hand_values_criterion_1(golden):
    c = golden["lorenz_jet_256_n6"]
    ulp = Fraction(1, 2**256)
    for (m, i), text in {(0, 1): "-16.8", (1, 1): "138.192", (2, 1): "181.144"}.items():
        got = frac(c["coeffs"][m][i])
        assert abs(got - Fraction(text)) <= 2 * ulp * abs(Fraction(text)) * 2
    assert abs(frac(c["coeffs"][0][2]) - Fraction("774.96")) < Fraction(1, 10**70)


def test_exponential_criterion_2(golden):
    c = golden["exp_tau1_n30_256"]
    e = Fraction(0)
    term = Fraction(1)
    for n in range(1, 80):
        e += term
        term /= n
    assert abs(frac(c["result"][0]) - e) < Fraction(1, 10**32)


def test_reference_regression_pair_agreement_series(golden):
    a, b = golden["cns_pair_128_n20"], golden["cns_pair_256_n30"]
    series = {}
    for ra, rb in zip(a["records"], b["records"]):
        series[ra["step"]] = agreement_digits([frac(h) for h in ra["state"]], [frac(h) for h in rb["state"]])
    assert series[0] == 38 and series[100] == 23 and series[2500] == 13
    assert min(series.values()) >= 6  # t_c = 25.00 at d = 6


def test_oracle_chunked_reduction_threads_do_not_change_bits():
    """reduction.py worker independence: OpenMP thread count never changes bits."""
    P = 256
    vals = [[R.from_decimal(str((k * 37 + s) % 101 - 50) + "." + str(k % 7), P) for k in range(300)]
            for s in range(4)]
    one = R.convolve(vals, 299, P, chunks=64, threshold=16, threads=1)
    four = R.convolve(vals, 299, P, chunks=64, threshold=16, threads=4)
    assert [R.dy_hex(v) for v in one] == [R.dy_hex(v) for v in four]
