"""Quick GPU check of the warp kernel: bit-exactness vs the model and speed.
    python tools/warp_check.py
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import numpy as np
import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

INIT = ("-15.8", "-17.48", "35.64")


def tables_for(K, N):
    P = M.bits_for_digits(K)
    ctx = M.PrecisionContext(P)
    fmt = FixedFormat(P)
    system = M.builtin_system("lorenz", ctx)
    t = SystemTables.build(system, fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
    base = [M.mp_from_decimal(x, ctx).as_fraction() for x in INIT]
    return P, ctx, fmt, t, base


for K, N, steps, n_traj in [(20, 14, 10, 2), (50, 40, 10, 1), (100, 60, 4, 9), (150, 90, 2, 3), (200, 120, 2, 33), (250, 150, 1, 2)]:
    P, ctx, fmt, t, base = tables_for(K, N)
    states = np.stack([fmt.to_digits([b + Fraction(5 * j - 7, 10**18) for b in base]) for j in range(n_traj)])
    with DevicePlan(t, fmt, N, n_traj) as plan:
        plan.configure("warp", 1)
        try:
            _, r, status = plan.integrate(states, steps, 0, 1)
        except Exception as e:
            print(K, N, "FAILED", e)
            continue
        jets = plan.compute_jet(states)
    bad = []
    for j in range(n_traj):
        _, rc = FX.integrate(t, fmt.frac_digits, N, P, states[j], steps, 0, 1, variant=3)
        jc = FX.compute_jet(t, fmt.frac_digits, N, states[j], variant=3)
        if not np.array_equal(r[:, j], rc):
            bad.append(("rec", j))
        if not np.array_equal(jets[j], jc):
            rows = [(m, i) for m in range(3) for i in range(N + 1) if not np.array_equal(jets[j][m, i], jc[m, i])]
            bad.append(("jet", j, rows[:4]))
    print(f"K={K} N={N} W={fmt.width} traj={n_traj}: status={status.tolist()[:4]} {'OK' if not bad else bad[:4]}", flush=True)

for name, K, N, S, n_traj in [("k50", 50, 40, 100, 1), ("ens100", 100, 60, 10, 4096), ("ens150v", 150, 90, 10, 4096),
                              ("ens200", 200, 120, 5, 4096), ("ens250v", 250, 150, 5, 4096)]:
    P, ctx, fmt, t, base = tables_for(K, N)
    rng = np.random.default_rng(0)
    states = np.stack([fmt.to_digits([b + Fraction(int(rng.integers(-10**6, 10**6)), 10**26) for b in base])
                       for j in range(n_traj)])
    for kern in ("warp", "team") if n_traj > 1 else ("warp", "mx"):
        with DevicePlan(t, fmt, N, n_traj) as plan:
            plan.configure(kern, 16 if kern == "mx" else 1)
            plan.upload(states)
            plan.run_device(S)
            plan.last_kernel_ms()
            plan.count_macs(True)
            plan.run_device(S)
            ms = plan.last_kernel_ms()
            u, x = plan.read_macs()
            print(f"{name} {kern}: {ms:.2f} ms per {S} steps -> {n_traj * S / ms * 1e3:.0f} traj-steps/s; useful {u:.3e} executed {x:.3e} "
                  f"useful MAC/s {u / ms * 1e3:.3e} info {plan.info()}", flush=True)
