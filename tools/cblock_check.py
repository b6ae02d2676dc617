"""Quick GPU check of the cblock kernel: bit-exactness vs the value-exact model (records and jet)
at several (K, N, cluster) shapes, then device-timed speed against mx.
    python tools/cblock_check.py [fast]
"""
import sys, os
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


fast = "fast" in sys.argv
shapes = [(50, 40, 6, 1, 2), (100, 60, 4, 2, 4), (300, 100, 3, 1, 8), (500, 200, 2, 1, 16), (500, 200, 2, 1, 8),
          (500, 200, 1, 1, 3), (700, 120, 2, 1, 16), (500, 37, 3, 3, 5)]
for K, N, steps, n_traj, G in shapes:
    P, ctx, fmt, t, base = tables_for(K, N)
    states = np.stack([fmt.to_digits([b + Fraction(5 * j - 7, 10**18) for b in base]) for j in range(n_traj)])
    with DevicePlan(t, fmt, N, n_traj) as plan:
        try:
            plan.configure("cblock", G)
            info = plan.info()
            _, r, status = plan.integrate(states, steps, 0, 1)
            jets = plan.compute_jet(states)
        except Exception as e:
            print(K, N, G, "FAILED", e, flush=True)
            continue
    bad = []
    for j in range(n_traj):
        _, rc = FX.integrate(t, fmt.frac_digits, N, P, states[j], steps, 0, 1, variant=3)
        jc = FX.compute_jet(t, fmt.frac_digits, N, states[j], variant=3)
        if not np.array_equal(r[:, j], rc):
            bad.append(("rec", j))
        if not np.array_equal(jets[j], jc):
            rows = [(m, i) for m in range(3) for i in range(N + 1) if not np.array_equal(jets[j][m, i], jc[m, i])]
            bad.append(("jet", j, rows[:4]))
    print(f"K={K} N={N} W={fmt.width} traj={n_traj} G={G}: status={status.tolist()[:4]} {'OK' if not bad else bad[:4]} {info}", flush=True)

perf = [("k500", 500, 200, 100, 1, ("cblock/16", "cblock/8", "mx/16")), ("k50", 50, 40, 100, 1, ("cblock/2", "cblock/4", "warp/1")),
        ("k300", 300, 150, 100, 1, ("cblock/16", "mx/16")), ("k800", 800, 300, 20, 1, ("cblock/16", "mx/16"))]
for name, K, N, S, n_traj, kerns in perf:
    P, ctx, fmt, t, base = tables_for(K, N)
    states = np.stack([fmt.to_digits(base) for j in range(n_traj)])
    for kc in kerns:
        kern, _, cl = kc.partition("/")
        try:
            with DevicePlan(t, fmt, N, n_traj) as plan:
                plan.configure(kern, int(cl))
                plan.upload(states)
                plan.run_device(S)
                plan.last_kernel_ms()
                ms = []
                for _ in range(3):
                    plan.run_device(S)
                    ms.append(plan.last_kernel_ms())
                plan.count_macs(True)
                plan.run_device(S)
                plan.last_kernel_ms()
                u, x = plan.read_macs()
                m = min(ms)
                print(f"{name} {kc}: {m:.2f} ms per {S} steps -> {n_traj * S / m * 1e3:.0f} steps/s ({m * 1e-3 * 1.965e9 / S / N:.0f} cycles/order); "
                      f"useful {u:.3e} executed {x:.3e} useful MAC/s {u / m * 1e3:.3e} info {plan.info()}", flush=True)
        except Exception as e:
            print(name, kc, "FAILED", e, flush=True)
