"""Device-timed Taylor steps/s of a few workloads with explicit kernels (no e2e, no CPU leg).
    python tools/quick_perf.py name:K:N:steps:n_traj:kernel[/cluster] ...
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import numpy as np
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

for spec in sys.argv[1:]:
    name, K, N, S, n_traj, kern = spec.split(":")
    K, N, S, n_traj = int(K), int(N), int(S), int(n_traj)
    kern, _, cl = kern.partition("/")
    P = M.bits_for_digits(K); ctx = M.PrecisionContext(P); fmt = FixedFormat(P)
    t = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
    base = [M.mp_from_decimal(x, ctx).as_fraction() for x in ("-15.8", "-17.48", "35.64")]
    rng = np.random.default_rng(0)
    states = np.stack([fmt.to_digits([b + Fraction(int(rng.integers(-10**6, 10**6)), 10**26) for b in base]) for _ in range(n_traj)])
    with DevicePlan(t, fmt, N, n_traj) as plan:
        plan.configure(kern, int(cl or (16 if n_traj == 1 else 1)))
        plan.upload(states)
        plan.run_device(S); plan.last_kernel_ms()
        ms = []
        for _ in range(3):
            plan.run_device(S); ms.append(plan.last_kernel_ms())
        plan.count_macs(True); plan.run_device(S); plan.last_kernel_ms(); u, x = plan.read_macs()
        m = min(ms)
        print(f"{name} {kern}: {m:.2f} ms per {S} steps -> {n_traj * S / m * 1e3:.0f} traj-steps/s; useful MAC/s {u / m * 1e3:.3e} (frac of 9.44e12: {u / m * 1e3 / 9.44e12:.4f}) {plan.info()}", flush=True)
