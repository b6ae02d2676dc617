"""One warm-up launch and one measured launch of a chosen kernel (for ncu -k ... --launch-skip 1).
    python tools/one_launch.py K N steps n_traj kernel cluster
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

K, N, S, n_traj = (int(x) for x in sys.argv[1:5])
kern, cl = sys.argv[5], int(sys.argv[6])
P = M.bits_for_digits(K); ctx = M.PrecisionContext(P); fmt = FixedFormat(P)
t = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
base = [M.mp_from_decimal(x, ctx).as_fraction() for x in ("-15.8", "-17.48", "35.64")]
states = np.stack([fmt.to_digits(base) for _ in range(n_traj)])
with DevicePlan(t, fmt, N, n_traj) as plan:
    plan.configure(kern, cl)
    plan.upload(states)
    for _ in range(2):
        plan.run_device(S)
        print(plan.info()["kernel"], plan.last_kernel_ms(), "ms")
