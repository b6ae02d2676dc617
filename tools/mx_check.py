"""Quick bit-exactness check of a kernel against oracle/fixmodel.c (test infrastructure).

    python tools/mx_check.py mx 16 167:40:5 1661:200:2
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

kern, G = sys.argv[1], int(sys.argv[2])
for spec in sys.argv[3:]:
    P, N, steps = (int(x) for x in spec.split(":"))
    ctx = M.PrecisionContext(P)
    system = M.builtin_system("lorenz", ctx)
    fmt = FixedFormat(P)
    tables = SystemTables.build(system, fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
    st = fmt.to_digits([M.mp_from_decimal(t, ctx) for t in ("-15.8", "-17.48", "35.64")])
    with DevicePlan(tables, fmt, N, 1) as plan:
        plan.configure(kern, G)
        info = plan.info()
        t = time.time()
        jet = plan.compute_jet(st)[0]
        s_gpu, r_gpu, status = plan.integrate(st, steps, 0, 1)
        dt = time.time() - t
        kw = plan.model_kwargs()
    cj = FX.compute_jet(tables, fmt.frac_digits, N, st, **kw)
    s_cpu, r_cpu = FX.integrate(tables, fmt.frac_digits, N, P, st, steps, 0, 1, **kw)
    ok_j = np.array_equal(jet, cj)
    ok_i = np.array_equal(r_gpu[:, 0], r_cpu)
    print(f"P={P} N={N} steps={steps} {info} model={kw} status={status.tolist()} jet_ok={ok_j} "
          f"integrate_ok={ok_i} ({dt:.2f}s)", flush=True)
    if not ok_j:
        bad = np.argwhere(jet != cj)
        m, i, d = bad[0]
        print("  first jet mismatch at var", m, "order", i, "digit", d, "gpu", jet[m, i, d], "model", cj[m, i, d],
              "n_bad", len(bad), "orders with mismatches", sorted(set(bad[:, 1].tolist()))[:10])
