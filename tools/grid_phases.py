"""Phase timestamps (clock64, MPT_DEBUG) of the grid kernel, CTA 0, thread 0, first step.
    python tools/grid_phases.py K N
0 order start, 1 Cauchy units done, 2 linear units + column sums added (RED), 3 after grid barrier 1,
4 numerators assembled, 5 U normalised, 6 C-product units + RED, 7 after grid barrier 2, 8 rows normalised, 9 published
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ["MPT_DEBUG"] = "1"
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

K, N = int(sys.argv[1]), int(sys.argv[2])
P = M.bits_for_digits(K); ctx = M.PrecisionContext(P); fmt = FixedFormat(P)
tab = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
st = fmt.to_digits([M.mp_from_decimal(x, ctx) for x in ("-15.8", "-17.48", "35.64")])
with DevicePlan(tab, fmt, N, 1) as plan:
    plan.configure("grid", 1)
    plan.upload(st)
    plan.run_device(1); plan.last_kernel_ms()
    buf = (ctypes.c_longlong * 65536)()
    plan.lib.mpt_debug_read(buf, 65536)
    os.environ.pop("MPT_DEBUG")
    plan.run_device(1)
    ms = plan.last_kernel_ms()
    info = plan.info()
n = min(N, 255)
d = np.array(list(buf)[: 256 * 16]).reshape(256, 16).astype(np.float64)
print(info, f"{ms:.3f} ms/step (no debug), {ms * 1.965e6 / N:.0f} cycles/order")
names = ["cauchy", "lin+red", "gbar1", "asm", "normU", "cprod+red", "gbar2", "normRow", "publish"]
for lo, hi in ((1, 32), (32, 128), (128, 255)):
    rr = [i for i in range(lo, min(hi, n - 1)) if d[i, 0] > 0 and d[i, 9] > 0]
    if not rr:
        continue
    seg = [np.mean([d[i, k + 1] - d[i, k] for i in rr]) for k in range(9)]
    tot = np.mean([d[i + 1, 0] - d[i, 0] for i in rr if d[i + 1, 0] > 0])
    print(f"orders {lo}-{hi} (only the first 255 orders are stamped): order-to-order {tot:.0f}: " + "  ".join(f"{nm} {v:.0f}" for nm, v in zip(names, seg)))
