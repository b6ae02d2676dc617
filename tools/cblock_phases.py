"""Phase timestamps (clock64, MPT_DEBUG) of the cblock kernel, rank 0, first step.
    python tools/cblock_phases.py K N G
per order, warps 0 (target + units), 8 (element sums + pushes), 13 (side warp with the non-integer linear product):
0 order start, 1 zmin done, 2 side job done, 3 unit products done, 4 arrival at S1, 5 pushes issued, 6 after the cluster
barrier, 7 U assembled, 9 U rounded, 11 U x C chunk done, 13 row rounded. Stamps taken right after a barrier are not
reliable (the clock read is scheduled before the barrier resolves): read arrivals.
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
os.environ["MPT_DEBUG"] = "1"
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

K, N, G = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
P = M.bits_for_digits(K); ctx = M.PrecisionContext(P); fmt = FixedFormat(P)
tab = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
st = fmt.to_digits([M.mp_from_decimal(x, ctx) for x in ("-15.8", "-17.48", "35.64")])
with DevicePlan(tab, fmt, N, 1) as plan:
    plan.configure("cblock", G)
    plan.upload(st)
    plan.run_device(1); plan.last_kernel_ms()
    buf = (ctypes.c_longlong * 65536)()
    plan.lib.mpt_debug_read(buf, 65536)
    os.environ.pop("MPT_DEBUG")
    plan.run_device(3)
    ms = plan.last_kernel_ms() / 3
    info = plan.info()
n = min(N, 256)
d = np.array(list(buf)[: n * 3 * 16]).reshape(n, 3, 16).astype(np.float64)
print(info, f"{ms:.3f} ms/step (no debug), {ms * 1.965e6 / N:.0f} cycles/order")
for lo, hi in ((1, 8), (8, 32), (32, 64), (64, 128), (128, 256)):
    rr = [i for i in range(lo, min(hi, n - 1))]
    if not rr:
        continue
    print(f"orders {lo}-{hi}: order-to-order {np.mean([d[i + 1, 0, 0] - d[i, 0, 0] for i in rr]):.0f}")
    for w, name in ((0, "w0 "), (1, "w8 "), (2, "w13")):
        row = [np.mean([d[i, w, k] - d[i, 0, 0] for i in rr if d[i, w, k] > 0] or [0]) for k in range(15)]
        print(f"  {name}: " + " ".join(f"{x:6.0f}" for x in row))
