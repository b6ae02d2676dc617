"""Per-warp phase timestamps (clock64, MPT_DEBUG) of the mx kernel's lead CTA, first step.
    python tools/mx_phases.py K N G
per order and warp: 0 start, 1 products/aux done, 2 after barrier, 3 roundings (+pushes) done,
4 cp.async landed, 5 after barrier, 6 after C-row info + barrier
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

os.environ["MPT_DEBUG"] = "1"
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import DevicePlan, SystemTables
from paper_1908_09301_b200.fixed import FixedFormat

K, N, G = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
P = M.bits_for_digits(K)
ctx = M.PrecisionContext(P)
fmt = FixedFormat(P)
tab = SystemTables.build(M.builtin_system("lorenz", ctx), fmt, N, M.mp_from_decimal("0.01", ctx).as_fraction())
st = fmt.to_digits([M.mp_from_decimal(x, ctx) for x in ("-15.8", "-17.48", "35.64")])
with DevicePlan(tab, fmt, N, 1) as plan:
    plan.configure("mx", G)
    plan.upload(st)
    plan.run_device(1)
    plan.last_kernel_ms()
    buf = (ctypes.c_longlong * 65536)()
    plan.lib.mpt_debug_read(buf, 65536)
    os.environ.pop("MPT_DEBUG")
    plan.run_device(3)
    ms = plan.last_kernel_ms() / 3
    info = plan.info()
d = np.array(list(buf)[: 256 * 16 * 8]).reshape(256, 16, 8).astype(np.float64)
bd = np.array(list(buf)[40000: 40000 + 2 * 256 * 8]).reshape(2, 256, 8).astype(np.float64)
print(info, f"{ms:.3f} ms/step (no debug), {ms * 1.965e6 / N:.0f} cycles/order")
for lo, hi in ((1, 8), (8, 32), (32, 64), (64, 128), (128, 256)):
    rr = [i for i in range(lo, min(hi, N - 1, 255)) if d[i, 0, 0] > 0 and d[i + 1, 0, 0] > 0]
    if not rr:
        continue
    t0 = np.array([d[i, 0, 0] for i in rr])
    print(f"orders {lo}-{hi}: order-to-order {np.mean([d[i + 1, 0, 0] - d[i, 0, 0] for i in rr]):.0f}")
    for w in (0, 3, 6, 15):
        row = [np.mean([d[i, w, k] - d[i, 0, 0] for i in rr]) for k in range(7)]
        print(f"  warp {w:2d}: " + " ".join(f"{x:7.0f}" for x in row))

# bulk ranks 1 and 2 (rank 2 owns k = 2: new terms every order): 0 loop top, 1 row arrived,
# 2 new terms absorbed, 3 L' pushed, 4 old terms absorbed
for o in range(2):
    for lo, hi in ((2, 32), (32, 128), (128, 256)):
        rr = [r for r in range(lo, min(hi, N - 3)) if bd[o, r, 0] > 0 and bd[o, r + 1, 0] > 0]
        if not rr:
            continue
        seg = lambda a, b: np.mean([bd[o, r, b] - bd[o, r, a] for r in rr])
        per = np.mean([bd[o, r + 1, 0] - bd[o, r, 0] for r in rr])
        print(f"bulk rank {o + 1} rows {lo}-{hi}: per-row {per:.0f}: wait {seg(0, 1):.0f} new {seg(1, 2):.0f} "
              f"push {seg(2, 3):.0f} old {seg(3, 4):.0f}")
