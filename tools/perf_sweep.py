"""Kernel sweep on one GPU: device ms per Taylor step for each kernel / cluster size.

    python tools/perf_sweep.py 500:200:20:mx/16,mx/8 2200:1000:1:grid/1

Each argument is K:N:steps:kernel/G[,kernel/G...]. Not part of the product path.
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat


def perf(K, N, steps, configs):
    P = M.bits_for_digits(K); ctx = M.PrecisionContext(P); sysm = M.builtin_system('lorenz', ctx); fmt = FixedFormat(P)
    tab = SystemTables.build(sysm, fmt, N, M.mp_from_decimal('0.01', ctx).as_fraction())
    st = fmt.to_digits([M.mp_from_decimal(x, ctx) for x in ('-15.8', '-17.48', '35.64')])
    for kern, G in configs:
        with DevicePlan(tab, fmt, N, 1) as plan:
            try:
                plan.configure(kern, G)
            except Exception as e:
                print(kern, G, 'unavailable', e, flush=True); continue
            plan.upload(st); plan.run_device(min(2, steps)); plan.last_kernel_ms()
            plan.count_macs(True); plan.run_device(steps); ms = plan.last_kernel_ms(); u, x = plan.read_macs()
            print(f'K={K} N={N} {plan.info()} : {ms/steps:.3f} ms/step = {1000*steps/ms:.1f} steps/s, '
                  f'{ms*1e3/steps/N:.2f} us/order; useful MAC/step {u/steps:.3e} executed {x/steps:.3e}', flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        K, N, steps, ks = arg.split(":")
        perf(int(K), int(N), int(steps), [(k.split("/")[0], int(k.split("/")[1])) for k in ks.split(",")])
