import time, sys, os
import numpy as np
sys.path.insert(0,'.')
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat
def perf(K, N, steps, configs):
    P=M.bits_for_digits(K); ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
    tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
    st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
    for kern, G in configs:
        with DevicePlan(tab,fmt,N,1) as plan:
            try: plan.configure(kern, G)
            except Exception as e: print(kern,G,'unavailable',e); continue
            plan.upload(st); plan.run_device(2); plan.last_kernel_ms()
            plan.count_macs(True); plan.run_device(steps); ms=plan.last_kernel_ms(); u,x=plan.read_macs()
            print(f'K={K} N={N} {plan.info()} : {ms/steps:.3f} ms/step = {1000*steps/ms:.1f} steps/s; useful MAC/step {u/steps:.3e} executed {x/steps:.3e}', flush=True)
perf(50,40,100,[('pipe',1)])
perf(500,200,20,[('cluster',16),('pipe',16)])
perf(500,200,20,[('grid',1)])
perf(800,480,2,[('team',1),('grid',1)])
perf(2200,1000,1,[('grid',1)])
perf(4200,3500,1,[('grid',1)])
