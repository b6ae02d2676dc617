import sys, os
sys.path.insert(0,'.')
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat
K,N,steps,kern,G=int(sys.argv[1]),int(sys.argv[2]),int(sys.argv[3]),sys.argv[4],int(sys.argv[5])
P=M.bits_for_digits(K); ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
with DevicePlan(tab,fmt,N,1) as plan:
    plan.configure(kern,G); plan.upload(st); plan.run_device(steps); ms=plan.last_kernel_ms()
    print(plan.info(), f'{ms/steps:.3f} ms/step')
