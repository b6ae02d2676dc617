import sys, ctypes, numpy as np
sys.path.insert(0,'.')
import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import SystemTables, DevicePlan, _p
from paper_1908_09301_b200.fixed import FixedFormat
for (P,N) in ((128,8),):
  ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
  tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
  st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
  cj=FX.compute_jet(tab,fmt.frac_digits,N,st)
  for kern,G in (('cluster',1),('cluster',2)):
    with DevicePlan(tab,fmt,N,1) as plan:
        plan.configure(kern,G)
        s=np.ascontiguousarray(st,dtype=np.int32)
        coef=np.zeros((1,3,N+1,fmt.width),np.int32); status=np.zeros(1,np.int32)
        rc=plan.lib.mpt_compute_jet(plan.h,_p(s),_p(coef),_p(status))
        gj=coef[0]
        print(kern,G,'rc',rc,'status',status)
        for i in range(N+1):
            for m in range(3):
                if not np.array_equal(gj[m,i],cj[m,i]):
                    print(' first diff m',m,'i',i); print('  gpu',gj[m,i].tolist()); print('  cpu',cj[m,i].tolist())
                    break
            else: continue
            break
