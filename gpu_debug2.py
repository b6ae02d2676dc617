import sys, ctypes, os, numpy as np
os.environ['MPT_DEBUG']='1'
sys.path.insert(0,'.')
import paper_1908_09301_b200 as M
from oracle import fix as FX
from paper_1908_09301_b200.engine import SystemTables, DevicePlan, _p
from paper_1908_09301_b200.fixed import FixedFormat
P,N=128,8
ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
with DevicePlan(tab,fmt,N,1) as plan:
    plan.configure('cluster',1)
    s=np.ascontiguousarray(st,dtype=np.int32)
    coef=np.zeros((1,3,N+1,fmt.width),np.int32); status=np.zeros(1,np.int32)
    rc=plan.lib.mpt_compute_jet(plan.h,_p(s),_p(coef),_p(status))
    buf=(ctypes.c_longlong*4096)()
    plan.lib.mpt_debug_read(buf,4096)
    d=list(buf)
    print('ucol',d[:16]); print('U',d[100:107]); print('CT',d[200:207]); print('info',d[300:308])
    for u in range(12): print('unit',u,d[400+u*64:400+u*64+16],'car',d[1400+u*8:1400+u*8+3])
