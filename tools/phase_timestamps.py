import sys, os, ctypes, numpy as np
os.environ['MPT_DEBUG']='1'
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat
K,N,kern,G=int(sys.argv[1]),int(sys.argv[2]),sys.argv[3],int(sys.argv[4])
P=M.bits_for_digits(K); ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
with DevicePlan(tab,fmt,N,1) as plan:
    plan.configure(kern,G); plan.upload(st); plan.run_device(1); plan.last_kernel_ms()
    os.environ.pop('MPT_DEBUG')
    plan.run_device(1); ms=plan.last_kernel_ms()
    buf=(ctypes.c_longlong*4096)(); plan.lib.mpt_debug_read(buf,4096)
    d=np.array(list(buf)[:200*16]).reshape(200,16)
    print(plan.info(), f'{ms:.3f} ms/step, {ms*1.965e6/N:.0f} cycles/order')
    rows=[r for r in range(min(N,200)) if d[r,0]>0]
    def seg(a,b,rr=rows):
        v=[d[r,b]-d[r,a] for r in rr if d[r,a]>0 and d[r,b]>0]
        return round(float(np.mean(v))) if v else float('nan')
    for lo,hi in ((0,50),(50,150),(150,200)):
        rr=[r for r in rows if lo<=r<hi]
        print(f' orders {lo}-{hi}: A-prod', seg(0,1,rr),' B-asm', seg(1,2,rr),' C-norm', seg(2,3,rr),' D-cprod', seg(3,4,rr),' E-norm', seg(4,5,rr),' publish', seg(5,6,rr),' barrier', seg(6,7,rr),' | bulk mac', seg(0,8,rr),' push', seg(8,9,rr), ' total', seg(0,7,rr))
