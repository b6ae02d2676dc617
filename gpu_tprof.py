import sys, os, ctypes, numpy as np
os.environ['MPT_DEBUG']='1'
sys.path.insert(0,'.')
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat
K,N,kern,G=int(sys.argv[1]),int(sys.argv[2]),sys.argv[3],int(sys.argv[4])
P=M.bits_for_digits(K); ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
tab=SystemTables.build(sysm,fmt,N,M.mp_from_decimal('0.01',ctx).as_fraction())
st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in ('-15.8','-17.48','35.64')])
with DevicePlan(tab,fmt,N,1) as plan:
    plan.configure(kern,G); plan.upload(st); plan.run_device(1); ms=plan.last_kernel_ms()
    buf=(ctypes.c_longlong*4096)(); plan.lib.mpt_debug_read(buf,4096)
    d=np.array(list(buf)[:200*16]).reshape(200,16)
    print(plan.info(), f'{ms:.3f} ms/step, {ms*1.965e6/N:.0f} cycles/order')
    names={1:'C0 list+bar',2:'C1 products',3:'C2 assemble',4:'C2 normalize',5:'C3 product',6:'C3 normalize',7:'publish',11:'barrier(wait)'}
    rows=[r for r in range(min(N,200)) if d[r,0]>0]
    def seg(a,b):
        v=[d[r,b]-d[r,a] for r in rows if d[r,a]>0 and d[r,b]>0]
        return np.mean(v) if v else float('nan')
    print(' chain: list', seg(0,1),' C1', seg(1,2),' assemble', seg(2,3),' norm1', seg(3,4),' cprod', seg(4,5), ' norm2', seg(5,6), ' publish', seg(6,7), ' ->barrier-exit', seg(7,11))
    print(' bulk : mac', seg(0,8), ' bar2', seg(8,9), ' reduce+push', seg(9,10), ' ->barrier-exit', seg(10,11))
    print(' total order', seg(0,11))
    for r in (2,50,150):
        if r < len(rows): print(' order',r,' chain->7', d[r,7]-d[r,0], ' bulk->10', d[r,10]-d[r,0], ' exit', d[r,11]-d[r,0])
