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
    d=np.array(list(buf)).reshape(256,16)
    print(plan.info(), f'{ms:.3f} ms/step, {ms*1.965e6/N:.0f} cycles/order')
    names=['A-bulk','A-lin+red','bar1','B-read','B-norm','C-prod','bar2','D-norm','D-pub']
    for lo,hi in ((0,50),(50,150),(150,255)):
        rows=[r for r in range(lo,hi) if d[r,0]>0 and d[r,9]>0]
        if not rows: continue
        segs=[np.mean([d[r,e+1]-d[r,e] for r in rows]) for e in range(9)]
        print(f' orders {lo}-{hi}: ' + '  '.join(f'{n}={s:.0f}' for n,s in zip(names,segs)) + f'  total={np.mean([d[r,9]-d[r,0] for r in rows]):.0f}')
