import json, time, sys
import numpy as np
sys.path.insert(0,'.')
from oracle import fix as FX
import paper_1908_09301_b200 as M
from paper_1908_09301_b200.engine import SystemTables, DevicePlan
from paper_1908_09301_b200.fixed import FixedFormat
from fractions import Fraction
def run(P, N, nsteps, stride, tau='0.01', init=('-15.8','-17.48','35.64')):
    ctx=M.PrecisionContext(P); sysm=M.builtin_system('lorenz',ctx); fmt=FixedFormat(P)
    t=M.mp_from_decimal(tau,ctx); tab=SystemTables.build(sysm,fmt,N,t.as_fraction())
    st=fmt.to_digits([M.mp_from_decimal(x,ctx) for x in init])
    # jet check
    cj=FX.compute_jet(tab,fmt.frac_digits,N,st)
    with DevicePlan(tab,fmt,N,1) as plan:
        print('plan info',plan.info(), flush=True)
        gj=plan.compute_jet(st)[0]
        bad=np.argwhere((gj!=cj).any(axis=2))
        print(f'P={P} N={N} jet mismatches:', len(bad), bad[:5].tolist(), flush=True)
        if len(bad):
            m,i=bad[0]; print(' first gpu',gj[m,i][:12].tolist(),'\n first cpu',cj[m,i][:12].tolist())
        t0=time.time(); steps,recs,status=plan.integrate(st,nsteps,0,stride); dt=time.time()-t0
        cs,cr=FX.integrate(tab,fmt.frac_digits,N,P,st,nsteps,0,stride)
        eq=(recs[:,0]==cr).all(axis=(1,2))
        print(f'  integrate {nsteps} steps: wall {dt:.3f}s kernel {plan.last_kernel_ms():.3f}ms status {status.tolist()} records equal: {eq.tolist()}', flush=True)
run(167,40,50,10)
run(256,30,20,5)
run(1661,200,3,1)
run(1661,200,20,10)
