import sys, time, numpy as np
sys.path.insert(0,'.')
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.stage import build_acopf
from oracle.stage import StageOracle
def cmp(name, a, b):
    a=np.asarray(a,float); b=np.asarray(b,float)
    bits=int(np.sum(a.view(np.int64)!=b.view(np.int64)))
    gate=np.abs(a-b) <= 1e-14 + 1e-12*np.abs(b)
    miss=int(np.sum(~gate))
    print(f'  {name}: n={a.size} bitdiff={bits} gate_miss={miss} maxrel={np.max(np.abs(a-b)/np.maximum(np.abs(b),1e-300)) if a.size else 0:.2e}')
    return miss
tot=0
for (nb,nc,ng,feat) in [(9,0,3,False),(30,10,6,True),(200,60,40,True),(2000,600,500,False),(10000,3000,2500,False)]:
    case = syn.make_case(nb,nc,ng,seed=nb, ring=(nb==9), features=feat)
    p, lay = build_acopf(case)
    o = StageOracle(case)
    kinds = syn.variable_kinds([(o.nb,o.ng)])
    print(nb)
    for s in range(2):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq+p.m_ineq, 100+s)
        tot+=cmp('obj',[p.objective(x)],[o.objective(x)])
        tot+=cmp('grad',p.gradient(x),o.gradient(x))
        tot+=cmp('cons',p.constraints(x),o.constraints(x))
        J=p.jacobian(x); Jo=o.jacobian(x)
        assert np.array_equal(J.indptr,Jo.indptr) and np.array_equal(J.indices,Jo.indices)
        tot+=cmp('jac',J.data,Jo.data)
        H=p.lagrangian_hessian(x,1.7,mult); Ho=o.lagrangian_hessian(x,1.7,mult)
        assert np.array_equal(H.indptr,Ho.indptr) and np.array_equal(H.indices,Ho.indices)
        tot+=cmp('hess',H.data,Ho.data)
print('TOTAL gate misses', tot)
