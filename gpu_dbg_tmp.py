import sys, numpy as np
sys.path.insert(0,'.')
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.stage import build_acopf
from oracle.stage import StageOracle
case = syn.make_case(2000,600,500,seed=2000)
p, lay = build_acopf(case)
o = StageOracle(case)
kinds = syn.variable_kinds([(o.nb,o.ng)])
x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq+p.m_ineq, 100)
print('oracle', o.objective(x))
for i in range(4): print('gpu', p.objective(x))
case = syn.make_case(2000,600,500,seed=2000)
p, lay = build_acopf(case)
g=p.gradient(x)
for i in range(2): print('gpu after grad', p.objective(x))
