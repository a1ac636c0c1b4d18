"""Breakdown of the batch-1 callback latency on the cfg1 network (development aid)."""
import time, statistics, ctypes, sys
sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
from paper_2203_10587_b200 import build_acopf, synthetic as syn, _lib as L

case = syn.config_case(1)
p, _ = build_acopf(case, device=0)
cb = p.objective.__self__
ev = cb.ev
kinds = syn.variable_kinds([(ev.topos[0].nb, ev.topos[0].ng)])
x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 4242)


def med(fn, n=50):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        t = time.perf_counter(); fn(); ts.append(time.perf_counter() - t)
    return 1e3 * statistics.median(ts)


print("objective", med(lambda: p.objective(x)))
print("jacobian", med(lambda: p.jacobian(x)))
print("hessian", med(lambda: p.lagrangian_hessian(x, 1.0, mult)))
print("_eval OBJ", med(lambda: cb._eval(x, None, 1.0, L.OBJ)))
print("_eval JAC", med(lambda: cb._eval(x, None, 1.0, L.JAC)))
print("_eval HESS", med(lambda: cb._eval(x, mult, 1.0, L.HESS)))
print("pinned alloc nnz_j", med(lambda: cb._pinned(ev.nnz_j)))
px = cb._pin_x.numpy()[:ev.n]
print("copyto x", med(lambda: np.copyto(px, x)))
vals = cb._eval(x, None, 1.0, L.JAC)
ip, ind = cb._patterns("J")
print("csr build", med(lambda: sp.csr_matrix((vals, ind.copy(), ip.copy()), shape=(ev.m, ev.n))))
print("index copies", med(lambda: (ind.copy(), ip.copy())))
out = cb._pinned(ev.nnz_j)
def raw(what, size, o):
    ptrs = [None] * 5
    ptrs[{L.OBJ: 0, L.GRAD: 1, L.CONS: 2, L.JAC: 3, L.HESS: 4}[what]] = o
    v = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
    nn = lambda t: 0 if t is None else size
    L.check(L.lib().acopf_batch_eval_host(ev._h, ctypes.c_void_p(cb._pin_x.data_ptr()), ev.n, 1.0, None, 0, int(what),
            v(ptrs[0]), nn(ptrs[0]), v(ptrs[1]), nn(ptrs[1]), v(ptrs[2]), nn(ptrs[2]), v(ptrs[3]), nn(ptrs[3]),
            v(ptrs[4]), nn(ptrs[4]), None))
o1 = cb._pinned(ev.n_obj)
print("raw OBJ", med(lambda: raw(L.OBJ, ev.n_obj, o1)))
print("raw JAC", med(lambda: raw(L.JAC, ev.nnz_j, out)))
import torch
s = torch.cuda.Stream()
print("n", ev.n, "m", ev.m, "nnz_j", ev.nnz_j, "nnz_h", ev.nnz_h)
