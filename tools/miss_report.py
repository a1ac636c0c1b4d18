"""Report gate misses on sampled full-size config-4 stages with their conditioning."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2203_10587_b200 as pkg
from paper_2203_10587_b200 import synthetic as syn, _lib as L
from paper_2203_10587_b200.types import CouplingMode
from oracle.stage import StageOracle
import common as C

base, scens, ctgs = syn.config4_inputs()
p, imap = pkg.compose_general(scens, ctgs, [base], CouplingMode(), 30.0)
kinds = syn.variable_kinds([(len(l.va), len(l.pg)) for l in imap.layouts])
x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 41)
ev = p.evaluator
out = ev.eval_host(x, mult, 1.0, L.ALL)
ip, ix = ev.pattern("J"); hp, hx = ev.pattern("H")
rep = []
for k in [0, 1, 32, 33, 1023, 500, 777]:
    o = StageOracle(imap.stages[k].case)
    lay = imap.layouts[k]
    a, b = imap.var_offset[k], imap.var_offset[k] + lay.n_vars
    e0, i0 = imap.eq_offset[k], p.m_eq + imap.ineq_offset[k]
    mk = np.concatenate([mult[e0:e0 + lay.n_eq], mult[i0:i0 + lay.n_ineq]])
    xs = x[a:b]
    rows = np.r_[e0:e0 + lay.n_eq, i0:i0 + lay.n_ineq]
    Jd = np.concatenate([out["jac"][ip[r]:ip[r + 1]] for r in rows])
    Hd = out["hess"][hp[a]:hp[b]]
    Jo = o.jacobian(xs); Ho = o.lagrangian_hessian(xs, imap.weights[k], mk)
    # conditioning: sum of |COO terms| per CSR entry, from the oracle's COO values
    import scipy.sparse as sp
    Jabs = sp.coo_matrix((np.abs(o.jacobian_coo_values(xs)), (o.jr, o.jc)), shape=Jo.shape).tocsr()
    Habs = sp.coo_matrix((np.abs(o.hessian_coo_values(xs, imap.weights[k], mk)), (o.hr, o.hc)), shape=Ho.shape).tocsr()
    cs = np.concatenate([out["cons"][e0:e0 + lay.n_eq], out["cons"][i0:i0 + lay.n_ineq]])
    for name, a_, b_, absm in (("J", Jd, Jo.data, Jabs.data), ("H", Hd, Ho.data, Habs.data), ("cons", cs, o.constraints(xs), None)):
        bad = ~(np.abs(a_ - b_) <= 1e-14 + 1e-12 * np.abs(b_))
        for i in np.flatnonzero(bad):
            cond = float(absm[i] / abs(b_[i])) if absm is not None and b_[i] != 0 else None
            rep.append(dict(stage=k, arr=name, idx=int(i), gpu=float(a_[i]), ref=float(b_[i]),
                            rel=float(abs(a_[i] - b_[i]) / max(abs(b_[i]), 1e-300)), cond=cond))
    print(k, "J bitdiff", C.bit_diffs(Jd, Jo.data), "H bitdiff", C.bit_diffs(Hd, Ho.data), "of", len(Jd) + len(Hd), flush=True)
print(json.dumps(rep, indent=1))
