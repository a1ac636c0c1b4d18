"""Device KKT assembly + Bunch-Kaufman factorisation (kkt.py) against the reference IPM's
dense Newton matrix (ipm.py:463-501, _BunchKaufman ipm.py:173-220), restated in numpy on
the oracle's Jacobian / Hessian."""

import time

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.linalg import lapack

import common as C
import paper_2203_10587_b200 as pkg
from golden.make_golden import STAGE_SPECS, stage_case
from paper_2203_10587_b200 import _lib as L
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.kkt import DeviceKKT, _inertia
from oracle.stage import StageOracle

pytestmark = pytest.mark.gpu


def _reference_k(o, x, mult, s_f, s_c, free, dx, ds, reg, delta):
    """The reference's K (ipm.py:463-477 and _BunchKaufman.__init__), both triangles."""
    me, mi = o.m_eq, o.m_ineq
    hess = o.lagrangian_hessian(x, 1.0 * s_f, mult * s_c)[free][:, free]
    jac = o.jacobian(x)[:, free]
    je = sp.diags(s_c[:me]) @ jac[:me]
    ji = sp.diags(s_c[me:]) @ jac[me:]
    hfull = hess + sp.diags(dx, format="csr")
    if mi:
        hfull = hfull + ji.T @ sp.diags(ds) @ ji
    hfull = np.asarray(hfull.todense())
    hfull = 0.5 * (hfull + hfull.T)
    n = len(free)
    k = np.zeros((n + me, n + me))
    k[:n, :n] = hfull
    k[n:, :n] = je.toarray()
    k[:n, n:] = je.toarray().T
    k[np.arange(n), np.arange(n)] += reg
    k[np.arange(n, n + me), np.arange(n, n + me)] -= delta
    return k


def _bk_inertia(k):
    ldu, ipiv, info = lapack.dsytrf(k, lower=1)
    d = np.diag(ldu)
    e = np.diag(ldu, -1)
    return _inertia(d, e, np.where(ipiv >= 0, ipiv + 1, ipiv)), info


@pytest.mark.parametrize("name", ["stage_ring9", "stage_feat30", "stage_feat200"])
def test_device_kkt_matches_reference(name):
    import torch
    case = stage_case(STAGE_SPECS[name])
    p, _ = pkg.build_acopf(case)
    o = StageOracle(case)
    rng = np.random.default_rng(7)
    kinds = syn.variable_kinds([(o.nb, o.ng)])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 21)
    free = np.flatnonzero(p.xl != p.xu)
    s_f = 0.37
    s_c = rng.uniform(0.2, 1.0, p.m_eq + p.m_ineq)
    dx = rng.uniform(0.0, 3.0, len(free))
    ds = rng.uniform(0.0, 2.0, p.m_ineq)
    kk = DeviceKKT(p)
    ev = p.evaluator
    out = ev.eval_device(torch.from_numpy(x).cuda(), torch.from_numpy(mult * s_c).cuda(), s_f, L.JAC | L.HESS)
    for reg, delta in ((0.0, 0.0), (1e-4, 1e-8)):
        K = kk.assemble(out["jac"], out["hess"], dx, ds, reg, delta, sc=s_c)
        Kref = _reference_k(o, x, mult, s_f, s_c, free, dx, ds, reg, delta)
        Kd = K.cpu().numpy()
        scale = max(1.0, float(np.abs(Kref).max()))
        assert np.allclose(Kd, Kref, rtol=1e-12, atol=1e-14 * scale), float(np.abs(Kd - Kref).max())
        LD, piv, inertia, info = kk.factor(K)
        ref_inertia, _ = _bk_inertia(Kref)
        assert inertia == ref_inertia
        b = rng.standard_normal(kk.dim)
        sol = kk.solve(LD, piv, b).cpu().numpy()
        ref = np.linalg.solve(Kref, b)
        assert np.linalg.norm(sol - ref) <= 1e-8 * max(1.0, np.linalg.norm(ref))
    C.record(f"kkt:{name}", dim=kk.dim, nf=kk.nf, me=kk.me)


@pytest.mark.slow
def test_device_kkt_config1_solve():
    """The config-1 Newton system (n + m_eq = 45 k; the dense reference cannot factor it in a
    usable time): assemble, factor, solve on the device; residual of the solve."""
    import torch
    case = syn.config_case(1)
    p, _ = pkg.build_acopf(case)
    kinds = syn.variable_kinds([(len(p.x0) // 2 - 1250, 2500)]) if False else None
    o_nb = p.evaluator.plans[0].topo.nb
    kinds = syn.variable_kinds([(o_nb, p.evaluator.plans[0].topo.ng)])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 5)
    rng = np.random.default_rng(3)
    kk = DeviceKKT(p)
    ev = p.evaluator
    out = ev.eval_device(torch.from_numpy(x).cuda(), torch.from_numpy(mult).cuda(), 1.0, L.JAC | L.HESS)
    dx = rng.uniform(1.0, 3.0, kk.nf)
    ds = rng.uniform(0.0, 2.0, p.m_ineq)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    K = kk.assemble(out["jac"], out["hess"], dx, ds, 1e-6, 1e-8)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    LD, piv, inertia, info = kk.factor(K)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    b = torch.as_tensor(rng.standard_normal(kk.dim), device="cuda")
    sol = kk.solve(LD, piv, b)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    K = kk.assemble(out["jac"], out["hess"], dx, ds, 1e-6, 1e-8, out=K)
    res = float(torch.linalg.norm(K @ sol - b) / torch.linalg.norm(b))
    C.record("kkt:cfg1", dim=kk.dim, assemble_s=t1 - t0, factor_s=t2 - t1, solve_s=t3 - t2,
             inertia=list(inertia), residual=res, info=info)
    assert info == 0 and res < 1e-8, res
