"""Solution extraction oracle -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/opfkit/acopf.py:448-546` (``_branch_flows_mw``,
``extract_solution``, ``solution_from_case``, ``residuals_at``) on top of
:class:`oracle.stage.StageOracle`'s flow quantities, returning plain dicts
of arrays.  Checked against fixtures made by the reference itself
(tests/golden/make_golden.py ``solutions``).
"""

from __future__ import annotations

import numpy as np

from .stage import StageOracle


def _stage_point(o: StageOracle, va_all, vm_all):
    x = np.zeros(o.n)
    x[:o.nb] = np.array([va_all[p] for p in o.active])
    x[o.nb:2 * o.nb] = np.array([vm_all[p] for p in o.active])
    return x


def branch_flows_mw(case, va_all, vm_all):
    """acopf.py:448-464."""
    o = StageOracle(case)
    nbrs = len(case.branches)
    out = {k: np.zeros(nbrs) for k in ("pf", "qf", "pt", "qt")}
    if o.nbr:
        q = o._flows(_stage_point(o, va_all, vm_all))
        live = np.array(o.live_branches, dtype=np.intp)
        for k in out:
            out[k][live] = q[k] * o.base
    return out


def _cost(case, gens, pg):
    total = 0
    for j in gens:
        c = case.gens[j].cost
        total = total + ((c.c2 * pg[j] + c.c1) * pg[j] + c.c0)
    return float(total)


def extract(case, layout, x):
    """acopf.py:467-488 (layout maps of the stage)."""
    vm = np.zeros(len(case.buses))
    va = np.zeros(len(case.buses))
    for pos in layout.va:
        va[pos] = x[layout.va[pos]]
        vm[pos] = x[layout.vm[pos]]
    pg = np.zeros(len(case.gens))
    qg = np.zeros(len(case.gens))
    for g, idx in layout.pg.items():
        pg[g] = x[idx] * case.base_mva
        qg[g] = x[layout.qg[g]] * case.base_mva
    sol = dict(vm=vm, va=va, pg=pg, qg=qg, **branch_flows_mw(case, va, vm))
    sol["objective"] = _cost(case, list(layout.pg), pg)
    return sol


def from_case(case):
    """acopf.py:504-515."""
    vm = np.array([b.vm for b in case.buses], dtype=np.float64)
    va = np.array([b.va for b in case.buses], dtype=np.float64)
    pg = np.array([g.pg if g.status else 0.0 for g in case.gens], dtype=np.float64)
    qg = np.array([g.qg if g.status else 0.0 for g in case.gens], dtype=np.float64)
    sol = dict(vm=vm, va=va, pg=pg, qg=qg, **branch_flows_mw(case, va, vm))
    sol["objective"] = _cost(case, [j for j, g in enumerate(case.gens) if g.status], pg)
    return sol


def residuals(case, va, vm, pg, qg):
    """acopf.py:518-546: generation - load - network injection, MW / MVAr."""
    o = StageOracle(case)
    x = _stage_point(o, va, vm)
    q = o._flows(x)
    vms = x[o.nb:2 * o.nb]
    p = np.zeros(o.nb)
    r = np.zeros(o.nb)
    np.add.at(p, o.f, q["pf"])
    np.add.at(p, o.t, q["pt"])
    np.add.at(r, o.f, q["qf"])
    np.add.at(r, o.t, q["qt"])
    p += o.gs * vms * vms
    r -= o.bs * vms * vms
    dp_s = -p * o.base
    dq_s = -r * o.base
    for k, pos in enumerate(o.active):
        dp_s[k] -= case.buses[pos].pd
        dq_s[k] -= case.buses[pos].qd
    pos_of = {b.id: k for k, b in enumerate(case.buses)}
    for j in o.live_gens:
        k = o.slot[pos_of[case.gens[j].bus]]
        dp_s[k] += pg[j]
        dq_s[k] += qg[j]
    dp = np.zeros(len(case.buses))
    dq = np.zeros(len(case.buses))
    for k, pos in enumerate(o.active):
        dp[pos] = dp_s[k]
        dq[pos] = dq_s[k]
    return dp, dq
