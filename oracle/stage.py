"""Per-stage ACOPF oracle (numpy + scipy.sparse) -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/opfkit/acopf.py` so that, on the same host, every output
is bit-identical to the reference:

* packing (acopf.py:77-149): active-bus slots, live generators/branches,
  per-unit bus data, CPython-complex branch admittances (network.py:215-229);
* COO patterns (acopf.py:153-195): the *order* of COO terms fixes scipy's
  duplicate-summation order, so it is reproduced exactly;
* first-order flow quantities (acopf.py:230-250), injections (:252-264),
  objective/gradient (:266-275), constraints (:277-288), Jacobian
  (:290-311), flow Hessians (:313-329) and the Lagrangian Hessian (:331-373),
  each with the reference's left-to-right association;
* bounds, start point and layout maps (acopf.py:197-221, :376-410).

Arithmetic dependencies (not vendored by the reference): numpy float64
sin/cos (glibc libm on this image), ``np.add.at`` (sequential), ``np.sum``
(pairwise), scipy ``coo_matrix.tocsr`` (counting sort by row, per-row
``std::sort`` on column, left-to-right duplicate sums).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

REF, ISOLATED = 3, 4

# the 10 unique (row-axis, col-axis) pairs of a branch's 4x4 Hessian block
# over (theta_f, theta_t, vm_f, vm_t), acopf.py:48-49
POSITIONS = ((0, 0), (0, 1), (0, 2), (0, 3), (1, 1), (1, 2), (1, 3),
             (2, 2), (2, 3), (3, 3))


def admittances(br):
    """Python-complex pi-model admittances, network.py:215-229."""
    ser = 1.0 / complex(br.r, br.x)
    sh = complex(0.0, br.b / 2.0)
    mag = br.ratio if br.ratio != 0.0 else 1.0
    import math
    tap = mag * complex(math.cos(br.angle), math.sin(br.angle))
    return ((ser + sh) / (tap * tap.conjugate()), -ser / tap.conjugate(),
            -ser / tap, ser + sh)


class StageOracle:
    """One NetworkCase packed into arrays with reference-exact callbacks."""

    def __init__(self, case):
        base = case.base_mva
        self.base = base
        pos = {b.id: k for k, b in enumerate(case.buses)}
        self.active = [k for k, b in enumerate(case.buses) if b.btype != ISOLATED]
        slot = {p: s for s, p in enumerate(self.active)}
        self.slot = slot
        nb = len(self.active)
        self.live_gens = [j for j, g in enumerate(case.gens) if g.status != 0]
        self.live_branches = []
        for k, br in enumerate(case.branches):
            if br.status == 0:
                continue
            if pos[br.fbus] not in slot or pos[br.tbus] not in slot:
                raise ValueError("in-service branch touches an isolated bus")
            self.live_branches.append(k)
        ng, nbr = len(self.live_gens), len(self.live_branches)
        self.nb, self.ng, self.nbr = nb, ng, nbr
        self.n = 2 * nb + 2 * ng
        self.pg0, self.qg0 = 2 * nb, 2 * nb + ng

        bl = [case.buses[p] for p in self.active]
        self.pd = np.array([b.pd for b in bl]) / base
        self.qd = np.array([b.qd for b in bl]) / base
        self.gs = np.array([b.gs for b in bl]) / base
        self.bs = np.array([b.bs for b in bl]) / base

        brs = [case.branches[k] for k in self.live_branches]
        self.f = np.array([slot[pos[b.fbus]] for b in brs], dtype=np.intp)
        self.t = np.array([slot[pos[b.tbus]] for b in brs], dtype=np.intp)
        ys = [admittances(b) for b in brs]
        # (gff, bff, gft, bft, gtf, btf, gtt, btt)
        self.y = [np.array([c[i // 2].imag if i % 2 else c[i // 2].real for c in ys])
                  for i in range(8)]
        self.rated = np.array([i for i, b in enumerate(brs) if b.rate_a > 0.0], dtype=np.intp)
        self.nr = len(self.rated)
        self.smax2 = np.array([(brs[i].rate_a / base) ** 2 for i in self.rated])

        gl = [case.gens[j] for j in self.live_gens]
        self.gbus = np.array([slot[pos[g.bus]] for g in gl], dtype=np.intp)
        self.ca = np.array([g.cost.c2 for g in gl]) * base * base
        self.cb = np.array([g.cost.c1 for g in gl]) * base
        self.cc = np.array([g.cost.c0 for g in gl])

        self.m_eq = 2 * nb
        self.m_ineq = 2 * self.nr
        self._coo()
        self._bounds(case)

    # -- structure ----------------------------------------------------------

    def _coo(self):
        nb, ng, nr = self.nb, self.ng, self.nr
        f, t = self.f, self.t
        axes = (f, t, f + nb, t + nb)                 # VA_f, VA_t, VM_f, VM_t
        quad = np.stack(axes, axis=1).ravel()          # per branch, 4 columns
        brow = (f, t, f + nb, t + nb)                  # P_f, P_t, Q_f, Q_t rows
        rows = [np.repeat(r, 4) for r in brow]
        cols = [quad] * 4
        rows += [np.arange(nb), np.arange(nb) + nb, self.gbus, self.gbus + nb]
        cols += [np.arange(nb) + nb, np.arange(nb) + nb,
                 np.arange(ng) + self.pg0, np.arange(ng) + self.qg0]
        if nr:
            srow = 2 * nb + 2 * np.arange(nr)
            rq = np.stack([a[self.rated] for a in axes], axis=1).ravel()
            rows += [np.repeat(srow, 4), np.repeat(srow + 1, 4)]
            cols += [rq, rq]
        self.jr = np.concatenate(rows)
        self.jc = np.concatenate(cols)
        hr, hc = [], []
        for a, b in POSITIONS:
            hr.append(axes[a])
            hc.append(axes[b])
            if a != b:
                hr.append(axes[b])
                hc.append(axes[a])
        hr += [np.arange(nb) + nb, np.arange(ng) + self.pg0]
        hc += [np.arange(nb) + nb, np.arange(ng) + self.pg0]
        self.hr = np.concatenate(hr)
        self.hc = np.concatenate(hc)

    def _bounds(self, case):
        nb, n = self.nb, self.n
        self.xl = np.full(n, -np.inf)
        self.xu = np.full(n, np.inf)
        self.x0 = np.zeros(n)
        self.ref_positions = []
        for s, p in enumerate(self.active):
            b = case.buses[p]
            self.x0[s] = b.va
            self.xl[nb + s], self.xu[nb + s] = b.vmin, b.vmax
            self.x0[nb + s] = min(max(b.vm, b.vmin), b.vmax)
            if b.btype == REF:
                self.xl[s] = self.xu[s] = b.va
                self.ref_positions.append(p)
        for j, gp in enumerate(self.live_gens):
            g = case.gens[gp]
            base = self.base
            self.xl[self.pg0 + j], self.xu[self.pg0 + j] = g.pmin / base, g.pmax / base
            self.x0[self.pg0 + j] = 0.5 * (g.pmin + g.pmax) / base
            self.xl[self.qg0 + j], self.xu[self.qg0 + j] = g.qmin / base, g.qmax / base
            self.x0[self.qg0 + j] = 0.5 * (g.qmin + g.qmax) / base
        self.gl = np.full(self.m_ineq, -np.inf)
        self.gu = np.repeat(self.smax2, 2) if self.nr else np.zeros(0)

    # -- evaluation ---------------------------------------------------------

    def _flows(self, x):
        """Flows, partials and the trig intermediates (acopf.py:230-250)."""
        nb = self.nb
        va, vm = x[:nb], x[nb:2 * nb]
        gff, bff, gft, bft, gtf, btf, gtt, btt = self.y
        vf, vt = vm[self.f], vm[self.t]
        ang = va[self.f] - va[self.t]
        c, s = np.cos(ang), np.sin(ang)
        u = gft * c + bft * s
        w = gft * s - bft * c
        u2 = gtf * c - btf * s
        w2 = -(gtf * s + btf * c)
        vv = vf * vt
        q = dict(u=u, w=w, u2=u2, w2=w2, vf=vf, vt=vt, vv=vv)
        q["pf"] = gff * vf * vf + vv * u
        q["qf"] = -bff * vf * vf + vv * w
        q["pt"] = gtt * vt * vt + vv * u2
        q["qt"] = -btt * vt * vt + vv * w2
        q["gpf"] = (-vv * w, vv * w, 2 * gff * vf + vt * u, vf * u)
        q["gqf"] = (vv * u, -vv * u, -2 * bff * vf + vt * w, vf * w)
        q["gpt"] = (vv * w2, -vv * w2, vt * u2, 2 * gtt * vt + vf * u2)
        q["gqt"] = (-vv * u2, vv * u2, vt * w2, -2 * btt * vt + vf * w2)
        return q

    def objective(self, x):
        pg = x[self.pg0:self.pg0 + self.ng]
        return float(np.sum((self.ca * pg + self.cb) * pg + self.cc))

    def gradient(self, x):
        g = np.zeros(self.n)
        pg = x[self.pg0:self.pg0 + self.ng]
        g[self.pg0:self.pg0 + self.ng] = 2 * self.ca * pg + self.cb
        return g

    def constraints(self, x):
        nb, ng = self.nb, self.ng
        vm = x[nb:2 * nb]
        q = self._flows(x)
        p = np.zeros(nb)
        r = np.zeros(nb)
        np.add.at(p, self.f, q["pf"])
        np.add.at(p, self.t, q["pt"])
        np.add.at(r, self.f, q["qf"])
        np.add.at(r, self.t, q["qt"])
        p += self.gs * vm * vm
        r -= self.bs * vm * vm
        cp = -(self.pd + p)
        cq = -(self.qd + r)
        np.add.at(cp, self.gbus, x[self.pg0:self.pg0 + ng])
        np.add.at(cq, self.gbus, x[self.qg0:self.qg0 + ng])
        lim = np.empty(self.m_ineq)
        k = self.rated
        lim[0::2] = q["pf"][k] ** 2 + q["qf"][k] ** 2
        lim[1::2] = q["pt"][k] ** 2 + q["qt"][k] ** 2
        return np.concatenate([cp, cq, lim])

    def jacobian_coo_values(self, x):
        nb = self.nb
        vm = x[nb:2 * nb]
        q = self._flows(x)
        bal = np.concatenate([np.stack(q[key], axis=1).ravel()
                              for key in ("gpf", "gpt", "gqf", "gqt")])
        vals = [-bal, -2 * self.gs * vm, 2 * self.bs * vm,
                np.ones(self.ng), np.ones(self.ng)]
        if self.nr:
            k = self.rated
            for flow in (("pf", "gpf", "qf", "gqf"), ("pt", "gpt", "qt", "gqt")):
                a, ga, b, gb = flow
                d = 0
                d = d + 2 * q[a][k, None] * np.stack(q[ga], axis=1)[k]
                d = d + 2 * q[b][k, None] * np.stack(q[gb], axis=1)[k]
                vals.append(d.ravel())
        return np.concatenate(vals)

    def jacobian(self, x):
        return sp.coo_matrix((self.jacobian_coo_values(x), (self.jr, self.jc)),
                             shape=(self.m_eq + self.m_ineq, self.n)).tocsr()

    def hessian_coo_values(self, x, obj_factor, mult):
        nb = self.nb
        q = self._flows(x)
        u, w, u2, w2 = q["u"], q["w"], q["u2"], q["w2"]
        vf, vt, vv = q["vf"], q["vt"], q["vv"]
        z = np.zeros(self.nbr)
        gff, bff, _, _, _, _, gtt, btt = self.y
        g2f, b2f, g2t, b2t = 2 * gff, 2 * bff, 2 * gtt, 2 * btt
        # second derivatives of Pf, Qf, Pt, Qt per POSITIONS entry (acopf.py:321-328)
        hpf = (-vv * u, vv * u, -vt * w, -vf * w, -vv * u, vt * w, vf * w, g2f, u, z)
        hqf = (-vv * w, vv * w, vt * u, vf * u, -vv * w, -vt * u, -vf * u, -b2f, w, z)
        hpt = (-vv * u2, vv * u2, vt * w2, vf * w2, -vv * u2, -vt * w2, -vf * w2, z, u2, g2t)
        hqt = (-vv * w2, vv * w2, -vt * u2, -vf * u2, -vv * w2, vt * u2, vf * u2, z, w2, -b2t)
        lpf, lpt = -mult[self.f], -mult[self.t]
        lqf, lqt = -mult[self.f + nb], -mult[self.t + nb]
        sf = np.zeros(self.nbr)
        st = np.zeros(self.nbr)
        if self.nr:
            ridx = 2 * np.arange(self.nr) + self.m_eq
            sf[self.rated] = mult[ridx]
            st[self.rated] = mult[ridx + 1]
        cpf = lpf + 2 * sf * q["pf"]
        cqf = lqf + 2 * sf * q["qf"]
        cpt = lpt + 2 * st * q["pt"]
        cqt = lqt + 2 * st * q["qt"]
        gpf, gqf, gpt, gqt = q["gpf"], q["gqf"], q["gpt"], q["gqt"]
        out = []
        for i, (a, b) in enumerate(POSITIONS):
            v = (cpf * hpf[i] + cqf * hqf[i] + cpt * hpt[i] + cqt * hqt[i]
                 + 2 * sf * (gpf[a] * gpf[b] + gqf[a] * gqf[b])
                 + 2 * st * (gpt[a] * gpt[b] + gqt[a] * gqt[b]))
            out.append(v)
            if a != b:
                out.append(v)
        lp, lq = -mult[:nb], -mult[nb:2 * nb]
        out.append(2 * (lp * self.gs - lq * self.bs))
        d = np.full(self.ng, 0.0)
        d += 2 * obj_factor * self.ca
        out.append(d)
        return np.concatenate(out)

    def lagrangian_hessian(self, x, obj_factor, mult):
        return sp.coo_matrix((self.hessian_coo_values(x, obj_factor, mult),
                              (self.hr, self.hc)), shape=(self.n, self.n)).tocsr()

    # -- layout (acopf.py:376-389) -------------------------------------------

    def layout_maps(self):
        nb = self.nb
        return dict(
            va={p: self.slot[p] for p in self.active},
            vm={p: self.slot[p] + nb for p in self.active},
            pg={gp: self.pg0 + j for j, gp in enumerate(self.live_gens)},
            qg={gp: self.qg0 + j for j, gp in enumerate(self.live_gens)},
            p_row={p: self.slot[p] for p in self.active},
            q_row={p: self.slot[p] + nb for p in self.active},
            sf_row={self.live_branches[i]: 2 * k for k, i in enumerate(self.rated)},
            st_row={self.live_branches[i]: 2 * k + 1 for k, i in enumerate(self.rated)},
            ref_buses=tuple(self.ref_positions))
