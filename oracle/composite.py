"""Composite (multi-stage) ACOPF oracle -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/opfkit/composer.py`:

* stage lattice, scenario-major / contingency / period order
  (composer.py:327-388) and the flat stochastic variant (:435-457);
* coupling rows: ramp (:157-162), corrective box / preventive pins
  (:164-188), scenario box (:190-197); pins after all stage equalities,
  boxes after all stage inequalities (:217-242);
* composite callbacks (:256-311): weighted objective summed left to right,
  weighted gradient slices, stage constraint blocks plus ``child - base``
  coupling values, Jacobian/Hessian stage blocks shifted into place and
  re-canonicalised by scipy.

The stage transforms it needs (network.py:312-357) are restated locally so
the checker shares no code with the product.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import scipy.sparse as sp

from .stage import REF, StageOracle


def _gen_at(case, bus, ordinal):
    hits = [k for k, g in enumerate(case.gens) if g.bus == bus]
    return hits[ordinal - 1]


def _apply_ctg(case, ctg):
    gens, brs = list(case.gens), list(case.branches)
    for o in ctg.outages:
        if o.kind == "GEN":
            k = _gen_at(case, o.bus, o.ordinal)
            gens[k] = replace(gens[k], status=0)
        else:
            hits = [k for k, b in enumerate(case.branches)
                    if b.fbus == o.bus and b.tbus == o.tbus]
            k = hits[o.ordinal - 1]
            brs[k] = replace(brs[k], status=0)
    return replace(case, gens=tuple(gens), branches=tuple(brs))


def _apply_scen(case, scen):
    gens = list(case.gens)
    for (bus, ordinal), mw in scen.wind_targets:
        k = _gen_at(case, bus, ordinal)
        gens[k] = replace(gens[k], pmax=mw, pmin=0.0)
    return replace(case, gens=tuple(gens))


class CompositeOracle:
    """Stages + coupling rows + composite callbacks, reference-exact."""

    def __init__(self):
        self.cases, self.weights, self.meta, self.pending = [], [], [], []

    # -- lattice ------------------------------------------------------------

    def _add(self, case, weight, meta):
        self.cases.append(case)
        self.weights.append(weight)
        self.meta.append(meta)
        return len(self.cases) - 1

    @staticmethod
    def _both_live(a, b):
        return [i for i, (ga, gb) in enumerate(zip(a.gens, b.gens))
                if ga.status != 0 and gb.status != 0]

    def _ramp(self, child, base, dt):
        bc = self.cases[base]
        for g in self._both_live(self.cases[child], bc):
            self.pending.append(("Ramp", child, base, g, None,
                                 bc.gens[g].ramp_30 * (dt / 30.0) / bc.base_mva, False))

    def _mode(self, child, base, mode, kind="ContingencyBox", scale=None):
        bc = self.cases[base]
        live = self._both_live(self.cases[child], bc)
        if mode.kind == "corrective":
            s = mode.contingency_scale if scale is None else scale
            for g in live:
                self.pending.append((kind, child, base, g, None,
                                     bc.gens[g].ramp_30 * s / bc.base_mva, False))
            return
        pos = {b.id: k for k, b in enumerate(bc.buses)}
        for g in live:
            if bc.buses[pos[bc.gens[g].bus]].btype == REF:
                continue
            self.pending.append(("PreventivePin", child, base, g, None, 0.0, True))
        if mode.pin_voltages:
            for bp in sorted({pos[bc.gens[g].bus] for g in live}):
                self.pending.append(("PreventivePin", child, base, None, bp, 0.0, True))

    def _scen(self, child, base, mode):
        bc = self.cases[base]
        for g in self._both_live(self.cases[child], bc):
            self.pending.append(("ScenarioBox", child, base, g, None,
                                 bc.gens[g].ramp_30 * mode.scenario_scale / bc.base_mva,
                                 False))

    @staticmethod
    def _scenario_order(scens):
        if scens is None:
            return [(None, 1.0)]
        items = list(scens.scenarios)
        tot = sum(s.weight for s in items)
        b = min(range(len(items)), key=lambda i: (-items[i].weight, items[i].id))
        rest = sorted((s for i, s in enumerate(items) if i != b), key=lambda s: s.id)
        return [(s, s.weight / tot) for s in [items[b]] + rest]

    @classmethod
    def general(cls, scens, ctgs, periods, mode, dt, assemble=True):
        """composer.py:327-388.  assemble=False stops after the lattice (cases, weights and
        the pending coupling rows), without building the stage oracles."""
        o = cls()
        ctg_list = [None] + (list(ctgs.by_id()) if ctgs is not None else [])
        idx = {}
        so = cls._scenario_order(scens)
        for si, (sc, w) in enumerate(so):
            sp_ = [_apply_scen(p, sc) if sc else p for p in periods]
            for ci, c in enumerate(ctg_list):
                cp = [_apply_ctg(p, c) for p in sp_] if c else sp_
                for t in range(len(periods)):
                    idx[(si, ci, t)] = o._add(cp[t], w, (sc, c, t))
        for si in range(len(so)):
            for ci in range(len(ctg_list)):
                for t in range(1, len(periods)):
                    o._ramp(idx[(si, ci, t)], idx[(si, ci, t - 1)], dt)
            for ci in range(1, len(ctg_list)):
                o._mode(idx[(si, ci, 0)], idx[(si, 0, 0)], mode)
            if si > 0:
                o._scen(idx[(si, 0, 0)], idx[(0, 0, 0)], mode)
        if assemble:
            o._assemble()
        return o

    @classmethod
    def sopf_flat(cls, base, scens, ctgs, mode):
        o = cls()
        ctg_list = [None] + (list(ctgs.by_id()) if ctgs is not None else [])
        ids = []
        for sc, w in cls._scenario_order(scens):
            sc_case = _apply_scen(base, sc) if sc else base
            for ci, c in enumerate(ctg_list):
                k = o._add(_apply_ctg(sc_case, c) if c else sc_case, w, (sc, c, 0))
                ids.append((ci, k))
        for ci, k in ids:
            if k == 0:
                continue
            o._mode(k, 0, mode, kind="ContingencyBox" if ci > 0 else "ScenarioBox",
                    scale=mode.contingency_scale if ci > 0 else mode.scenario_scale)
        o._assemble()
        return o

    # -- assembly (composer.py:199-324) -----------------------------------------

    def _assemble(self):
        st = [StageOracle(c) for c in self.cases]
        self.stage = st
        ns = len(st)
        self.var_off = np.concatenate([[0], np.cumsum([s.n for s in st])[:-1]]).astype(int)
        self.eq_off = np.concatenate([[0], np.cumsum([s.m_eq for s in st])[:-1]]).astype(int)
        self.ineq_off = np.concatenate([[0], np.cumsum([s.m_ineq for s in st])[:-1]]).astype(int)
        nv = sum(s.n for s in st)
        me_st = sum(s.m_eq for s in st)
        mi_st = sum(s.m_ineq for s in st)
        pins = [r for r in self.pending if r[6]]
        boxes = [r for r in self.pending if not r[6]]
        self.n = nv
        self.m_eq = me_st + len(pins)
        self.m_ineq = mi_st + len(boxes)
        lay = [s.layout_maps() for s in st]
        self.layouts = lay

        def var(r, k):
            m = lay[k]["pg"][r[3]] if r[3] is not None else lay[k]["vm"][r[4]]
            return int(self.var_off[k] + m)

        self.coupling = []
        cr, cc, cv = [], [], []
        for i, r in enumerate(pins + boxes):
            row = me_st + i if r[6] else self.m_eq + mi_st + (i - len(pins))
            self.coupling.append(dict(kind=r[0], stage_a=r[1], stage_b=r[2], gen=r[3],
                                      bus=r[4], bound=r[5], row=row, is_equality=r[6]))
            cr += [row, row]
            cc += [var(r, r[1]), var(r, r[2])]
            cv += [1.0, -1.0]
        self.c_rows = np.asarray(cr, dtype=int)
        self.c_cols = np.asarray(cc, dtype=int)
        self.c_vals = np.asarray(cv)
        self.w = np.asarray(self.weights)
        self.xl = np.concatenate([s.xl for s in st])
        self.xu = np.concatenate([s.xu for s in st])
        self.x0 = np.concatenate([s.x0 for s in st])
        self.gl = np.concatenate([s.gl for s in st] + [np.array([-r[5] for r in boxes])])
        self.gu = np.concatenate([s.gu for s in st] + [np.array([r[5] for r in boxes])])
        self.slices = [(int(self.var_off[k]), int(self.var_off[k]) + st[k].n) for k in range(ns)]

    # -- callbacks --------------------------------------------------------------

    def objective(self, x):
        return float(sum(self.w[k] * self.stage[k].objective(x[a:b])
                         for k, (a, b) in enumerate(self.slices)))

    def gradient(self, x):
        g = np.zeros(self.n)
        for k, (a, b) in enumerate(self.slices):
            g[a:b] = self.w[k] * self.stage[k].gradient(x[a:b])
        return g

    def constraints(self, x):
        out = np.zeros(self.m_eq + self.m_ineq)
        for k, (a, b) in enumerate(self.slices):
            s = self.stage[k]
            c = s.constraints(x[a:b])
            out[self.eq_off[k]:self.eq_off[k] + s.m_eq] = c[:s.m_eq]
            lo = self.m_eq + self.ineq_off[k]
            out[lo:lo + s.m_ineq] = c[s.m_eq:]
        if len(self.coupling):
            out[self.c_rows[0::2]] = x[self.c_cols[0::2]] - x[self.c_cols[1::2]]
        return out

    def jacobian(self, x):
        rows, cols, vals = [self.c_rows], [self.c_cols], [self.c_vals]
        for k, (a, b) in enumerate(self.slices):
            s = self.stage[k]
            j = s.jacobian(x[a:b]).tocoo()
            eq = j.row < s.m_eq
            rows.append(np.where(eq, self.eq_off[k] + j.row,
                                 self.m_eq + self.ineq_off[k] + (j.row - s.m_eq)))
            cols.append(a + j.col)
            vals.append(j.data)
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.m_eq + self.m_ineq, self.n))

    def lagrangian_hessian(self, x, obj_factor, mult):
        rows, cols, vals = [], [], []
        for k, (a, b) in enumerate(self.slices):
            s = self.stage[k]
            lo = self.m_eq + self.ineq_off[k]
            mk = np.concatenate([mult[self.eq_off[k]:self.eq_off[k] + s.m_eq],
                                 mult[lo:lo + s.m_ineq]])
            h = s.lagrangian_hessian(x[a:b], obj_factor * self.w[k], mk).tocoo()
            rows.append(a + h.row)
            cols.append(a + h.col)
            vals.append(h.data)
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.n, self.n))
