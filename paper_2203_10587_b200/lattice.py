"""``compose_*``: multiperiod / SCOPF / stochastic composites on the B200.

Drop-in for `pkg/src/opfkit/composer.py:391-457` (same signatures and
return types).  The lattice, coupling rows and index maps follow the
reference exactly (composer.py:145-388):

* stages enumerate scenario-major (most probable scenario first, the rest
  by id), then contingency (base, then by id), then period;
* ramp rows chain consecutive periods; contingency rows (corrective box or
  preventive pins, optional VM pins) tie each post-contingency stage's first
  period to its scenario base; scenario boxes tie scenario bases to the
  first scenario's base; pins sit after all stage equalities, boxes after
  all stage inequalities; every row reads child - base.

What changes is how stages are represented: instead of one packed engine per
stage, a stage is (shared packed topology, removed branches, load set,
bound overrides).  Generator outages get their own topology; branch outages
are per-stage removal lists handled by the device planner; loads of a
period are a per-stage load set.  All stages are evaluated by one kernel
launch.  ``CompositeIndexMap.stages``, ``.layouts`` and ``.coupling_rows``
are materialised lazily (they hold a NetworkCase / dicts per element).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import EmptyScenarioSet, InvalidPlan, IslandingDetected, TopologyMismatch
from . import _lib as L
from .evaluator import BatchEvaluator, Coupling, StagePlan
from .grid import ISOLATED, REF, apply_contingency, apply_scenario, check_connectivity, resolve_outages, scenario_targets
from .packer import PackedCase, Topology
from .stage import CallbackSet
from .types import (
    CONTINGENCY_BOX, CORRECTIVE, PREVENTIVE_PIN, RAMP, SCENARIO_BOX,
    AcopfLayout, CompositeIndexMap, CouplingMode, CouplingRow, NlpProblem, StageSpec,
)
from .errors import Disconnected

KINDS = (RAMP, CONTINGENCY_BOX, SCENARIO_BOX, PREVENTIVE_PIN)


class LazySeq:
    """Read-only sequence whose items are built on first access."""

    def __init__(self, n: int, make):
        self._n = n
        self._make = make
        self._cache: dict = {}

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        if i not in self._cache:
            self._cache[i] = self._make(i)
        return self._cache[i]

    def __iter__(self):
        return (self[i] for i in range(self._n))

    def __eq__(self, other):
        try:
            return len(other) == self._n and all(a == b for a, b in zip(self, other))
        except TypeError:
            return NotImplemented

    def __contains__(self, item):
        return any(item == v for v in self)

    def index(self, item):
        for i, v in enumerate(self):
            if v == item:
                return i
        raise ValueError(f"{item!r} is not in the sequence")

    def count(self, item):
        return sum(1 for v in self if v == item)

    def __reversed__(self):
        return (self[i] for i in range(self._n - 1, -1, -1))

    def __repr__(self):
        return f"LazySeq(len={self._n})"


# a read-only sequence for isinstance checks (collections.abc.Sequence), like the
# reference's tuples; items are built on first access (cfg4: 6.1 M coupling rows)
import collections.abc as _abc  # noqa: E402
_abc.Sequence.register(LazySeq)


def _same_topology(a: PackedCase, b: PackedCase) -> bool:
    """Everything but loads equal (composer.py:112-126 checks a subset)."""
    pairs = [(a.active, b.active), (a.gs, b.gs), (a.bs, b.bs), (a.gen_bus, b.gen_bus),
             (a.gen_status, b.gen_status), (a.c2, b.c2), (a.c1, b.c1), (a.c0, b.c0),
             (a.br_f, b.br_f), (a.br_t, b.br_t), (a.br_status, b.br_status), (a.adm, b.adm),
             (a.smax2, b.smax2), (a.rate_a > 0, b.rate_a > 0)]
    return a.base == b.base and all(x.shape == y.shape and np.array_equal(x, y) for x, y in pairs)


def _check_topology(ref, other) -> None:
    same = (ref.base_mva == other.base_mva
            and len(ref.buses) == len(other.buses)
            and len(ref.gens) == len(other.gens)
            and len(ref.branches) == len(other.branches)
            and all(a.id == b.id and a.btype == b.btype for a, b in zip(ref.buses, other.buses))
            and all(a.bus == b.bus and a.status == b.status for a, b in zip(ref.gens, other.gens))
            and all(a.fbus == b.fbus and a.tbus == b.tbus and a.status == b.status
                    for a, b in zip(ref.branches, other.branches)))
    if not same:
        raise TopologyMismatch("periods must share one topology (loads may differ)")


def _bridges(pc: PackedCase) -> set:
    """Case positions of live branches whose outage islands the network (native Tarjan,
    acopf_graph_bridges, over the live multigraph)."""
    import ctypes
    ea = L.i32(pc.br_f[pc.live_br])
    eb = L.i32(pc.br_t[pc.live_br])
    out = np.zeros(max(len(ea), 1), dtype=np.uint8)
    if len(ea):
        L.check(L.lib().acopf_graph_bridges(len(pc.bus_id), len(ea), L.ptr(ea, ctypes.c_int32),
                                            L.ptr(eb, ctypes.c_int32), None, L.ptr(out, ctypes.c_uint8)))
    return set(int(k) for k in np.asarray(pc.live_br)[out[:len(ea)].astype(bool)])


def _islands_without(pc: PackedCase, removed_case_branches) -> int:
    """Island count of the in-service network minus some branches (check_connectivity, native)."""
    import ctypes
    live = np.asarray(pc.live_br)
    keep = ~np.isin(live, np.asarray(removed_case_branches, dtype=np.int64))
    ea, eb = L.i32(pc.br_f[live]), L.i32(pc.br_t[live])
    el = np.ascontiguousarray(keep, dtype=np.uint8)
    alive = np.ascontiguousarray(pc.btype != ISOLATED, dtype=np.uint8)
    n = ctypes.c_int32()
    L.check(L.lib().acopf_graph_islands(len(alive), L.ptr(alive, ctypes.c_uint8), len(ea), L.ptr(ea, ctypes.c_int32),
                                        L.ptr(eb, ctypes.c_int32), L.ptr(el, ctypes.c_uint8) if len(el) else None,
                                        ctypes.byref(n), None))
    return int(n.value)


@dataclass
class CompositeSpec:
    """A composite lattice without its evaluator (used for sharding across GPUs)."""
    plans: list
    cp: dict                  # coupling rows: kind, stage_a/b, gen, bus, bound, row, col_a/b (global)
    n_pins: int
    n_s: np.ndarray           # per-stage n, m_eq, m_ineq
    meq_s: np.ndarray
    mineq_s: np.ndarray
    var_off: np.ndarray
    eq_off: np.ndarray
    ineq_off: np.ndarray
    m_eq: int
    m_ineq: int
    stage_dims: list          # (nb, ng) per stage


class _Stage:
    __slots__ = ("s_pos", "c_pos", "t", "scen", "ctg", "weight", "topo", "removed", "pt",
                 "pmin", "pmax", "gen_live", "case_gen_live")

    def __init__(self, **kw):
        for k, v in kw.items():
            setattr(self, k, v)


class _Lattice:
    def __init__(self, periods, name: str, device: int):
        self.name = name
        self.device = device
        self.periods = list(periods)
        self.pcs = []
        self.period_topo = []          # period -> representative period index
        for t, case in enumerate(self.periods):
            pc = PackedCase(case)
            rep = next((r for r in sorted(set(self.period_topo)) if _same_topology(self.pcs[r], pc)), t)
            self.pcs.append(pc)
            self.period_topo.append(rep)
        for r in sorted(set(self.period_topo)):
            n_islands, _ = check_connectivity(self.periods[r])
            if n_islands != 1:
                raise Disconnected(f"case {self.periods[r].name!r} has {n_islands} islands")
        self._topos: dict = {}
        self._bridges: dict = {}
        self.stages: list = []
        self.rows: list = []           # (kind, child, base, gens or None, buses or None, bounds, is_eq)

    # -- stage construction ----------------------------------------------------

    def topo(self, rep: int, gen_off: frozenset) -> Topology:
        key = (rep, gen_off)
        if key not in self._topos:
            self._topos[key] = Topology(self.pcs[rep], gen_off)
        return self._topos[key]

    def islands_after(self, rep: int, case_branches, ctg) -> None:
        if not case_branches:
            return
        if len(case_branches) == 1:
            # a single outage islands exactly when the branch is a bridge of the
            # live multigraph (a parallel twin is a back edge, so not a bridge)
            if rep not in self._bridges:
                self._bridges[rep] = _bridges(self.pcs[rep])
            if int(case_branches[0]) in self._bridges[rep]:
                raise IslandingDetected(f"contingency {ctg.id} splits the network into 2 islands")
            return
        n = _islands_without(self.pcs[rep], case_branches)      # one native check per contingency
        if n != 1:
            raise IslandingDetected(f"contingency {ctg.id} splits the network into {n} islands")

    def add_stage(self, s_pos, c_pos, t, scen, ctg, weight, targets, outages) -> int:
        rep = self.period_topo[t]
        pc = self.pcs[t]
        gen_off, br_off = outages if outages is not None else ((), ())
        topo = self.topo(rep, frozenset(gen_off))
        removed = topo.removed_local(br_off) if br_off else np.zeros(0, dtype=np.int32)
        pmin = pmax = None
        if targets:
            pmin, pmax = pc.pmin.copy(), pc.pmax.copy()
            for k, mw in targets.items():
                pmax[k] = mw
                pmin[k] = 0.0
        case_live = pc.gen_status.copy()
        for g in gen_off:
            case_live[g] = False
        self.stages.append(_Stage(s_pos=s_pos, c_pos=c_pos, t=t, scen=scen, ctg=ctg, weight=weight,
                                  topo=topo, removed=removed, pt=pc, pmin=pmin, pmax=pmax,
                                  case_gen_live=case_live))
        return len(self.stages) - 1

    # -- coupling rows (composer.py:157-197) -------------------------------------

    def _live_both(self, a: int, b: int) -> np.ndarray:
        return np.flatnonzero(self.stages[a].case_gen_live & self.stages[b].case_gen_live)

    def ramp_rows(self, child, base, dt):
        pc = self.stages[base].pt
        g = self._live_both(child, base)
        self.rows.append((RAMP, child, base, g, None, pc.ramp[g] * (dt / 30.0) / pc.base, False))

    def mode_rows(self, child, base, mode, box_kind=CONTINGENCY_BOX, scale=None):
        pc = self.stages[base].pt
        g = self._live_both(child, base)
        if mode.kind == CORRECTIVE:
            m = mode.contingency_scale if scale is None else scale
            self.rows.append((box_kind, child, base, g, None, pc.ramp[g] * m / pc.base, False))
            return
        bus_of = pc.gen_bus[g]
        keep = pc.btype[bus_of] != REF
        gp = g[keep]
        self.rows.append((PREVENTIVE_PIN, child, base, gp, None, np.zeros(len(gp)), True))
        if mode.pin_voltages:
            buses = np.array(sorted(set(int(b) for b in bus_of)), dtype=np.int64)
            self.rows.append((PREVENTIVE_PIN, child, base, None, buses, np.zeros(len(buses)), True))

    def scenario_rows(self, child, base, mode):
        pc = self.stages[base].pt
        g = self._live_both(child, base)
        self.rows.append((SCENARIO_BOX, child, base, g, None, pc.ramp[g] * mode.scenario_scale / pc.base, False))

    # -- assembly -------------------------------------------------------------------

    def spec(self) -> "CompositeSpec":
        """Stage plans, offsets and coupling rows -- everything but the evaluator."""
        st = self.stages
        ns = len(st)
        plans = []
        for s in st:
            pc = s.pt
            plans.append(StagePlan(topo=s.topo, removed=s.removed, pd=pc.pd, qd=pc.qd,
                                   load_key=("t", s.t), weight=s.weight))
        n_s = np.array([s.topo.n for s in st], dtype=np.int64)
        meq_s = np.array([2 * s.topo.nb for s in st], dtype=np.int64)
        rated_live = []
        rated_mask = {}                # topology -> per local branch: 1 when rated
        for s in st:
            key = id(s.topo)
            if key not in rated_mask:
                m = np.zeros(s.topo.nbr, dtype=bool)
                m[s.topo.rated_pos] = True
                rated_mask[key] = m
            nr = len(s.topo.rated_pos)
            gone = int(np.count_nonzero(rated_mask[key][s.removed])) if len(s.removed) else 0
            rated_live.append(nr - gone)
        mineq_s = 2 * np.array(rated_live, dtype=np.int64)
        var_off = np.concatenate([[0], np.cumsum(n_s)[:-1]]).astype(np.int64)
        eq_off = np.concatenate([[0], np.cumsum(meq_s)[:-1]]).astype(np.int64)
        ineq_off = np.concatenate([[0], np.cumsum(mineq_s)[:-1]]).astype(np.int64)
        nv = int(n_s.sum())
        me_st, mi_st = int(meq_s.sum()), int(mineq_s.sum())

        # flatten coupling rows: pins (in order), then boxes (in order)
        pins = [r for r in self.rows if r[6]]
        boxes = [r for r in self.rows if not r[6]]
        n_pins = sum(len(r[5]) for r in pins)
        n_box = sum(len(r[5]) for r in boxes)
        m_eq, m_ineq = me_st + n_pins, mi_st + n_box

        def var_cols(stage, gens, buses):
            s = st[stage]
            if gens is not None:
                pos = np.searchsorted(s.topo.live_gens, gens)
                return var_off[stage] + 2 * s.topo.nb + pos
            return var_off[stage] + s.topo.nb + s.topo.pc.slot[buses]

        # one preallocated array per field, filled group by group (6.1 M rows for cfg4)
        total = sum(len(r[5]) for r in pins) + sum(len(r[5]) for r in boxes)
        cp = dict(kind=np.empty(total, dtype=np.int8), stage_a=np.empty(total, dtype=np.int64),
                  stage_b=np.empty(total, dtype=np.int64), gen=np.empty(total, dtype=np.int64),
                  bus=np.empty(total, dtype=np.int64), bound=np.empty(total, dtype=np.float64),
                  row=np.empty(total, dtype=np.int64), col_a=np.empty(total, dtype=np.int64),
                  col_b=np.empty(total, dtype=np.int64))
        gen_pos = {}                   # topology -> variable position of each case generator (-1: off)

        def var_cols_fast(stage, gens, buses):
            s = st[stage]
            if gens is not None:
                key = id(s.topo)
                if key not in gen_pos:
                    m = np.full(int(s.topo.live_gens.max()) + 1 if len(s.topo.live_gens) else 1, -1, dtype=np.int64)
                    m[s.topo.live_gens] = np.arange(len(s.topo.live_gens))
                    gen_pos[key] = m
                return var_off[stage] + 2 * s.topo.nb + gen_pos[key][gens]
            return var_cols(stage, gens, buses)

        at = 0
        nxt_pin, nxt_box = me_st, m_eq + mi_st
        for group in (pins, boxes):
            for kind, child, base, gens, buses, bnd, is_eq in group:
                k = len(bnd)
                if k == 0:
                    continue
                sl = slice(at, at + k)
                start = nxt_pin if is_eq else nxt_box
                cp["row"][sl] = np.arange(start, start + k, dtype=np.int64)
                if is_eq:
                    nxt_pin += k
                else:
                    nxt_box += k
                cp["kind"][sl] = KINDS.index(kind)
                cp["stage_a"][sl] = child
                cp["stage_b"][sl] = base
                cp["gen"][sl] = gens if gens is not None else -1
                cp["bus"][sl] = buses if buses is not None else -1
                cp["bound"][sl] = bnd
                cp["col_a"][sl] = var_cols_fast(child, gens, buses)
                cp["col_b"][sl] = var_cols_fast(base, gens, buses)
                at += k
        return CompositeSpec(plans=plans, cp=cp, n_pins=n_pins, n_s=n_s, meq_s=meq_s, mineq_s=mineq_s,
                             var_off=var_off, eq_off=eq_off, ineq_off=ineq_off, m_eq=m_eq, m_ineq=m_ineq,
                             stage_dims=[(s.topo.nb, s.topo.ng) for s in st])

    def assemble(self):
        sp = self.spec()
        st = self.stages
        ns = len(st)
        plans, cp, n_pins = sp.plans, sp.cp, sp.n_pins
        n_s, meq_s, mineq_s = sp.n_s, sp.meq_s, sp.mineq_s
        var_off, eq_off, ineq_off = sp.var_off, sp.eq_off, sp.ineq_off
        nv, m_eq, m_ineq = int(n_s.sum()), sp.m_eq, sp.m_ineq
        self.cp = cp
        ev = BatchEvaluator(plans, device=self.device, layout="composite",
                            coupling=Coupling(row=cp["row"], col_a=cp["col_a"], col_b=cp["col_b"]),
                            n_pins=n_pins)
        if (ev.n, ev.m_eq, ev.m_ineq) != (nv, m_eq, m_ineq):
            raise RuntimeError("native planner sizes disagree with the lattice")

        # bounds: one (xl, xu, x0) per distinct (topology, period, scenario limits) and one
        # (gl, gu) per distinct (topology, removed branches); the flat vectors are filled by
        # the library's threaded run copy (acopf_copy_runs)
        xl, xu, x0 = (np.empty(nv) for _ in range(3))
        is_box = cp["row"] >= m_eq
        n_box = int(np.count_nonzero(is_box))
        mi_st = int(mineq_s.sum())
        gl, gu = np.empty(mi_st + n_box), np.empty(mi_st + n_box)
        xkeys, gkeys = {}, {}
        xsrc, gsrc = [], []
        x_src_off = np.empty(ns, dtype=np.int64)
        g_src_off = np.empty(ns, dtype=np.int64)
        xo = go = 0
        for k, s in enumerate(st):
            kx = (id(s.topo), s.t, s.s_pos if s.pmin is not None else -1)
            if kx not in xkeys:
                xkeys[kx] = xo
                xsrc.append(stage_bounds(s.topo, s.pt, s.pmin, s.pmax))
                xo += s.topo.n
            x_src_off[k] = xkeys[kx]
            kg = (id(s.topo), s.removed.tobytes())
            if kg not in gkeys:
                gkeys[kg] = go
                gsrc.append(s.topo.ineq_bounds(s.removed))
                go += len(gsrc[-1][0])
            g_src_off[k] = gkeys[kg]
        lens = n_s.astype(np.int64)
        for dst, j in ((xl, 0), (xu, 1), (x0, 2)):
            copy_runs(dst, var_off, np.concatenate([b[j] for b in xsrc]), x_src_off, lens)
        glens = mineq_s.astype(np.int64)
        for dst, j in ((gl, 0), (gu, 1)):
            src = np.concatenate([b[j] for b in gsrc]) if gsrc else np.zeros(0)
            copy_runs(dst, ineq_off, src, g_src_off, glens)
        gl[mi_st:] = -cp["bound"][is_box]
        gu[mi_st:] = cp["bound"][is_box]

        cbk = CallbackSet(ev)
        problem = NlpProblem(n=nv, m_eq=m_eq, m_ineq=m_ineq, xl=xl, xu=xu, gl=gl, gu=gu, x0=x0,
                             objective=cbk.objective, gradient=cbk.gradient, constraints=cbk.constraints,
                             jacobian=cbk.jacobian, lagrangian_hessian=cbk.lagrangian_hessian, name=self.name)
        problem.evaluator = ev

        periods = self.periods

        def make_spec(k):
            s = st[k]
            case = periods[s.t]
            if s.scen is not None:
                case = apply_scenario(case, s.scen)
            if s.ctg is not None:
                case = apply_contingency(case, s.ctg)
            return StageSpec(scenario=s.scen, contingency=s.ctg, period=s.t, dt_minutes=self.dt, case=case)

        def make_layout(k):
            s = st[k]
            maps = s.topo.layout_maps(s.removed)
            return AcopfLayout(n_vars=int(n_s[k]), n_eq=int(meq_s[k]), n_ineq=int(mineq_s[k]), **maps)

        def make_row(i):
            g, b = int(cp["gen"][i]), int(cp["bus"][i])
            return CouplingRow(kind=KINDS[cp["kind"][i]], stage_a=int(cp["stage_a"][i]),
                               stage_b=int(cp["stage_b"][i]), gen=None if g < 0 else g,
                               bus=None if b < 0 else b, bound=float(cp["bound"][i]), row=int(cp["row"][i]),
                               is_equality=bool(cp["row"][i] < m_eq))

        index = CompositeIndexMap(
            stages=LazySeq(ns, make_spec), var_offset=tuple(int(v) for v in var_off),
            eq_offset=tuple(int(v) for v in eq_off), ineq_offset=tuple(int(v) for v in ineq_off),
            coupling_rows=LazySeq(len(cp["row"]), make_row), weights=tuple(float(s.weight) for s in st),
            layouts=LazySeq(ns, make_layout), n_vars=nv, m_eq=m_eq, m_ineq=m_ineq)
        # extension (not a reference field): the coupling rows as arrays -- kind code (KINDS),
        # stage_a, stage_b, gen, bus (-1 = none), bound, row, and the x columns col_a / col_b
        object.__setattr__(index, "coupling_arrays", cp)
        return problem, index


def copy_runs(dst: np.ndarray, dst_off, src: np.ndarray, src_off, lens) -> None:
    """dst[dst_off[i]:+lens[i]] = src[src_off[i]:+lens[i]] for every run (acopf_copy_runs, threaded)."""
    import ctypes
    n = len(lens)
    if n == 0:
        return
    do, so, ln = L.i64(dst_off), L.i64(src_off), L.i64(lens)
    src = L.f64(src) if len(src) else np.zeros(1)
    L.check(L.lib().acopf_copy_runs(n, dst.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), L.ptr(do, ctypes.c_int64),
                                    L.ptr(src, ctypes.c_double), L.ptr(so, ctypes.c_int64), L.ptr(ln, ctypes.c_int64)))


def stage_bounds(topo: Topology, pc: PackedCase, pmin=None, pmax=None):
    """(xl, xu, x0) of one stage (acopf.py:197-221) from its own period data."""
    nb, ng = topo.nb, topo.ng
    base = pc.base
    n = topo.n
    xl = np.full(n, -np.inf)
    xu = np.full(n, np.inf)
    x0 = np.zeros(n)
    x0[:nb] = pc.va
    xl[nb:2 * nb] = pc.vmin
    xu[nb:2 * nb] = pc.vmax
    x0[nb:2 * nb] = np.minimum(np.maximum(pc.vm, pc.vmin), pc.vmax)
    ref = np.flatnonzero(pc.is_ref)
    xl[ref] = pc.va[ref]
    xu[ref] = pc.va[ref]
    g = topo.live_gens
    lo = (pc.pmin if pmin is None else pmin)[g]
    hi = (pc.pmax if pmax is None else pmax)[g]
    o = 2 * nb
    xl[o:o + ng] = lo / base
    xu[o:o + ng] = hi / base
    x0[o:o + ng] = 0.5 * (lo + hi) / base
    o += ng
    xl[o:o + ng] = pc.qmin[g] / base
    xu[o:o + ng] = pc.qmax[g] / base
    x0[o:o + ng] = 0.5 * (pc.qmin[g] + pc.qmax[g]) / base
    return xl, xu, x0


def _scenario_order(scenarios):
    if scenarios is None:
        return [(None, 1.0)]
    items = list(scenarios.scenarios)
    if not items:
        raise EmptyScenarioSet("no scenarios to compose")
    total = sum(s.weight for s in items)
    if not total > 0.0:
        raise EmptyScenarioSet("scenario weights sum to zero")
    b = scenarios.base_index()
    rest = sorted((s for i, s in enumerate(items) if i != b), key=lambda s: s.id)
    return [(s, s.weight / total) for s in [items[b]] + rest]


def _ctg_order(ctgs):
    return [None] if ctgs is None else [None] + list(ctgs.by_id())


def _general_impl(scenarios, ctgs, periods, mode, dt_minutes, name, device, spec_only=False):
    if not periods:
        raise InvalidPlan("at least one period is required")
    nt = len(periods)
    if nt > 1 and not dt_minutes > 0:
        raise InvalidPlan("dt_minutes must be positive for multiple periods")
    for t in range(1, nt):
        _check_topology(periods[0], periods[t])
    lat = _Lattice(periods, name, device)
    lat.dt = dt_minutes
    so = _scenario_order(scenarios)
    co = _ctg_order(ctgs)
    # validate transforms once (they only depend on the shared topology)
    targets = [None if sc is None else scenario_targets(periods[0], sc) for sc, _ in so]
    outages = []
    for c in co:
        if c is None:
            outages.append(None)
            continue
        goff, boff = resolve_outages(periods[0], c)
        lat.islands_after(lat.period_topo[0], list(boff), c)
        outages.append((goff, boff))
    idx = {}
    for si, (sc, w) in enumerate(so):
        for ci, c in enumerate(co):
            for t in range(nt):
                idx[(si, ci, t)] = lat.add_stage(si, ci, t, sc, c, w, targets[si], outages[ci])
    for si in range(len(so)):
        for ci in range(len(co)):
            for t in range(1, nt):
                lat.ramp_rows(idx[(si, ci, t)], idx[(si, ci, t - 1)], dt_minutes)
        for ci in range(1, len(co)):
            lat.mode_rows(idx[(si, ci, 0)], idx[(si, 0, 0)], mode)
        if si > 0:
            lat.scenario_rows(idx[(si, 0, 0)], idx[(0, 0, 0)], mode)
    return lat.spec() if spec_only else lat.assemble()


def compose_multiperiod(cases, dt_minutes: float, *, device: int = 0):
    """Ramp-coupled horizon; one stage per period (composer.py:391-394)."""
    return _general_impl(None, None, list(cases), CouplingMode(), dt_minutes,
                         f"tcopf(nt={len(cases)})", device)


def compose_scopf(base, ctgs, mode, *, device: int = 0):
    """Base plus post-contingency stages (composer.py:397-401)."""
    return _general_impl(None, ctgs, [base], mode, 30.0, f"scopf(nc={len(ctgs)})", device)


def compose_multiperiod_scopf(base_periods, ctgs, mode, dt_minutes: float, *, device: int = 0):
    """Every (contingency, period) stage (composer.py:404-411)."""
    return _general_impl(None, ctgs, list(base_periods), mode, dt_minutes,
                         f"tcopf-scopf(nc={len(ctgs)},nt={len(base_periods)})", device)


def compose_sopf_full(base, scenarios, ctgs, mode, *, device: int = 0):
    """Three-stage tree (composer.py:414-420)."""
    nc = 0 if ctgs is None else len(ctgs)
    return _general_impl(scenarios, ctgs, [base], mode, 30.0,
                         f"sopf-full(ns={len(scenarios)},nc={nc})", device)


def compose_general(scenarios, ctgs, periods, mode, dt_minutes: float, *, device: int = 0):
    """Full (scenario, contingency, period) lattice (composer.py:423-432)."""
    n_s = 1 if scenarios is None else len(scenarios)
    n_c = 0 if ctgs is None else len(ctgs)
    return _general_impl(scenarios, ctgs, list(periods), mode, dt_minutes,
                         f"sopf-general(ns={n_s},nc={n_c},nt={len(periods)})", device)


def compose_sopf_flat(base, scenarios, ctgs, mode, *, device: int = 0):
    """All stages couple to the most probable scenario's base (composer.py:435-457)."""
    lat = _Lattice([base], f"sopf-flat(ns={len(scenarios)},nc={0 if ctgs is None else len(ctgs)})", device)
    lat.dt = 30.0
    co = _ctg_order(ctgs)
    outages = []
    for c in co:
        if c is None:
            outages.append(None)
            continue
        goff, boff = resolve_outages(base, c)
        lat.islands_after(0, list(boff), c)
        outages.append((goff, boff))
    ids = []
    for si, (sc, w) in enumerate(_scenario_order(scenarios)):
        tg = None if sc is None else scenario_targets(base, sc)
        for ci, c in enumerate(co):
            k = lat.add_stage(si, ci, 0, sc, c, w, tg, outages[ci])
            ids.append((ci, k))
    for ci, k in ids:
        if k == 0:
            continue
        lat.mode_rows(k, 0, mode, box_kind=CONTINGENCY_BOX if ci > 0 else SCENARIO_BOX,
                      scale=mode.contingency_scale if ci > 0 else mode.scenario_scale)
    return lat.assemble()


def composite_spec(kind: str, *args, **kw) -> CompositeSpec:
    """The lattice of compose_<kind>(*args) without building an evaluator.

    kind: "multiperiod" (cases, dt), "scopf" (base, ctgs, mode), "general"
    (scenarios, ctgs, periods, mode, dt).  Used by :mod:`dispatch` to shard
    the stages over ranks.
    """
    if kind == "multiperiod":
        cases, dt = args
        return _general_impl(None, None, list(cases), CouplingMode(), dt, "tcopf", 0, spec_only=True)
    if kind == "scopf":
        base, ctgs, mode = args
        return _general_impl(None, ctgs, [base], mode, 30.0, "scopf", 0, spec_only=True)
    if kind == "general":
        scens, ctgs, periods, mode, dt = args
        return _general_impl(scens, ctgs, list(periods), mode, dt, "general", 0, spec_only=True)
    raise ValueError(f"unknown composite kind {kind!r}")
