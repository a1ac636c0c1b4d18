"""Pack NetworkCase objects into structure-of-arrays tables.

Mirrors the reference's ``_Engine.__init__`` (`acopf.py:77-149`) and
``_build_bounds`` (`acopf.py:197-221`) with the same per-unit conversions and
the same floating-point expressions, so the packed doubles (and therefore
every evaluated value) are bit-identical to the reference's:

* active buses = type != 4, in case order; live generators/branches =
  status != 0 in case order; a live branch on an isolated bus raises
  :class:`Disconnected` (acopf.py:91-102);
* ``pd/qd/gs/bs = value / base``; ``cost_a = c2 * base * base``,
  ``cost_b = c1 * base``, ``cost_c = c0``;
* branch admittances in CPython ``complex`` (network.py:215-229);
* ``smax2 = (rate_a / base) ** 2`` per rated branch, in Python floats.

A :class:`PackedCase` holds every element of one case (including
out-of-service ones) so that contingency / scenario / period variants of
the same grid are derived by masking instead of re-packing.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import Disconnected
from .grid import ISOLATED, REF, check_connectivity

def _admittance8(br) -> tuple:
    ys = 1.0 / complex(br.r, br.x)
    half_b = complex(0.0, br.b / 2.0)
    m = 1.0 if br.ratio == 0.0 else br.ratio
    t = m * complex(math.cos(br.angle), math.sin(br.angle))
    tc = t.conjugate()
    yff, yft, ytf, ytt = (ys + half_b) / (t * tc), -ys / tc, -ys / t, ys + half_b
    return (yff.real, yff.imag, yft.real, yft.imag, ytf.real, ytf.imag, ytt.real, ytt.imag)


class PackedCase:
    """Every element of one case as numpy arrays (no liveness applied yet)."""

    def __init__(self, case):
        self.case = case
        base = float(case.base_mva)
        self.base = base
        buses, gens, brs = case.buses, case.gens, case.branches
        self.bus_id = np.array([b.id for b in buses], dtype=np.int64)
        self.btype = np.array([b.btype for b in buses], dtype=np.int64)
        self.bus_pos = {int(b): k for k, b in enumerate(self.bus_id)}
        self.active = np.flatnonzero(self.btype != ISOLATED)
        self.slot = np.full(len(buses), -1, dtype=np.int64)
        self.slot[self.active] = np.arange(len(self.active))
        act = [buses[p] for p in self.active]
        self.pd = np.array([b.pd for b in act], dtype=np.float64) / base
        self.qd = np.array([b.qd for b in act], dtype=np.float64) / base
        self.gs = np.array([b.gs for b in act], dtype=np.float64) / base
        self.bs = np.array([b.bs for b in act], dtype=np.float64) / base
        self.vm = np.array([b.vm for b in act], dtype=np.float64)
        self.va = np.array([b.va for b in act], dtype=np.float64)
        self.vmin = np.array([b.vmin for b in act], dtype=np.float64)
        self.vmax = np.array([b.vmax for b in act], dtype=np.float64)
        self.is_ref = np.array([b.btype == REF for b in act], dtype=bool)

        pos = self.bus_pos
        self.gen_bus = np.array([pos[g.bus] for g in gens], dtype=np.int64)
        self.gen_status = np.array([g.status != 0 for g in gens], dtype=bool)
        self.pmin = np.array([g.pmin for g in gens], dtype=np.float64)
        self.pmax = np.array([g.pmax for g in gens], dtype=np.float64)
        self.qmin = np.array([g.qmin for g in gens], dtype=np.float64)
        self.qmax = np.array([g.qmax for g in gens], dtype=np.float64)
        self.c2 = np.array([g.cost.c2 for g in gens], dtype=np.float64)
        self.c1 = np.array([g.cost.c1 for g in gens], dtype=np.float64)
        self.c0 = np.array([g.cost.c0 for g in gens], dtype=np.float64)
        self.ramp = np.array([g.ramp_30 for g in gens], dtype=np.float64)

        self.br_f = np.array([pos[b.fbus] for b in brs], dtype=np.int64)
        self.br_t = np.array([pos[b.tbus] for b in brs], dtype=np.int64)
        self.br_status = np.array([b.status != 0 for b in brs], dtype=bool)
        self.rate_a = np.array([b.rate_a for b in brs], dtype=np.float64)
        self.live_br = np.flatnonzero(self.br_status)
        bad = (self.slot[self.br_f[self.live_br]] < 0) | (self.slot[self.br_t[self.live_br]] < 0)
        if bad.any():
            br = brs[int(self.live_br[np.flatnonzero(bad)[0]])]
            raise Disconnected(f"in-service branch {br.fbus}-{br.tbus} touches an isolated bus")
        self.adm = np.zeros((len(brs), 8), dtype=np.float64)
        for k in self.live_br:
            self.adm[k] = _admittance8(brs[int(k)])
        self.smax2 = np.zeros(len(brs), dtype=np.float64)
        for k in self.live_br:
            ra = brs[int(k)].rate_a
            if ra > 0.0:
                self.smax2[k] = (ra / base) ** 2

    def n_islands(self) -> int:
        return check_connectivity(self.case)[0]


class Topology:
    """One packed topology: a PackedCase with a fixed set of live generators.

    Branch outages of contingency stages are *not* part of the topology;
    they are passed to the device as per-stage removed lists.
    """

    def __init__(self, pc: PackedCase, gen_off: frozenset = frozenset()):
        self.pc = pc
        self.gen_off = gen_off
        live_g = pc.gen_status.copy()
        for g in gen_off:
            live_g[g] = False
        self.live_gens = np.flatnonzero(live_g)
        self.live_br = pc.live_br
        self.br_index = np.full(len(pc.br_status), -1, dtype=np.int64)
        self.br_index[self.live_br] = np.arange(len(self.live_br))
        self.nb = len(pc.active)
        self.ng = len(self.live_gens)
        self.nbr = len(self.live_br)
        self.fo = pc.slot[pc.br_f[self.live_br]].astype(np.int32)
        self.to = pc.slot[pc.br_t[self.live_br]].astype(np.int32)
        self.adm = np.ascontiguousarray(pc.adm[self.live_br])
        self.rated = (pc.rate_a[self.live_br] > 0.0).astype(np.uint8)
        self.rated_pos = np.flatnonzero(self.rated)          # live index of each rated branch
        self.gbus = pc.slot[pc.gen_bus[self.live_gens]].astype(np.int32)
        base = pc.base
        self.ca = pc.c2[self.live_gens] * base * base
        self.cb = pc.c1[self.live_gens] * base
        self.cc = pc.c0[self.live_gens].copy()
        self.n = 2 * self.nb + 2 * self.ng
        self._handle = None

    def handle(self):
        """Native topology handle (created on first use)."""
        if self._handle is None:
            import ctypes
            from . import _lib as L
            h = ctypes.c_void_p()
            fo, to = L.i32(self.fo), L.i32(self.to)
            adm = L.f64(self.adm.reshape(-1))
            rated = np.ascontiguousarray(self.rated, dtype=np.uint8)
            gbus = L.i32(self.gbus)
            gs, bs = L.f64(self.pc.gs), L.f64(self.pc.bs)
            L.check(L.lib().acopf_topo_create(
                self.nb, self.nbr, self.ng, L.ptr(fo, ctypes.c_int32), L.ptr(to, ctypes.c_int32),
                L.ptr(adm, ctypes.c_double), L.ptr(rated, ctypes.c_uint8), L.ptr(gbus, ctypes.c_int32),
                L.ptr(gs, ctypes.c_double), L.ptr(bs, ctypes.c_double), ctypes.byref(h)))
            self._handle = h
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                from . import _lib as L
                L.lib().acopf_topo_destroy(h)
            except Exception:
                pass

    # -- per-stage host data ---------------------------------------------------

    def bounds(self, pmin=None, pmax=None):
        """(xl, xu, x0) like acopf.py:197-221; pmin/pmax override (all gens, MW)."""
        pc, nb, ng = self.pc, self.nb, self.ng
        base = pc.base
        n = self.n
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
        g = self.live_gens
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

    def ref_positions(self) -> tuple:
        return tuple(int(p) for p in self.pc.active[self.pc.is_ref])

    def removed_local(self, case_branches) -> np.ndarray:
        """Topology-local indices of case branch positions (must be live)."""
        idx = self.br_index[np.asarray(case_branches, dtype=np.int64)]
        if (idx < 0).any():
            raise ValueError("removed branch is not live in the topology")
        return np.sort(idx).astype(np.int32)

    def ineq_bounds(self, removed_local=()) -> tuple:
        """(gl, gu) of the stage inequality rows after branch removals."""
        keep = np.ones(self.nbr, dtype=bool)
        keep[np.asarray(removed_local, dtype=np.int64)] = False
        live_rated = self.rated_pos[keep[self.rated_pos]]
        smax2 = self.pc.smax2[self.live_br[live_rated]]
        gu = np.repeat(smax2, 2) if len(smax2) else np.zeros(0)
        return np.full(len(gu), -np.inf), gu

    def layout_maps(self, removed_local=()) -> dict:
        """AcopfLayout maps (acopf.py:376-389) of the topology minus removals."""
        pc, nb = self.pc, self.nb
        act = [int(p) for p in pc.active]
        keep = np.ones(self.nbr, dtype=bool)
        keep[np.asarray(removed_local, dtype=np.int64)] = False
        live_rated = self.rated_pos[keep[self.rated_pos]]
        case_idx = self.live_br[live_rated]
        off_pg, off_qg = 2 * nb, 2 * nb + self.ng
        return dict(
            va={p: s for s, p in enumerate(act)},
            vm={p: s + nb for s, p in enumerate(act)},
            pg={int(g): off_pg + j for j, g in enumerate(self.live_gens)},
            qg={int(g): off_qg + j for j, g in enumerate(self.live_gens)},
            p_row={p: s for s, p in enumerate(act)},
            q_row={p: s + nb for s, p in enumerate(act)},
            sf_row={int(k): 2 * j for j, k in enumerate(case_idx)},
            st_row={int(k): 2 * j + 1 for j, k in enumerate(case_idx)},
            ref_buses=self.ref_positions())
