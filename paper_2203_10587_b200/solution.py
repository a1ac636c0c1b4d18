"""Solutions at an NLP point: line flows and power-balance residuals on the B200.

Drop-in for `pkg/src/opfkit/acopf.py:413-546` (``SolvedCase``,
``extract_solution``, ``pack_solution``, ``solution_from_case``,
``residuals_at``): same signatures, same arrays, same errors.  The network
part -- per-branch flows and per-bus injections (acopf.py:230-264) -- runs in
the evaluation kernel's flows mode (``acopf_batch_flows``); the host only
applies the reference's MVA scaling, load and dispatch terms in the
reference's order, so every array is bit-identical to the reference's.

``extract_solutions`` is the batched form the runner needs after a composite
solve (runner.py:209, 260-262): the flows of every stage of a composite come
from ONE launch over the composite's device evaluator.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .errors import DimensionMismatch
from .evaluator import BatchEvaluator
from .packer import PackedCase, Topology
from .stage import stage_plan


@dataclass(frozen=True)
class SolvedCase:
    """A case with an operating point and its line flows (acopf.py:413-431).

    Arrays align with case.buses / case.gens / case.branches; out-of-service
    elements are zero.  MW / MVAr, radians, $/h.
    """

    case: object
    vm: np.ndarray
    va: np.ndarray
    pg: np.ndarray
    qg: np.ndarray
    pf: np.ndarray
    qf: np.ndarray
    pt: np.ndarray
    qt: np.ndarray
    objective: float

    def to_raw(self, name=None):
        """RawCase with solved voltages, dispatch and flow columns (acopf.py:433-446)."""
        from .matpower import solved_to_raw
        return solved_to_raw(self, name=name)


def device_flows(ev: BatchEvaluator, x_dev, stream=None):
    """(flows, inj) device tensors of every stage of ``ev`` at device ``x_dev``.

    Layout per stage in batch order (include/acopf_b200.h, acopf_batch_flows):
    flows = [pf | qf | pt | qt] over the topology's branches (removed ones 0),
    inj = [p | q] over the active buses, per unit.
    """
    import torch
    nf = sum(4 * p.topo.nbr for p in ev.plans)
    ni = sum(2 * p.topo.nb for p in ev.plans)
    dev = torch.device("cuda", ev.device)
    flows = torch.zeros(max(nf, 1), dtype=torch.float64, device=dev)
    inj = torch.zeros(max(ni, 1), dtype=torch.float64, device=dev)
    st = ev.stream_handle(stream)        # torch's current stream unless given: ordered with the zero-fills
    L.check(L.lib().acopf_batch_flows(ev._h, ctypes.c_void_p(x_dev.data_ptr()),
                                      ctypes.c_void_p(flows.data_ptr()), ctypes.c_void_p(inj.data_ptr()), st))
    return flows, inj


def _host_flows(ev: BatchEvaluator, x: np.ndarray):
    """device_flows from a host point; returns per-stage host views."""
    import torch
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(torch.device("cuda", ev.device))
    flows, inj = device_flows(ev, xd)
    flows, inj = flows.cpu().numpy(), inj.cpu().numpy()
    out, fo, io = [], 0, 0
    for p in ev.plans:
        nbr, nb = p.topo.nbr, p.topo.nb
        out.append((flows[fo:fo + 4 * nbr].reshape(4, nbr), inj[io:io + 2 * nb].reshape(2, nb)))
        fo += 4 * nbr
        io += 2 * nb
    return out


_SINGLE_CACHE: "dict" = {}


def _single(case):
    """(PackedCase, Topology, one-stage evaluator) of a case, as _Engine(case) (acopf.py:77-149).

    Cached per case object (cases are frozen dataclasses): repeated extract_solution /
    residuals_at calls on one case reuse the packing, the planner's tables and the device
    upload instead of rebuilding them (a few most recent cases are kept)."""
    key = id(case)
    hit = _SINGLE_CACHE.get(key)
    if hit is not None and hit[0] is case:
        return hit[1]
    pc = PackedCase(case)
    topo = Topology(pc)
    ev = BatchEvaluator([stage_plan(topo)], layout="independent")
    if len(_SINGLE_CACHE) >= 8:
        _SINGLE_CACHE.pop(next(iter(_SINGLE_CACHE)))
    _SINGLE_CACHE[key] = (case, (pc, topo, ev))
    return pc, topo, ev


def _flows_mw(case, topo, removed, fl, base):
    """_branch_flows_mw (acopf.py:448-464): pu flows of the live branches x base, zeros elsewhere."""
    nbrs = len(case.branches)
    pf, qf, pt, qt = (np.zeros(nbrs) for _ in range(4))
    keep = np.ones(topo.nbr, dtype=bool)
    keep[np.asarray(removed, dtype=np.int64)] = False
    if keep.any():
        live = topo.live_br[keep]
        pf[live] = fl[0][keep] * base
        qf[live] = fl[1][keep] * base
        pt[live] = fl[2][keep] * base
        qt[live] = fl[3][keep] * base
    return pf, qf, pt, qt


def _unpack(case, layout, x):
    nb_all, ng_all = len(case.buses), len(case.gens)
    vm = np.zeros(nb_all)
    va = np.zeros(nb_all)
    if layout.va:
        pos = np.fromiter(layout.va.keys(), dtype=np.int64, count=len(layout.va))
        va[pos] = x[np.fromiter(layout.va.values(), dtype=np.int64, count=len(pos))]
        vm[pos] = x[np.array([layout.vm[p] for p in pos.tolist()], dtype=np.int64)]
    pg = np.zeros(ng_all)
    qg = np.zeros(ng_all)
    if layout.pg:
        gpos = np.fromiter(layout.pg.keys(), dtype=np.int64, count=len(layout.pg))
        pg[gpos] = x[np.fromiter(layout.pg.values(), dtype=np.int64, count=len(gpos))] * case.base_mva
        qg[gpos] = x[np.array([layout.qg[g] for g in gpos.tolist()], dtype=np.int64)] * case.base_mva
    return vm, va, pg, qg


def _objective(case, gens, pg):
    """$/h in generator order, Python's builtin sum (acopf.py:486, 513)."""
    return float(sum(case.gens[g].cost.at(pg[g]) for g in gens))


def _stage_x(topo, va, vm):
    """A stage point carrying the given voltages (dispatch zero: flows ignore it)."""
    x = np.zeros(topo.n)
    act = topo.pc.active
    x[:topo.nb] = va[act]
    x[topo.nb:2 * topo.nb] = vm[act]
    return x


def extract_solution(case, layout, x) -> SolvedCase:
    """Unpack an NLP point into a SolvedCase with computed line flows (acopf.py:467-488)."""
    x = np.asarray(x)
    if x.shape != (layout.n_vars,):
        raise DimensionMismatch(f"x has shape {x.shape}, layout expects ({layout.n_vars},)")
    pc, topo, ev = _single(case)
    vm, va, pg, qg = _unpack(case, layout, x)
    flows = (np.zeros(len(case.branches)),) * 4
    if topo.nbr:
        (fl, _), = _host_flows(ev, _stage_x(topo, va, vm))
        flows = _flows_mw(case, topo, (), fl, pc.base)
    return SolvedCase(case=case, vm=vm, va=va, pg=pg, qg=qg, pf=flows[0], qf=flows[1], pt=flows[2],
                      qt=flows[3], objective=_objective(case, layout.pg, pg))


def pack_solution(case, layout, sol: SolvedCase) -> np.ndarray:
    """Inverse of extract_solution, flows ignored (acopf.py:491-501)."""
    x = np.zeros(layout.n_vars)
    for pos, idx in layout.va.items():
        x[idx] = sol.va[pos]
        x[layout.vm[pos]] = sol.vm[pos]
    for gpos, idx in layout.pg.items():
        x[idx] = sol.pg[gpos] / case.base_mva
        x[layout.qg[gpos]] = sol.qg[gpos] / case.base_mva
    return x


def solution_from_case(case) -> SolvedCase:
    """The case's stored voltages and dispatch as a solution (acopf.py:504-515)."""
    pc, topo, ev = _single(case)
    vm = np.array([b.vm for b in case.buses], dtype=np.float64)
    va = np.array([b.va for b in case.buses], dtype=np.float64)
    pg = np.array([g.pg if g.status else 0.0 for g in case.gens], dtype=np.float64)
    qg = np.array([g.qg if g.status else 0.0 for g in case.gens], dtype=np.float64)
    flows = (np.zeros(len(case.branches)),) * 4
    if topo.nbr:
        (fl, _), = _host_flows(ev, _stage_x(topo, va, vm))
        flows = _flows_mw(case, topo, (), fl, pc.base)
    live = [j for j, g in enumerate(case.gens) if g.status]
    return SolvedCase(case=case, vm=vm, va=va, pg=pg, qg=qg, pf=flows[0], qf=flows[1], pt=flows[2],
                      qt=flows[3], objective=_objective(case, live, pg))


def residuals_at(case, sol: SolvedCase):
    """Per-bus balance residuals, generation - load - injection (acopf.py:518-546)."""
    for attr, count in (("vm", len(case.buses)), ("pg", len(case.gens))):
        if np.shape(getattr(sol, attr)) != (count,):
            raise DimensionMismatch(f"solution {attr} has wrong length")
    pc, topo, ev = _single(case)
    nb_all = len(case.buses)
    dp, dq = np.zeros(nb_all), np.zeros(nb_all)
    if topo.nb == 0:
        return dp, dq
    (_, inj), = _host_flows(ev, _stage_x(topo, np.asarray(sol.va, dtype=np.float64),
                                         np.asarray(sol.vm, dtype=np.float64)))
    base = pc.base
    act = pc.active
    dp_s = -inj[0] * base
    dq_s = -inj[1] * base
    dp_s -= np.array([case.buses[p].pd for p in act], dtype=np.float64)
    dq_s -= np.array([case.buses[p].qd for p in act], dtype=np.float64)
    # generators in case order, one at a time (np.add.at is sequential)
    np.add.at(dp_s, topo.gbus, np.asarray(sol.pg, dtype=np.float64)[topo.live_gens])
    np.add.at(dq_s, topo.gbus, np.asarray(sol.qg, dtype=np.float64)[topo.live_gens])
    dp[act] = dp_s
    dq[act] = dq_s
    return dp, dq


def extract_solutions(problem, imap, x) -> list:
    """extract_solution for every stage of a composite, flows from one device launch.

    ``problem`` / ``imap`` come from a ``compose_*`` builder of this package;
    stage k's result equals ``extract_solution(imap.stages[k].case,
    imap.layouts[k], x[var_offset[k]:var_offset[k] + n_k])``.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (imap.n_vars,):
        raise DimensionMismatch(f"x has shape {x.shape}, composite expects ({imap.n_vars},)")
    ev = problem.evaluator
    per_stage = _host_flows(ev, _full_x(ev, x))
    out = []
    for k, plan in enumerate(ev.plans):
        case, layout = imap.stages[k].case, imap.layouts[k]
        o = imap.var_offset[k]
        xk = x[o:o + layout.n_vars]
        vm, va, pg, qg = _unpack(case, layout, xk)
        fl = per_stage[k][0]
        flows = _flows_mw(case, plan.topo, plan.removed, fl, plan.topo.pc.base)
        out.append(SolvedCase(case=case, vm=vm, va=va, pg=pg, qg=qg, pf=flows[0], qf=flows[1],
                              pt=flows[2], qt=flows[3], objective=_objective(case, layout.pg, pg)))
    return out


def _full_x(ev, x):
    """The evaluator's flat x (composite x, padded when the layout carries a halo)."""
    if len(x) == ev.n:
        return x
    buf = np.zeros(ev.n)
    buf[:len(x)] = x
    return buf
