"""``build_acopf``: the reference's stage NLP, evaluated on the B200.

Drop-in for `pkg/src/opfkit/acopf.py:392-410`: same signature, returns a
plain :class:`NlpProblem` (mutable dataclass, same bounds/start point) and an
:class:`AcopfLayout` with identical maps.  The five callbacks copy the point
to the GPU, run the fused evaluation kernel for the requested outputs only,
and copy the result back; ``jacobian`` / ``lagrangian_hessian`` wrap the
values into scipy CSR matrices whose (fixed, canonical) pattern was computed
once by the native planner -- bit-identical to what scipy produces from the
reference's COO triplets.
"""

from __future__ import annotations

import threading

import numpy as np
import scipy.sparse as sp

from . import _lib as L
from .errors import Disconnected
from .evaluator import BatchEvaluator, StagePlan
from .grid import check_connectivity
from .packer import PackedCase, Topology
from .types import AcopfLayout, NlpProblem


def csr_index_arrays(indptr: np.ndarray, indices: np.ndarray):
    """scipy's index dtype choice: int32 unless the matrix needs int64."""
    if len(indices) < 2 ** 31 - 1 and (len(indptr) == 0 or indptr[-1] < 2 ** 31 - 1):
        return indptr.astype(np.int32), indices.astype(np.int32)
    return indptr, indices.astype(np.int64)


class CallbackSet:
    """The five NlpProblem callbacks over one BatchEvaluator (host buffers).

    Latency path (the reference's IPM calls one callback at a time, ipm.py:389-578): the
    point is copied into a persistent pinned buffer, every output is written by an
    asynchronous D2H copy straight into a FRESH pinned array from torch's caching host
    allocator (so each call returns new arrays the caller owns, as the reference does,
    without a pageable copy), and the C ABI call itself is one ctypes call
    (acopf_batch_eval_host: H2D, the requested kernels only, D2H, synchronise)."""

    def __init__(self, ev: BatchEvaluator, obj_index: int = 0):
        self.ev = ev
        self._lock = threading.Lock()
        self._jp = self._hp = None
        self.obj_index = obj_index
        self._pin_x = self._pin_m = None

    def _patterns(self, which):
        if which == "J":
            if self._jp is None:
                self._jp = csr_index_arrays(*self.ev.pattern("J"))
            return self._jp
        if self._hp is None:
            self._hp = csr_index_arrays(*self.ev.pattern("H"))
        return self._hp

    @staticmethod
    def _pinned(n):
        import torch
        return torch.empty(max(int(n), 1), dtype=torch.float64, pin_memory=True)

    def _eval(self, x, mult, of, what):
        """One evaluation of `what` (a single output) into a fresh pinned array."""
        import ctypes
        ev = self.ev
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (ev.n,):
            raise ValueError(f"x must have shape ({ev.n},)")
        with self._lock:
            if self._pin_x is None:
                self._pin_x = self._pinned(ev.n)
                self._pin_m = self._pinned(ev.m)
            px = self._pin_x.numpy()[:ev.n]
            np.copyto(px, x)
            pm = 0
            if mult is not None:
                mult = np.asarray(mult, dtype=np.float64)
                if mult.shape != (ev.m,):
                    raise ValueError(f"mult must have shape ({ev.m},)")
                np.copyto(self._pin_m.numpy()[:ev.m], mult)
                pm = self._pin_m.data_ptr()
            size = {L.OBJ: ev.n_obj, L.GRAD: ev.n, L.CONS: ev.m, L.JAC: ev.nnz_j, L.HESS: ev.nnz_h}[what]
            out = self._pinned(size)
            ptrs = [None] * 5
            ptrs[{L.OBJ: 0, L.GRAD: 1, L.CONS: 2, L.JAC: 3, L.HESS: 4}[what]] = out
            v = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
            nn = lambda t: 0 if t is None else size
            L.check(L.lib().acopf_batch_eval_host(
                ev._h, ctypes.c_void_p(self._pin_x.data_ptr()), ev.n, float(of), ctypes.c_void_p(pm or None),
                ev.m if pm else 0, int(what), v(ptrs[0]), nn(ptrs[0]), v(ptrs[1]), nn(ptrs[1]), v(ptrs[2]),
                nn(ptrs[2]), v(ptrs[3]), nn(ptrs[3]), v(ptrs[4]), nn(ptrs[4]), None))
            return out.numpy()[:size]

    def objective(self, x) -> float:
        return float(self._eval(x, None, 1.0, L.OBJ)[self.obj_index])

    def gradient(self, x) -> np.ndarray:
        return self._eval(x, None, 1.0, L.GRAD)

    def constraints(self, x) -> np.ndarray:
        return self._eval(x, None, 1.0, L.CONS)

    def jacobian(self, x) -> sp.csr_matrix:
        vals = self._eval(x, None, 1.0, L.JAC)
        indptr, indices = self._patterns("J")
        return sp.csr_matrix((vals, indices.copy(), indptr.copy()), shape=(self.ev.m, self.ev.n))

    def lagrangian_hessian(self, x, obj_factor, mult) -> sp.csr_matrix:
        mult = np.asarray(mult, dtype=np.float64)
        vals = self._eval(x, mult, float(obj_factor), L.HESS)
        indptr, indices = self._patterns("H")
        return sp.csr_matrix((vals, indices.copy(), indptr.copy()), shape=(self.ev.n, self.ev.n))


def stage_plan(topo: Topology, removed=(), weight: float = 1.0, load_key=0) -> StagePlan:
    pc = topo.pc
    return StagePlan(topo=topo, removed=np.asarray(removed, dtype=np.int32), pd=pc.pd, qd=pc.qd,
                     load_key=load_key, weight=weight)


def build_acopf(case, *, device: int = 0):
    """Build the stage NLP.  Returns (NlpProblem, AcopfLayout).

    Raises Disconnected when the in-service network is not one island
    (acopf.py:398-400) or a live branch touches an isolated bus (:97-99).
    """
    n_islands, _ = check_connectivity(case)
    if n_islands != 1:
        raise Disconnected(f"case {case.name!r} has {n_islands} islands")
    pc = PackedCase(case)
    topo = Topology(pc)
    ev = BatchEvaluator([stage_plan(topo)], device=device, layout="independent")
    cb = CallbackSet(ev)
    xl, xu, x0 = topo.bounds()
    gl, gu = topo.ineq_bounds()
    maps = topo.layout_maps()
    layout = AcopfLayout(n_vars=ev.n, n_eq=ev.m_eq, n_ineq=ev.m_ineq, **maps)
    problem = NlpProblem(n=ev.n, m_eq=ev.m_eq, m_ineq=ev.m_ineq, xl=xl, xu=xu, gl=gl, gu=gu, x0=x0,
                         objective=cb.objective, gradient=cb.gradient, constraints=cb.constraints,
                         jacobian=cb.jacobian, lagrangian_hessian=cb.lagrangian_hessian,
                         name=f"acopf:{case.name}")
    problem.evaluator = ev          # device-resident batched entry point (not a reference field)
    return problem, layout
