"""Device-resident batched evaluation of ACOPF callbacks over many stages.

A :class:`StagePlan` says what one stage is (topology, removed branches,
loads, costs, objective weight); :class:`BatchEvaluator` hands the plans to
the native planner (libacopf_b200.so), lays their outputs into flat buffers
and evaluates every stage in one kernel launch.

Two layouts:

* ``"composite"`` -- the reference's composite NLP ordering
  (`composer.py:206-242`): variables stage by stage; constraints
  ``[stage eq blocks | pins | stage ineq blocks | boxes]``; J/H values in
  the composite CSR's order; weighted objective summed in stage order.
* ``"independent"`` -- every stage is its own NLP (stage-contiguous
  ``[eq; ineq]`` blocks and CSR values), objective per stage.  This is how
  many evaluation points of one network are batched (BASELINE config 1).

Device buffers are torch tensors on ``cuda:<device>`` (PyTorch is only the
allocator/stream plumbing; all arithmetic happens in the CUDA kernel).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass
class StagePlan:
    topo: object                      # packer.Topology
    removed: np.ndarray               # topology-local branch ids removed in this stage
    pd: np.ndarray                    # per-unit loads of the active buses
    qd: np.ndarray
    load_key: object                  # stages with equal keys share one load set
    cost_key: object = None           # stages with equal keys share one cost set (None: topology's)
    ca: np.ndarray | None = None
    cb: np.ndarray | None = None
    cc: np.ndarray | None = None
    weight: float = 1.0


@dataclass
class Coupling:
    """Coupling rows in flat-buffer coordinates (composer.py:229-242)."""
    row: np.ndarray                   # cons row
    col_a: np.ndarray                 # x index of the child quantity
    col_b: np.ndarray                 # x index of the base quantity (may point into a halo)
    base_first: np.ndarray | None = None   # base column sorts first (default: col_b < col_a)


class BatchEvaluator:
    def __init__(self, plans, *, device: int = 0, layout: str = "independent",
                 coupling: Coupling | None = None, n_pins: int = 0, obj_terms: bool = False):
        if layout not in ("independent", "composite"):
            raise ValueError("layout must be 'independent' or 'composite'")
        self.plans = list(plans)
        self.device = int(device)
        self.layout = layout
        lib = L.lib()
        topos = []
        tindex = {}
        for p in self.plans:
            if id(p.topo) not in tindex:
                tindex[id(p.topo)] = len(topos)
                topos.append(p.topo)
        self.topos = topos
        S = len(self.plans)
        stage_topo = L.i32([tindex[id(p.topo)] for p in self.plans])
        rem_ptr = np.zeros(S + 1, dtype=np.int64)
        rems = []
        for s, p in enumerate(self.plans):
            r = np.asarray(p.removed, dtype=np.int32)
            rems.append(r)
            rem_ptr[s + 1] = rem_ptr[s] + len(r)
        rem_idx = L.i32(np.concatenate(rems) if rems and rem_ptr[-1] else np.zeros(1))
        # load and cost sets (deduplicated by key)
        load_sets, load_of, lkeys = [], [], {}
        cost_sets, cost_of, ckeys = [], [], {}
        for p in self.plans:
            lk = (id(p.topo), p.load_key)
            if lk not in lkeys:
                lkeys[lk] = len(load_sets)
                load_sets.append((L.f64(p.pd), L.f64(p.qd)))
            load_of.append(lkeys[lk])
            ck = (id(p.topo), p.cost_key)
            if ck not in ckeys:
                ckeys[ck] = len(cost_sets)
                if p.ca is None:
                    cost_sets.append((p.topo.ca, p.topo.cb, p.topo.cc))
                else:
                    cost_sets.append((p.ca, p.cb, p.cc))
            cost_of.append(ckeys[ck])
        load_off = np.zeros(len(load_sets) + 1, dtype=np.int64)
        for i, (a, _) in enumerate(load_sets):
            load_off[i + 1] = load_off[i] + len(a)
        pd_all = L.f64(np.concatenate([a for a, _ in load_sets] + [np.zeros(1)]))
        qd_all = L.f64(np.concatenate([b for _, b in load_sets] + [np.zeros(1)]))
        cost_off = np.zeros(len(cost_sets) + 1, dtype=np.int64)
        for i, c in enumerate(cost_sets):
            cost_off[i + 1] = cost_off[i] + len(c[0])
        ca_all = L.f64(np.concatenate([c[0] for c in cost_sets] + [np.zeros(1)]))
        cb_all = L.f64(np.concatenate([c[1] for c in cost_sets] + [np.zeros(1)]))
        cc_all = L.f64(np.concatenate([c[2] for c in cost_sets] + [np.zeros(1)]))
        weights = L.f64([p.weight for p in self.plans])
        handles = (ctypes.c_void_p * max(len(topos), 1))(*[t.handle() for t in topos])
        h = ctypes.c_void_p()
        stage_load, stage_cost = L.i32(load_of), L.i32(cost_of)
        L.check(lib.acopf_batch_create(
            self.device, len(topos), handles, S, L.ptr(stage_topo, ctypes.c_int32),
            L.ptr(rem_ptr, ctypes.c_int64), L.ptr(rem_idx, ctypes.c_int32),
            L.ptr(stage_load, ctypes.c_int32), L.ptr(load_off, ctypes.c_int64), int(load_off[-1]),
            L.ptr(pd_all, ctypes.c_double), L.ptr(qd_all, ctypes.c_double),
            L.ptr(stage_cost, ctypes.c_int32), L.ptr(cost_off, ctypes.c_int64), int(cost_off[-1]),
            L.ptr(ca_all, ctypes.c_double), L.ptr(cb_all, ctypes.c_double), L.ptr(cc_all, ctypes.c_double),
            L.ptr(weights, ctypes.c_double), ctypes.byref(h)))
        self._h = h
        sizes = np.zeros((S, 6), dtype=np.int64)
        L.check(lib.acopf_batch_stage_sizes(h, L.ptr(sizes, ctypes.c_int64)))
        self.sizes = sizes
        self.obj_terms = obj_terms
        self._layout(coupling, n_pins)

    # -- layout ---------------------------------------------------------------

    def _layout(self, coupling, n_pins):
        sz = self.sizes
        S = len(self.plans)
        n, meq, mineq, jeq, jin, hnz = (sz[:, i] for i in range(6))

        def prefix(a):
            out = np.zeros(len(a) + 1, dtype=np.int64)
            np.cumsum(a, out=out[1:])
            return out

        var_off = prefix(n)
        self.n = int(var_off[-1])
        h_base = prefix(hnz)
        self.nnz_h = int(h_base[-1])
        ncp = 0 if coupling is None else len(coupling.row)
        if self.layout == "independent":
            m = meq + mineq
            row0 = prefix(m)
            eq_row, ineq_row = row0[:-1], row0[:-1] + meq
            jnz = prefix(jeq + jin)
            jeq_base, jin_base = jnz[:-1], jnz[:-1] + jeq
            self.m_eq = int(meq.sum())
            self.m_ineq = int(mineq.sum())
            self.m = int(row0[-1])
            self.nnz_j = int(jnz[-1])
            obj_mode, obj_slot, self.n_obj = L.OBJ_PER_STAGE, np.arange(S), S
            cp = None
        else:
            me_st, mi_st = int(meq.sum()), int(mineq.sum())
            n_box = ncp - n_pins
            self.m_eq = me_st + n_pins
            self.m_ineq = mi_st + n_box
            self.m = self.m_eq + self.m_ineq
            eq_row = prefix(meq)[:-1]
            ineq_row = self.m_eq + prefix(mineq)[:-1]
            jeq_all = int(jeq.sum())
            jeq_base = prefix(jeq)[:-1]
            jin_base = jeq_all + 2 * n_pins + prefix(jin)[:-1]
            self.nnz_j = jeq_all + 2 * n_pins + int(jin.sum()) + 2 * n_box
            if self.obj_terms:
                obj_mode, obj_slot, self.n_obj = L.OBJ_TERMS, np.arange(S), S
            else:
                obj_mode, obj_slot, self.n_obj = L.OBJ_WEIGHTED, np.arange(S), 1
            cp = coupling
        self.var_off = var_off[:-1]
        self.eq_row, self.ineq_row = np.asarray(eq_row), np.asarray(ineq_row)
        self.jeq_base, self.jin_base, self.h_base = np.asarray(jeq_base), np.asarray(jin_base), h_base[:-1]
        off6 = L.i64(np.stack([self.var_off, self.eq_row, self.ineq_row,
                               self.jeq_base, self.jin_base, self.h_base], axis=1))
        if cp is not None and ncp:
            rows = L.i64(cp.row)
            # J position of a coupling row: pins follow the eq blocks, boxes the ineq blocks
            me_st = int(meq.sum())
            jpos = 2 * rows
            jpos += np.where(rows < self.m_eq, int(jeq.sum()) - 2 * me_st,
                             int(jeq.sum()) + 2 * n_pins + int(jin.sum()) - 2 * (self.m_eq + int(mineq.sum())))
            ca, cb = L.i64(cp.col_a), L.i64(cp.col_b)
            first = np.ascontiguousarray(cb < ca if cp.base_first is None else cp.base_first, dtype=np.int8)
        else:
            rows = jpos = ca = cb = L.i64(np.zeros(1))
            first = np.zeros(1, dtype=np.int8)
            ncp = 0
        slots = L.i32(obj_slot)
        L.check(L.lib().acopf_batch_set_layout(
            self._h, L.ptr(off6, ctypes.c_int64), obj_mode, L.ptr(slots, ctypes.c_int32), ncp,
            L.ptr(rows, ctypes.c_int64), L.ptr(jpos, ctypes.c_int64), L.ptr(ca, ctypes.c_int64),
            L.ptr(cb, ctypes.c_int64), L.ptr(first, ctypes.c_int8)))
        # (the library keeps its own copies of the coupling arrays)

    # -- patterns ---------------------------------------------------------------

    def pattern(self, which: str, stage: int = -1):
        """(indptr int64, indices int32) of J ('J') or H ('H')."""
        w = 0 if which == "J" else 1
        if stage >= 0:
            n, meq, mineq = self.sizes[stage, :3]
            rows = int(meq + mineq) if w == 0 else int(n)
            nnz = int(self.sizes[stage, 3] + self.sizes[stage, 4]) if w == 0 else int(self.sizes[stage, 5])
        else:
            rows = self.m if w == 0 else self.n
            nnz = self.nnz_j if w == 0 else self.nnz_h
        indptr = np.zeros(rows + 1, dtype=np.int64)
        indices = np.zeros(max(nnz, 1), dtype=np.int32)
        L.check(L.lib().acopf_batch_pattern(self._h, int(stage), w, rows,
                                            L.ptr(indptr, ctypes.c_int64), L.ptr(indices, ctypes.c_int32)))
        return indptr, indices[:nnz]

    # -- evaluation ---------------------------------------------------------------

    def alloc(self, what: int = L.ALL):
        """Fresh torch output buffers on the device."""
        import torch
        dev = torch.device("cuda", self.device)
        mk = lambda k: torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        return dict(obj=mk(self.n_obj), grad=mk(self.n), cons=mk(self.m),
                    jac=mk(self.nnz_j), hess=mk(self.nnz_h))

    def stream_handle(self, stream=None) -> ctypes.c_void_p:
        """The cudaStream_t to launch on: ``stream`` (a raw handle or a torch stream), else
        torch's current stream on this device, so the kernels are ordered with the torch
        work that produced the inputs and that reads the outputs."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(torch.device("cuda", self.device))
        if hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        return ctypes.c_void_p(int(stream) or None)

    def eval_device(self, x, mult, obj_factor: float = 1.0, what: int = L.ALL, out=None, stream=None):
        """Evaluate with torch device tensors on ``stream`` (default: torch's current
        stream); returns the output dict."""
        out = out if out is not None else self.alloc(what)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        st = self.stream_handle(stream)
        L.check(L.lib().acopf_batch_eval(
            self._h, ptr(x), float(obj_factor), ptr(mult), int(what), ptr(out["obj"]), ptr(out["grad"]),
            ptr(out["cons"]), ptr(out["jac"]), ptr(out["hess"]), st))
        return out

    def eval_host(self, x: np.ndarray, mult: np.ndarray | None, obj_factor: float = 1.0,
                  what: int = L.ALL, out: dict | None = None) -> dict:
        """Evaluate from host numpy arrays (copies in and out, synchronises)."""
        x = L.f64(x)
        if x.shape != (self.n,):
            raise ValueError(f"x must have shape ({self.n},)")
        if mult is not None:
            mult = L.f64(mult)
            if mult.shape != (self.m,):
                raise ValueError(f"mult must have shape ({self.m},)")
        if out is None:
            out = {}
        def buf(key, k, bit):
            if not (what & bit):
                return None
            if key not in out or out[key].shape != (k,):
                out[key] = np.empty(k)
            return out[key]
        o = buf("obj", self.n_obj, L.OBJ)
        g = buf("grad", self.n, L.GRAD)
        c = buf("cons", self.m, L.CONS)
        j = buf("jac", self.nnz_j, L.JAC)
        h = buf("hess", self.nnz_h, L.HESS)
        vp = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a is not None else None
        sz = lambda a: 0 if a is None else len(a)
        L.check(L.lib().acopf_batch_eval_host(
            self._h, vp(x), len(x), float(obj_factor), vp(mult), sz(mult), int(what), vp(o), sz(o),
            vp(g), sz(g), vp(c), sz(c), vp(j), sz(j), vp(h), sz(h), None))
        return out

    def eval_host_ptrs(self, x_ptr: int, mult_ptr: int, obj_factor: float, what: int, outs: dict,
                       stream=None) -> None:
        """Host-buffer evaluation on raw pointers (pinned torch tensors in bench.py)."""
        v = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        n = lambda t: 0 if t is None else t.numel()
        L.check(L.lib().acopf_batch_eval_host(
            self._h, ctypes.c_void_p(x_ptr), self.n, float(obj_factor), ctypes.c_void_p(mult_ptr),
            self.m if mult_ptr else 0, int(what), v(outs.get("obj")), n(outs.get("obj")),
            v(outs.get("grad")), n(outs.get("grad")), v(outs.get("cons")), n(outs.get("cons")),
            v(outs.get("jac")), n(outs.get("jac")), v(outs.get("hess")), n(outs.get("hess")),
            ctypes.c_void_p(stream) if stream else None))

    def launches(self) -> int:
        return int(L.lib().acopf_batch_launches(self._h))

    def verify_plan(self) -> dict:
        """Host check of the tile tables' invariants (acopf_batch_verify); no GPU needed."""
        st = np.zeros(12, dtype=np.int64)
        L.check(L.lib().acopf_batch_verify(self._h, L.ptr(st, ctypes.c_int64)))
        keys = ("tables", "tiles", "ends", "area_doubles", "pad_slots", "max_smem_bytes",
                "sum_rounds", "round_lane_terms", "round_chain_terms", "store_wavefronts_half",
                "store_wavefronts_warp", "store_wavefronts_ideal")
        return dict(zip(keys, (int(v) for v in st)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None:
            try:
                L.lib().acopf_batch_destroy(h)
            except Exception:
                pass
