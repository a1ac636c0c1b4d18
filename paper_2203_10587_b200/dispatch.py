"""Multi-GPU dispatcher: one composite sharded over ranks.

One process per GPU (torch.distributed, NCCL over NVLink on B200; gloo in the
CPU tests).  Rank r owns a contiguous block of stages -- scenario-major for
the stochastic composites, so contingency rows stay rank-local -- and builds
the native evaluator for its stages only.  Its flat buffers hold, in the
global order, its stage variables (plus a halo), its constraint rows
``[eq blocks | pins | ineq blocks | boxes]`` and the matching J / H values.

Collectives (the only data exchanged; both inside the C ABI's
``acopf_batch_eval_multi``, NCCL over NVLink):

* halo: coupling rows ``x[child] - x[base]`` whose base stage lives on another
  rank read the base values from a halo filled by one ``ncclAllGather`` of
  each rank's exported values (base-stage Pg / VM; a period neighbour's Pg),
  packed and unpacked by the library's kernels on a stream beside the tile
  kernel;
* objective: every rank writes its per-stage ``w_s f_s`` (ACOPF_OBJ_TERMS);
  the terms are all-gathered and summed in global stage order on the device,
  which keeps the composite objective bit-identical to the single-GPU
  evaluation (composer.py:256-258 sums left to right).
"""

from __future__ import annotations

import numpy as np

from .evaluator import BatchEvaluator, Coupling


def partition_stages(spec, world: int, align=None) -> list:
    """Contiguous stage blocks balanced by variable count.

    ``align``: optional per-stage group ids (e.g. scenario index); block
    boundaries are placed on group boundaries when there are enough groups.
    """
    S = len(spec.plans)
    w = np.asarray(spec.n_s, dtype=np.float64)
    cut_ok = np.ones(S + 1, dtype=bool)
    if align is not None and len(set(align)) >= world:
        a = np.asarray(align)
        cut_ok[1:S] = a[1:] != a[:-1]
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        cands = np.flatnonzero(cut_ok)
        cands = cands[(cands > cuts[-1]) & (cands < S)]
        if len(cands) == 0:
            cuts.append(cuts[-1])
            continue
        cuts.append(int(cands[np.argmin(np.abs(cum[cands] - target))]))
    cuts.append(S)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


class ShardPlan:
    """Host-side bookkeeping of one rank's share of a composite (no device work)."""

    def __init__(self, spec, rank: int, world: int, align=None):
        self.spec, self.rank, self.world = spec, rank, world
        self.blocks = partition_stages(spec, world, align)
        s0, s1 = self.blocks[rank]
        self.s0, self.s1 = s0, s1
        S = len(spec.plans)
        var_end = np.concatenate([spec.var_off, [int(spec.n_s.sum())]])
        self.x_lo, self.x_hi = int(var_end[s0]), int(var_end[s1])
        self.var_end = var_end
        cp = spec.cp
        me_st = int(spec.meq_s.sum())
        mi_st = int(spec.mineq_s.sum())
        self.me_st, self.mi_st = me_st, mi_st
        mine = (cp["stage_a"] >= s0) & (cp["stage_a"] < s1)
        rows = cp["row"][mine]
        is_pin = rows < spec.m_eq
        pin_idx = rows[is_pin] - me_st
        box_idx = rows[~is_pin] - spec.m_eq - mi_st
        for idx in (pin_idx, box_idx):
            if len(idx) and not np.array_equal(idx, np.arange(idx[0], idx[0] + len(idx))):
                raise NotImplementedError("this lattice's coupling rows are not contiguous per rank")
        self.pin_lo = int(pin_idx[0]) if len(pin_idx) else 0
        self.box_lo = int(box_idx[0]) if len(box_idx) else 0
        self.n_pins, self.n_box = int(len(pin_idx)), int(len(box_idx))
        self.me_loc = int(spec.meq_s[s0:s1].sum())
        self.mi_loc = int(spec.mineq_s[s0:s1].sum())
        self.n_loc = self.x_hi - self.x_lo
        self.m_eq_loc = self.me_loc + self.n_pins
        # local coupling rows and columns (base values outside the block -> halo)
        col_a, col_b = cp["col_a"][mine], cp["col_b"][mine]
        remote = (col_b < self.x_lo) | (col_b >= self.x_hi)
        self.halo_idx = np.unique(col_b[remote])              # global x indices this rank imports
        loc_b = col_b - self.x_lo
        loc_b[remote] = self.n_loc + np.searchsorted(self.halo_idx, col_b[remote])
        loc_rows = np.empty(len(rows), dtype=np.int64)
        loc_rows[is_pin] = self.me_loc + (pin_idx - self.pin_lo)
        loc_rows[~is_pin] = self.m_eq_loc + self.mi_loc + (box_idx - self.box_lo)
        self.coupling = Coupling(row=loc_rows, col_a=col_a - self.x_lo, col_b=loc_b,
                                 base_first=col_b < col_a)

    def owner(self, g: np.ndarray) -> np.ndarray:
        """Rank owning global x index g."""
        starts = np.array([self.var_end[a] for a, _ in self.blocks])
        return np.searchsorted(starts, g, side="right") - 1


class ShardedComposite:
    """One rank's evaluator for a sharded composite.

    ``dist`` is ``torch.distributed`` (initialised); tensors live on
    ``device``.  The exchange runs inside the C ABI: ``acopf_multi_create``
    computes the plan (exports, halo positions, objective counts) from every
    rank's halo needs and makes the NCCL communicator (its id is made by rank 0
    and broadcast through ``dist``); ``acopf_batch_eval_multi`` runs the halo
    pack -> ncclAllGather -> unpack -> coupling-row chain on a forked stream
    beside the tile kernel and sums every rank's objective terms in stage order
    on the device.  ``local_eval`` (CPU tests, gloo) replaces the device
    evaluation: the native plan is then executed by this class's emulation of
    the same exchange over ``dist``.
    """

    def __init__(self, spec, dist, rank: int, world: int, device="cuda", align=None, local_eval=None):
        import ctypes
        import torch
        from . import _lib as L
        self.torch, self.dist, self.L = torch, dist, L
        self.plan = plan = ShardPlan(spec, rank, world, align)
        self.device = torch.device(device)
        dev_index = self.device.index or 0
        self.ev = BatchEvaluator(spec.plans[plan.s0:plan.s1], device=dev_index, layout="composite",
                                 coupling=plan.coupling, n_pins=plan.n_pins, obj_terms=True)
        assert self.ev.n == plan.n_loc and self.ev.m_eq == plan.m_eq_loc
        self.local_eval = local_eval
        # every rank's halo needs, x range and stage count (host exchange, once)
        info = [None] * world
        dist.all_gather_object(info, (plan.halo_idx.tolist(), plan.x_lo, plan.x_hi, plan.s1 - plan.s0))
        need_ptr = np.zeros(world + 1, dtype=np.int64)
        for r, (nd, _, _, _) in enumerate(info):
            need_ptr[r + 1] = need_ptr[r] + len(nd)
        need_idx = L.i64(np.concatenate([np.asarray(nd, dtype=np.int64) for nd, _, _, _ in info] + [np.zeros(1)]))
        x_lo = L.i64([a for _, a, _, _ in info])
        x_hi = L.i64([b for _, _, b, _ in info])
        self.obj_counts = counts = L.i32([c for _, _, _, c in info])
        nccl_id = None
        if local_eval is None and self.device.type == "cuda":
            idbuf = ctypes.create_string_buffer(128)
            if rank == 0:
                L.check(L.lib().acopf_nccl_unique_id(idbuf))
            box = [idbuf.raw if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            idbuf = ctypes.create_string_buffer(box[0], 128)
            nccl_id = idbuf
        h = ctypes.c_void_p()
        L.check(L.lib().acopf_multi_create(self.ev._h, rank, world, L.ptr(x_lo, ctypes.c_int64),
                                           L.ptr(x_hi, ctypes.c_int64), L.ptr(need_ptr, ctypes.c_int64),
                                           L.ptr(need_idx, ctypes.c_int64), plan.n_loc,
                                           L.ptr(counts, ctypes.c_int32), nccl_id, ctypes.byref(h)))
        self._m = h
        sizes = np.zeros(3, dtype=np.int64)
        L.check(L.lib().acopf_multi_plan(h, L.ptr(sizes, ctypes.c_int64), None, None))
        exp_idx = np.zeros(max(int(sizes[0]), 1), dtype=np.int64)
        halo_src = np.zeros(max(int(sizes[2]), 1), dtype=np.int64)
        L.check(L.lib().acopf_multi_plan(h, None, L.ptr(exp_idx, ctypes.c_int64), L.ptr(halo_src, ctypes.c_int64)))
        self.export_local = exp_idx[:int(sizes[0])]
        self.export_max = int(sizes[1])
        self.halo_src = halo_src[:int(sizes[2])]
        self.obj_max = max(int(counts.max()), 1)
        self.n_x = plan.n_loc + len(plan.halo_idx)
        self._obj = None

    def launches(self) -> int:
        return self.ev.launches()

    # -- buffers -----------------------------------------------------------------

    def alloc_x(self):
        return self.torch.zeros(max(self.n_x, 1), dtype=self.torch.float64, device=self.device)

    def evaluate(self, x, mult, obj_factor: float = 1.0, what: int = 31, out=None, stream=None):
        """One sharded evaluation.  Returns (out, objective): the objective is a 1-element
        tensor on the device (no host synchronisation), None unless OBJ is requested."""
        import ctypes
        L = self.L
        if self.local_eval is not None:
            return self._emulated(x, mult, obj_factor, what)
        out = out if out is not None else self.ev.alloc(what)
        if self._obj is None:
            self._obj = self.torch.zeros(1, dtype=self.torch.float64, device=self.device)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        L.check(L.lib().acopf_batch_eval_multi(
            self._m, ptr(x), float(obj_factor), ptr(mult), int(what), ptr(self._obj), ptr(out["grad"]),
            ptr(out["cons"]), ptr(out["jac"]), ptr(out["hess"]), self.ev.stream_handle(stream)))
        return out, (self._obj if what & L.OBJ else None)

    # -- CPU emulation of the native exchange (tests over gloo) ----------------------

    def _emulated(self, x, mult, obj_factor, what):
        torch, L = self.torch, self.L
        world = self.plan.world
        if what & (L.CONS | L.JAC):
            send = torch.zeros(self.export_max, dtype=torch.float64, device=self.device)
            if len(self.export_local):
                send[:len(self.export_local)] = x[torch.as_tensor(self.export_local)]
            recv = torch.empty(world * self.export_max, dtype=torch.float64, device=self.device)
            self.dist.all_gather_into_tensor(recv, send)
            if len(self.halo_src):
                x[self.plan.n_loc:self.n_x] = recv[torch.as_tensor(self.halo_src)]
        out = self.local_eval(x, mult, obj_factor, what)
        obj = None
        if what & L.OBJ:
            buf = torch.zeros(self.obj_max, dtype=torch.float64, device=self.device)
            terms = out["obj"][:self.plan.s1 - self.plan.s0]
            buf[:len(terms)] = terms
            allt = torch.empty(world * self.obj_max, dtype=torch.float64, device=self.device)
            self.dist.all_gather_into_tensor(allt, buf)
            host = allt.cpu().numpy().reshape(world, self.obj_max)
            acc = 0.0
            for r, c in enumerate(self.obj_counts):            # acopf_objsum_multi_kernel's order
                for v in host[r, :c]:
                    acc = acc + float(v)
            obj = torch.tensor([acc], dtype=torch.float64)
        return out, obj

    def __del__(self):
        h = getattr(self, "_m", None)
        if h is not None:
            try:
                self.L.lib().acopf_multi_destroy(h)
            except Exception:
                pass

    # -- placing local results in the global vectors (tests, drop-in API) -----------

    def global_ranges(self, all_sizes):
        """(x, cons, jac, hess) lists of (global_start, local_start, length) for this rank.

        all_sizes: per-stage (n, m_eq, m_ineq, nnz_jeq, nnz_jin, nnz_h) of the whole composite.
        """
        p, spec = self.plan, self.plan.spec
        sz = np.asarray(all_sizes)
        s0, s1 = p.s0, p.s1
        pre = lambda a, k: int(a[:k].sum())
        jeq_all, jin_all = int(sz[:, 3].sum()), int(sz[:, 4].sum())
        n_pins_all = int(np.count_nonzero(spec.cp["row"] < spec.m_eq))
        loc_jeq = int(sz[s0:s1, 3].sum())
        loc_jin = int(sz[s0:s1, 4].sum())
        x = [(p.x_lo, 0, p.n_loc)]
        cons = [(pre(spec.meq_s, s0), 0, p.me_loc),
                (p.me_st + p.pin_lo, p.me_loc, p.n_pins),
                (spec.m_eq + pre(spec.mineq_s, s0), p.m_eq_loc, p.mi_loc),
                (spec.m_eq + p.mi_st + p.box_lo, p.m_eq_loc + p.mi_loc, p.n_box)]
        jac = [(pre(sz[:, 3], s0), 0, loc_jeq),
               (jeq_all + 2 * p.pin_lo, loc_jeq, 2 * p.n_pins),
               (jeq_all + 2 * n_pins_all + pre(sz[:, 4], s0), loc_jeq + 2 * p.n_pins, loc_jin),
               (jeq_all + 2 * n_pins_all + jin_all + 2 * p.box_lo, loc_jeq + 2 * p.n_pins + loc_jin, 2 * p.n_box)]
        hess = [(pre(sz[:, 5], s0), 0, int(sz[s0:s1, 5].sum()))]
        return dict(x=x, grad=x, cons=cons, jac=jac, hess=hess)
