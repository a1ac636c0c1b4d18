"""Sharded composites across ranks (world_size 2, gloo, CPU).

The device evaluation is replaced by the oracle (test-only); everything else
is the product path: stage partition, each rank's native planner (host side),
the exchange plan computed by the C ABI (acopf_multi_create, plan-only
handle: exports, halo positions, objective counts), executed over gloo by
ShardedComposite's emulation of acopf_batch_eval_multi's exchange, the ordered
objective combination, and the local -> global range mapping, which is
checked against the oracle's global CSR patterns.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import common as C


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    from paper_2203_10587_b200 import synthetic as syn
    from paper_2203_10587_b200.lattice import composite_spec
    from paper_2203_10587_b200.types import CouplingMode
    from oracle.composite import CompositeOracle
    base, ctgs = syn.config2_inputs(n_ctg=7, nb=40, n_chords=12, ng=8, features=True)
    yield "scopf", composite_spec("scopf", base, ctgs, CouplingMode()), \
        CompositeOracle.general(None, ctgs, [base], CouplingMode(), 30.0), None
    periods = syn.config3_periods(6, nb=30, n_chords=8, ng=6)
    yield "multiperiod", composite_spec("multiperiod", periods, 15.0), \
        CompositeOracle.general(None, None, periods, CouplingMode(), 15.0), None
    base, scens, ctgs = syn.config4_inputs(n_scen=4, n_ctg=2, nb=30, n_chords=8, ng=10)
    mode = CouplingMode(kind="preventive", pin_voltages=True)
    spec = composite_spec("general", scens, ctgs, [base], mode, 30.0)
    align = [k // 3 for k in range(len(spec.plans))]          # scenario of each stage
    yield "general", spec, CompositeOracle.general(scens, ctgs, [base], mode, 30.0), align


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_10587_b200 import synthetic as syn
    from paper_2203_10587_b200.dispatch import ShardedComposite
    out = {}
    for name, spec, o, align in _cases():
        kinds = syn.variable_kinds(spec.stage_dims)
        x, mult = syn.random_point(kinds, o.xl, o.xu, o.m_eq + o.m_ineq, 17)
        g_cons, g_grad = o.constraints(x), o.gradient(x)
        J, H = o.jacobian(x), o.lagrangian_hessian(x, 0.8, mult)

        holder = {}

        def local_eval(xl, ml, of, what):
            sc = holder["sc"]
            rg = sc.global_ranges(holder["sizes"])
            def take(vec, ranges):
                n = sum(ln for _, _, ln in ranges)
                loc = np.zeros(n)
                for g0, l0, ln in ranges:
                    loc[l0:l0 + ln] = vec[g0:g0 + ln]
                return loc
            cons = take(g_cons, rg["cons"])
            cp = sc.plan.coupling
            xs = xl.numpy()
            cons[cp.row] = xs[cp.col_a] - xs[cp.col_b]            # from the exchanged halo
            p = sc.plan
            terms = [o.w[k] * o.stage[k].objective(x[o.slices[k][0]:o.slices[k][1]])
                     for k in range(p.s0, p.s1)]
            return dict(obj=torch.tensor(terms, dtype=torch.float64), grad=take(g_grad, rg["grad"]), cons=cons,
                        jac=take(J.data, rg["jac"]), hess=take(H.data, rg["hess"]))

        sc = ShardedComposite(spec, dist, rank, world, device="cpu", align=align, local_eval=local_eval)
        holder["sc"] = sc
        sizes = [None] * world
        dist.all_gather_object(sizes, sc.ev.sizes.tolist())
        holder["sizes"] = [row for part in sizes for row in part]
        xl = sc.alloc_x()
        xl[:sc.plan.n_loc] = torch.from_numpy(x[sc.plan.x_lo:sc.plan.x_hi])
        res, obj = sc.evaluate(xl, None, 0.8, 31)
        rg = sc.global_ranges(holder["sizes"])
        # local planner patterns placed at the global ranges == oracle's global patterns
        lj_ptr, lj_idx = sc.ev.pattern("J")
        lh_ptr, lh_idx = sc.ev.pattern("H")
        g0, l0, ln = rg["jac"][0]
        ok_j = np.array_equal(lj_idx[l0:l0 + ln] + sc.plan.x_lo, J.indices[g0:g0 + ln])
        g0, l0, ln = rg["jac"][2]
        ok_j &= np.array_equal(lj_idx[l0:l0 + ln] + sc.plan.x_lo, J.indices[g0:g0 + ln])
        g0, l0, ln = rg["hess"][0]
        ok_h = np.array_equal(lh_idx[l0:l0 + ln] + sc.plan.x_lo, H.indices[g0:g0 + ln])
        parts = [None] * world
        dist.all_gather_object(parts, (rg, {k: np.asarray(v) for k, v in res.items() if k != "obj"}))
        if rank == 0:
            glob = dict(cons=np.zeros_like(g_cons), grad=np.zeros_like(g_grad), jac=np.zeros_like(J.data),
                        hess=np.zeros_like(H.data))
            for prg, pres in parts:
                for key in glob:
                    for gs, ls, ln in prg[key]:
                        glob[key][gs:gs + ln] = pres[key][ls:ls + ln]
            out[name] = dict(obj=float(obj[0]) == o.objective(x), ok_j=bool(ok_j), ok_h=bool(ok_h),
                             cons=C.bit_diffs(glob["cons"], g_cons), grad=C.bit_diffs(glob["grad"], g_grad),
                             jac=C.bit_diffs(glob["jac"], J.data), hess=C.bit_diffs(glob["hess"], H.data),
                             halo=len(sc.plan.halo_idx))
        else:
            out[name] = dict(ok_j=bool(ok_j), ok_h=bool(ok_h), halo=len(sc.plan.halo_idx))
    results[rank] = out
    dist.destroy_process_group()


def test_two_rank_sharded_composites():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    mp.start_processes(_worker, args=(world, port, results), nprocs=world, start_method="spawn", join=True)
    r0, r1 = results[0], results[1]
    for name in ("scopf", "multiperiod", "general"):
        a = r0[name]
        assert a["obj"], name
        assert a["cons"] == 0 and a["grad"] == 0 and a["jac"] == 0 and a["hess"] == 0, (name, a)
        assert a["ok_j"] and a["ok_h"] and r1[name]["ok_j"] and r1[name]["ok_h"], name
    # rank 1 imports base-stage values for the cross-rank coupling rows
    assert r1["scopf"]["halo"] > 0 and r1["multiperiod"]["halo"] > 0
