"""GPU parity: the CUDA path (through the C ABI) against the oracle and goldens.

Gate (BASELINE.json north_star): patterns and index maps bit-exact; every
value within |a - b| <= 1e-14 + 1e-12 |b|.  Bitwise-different counts are
recorded alongside (the only source is the device sincos vs glibc's, which
differ in the last bit on ~0.25 % of angles).
"""

import json
import os

import numpy as np
import pytest

import common as C
from golden.make_golden import COMPOSITE_SPECS, STAGE_SPECS, composite_inputs, compose, stage_case
import paper_2203_10587_b200 as pkg
from paper_2203_10587_b200 import _lib as L
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.grid import BRANCH, GEN, Contingency, ContingencySet, Outage
from paper_2203_10587_b200.types import CouplingMode
from oracle.composite import CompositeOracle
from oracle.stage import StageOracle

pytestmark = pytest.mark.gpu

REPORT = {}


def _record(name, **kw):
    REPORT.setdefault(name, {}).update(kw)
    out = os.environ.get("PARITY_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump(REPORT, fh, indent=1, sort_keys=True)


def _compare_problem(p, ref, pts, name):
    """ref: object with objective/gradient/constraints/jacobian/lagrangian_hessian (or golden dict)."""
    misses = bits = total = 0
    for i, (x, mult, of) in enumerate(pts):
        if isinstance(ref, dict):
            r_obj = float(ref[f"obj{i}"][0])
            r_grad, r_cons = ref[f"grad{i}"], ref[f"cons{i}"]
            r_j = (ref["jindptr"], ref["jindices"], ref[f"jdata{i}"])
            r_h = (ref["hindptr"], ref["hindices"], ref[f"hdata{i}"])
        else:
            r_obj, r_grad, r_cons = ref.objective(x), ref.gradient(x), ref.constraints(x)
            J, H = ref.jacobian(x), ref.lagrangian_hessian(x, of, mult)
            r_j, r_h = (J.indptr, J.indices, J.data), (H.indptr, H.indices, H.data)
        J = p.jacobian(x)
        H = p.lagrangian_hessian(x, of, mult)
        assert np.array_equal(J.indptr, r_j[0]) and np.array_equal(J.indices, r_j[1])
        assert np.array_equal(H.indptr, r_h[0]) and np.array_equal(H.indices, r_h[1])
        assert J.indices.dtype == np.int32 and H.indptr.dtype == np.int32
        pairs = [([p.objective(x)], [r_obj]), (p.gradient(x), r_grad), (p.constraints(x), r_cons),
                 (J.data, r_j[2]), (H.data, r_h[2])]
        for a, b in pairs:
            misses += C.gate_misses(a, b)
            bits += C.bit_diffs(a, b)
            total += len(b)
    _record(name, gate_misses=misses, bit_diffs=bits, values=total)
    assert misses == 0, f"{misses} values outside the 1e-12/1e-14 gate"


@pytest.mark.parametrize("name", C.STAGE_FIXTURES)
def test_stage_vs_golden(name):
    g = C.load(name)
    p, _ = pkg.build_acopf(stage_case(STAGE_SPECS[name]))
    _compare_problem(p, g, C.points(g), "golden:" + name)


@pytest.mark.parametrize("name", C.COMPOSITE_FIXTURES)
def test_composite_vs_golden(name):
    g = C.load(name)
    spec = COMPOSITE_SPECS[name]
    a, _ = composite_inputs(spec)
    p, _ = compose(pkg, spec["kind"], a)
    _compare_problem(p, g, C.points(g), "golden:" + name)


def test_small_cases_are_bit_exact():
    """Ring and feature cases: every output bitwise equal to the reference."""
    for name in ("stage_ring9", "stage_feat30"):
        g = C.load(name)
        p, _ = pkg.build_acopf(stage_case(STAGE_SPECS[name]))
        for i, (x, mult, of) in enumerate(C.points(g)):
            assert p.objective(x) == float(g[f"obj{i}"][0])
            assert C.bit_diffs(p.constraints(x), g[f"cons{i}"]) == 0
            assert C.bit_diffs(p.jacobian(x).data, g[f"jdata{i}"]) == 0
            assert C.bit_diffs(p.lagrangian_hessian(x, of, mult).data, g[f"hdata{i}"]) == 0


def _oracle_points(p, o, n, seed):
    kinds = syn.variable_kinds([(s.nb, s.ng) for s in getattr(o, "stage", [o])])
    out = []
    for s in range(n):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, seed + s)
        out.append((x, mult, 1.0))
    return out


def test_config1_network_vs_oracle():
    """BASELINE config 1 network (10k buses) at seeded points."""
    case = syn.config_case(1)
    p, _ = pkg.build_acopf(case)
    o = StageOracle(case)
    _compare_problem(p, o, _oracle_points(p, o, 3, 11), "oracle:cfg1")


def test_generator_and_multi_outage_contingencies():
    """GEN outages (new topology), a double outage, preventive pins (ctgc.cont-like)."""
    base = syn.make_case(40, 12, 8, seed=5, features=True)
    nb = syn.non_bridge_branches(base)
    b1, b2 = base.branches[nb[0]], base.branches[nb[3]]
    o1 = base.branches_between(b1.fbus, b1.tbus).index(nb[0]) + 1
    o2 = base.branches_between(b2.fbus, b2.tbus).index(nb[3]) + 1
    g0 = base.gens[1]
    ctgs = ContingencySet((
        Contingency(1, (Outage(GEN, g0.bus, None, 1),)),
        Contingency(2, (Outage(BRANCH, b1.fbus, b1.tbus, o1),)),
        Contingency(3, (Outage(GEN, g0.bus, None, 1), Outage(BRANCH, b2.fbus, b2.tbus, o2))),
        Contingency(4, (Outage(BRANCH, b1.fbus, b1.tbus, o1), Outage(BRANCH, b2.fbus, b2.tbus, o2))),
    ))
    for mode in (CouplingMode(), CouplingMode(kind="preventive", pin_voltages=True)):
        p, imap = pkg.compose_scopf(base, ctgs, mode)
        o = CompositeOracle.general(None, ctgs, [base], mode, 30.0)
        _compare_problem(p, o, _oracle_points(p, o, 2, 21), f"oracle:ctg-mix-{mode.kind}")


def test_batched_points_equal_single_evaluations():
    """Independent-layout batch of 6 points == 6 single evaluations, bitwise."""
    case = syn.make_case(500, 150, 100, seed=8, features=True)
    p, _ = pkg.build_acopf(case)
    topo = p.evaluator.plans[0].topo
    from paper_2203_10587_b200.stage import stage_plan
    ev = pkg.BatchEvaluator([stage_plan(topo) for _ in range(6)], layout="independent")
    kinds = syn.variable_kinds([(topo.nb, topo.ng)])
    xs, ms = [], []
    for s in range(6):
        x, m = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 300 + s)
        xs.append(x)
        ms.append(m)
    out = ev.eval_host(np.concatenate(xs), np.concatenate(ms), 1.5, L.ALL)
    one = p.evaluator
    for s in range(6):
        r = one.eval_host(xs[s], ms[s], 1.5, L.ALL)
        assert out["obj"][s] == r["obj"][0]
        for key, size in (("grad", one.n), ("cons", one.m), ("jac", one.nnz_j), ("hess", one.nnz_h)):
            assert C.bit_diffs(out[key][s * size:(s + 1) * size], r[key]) == 0, key


def test_composite_blocks_equal_standalone_stages():
    """each stage block of a composite equals the standalone stage, bitwise."""
    base, ctgs = syn.config2_inputs(n_ctg=12, nb=300, n_chords=90, ng=60)
    p, imap = pkg.compose_scopf(base, ctgs, CouplingMode())
    kinds = syn.variable_kinds([(len(l.va), len(l.pg)) for l in imap.layouts])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 5)
    J = p.jacobian(x)
    H = p.lagrangian_hessian(x, 1.0, mult)
    c = p.constraints(x)
    for k in (0, 1, 7, 12):
        sp_, lay = pkg.build_acopf(imap.stages[k].case)
        a, b = imap.var_offset[k], imap.var_offset[k] + lay.n_vars
        e0, i0 = imap.eq_offset[k], p.m_eq + imap.ineq_offset[k]
        mk = np.concatenate([mult[e0:e0 + lay.n_eq], mult[i0:i0 + lay.n_ineq]])
        Js = sp_.jacobian(x[a:b])
        Hs = sp_.lagrangian_hessian(x[a:b], 1.0 * imap.weights[k], mk)
        rows = np.r_[e0:e0 + lay.n_eq, i0:i0 + lay.n_ineq]
        assert C.bit_diffs(J[rows][:, a:b].toarray(), Js.toarray()) == 0
        assert C.bit_diffs(H[a:b][:, a:b].toarray(), Hs.toarray()) == 0
        assert C.bit_diffs(c[rows], sp_.constraints(x[a:b])) == 0


def test_what_mask_writes_only_requested_outputs():
    case = syn.make_case(200, 60, 40, seed=3, features=True)
    p, _ = pkg.build_acopf(case)
    import torch
    ev = p.evaluator
    x = torch.tensor(p.x0, device="cuda")
    mult = torch.ones(ev.m, dtype=torch.float64, device="cuda")
    for what, key in ((L.OBJ, "obj"), (L.GRAD, "grad"), (L.CONS, "cons"), (L.JAC, "jac"), (L.HESS, "hess")):
        out = ev.alloc()
        for t in out.values():
            t.fill_(12345.0)
        ev.eval_device(x, mult, 1.0, what, out=out)
        torch.cuda.synchronize()
        for k, t in out.items():
            if k == key:
                assert not bool((t == 12345.0).all())
            else:
                assert bool((t == 12345.0).all()), (what, k)
    full = ev.eval_device(x, mult, 1.0, L.ALL)
    host = ev.eval_host(p.x0, np.ones(ev.m), 1.0, L.ALL)
    for k in ("obj", "grad", "cons", "jac", "hess"):
        assert C.bit_diffs(full[k].cpu().numpy()[:len(host[k])], host[k]) == 0


def test_edge_cases():
    """No rated branches, single bus, no live generators, NaN propagation."""
    from dataclasses import replace
    case = syn.make_case(12, 3, 3, seed=2)
    unrated = replace(case, branches=tuple(replace(b, rate_a=0.0) for b in case.branches))
    lone = replace(case, buses=case.buses[:1], gens=case.gens[:1], branches=())
    nogen = replace(case, gens=tuple(replace(g, status=0) for g in case.gens))
    for c in (unrated, lone, nogen):
        p, _ = pkg.build_acopf(c)
        o = StageOracle(c)
        _compare_problem(p, o, _oracle_points(p, o, 2, 40), "oracle:edge")
    p, _ = pkg.build_acopf(case)
    o = StageOracle(case)
    x = p.x0.copy()
    x[3] = np.nan
    mult = np.ones(p.m_eq + p.m_ineq)
    assert np.array_equal(np.isnan(p.constraints(x)), np.isnan(o.constraints(x)))
    assert np.array_equal(np.isnan(p.jacobian(x).data), np.isnan(o.jacobian(x).data))
    assert np.array_equal(np.isnan(p.lagrangian_hessian(x, 1.0, mult).data),
                          np.isnan(o.lagrangian_hessian(x, 1.0, mult).data))


def test_finite_difference_consistency():
    """The reference's own known-answer check (tests/test_acopf.py:106-126): FD 1e-6 / 1e-5."""
    case = syn.make_case(14, 4, 4, seed=6, features=True)
    p, _ = pkg.build_acopf(case)
    rng = np.random.default_rng(3)
    m = p.m_eq + p.m_ineq
    mult = rng.uniform(-1.0, 1.0, m)
    lo = np.where(np.isfinite(p.xl), p.xl, -0.5)
    hi = np.where(np.isfinite(p.xu), p.xu, 0.5)
    x = lo + rng.uniform(0.1, 0.9, p.n) * (hi - lo)
    x[p.xl == p.xu] = p.xl[p.xl == p.xu]
    rel = lambda a, b: 0.0 if max(abs(a), abs(b)) <= 1e-8 else abs(a - b) / max(1.0, abs(a), abs(b))
    g, J, H = p.gradient(x), p.jacobian(x).toarray(), p.lagrangian_hessian(x, 1.0, mult).toarray()
    lag = lambda z: p.gradient(z) + p.jacobian(z).T @ mult
    h = 1e-6
    worst = [0.0, 0.0, 0.0]
    for i in range(p.n):
        e = np.zeros(p.n)
        e[i] = h
        worst[0] = max(worst[0], rel(g[i], (p.objective(x + e) - p.objective(x - e)) / (2 * h)))
        fdc = (p.constraints(x + e) - p.constraints(x - e)) / (2 * h)
        worst[1] = max(worst[1], max(rel(J[k, i], fdc[k]) for k in range(m)))
        fdh = (lag(x + e) - lag(x - e)) / (2 * h)
        worst[2] = max(worst[2], max(rel(H[k, i], fdh[k]) for k in range(p.n)))
    assert worst[0] <= 1e-6 and worst[1] <= 1e-6 and worst[2] <= 1e-5, worst


def test_disconnected_and_bad_inputs():
    from dataclasses import replace
    case = syn.make_case(12, 0, 3, seed=2)
    with pytest.raises(pkg.Disconnected):
        pkg.build_acopf(replace(case, branches=case.branches[1:]))
    p, _ = pkg.build_acopf(case)
    with pytest.raises(ValueError):
        p.constraints(np.zeros(p.n + 1))


def test_sharded_path_single_rank_nccl():
    """ShardedComposite on one NCCL rank == the unsharded composite, bitwise (collectives on GPU)."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2203_10587_b200.dispatch import ShardedComposite
    from paper_2203_10587_b200.lattice import composite_spec
    base, ctgs = syn.config2_inputs(n_ctg=9, nb=200, n_chords=60, ng=40)
    spec = composite_spec("scopf", base, ctgs, CouplingMode())
    p, _ = pkg.compose_scopf(base, ctgs, CouplingMode())
    kinds = syn.variable_kinds(spec.stage_dims)
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 9)
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        sc = ShardedComposite(spec, dist, 0, 1, device="cuda:0")
        xd = sc.alloc_x()
        xd[:sc.plan.n_loc] = torch.from_numpy(x).cuda()
        out, obj = sc.evaluate(xd, torch.from_numpy(mult).cuda(), 1.25, L.ALL)
        torch.cuda.synchronize()
        ref = p.evaluator.eval_host(x, mult, 1.25, L.ALL)
        assert obj == float(ref["obj"][0])
        for k in ("grad", "cons", "jac", "hess"):
            assert C.bit_diffs(out[k].cpu().numpy()[:len(ref[k])], ref[k]) == 0, k
    finally:
        dist.destroy_process_group()


def _check_composite_samples(p, imap, stages, seed):
    """Sampled stage blocks vs the oracle (gate) and vs standalone GPU stages (bitwise)."""
    kinds = syn.variable_kinds([(len(l.va), len(l.pg)) for l in imap.layouts])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, seed)
    ev = p.evaluator
    out = ev.eval_host(x, mult, 1.0, L.ALL)
    # composite objective = ((0 + w_0 f_0) + w_1 f_1) + ... over all stages (composer.py:256-258)
    terms_ev = pkg.BatchEvaluator(ev.plans, layout="composite", coupling=None, obj_terms=True)
    t = terms_ev.eval_host(x, None, 1.0, L.OBJ)["obj"]
    acc = 0.0
    for v in t:
        acc = acc + float(v)
    assert acc == float(out["obj"][0])
    ip, ix = ev.pattern("J")
    hp, hx = ev.pattern("H")
    misses = 0
    for k in stages:
        case = imap.stages[k].case
        o = StageOracle(case)
        lay = imap.layouts[k]
        a, b = imap.var_offset[k], imap.var_offset[k] + lay.n_vars
        e0, i0 = imap.eq_offset[k], p.m_eq + imap.ineq_offset[k]
        mk = np.concatenate([mult[e0:e0 + lay.n_eq], mult[i0:i0 + lay.n_ineq]])
        xs = x[a:b]
        # constraints of the stage block
        cs = np.concatenate([out["cons"][e0:e0 + lay.n_eq], out["cons"][i0:i0 + lay.n_ineq]])
        misses += C.gate_misses(cs, o.constraints(xs))
        # J rows of the stage (eq then ineq), H rows of the stage
        rows = np.r_[e0:e0 + lay.n_eq, i0:i0 + lay.n_ineq]
        Jd = np.concatenate([out["jac"][ip[r]:ip[r + 1]] for r in rows])
        Hd = out["hess"][hp[a]:hp[b]]
        Jo = o.jacobian(xs)
        Ho = o.lagrangian_hessian(xs, 1.0 * imap.weights[k], mk)
        assert len(Jd) == Jo.nnz and len(Hd) == Ho.nnz
        misses += C.gate_misses(Jd, Jo.data) + C.gate_misses(Hd, Ho.data)
        g = out["grad"][a:b]
        misses += C.gate_misses(g, imap.weights[k] * o.gradient(xs))
    # coupling rows read child - base
    for r in list(imap.coupling_rows)[:50]:
        child = imap.var_offset[r.stage_a] + imap.layouts[r.stage_a].pg[r.gen]
        base_ = imap.var_offset[r.stage_b] + imap.layouts[r.stage_b].pg[r.gen]
        assert out["cons"][r.row] == x[child] - x[base_]
    return misses


@pytest.mark.slow
def test_config2_full_composite_samples():
    """BASELINE config 2 at full size (1,025 stages): sampled stages vs the oracle."""
    base, ctgs = syn.config2_inputs()
    p, imap = pkg.compose_scopf(base, ctgs, CouplingMode())
    misses = _check_composite_samples(p, imap, [0, 1, 513, 1024], 31)
    _record("oracle:cfg2-full-samples", gate_misses=misses)
    assert misses == 0


@pytest.mark.slow
def test_config4_full_composite_samples():
    """BASELINE config 4 at full size (1,024 stages, 25k buses): sampled stages vs the oracle."""
    base, scens, ctgs = syn.config4_inputs()
    p, imap = pkg.compose_general(scens, ctgs, [base], CouplingMode(), 30.0)
    misses = _check_composite_samples(p, imap, [0, 1, 32, 33, 1023], 41)
    _record("oracle:cfg4-full-samples", gate_misses=misses)
    assert misses == 0
