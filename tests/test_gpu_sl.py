"""The stage-lane kernel (sl_kernel.cuh; full evaluations of stages sharing their tiles'
topology) against the per-callback path (tile kernel) and the reference's outputs, bitwise.

A full evaluation (ACOPF_ALL) of a batch runs the transposition pre-pass, the SL kernel and
the tile kernel for the (tile, stage) pairs SL does not cover (contingency-patched tiles, hub
buses); the single-callback what-masks run the tile kernel alone.  Every case compares both,
value for value, and the small fixtures also against the reference's goldens."""

import numpy as np
import pytest

import common as C
import paper_2203_10587_b200 as pkg
from golden.make_golden import COMPOSITE_SPECS, STAGE_SPECS, composite_inputs, compose, stage_case
from paper_2203_10587_b200 import _lib as L
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.grid import BRANCH, GEN, Contingency, ContingencySet, Outage
from paper_2203_10587_b200.types import CouplingMode

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _sl_on(monkeypatch):
    """The stage-lane path is opt-in (ACOPF_SL=1, read when a batch is first uploaded)."""
    monkeypatch.setenv("ACOPF_SL", "1")


def _per_callback(ev, x, mult, of):
    """The five outputs from five single-callback evaluations (tile kernel only)."""
    out = {}
    for what, key in ((L.OBJ, "obj"), (L.GRAD, "grad"), (L.CONS, "cons"), (L.JAC, "jac"), (L.HESS, "hess")):
        out[key] = ev.eval_host(x, mult, of, what)[key].copy()
    return out


def _full_device(ev, x, mult, of):
    import torch
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    md = torch.from_numpy(np.ascontiguousarray(mult)).cuda()
    o = ev.eval_device(xd, md, of, L.ALL)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items()}


def _check(ev, x, mult, of, name, golden=None):
    full = _full_device(ev, x, mult, of)
    ref = _per_callback(ev, x, mult, of)
    bits = vals = 0
    for k in ("obj", "grad", "cons", "jac", "hess"):
        a = full[k][:len(ref[k])]
        bits += C.bit_diffs(a, ref[k])
        vals += len(ref[k])
        if golden is not None:
            assert C.bit_diffs(a, golden[k]) == 0, (name, k)
    C.record("sl:" + name, bit_diffs=bits, values=vals)
    assert bits == 0, f"{name}: {bits} values differ between the SL and tile-kernel paths"


def _stage_batch(case, npts, seed):
    from paper_2203_10587_b200.packer import PackedCase, Topology
    from paper_2203_10587_b200.stage import stage_plan
    topo = Topology(PackedCase(case))
    ev = pkg.BatchEvaluator([stage_plan(topo) for _ in range(npts)], layout="independent")
    xl, xu, _ = topo.bounds()
    kinds = syn.variable_kinds([(topo.nb, topo.ng)])
    m1 = ev.m // npts
    pts = [syn.random_point(kinds, xl, xu, m1, seed + i) for i in range(npts)]
    return ev, np.concatenate([p[0] for p in pts]), np.concatenate([p[1] for p in pts])


@pytest.mark.parametrize("name", C.STAGE_FIXTURES)
def test_sl_stage_goldens(name):
    g = C.load(name)
    p, _ = pkg.build_acopf(stage_case(STAGE_SPECS[name]))
    for i, (x, mult, of) in enumerate(C.points(g)):
        gold = dict(obj=g[f"obj{i}"], grad=g[f"grad{i}"], cons=g[f"cons{i}"], jac=g[f"jdata{i}"],
                    hess=g[f"hdata{i}"])
        _check(p.evaluator, x, mult, of, f"{name}-{i}", gold)


@pytest.mark.parametrize("name", C.COMPOSITE_FIXTURES)
def test_sl_composite_goldens(name):
    g = C.load(name)
    spec = COMPOSITE_SPECS[name]
    a, _ = composite_inputs(spec)
    p, _ = compose(pkg, spec["kind"], a)
    for i, (x, mult, of) in enumerate(C.points(g)):
        gold = dict(obj=g[f"obj{i}"], grad=g[f"grad{i}"], cons=g[f"cons{i}"], jac=g[f"jdata{i}"],
                    hess=g[f"hdata{i}"])
        _check(p.evaluator, x, mult, of, f"{name}-{i}", gold)


@pytest.mark.parametrize("npts", [1, 5, 33, 100])
def test_sl_batches_of_points(npts):
    """Independent points of one network: partial and several lane groups."""
    ev, x, m = _stage_batch(syn.make_case(300, 90, 60, seed=12, features=True), npts, 40)
    _check(ev, x, m, 1.25, f"batch{npts}")


def test_sl_config1_network():
    ev, x, m = _stage_batch(syn.config_case(1), 40, 1000)
    _check(ev, x, m, 1.0, "cfg1x40")


def test_sl_hub_and_wide_angles():
    case = C.hub_case()
    ev, x, m = _stage_batch(case, 34, 70)
    _check(ev, x, m, 0.7, "hub")
    case = stage_case(STAGE_SPECS["stage_feat200"])
    ev, x, m = _stage_batch(case, 32, 5)
    nb = ev.plans[0].topo.nb
    xs = x.reshape(32, -1)
    xs[:, :nb] = np.random.default_rng(9).uniform(-1.6, 1.6, (32, nb))
    _check(ev, xs.reshape(-1), m, 1.0, "wide")


def test_sl_contingency_mixes():
    """GEN outages (other topologies), double outages, preventive pins: patched tiles fall back."""
    base = syn.make_case(60, 18, 12, seed=5, features=True)
    nb = syn.non_bridge_branches(base)
    ctgs = [Contingency(1, (Outage(GEN, base.gens[1].bus, None, 1),))]
    for j, k in enumerate(nb[:40]):
        br = base.branches[k]
        o = base.branches_between(br.fbus, br.tbus).index(k) + 1
        ctgs.append(Contingency(2 + j, (Outage(BRANCH, br.fbus, br.tbus, o),)))
    for mode in (CouplingMode(), CouplingMode(kind="preventive", pin_voltages=True)):
        p, imap = pkg.compose_scopf(base, ContingencySet(tuple(ctgs)), mode)
        kinds = syn.variable_kinds([(len(l.va), len(l.pg)) for l in imap.layouts])
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 77)
        _check(p.evaluator, x, mult, 1.0, f"ctgmix-{mode.kind}")


def test_sl_scenario_contingency_lattice():
    """A small cfg4-shaped lattice: 6 scenarios x (base + 5 N-1), wind targets."""
    base, scens, ctgs = syn.config4_inputs(n_scen=6, n_ctg=5, nb=300, n_chords=90, ng=60)
    p, imap = pkg.compose_general(scens, ctgs, [base], CouplingMode(), 30.0)
    kinds = syn.variable_kinds([(len(l.va), len(l.pg)) for l in imap.layouts])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 78)
    _check(p.evaluator, x, mult, 1.0, "lattice")
