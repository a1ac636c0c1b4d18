"""Full-size GPU parity at every BASELINE.json config, with bit counts (slow; GPU).

Every value of the full workload is compared, not a sample:

* cfg0: the 9-bus ring at CONFIG_SEEDS[0] against the reference's own outputs
  (tests/golden/cfg0_stage.npz, make_golden.py configs) and the oracle;
* cfg1: the bench's whole 100-point batch of the 10,000-bus network against
  the oracle, point by point;
* cfg2 / cfg3: the complete composites (1,025 / 96 stages) against the
  oracle's composite callbacks (composer.py:256-311 restated), CSR patterns
  included;
* cfg4: all 1,024 stage blocks against per-stage oracles (a
  composite's stage block is the standalone stage with the stage weight), in
  a process pool; every one of the 6,138,000 coupling rows (structure against
  the oracle's lattice, values child - base, +-1 Jacobian entries); the
  composite objective as the stage-order sum.

Plus the reference's own fixtures (case9.m with ctgc.cont, scenarios.csv and
the load profile, tests/data of the reference) and branch angles up to ~pi
(glibc's wide-range sin/cos paths), against reference-generated goldens.

Gate (north_star): |a - b| <= 1e-14 + 1e-12 |b|; the path is bit-exact, so
every comparison also asserts 0 differing bits and records the counts in the
parity report (PARITY_REPORT=<path>).
"""

import multiprocessing as mp
import os

import numpy as np
import pytest

import common as C
import paper_2203_10587_b200 as pkg
from golden.make_golden import STAGE_SPECS, stage_case
from paper_2203_10587_b200 import _lib as L
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.lattice import KINDS
from paper_2203_10587_b200.types import CouplingMode
from oracle.composite import CompositeOracle
from oracle.stage import StageOracle

pytestmark = pytest.mark.gpu


class Tally:
    """Gate misses, differing bits and value counts over many comparisons."""

    def __init__(self):
        self.misses = self.bits = self.values = 0

    def add(self, a, b):
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        assert a.shape == b.shape, (a.shape, b.shape)
        self.misses += C.gate_misses(a, b)
        self.bits += C.bit_diffs(a, b)
        self.values += b.size

    def finish(self, name, **extra):
        C.record(name, gate_misses=self.misses, bit_diffs=self.bits, values=self.values, **extra)
        if self.bits:
            print(name, extra)
        assert self.misses == 0, f"{name}: {self.misses} values outside the gate"
        assert self.bits == 0, f"{name}: {self.bits} values differ in some bit"


def _problem_vs(t: Tally, p, ref, x, mult, of, patterns=True):
    """All five callbacks of p against ref (an oracle or a golden dict entry)."""
    J, H = p.jacobian(x), p.lagrangian_hessian(x, of, mult)
    if isinstance(ref, tuple):
        r_obj, r_grad, r_cons, (rjp, rji, rjd), (rhp, rhi, rhd) = ref
    else:
        Jo, Ho = ref.jacobian(x), ref.lagrangian_hessian(x, of, mult)
        r_obj, r_grad, r_cons = ref.objective(x), ref.gradient(x), ref.constraints(x)
        rjp, rji, rjd, rhp, rhi, rhd = Jo.indptr, Jo.indices, Jo.data, Ho.indptr, Ho.indices, Ho.data
    if patterns:
        assert np.array_equal(J.indptr, rjp) and np.array_equal(J.indices, rji)
        assert np.array_equal(H.indptr, rhp) and np.array_equal(H.indices, rhi)
    t.add([p.objective(x)], [r_obj])
    t.add(p.gradient(x), r_grad)
    t.add(p.constraints(x), r_cons)
    t.add(J.data, rjd)
    t.add(H.data, rhd)


def _golden_ref(g, i):
    return (float(g[f"obj{i}"][0]), g[f"grad{i}"], g[f"cons{i}"], (g["jindptr"], g["jindices"], g[f"jdata{i}"]),
            (g["hindptr"], g["hindices"], g[f"hdata{i}"]))


# ---------------------------------------------------------------------------
# cfg0, wide angles, the reference's fixtures


@pytest.fixture(params=["0", "1"], ids=["gather", "interleaved"])
def bus_inputs(request, monkeypatch):
    monkeypatch.setenv("ACOPF_INTERLEAVE", request.param)
    return request.param


def test_config0_full(bus_inputs):
    """BASELINE config 0: the reference's own outputs at 4 points, then the oracle at 40 more."""
    case = syn.config_case(0)
    p, _ = pkg.build_acopf(case)
    g = C.load("cfg0_stage")
    t = Tally()
    for i, (x, mult, of) in enumerate(C.points(g)):
        _problem_vs(t, p, _golden_ref(g, i), x, mult, of)
    o = StageOracle(case)
    kinds = syn.variable_kinds([(o.nb, o.ng)])
    for s in range(40):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, syn.CONFIG_SEEDS[0] + 100 + s)
        _problem_vs(t, p, o, x, mult, 1.0 + 0.1 * s)
    t.finish(f"oracle:cfg0-full-{bus_inputs}", points=44)


def test_wide_branch_angles_golden(bus_inputs):
    """Branch angles up to ~pi (Va ~ U(-1.6, 1.6)): glibc's reflection and Cody-Waite paths of
    sin/cos, against the reference's outputs (cfg_feat200_wide.npz), bit for bit."""
    g = C.load("cfg_feat200_wide")
    p, _ = pkg.build_acopf(stage_case(STAGE_SPECS["stage_feat200"]))
    t = Tally()
    for i, (x, mult, of) in enumerate(C.points(g)):
        _problem_vs(t, p, _golden_ref(g, i), x, mult, of)
    t.finish(f"golden:wide-angles-{bus_inputs}")


def test_wide_branch_angles_config1_network():
    """The 10,000-bus network at Va ~ U(-pi/2, pi/2) (|theta| up to pi) against the oracle."""
    case = syn.config_case(1)
    p, _ = pkg.build_acopf(case)
    o = StageOracle(case)
    kinds = syn.variable_kinds([(o.nb, o.ng)])
    t = Tally()
    for s in range(2):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 700 + s)
        va = kinds == syn.VA
        x[va] = np.random.default_rng(800 + s).uniform(-np.pi / 2, np.pi / 2, int(va.sum()))
        x[p.xl == p.xu] = p.xl[p.xl == p.xu]
        _problem_vs(t, p, o, x, mult, 1.0)
    t.finish("oracle:cfg1-wide-angles")


def test_reference_fixture_case9_stage(bus_inputs):
    """The reference's case9.m at x0, two seeded points and a wide-angle point."""
    g = C.load("ref_case9_stage")
    p, _ = pkg.build_acopf(C.case_from_json(str(g["case"])))
    t = Tally()
    for i, (x, mult, of) in enumerate(C.points(g)):
        _problem_vs(t, p, _golden_ref(g, i), x, mult, of)
    t.finish(f"golden:ref_case9_stage-{bus_inputs}")


@pytest.mark.parametrize("name", C.REF_FIXTURES)
def test_reference_fixture_composites(name, bus_inputs):
    """case9 + ctgc.cont / scenarios.csv / load_p,q.csv through compose_* (the reference's
    tests/test_composer.py usage), against the reference's composite callbacks."""
    g = C.load(name)
    p, _ = C.ref_fixture_compose(pkg, g, CouplingMode)
    t = Tally()
    for i, (x, mult, of) in enumerate(C.points(g)):
        _problem_vs(t, p, _golden_ref(g, i), x, mult, of)
    t.finish(f"golden:{name}-{bus_inputs}")


# ---------------------------------------------------------------------------
# cfg1: the whole 100-point batch


@pytest.mark.slow
def test_config1_full_batch():
    """The bench's 100 seeded points in ONE batched launch, every value against the oracle."""
    from paper_2203_10587_b200.packer import PackedCase, Topology
    from paper_2203_10587_b200.stage import stage_plan
    case = syn.config_case(1)
    topo = Topology(PackedCase(case))
    npts = 100
    ev = pkg.BatchEvaluator([stage_plan(topo) for _ in range(npts)], layout="independent")
    xl, xu, _ = topo.bounds()
    kinds = syn.variable_kinds([(topo.nb, topo.ng)])
    m1 = ev.m // npts
    pts = [syn.random_point(kinds, xl, xu, m1, 1_000_000 + i) for i in range(npts)]
    out = ev.eval_host(np.concatenate([p[0] for p in pts]), np.concatenate([p[1] for p in pts]), 1.0, L.ALL)
    o = StageOracle(case)
    n1, nj, nh = ev.n // npts, ev.nnz_j // npts, ev.nnz_h // npts
    t = Tally()
    jp, ji = ev.pattern("J", 0)
    hp, hi = ev.pattern("H", 0)
    for i, (x, mult) in enumerate(pts):
        J, H = o.jacobian(x), o.lagrangian_hessian(x, 1.0, mult)
        if i == 0:
            assert np.array_equal(jp, J.indptr) and np.array_equal(ji, J.indices)
            assert np.array_equal(hp, H.indptr) and np.array_equal(hi, H.indices)
        t.add(out["obj"][i:i + 1], [o.objective(x)])
        t.add(out["grad"][i * n1:(i + 1) * n1], o.gradient(x))
        t.add(out["cons"][i * m1:(i + 1) * m1], o.constraints(x))
        t.add(out["jac"][i * nj:(i + 1) * nj], J.data)
        t.add(out["hess"][i * nh:(i + 1) * nh], H.data)
    t.finish("oracle:cfg1-full", points=npts)


# ---------------------------------------------------------------------------
# cfg2 / cfg3: complete composites against the oracle's composite callbacks


def _full_composite(name, p, o, seed):
    kinds = syn.variable_kinds([(s.nb, s.ng) for s in o.stage])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, seed)
    for a in ("xl", "xu", "x0", "gl", "gu"):
        assert C.bit_diffs(getattr(p, a), getattr(o, a)) == 0, a
    t = Tally()
    _problem_vs(t, p, o, x, mult, 1.0)
    t.finish(name, stages=len(o.stage))


@pytest.mark.slow
def test_config2_full_composite():
    """BASELINE config 2 (1,025 stages): every output value and both CSR patterns."""
    base, ctgs = syn.config2_inputs()
    p, imap = pkg.compose_scopf(base, ctgs, CouplingMode())
    o = CompositeOracle.general(None, ctgs, [base], CouplingMode(), 30.0)
    assert list(imap.var_offset) == [int(v) for v in o.var_off]
    _full_composite("oracle:cfg2-full", p, o, 31)


@pytest.mark.slow
def test_config3_full_composite():
    """BASELINE config 3 (96 periods, ramp rows): every output value and both CSR patterns."""
    periods = syn.config3_periods()
    p, imap = pkg.compose_multiperiod(periods, 15.0)
    o = CompositeOracle.general(None, None, periods, CouplingMode(), 15.0)
    assert list(imap.var_offset) == [int(v) for v in o.var_off]
    _full_composite("oracle:cfg3-full", p, o, 33)


# ---------------------------------------------------------------------------
# cfg4: all 1,024 stage blocks in a process pool, every coupling row

_W = {}


def _cfg4_stage(k):
    """Worker: stage k of the cfg4 composite against its own oracle (stage-local CSR)."""
    o_lat, ev, out, x, mult = _W["lat"], _W["ev"], _W["out"], _W["x"], _W["mult"]
    so = StageOracle(o_lat.cases[k])
    n, meq, mineq, njeq, njin, nh = (int(v) for v in ev.sizes[k])
    assert (so.n, so.m_eq, so.m_ineq) == (n, meq, mineq)
    a = int(ev.var_off[k])
    e0, i0 = int(ev.eq_row[k]), int(ev.ineq_row[k])
    xk = x[a:a + n]
    mk = np.concatenate([mult[e0:e0 + meq], mult[i0:i0 + mineq]])
    w = float(o_lat.weights[k])
    J, H = so.jacobian(xk), so.lagrangian_hessian(xk, 1.0 * w, mk)
    jp, ji = ev.pattern("J", k)
    hp, hi = ev.pattern("H", k)
    pat = (np.array_equal(jp, J.indptr) and np.array_equal(ji, J.indices) and np.array_equal(hp, H.indptr)
           and np.array_equal(hi, H.indices))
    jb, jn, hb = int(ev.jeq_base[k]), int(ev.jin_base[k]), int(ev.h_base[k])
    pairs = [(out["grad"][a:a + n], w * so.gradient(xk)),
             (np.concatenate([out["cons"][e0:e0 + meq], out["cons"][i0:i0 + mineq]]), so.constraints(xk)),
             (np.concatenate([out["jac"][jb:jb + njeq], out["jac"][jn:jn + njin]]), J.data),
             (out["hess"][hb:hb + nh], H.data)]
    t = Tally()
    where = []
    for name, (u, v) in zip(("grad", "cons", "jac", "hess"), pairs):
        b0 = t.bits
        t.add(u, v)
        if t.bits > b0:
            d = np.flatnonzero(np.asarray(u).view(np.int64) != np.asarray(v).view(np.int64))[:4]
            where.append((k, name, [(int(i), float(u[i]), float(v[i])) for i in d]))
    pg = so.layout_maps()["pg"]
    return k, so.objective(xk), t.misses, t.bits, t.values, pat, pg, where


@pytest.mark.slow
def test_config4_full_all_stages():
    """BASELINE config 4: all 1,024 stage blocks (25k buses each) and all 6,138,000 coupling rows."""
    base, scens, ctgs = syn.config4_inputs()
    mode = CouplingMode()
    p, imap = pkg.compose_general(scens, ctgs, [base], mode, 30.0)
    ev = p.evaluator
    S = len(ev.plans)
    assert S == 1024
    kinds = syn.variable_kinds([(pl.topo.nb, pl.topo.ng) for pl in ev.plans])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 41)
    out = ev.eval_host(x, mult, 1.0, L.ALL)
    lat = CompositeOracle.general(scens, ctgs, [base], mode, 30.0, assemble=False)
    assert len(lat.cases) == S
    assert np.array_equal(np.asarray(imap.weights), np.asarray(lat.weights))
    _W.update(lat=lat, ev=ev, out=out, x=x, mult=mult)
    workers = max(1, min(16, (os.cpu_count() or 2) - 1))
    t = Tally()
    fs = [None] * S
    pgs = [None] * S
    where = []
    with mp.get_context("fork").Pool(workers) as pool:
        for k, f, mi, bi, vi, pat, pg, wh in pool.imap_unordered(_cfg4_stage, range(S), chunksize=4):
            assert pat, f"stage {k}: CSR pattern differs"
            fs[k], pgs[k] = f, pg
            where += wh
            t.misses += mi
            t.bits += bi
            t.values += vi
    _W.clear()
    # composite objective: sum(w[k] f_k) with w = np.asarray(weights) (composer.py:244,256-258):
    # np.float64 items, so CPython's sum adds them left to right (its compensated float
    # path, 3.12+, only applies to exact Python floats)
    w = np.asarray(lat.weights)
    ref_obj = float(sum(w[k] * fs[k] for k in range(S)))
    b0 = t.bits
    t.add(out["obj"][:1], [ref_obj])
    if t.bits > b0:
        where.append(("objective", float(out["obj"][0]), ref_obj))
    # coupling rows: the oracle lattice's pending rows, in order (pins first, then boxes)
    cp = imap.coupling_arrays
    pend = [r for r in lat.pending if r[6]] + [r for r in lat.pending if not r[6]]
    assert len(pend) == len(cp["row"]) == 6_138_000
    kind = np.array([KINDS.index(r[0]) for r in pend], dtype=np.int8)
    sa = np.array([r[1] for r in pend], dtype=np.int64)
    sb = np.array([r[2] for r in pend], dtype=np.int64)
    gen = np.array([r[3] for r in pend], dtype=np.int64)
    bound = np.array([r[5] for r in pend], dtype=np.float64)
    assert np.array_equal(cp["kind"], kind) and np.array_equal(cp["stage_a"], sa)
    assert np.array_equal(cp["stage_b"], sb) and np.array_equal(cp["gen"], gen)
    assert C.bit_diffs(cp["bound"], bound) == 0
    rows = np.arange(p.m_eq + int(ev.sizes[:, 2].sum()), p.m_eq + p.m_ineq)
    assert np.array_equal(cp["row"], rows)
    # columns from the oracle's own stage layouts (cfg4 contingencies are branch outages: every
    # stage has the same live generators): x[var_off[a] + pg[g]] - x[var_off[b] + pg[g]]
    assert all(pg == pgs[0] for pg in pgs[1:])
    var_off = np.asarray(ev.var_off)
    pgarr = np.full(len(base.gens), -1, dtype=np.int64)
    for g_, v_ in pgs[0].items():
        pgarr[g_] = v_
    assert (pgarr[gen] >= 0).all()
    ca, cb = var_off[sa] + pgarr[gen], var_off[sb] + pgarr[gen]
    t.add(out["cons"][rows], x[ca] - x[cb])
    # +-1 Jacobian entries at the coupling rows' CSR positions, ordered by column
    jp, _ = ev.pattern("J")
    pos = jp[rows]
    first = np.where(cb < ca, -1.0, 1.0)
    t.add(out["jac"][pos], first)
    t.add(out["jac"][pos + 1], -first)
    t.finish("oracle:cfg4-full", stages=S, coupling_rows=int(len(rows)), differing=repr(where[:20]))


def test_matpower_text_from_gpu_solutions():
    """extract_solution on the GPU, then write_case (acopf_format_matrix): the reference's text."""
    from paper_2203_10587_b200 import matpower as M
    from paper_2203_10587_b200.solution import extract_solution
    g = C.load("matpower_text")
    for i in range(int(g["n"])):
        case = C.case_from_json(str(g[f"case{i}"]))
        _, lay = pkg.build_acopf(case)
        sol = extract_solution(case, lay, g[f"x{i}"])
        assert M.write_case(sol, name=f"t_{i}") == str(g[f"text{i}"])
        assert M.write_case(sol) == str(g[f"text_default{i}"])
