"""The oracle (test infrastructure) is pinned to the reference's own outputs.

* against the committed golden fixtures (made by tests/golden/make_golden.py
  from the real reference): bit for bit, everywhere;
* against the live reference when it is mounted (build container only).
"""

import numpy as np
import pytest

import common as C
from oracle.composite import CompositeOracle
from oracle.stage import StageOracle
from golden.make_golden import STAGE_SPECS, COMPOSITE_SPECS, case_digest, composite_inputs, stage_case
from paper_2203_10587_b200.types import CouplingMode


def _same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and C.bit_diffs(a, b) == 0


def _composite_oracle(spec):
    a, bases = composite_inputs(spec)
    k = spec["kind"]
    if k == "scopf":
        return CompositeOracle.general(None, a["ctgs"], [a["base"]], a["mode"], 30.0), bases
    if k == "multiperiod":
        return CompositeOracle.general(None, None, a["periods"], CouplingMode(), a["dt"]), bases
    if k == "general":
        return CompositeOracle.general(a["scens"], a["ctgs"], a["periods"], a["mode"], a["dt"]), bases
    return CompositeOracle.sopf_flat(a["base"], a["scens"], a["ctgs"], a["mode"]), bases


def _check_problem(o, g):
    assert (o.n, o.m_eq, o.m_ineq) == (int(g["n"]), int(g["m_eq"]), int(g["m_ineq"]))
    for a in ("xl", "xu", "x0", "gl", "gu"):
        assert _same(getattr(o, a), g[a]), a
    for i, (x, mult, of) in enumerate(C.points(g)):
        assert o.objective(x) == float(g[f"obj{i}"][0])
        assert _same(o.gradient(x), g[f"grad{i}"])
        assert _same(o.constraints(x), g[f"cons{i}"])
        J = o.jacobian(x)
        assert np.array_equal(J.indptr, g["jindptr"]) and np.array_equal(J.indices, g["jindices"])
        assert _same(J.data, g[f"jdata{i}"])
        H = o.lagrangian_hessian(x, of, mult)
        assert np.array_equal(H.indptr, g["hindptr"]) and np.array_equal(H.indices, g["hindices"])
        assert _same(H.data, g[f"hdata{i}"])


@pytest.mark.parametrize("name", C.STAGE_FIXTURES)
def test_stage_oracle_matches_golden(name):
    g = C.load(name)
    case = stage_case(STAGE_SPECS[name])
    assert case_digest(case) == str(g["case_digest"]), "synthetic generator drifted"
    _check_problem(StageOracle(case), g)


@pytest.mark.parametrize("name", C.COMPOSITE_FIXTURES)
def test_composite_oracle_matches_golden(name):
    g = C.load(name)
    o, bases = _composite_oracle(COMPOSITE_SPECS[name])
    assert case_digest(bases[0]) == str(g["case_digest"])
    assert list(o.var_off) == list(g["var_offset"])
    rows = np.array([[c["stage_a"], c["stage_b"], -1 if c["gen"] is None else c["gen"],
                      -1 if c["bus"] is None else c["bus"], c["row"], int(c["is_equality"])]
                     for c in o.coupling], dtype=np.int64).reshape(-1, 6)
    assert np.array_equal(rows, g["cp_rows"])
    assert [c["kind"] for c in o.coupling] == list(g["cp_kinds"])
    assert _same([c["bound"] for c in o.coupling], g["cp_bounds"])
    _check_problem(o, g)


def test_oracle_matches_live_reference():
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        pytest.skip("reference not mounted")
    from paper_2203_10587_b200 import synthetic as syn
    case = syn.make_case(120, 40, 25, seed=77, features=True)
    p, lay = ok.build_acopf(rb.to_ref_case(case))
    o = StageOracle(case)
    kinds = syn.variable_kinds([(o.nb, o.ng)])
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 5)
    assert p.objective(x) == o.objective(x)
    assert _same(p.constraints(x), o.constraints(x))
    assert _same(p.jacobian(x).data, o.jacobian(x).data)
    assert _same(p.lagrangian_hessian(x, 2.0, mult).data, o.lagrangian_hessian(x, 2.0, mult).data)
    for k, v in o.layout_maps().items():
        assert getattr(lay, k) == v


def test_numpy_pairwise_sum_model():
    """np.sum over float64 is the pairwise scheme the kernel restates (n <= 128 blocks)."""
    def pw(a):
        n = len(a)
        if n < 8:
            r = 0.0
            for v in a:
                r += v
            return r
        if n <= 128:
            r = list(a[:8])
            i = 8
            while i < n - n % 8:
                for j in range(8):
                    r[j] += a[i + j]
                i += 8
            s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                s += a[i]
                i += 1
            return s
        n2 = n // 2
        n2 -= n2 % 8
        return pw(a[:n2]) + pw(a[n2:])
    rng = np.random.default_rng(0)
    for n in [0, 1, 7, 8, 9, 127, 128, 129, 500, 2500, 6000, 17000]:
        a = rng.standard_normal(n) * 1e3
        assert float(np.sum(a)) == pw(list(a))


def test_stage_oracle_matches_reference_fixture_case9():
    """The reference's own case9.m (tests/data), parsed by the reference, stored in the golden."""
    g = C.load("ref_case9_stage")
    _check_problem(StageOracle(C.case_from_json(str(g["case"]))), g)


@pytest.mark.parametrize("name", C.REF_FIXTURES)
def test_composite_oracle_matches_reference_fixtures(name):
    """case9 + ctgc.cont / scenarios.csv / load profile through the reference's compose_*."""
    g = C.load(name)
    o = C.ref_fixture_oracle(g)
    assert list(o.var_off) == list(g["var_offset"])
    rows = np.array([[c["stage_a"], c["stage_b"], -1 if c["gen"] is None else c["gen"],
                      -1 if c["bus"] is None else c["bus"], c["row"], int(c["is_equality"])]
                     for c in o.coupling], dtype=np.int64).reshape(-1, 6)
    assert np.array_equal(rows, g["cp_rows"])
    assert _same([c["bound"] for c in o.coupling], g["cp_bounds"])
    _check_problem(o, g)


@pytest.mark.parametrize("name", ["cfg0_stage", "cfg_feat200_wide"])
def test_stage_oracle_matches_config_goldens(name):
    """BASELINE config 0 and the wide-angle (|theta| up to ~pi) golden."""
    from paper_2203_10587_b200 import synthetic as syn
    g = C.load(name)
    case = syn.config_case(0) if name == "cfg0_stage" else stage_case(STAGE_SPECS["stage_feat200"])
    assert case_digest(case) == str(g["case_digest"]), "synthetic generator drifted"
    _check_problem(StageOracle(case), g)
