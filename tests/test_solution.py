"""Solution extraction (acopf.py:413-546): oracle vs reference fixtures, device path vs both."""

import json
from types import SimpleNamespace

import numpy as np
import pytest

import common as C
from golden.make_golden import COMPOSITE_SPECS, STAGE_SPECS, composite_inputs, compose, stage_case
import paper_2203_10587_b200 as pkg
from paper_2203_10587_b200 import solution as S
from paper_2203_10587_b200 import synthetic as syn
from oracle import solution as OS
from oracle.stage import StageOracle

FIELDS = ("vm", "va", "pg", "qg", "pf", "qf", "pt", "qt")
STAGES = ["stage_ring9", "stage_feat30", "stage_feat200"]
COMPOSITES = ["scopf_corrective", "general"]


def _layout(case):
    o = StageOracle(case)
    return SimpleNamespace(n_vars=o.n, **o.layout_maps())


def _same(sol, g, prefix):
    get = (lambda f: sol[f]) if isinstance(sol, dict) else (lambda f: getattr(sol, f))
    for f in FIELDS:
        assert C.bit_diffs(get(f), g[prefix + f]) == 0, (prefix, f)
    assert get("objective") == float(g[prefix + "objective"][0]), prefix


def _composite(name):
    spec = COMPOSITE_SPECS[name]
    a, _ = composite_inputs(spec)
    return compose(pkg, spec["kind"], a)


# -- CPU: the oracle is pinned to the reference --------------------------------

@pytest.mark.parametrize("name", STAGES)
def test_oracle_extract_matches_reference(name):
    g = C.load("solution_" + name)
    case = stage_case(json.loads(str(g["spec"])))
    sol = OS.extract(case, _layout(case), g["x"])
    _same(sol, g, "ex_")
    dp, dq = OS.residuals(case, sol["va"], sol["vm"], sol["pg"], sol["qg"])
    assert C.bit_diffs(dp, g["ex_dp"]) == 0 and C.bit_diffs(dq, g["ex_dq"]) == 0
    fc = OS.from_case(case)
    _same(fc, g, "fc_")
    dp, dq = OS.residuals(case, fc["va"], fc["vm"], fc["pg"], fc["qg"])
    assert C.bit_diffs(dp, g["fc_dp"]) == 0 and C.bit_diffs(dq, g["fc_dq"]) == 0


@pytest.mark.parametrize("name", COMPOSITES)
def test_oracle_stage_extract_matches_reference(name):
    g = C.load("solution_" + name)
    _, imap = _composite(name)
    x = g["x"]
    assert len(imap.stages) == int(g["n_stages"][0])
    for k, st in enumerate(imap.stages):
        o, lay = imap.var_offset[k], imap.layouts[k]
        sol = OS.extract(st.case, lay, x[o:o + lay.n_vars])
        _same(sol, g, f"s{k}_")
        dp, dq = OS.residuals(st.case, sol["va"], sol["vm"], sol["pg"], sol["qg"])
        assert C.bit_diffs(dp, g[f"s{k}_dp"]) == 0 and C.bit_diffs(dq, g[f"s{k}_dq"]) == 0


@pytest.mark.parametrize("name", STAGES)
def test_pack_solution_matches_reference(name):
    g = C.load("solution_" + name)
    case = stage_case(json.loads(str(g["spec"])))
    _, lay = pkg.build_acopf(case)
    sol = S.SolvedCase(case=case, objective=float(g["ex_objective"][0]),
                       **{f: g["ex_" + f] for f in FIELDS})
    assert C.bit_diffs(S.pack_solution(case, lay, sol), g["packed"]) == 0


def test_shape_errors_before_any_device_work():
    case = stage_case(STAGE_SPECS["stage_ring9"])
    _, lay = pkg.build_acopf(case)
    with pytest.raises(pkg.DimensionMismatch):
        S.extract_solution(case, lay, np.zeros(lay.n_vars - 1))
    bad = S.SolvedCase(case=case, vm=np.zeros(3), va=np.zeros(3), pg=np.zeros(len(case.gens)),
                       qg=np.zeros(len(case.gens)), pf=None, qf=None, pt=None, qt=None, objective=0.0)
    with pytest.raises(pkg.DimensionMismatch):
        S.residuals_at(case, bad)
    with pytest.raises(IndexError):           # the reference's to_raw indexes vm per bus too
        bad.to_raw()


# -- GPU: the device flows mode -------------------------------------------------

@pytest.fixture(params=["0", "1"], ids=["gather", "interleaved"])
def bus_inputs(request, monkeypatch):
    """Both bus-input paths of the tile kernel (see test_gpu_parity.bus_inputs)."""
    monkeypatch.setenv("ACOPF_INTERLEAVE", request.param)
    return request.param


@pytest.mark.gpu
@pytest.mark.parametrize("name", STAGES)
def test_device_extract_matches_reference(name, bus_inputs):
    g = C.load("solution_" + name)
    case = stage_case(json.loads(str(g["spec"])))
    _, lay = pkg.build_acopf(case)
    sol = S.extract_solution(case, lay, g["x"])
    _same(sol, g, "ex_")
    dp, dq = S.residuals_at(case, sol)
    assert C.bit_diffs(dp, g["ex_dp"]) == 0 and C.bit_diffs(dq, g["ex_dq"]) == 0
    fc = S.solution_from_case(case)
    _same(fc, g, "fc_")
    dp, dq = S.residuals_at(case, fc)
    assert C.bit_diffs(dp, g["fc_dp"]) == 0 and C.bit_diffs(dq, g["fc_dq"]) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", COMPOSITES)
def test_device_composite_extract_matches_reference(name, bus_inputs):
    """All stages' flows from one launch over the composite evaluator."""
    g = C.load("solution_" + name)
    p, imap = _composite(name)
    sols = S.extract_solutions(p, imap, g["x"])
    assert len(sols) == int(g["n_stages"][0])
    for k, sol in enumerate(sols):
        _same(sol, g, f"s{k}_")
        dp, dq = S.residuals_at(sol.case, sol)
        assert C.bit_diffs(dp, g[f"s{k}_dp"]) == 0 and C.bit_diffs(dq, g[f"s{k}_dq"]) == 0


@pytest.mark.gpu
def test_device_residuals_large_case_vs_oracle():
    """10k-bus configuration: flows and residuals bit-identical to the oracle."""
    case = syn.config_case(1)
    p, lay = pkg.build_acopf(case)
    kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
    x, _ = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 5)
    sol = S.extract_solution(case, lay, x)
    ref = OS.extract(case, lay, x)
    _same(sol, {"o_" + k: (np.array([v]) if k == "objective" else v) for k, v in ref.items()}, "o_")
    dp, dq = S.residuals_at(case, sol)
    rdp, rdq = OS.residuals(case, sol.va, sol.vm, sol.pg, sol.qg)
    assert C.bit_diffs(dp, rdp) == 0 and C.bit_diffs(dq, rdq) == 0


@pytest.mark.gpu
def test_device_residuals_linear_in_dispatch():
    """Residuals are generation - load - injection: removing all dispatch moves
    each bus's residual by exactly its generation (up to rounding)."""
    case = stage_case(STAGE_SPECS["stage_feat200"])
    _, lay = pkg.build_acopf(case)
    fc = S.solution_from_case(case)
    dp, dq = S.residuals_at(case, fc)
    assert np.all(np.isfinite(dp)) and np.all(np.isfinite(dq))
    zero = S.SolvedCase(case=case, vm=fc.vm, va=fc.va, pg=np.zeros_like(fc.pg), qg=np.zeros_like(fc.qg),
                        pf=fc.pf, qf=fc.qf, pt=fc.pt, qt=fc.qt, objective=0.0)
    dp0, dq0 = S.residuals_at(case, zero)
    # moving all generation out changes each bus's residual by its generation exactly
    gen_p = np.zeros(len(case.buses))
    pos = {b.id: k for k, b in enumerate(case.buses)}
    for j, gn in enumerate(case.gens):
        if gn.status and case.buses[pos[gn.bus]].btype != pkg.ISOLATED:
            gen_p[pos[gn.bus]] += fc.pg[j]
    assert np.allclose(dp - dp0, gen_p, rtol=1e-12, atol=1e-9)
