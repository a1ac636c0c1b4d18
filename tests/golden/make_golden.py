"""Generate the golden fixtures in this directory from the REAL reference.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on GPU boxes):

    python tests/golden/make_golden.py

Every fixture is one seeded synthetic input (rebuilt in tests from the
``spec`` JSON through ``paper_2203_10587_b200.synthetic``) evaluated by the
reference's own ``build_acopf`` / ``compose_*`` callbacks: objective,
gradient, constraints, Jacobian and Lagrangian-Hessian CSR, bounds and
(for composites) offsets and coupling rows.  ``case_digest`` pins the
generator: a test fails if the synthetic inputs drift.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2203_10587_b200 import synthetic as syn  # noqa: E402
from paper_2203_10587_b200.types import CouplingMode  # noqa: E402

STAGE_SPECS = {
    "stage_ring9": dict(nb=9, nc=0, ng=3, seed=9, ring=True, features=False, points=3),
    "stage_feat30": dict(nb=30, nc=10, ng=6, seed=30, ring=False, features=True, points=3),
    "stage_feat200": dict(nb=200, nc=60, ng=40, seed=200, ring=False, features=True, points=2),
    "stage_synth2000": dict(nb=2000, nc=600, ng=500, seed=2000, ring=False, features=False, points=1),
}

COMPOSITE_SPECS = {
    "scopf_corrective": dict(kind="scopf", nb=60, nc=20, ng=12, n_ctg=6, features=True,
                             mode=dict(kind="corrective")),
    "scopf_preventive": dict(kind="scopf", nb=60, nc=20, ng=12, n_ctg=6, features=True,
                             mode=dict(kind="preventive", pin_voltages=True)),
    "multiperiod": dict(kind="multiperiod", nb=50, nc=15, ng=10, n_periods=5, dt=15.0),
    "general": dict(kind="general", nb=80, nc=25, ng=20, n_scen=3, n_ctg=2, n_periods=2, dt=15.0,
                    mode=dict(kind="preventive")),
    "sopf_flat": dict(kind="flat", nb=80, nc=25, ng=20, n_scen=3, n_ctg=2,
                      mode=dict(kind="corrective", contingency_scale=0.5, scenario_scale=2.0)),
}


def case_digest(case) -> str:
    """Stable hash of every field of a case (pins the synthetic generator)."""
    h = hashlib.sha256()
    for b in case.buses:
        h.update(repr((b.id, b.btype, b.pd, b.qd, b.gs, b.bs, b.vm, b.va, b.vmin, b.vmax)).encode())
    for g in case.gens:
        h.update(repr((g.bus, g.status, g.pmin, g.pmax, g.qmin, g.qmax, g.ramp_30, g.cost.c2,
                       g.cost.c1, g.cost.c0, g.is_wind)).encode())
    for br in case.branches:
        h.update(repr((br.fbus, br.tbus, br.r, br.x, br.b, br.rate_a, br.ratio, br.angle,
                       br.status)).encode())
    return h.hexdigest()


def stage_case(spec):
    return syn.make_case(spec["nb"], spec["nc"], spec["ng"], seed=spec["seed"], ring=spec["ring"],
                         features=spec["features"])


def composite_inputs(spec):
    """(kind, args for compose_*, list of base cases) rebuilt from a spec."""
    kind = spec["kind"]
    mode = CouplingMode(**spec.get("mode", {}))
    size = dict(nb=spec["nb"], n_chords=spec["nc"], ng=spec["ng"])
    if kind == "scopf":
        base, ctgs = syn.config2_inputs(n_ctg=spec["n_ctg"], features=spec.get("features", False), **size)
        return dict(base=base, ctgs=ctgs, mode=mode), [base]
    if kind == "multiperiod":
        periods = syn.config3_periods(spec["n_periods"], **size)
        return dict(periods=periods, dt=spec["dt"]), periods
    base, scens, ctgs = syn.config4_inputs(n_scen=spec["n_scen"], n_ctg=spec["n_ctg"], **size)
    if kind == "general":
        return dict(scens=scens, ctgs=ctgs, periods=[base] * spec["n_periods"], mode=mode,
                    dt=spec["dt"]), [base]
    return dict(base=base, scens=scens, ctgs=ctgs, mode=mode), [base]


def compose(api, kind, a, conv=None):
    """Call the right compose_* of ``api`` (reference module or this package)."""
    c = conv or (lambda kind_, v: v)
    if kind == "scopf":
        return api.compose_scopf(c("case", a["base"]), c("ctgs", a["ctgs"]), c("mode", a["mode"]))
    if kind == "multiperiod":
        return api.compose_multiperiod([c("case", p) for p in a["periods"]], a["dt"])
    if kind == "general":
        return api.compose_general(c("scens", a["scens"]), c("ctgs", a["ctgs"]),
                                   [c("case", p) for p in a["periods"]], c("mode", a["mode"]), a["dt"])
    return api.compose_sopf_flat(c("case", a["base"]), c("scens", a["scens"]), c("ctgs", a["ctgs"]),
                                 c("mode", a["mode"]))


def variable_kinds_from_layouts(layouts):
    return syn.variable_kinds([(len(l.va), len(l.pg)) for l in layouts])


def dump(path, p, points, extra):
    out = dict(extra)
    out["n"], out["m_eq"], out["m_ineq"] = p.n, p.m_eq, p.m_ineq
    for a in ("xl", "xu", "x0", "gl", "gu"):
        out[a] = getattr(p, a)
    for i, (x, mult, of) in enumerate(points):
        out[f"px{i}"], out[f"pmult{i}"], out[f"pof{i}"] = x, mult, of
        out[f"obj{i}"] = np.array([p.objective(x)])
        out[f"grad{i}"] = p.gradient(x)
        out[f"cons{i}"] = p.constraints(x)
        J = p.jacobian(x)
        H = p.lagrangian_hessian(x, of, mult)
        out[f"jdata{i}"], out[f"hdata{i}"] = J.data, H.data
        if i == 0:
            out["jindptr"], out["jindices"] = J.indptr, J.indices
            out["hindptr"], out["hindices"] = H.indptr, H.indices
    out["npoints"] = len(points)
    np.savez_compressed(path, **out)


def main():
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        raise SystemExit("reference not mounted at /root/reference")
    for name, spec in STAGE_SPECS.items():
        case = stage_case(spec)
        p, lay = ok.build_acopf(rb.to_ref_case(case))
        kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
        pts = []
        for s in range(spec["points"]):
            x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 1000 + s)
            pts.append((x, mult, 1.0 + 0.25 * s))
        dump(os.path.join(HERE, name + ".npz"), p, pts,
             dict(spec=json.dumps(spec), case_digest=case_digest(case)))
        print(name, p.n, p.m_eq + p.m_ineq)
    conv_map = dict(case=rb.to_ref_case, ctgs=rb.to_ref_ctgs, scens=rb.to_ref_scens, mode=rb.to_ref_mode)
    for name, spec in COMPOSITE_SPECS.items():
        a, bases = composite_inputs(spec)
        p, imap = compose(ok, spec["kind"], a, conv=lambda k, v: conv_map[k](v))
        kinds = variable_kinds_from_layouts(imap.layouts)
        pts = []
        for s in range(2):
            x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 2000 + s)
            pts.append((x, mult, 0.5 + s))
        rows = np.array([[r.stage_a, r.stage_b, -1 if r.gen is None else r.gen,
                          -1 if r.bus is None else r.bus, r.row, int(r.is_equality)]
                         for r in imap.coupling_rows], dtype=np.int64).reshape(-1, 6)
        kinds_s = np.array([r.kind for r in imap.coupling_rows])
        bounds = np.array([r.bound for r in imap.coupling_rows], dtype=np.float64)
        dump(os.path.join(HERE, name + ".npz"), p, pts,
             dict(spec=json.dumps(spec), case_digest=case_digest(bases[0]),
                  var_offset=np.array(imap.var_offset), eq_offset=np.array(imap.eq_offset),
                  ineq_offset=np.array(imap.ineq_offset), weights=np.array(imap.weights),
                  cp_rows=rows, cp_kinds=kinds_s, cp_bounds=bounds))
        print(name, p.n, p.m_eq + p.m_ineq, len(imap.coupling_rows))


SOLUTION_STAGES = ["stage_ring9", "stage_feat30", "stage_feat200"]
SOLUTION_FIELDS = ("vm", "va", "pg", "qg", "pf", "qf", "pt", "qt")


def _dump_solution(out, prefix, sol, ok):
    for f in SOLUTION_FIELDS:
        out[prefix + f] = getattr(sol, f)
    out[prefix + "objective"] = np.array([sol.objective])
    dp, dq = ok.residuals_at(sol.case, sol)
    out[prefix + "dp"], out[prefix + "dq"] = dp, dq


def solutions():
    """solution_*.npz: extract_solution / solution_from_case / residuals_at (acopf.py:413-546)."""
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        raise SystemExit("reference not mounted at /root/reference")
    for name in SOLUTION_STAGES:
        spec = STAGE_SPECS[name]
        case = stage_case(spec)
        rc = rb.to_ref_case(case)
        p, lay = ok.build_acopf(rc)
        kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
        x, _ = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 3000)
        out = dict(spec=json.dumps(spec), case_digest=case_digest(case), x=x)
        sol = ok.extract_solution(rc, lay, x)
        _dump_solution(out, "ex_", sol, ok)
        out["packed"] = ok.pack_solution(rc, lay, sol)
        _dump_solution(out, "fc_", ok.solution_from_case(rc), ok)
        np.savez_compressed(os.path.join(HERE, "solution_" + name + ".npz"), **out)
        print("solution", name)
    conv_map = dict(case=rb.to_ref_case, ctgs=rb.to_ref_ctgs, scens=rb.to_ref_scens, mode=rb.to_ref_mode)
    for name in ("scopf_corrective", "general"):
        spec = COMPOSITE_SPECS[name]
        a, bases = composite_inputs(spec)
        p, imap = compose(ok, spec["kind"], a, conv=lambda k, v: conv_map[k](v))
        kinds = variable_kinds_from_layouts(imap.layouts)
        x, _ = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 3001)
        out = dict(spec=json.dumps(spec), case_digest=case_digest(bases[0]), x=x,
                   n_stages=np.array([len(imap.stages)]))
        for k, st in enumerate(imap.stages):
            o, lay = imap.var_offset[k], imap.layouts[k]
            _dump_solution(out, f"s{k}_", ok.extract_solution(st.case, lay, x[o:o + lay.n_vars]), ok)
        np.savez_compressed(os.path.join(HERE, "solution_" + name + ".npz"), **out)
        print("solution", name, len(imap.stages))


# ---------------------------------------------------------------------------
# the reference's own test fixtures (pkg/tests/conftest.py:20-57): case9.m, ctgc.cont,
# scenarios.csv, load_p.csv / load_q.csv, parsed by the reference's own readers and
# evaluated by its own build_acopf / compose_*; the parsed inputs are stored (as this
# package's dataclass fields) next to the outputs, so the GPU box needs no reference files

REF_DATA = "/root/reference/pkg/tests/data"


def _to_ours(ok, case):
    import common as C
    return C.case_to_json(case)


def fixture_inputs(ok):
    """Reference-parsed fixtures: (case9, ctgs, scens, period cases)."""
    case9 = ok.load_case(os.path.join(REF_DATA, "case9.m"))
    ctgs = ok.parse_contingencies_file(os.path.join(REF_DATA, "ctgc.cont"))
    scens = ok.parse_scenarios_file(os.path.join(REF_DATA, "scenarios.csv"))
    prof = ok.parse_load_profile_files(os.path.join(REF_DATA, "load_p.csv"), os.path.join(REF_DATA, "load_q.csv"))
    periods = [ok.network.apply_load_step(case9, prof, t) for t in range(len(prof.times))]
    return case9, ctgs, scens, periods


FIXTURE_SPECS = {
    # name: (builder, args) over the reference fixtures; mirrors pkg/tests/test_composer.py usage
    "ref_case9_scopf_corrective": ("scopf", dict(mode=dict(kind="corrective"))),
    "ref_case9_scopf_preventive": ("scopf", dict(mode=dict(kind="preventive", pin_voltages=True))),
    "ref_case9_general": ("general", dict(n_ctg=2, n_periods=2, dt=5.0, mode=dict(kind="preventive"))),
    "ref_case9_multiperiod": ("multiperiod", dict(dt=5.0)),
    "ref_case9_sopf_full": ("sopf_full", dict(mode=dict(kind="corrective"))),
    "ref_case9_mp_scopf": ("mp_scopf", dict(n_ctg=3, dt=5.0, mode=dict(kind="corrective"))),
}


def fixture_compose(api, kind, args, case9, ctgs, scens, periods, mode, trunc):
    """compose_* of ``api`` (the reference or this package) for one FIXTURE_SPECS entry."""
    if kind == "scopf":
        return api.compose_scopf(case9, ctgs, mode)
    if kind == "general":
        return api.compose_general(scens, trunc(ctgs, args["n_ctg"]), [case9] * args["n_periods"], mode, args["dt"])
    if kind == "multiperiod":
        return api.compose_multiperiod(periods, args["dt"])
    if kind == "sopf_full":
        return api.compose_sopf_full(case9, scens, ctgs, mode)
    return api.compose_multiperiod_scopf(periods, trunc(ctgs, args["n_ctg"]), mode, args["dt"])


def fixtures():
    """ref_case9_*.npz: the reference's fixtures through its own stage and composite builders,
    at seeded points (one with branch angles up to ~pi, glibc's wide-range sin/cos)."""
    import common as C
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        raise SystemExit("reference not mounted at /root/reference")
    case9, ctgs, scens, periods = fixture_inputs(ok)
    inputs = dict(case=C.case_to_json(case9), ctgs=C.ctgs_to_json(ctgs), scens=C.scens_to_json(scens),
                  periods=json.dumps([json.loads(C.case_to_json(c)) for c in periods]))
    # stage: x0 plus seeded points, one with large branch angles
    p, lay = ok.build_acopf(case9)
    kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
    pts = [(p.x0.copy(), np.ones(p.m_eq + p.m_ineq), 1.0)]
    for s in range(2):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 4000 + s)
        pts.append((x, mult, 1.0 + 0.5 * s))
    x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 4100)
    va = kinds == syn.VA
    x[va] = np.random.default_rng(4101).uniform(-1.6, 1.6, int(va.sum()))
    x[p.xl == p.xu] = p.xl[p.xl == p.xu]
    pts.append((x, mult, 1.0))
    dump(os.path.join(HERE, "ref_case9_stage.npz"), p, pts, dict(spec=json.dumps(dict(kind="stage")), **inputs))
    print("ref_case9_stage", p.n, p.m_eq + p.m_ineq)
    trunc = lambda c, n: c.truncated(n)
    for name, (kind, args) in FIXTURE_SPECS.items():
        mode = ok.composer.CouplingMode(**args.get("mode", {}))
        p, imap = fixture_compose(ok, kind, args, case9, ctgs, scens, periods, mode, trunc)
        kinds = variable_kinds_from_layouts(imap.layouts)
        pts = []
        for s in range(2):
            x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 4200 + s)
            pts.append((x, mult, 0.75 + s))
        rows = np.array([[r.stage_a, r.stage_b, -1 if r.gen is None else r.gen,
                          -1 if r.bus is None else r.bus, r.row, int(r.is_equality)]
                         for r in imap.coupling_rows], dtype=np.int64).reshape(-1, 6)
        dump(os.path.join(HERE, name + ".npz"), p, pts,
             dict(spec=json.dumps(dict(kind=kind, **args)), **inputs,
                  var_offset=np.array(imap.var_offset), eq_offset=np.array(imap.eq_offset),
                  ineq_offset=np.array(imap.ineq_offset), weights=np.array(imap.weights),
                  cp_rows=rows, cp_kinds=np.array([r.kind for r in imap.coupling_rows]),
                  cp_bounds=np.array([r.bound for r in imap.coupling_rows], dtype=np.float64)))
        print(name, p.n, p.m_eq + p.m_ineq, len(imap.coupling_rows))


def configs():
    """cfg0_stage.npz: BASELINE config 0 (the 9-bus ring at CONFIG_SEEDS[0]) from the reference,
    at 4 seeded points; cfg_feat200_wide.npz: a 200-bus feature network at branch angles up to
    ~pi (Va ~ U(-1.6, 1.6)), the non-table paths of glibc's sin/cos."""
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        raise SystemExit("reference not mounted at /root/reference")
    case = syn.config_case(0)
    p, lay = ok.build_acopf(rb.to_ref_case(case))
    kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
    pts = []
    for s in range(4):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, syn.CONFIG_SEEDS[0] + s)
        pts.append((x, mult, 1.0))
    dump(os.path.join(HERE, "cfg0_stage.npz"), p, pts,
         dict(spec=json.dumps(dict(config=0)), case_digest=case_digest(case)))
    print("cfg0_stage", p.n, p.m_eq + p.m_ineq)
    spec = STAGE_SPECS["stage_feat200"]
    case = stage_case(spec)
    p, lay = ok.build_acopf(rb.to_ref_case(case))
    kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
    pts = []
    for s in range(3):
        x, mult = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 5000 + s)
        va = kinds == syn.VA
        x[va] = np.random.default_rng(5100 + s).uniform(-1.6, 1.6, int(va.sum()))
        x[p.xl == p.xu] = p.xl[p.xl == p.xu]
        pts.append((x, mult, 1.0))
    dump(os.path.join(HERE, "cfg_feat200_wide.npz"), p, pts,
         dict(spec=json.dumps(spec), case_digest=case_digest(case)))
    print("cfg_feat200_wide", p.n)


def writer():
    """matpower_text.npz: the reference's write_case text (matpower.py:180-187) of solved cases --
    extract_solution outputs of the stage goldens' cases and of case9 (reference-parsed, with
    its ramp / tail columns) at seeded points."""
    import common as C
    import refbridge as rb
    ok = rb.opfkit()
    if ok is None:
        raise SystemExit("reference not mounted at /root/reference")
    out = {}
    case9, _, _, _ = fixture_inputs(ok)
    cases = [("case9", case9, C.case_to_json(case9))]
    for name in ("stage_ring9", "stage_feat30", "stage_feat200"):
        c = stage_case(STAGE_SPECS[name])
        cases.append((name, rb.to_ref_case(c), C.case_to_json(c)))
    for i, (name, rc, js) in enumerate(cases):
        p, lay = ok.build_acopf(rc)
        kinds = syn.variable_kinds([(len(lay.va), len(lay.pg))])
        x, _ = syn.random_point(kinds, p.xl, p.xu, p.m_eq + p.m_ineq, 6000 + i)
        sol = ok.extract_solution(rc, lay, x)
        out[f"case{i}"] = js
        out[f"x{i}"] = x
        out[f"text{i}"] = ok.matpower.write_case(sol, name=f"t_{i}")
        out[f"text_default{i}"] = ok.matpower.write_case(sol)
    out["n"] = len(cases)
    np.savez_compressed(os.path.join(HERE, "matpower_text.npz"), **out)
    print("matpower_text", len(cases))


if __name__ == "__main__":
    if sys.argv[1:] == ["solutions"]:
        solutions()
    elif sys.argv[1:] == ["fixtures"]:
        fixtures()
    elif sys.argv[1:] == ["configs"]:
        configs()
    elif sys.argv[1:] == ["writer"]:
        writer()
    else:
        main()
