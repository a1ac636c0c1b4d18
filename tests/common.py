"""Shared helpers for the parity tests (golden fixtures, comparisons)."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_2203_10587_b200 import synthetic as syn

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STAGE_FIXTURES = ["stage_ring9", "stage_feat30", "stage_feat200", "stage_synth2000"]
COMPOSITE_FIXTURES = ["scopf_corrective", "scopf_preventive", "multiperiod", "general", "sopf_flat"]

# the parity gate of BASELINE.json north_star: |a - b| <= 1e-14 + 1e-12 |b|
ATOL, RTOL = 1e-14, 1e-12


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    return {k: z[k] for k in z.files}


def spec(g):
    return json.loads(str(g["spec"]))


REPORT = {}


def record(name, **kw):
    """Add one comparison to the parity report (PARITY_REPORT=<path> writes it as JSON)."""
    REPORT.setdefault(name, {}).update(kw)
    out = os.environ.get("PARITY_REPORT")
    if out:
        with open(out, "w") as fh:
            json.dump(REPORT, fh, indent=1, sort_keys=True)


def gate_misses(a, b) -> int:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    ok = np.abs(a - b) <= ATOL + RTOL * np.abs(b)
    ok |= (a == b) | (np.isnan(a) & np.isnan(b))
    return int(np.count_nonzero(~ok))


def bit_diffs(a, b) -> int:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return int(np.count_nonzero(a.view(np.int64) != b.view(np.int64)))


def points(g):
    return [(g[f"px{i}"], g[f"pmult{i}"], float(g[f"pof{i}"])) for i in range(int(g["npoints"]))]


def hub_case(n_hub=200, n_gen_hub=150, seed=5):
    """A network with one hub bus carrying n_hub extra branches (half as the from-bus, half as
    the to-bus, some parallel) and n_gen_hub generators: exercises a tile whose one bus has
    more branch ends than the tile CTA has threads (128), long duplicate sums, and more
    generators than threads per tile."""
    from dataclasses import replace
    case = syn.make_case(200, 40, 20, seed=seed, features=True)
    rng = np.random.default_rng(seed)
    hub = case.buses[3].id
    others = [b.id for b in case.buses if b.id != hub and b.btype != 4]
    extra = []
    for k, j in enumerate(rng.choice(others, size=n_hub, replace=True)):
        base = case.branches[k % 50]
        fb, tb = (hub, int(j)) if k % 2 == 0 else (int(j), hub)
        extra.append(replace(base, fbus=fb, tbus=tb, r=float(rng.uniform(0.005, 0.02)),
                             x=float(rng.uniform(0.05, 0.2)), status=1))
    g0 = case.gens[1]
    gens = [replace(g0, bus=hub, pmax=float(rng.uniform(50, 300)),
                    cost=replace(g0.cost, c1=float(rng.uniform(1, 40)))) for _ in range(n_gen_hub)]
    return replace(case, branches=case.branches + tuple(extra), gens=case.gens + tuple(gens))


# -- case / input (de)serialisation for the reference-fixture goldens ---------------------------

def case_to_json(case) -> str:
    import dataclasses
    d = dict(name=case.name, base_mva=case.base_mva,
             buses=[dataclasses.asdict(b) for b in case.buses],
             gens=[dict(dataclasses.asdict(g), cost=dataclasses.asdict(g.cost)) for g in case.gens],
             branches=[dataclasses.asdict(b) for b in case.branches])
    return json.dumps(d)


def _tup(v):
    return tuple(_tup(x) for x in v) if isinstance(v, list) else v


def case_from_json(s):
    """This package's NetworkCase from case_to_json output (fields of the reference's dataclasses)."""
    from paper_2203_10587_b200.grid import Branch, Bus, GenCost, Generator, NetworkCase
    d = json.loads(s) if isinstance(s, str) else s
    fix = lambda r: {k: _tup(v) for k, v in r.items()}
    buses = tuple(Bus(**fix(b)) for b in d["buses"])
    gens = tuple(Generator(**dict(fix(g), cost=GenCost(**fix(g["cost"])))) for g in d["gens"])
    branches = tuple(Branch(**fix(b)) for b in d["branches"])
    return NetworkCase(name=d["name"], base_mva=d["base_mva"], buses=buses, gens=gens, branches=branches)


def ctgs_to_json(ctgs) -> str:
    return json.dumps([[c.id, [[o.kind, o.bus, o.tbus, o.ordinal] for o in c.outages]]
                       for c in ctgs.contingencies])


def ctgs_from_json(s):
    from paper_2203_10587_b200.grid import Contingency, ContingencySet, Outage
    return ContingencySet(tuple(Contingency(id=i, outages=tuple(Outage(k, b, t, o) for k, b, t, o in outs))
                                for i, outs in json.loads(s)))


def scens_to_json(scens) -> str:
    return json.dumps([[s.id, s.weight, [[list(k), v] for k, v in s.wind_targets]] for s in scens.scenarios])


def scens_from_json(s):
    from paper_2203_10587_b200.grid import Scenario, ScenarioSet
    return ScenarioSet(tuple(Scenario(id=i, weight=w, wind_targets=tuple((tuple(k), v) for k, v in wt))
                             for i, w, wt in json.loads(s)))


# -- the reference's own fixtures (tests/golden/ref_case9_*.npz, make_golden.py fixtures) --------

REF_FIXTURES = ["ref_case9_scopf_corrective", "ref_case9_scopf_preventive", "ref_case9_general",
                "ref_case9_multiperiod", "ref_case9_sopf_full", "ref_case9_mp_scopf"]


def ref_fixture_inputs(g):
    """(case9, ctgs, scens, periods) of a ref_case9_* golden, as this package's dataclasses."""
    case9 = case_from_json(str(g["case"]))
    ctgs = ctgs_from_json(str(g["ctgs"]))
    scens = scens_from_json(str(g["scens"]))
    periods = [case_from_json(c) for c in json.loads(str(g["periods"]))]
    return case9, ctgs, scens, periods


def ref_fixture_args(g):
    """(kind, args, inputs, CouplingMode kwargs) of a ref_case9_* composite golden."""
    sp = spec(g)
    kind = sp.pop("kind")
    mode = sp.pop("mode", {})
    return kind, sp, ref_fixture_inputs(g), mode


def truncate_ctgs(ctgs, n):
    from paper_2203_10587_b200.grid import ContingencySet
    return ContingencySet(tuple(ctgs.by_id()[:n]))


def ref_fixture_compose(api, g, mode_cls):
    """Compose a ref_case9_* fixture with ``api`` (this package)."""
    from golden.make_golden import fixture_compose
    kind, args, (case9, ctgs, scens, periods), mode = ref_fixture_args(g)
    return fixture_compose(api, kind, args, case9, ctgs, scens, periods, mode_cls(**mode), truncate_ctgs)


def ref_fixture_oracle(g):
    """The oracle's composite for a ref_case9_* golden (compose_* are _general_impl, composer.py:391-432)."""
    from oracle.composite import CompositeOracle
    from paper_2203_10587_b200.types import CouplingMode
    kind, args, (case9, ctgs, scens, periods), mode = ref_fixture_args(g)
    mode = CouplingMode(**mode)
    if kind == "scopf":
        return CompositeOracle.general(None, ctgs, [case9], mode, 30.0)
    if kind == "general":
        return CompositeOracle.general(scens, truncate_ctgs(ctgs, args["n_ctg"]), [case9] * args["n_periods"],
                                       mode, args["dt"])
    if kind == "multiperiod":
        return CompositeOracle.general(None, None, periods, mode, args["dt"])
    if kind == "sopf_full":
        return CompositeOracle.general(scens, ctgs, [case9], mode, 30.0)
    return CompositeOracle.general(None, truncate_ctgs(ctgs, args["n_ctg"]), periods, mode, args["dt"])
