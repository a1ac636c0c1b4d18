"""Error semantics of the drop-in builders (CPU; planner only, no GPU).

Each case builds an invalid input and checks that this package raises the
reference's exception (same class name, same ``opfkit.errors`` hierarchy
position) at the same call: composer.py:55-66 (InvalidPlan on a coupling
kind), :112-126 (TopologyMismatch), :327-357 (EmptyScenarioSet, InvalidPlan),
network.py:296-357 (UnknownOutage, IslandingDetected, TargetOnNonWind),
acopf.py:97-99,398-400 (Disconnected).  Where the reference is mounted
(the build container), the same input is also fed to the reference and the
raised class names must agree.
"""

from dataclasses import replace

import pytest

import paper_2203_10587_b200 as pkg
import refbridge as rb
from paper_2203_10587_b200 import errors as E
from paper_2203_10587_b200 import synthetic as syn
from paper_2203_10587_b200.grid import (BRANCH, GEN, Contingency, ContingencySet, Outage, Scenario,
                                        ScenarioSet)
from paper_2203_10587_b200.types import CouplingMode


def _bridge(case):
    nb = set(syn.non_bridge_branches(case))
    return next(k for k, b in enumerate(case.branches) if b.status and k not in nb and b.fbus != b.tbus)


def _ctg_of(case, k, cid=1):
    br = case.branches[k]
    ordinal = case.branches_between(br.fbus, br.tbus).index(k) + 1
    return Contingency(cid, (Outage(BRANCH, br.fbus, br.tbus, ordinal),))


def _base():
    return syn.make_case(40, 12, 8, seed=5, features=True)


def _cases():
    """(name, expected error, call(api, conv)) -- conv maps this package's inputs to the api's."""
    base = _base()
    out = []
    bridge = ContingencySet((_ctg_of(base, _bridge(base)),))
    out.append(("bridge outage", E.IslandingDetected,
                lambda api, c: api.compose_scopf(c["case"](base), c["ctgs"](bridge), c["mode"](CouplingMode()))))
    nb = syn.non_bridge_branches(base)
    k1, k2 = nb[0], nb[1]
    double = ContingencySet((Contingency(1, _ctg_of(base, k1).outages + _ctg_of(base, k2).outages),))
    # a double outage of two non-bridges may or may not island; pick one that does if any
    nogen = ContingencySet((Contingency(1, (Outage(GEN, base.buses[-2].id, None, 7),)),))
    out.append(("generator that does not exist", E.UnknownOutage,
                lambda api, c: api.compose_scopf(c["case"](base), c["ctgs"](nogen), c["mode"](CouplingMode()))))
    br = base.branches[k1]
    nobr = ContingencySet((Contingency(1, (Outage(BRANCH, br.fbus, br.tbus, 9),)),))
    out.append(("branch ordinal out of range", E.UnknownOutage,
                lambda api, c: api.compose_scopf(c["case"](base), c["ctgs"](nobr), c["mode"](CouplingMode()))))
    off = next(k for k, b in enumerate(base.branches) if b.status == 0 and b.fbus != b.tbus)
    offc = ContingencySet((_ctg_of(base, off),))
    out.append(("branch already off", E.UnknownOutage,
                lambda api, c: api.compose_scopf(c["case"](base), c["ctgs"](offc), c["mode"](CouplingMode()))))
    other = replace(base, branches=tuple(replace(b, status=0) if i == k1 else b
                                         for i, b in enumerate(base.branches)))
    out.append(("periods with different topologies", E.TopologyMismatch,
                lambda api, c: api.compose_multiperiod([c["case"](base), c["case"](other)], 15.0)))
    out.append(("no periods", E.InvalidPlan,
                lambda api, c: api.compose_general(None, None, [], c["mode"](CouplingMode()), 15.0)))
    out.append(("non-positive dt with two periods", E.InvalidPlan,
                lambda api, c: api.compose_multiperiod([c["case"](base), c["case"](base)], 0.0)))
    out.append(("empty scenario set", E.EmptyScenarioSet,
                lambda api, c: api.compose_sopf_full(c["case"](base), c["scens"](ScenarioSet(())), None,
                                                     c["mode"](CouplingMode()))))
    g1 = base.gens[1]
    zero_w = ScenarioSet((Scenario(1, 0.0, ()), Scenario(2, 0.0, ())))
    out.append(("scenario weights sum to zero", E.EmptyScenarioSet,
                lambda api, c: api.compose_sopf_full(c["case"](base), c["scens"](zero_w), None,
                                                     c["mode"](CouplingMode()))))
    nonwind = ScenarioSet((Scenario(1, 1.0, (((g1.bus, 1), 50.0),)),))
    out.append(("target on a non-wind generator", E.TargetOnNonWind,
                lambda api, c: api.compose_sopf_full(c["case"](base), c["scens"](nonwind), None,
                                                     c["mode"](CouplingMode()))))
    split = replace(base, branches=tuple(replace(b, status=0) if i == _bridge(base) else b
                                         for i, b in enumerate(base.branches)))
    out.append(("disconnected stage network", E.Disconnected,
                lambda api, c: api.build_acopf(c["case"](split))))
    out.append(("disconnected composite period", E.Disconnected,
                lambda api, c: api.compose_scopf(c["case"](split), c["ctgs"](ContingencySet(())),
                                                 c["mode"](CouplingMode()))))
    del double
    return out


OURS = dict(case=lambda v: v, ctgs=lambda v: v, scens=lambda v: v, mode=lambda v: v)


@pytest.mark.parametrize("idx", range(12))
def test_builder_errors_match_reference(idx):
    name, exc, call = _cases()[idx]
    with pytest.raises(exc):
        call(pkg, OURS)
    ok = rb.opfkit()
    if ok is None:
        return                              # GPU box: the reference is not mounted
    conv = dict(case=rb.to_ref_case, ctgs=rb.to_ref_ctgs, scens=rb.to_ref_scens, mode=rb.to_ref_mode)
    with pytest.raises(Exception) as info:
        call(ok, conv)
    assert type(info.value).__name__ == exc.__name__, (name, type(info.value).__name__)


def test_invalid_coupling_kind():
    with pytest.raises(E.InvalidPlan):
        CouplingMode(kind="bogus")


def test_errors_are_caught_by_the_reference_classes_when_it_is_importable():
    """With opfkit importable, each error also derives from the same-named opfkit.errors class, so
    callers that catch the reference's exceptions keep working after the switch."""
    if rb.opfkit() is None:
        pytest.skip("reference not mounted")
    import subprocess
    import sys
    code = (f"import sys; sys.path.insert(0, {rb.REF_SRC!r}); import opfkit\n"
            "import paper_2203_10587_b200 as pkg\n"
            "from paper_2203_10587_b200 import errors as E, synthetic as syn\n"
            "for n in ('IslandingDetected', 'UnknownOutage', 'TopologyMismatch', 'EmptyScenarioSet',\n"
            "          'InvalidPlan', 'TargetOnNonWind', 'Disconnected', 'DimensionMismatch'):\n"
            "    assert issubclass(getattr(E, n), getattr(opfkit.errors, n)), n\n"
            "    assert issubclass(getattr(E, n), E.OpfkitError), n\n"
            "from dataclasses import replace\n"
            "case = syn.make_case(12, 0, 3, seed=2)\n"
            "try:\n"
            "    pkg.build_acopf(replace(case, branches=case.branches[1:]))\n"
            "except opfkit.errors.Disconnected:\n"
            "    print('caught')\n")
    import os
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(sys.path))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    assert r.returncode == 0 and "caught" in r.stdout, r.stderr
