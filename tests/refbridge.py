"""Test helper: import the real reference (build container only) and convert
this package's grid objects into the reference's own dataclasses.

The reference lives read-only at /root/reference (absent on GPU boxes), so
every user of this module must skip when :func:`opfkit` returns None.
"""

from __future__ import annotations

import dataclasses
import os
import sys

REF_SRC = "/root/reference/pkg/src"


def opfkit():
    """The reference package, or None where it is not mounted."""
    if not os.path.isdir(REF_SRC):
        return None
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    sys.dont_write_bytecode = True
    import opfkit as ok  # noqa: E402
    return ok


def _conv(obj, cls, **over):
    vals = {f.name: getattr(obj, f.name) for f in dataclasses.fields(cls)}
    vals.update(over)
    return cls(**vals)


def to_ref_case(case):
    ok = opfkit()
    net = ok.network
    buses = tuple(_conv(b, net.Bus) for b in case.buses)
    gens = tuple(_conv(g, net.Generator, cost=_conv(g.cost, net.GenCost)) for g in case.gens)
    branches = tuple(_conv(b, net.Branch) for b in case.branches)
    return net.NetworkCase(name=case.name, base_mva=case.base_mva, buses=buses,
                           gens=gens, branches=branches)


def to_ref_ctgs(ctgs):
    ok = opfkit()
    net = ok.network
    out = []
    for c in ctgs.contingencies:
        out.append(net.Contingency(id=c.id, outages=tuple(
            net.Outage(kind=o.kind, bus=o.bus, tbus=o.tbus, ordinal=o.ordinal)
            for o in c.outages)))
    return ok.inputs.ContingencySet(tuple(out))


def to_ref_scens(scens):
    ok = opfkit()
    net = ok.network
    return ok.inputs.ScenarioSet(tuple(
        net.Scenario(id=s.id, weight=s.weight, wind_targets=s.wind_targets)
        for s in scens.scenarios))


def to_ref_mode(mode):
    ok = opfkit()
    return ok.composer.CouplingMode(kind=mode.kind, pin_voltages=mode.pin_voltages,
                                    contingency_scale=mode.contingency_scale,
                                    scenario_scale=mode.scenario_scale)
