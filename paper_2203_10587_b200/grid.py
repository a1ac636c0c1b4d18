"""Typed grid model consumed by the packer, plus the per-stage transforms.

This is the *input side* of the hot path:
the dataclasses carry the same field names as the reference's
``opfkit.network`` types (`pkg/src/opfkit/network.py:31-153`) so either the
reference's own ``NetworkCase`` objects or these can be handed to
:func:`paper_2203_10587_b200.build_acopf` / ``compose_*`` (duck typing: only
attribute reads are used).  Transforms return new cases and never mutate
their inputs, like the reference's (`network.py:312-388`).

Units follow the reference: loads and generator limits in MW / MVAr,
impedances per unit, angles in radians.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from functools import cached_property

from .errors import (
    EmptyScenarioSet,
    IndexOutOfRange,
    IslandingDetected,
    TargetOnNonWind,
    UnknownBus,
    UnknownOutage,
)

# bus types (MATPOWER numbering, network.py:28)
PQ, PV, REF, ISOLATED = 1, 2, 3, 4
# outage kinds (network.py:265)
GEN, BRANCH = "GEN", "BRANCH"


@dataclass(frozen=True)
class Bus:
    id: int
    btype: int
    pd: float
    qd: float
    gs: float
    bs: float
    area: int
    vm: float
    va: float
    base_kv: float
    zone: int
    vmax: float
    vmin: float
    extra: tuple = ()


@dataclass(frozen=True)
class GenCost:
    c2: float
    c1: float
    c0: float
    startup: float = 0.0
    shutdown: float = 0.0
    ncost: int = 3

    def is_zero(self) -> bool:
        return not (self.c2 or self.c1 or self.c0)

    def at(self, p_mw: float) -> float:
        return (self.c2 * p_mw + self.c1) * p_mw + self.c0


@dataclass(frozen=True)
class Generator:
    bus: int
    pg: float
    qg: float
    qmax: float
    qmin: float
    vg: float
    mbase: float
    status: int
    pmax: float
    pmin: float
    ramp_30: float
    cost: GenCost
    is_wind: bool
    tail: tuple = ()


@dataclass(frozen=True)
class Branch:
    fbus: int
    tbus: int
    r: float
    x: float
    b: float
    rate_a: float
    rate_b: float
    rate_c: float
    ratio: float
    angle: float
    status: int
    angmin: float
    angmax: float
    extra: tuple = ()

    @property
    def tap(self) -> complex:
        """Complex tap ratio; ratio 0 means no transformer (network.py:101-104)."""
        m = 1.0 if self.ratio == 0.0 else self.ratio
        return m * complex(math.cos(self.angle), math.sin(self.angle))


@dataclass(frozen=True)
class NetworkCase:
    name: str
    base_mva: float
    buses: tuple
    gens: tuple
    branches: tuple

    @cached_property
    def bus_pos(self) -> dict:
        return {b.id: k for k, b in enumerate(self.buses)}

    @cached_property
    def _gens_by_bus(self) -> dict:
        out = {}
        for k, g in enumerate(self.gens):
            out.setdefault(g.bus, []).append(k)
        return out

    @cached_property
    def _branches_by_ends(self) -> dict:
        out = {}
        for k, br in enumerate(self.branches):
            out.setdefault((br.fbus, br.tbus), []).append(k)
        return out

    def gens_at(self, bus_id: int) -> list:
        """Positions of the generators at a bus, case order (network.py:120-122)."""
        return list(self._gens_by_bus.get(bus_id, ()))

    def branches_between(self, fbus: int, tbus: int) -> list:
        """Positions of the branches fbus -> tbus, case order (network.py:124-127)."""
        return list(self._branches_by_ends.get((fbus, tbus), ()))


@dataclass(frozen=True)
class Outage:
    kind: str
    bus: int
    tbus: int | None
    ordinal: int


@dataclass(frozen=True)
class Contingency:
    id: int
    outages: tuple


@dataclass(frozen=True)
class Scenario:
    id: int
    weight: float
    wind_targets: tuple


@dataclass(frozen=True)
class LoadProfile:
    times: tuple
    buses: tuple
    pd: tuple
    qd: tuple


@dataclass(frozen=True)
class ContingencySet:
    """Ordered contingency list (reference: inputs.py:42-58)."""
    contingencies: tuple

    def __len__(self) -> int:
        return len(self.contingencies)

    def __iter__(self):
        return iter(self.contingencies)

    def by_id(self) -> tuple:
        return tuple(sorted(self.contingencies, key=lambda c: c.id))

    def truncated(self, nc: int) -> "ContingencySet":
        return ContingencySet(self.contingencies[:max(nc, 0)])


@dataclass(frozen=True)
class ScenarioSet:
    """Weighted scenario list (reference: inputs.py:61-95)."""
    scenarios: tuple

    def __len__(self) -> int:
        return len(self.scenarios)

    def __iter__(self):
        return iter(self.scenarios)

    @property
    def total_weight(self) -> float:
        return sum(s.weight for s in self.scenarios)

    def base_index(self) -> int:
        """Most probable scenario, ties to the lowest id."""
        if not self.scenarios:
            raise EmptyScenarioSet("no scenarios")
        order = sorted(range(len(self.scenarios)),
                       key=lambda k: (-self.scenarios[k].weight,
                                      self.scenarios[k].id))
        return order[0]

    def wind_keys(self) -> tuple:
        keys: dict = {}
        for s in self.scenarios:
            for key, _ in s.wind_targets:
                keys.setdefault(key, None)
        return tuple(keys)

    def truncated(self, ns: int) -> "ScenarioSet":
        return ScenarioSet(self.scenarios[:max(ns, 0)])


# ---------------------------------------------------------------------------
# admittances and connectivity (packer inputs)

def branch_admittance(br) -> tuple:
    """(yff, yft, ytf, ytt) of the pi model, in CPython ``complex``.

    Same formulas as network.py:215-229; evaluated with Python complex
    arithmetic on purpose so the packed doubles are bit-identical to the
    reference's (CPython's complex division is part of the contract).
    """
    ys = 1.0 / complex(br.r, br.x)
    half_b = complex(0.0, br.b / 2.0)
    t = br.tap
    tc = t.conjugate()
    return (ys + half_b) / (t * tc), -ys / tc, -ys / t, ys + half_b


def check_connectivity(case) -> tuple:
    """(island count, per-bus label) over in-service branches (network.py:232-262).

    Isolated (type 4) buses carry label -1 and are not counted.
    """
    pos = case.bus_pos
    nbus = len(case.buses)
    alive = [b.btype != ISOLATED for b in case.buses]
    nbrs: list = [[] for _ in range(nbus)]
    for br in case.branches:
        if br.status == 0:
            continue
        a, b = pos[br.fbus], pos[br.tbus]
        if alive[a] and alive[b]:
            nbrs[a].append(b)
            nbrs[b].append(a)
    label = [-1] * nbus
    count = 0
    for root in range(nbus):
        if not alive[root] or label[root] >= 0:
            continue
        label[root] = count
        todo = [root]
        while todo:
            u = todo.pop()
            for v in nbrs[u]:
                if label[v] < 0:
                    label[v] = count
                    todo.append(v)
        count += 1
    return count, label


# ---------------------------------------------------------------------------
# stage transforms

def _gen_index(case, bus: int, ordinal: int) -> int:
    hits = case.gens_at(bus)
    if not 1 <= ordinal <= len(hits):
        raise UnknownOutage(f"no generator #{ordinal} at bus {bus}")
    return hits[ordinal - 1]


def _branch_index(case, fbus: int, tbus: int, ordinal: int) -> int:
    hits = case.branches_between(fbus, tbus)
    if not 1 <= ordinal <= len(hits):
        raise UnknownOutage(f"no branch #{ordinal} from bus {fbus} to {tbus}")
    return hits[ordinal - 1]


def resolve_outages(case, ctg) -> tuple:
    """(gen positions, branch positions) a contingency switches off.

    Raises like network.py:312-336 for unknown or already-off elements.
    """
    gens, branches = [], []
    gst = {}
    bst = {}
    for o in ctg.outages:
        if o.kind == GEN:
            k = _gen_index(case, o.bus, o.ordinal)
            if gst.get(k, case.gens[k].status) == 0:
                raise UnknownOutage(
                    f"generator #{o.ordinal} at bus {o.bus} is already off")
            gst[k] = 0
            gens.append(k)
        elif o.kind == BRANCH:
            k = _branch_index(case, o.bus, o.tbus, o.ordinal)
            if bst.get(k, case.branches[k].status) == 0:
                raise UnknownOutage(
                    f"branch #{o.ordinal} {o.bus}-{o.tbus} is already off")
            bst[k] = 0
            branches.append(k)
        else:
            raise UnknownOutage(f"outage kind {o.kind!r}")
    return tuple(gens), tuple(branches)


def apply_contingency(case, ctg):
    """Case with the contingency's elements off (network.py:312-345)."""
    goff, boff = resolve_outages(case, ctg)
    gens = list(case.gens)
    for k in goff:
        gens[k] = replace(gens[k], status=0)
    branches = list(case.branches)
    for k in boff:
        branches[k] = replace(branches[k], status=0)
    out = replace(case, gens=tuple(gens), branches=tuple(branches))
    if boff:
        n_islands, _ = check_connectivity(out)
        if n_islands != 1:
            raise IslandingDetected(
                f"contingency {ctg.id} splits the network into "
                f"{n_islands} islands")
    return out


def scenario_targets(case, scenario) -> dict:
    """{gen position: target MW} after validation (network.py:348-357)."""
    out = {}
    for (bus, ordinal), mw in scenario.wind_targets:
        k = _gen_index(case, bus, ordinal)
        if not case.gens[k].is_wind:
            raise TargetOnNonWind(
                f"generator #{ordinal} at bus {bus} is not wind")
        out[k] = mw
    return out


def apply_scenario(case, scenario):
    """Case with wind Pmax set to the scenario targets, Pmin 0."""
    gens = list(case.gens)
    for k, mw in scenario_targets(case, scenario).items():
        gens[k] = replace(gens[k], pmax=mw, pmin=0.0)
    return replace(case, gens=tuple(gens))


def declare_wind(case, keys):
    """Mark (bus, ordinal) generators as zero-cost wind (network.py:360-373)."""
    gens = list(case.gens)
    for bus, ordinal in keys:
        k = _gen_index(case, bus, ordinal)
        g = gens[k]
        if not g.is_wind:
            gens[k] = replace(g, cost=replace(g.cost, c2=0.0, c1=0.0, c0=0.0),
                              pmin=0.0, is_wind=True)
    return replace(case, gens=tuple(gens))


def apply_load_step(case, profile, t: int):
    """Case with loads replaced by profile step t (network.py:376-388)."""
    if not 0 <= t < len(profile.times):
        raise IndexOutOfRange(
            f"step {t} outside profile horizon of {len(profile.times)}")
    buses = list(case.buses)
    for col, bid in enumerate(profile.buses):
        k = case.bus_pos.get(bid)
        if k is None:
            raise UnknownBus(f"profile bus {bid} not in case")
        buses[k] = replace(buses[k], pd=profile.pd[t][col], qd=profile.qd[t][col])
    return replace(case, buses=tuple(buses))
