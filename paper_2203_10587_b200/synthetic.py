"""Seeded synthetic networks and evaluation points for BASELINE.json's configs.

The reference's benchmark networks (ACTIVSg, `PAPER.md:175,218-231`) are not
available here; BASELINE.json names synthetic networks instead and
SURVEY.md §8(d) gives the recipe this module implements:

* topology: random recursive spanning tree (parent(i) ~ U{0..i-1}) plus
  distinct random chords without self-loops or parallel edges; config 0
  is the 9-bus ring i -> (i+1) mod 9;
* branches: r ~ U(0.005,0.02), x ~ U(0.05,0.2), b ~ U(0,0.2), ratio 1,
  angle 0, rate_a ~ U(1.5,3.0)*100 MVA (every branch rated);
* buses: bus 0 is REF, generator buses PV, others PQ; Vm in [0.9,1.1];
  Pd ~ U(0.5,1.5)*100 MW with Qd = 0.3 Pd on 60 % of the buses;
* generators on bus 0 plus random distinct buses, P in [10,300] MW,
  Q in [-300,300] MVAr, c2 ~ U(0.01,0.1), c1 ~ U(1,40), c0 = 0;
* evaluation points: Vm ~ U(0.95,1.05), Va ~ U(-0.3,0.3) (pinned REF
  angle kept), Pg/Qg ~ U(bounds), multipliers ~ N(0,1).

``features=True`` additionally exercises everything the reference's stage
model supports (taps, phase shifts, shunts, unrated and out-of-service
branches, parallel branches, a self-loop, out-of-service generators,
several generators per bus, isolated buses, nonzero c0) for parity tests.
Seeds are fixed per config (CONFIG_SEEDS) so every run sees the same inputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from .grid import (
    BRANCH, ISOLATED, PQ, PV, REF,
    Branch, Bus, Contingency, ContingencySet, GenCost, Generator,
    LoadProfile, NetworkCase, Outage, Scenario, ScenarioSet,
    apply_load_step, declare_wind,
)

CONFIG_SEEDS = {0: 20220310, 1: 20220311, 2: 20220312, 3: 20220313, 4: 20220314}

# BASELINE.json configs[k] network sizes: (buses, chords, generators)
CONFIG_SIZES = {
    0: (9, 0, 3),
    1: (10_000, 3_000, 2_500),
    2: (2_000, 600, 500),
    3: (2_000, 600, 500),
    4: (25_000, 8_000, 6_000),
}


def _tree_and_chords(nb: int, n_chords: int, rng) -> list:
    edges = []
    if nb > 1:
        parents = np.floor(rng.random(nb - 1) * np.arange(1, nb)).astype(np.int64)
        edges = [(int(p), i + 1) for i, p in enumerate(parents)]
    seen = {(min(a, b), max(a, b)) for a, b in edges}
    max_chords = nb * (nb - 1) // 2 - len(seen)
    if n_chords > max_chords:
        raise ValueError("too many chords for this bus count")
    chords = []
    while len(chords) < n_chords:
        need = n_chords - len(chords)
        cand = rng.integers(0, nb, size=(2 * need + 8, 2))
        for a, b in cand:
            a, b = int(a), int(b)
            key = (min(a, b), max(a, b))
            if a == b or key in seen:
                continue
            seen.add(key)
            chords.append((a, b))
            if len(chords) == n_chords:
                break
    return edges + chords


def make_case(nb: int, n_chords: int, ng: int, seed: int, *, ring: bool = False,
              name: str | None = None, features: bool = False,
              ramp_30: float | None = 10.0) -> NetworkCase:
    """One synthetic network (SURVEY §8d recipe); see the module docstring."""
    rng = np.random.default_rng(seed)
    if ring:
        edges = [(i, (i + 1) % nb) for i in range(nb)]
    else:
        edges = _tree_and_chords(nb, n_chords, rng)
    nbr = len(edges)
    r = rng.uniform(0.005, 0.02, nbr)
    x = rng.uniform(0.05, 0.2, nbr)
    bch = rng.uniform(0.0, 0.2, nbr)
    rate = rng.uniform(1.5, 3.0, nbr) * 100.0

    if ring and nb == 9 and ng == 3:
        gen_buses = np.array([0, 3, 6])
    else:
        others = rng.choice(np.arange(1, nb), size=ng - 1, replace=False)
        gen_buses = np.sort(np.concatenate([[0], others]))
    gen_set = set(int(b) for b in gen_buses)
    if ring and nb == 9 and ng == 3:
        load_buses = np.array([b for b in range(nb) if b not in gen_set])
    else:
        load_buses = rng.choice(nb, size=int(round(0.6 * nb)), replace=False)
    pd = np.zeros(nb)
    pd[load_buses] = rng.uniform(0.5, 1.5, len(load_buses)) * 100.0
    c2 = rng.uniform(0.01, 0.1, ng)
    c1 = rng.uniform(1.0, 40.0, ng)

    buses = []
    for i in range(nb):
        btype = REF if i == 0 else (PV if i in gen_set else PQ)
        buses.append(Bus(id=i + 1, btype=btype, pd=float(pd[i]), qd=float(0.3 * pd[i]),
                         gs=0.0, bs=0.0, area=1, vm=1.0, va=0.0, base_kv=230.0,
                         zone=1, vmax=1.1, vmin=0.9))
    gens = []
    for j, b in enumerate(gen_buses):
        gens.append(Generator(bus=int(b) + 1, pg=0.0, qg=0.0, qmax=300.0, qmin=-300.0,
                              vg=1.0, mbase=100.0, status=1, pmax=300.0, pmin=10.0,
                              ramp_30=float(ramp_30 if ramp_30 is not None else 0.0),
                              cost=GenCost(c2=float(c2[j]), c1=float(c1[j]), c0=0.0),
                              is_wind=False))
    branches = []
    for k, (a, b) in enumerate(edges):
        branches.append(Branch(fbus=a + 1, tbus=b + 1, r=float(r[k]), x=float(x[k]),
                               b=float(bch[k]), rate_a=float(rate[k]), rate_b=0.0,
                               rate_c=0.0, ratio=1.0, angle=0.0, status=1,
                               angmin=-360.0, angmax=360.0))
    case = NetworkCase(name=name or f"synth{nb}", base_mva=100.0, buses=tuple(buses),
                       gens=tuple(gens), branches=tuple(branches))
    if features:
        case = _add_features(case, rng)
    return case


def _add_features(case: NetworkCase, rng) -> NetworkCase:
    """Sprinkle every modelled feature over a connected synthetic case."""
    buses = list(case.buses)
    branches = list(case.branches)
    gens = list(case.gens)
    nb, nbr = len(buses), len(branches)
    # shunts on a third of the buses
    for i in rng.choice(nb, size=max(1, nb // 3), replace=False):
        buses[i] = replace(buses[i], gs=float(rng.uniform(-5, 5)), bs=float(rng.uniform(-20, 20)))
    # off-nominal taps and phase shifts
    for k in rng.choice(nbr, size=max(1, nbr // 4), replace=False):
        branches[k] = replace(branches[k], ratio=float(rng.uniform(0.9, 1.1)),
                              angle=math.radians(float(rng.uniform(-5, 5))))
    # ratio 0 means "no transformer"
    k0 = int(rng.integers(0, nbr))
    branches[k0] = replace(branches[k0], ratio=0.0)
    # unrated branches
    for k in rng.choice(nbr, size=max(1, nbr // 6), replace=False):
        branches[k] = replace(branches[k], rate_a=0.0)
    # parallel twins (same orientation and reversed), a self-loop
    twins = []
    for k in rng.choice(nbr, size=max(1, nbr // 10), replace=False):
        br = branches[k]
        twins.append(replace(br, r=br.r * 1.3, x=br.x * 0.8))
    br = branches[int(rng.integers(0, nbr))]
    twins.append(replace(br, fbus=br.tbus, tbus=br.fbus, b=0.01))
    loop_bus = buses[int(rng.integers(1, nb))].id
    twins.append(replace(branches[0], fbus=loop_bus, tbus=loop_bus, r=0.01, x=0.1, b=0.05))
    branches.extend(twins)
    # a parallel out-of-service branch (must not appear in the model)
    branches.append(replace(branches[1], status=0, r=0.02))
    # extra generators on existing generator buses, one out of service
    extra = []
    for j in rng.choice(len(gens), size=max(1, len(gens) // 3), replace=False):
        g = gens[j]
        extra.append(replace(g, cost=GenCost(c2=float(rng.uniform(0.01, 0.1)),
                                             c1=float(rng.uniform(1, 40)),
                                             c0=float(rng.uniform(0, 50)))))
    gens.extend(extra)
    gens[-1] = replace(gens[-1], status=0)
    # an isolated bus appended at the end (no in-service branch touches it),
    # and an isolated bus hanging off an out-of-service branch
    iso_id = max(b.id for b in buses) + 1
    buses.append(replace(buses[1], id=iso_id, btype=ISOLATED, pd=0.0, qd=0.0))
    branches.append(replace(branches[2], fbus=iso_id, tbus=buses[0].id, status=0))
    return replace(case, buses=tuple(buses), branches=tuple(branches), gens=tuple(gens))


def config_case(k: int, *, nb: int | None = None, n_chords: int | None = None,
                ng: int | None = None, **kw) -> NetworkCase:
    """Base network of BASELINE.json config k (optionally resized for tests)."""
    nb0, nc0, ng0 = CONFIG_SIZES[k]
    nb = nb0 if nb is None else nb
    n_chords = nc0 if n_chords is None else n_chords
    ng = ng0 if ng is None else ng
    return make_case(nb, n_chords, ng, CONFIG_SEEDS[k] + nb, ring=(k == 0),
                     name=f"cfg{k}-{nb}", **kw)


# ---------------------------------------------------------------------------
# bridges (an outage of a bridge islands the network, network.py:339-344)

def non_bridge_branches(case) -> list:
    """Positions of in-service branches whose outage keeps one island."""
    pos = case.bus_pos
    nbus = len(case.buses)
    adj: list = [[] for _ in range(nbus)]
    live = [k for k, br in enumerate(case.branches) if br.status != 0]
    for k in live:
        br = case.branches[k]
        a, b = pos[br.fbus], pos[br.tbus]
        adj[a].append((b, k))
        adj[b].append((a, k))
    disc = [-1] * nbus
    low = [0] * nbus
    bridges = set()
    t = 0
    for root in range(nbus):
        if disc[root] >= 0 or not adj[root]:
            continue
        disc[root] = low[root] = t
        t += 1
        stack = [(root, -1, iter(adj[root]))]
        while stack:
            u, via, it = stack[-1]
            advanced = False
            for v, k in it:
                if k == via:
                    continue
                if disc[v] < 0:
                    disc[v] = low[v] = t
                    t += 1
                    stack.append((v, k, iter(adj[v])))
                    advanced = True
                    break
                low[u] = min(low[u], disc[v])
            if not advanced:
                stack.pop()
                if stack:
                    p = stack[-1][0]
                    low[p] = min(low[p], low[u])
                    if low[u] > disc[p]:
                        bridges.add(via)
    return [k for k in live if k not in bridges and
            case.branches[k].fbus != case.branches[k].tbus]


def branch_contingencies(case, count: int, seed: int) -> ContingencySet:
    """``count`` distinct single non-bridge branch outages, ids 1..count."""
    rng = np.random.default_rng(seed)
    cand = np.array(non_bridge_branches(case))
    pick = rng.choice(len(cand), size=count, replace=False)
    ctgs = []
    for cid, j in enumerate(pick, start=1):
        k = int(cand[j])
        br = case.branches[k]
        ordinal = case.branches_between(br.fbus, br.tbus).index(k) + 1
        ctgs.append(Contingency(id=cid, outages=(Outage(BRANCH, br.fbus, br.tbus, ordinal),)))
    return ContingencySet(tuple(ctgs))


# ---------------------------------------------------------------------------
# BASELINE.json configs 2-4 as compose_* inputs

def config2_inputs(n_ctg: int = 1024, **kw):
    """(base case, ContingencySet) for the N-1 SCOPF (ramp_30 = 10 MW: delta_c = 0.1 pu)."""
    base = config_case(2, ramp_30=10.0, **kw)
    return base, branch_contingencies(base, n_ctg, CONFIG_SEEDS[2] + 1)


def config3_periods(n_periods: int = 96, **kw) -> list:
    """Period cases with the seeded daily load profile; ramp_30 = 0.1 Pmax."""
    base = config_case(3, ramp_30=30.0, **kw)
    rng = np.random.default_rng(CONFIG_SEEDS[3] + 1)
    phi = float(rng.uniform(0.0, 2.0 * math.pi))
    load_ids = [b.id for b in base.buses if b.pd > 0.0]
    pd0 = np.array([base.buses[base.bus_pos[i]].pd for i in load_ids])
    pds, qds = [], []
    for t in range(n_periods):
        noise = 1.0 + rng.uniform(-0.05, 0.05, len(load_ids))
        p = pd0 * (0.7 + 0.3 * math.sin(2.0 * math.pi * t / 96.0 + phi)) * noise
        pds.append(tuple(float(v) for v in p))
        qds.append(tuple(float(v) for v in 0.3 * p))
    profile = LoadProfile(times=tuple(15.0 * t for t in range(n_periods)),
                          buses=tuple(load_ids), pd=tuple(pds), qd=tuple(qds))
    return [apply_load_step(base, profile, t) for t in range(n_periods)]


def config4_inputs(n_scen: int = 32, n_ctg: int = 31, **kw):
    """(wind-declared base, ScenarioSet, ContingencySet) for the stochastic SCOPF."""
    base = config_case(4, ramp_30=10.0, **kw)
    rng = np.random.default_rng(CONFIG_SEEDS[4] + 1)
    ng = len(base.gens)
    wind = np.sort(rng.choice(np.arange(1, ng), size=max(1, ng // 5), replace=False))
    keys = [(base.gens[j].bus, 1) for j in wind]
    base = declare_wind(base, keys)
    scens = []
    for s in range(n_scen):
        frac = rng.uniform(0.3, 1.0, len(wind))
        targets = tuple((key, float(base.gens[j].pmax * f))
                        for key, j, f in zip(keys, wind, frac))
        scens.append(Scenario(id=s + 1, weight=1.0, wind_targets=targets))
    ctgs = branch_contingencies(base, n_ctg, CONFIG_SEEDS[4] + 2)
    return base, ScenarioSet(tuple(scens)), ctgs


# ---------------------------------------------------------------------------
# evaluation points

VA, VM, PG, QG = 0, 1, 2, 3


def variable_kinds(stage_dims) -> np.ndarray:
    """Per-variable kind code for stacked stages given [(nb, ng), ...]."""
    parts = []
    for nb, ng in stage_dims:
        parts += [np.full(nb, VA), np.full(nb, VM), np.full(ng, PG), np.full(ng, QG)]
    return np.concatenate(parts).astype(np.int8) if parts else np.zeros(0, np.int8)


def random_point(kinds, xl, xu, m: int, seed: int):
    """(x, mult) drawn as in SURVEY §8d; pinned coordinates keep their value."""
    rng = np.random.default_rng(seed)
    n = len(kinds)
    x = np.empty(n)
    va = kinds == VA
    vm = kinds == VM
    gq = (kinds == PG) | (kinds == QG)
    x[va] = rng.uniform(-0.3, 0.3, int(va.sum()))
    x[vm] = rng.uniform(0.95, 1.05, int(vm.sum()))
    u = rng.random(int(gq.sum()))
    x[gq] = xl[gq] + u * (xu[gq] - xl[gq])
    fixed = xl == xu
    x[fixed] = xl[fixed]
    mult = rng.standard_normal(m)
    return x, mult
