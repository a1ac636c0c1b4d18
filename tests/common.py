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
