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
