"""MATPOWER output: write_case text byte-identical to the reference's
(matpower.py:146-190, acopf.py:433-446), formatted by acopf_format_matrix (C++).

The solved cases come from extract_solution on the GPU in the reference; here (CPU) the
SolvedCase is rebuilt from the same x through the oracle's flows, so the test needs no GPU."""

import os
import tempfile

import numpy as np
import pytest

import common as C
import paper_2203_10587_b200 as pkg
from paper_2203_10587_b200 import matpower as M
from paper_2203_10587_b200.solution import SolvedCase
from oracle.solution import extract
from oracle.stage import StageOracle


def _solved(g, i):
    """The SolvedCase of extract_solution at golden point i, via the oracle's flows (CPU)."""
    case = C.case_from_json(str(g[f"case{i}"]))
    o = StageOracle(case)
    lay = pkg.AcopfLayout(n_vars=o.n, n_eq=o.m_eq, n_ineq=o.m_ineq, **o.layout_maps())
    d = extract(case, lay, g[f"x{i}"])
    return SolvedCase(case=case, **d)


@pytest.mark.parametrize("i", range(4))
def test_write_case_matches_reference_text(i):
    g = C.load("matpower_text")
    sol = _solved(g, i)
    assert M.write_case(sol, name=f"t_{i}") == str(g[f"text{i}"])
    assert M.write_case(sol) == str(g[f"text_default{i}"])


def test_write_case_files_concurrently():
    g = C.load("matpower_text")
    sols = [_solved(g, i) for i in range(int(g["n"]))]
    d = tempfile.mkdtemp()
    paths = [os.path.join(d, f"t_{i}.m") for i in range(len(sols))]
    M.write_case_files(sols, paths, names=[f"t_{i}" for i in range(len(sols))])
    for i, path in enumerate(paths):
        assert open(path).read() == str(g[f"text{i}"])


def test_format_matrix_edge_values():
    rows = ((0.0, -0.0, 1e20, -1e-300, np.inf, -np.inf, np.nan, -np.nan, 123456789.123, 1 / 3),
            (), (2.5,))
    expect = "mpc.x = [\n\t" + "\t".join("%.10g" % v for v in rows[0]) + ";\n\t;\n\t2.5;\n];"
    assert M.format_matrix("x", rows) == expect
    assert M.format_matrix("y", ()) == "mpc.y = [\n];"
