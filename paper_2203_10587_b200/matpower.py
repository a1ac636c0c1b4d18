"""MATPOWER output of solved stages: the reference's writer side, formatted natively.

Drop-in for `pkg/src/opfkit/matpower.py:34-190` (``RawCase``, ``format_case``,
``write_case``, ``write_case_file``) and the per-stage output tree of
`runner.py:381-451` (``write_output_tree``'s MATPOWER files).  The text is
byte-identical to the reference's: every value is printed with ``%.10g``
(matpower.py:146-148) by ``acopf_format_matrix`` in libacopf_b200.so, which
formats whole matrices in C++ (and runs concurrently over stages: ctypes
releases the GIL), instead of one Python %-format per value.  Parsing (the
input side) is not part of this package.
"""

from __future__ import annotations

import ctypes
import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass(frozen=True)
class RawCase:
    """Numeric contents of a case file (matpower.py:34-44): rows of floats per section."""
    name: str
    base_mva: float
    bus: tuple
    gen: tuple
    branch: tuple
    gencost: tuple


def _ragged(rows):
    """(row_ptr int64, values float64) of a tuple of float tuples (or a 2-D array)."""
    if isinstance(rows, np.ndarray):
        a = np.ascontiguousarray(rows, dtype=np.float64)
        r, c = a.shape if a.ndim == 2 else (0, 0)
        return np.arange(r + 1, dtype=np.int64) * c, a.reshape(-1)
    lens = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    vals = np.fromiter((v for r in rows for v in r), dtype=np.float64, count=int(ptr[-1]))
    return ptr, vals


def format_matrix(section: str, rows) -> str:
    """``mpc.<section> = [ ... ];`` exactly as matpower._fmt_matrix (matpower.py:151-157)."""
    ptr, vals = _ragged(rows)
    lib = L.lib()
    n = len(ptr) - 1
    out_len = ctypes.c_int64()
    cap = max(64, 24 * len(vals) + 4 * n + 64)
    buf = ctypes.create_string_buffer(cap)
    L.check(lib.acopf_format_matrix(section.encode(), n, L.ptr(ptr, ctypes.c_int64),
                                    L.ptr(vals if len(vals) else np.zeros(1), ctypes.c_double),
                                    buf, cap, ctypes.byref(out_len)))
    return buf.raw[:out_len.value].decode("ascii")


def _fmt(v: float) -> str:
    return "%.10g" % v


def format_case(raw: RawCase) -> str:
    """MATPOWER text of a RawCase, tab separated (matpower.py:160-177)."""
    parts = [f"function mpc = {raw.name}", "", f"mpc.baseMVA = {_fmt(raw.base_mva)};", "",
             format_matrix("bus", raw.bus), "", format_matrix("gen", raw.gen), "",
             format_matrix("branch", raw.branch), "", format_matrix("gencost", raw.gencost), ""]
    return "\n".join(parts)


def case_to_raw(case) -> RawCase:
    """NetworkCase.to_raw (network.py:129-153): MATPOWER columns, angles in degrees."""
    bus = tuple((float(b.id), float(b.btype), b.pd, b.qd, b.gs, b.bs, float(b.area), b.vm,
                 math.degrees(b.va), b.base_kv, float(b.zone), b.vmax, b.vmin) + tuple(b.extra)
                for b in case.buses)
    gen = tuple((float(g.bus), g.pg, g.qg, g.qmax, g.qmin, g.vg, g.mbase, float(g.status), g.pmax, g.pmin)
                + tuple(g.tail) for g in case.gens)
    branch = tuple((float(br.fbus), float(br.tbus), br.r, br.x, br.b, br.rate_a, br.rate_b, br.rate_c,
                    br.ratio, math.degrees(br.angle), float(br.status), br.angmin, br.angmax)
                   + tuple(br.extra) for br in case.branches)
    cost = []
    for g in case.gens:
        c = g.cost
        cost.append((2.0, c.startup, c.shutdown, float(c.ncost)) + (c.c2, c.c1, c.c0)[3 - c.ncost:])
    return RawCase(name=case.name, base_mva=case.base_mva, bus=bus, gen=gen, branch=branch, gencost=tuple(cost))


def solved_to_raw(sol, name: str | None = None) -> RawCase:
    """SolvedCase.to_raw (acopf.py:433-446): solved Vm/Va, dispatch and flow columns."""
    base = case_to_raw(sol.case)
    bus = tuple(row[:7] + (sol.vm[i], math.degrees(sol.va[i])) + row[9:] for i, row in enumerate(base.bus))
    gen = tuple((row[0], sol.pg[i], sol.qg[i]) + row[3:] for i, row in enumerate(base.gen))
    branch = tuple(row[:13] + (sol.pf[i], sol.qf[i], sol.pt[i], sol.qt[i]) for i, row in enumerate(base.branch))
    return RawCase(name=name or base.name, base_mva=base.base_mva, bus=bus, gen=gen, branch=branch,
                   gencost=base.gencost)


def write_case(solved, name: str | None = None) -> str:
    """MATPOWER text of a solved case (matpower.py:180-187)."""
    return format_case(solved.to_raw(name=name))


def write_case_file(solved, path: str, name: str | None = None) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(write_case(solved, name=name))


def write_case_files(solved, paths, names=None, workers: int | None = None) -> None:
    """write_case_file for many stages at once (the MATPOWER files of runner.write_output_tree,
    runner.py:394-423), formatted concurrently on the host cores."""
    names = list(names) if names is not None else [None] * len(paths)
    jobs = list(zip(solved, paths, names))
    with ThreadPoolExecutor(max_workers=workers or min(32, os.cpu_count() or 1)) as pool:
        list(pool.map(lambda j: write_case_file(j[0], j[1], name=j[2]), jobs))
