"""Native library host side (no GPU): symbols, scipy-order replay, sincos, planner."""

import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest
from scipy.sparse import _sparsetools

import common as C
from golden.make_golden import STAGE_SPECS, COMPOSITE_SPECS, composite_inputs, compose, stage_case
import paper_2203_10587_b200 as pkg
from paper_2203_10587_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "acopf_b200.h")
CSRC = os.path.join(ROOT, "paper_2203_10587_b200", "csrc")


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(L.LIB_PATH)
    names = set(re.findall(r"\b(acopf_\w+)\s*\(", open(HEADER).read()))
    assert len(names) >= 12
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert L.lib().acopf_version() == 1


def _scipy_order(cols):
    """Term order scipy's csr_sort_indices gives one row (payload replay)."""
    n = len(cols)
    indptr = np.array([0, n], dtype=np.int32)
    idx = np.asarray(cols, dtype=np.int32).copy()
    payload = np.arange(n, dtype=np.float64)
    _sparsetools.csr_sort_indices(1, indptr, idx, payload)
    return payload.astype(np.int32)


def _ours(cols):
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    perm = np.zeros(len(cols), dtype=np.int32)
    L.check(L.lib().acopf_canonical_order(len(cols), L.ptr(cols, ctypes.c_int32), L.ptr(perm, ctypes.c_int32)))
    return perm


@pytest.mark.parametrize("seed", range(40))
def test_canonical_order_replays_scipy(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 80))
    cols = rng.integers(0, max(2, n // 3), size=n)
    assert np.array_equal(_ours(cols), _scipy_order(cols))


def test_canonical_order_real_rows_longer_than_16():
    """Rows above the insertion-sort threshold (introsort: not stable)."""
    rng = np.random.default_rng(1)
    for n in (17, 24, 33, 64, 200, 1000):
        cols = np.repeat(rng.integers(0, 6, size=n // 3 + 1), 3)[:n]
        assert np.array_equal(_ours(cols), _scipy_order(cols))


@pytest.fixture(scope="module")
def sincos_bin():
    d = tempfile.mkdtemp()
    src = os.path.join(d, "t.cpp")
    with open(src, "w") as fh:
        fh.write('#include <cstdio>\n#include <cstdlib>\n#include "sincos.cuh"\n'
                 'int main(){size_t n; if(fread(&n,8,1,stdin)!=1) return 1; double* x=(double*)malloc(8*n);'
                 'if(fread(x,8,n,stdin)!=n) return 1; double* o=(double*)malloc(16*n);'
                 'for(size_t i=0;i<n;i++) acc_sincos(x[i],&o[2*i],&o[2*i+1]); fwrite(o,16,n,stdout); return 0;}\n')
    exe = os.path.join(d, "t")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", CSRC, src, "-o", exe], check=True)
    return exe


@pytest.fixture(scope="module")
def libm_sincos_bin():
    d = tempfile.mkdtemp()
    src = os.path.join(d, "t.cpp")
    with open(src, "w") as fh:
        fh.write('#include <cstdio>\n#include <cstdlib>\n#include "sincos.cuh"\n'
                 'int main(){size_t n; if(fread(&n,8,1,stdin)!=1) return 1; double* x=(double*)malloc(8*n);'
                 'if(fread(x,8,n,stdin)!=n) return 1; double* o=(double*)malloc(16*n);'
                 'for(size_t i=0;i<n;i++) libm_sincos(x[i],&o[2*i],&o[2*i+1]); fwrite(o,16,n,stdout); return 0;}\n')
    exe = os.path.join(d, "t")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", CSRC, src, "-o", exe], check=True)
    return exe


def test_libm_sincos_bit_identical_to_numpy(libm_sincos_bin):
    """The kernels' sincos equals np.sin / np.cos (glibc) bit for bit on |x| < 0.8555."""
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(-0.8554, 0.8554, 1_000_000), rng.uniform(-0.13, 0.13, 200_000),
                         rng.uniform(-1e-7, 1e-7, 10_000),
                         [0.0, -0.0, 0.126, -0.126, 1 / 256, 0.85546874999999989, 7.45e-9, 1.49e-8]])
    inp = np.array([len(xs)], dtype=np.uint64).tobytes() + xs.tobytes()
    out = np.frombuffer(subprocess.run([libm_sincos_bin], input=inp, capture_output=True, check=True).stdout)
    assert C.bit_diffs(out[0::2], np.sin(xs)) == 0
    assert C.bit_diffs(out[1::2], np.cos(xs)) == 0


def test_libm_sincos_wide_range_bit_identical_to_numpy(libm_sincos_bin):
    """glibc's wide-range paths (0.8555 <= |x| < 105414336, large branch angles an IPM can
    visit): np.sin / np.cos bit for bit, including near multiples of pi/2."""
    rng = np.random.default_rng(12)
    xs = np.concatenate([rng.uniform(0.85546875, 2.4262638092041016, 600_000),
                         -rng.uniform(0.85546875, 2.4262638092041016, 200_000),
                         rng.uniform(-20.0, 20.0, 300_000), rng.uniform(-1e6, 1e6, 50_000),
                         np.pi / 2 + rng.uniform(-1e-6, 1e-6, 20_000),
                         np.pi * rng.integers(-40, 40, 20_000) + rng.uniform(-1e-9, 1e-9, 20_000),
                         [0.85546875, -0.85546875, 2.4262638092041016, np.nextafter(2.4262638092041016, 0),
                          np.pi, -np.pi, 3 * np.pi / 2, 105414335.0]])
    inp = np.array([len(xs)], dtype=np.uint64).tobytes() + xs.tobytes()
    out = np.frombuffer(subprocess.run([libm_sincos_bin], input=inp, capture_output=True, check=True).stdout)
    assert C.bit_diffs(out[0::2], np.sin(xs)) == 0
    assert C.bit_diffs(out[1::2], np.cos(xs)) == 0


def test_accurate_sincos_vs_libm(sincos_bin):
    """Device sincos (same source, host build) is within 1 ulp of libm and equal on >99.5%."""
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.uniform(-0.6, 0.6, 200000), rng.uniform(-4, 4, 50000),
                         rng.uniform(-1e4, 1e4, 5000), [0.0, -0.0, 1e-300, -3e-9, np.pi / 4]])
    inp = np.array([len(xs)], dtype=np.uint64).tobytes() + xs.tobytes()
    out = np.frombuffer(subprocess.run([sincos_bin], input=inp, capture_output=True, check=True).stdout)
    s, c = out[0::2], out[1::2]
    ns, nc = np.sin(xs), np.cos(xs)
    ulp = lambda a, b: np.abs(a.view(np.int64) - b.view(np.int64))
    assert ulp(s, ns).max() <= 1 and ulp(c, nc).max() <= 1
    assert np.count_nonzero(s != ns) < 0.005 * len(xs)
    assert np.count_nonzero(c != nc) < 0.005 * len(xs)
    assert np.signbit(s[len(xs) - 4])      # sin(-0.0) = -0.0


@pytest.mark.parametrize("name", C.STAGE_FIXTURES)
def test_stage_structure_matches_golden(name):
    """Patterns, bounds and sizes of build_acopf (planner only, no GPU)."""
    g = C.load(name)
    p, lay = pkg.build_acopf(stage_case(STAGE_SPECS[name]))
    assert (p.n, p.m_eq, p.m_ineq) == (int(g["n"]), int(g["m_eq"]), int(g["m_ineq"]))
    for a in ("xl", "xu", "x0", "gl", "gu"):
        assert C.bit_diffs(getattr(p, a), g[a]) == 0, a
    ip, ix = p.evaluator.pattern("J")
    assert np.array_equal(ip, g["jindptr"]) and np.array_equal(ix, g["jindices"])
    ip, ix = p.evaluator.pattern("H")
    assert np.array_equal(ip, g["hindptr"]) and np.array_equal(ix, g["hindices"])


@pytest.mark.parametrize("name", C.COMPOSITE_FIXTURES)
def test_composite_structure_matches_golden(name):
    g = C.load(name)
    spec = COMPOSITE_SPECS[name]
    a, _ = composite_inputs(spec)
    p, imap = compose(pkg, spec["kind"], a)
    assert (p.n, p.m_eq, p.m_ineq) == (int(g["n"]), int(g["m_eq"]), int(g["m_ineq"]))
    for k in ("xl", "xu", "x0", "gl", "gu"):
        assert C.bit_diffs(getattr(p, k), g[k]) == 0, k
    assert list(imap.var_offset) == list(g["var_offset"])
    assert list(imap.eq_offset) == list(g["eq_offset"])
    assert list(imap.ineq_offset) == list(g["ineq_offset"])
    assert np.array_equal(np.array(imap.weights), g["weights"])
    rows = np.array([[r.stage_a, r.stage_b, -1 if r.gen is None else r.gen, -1 if r.bus is None else r.bus,
                      r.row, int(r.is_equality)] for r in imap.coupling_rows], dtype=np.int64).reshape(-1, 6)
    assert np.array_equal(rows, g["cp_rows"])
    assert [r.kind for r in imap.coupling_rows] == list(g["cp_kinds"])
    assert C.bit_diffs([r.bound for r in imap.coupling_rows], g["cp_bounds"]) == 0
    ip, ix = p.evaluator.pattern("J")
    assert np.array_equal(ip, g["jindptr"]) and np.array_equal(ix, g["jindices"])
    ip, ix = p.evaluator.pattern("H")
    assert np.array_equal(ip, g["hindptr"]) and np.array_equal(ix, g["hindices"])


@pytest.mark.parametrize("name", C.STAGE_FIXTURES + C.COMPOSITE_FIXTURES)
def test_tile_tables_satisfy_planner_invariants(name):
    """Every staging position and round slot has exactly one producer (no GPU)."""
    if name in C.STAGE_FIXTURES:
        p, _ = pkg.build_acopf(stage_case(STAGE_SPECS[name]))
    else:
        spec = COMPOSITE_SPECS[name]
        a, _ = composite_inputs(spec)
        p, _ = compose(pkg, spec["kind"], a)
    st = p.evaluator.verify_plan()
    assert st["tables"] >= st["tiles"] >= 1
    assert st["max_smem_bytes"] <= 220 * 1024


def test_tile_tables_config1_network():
    """The 10k-bus network: invariants, tile fill and the CTA shared-memory budget."""
    from paper_2203_10587_b200 import synthetic as syn
    p, _ = pkg.build_acopf(syn.config_case(1))
    st = p.evaluator.verify_plan()
    assert st["ends"] == 2 * 12999
    assert st["ends"] / st["tiles"] > 80          # tile fill (128 ends per 4-warp CTA)
    assert st["max_smem_bytes"] <= 75 * 1024      # 3 CTAs (12 warps) per SM


def test_tile_tables_hub_network():
    """A hub bus with more branch ends than a tile CTA has threads: invariants and the
    modeled shared-memory store cost (conflicts included) against its conflict-free bound."""
    p, _ = pkg.build_acopf(C.hub_case())
    st = p.evaluator.verify_plan()
    assert st["ends"] > 128 and st["max_smem_bytes"] <= 220 * 1024
    assert st["store_wavefronts_ideal"] <= st["store_wavefronts_half"] <= 4 * st["store_wavefronts_ideal"]


def test_parallel_planner_is_deterministic():
    """Tile tables are built on all host cores: two builds of a contingency composite
    give identical plans (table counts, areas, rounds, modeled store cost)."""
    spec = COMPOSITE_SPECS["scopf_corrective"]
    stats = []
    for _ in range(2):
        a, _ = composite_inputs(spec)
        p, _ = compose(pkg, spec["kind"], a)
        stats.append(p.evaluator.verify_plan())
    assert stats[0] == stats[1]


def test_reference_fixture_case9_stage_structure():
    """build_acopf on the reference's own case9.m (parsed by the reference, stored in the golden)."""
    g = C.load("ref_case9_stage")
    p, lay = pkg.build_acopf(C.case_from_json(str(g["case"])))
    assert (p.n, p.m_eq, p.m_ineq) == (int(g["n"]), int(g["m_eq"]), int(g["m_ineq"]))
    for a in ("xl", "xu", "x0", "gl", "gu"):
        assert C.bit_diffs(getattr(p, a), g[a]) == 0, a
    ip, ix = p.evaluator.pattern("J")
    assert np.array_equal(ip, g["jindptr"]) and np.array_equal(ix, g["jindices"])
    ip, ix = p.evaluator.pattern("H")
    assert np.array_equal(ip, g["hindptr"]) and np.array_equal(ix, g["hindices"])


@pytest.mark.parametrize("name", C.REF_FIXTURES)
def test_reference_fixture_composite_structure(name):
    """compose_* on case9 + ctgc.cont / scenarios.csv / load profile (the reference's fixtures):
    sizes, bounds, offsets, weights, coupling rows and CSR patterns equal the reference's."""
    from paper_2203_10587_b200.types import CouplingMode
    g = C.load(name)
    p, imap = C.ref_fixture_compose(pkg, g, CouplingMode)
    assert (p.n, p.m_eq, p.m_ineq) == (int(g["n"]), int(g["m_eq"]), int(g["m_ineq"]))
    for k in ("xl", "xu", "x0", "gl", "gu"):
        assert C.bit_diffs(getattr(p, k), g[k]) == 0, k
    assert list(imap.var_offset) == list(g["var_offset"])
    assert list(imap.eq_offset) == list(g["eq_offset"])
    assert list(imap.ineq_offset) == list(g["ineq_offset"])
    assert np.array_equal(np.array(imap.weights), g["weights"])
    rows = np.array([[r.stage_a, r.stage_b, -1 if r.gen is None else r.gen, -1 if r.bus is None else r.bus,
                      r.row, int(r.is_equality)] for r in imap.coupling_rows], dtype=np.int64).reshape(-1, 6)
    assert np.array_equal(rows, g["cp_rows"])
    assert [r.kind for r in imap.coupling_rows] == list(g["cp_kinds"])
    assert C.bit_diffs([r.bound for r in imap.coupling_rows], g["cp_bounds"]) == 0
    ip, ix = p.evaluator.pattern("J")
    assert np.array_equal(ip, g["jindptr"]) and np.array_equal(ix, g["jindices"])
    ip, ix = p.evaluator.pattern("H")
    assert np.array_equal(ip, g["hindptr"]) and np.array_equal(ix, g["hindices"])


def test_native_graph_checks_match_the_python_restatements():
    """acopf_graph_bridges / acopf_graph_islands (the lattice's islanding checks) against
    grid.check_connectivity (network.py:232-262) and a Python Tarjan, incl. parallel twins."""
    from dataclasses import replace
    from paper_2203_10587_b200 import lattice as Lt
    from paper_2203_10587_b200 import synthetic as syn
    from paper_2203_10587_b200.grid import check_connectivity
    from paper_2203_10587_b200.packer import PackedCase
    for case in (syn.make_case(300, 60, 40, seed=5, features=True), C.hub_case(), syn.config_case(2)):
        pc = PackedCase(case)
        nb = set(syn.non_bridge_branches(case))
        br = Lt._bridges(pc)
        for k in pc.live_br:
            if case.branches[int(k)].fbus != case.branches[int(k)].tbus:
                assert (int(k) in br) == (int(k) not in nb)
        rng = np.random.default_rng(1)
        live = sorted(int(k) for k in pc.live_br)
        for _ in range(10):
            rem = set(rng.choice(live, size=4, replace=False).tolist())
            c2 = replace(case, branches=tuple(replace(b, status=0) if i in rem else b
                                              for i, b in enumerate(case.branches)))
            assert Lt._islands_without(pc, sorted(rem)) == check_connectivity(c2)[0]


def test_eval_host_rejects_short_or_missing_buffers_before_device_work():
    """acopf_batch_eval_host validates every requested output against the layout:
    a short buffer or a missing multiplier vector fails with a message, before any copy."""
    import ctypes
    from paper_2203_10587_b200 import _lib as L
    p, _ = pkg.build_acopf(stage_case(STAGE_SPECS["stage_feat30"]))
    ev = p.evaluator
    x = np.zeros(ev.n)
    short = np.zeros(max(ev.nnz_h - 1, 1))
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a is not None else None

    def call(what, nx=ev.n, mult=None, nm=0, h=None, nh=0, j=None, nj=0):
        return L.lib().acopf_batch_eval_host(ev._h, vp(x), nx, 1.0, vp(mult), nm, what, None, 0, None, 0, None, 0,
                                             vp(j), nj, vp(h), nh, None)

    assert call(L.HESS, h=short, nh=len(short), mult=np.zeros(ev.m), nm=ev.m) != 0
    assert b"hval" in L.lib().acopf_last_error()
    assert call(L.HESS, h=np.zeros(ev.nnz_h), nh=ev.nnz_h) != 0
    assert b"mult" in L.lib().acopf_last_error()
    assert call(L.JAC, j=np.zeros(3), nj=3) != 0
    assert b"jval" in L.lib().acopf_last_error()
    assert call(L.JAC, nx=ev.n - 1, j=np.zeros(ev.nnz_j), nj=ev.nnz_j) != 0
    assert b"x has" in L.lib().acopf_last_error()
