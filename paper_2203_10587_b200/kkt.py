"""The reference IPM's Newton system on the device.

The reference solves every Newton step with a dense Bunch-Kaufman LDL^T of

    K = [ 0.5 (Hfull + Hfull^T) + reg I    Je^T    ]      Hfull = H + diag(dx) + Ji^T diag(ds) Ji
        [ Je                              -delta I ]

over the free variables (`pkg/src/opfkit/ipm.py:463-501`: `hfull.todense()` at :471, the
factorisation `_BunchKaufman` with LAPACK `dsytrf` and the inertia test at :173-220).  With
the callbacks on the GPU, its host-side `todense()` and `dsytrf` become the cost of every
iteration at configs 1-4.  :class:`DeviceKKT` keeps the step on the device:

* **assembly** -- ``acopf_kkt_assemble`` (csrc/kkt.cuh) writes K straight from the
  evaluator's device-resident J / H values (``BatchEvaluator.eval_device``) with the
  reference view's row scaling; deterministic, one thread per column;
* **factorisation** -- cuSOLVER's Bunch-Kaufman ``sytrf`` (``torch.linalg.ldl_factor_ex``;
  a library solver, as SURVEY §8(f) allows), inertia read off the pivot blocks exactly as
  ``_BunchKaufman._inertia``;
* **solve** -- ``sytrs`` (``torch.linalg.ldl_solve``).

Scope: dense, like the reference (the cfg1 system, n + m_eq = 45 k, is a 16 GB matrix that
fits one B200); a sparse LDL^T for configs 2-4 is the next step.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L


def _csr_sub(indptr, indices, rows, col_map):
    """CSR of the given rows with columns mapped through col_map (-1 dropped):
    (ptr int64, col int32, value index int64)."""
    ptr = [0]
    cols, vi = [], []
    for r in rows:
        a, b = int(indptr[r]), int(indptr[r + 1])
        c = col_map[indices[a:b]]
        keep = c >= 0
        cols.append(c[keep])
        vi.append(np.arange(a, b, dtype=np.int64)[keep])
        ptr.append(ptr[-1] + int(keep.sum()))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dtype=dt)
    return np.asarray(ptr, dtype=np.int64), cat(cols, np.int32), cat(vi, np.int64)


class DeviceKKT:
    """Newton matrix of the reference IPM for one NlpProblem of this package, on its device."""

    def __init__(self, problem):
        import torch
        self.torch = torch
        self.p = problem
        ev = problem.evaluator
        self.ev = ev
        self.dev = torch.device("cuda", ev.device)
        fixed = problem.xl == problem.xu
        self.free = np.flatnonzero(~fixed)
        self.nf = len(self.free)
        self.me = problem.m_eq
        self.mi = problem.m_ineq
        col_map = np.full(problem.n, -1, dtype=np.int64)
        col_map[self.free] = np.arange(self.nf)
        jp, ji = ev.pattern("J")
        hp, hi = ev.pattern("H")
        h = _csr_sub(hp, hi, self.free, col_map)
        je = _csr_sub(jp, ji, range(self.me), col_map)
        jin = _csr_sub(jp, ji, range(self.me, self.me + self.mi), col_map)
        # Ji as CSC over free columns (rows ascending within a column)
        ji_ptr, ji_col, ji_vi = jin
        rows = np.repeat(np.arange(self.mi, dtype=np.int32), np.diff(ji_ptr))
        order = np.lexsort((rows, ji_col))
        jt_ptr = np.zeros(self.nf + 1, dtype=np.int64)
        np.cumsum(np.bincount(ji_col, minlength=self.nf), out=jt_ptr[1:])
        jt = (jt_ptr, rows[order].astype(np.int32), ji_vi[order])
        up = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=self.dev)
        self._h = [up(a) for a in h]
        self._je = [up(a) for a in je]
        self._ji = [up(a) for a in jin]
        self._jt = [up(a) for a in jt]
        self.dim = self.nf + self.me

    def assemble(self, jval, hval, dx, ds, reg: float = 0.0, delta: float = 0.0, sc=None, out=None):
        """K (dim x dim, float64, symmetric) on the device from device J / H values.
        dx: per free variable; ds: per inequality row; sc: the view's row scales (m) or None."""
        torch = self.torch
        K = out if out is not None else torch.zeros((self.dim, self.dim), dtype=torch.float64, device=self.dev)
        if out is not None:
            K.zero_()
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=self.dev) \
            if not isinstance(a, torch.Tensor) else a.to(self.dev, torch.float64).contiguous()
        dx_d, ds_d = t(dx), t(ds if self.mi else np.zeros(1))
        sc_d = t(sc) if sc is not None else None
        vp = lambda a: ctypes.c_void_p(a.data_ptr()) if a is not None else None
        sc_e = vp(sc_d[:self.me]) if sc_d is not None and self.me else None
        sc_i = vp(sc_d[self.me:]) if sc_d is not None and self.mi else None
        h, je, ji, jt = self._h, self._je, self._ji, self._jt
        st = self.ev.stream_handle(None)
        L.check(L.lib().acopf_kkt_assemble(
            self.nf, self.me, vp(K), vp(h[0]), vp(h[1]), vp(h[2]), vp(hval), vp(dx_d), vp(jt[0]), vp(jt[1]),
            vp(jt[2]), vp(ji[0]), vp(ji[1]), vp(ji[2]), vp(jval), vp(ds_d), vp(je[0]), vp(je[1]), vp(je[2]),
            sc_e, sc_i, float(reg), float(delta), st))
        self._keep = (dx_d, ds_d, sc_d)
        return K

    def factor(self, K):
        """(LD, pivots, (positive, negative) inertia) of Bunch-Kaufman LDL^T (cuSOLVER sytrf)."""
        torch = self.torch
        LD, piv, info = torch.linalg.ldl_factor_ex(K)
        d = torch.diagonal(LD).cpu().numpy()
        e = torch.diagonal(LD, -1).cpu().numpy()
        p = piv.cpu().numpy()
        return LD, piv, _inertia(d, e, p), int(info.item())

    def solve(self, LD, piv, rhs):
        torch = self.torch
        b = rhs if isinstance(rhs, torch.Tensor) else torch.as_tensor(np.asarray(rhs, dtype=np.float64), device=self.dev)
        return torch.linalg.ldl_solve(LD, piv, b.reshape(-1, 1)).reshape(-1)


def _inertia(d, e, piv):
    """(positive, negative) eigenvalue counts of D from LAPACK-style pivots (1-based; a 2x2 block
    has equal negative entries) -- _BunchKaufman._inertia (ipm.py:193-215)."""
    pos = neg = 0
    k, n = 0, len(d)
    while k < n:
        if piv[k] > 0:
            if d[k] > 0.0:
                pos += 1
            elif d[k] < 0.0:
                neg += 1
            k += 1
        else:
            a, c, b = d[k], d[k + 1], e[k]
            det = a * c - b * b
            if det < 0.0:
                pos += 1
                neg += 1
            elif a + c > 0.0:
                pos += 2
            else:
                neg += 2
            k += 2
    return pos, neg
