"""CPU ORACLE binding — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The product path
(paper_1607_00315_b200/) never imports, links or executes anything here.

The oracle (mlo.c) is a plain single-threaded fp64 C implementation of the
multilevel proximal-Newton method written from PAPER.md (Algorithm 1
P:155-173, Eqs. 3-6); see mlo.h and
DESIGN.md "Oracle".  It shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmlo.so")

OK, E_INVAL, E_STAGNATION, E_NOT_CONVERGED, E_CONTRACT = 0, 1, 4, 5, 6
R_UPDATED, R_CONVERGED, R_NOSTEP, R_STAGNATION = 0, 1, 2, 3


class Opts(ctypes.Structure):
    _fields_ = [("tol_kkt", ctypes.c_double), ("max_cycles", ctypes.c_int32), ("nu", ctypes.c_int32),
                ("nu_c", ctypes.c_int32), ("K_fine", ctypes.c_int32), ("K_mid", ctypes.c_int32),
                ("K_coarse", ctypes.c_int32), ("sigma_out", ctypes.c_double), ("sigma_in", ctypes.c_double),
                ("beta", ctypes.c_double), ("max_ls", ctypes.c_int32), ("eps_h", ctypes.c_double),
                ("multilevel", ctypes.c_int32), ("inner_cg", ctypes.c_int32), ("eta", ctypes.c_double),
                ("pcd_snap", ctypes.c_int32), ("continuation", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("F", ctypes.c_double), ("kappa", ctypes.c_double), ("vinf", ctypes.c_double),
                ("v1", ctypes.c_double), ("paper_ratio", ctypes.c_double),
                ("status", ctypes.c_int32), ("cycles", ctypes.c_int32),
                ("relaxations", ctypes.c_int64), ("relax_per_level", ctypes.c_int64 * 32),
                ("max_supp", ctypes.c_int64), ("nnz_w", ctypes.c_int64),
                ("nnz_touched", ctypes.c_int64), ("x_passes", ctypes.c_int64)]


class TraceRow(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("outcome", ctypes.c_int32), ("inner_iters", ctypes.c_int32),
                ("nA", ctypes.c_int32), ("nC", ctypes.c_int64), ("F_before", ctypes.c_double),
                ("F_after", ctypes.c_double), ("alpha", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile liboracle in-tree: plain C, -O2 -ffp-contract=off, no fast-math."""
    src = os.path.join(_HERE, "mlo.c")
    hdr = os.path.join(_HERE, "mlo.h")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(os.path.getmtime(src), os.path.getmtime(hdr)):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", _SO, src, "-lm"])
    return _SO


_lib = None
_P = ctypes.c_void_p


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(_SO)
    d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int32
    L.mlo_default_opts.argtypes = [ctypes.POINTER(Opts)]
    L.mlo_create.restype = _P
    L.mlo_create.argtypes = [i64, i64, i64, _P, _P, _P, _P, _P, _P, _P, d]
    L.mlo_create_lasso.restype = _P
    L.mlo_create_lasso.argtypes = [i64, i64, i64, _P, _P, _P, _P, _P, _P, _P, d]
    L.mlo_destroy.argtypes = [_P]
    L.mlo_set_w.argtypes = [_P, _P]
    L.mlo_get_w.argtypes = [_P, _P]
    L.mlo_get_rows.argtypes = [_P, _P, _P, _P, _P]
    L.mlo_eval_f_grad.argtypes = [_P, _P, i64, ctypes.POINTER(d), _P, _P]
    L.mlo_diag_hess.argtypes = [_P, _P, i64, _P]
    L.mlo_hessvec.argtypes = [_P, _P, i64, _P, _P]
    L.mlo_shrink_linesearch.argtypes = [_P, _P, i64, _P, _P, _P, _P, ctypes.POINTER(Opts),
                                        ctypes.POINTER(d), ctypes.POINTER(d)]
    L.mlo_select_coarse.argtypes = [_P, _P, i64, _P, ctypes.POINTER(i64)]
    L.mlo_relax.argtypes = [_P, _P, i64, i32, ctypes.POINTER(Opts), ctypes.POINTER(i32)]
    L.mlo_solve.argtypes = [_P, ctypes.POINTER(Opts), ctypes.POINTER(Report)]
    L.mlo_level_sizes.restype = i32
    L.mlo_level_sizes.argtypes = [i64, i64, i64, _P]
    L.mlo_trace_len.restype = i64
    L.mlo_trace_len.argtypes = [_P]
    L.mlo_trace_get.argtypes = [_P, i64, ctypes.POINTER(TraceRow)]
    L.mlo_trace_clear.argtypes = [_P]
    for f in ("mlo_soft_shrink", "mlo_logloss", "mlo_tau", "mlo_weight"):
        getattr(L, f).restype = d
    L.mlo_soft_shrink.argtypes = [d, d]
    L.mlo_logloss.argtypes = [d]
    L.mlo_tau.argtypes = [d]
    L.mlo_weight.argtypes = [d]
    L.mlo_scalar_prox.restype = d
    L.mlo_scalar_prox.argtypes = [d, d, d]
    _lib = L
    return L


def lib():
    return _load()


def default_opts(**over) -> Opts:
    o = Opts()
    _load().mlo_default_opts(ctypes.byref(o))
    for k, v in over.items():
        setattr(o, k, v)
    return o


def level_sizes(nAf: int, nS: int, n: int) -> list[int]:
    k = np.zeros(64, np.int64)
    L = _load().mlo_level_sizes(int(nAf), int(nS), int(n), k.ctypes.data_as(_P))
    return [int(x) for x in k[:L + 1]]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _C(C, n):
    if C is None:
        return None, n
    C = np.ascontiguousarray(C, np.int32)
    return C, len(C)


class Oracle:
    """ctypes wrapper over one oracle context (host arrays, kept alive here)."""

    def __init__(self, ds):
        L = _load()
        self.ds = ds
        self._keep = [np.ascontiguousarray(a) for a in (ds.csr_rowptr, ds.csr_col, ds.csr_val, ds.csc_colptr,
                                                         ds.csc_row, ds.csc_val, ds.y)]
        k = self._keep
        self.m, self.n = ds.m, ds.n
        if getattr(ds, "b", None) is not None:   # squared loss (LASSO): targets b in place of the labels
            k[-1] = np.ascontiguousarray(ds.b, np.float64)
            self.h = L.mlo_create_lasso(ds.m, ds.n, ds.nnz, *[_ptr(a) for a in k], float(ds.lam))
        else:
            self.h = L.mlo_create(ds.m, ds.n, ds.nnz, *[_ptr(a) for a in k], float(ds.lam))
        if not self.h:
            raise ValueError("mlo_create rejected the input")

    def __del__(self):
        if getattr(self, "h", None):
            _load().mlo_destroy(self.h)
            self.h = None

    def set_w(self, w):
        w = np.ascontiguousarray(w, np.float64)
        _load().mlo_set_w(self.h, _ptr(w))

    def get_w(self):
        w = np.zeros(self.n)
        _load().mlo_get_w(self.h, _ptr(w))
        return w

    def rows(self):
        z, r, D, ell = (np.zeros(self.m) for _ in range(4))
        _load().mlo_get_rows(self.h, _ptr(z), _ptr(r), _ptr(D), _ptr(ell))
        return z, r, D, ell

    def eval_f_grad(self, C=None):
        C, nC = _C(C, self.n)
        F = ctypes.c_double()
        g, h = np.zeros(nC), np.zeros(nC)
        st = _load().mlo_eval_f_grad(self.h, _ptr(C), nC, ctypes.byref(F), _ptr(g), _ptr(h))
        if st:
            raise ValueError(f"mlo_eval_f_grad status {st}")
        return F.value, g, h

    def diag_hess(self, C=None):
        C, nC = _C(C, self.n)
        h = np.zeros(nC)
        st = _load().mlo_diag_hess(self.h, _ptr(C), nC, _ptr(h))
        if st:
            raise ValueError(f"status {st}")
        return h

    def hessvec(self, C, v):
        C, nC = _C(C, self.n)
        v = np.ascontiguousarray(v, np.float64)
        Hv = np.zeros(nC)
        st = _load().mlo_hessvec(self.h, _ptr(C), nC, _ptr(v), _ptr(Hv))
        if st:
            raise ValueError(f"status {st}")
        return Hv

    def shrink_linesearch(self, C, g, h=None, d=None, Xd=None, opts=None):
        C, nC = _C(C, self.n)
        opts = opts or default_opts()
        a, F = ctypes.c_double(), ctypes.c_double()
        arrs = [None if x is None else np.ascontiguousarray(x, np.float64) for x in (g, h, d, Xd)]
        st = _load().mlo_shrink_linesearch(self.h, _ptr(C), nC, *[_ptr(x) for x in arrs], ctypes.byref(opts),
                                           ctypes.byref(a), ctypes.byref(F))
        return a.value, F.value, st

    def select_coarse(self, g, k_total):
        g = np.ascontiguousarray(g, np.float64)
        out = np.zeros(self.n, np.int32)
        nout = ctypes.c_int64()
        _load().mlo_select_coarse(self.h, _ptr(g), int(k_total), _ptr(out), ctypes.byref(nout))
        return out[:nout.value].copy()

    def relax(self, C, K, opts=None):
        C, nC = _C(C, self.n)
        opts = opts or default_opts()
        oc = ctypes.c_int32()
        st = _load().mlo_relax(self.h, _ptr(C), nC, int(K), ctypes.byref(opts), ctypes.byref(oc))
        return st, oc.value

    def solve(self, opts=None):
        opts = opts or default_opts()
        rep = Report()
        _load().mlo_solve(self.h, ctypes.byref(opts), ctypes.byref(rep))
        d = {f: getattr(rep, f) for f, _ in Report._fields_ if f != "relax_per_level"}
        d["relax_per_level"] = list(rep.relax_per_level)
        return d

    def trace(self):
        L = _load()
        out = []
        for i in range(L.mlo_trace_len(self.h)):
            r = TraceRow()
            L.mlo_trace_get(self.h, i, ctypes.byref(r))
            out.append({f: getattr(r, f) for f, _ in TraceRow._fields_})
        return out

    def clear_trace(self):
        _load().mlo_trace_clear(self.h)
