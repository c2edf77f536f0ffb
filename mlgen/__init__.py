"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic.  It draws X (CSR + CSC,
fp32 values / int32 indices), labels y in {-1,+1}, a planted w* and the
configuration's lambda (BASELINE.json defines lambda = factor * lambda_max,
lambda_max = 1/2 ||X^T y||_inf).  The recipe is DESIGN.md "Input recipe";
the synthetic data stand in for the paper's data sets.

`make(cfg)` builds BASELINE.json config 1..5 (C generator, mlgen.c); the
numpy helpers build the small structured designs the oracle pins use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmlgen.so")

DENSE_IID, DENSE_BLOCK, ZIPF = 0, 1, 2
LABEL_SIGN_NOISE, LABEL_LOGISTIC = 0, 1


class _Params(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("label", ctypes.c_int32),
                ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("mean_row_nnz", ctypes.c_double), ("zipf_s", ctypes.c_double),
                ("block", ctypes.c_int64), ("nnz_w", ctypes.c_int64),
                ("w_var", ctypes.c_double), ("label_noise", ctypes.c_double),
                ("flip_prob", ctypes.c_double), ("lambda_factor", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


class _Data(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("nnz_w", ctypes.c_int64),
                ("csr_rowptr", ctypes.POINTER(ctypes.c_int32)), ("csr_col", ctypes.POINTER(ctypes.c_int32)),
                ("csr_val", ctypes.POINTER(ctypes.c_float)),
                ("csc_colptr", ctypes.POINTER(ctypes.c_int32)), ("csc_row", ctypes.POINTER(ctypes.c_int32)),
                ("csc_val", ctypes.POINTER(ctypes.c_float)),
                ("y", ctypes.POINTER(ctypes.c_int8)),
                ("wstar_idx", ctypes.POINTER(ctypes.c_int32)), ("wstar_val", ctypes.POINTER(ctypes.c_double)),
                ("lambda_max", ctypes.c_double), ("lam", ctypes.c_double)]


def build(force: bool = False) -> str:
    """Compile libmlgen.so in-tree (gcc, OpenMP)."""
    src = os.path.join(_HERE, "mlgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "mlgen.h"))):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.mlgen_generate.restype = ctypes.POINTER(_Data)
        lib.mlgen_generate.argtypes = [ctypes.POINTER(_Params)]
        lib.mlgen_free.argtypes = [ctypes.POINTER(_Data)]
        lib.mlgen_preset.argtypes = [ctypes.c_int, ctypes.POINTER(_Params)]
        _lib = lib
    return _lib


@dataclass
class Dataset:
    """X (m x n, rows = samples) in CSR and CSC, labels, lambda."""
    m: int
    n: int
    csr_rowptr: np.ndarray
    csr_col: np.ndarray
    csr_val: np.ndarray
    csc_colptr: np.ndarray
    csc_row: np.ndarray
    csc_val: np.ndarray
    y: np.ndarray
    lam: float
    lambda_max: float = float("nan")
    wstar_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    wstar_val: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    name: str = ""
    b: np.ndarray | None = None   # squared-loss (LASSO) targets [m], fp64; None = logistic labels y

    @property
    def nnz(self) -> int:
        return int(self.csr_rowptr[-1])

    def with_lambda(self, lam: float) -> "Dataset":
        import copy
        d = copy.copy(self)
        d.lam = float(lam)
        return d

    def dense(self) -> np.ndarray:
        X = np.zeros((self.m, self.n), np.float64)
        for i in range(self.m):
            s, e = self.csr_rowptr[i], self.csr_rowptr[i + 1]
            X[i, self.csr_col[s:e]] = self.csr_val[s:e]
        return X


def params(cfg: int, **over) -> _Params:
    p = _Params()
    _load().mlgen_preset(cfg, ctypes.byref(p))
    for k, v in over.items():
        setattr(p, k, v)
    return p


def generate(p: _Params, name: str = "") -> Dataset:
    lib = _load()
    ptr = lib.mlgen_generate(ctypes.byref(p))
    if not ptr:
        raise ValueError("mlgen_generate failed (bad sizes or out of memory)")
    d = ptr.contents
    m, n, nnz, nw = d.m, d.n, d.nnz, d.nnz_w

    def arr(p_, count, dt):
        if count == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(p_, shape=(count,)).astype(dt, copy=True)

    ds = Dataset(m=m, n=n,
                 csr_rowptr=arr(d.csr_rowptr, m + 1, np.int32), csr_col=arr(d.csr_col, nnz, np.int32),
                 csr_val=arr(d.csr_val, nnz, np.float32),
                 csc_colptr=arr(d.csc_colptr, n + 1, np.int32), csc_row=arr(d.csc_row, nnz, np.int32),
                 csc_val=arr(d.csc_val, nnz, np.float32),
                 y=arr(d.y, m, np.int8), lam=d.lam, lambda_max=d.lambda_max,
                 wstar_idx=arr(d.wstar_idx, nw, np.int32), wstar_val=arr(d.wstar_val, nw, np.float64),
                 name=name)
    lib.mlgen_free(ptr)
    return ds


def make(cfg: int, **over) -> Dataset:
    """BASELINE.json config `cfg` (1..5), optionally with overridden fields (e.g. m, n for scaled variants)."""
    return generate(params(cfg, **over), name=f"cfg{cfg}" + ("" if not over else "-" + "-".join(
        f"{k}{v}" for k, v in sorted(over.items()))))


# ----------------------------------------------------------------- small structured designs
def from_dense(X: np.ndarray, y: np.ndarray, lam: float, name: str = "dense") -> Dataset:
    """CSR/CSC of the nonzeros of a dense fp32 matrix (explicit zeros are dropped)."""
    X = np.asarray(X, np.float32)
    m, n = X.shape
    rows, cols = np.nonzero(X)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    vals = X[rows, cols]
    rowptr = np.zeros(m + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    corder = np.lexsort((rows, cols))
    colptr = np.zeros(n + 1, np.int64)
    np.add.at(colptr, cols + 1, 1)
    colptr = np.cumsum(colptr)
    return Dataset(m=m, n=n, csr_rowptr=rowptr.astype(np.int32), csr_col=cols.astype(np.int32),
                   csr_val=vals.astype(np.float32), csc_colptr=colptr.astype(np.int32),
                   csc_row=rows[corder].astype(np.int32), csc_val=vals[corder].astype(np.float32),
                   y=np.asarray(y, np.int8), lam=float(lam), name=name)


def random_sparse(m: int, n: int, density: float, seed: int, lam_factor: float = 0.1,
                  empty_rows: int = 0, empty_cols: int = 0) -> Dataset:
    """Small random sparse design (N(0,1) values) with optional empty rows/columns; labels +-1 uniform."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((m, n)).astype(np.float32)
    X[rng.random((m, n)) >= density] = 0.0
    if empty_rows:
        X[rng.choice(m, empty_rows, replace=False)] = 0.0
    if empty_cols:
        X[:, rng.choice(n, empty_cols, replace=False)] = 0.0
    y = np.where(rng.random(m) < 0.5, 1, -1).astype(np.int8)
    lmax = 0.5 * np.max(np.abs(X.astype(np.float64).T @ y.astype(np.float64))) if X.any() else 1.0
    return from_dense(X, y, lam_factor * lmax if lmax > 0 else 1.0, name=f"rs{m}x{n}s{seed}")


def onehot(n: int, seed: int, rows_per_col=(2, 12), lam: float | None = None) -> tuple[Dataset, np.ndarray, np.ndarray, np.ndarray]:
    """One-hot separable design: row i has a single nonzero X[i, c(i)] = a_{c(i)}.

    Column j has p_j positive and q_j negative rows; a_j distinct in [0.5, 1.5].
    Returns (dataset, a, p, q).  Rows are shuffled so columns interleave in CSR order.
    """
    rng = np.random.default_rng(seed)
    a = np.sort(rng.uniform(0.5, 1.5, n))
    a = rng.permutation(a)
    p = rng.integers(rows_per_col[0], rows_per_col[1] + 1, n)
    q = rng.integers(rows_per_col[0], rows_per_col[1] + 1, n)
    cols = np.concatenate([np.full(p[j] + q[j], j) for j in range(n)])
    lab = np.concatenate([np.r_[np.ones(p[j]), -np.ones(q[j])] for j in range(n)])
    perm = rng.permutation(len(cols))
    cols, lab = cols[perm], lab[perm]
    m = len(cols)
    rowptr = np.arange(m + 1, dtype=np.int32)
    vals = a[cols].astype(np.float32)
    corder = np.lexsort((np.arange(m), cols))
    colptr = np.zeros(n + 1, np.int64)
    np.add.at(colptr, cols + 1, 1)
    colptr = np.cumsum(colptr)
    a32 = a.astype(np.float32).astype(np.float64)  # the stored (fp32) scales
    if lam is None:
        lmax = 0.5 * np.max(a32 * np.abs(p - q))
        lam = 0.3 * lmax
    ds = Dataset(m=m, n=n, csr_rowptr=rowptr, csr_col=cols.astype(np.int32), csr_val=vals,
                 csc_colptr=colptr.astype(np.int32), csc_row=corder.astype(np.int32),
                 csc_val=vals[corder], y=lab.astype(np.int8), lam=float(lam), name=f"onehot{n}s{seed}")
    return ds, a32, p, q


# ----------------------------------------------------------------- squared-loss (LASSO) instances
def lasso(base: Dataset, seed: int, k: int = 10, noise: float = 0.1, lam_factor: float = 0.1) -> Dataset:
    """The LASSO instance of Eq. 2 on the design of `base`: targets b = X w* + noise, with w* holding k
    N(0, 1) values at uniform random columns; lambda = lam_factor * lambda_max, lambda_max = ||X^T b||_inf (w = 0 is
    optimal iff lambda >= lambda_max).  Targets and lambda are inputs: no solver arithmetic here."""
    import copy
    rng = np.random.default_rng(seed)
    wi = np.sort(rng.choice(base.n, min(k, base.n), replace=False)).astype(np.int32)
    wv = rng.standard_normal(len(wi))
    w = np.zeros(base.n)
    w[wi] = wv
    rp, ci, cv = base.csr_rowptr, base.csr_col, base.csr_val.astype(np.float64)
    rows = np.repeat(np.arange(base.m), np.diff(rp))
    z = np.zeros(base.m)
    np.add.at(z, rows, cv * w[ci])
    b = z + noise * rng.standard_normal(base.m)
    g0 = np.zeros(base.n)
    np.add.at(g0, ci, cv * b[rows])
    lmax = float(np.max(np.abs(g0))) if base.nnz else 1.0
    d = copy.copy(base)
    d.b = b
    d.lambda_max = lmax
    d.lam = lam_factor * lmax if lmax > 0 else 1.0
    d.wstar_idx, d.wstar_val = wi, wv
    d.name = base.name + f"-lasso{seed}"
    return d
