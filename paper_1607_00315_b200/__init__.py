"""Thin Python binding of libml (include/ml.h) — argument marshalling only.

Every step of the hot path runs in libml's sm_100a kernels.  PyTorch is used only to allocate device memory and to
supply the CUDA stream.  There is no CPU fallback: `load()` raises when libml.so is missing, and `Context` raises
when no CUDA device is present.

Names follow the C ABI: ml_create, ml_eval_f_grad, ml_diag_hess, ml_hessvec, ml_shrink_linesearch,
ml_select_coarse, ml_solve (Algorithm 1 P:155-173 applied to l1-logistic regression P:783-798).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libml.so")
_SRC = os.path.join(_HERE, "csrc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

(ML_OK, ML_E_INVAL, ML_E_CUDA, ML_E_WORKSPACE, ML_E_STAGNATION, ML_E_NOT_CONVERGED, ML_E_CONTRACT,
 ML_E_NONFINITE) = range(8)


def _sources():
    return [os.path.join(_SRC, f) for f in sorted(os.listdir(_SRC))] + [os.path.join(_HERE, "..", "include", "ml.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libml.so in-tree for sm_100a (nvcc; no GPU needed)."""
    newest = max(os.path.getmtime(p) for p in _sources())
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["nvcc", *NVCC_FLAGS, "-o", _SO, os.path.join(_SRC, "ml.cu")]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
    return _SO


class MLData(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("csr_rowptr", ctypes.c_void_p), ("csr_col", ctypes.c_void_p), ("csr_val", ctypes.c_void_p),
                ("csc_colptr", ctypes.c_void_p), ("csc_row", ctypes.c_void_p), ("csc_val", ctypes.c_void_p),
                ("y", ctypes.c_void_p)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("tol_kkt", ctypes.c_double), ("max_cycles", ctypes.c_int32), ("nu", ctypes.c_int32),
                ("nu_c", ctypes.c_int32), ("K_fine", ctypes.c_int32), ("K_mid", ctypes.c_int32),
                ("K_coarse", ctypes.c_int32), ("sigma_out", ctypes.c_double), ("sigma_in", ctypes.c_double),
                ("beta", ctypes.c_double), ("max_ls", ctypes.c_int32), ("eps_h", ctypes.c_double),
                ("multilevel", ctypes.c_int32), ("inner_cg", ctypes.c_int32), ("eta", ctypes.c_double),
                ("pcd_snap", ctypes.c_int32), ("continuation", ctypes.c_int32)]


class SolveReport(ctypes.Structure):
    _fields_ = [("F", ctypes.c_double), ("kappa", ctypes.c_double), ("vinf", ctypes.c_double),
                ("v1", ctypes.c_double), ("paper_ratio", ctypes.c_double),
                ("status", ctypes.c_int32), ("cycles", ctypes.c_int32),
                ("relaxations", ctypes.c_int64), ("relax_per_level", ctypes.c_int64 * 32),
                ("max_supp", ctypes.c_int64), ("nnz_w", ctypes.c_int64),
                ("nnz_touched", ctypes.c_int64), ("x_passes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64)]


class TraceRow(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("outcome", ctypes.c_int32), ("inner_iters", ctypes.c_int32),
                ("nA", ctypes.c_int32), ("nC", ctypes.c_int64), ("F_before", ctypes.c_double),
                ("F_after", ctypes.c_double), ("alpha", ctypes.c_double)]


EXPORTS = ["ml_default_opts", "ml_workspace_bytes", "ml_create", "ml_create_lasso", "ml_destroy", "ml_set_w", "ml_get_w", "ml_get_rows",
           "ml_eval_f_grad", "ml_diag_hess", "ml_hessvec", "ml_shrink_linesearch", "ml_select_coarse", "ml_solve",
           "ml_status_str", "ml_last_error", "ml_kernel_launches", "ml_trace", "ml_profile",
           "ml_profile_read", "ml_inner_phases", "ml_set_sm_share", "ml_set_engine", "ml_heavy_info"]

_lib = None


def load(path: str | None = None):
    """Load libml.so (raises OSError if it is missing — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("ML_LIB") or _SO   # ML_LIB: an alternative build of the same library (tools)
    if not os.path.exists(p):
        raise OSError(f"libml.so not built ({p}); run paper_1607_00315_b200.build()")
    L = ctypes.CDLL(p)
    P, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    L.ml_default_opts.argtypes = [ctypes.POINTER(SolveOpts)]
    L.ml_workspace_bytes.restype = ctypes.c_size_t
    L.ml_workspace_bytes.argtypes = [i64, i64, i64]
    L.ml_create.restype = i32
    L.ml_create.argtypes = [ctypes.POINTER(MLData), d, P, P, ctypes.c_size_t, ctypes.POINTER(P)]
    if hasattr(L, "ml_create_lasso"):   # (older builds, e.g. ML_LIB bisection, predate these entry points)
        L.ml_create_lasso.restype = i32
        L.ml_create_lasso.argtypes = [ctypes.POINTER(MLData), P, d, P, P, ctypes.c_size_t, ctypes.POINTER(P)]
    for f in ("ml_destroy",):
        getattr(L, f).restype = i32
        getattr(L, f).argtypes = [P]
    for f in ("ml_set_w", "ml_get_w"):
        getattr(L, f).restype = i32
        getattr(L, f).argtypes = [P, P]
    L.ml_get_rows.restype = i32
    L.ml_get_rows.argtypes = [P, P, P, P]
    L.ml_eval_f_grad.restype = i32
    L.ml_eval_f_grad.argtypes = [P, P, i64, ctypes.POINTER(d), P, P]
    L.ml_diag_hess.restype = i32
    L.ml_diag_hess.argtypes = [P, P, i64, P]
    L.ml_hessvec.restype = i32
    L.ml_hessvec.argtypes = [P, P, i64, P, P]
    L.ml_shrink_linesearch.restype = i32
    L.ml_shrink_linesearch.argtypes = [P, P, i64, P, P, P, P, ctypes.POINTER(SolveOpts), ctypes.POINTER(d),
                                       ctypes.POINTER(d)]
    L.ml_select_coarse.restype = i32
    L.ml_select_coarse.argtypes = [P, P, i64, P, ctypes.POINTER(i64)]
    L.ml_solve.restype = i32
    L.ml_solve.argtypes = [P, ctypes.POINTER(SolveOpts), ctypes.POINTER(SolveReport)]
    L.ml_status_str.restype = ctypes.c_char_p
    L.ml_status_str.argtypes = [i32]
    L.ml_last_error.restype = ctypes.c_char_p
    L.ml_last_error.argtypes = [P]
    L.ml_kernel_launches.restype = i64
    L.ml_kernel_launches.argtypes = [P]
    L.ml_profile.restype = i32
    L.ml_profile.argtypes = [P, ctypes.c_uint32]
    L.ml_profile_read.restype = i32
    L.ml_profile_read.argtypes = [P, P, P, P, P]
    L.ml_inner_phases.restype = i32
    L.ml_inner_phases.argtypes = [P, P, i32]
    if hasattr(L, "ml_set_sm_share"):
        L.ml_set_sm_share.restype = i32
        L.ml_set_sm_share.argtypes = [P, i32]
    if hasattr(L, "ml_set_engine"):
        L.ml_set_engine.restype = i32
        L.ml_set_engine.argtypes = [P, ctypes.c_uint32]
    L.ml_trace.restype = i64
    L.ml_trace.argtypes = [P, P, i64]
    L.ml_heavy_info.restype = i32
    L.ml_heavy_info.argtypes = [P, P]
    _lib = L
    return L


def default_opts(**over) -> SolveOpts:
    o = SolveOpts()
    load().ml_default_opts(ctypes.byref(o))
    for k, v in over.items():
        setattr(o, k, v)
    return o


class MLError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libml status {status}: {msg}")
        self.status = status


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Context:
    """One ml_ctx bound to device copies of X (CSR + CSC), y and a workspace.

    `ds` is an mlgen.Dataset (host numpy arrays); the arrays are copied once to the device (outside any timed
    region).  All methods take / return torch CUDA tensors.
    """

    def __init__(self, ds, lam: float | None = None, device: str = "cuda:0", stream=None, host_tensors=None,
                 csr: bool = True, ws_fill: int | None = None, dense: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libml needs a CUDA device (no CPU fallback)")
        L = load()
        self.torch = torch
        self.device = torch.device(device)
        self.m, self.n, self.nnz = int(ds.m), int(ds.n), int(ds.nnz)
        self.lam = float(ds.lam if lam is None else lam)
        dev = self.device

        if host_tensors is not None:   # pinned host tensors (rowptr, col, val, colptr, row, val, y): H2D copies
            (self.csr_rowptr, self.csr_col, self.csr_val, self.csc_colptr, self.csc_row, self.csc_val,
             self.y) = (None if t is None else t.to(dev, non_blocking=True) for t in host_tensors)
        else:
            def up(a, dt):
                return torch.from_numpy(a).to(dev, dt)

            # csr=False: columns only (accepted by ml_create for m <= 8192, include/ml.h); dense=True: the index-free
            # dense X (column-major values only: no CSR, no CSC pointers or row indices; nnz = m n, m <= 8192)
            if dense:
                csr = False
            self.csr_rowptr = up(ds.csr_rowptr, torch.int32) if csr else None
            self.csr_col = up(ds.csr_col, torch.int32) if csr else None
            self.csr_val = up(ds.csr_val, torch.float32) if csr else None
            self.csc_colptr = None if dense else up(ds.csc_colptr, torch.int32)
            self.csc_row = None if dense else up(ds.csc_row, torch.int32)
            self.csc_val = up(ds.csc_val, torch.float32)
            self.y = up(ds.y, torch.int8)
        self.stream = stream or torch.cuda.current_stream(dev)
        wsb = int(L.ml_workspace_bytes(self.m, self.n, self.nnz))
        self.ws = torch.empty(wsb + 512, dtype=torch.uint8, device=dev)
        if ws_fill is not None:   # (tests: a workspace that held other data before; ml_create must not depend on it)
            words = self.ws[: (wsb + 512) // 8 * 8].view(torch.int64)
            if ws_fill == "epochs":   # look-back status words of epochs 0..63 (flag 1, count 5), cycling
                words.copy_(((torch.arange(words.numel(), device=dev, dtype=torch.int64) % 64) << 34) | (1 << 32) | 5)
            else:
                words.fill_(int(ws_fill))
        self.data = MLData(self.m, self.n, self.nnz, *[0 if t is None else t.data_ptr() for t in (
            self.csr_rowptr, self.csr_col, self.csr_val, self.csc_colptr, self.csc_row, self.csc_val, self.y)])
        h = ctypes.c_void_p()
        self.b = None if getattr(ds, "b", None) is None else torch.from_numpy(np.asarray(ds.b, np.float64)).to(dev)
        if self.b is not None:   # the squared-loss (LASSO) instance
            st = L.ml_create_lasso(ctypes.byref(self.data), ctypes.c_void_p(self.b.data_ptr()), self.lam,
                                   ctypes.c_void_p(self.stream.cuda_stream), ctypes.c_void_p(self.ws.data_ptr()),
                                   self.ws.numel(), ctypes.byref(h))
        else:
            st = L.ml_create(ctypes.byref(self.data), self.lam, ctypes.c_void_p(self.stream.cuda_stream),
                             ctypes.c_void_p(self.ws.data_ptr()), self.ws.numel(), ctypes.byref(h))
        if st != ML_OK:
            raise MLError(st, L.ml_status_str(st).decode())
        self.h = h

    @classmethod
    def from_host(cls, ds, pinned, device="cuda:0"):
        """Public entry with host buffers: H2D of X and y from pinned memory, then ml_create.  `pinned` lists
        (csr_rowptr, csr_col, csr_val, csc_colptr, csc_row, csc_val, y); the CSR entries may be None for m <= 8192."""
        return cls(ds, device=device, host_tensors=pinned)

    # ------------------------------------------------------------------ helpers
    def _check(self, st, allow=()):
        if st != ML_OK and st not in allow:
            L = load()
            raise MLError(st, f"{L.ml_status_str(st).decode()} {L.ml_last_error(self.h).decode()}")
        return st

    def _C(self, C):
        if C is None:
            return None, self.n
        return C, int(C.numel())

    def dvec(self, k):
        return self.torch.zeros(k, dtype=self.torch.float64, device=self.device)

    def close(self):
        if getattr(self, "h", None):
            load().ml_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ the C ABI
    def ml_set_w(self, w):
        return self._check(load().ml_set_w(self.h, _ptr(w.contiguous())))

    def ml_get_w(self):
        w = self.dvec(self.n)
        self._check(load().ml_get_w(self.h, _ptr(w)))
        return w

    def ml_get_rows(self):
        z, r, D = self.dvec(self.m), self.dvec(self.m), self.dvec(self.m)
        self._check(load().ml_get_rows(self.h, _ptr(z), _ptr(r), _ptr(D)))
        return z, r, D

    def ml_eval_f_grad(self, C=None, want_g=True, want_h=True):
        C, nC = self._C(C)
        g = self.dvec(nC) if want_g else None
        h = self.dvec(nC) if want_h else None
        F = ctypes.c_double()
        self._check(load().ml_eval_f_grad(self.h, _ptr(C), nC, ctypes.byref(F), _ptr(g), _ptr(h)))
        return F.value, g, h

    def ml_diag_hess(self, C=None):
        C, nC = self._C(C)
        h = self.dvec(nC)
        self._check(load().ml_diag_hess(self.h, _ptr(C), nC, _ptr(h)))
        return h

    def ml_hessvec(self, C, v):
        C, nC = self._C(C)
        Hv = self.dvec(nC)
        self._check(load().ml_hessvec(self.h, _ptr(C), nC, _ptr(v.contiguous()), _ptr(Hv)))
        return Hv

    def ml_shrink_linesearch(self, C, g, h=None, d=None, Xd=None, opts=None):
        C, nC = self._C(C)
        a, F = ctypes.c_double(), ctypes.c_double()
        opts = opts or default_opts()
        st = load().ml_shrink_linesearch(self.h, _ptr(C), nC, _ptr(g), _ptr(h), _ptr(d), _ptr(Xd),
                                         ctypes.byref(opts), ctypes.byref(a), ctypes.byref(F))
        self._check(st, allow=(ML_E_STAGNATION,))
        return a.value, F.value, st

    def ml_select_coarse(self, g, k_total):
        out = self.torch.zeros(self.n, dtype=self.torch.int32, device=self.device)
        nout = ctypes.c_int64()
        self._check(load().ml_select_coarse(self.h, _ptr(g.contiguous()), int(k_total), _ptr(out),
                                            ctypes.byref(nout)))
        self.torch.cuda.synchronize(self.device)
        return out[: nout.value].clone()

    def ml_solve(self, opts=None):
        rep = SolveReport()
        st = load().ml_solve(self.h, ctypes.byref(opts or default_opts()), ctypes.byref(rep))
        self._check(st, allow=(ML_E_NOT_CONVERGED,))
        d = {f: getattr(rep, f) for f, _ in SolveReport._fields_ if f != "relax_per_level"}
        d["relax_per_level"] = list(rep.relax_per_level)
        return d

    CLASSES = ["margins", "gather_fine", "gather_coarse", "scatter_XAs", "gather_Hs", "inner_dir", "mpass", "apply",
               "outer_ls", "update", "select", "book", "api", "inner_fused"]

    def ml_profile(self, mask=0):
        return self._check(load().ml_profile(self.h, int(mask)))

    def ml_profile_read(self):
        ms = (ctypes.c_double * 16)()
        ps, nz, sg = ((ctypes.c_int64 * 16)() for _ in range(3))
        self._check(load().ml_profile_read(self.h, ms, ps, nz, sg))
        return {name: {"ms": ms[k], "passes": ps[k], "nnz": nz[k], "segs": sg[k]}
                for k, name in enumerate(self.CLASSES)}

    def ml_set_engine(self, flags):
        return self._check(load().ml_set_engine(self.h, int(flags)))

    HEAVY_INFO = ("built", "nh", "nnzh", "s_tiles", "g_chunks", "bands", "relaxations", "mode")

    def ml_heavy_info(self):
        v = (ctypes.c_int64 * 8)()
        self._check(load().ml_heavy_info(self.h, v))
        return dict(zip(self.HEAVY_INFO, (int(x) for x in v)))

    def ml_set_sm_share(self, blocks):
        return self._check(load().ml_set_sm_share(self.h, int(blocks)))

    def ml_inner_phases(self, reset=True):
        ns = (ctypes.c_uint64 * 16)()
        self._check(load().ml_inner_phases(self.h, ns, int(reset)))
        return [int(x) for x in ns]

    def ml_kernel_launches(self):
        return int(load().ml_kernel_launches(self.h))

    def trace(self):
        L = load()
        n = L.ml_trace(self.h, None, 0)
        rows = (TraceRow * max(n, 1))()
        L.ml_trace(self.h, ctypes.cast(rows, ctypes.c_void_p), n)
        return [{f: getattr(rows[i], f) for f, _ in TraceRow._fields_} for i in range(n)]
