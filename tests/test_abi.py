"""The C-ABI library builds, loads and exports every symbol include/ml.h declares (no GPU needed, no compute)."""
import ctypes
import os
import re

import pytest

import paper_1607_00315_b200 as ml

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ml.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ml_[a-z_]+)\s*\(", txt)))


def test_build_and_exports():
    so = ml.build()
    lib = ctypes.CDLL(so)
    syms = header_symbols()
    assert "ml_solve" in syms and "ml_create" in syms and "ml_select_coarse" in syms
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(ml.EXPORTS)


def test_sm100a_code_in_library():
    import subprocess
    so = ml.build()
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_and_validation_host_only():
    L = ml.load()
    b1 = L.ml_workspace_bytes(200, 1000, 200000)
    b2 = L.ml_workspace_bytes(2000, 20000, 40000000)
    assert 0 < b1 < b2
    assert L.ml_workspace_bytes(0, 10, 0) == 0
    # invalid arguments are rejected before any device work
    d = ml.MLData(0, 5, 0, None, None, None, None, None, None, None)
    h = ctypes.c_void_p()
    assert L.ml_create(ctypes.byref(d), 1.0, None, None, 0, ctypes.byref(h)) == ml.ML_E_INVAL
    d = ml.MLData(3, 5, 4, 16, 16, 16, 16, 16, 16, 16)   # (fake, never dereferenced: checks come first)
    assert L.ml_create(ctypes.byref(d), -1.0, None, None, 0, ctypes.byref(h)) == ml.ML_E_INVAL
    assert L.ml_create(ctypes.byref(d), float("nan"), None, None, 0, ctypes.byref(h)) == ml.ML_E_INVAL
    assert L.ml_create(ctypes.byref(d), 1.0, None, None, 10, ctypes.byref(h)) == ml.ML_E_WORKSPACE
    # include/ml.h alignment: a value / index array not 16-byte aligned is rejected before any device work
    for k in range(4):
        p = [16] * 7
        p[[1, 2, 4, 5][k]] = 20
        d2 = ml.MLData(3, 5, 4, *p)
        assert L.ml_create(ctypes.byref(d2), 1.0, None, None, 10, ctypes.byref(h)) == ml.ML_E_INVAL
    assert L.ml_status_str(ml.ML_E_NONFINITE) == b"non-finite input"
    # index-free dense X (include/ml.h): NULL CSC pointers / rows are accepted only with nnz = m n, m <= 8192, no CSR
    for (mm, nn, nz, csr) in ((3, 5, 14, 0), (9000, 2, 18000, 0), (3, 5, 15, 16)):
        d3 = ml.MLData(mm, nn, nz, csr, csr, csr, None, None, 16, 16)
        assert L.ml_create(ctypes.byref(d3), 1.0, None, None, 10, ctypes.byref(h)) == ml.ML_E_INVAL
    assert L.ml_status_str(ml.ML_E_STAGNATION) == b"line search stagnation"
    o = ml.default_opts()
    assert o.tol_kkt == 1e-6 and o.K_fine == 2 and o.K_mid == 3 and o.K_coarse == 5 and o.inner_cg == 2 and o.pcd_snap == 1


def test_defaults_match_oracle():
    """Both sides run the same algorithm with the same frozen defaults."""
    import oracle
    a, b = ml.default_opts(), oracle.default_opts()
    for f, _ in ml.SolveOpts._fields_:
        assert getattr(a, f) == getattr(b, f), f


def test_product_path_does_not_import_oracle():
    """The CUDA path never imports, links or executes the oracle."""
    pkg = os.path.join(ROOT, "paper_1607_00315_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace("no cpu fallback", ""), f
