"""CUDA path (through the C ABI) vs the CPU oracle on identical seeded inputs.  Marked gpu.

Tolerances: per-kernel outputs F, g, h, Hv, z, r, D: relative L2 <= 1e-9; selection: exact
set equality given the oracle's gradient bits; line search: identical alpha unless the Armijo decision is a
near-tie; solve: F relative <= 1e-6 with both runs at kappa <= 1e-6, supports equal outside the band
||g_j| - lambda| < 1e-4 (BASELINE.json north_star).
"""
import numpy as np
import pytest

import mlgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1607_00315_b200 as ml  # noqa: E402

ml.build()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def absX(ds):
    """|X| as a scipy CSC (for the elementwise tolerances: each output's sum of absolute terms)."""
    import scipy.sparse as sp
    return sp.csc_matrix((np.abs(ds.csc_val.astype(np.float64)), ds.csc_row, ds.csc_colptr), shape=(ds.m, ds.n))


def elem(a, b, scale, tol=1e-9, what=""):
    """Elementwise: |a_k - b_k| <= tol * scale_k, scale_k = the sum of the absolute values of the terms of output k
    (a relative-L2 check alone lets a wrong light column hide under a few heavy ones)."""
    a, b, scale = (np.asarray(x, np.float64) for x in (a, b, scale))
    bad = np.abs(a - b) > tol * scale + 1e-300
    assert not bad.any(), (what, int(bad.sum()), np.flatnonzero(bad)[:5])


def dt(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0", dtype)


_CACHE = {}


def _full(cfg):
    """A full-size BASELINE config, generated once per test session (cfg 5: 23 s, 3.3 GB of host memory)."""
    key = f"full{cfg}"
    if key not in _CACHE:
        _CACHE[key] = mlgen.make(cfg)
    return _CACHE[key]


def _coo_dataset(m, n, per_row, seed, lam_factor):
    """A sparse design from coordinates (no dense m x n array): row i holds Poisson(per_row) distinct random columns
    (some rows stay empty), N(0,1) values, uniform labels; lambda = lam_factor * lambda_max."""
    rng = np.random.default_rng(seed)
    cnt = rng.poisson(per_row, m)
    rows = np.repeat(np.arange(m), cnt)
    cols = rng.integers(0, n, rows.size)
    key = np.unique(rows.astype(np.int64) * n + cols)          # sorted by (row, col), duplicates dropped
    rows, cols = (key // n).astype(np.int64), (key % n).astype(np.int64)
    vals = rng.standard_normal(rows.size).astype(np.float32)
    vals[vals == 0] = 1.0
    rowptr = np.zeros(m + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    corder = np.lexsort((rows, cols))
    colptr = np.zeros(n + 1, np.int64)
    np.add.at(colptr, cols + 1, 1)
    y = np.where(rng.random(m) < 0.5, 1, -1).astype(np.int8)
    g0 = np.zeros(n)
    np.add.at(g0, cols, vals.astype(np.float64) * y[rows])
    lam = lam_factor * 0.5 * np.max(np.abs(g0))
    return mlgen.Dataset(m=m, n=n, csr_rowptr=np.cumsum(rowptr).astype(np.int32), csr_col=cols.astype(np.int32),
                         csr_val=vals, csc_colptr=np.cumsum(colptr).astype(np.int32),
                         csc_row=rows[corder].astype(np.int32), csc_val=vals[corder], y=y, lam=float(lam),
                         name=f"coo{m}x{n}s{seed}")


def dataset(name):
    if name in _CACHE:
        return _CACHE[name]
    if name == "cfg1":
        ds = mlgen.make(1)
    elif name == "cfg2s":      # dense, correlated blocks; rows heavy (split path), columns light
        ds = mlgen.make(2, m=300, n=3000)
    elif name == "cfg2m":      # dense with heavy columns (> SPLIT)
        ds = mlgen.make(2, m=2500, n=600)
    elif name == "cfg3s":
        ds = mlgen.make(3, m=8000, n=16000)
    elif name == "cfg3":
        ds = mlgen.make(3)
    elif name == "cfg4s":
        ds = mlgen.make(4, m=20000, n=40000)
    elif name == "mid6k":      # 6000 rows: the small-m solver with 512-element column chunks (the 1024 rings do not fit)
        ds = mlgen.make(3, m=6000, n=12000)
    elif name == "sparse_edges":   # empty rows and columns, ragged
        ds = mlgen.random_sparse(777, 1301, 0.02, seed=5, empty_rows=9, empty_cols=40)
    elif name == "onehot":
        ds = mlgen.onehot(3000, 3)[0]
    elif name == "shortcols":   # large m, ~4 nonzeros per column (45 % of cfg 5's columns are this short): one thread
        # per column in the gather tiles, the finest gather in two passes, a look-back over > 32 groups
        ds = mlgen.make(5, m=12000, n=120000)   # (cfg 5's recipe: Zipf columns, mean length 10, many empty)
    elif name == "shortrows":   # large m, 1-7 nonzeros per row (some rows empty): one thread per row in the margins tiles
        ds = _coo_dataset(90000, 12000, 4, seed=12, lam_factor=0.05)
    elif name == "lasso2s":    # squared loss (Q29) on the small-m dense design
        ds = mlgen.lasso(mlgen.make(2, m=300, n=3000), 1, k=40, noise=0.5, lam_factor=0.1)
    elif name == "lasso4s":    # squared loss on the large-m (global m-vector) path
        ds = mlgen.lasso(mlgen.make(4, m=20000, n=40000), 2, k=200, noise=0.05, lam_factor=0.05)
    elif name == "lasso_mid6k":
        ds = mlgen.lasso(mlgen.make(3, m=6000, n=12000), 3, k=100, noise=0.05, lam_factor=0.05)
    elif name.startswith("tail"):   # X's last nonzeros past its last 16-byte boundary, in a short last column (the
        # chunk of that column starts after the staged part ends: its elements come from the global tail)
        r = int(name[4:])
        rng = np.random.default_rng(40 + r)
        X = rng.standard_normal((300, 40)).astype(np.float32)
        X[rng.random(X.shape) > 0.15] = 0.0
        X[:, -1] = 0.0
        k = max(1, r - 1)                        # the last column's nonzeros: it starts past the 16-byte boundary
        i = 0
        while (int(np.count_nonzero(X)) + k) % 4 != r:   # nnz = r mod 4
            X[i, 0] = 0.0 if X[i, 0] != 0.0 else 1.0
            i += 1
        X[:k, -1] = rng.uniform(0.5, 1.5, k)
        y = np.where(X @ rng.standard_normal(40) + 0.3 * rng.standard_normal(300) > 0, 1, -1).astype(np.int8)
        lmax = 0.5 * np.max(np.abs(X.astype(np.float64).T @ y))
        ds = mlgen.from_dense(X, y, 0.05 * lmax, name=name)
    elif name == "m1":
        ds = mlgen.from_dense(np.array([[0.5, -1.0, 2.0, 0.0, 1.5]], np.float32), np.array([1], np.int8), 0.1)
    elif name == "n1":
        rng = np.random.default_rng(1)
        ds = mlgen.from_dense(rng.uniform(0.1, 1, (57, 1)).astype(np.float32),
                              np.where(rng.random(57) < 0.7, 1, -1).astype(np.int8), 0.5)
    else:
        raise KeyError(name)
    _CACHE[name] = ds
    return ds


def random_w(n, kind, seed):
    rng = np.random.default_rng(seed)
    w = np.zeros(n)
    k = {"zero": 0, "ten": min(10, n), "pct": max(1, n // 100), "all": n}[kind]
    idx = rng.choice(n, k, replace=False)
    w[idx] = rng.normal(0, 0.1, k) * (3.0 if kind == "ten" else 1.0)
    return w


PER_KERNEL = ["cfg1", "cfg2s", "cfg2m", "cfg3s", "cfg4s", "sparse_edges", "onehot", "m1", "n1", "shortcols", "shortrows"]


@pytest.mark.parametrize("name", PER_KERNEL)
@pytest.mark.parametrize("wkind", ["zero", "ten", "pct", "all"])
def test_eval_f_grad_parity(name, wkind):
    """A1 + A2: F, g, h, z, r, D at the same w."""
    ds = dataset(name)
    w = random_w(ds.n, wkind, 17)
    o = oracle.Oracle(ds)
    o.set_w(w)
    F_o, g_o, h_o = o.eval_f_grad()
    z_o, r_o, D_o, _ = o.rows()
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    F_g, g_g, h_g = ctx.ml_eval_f_grad()
    z_g, r_g, D_g = (t.cpu().numpy() for t in ctx.ml_get_rows())
    assert abs(F_g - F_o) <= 1e-9 * abs(F_o)
    assert rel(g_g.cpu().numpy(), g_o) <= 1e-9
    assert rel(h_g.cpu().numpy(), h_o) <= 1e-9
    assert rel(z_g, z_o) <= 1e-9 and rel(r_g, r_o) <= 1e-9 and rel(D_g, D_o) <= 1e-9
    A = absX(ds)
    zs = A @ np.abs(w)
    elem(z_g, z_o, zs, what="z")
    elem(r_g, r_o, np.abs(r_o) + 0.25 * zs, what="r")     # |dr/dz| = D <= 1/4
    elem(D_g, D_o, np.abs(D_o) + 0.1 * zs, what="D")      # |dD/dz| <= 0.1
    elem(g_g.cpu().numpy(), g_o, A.T @ np.abs(r_o) + A.T @ (0.25 * zs), what="g")
    elem(h_g.cpu().numpy(), h_o, h_o + A.multiply(A).T @ (0.1 * zs), what="h")


def _lists(ds, seed):
    rng = np.random.default_rng(seed)
    lens = np.diff(ds.csc_colptr)
    heavy = int(np.argmax(lens))
    out = {"empty": np.zeros(0, np.int32), "single": np.array([ds.n // 2], np.int32),
           "heaviest": np.array([heavy], np.int32),
           "pct": np.sort(rng.choice(ds.n, max(1, ds.n // 100), replace=False)).astype(np.int32),
           "half": np.sort(rng.choice(ds.n, max(1, ds.n // 2), replace=False)).astype(np.int32)}
    return out


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg2m", "cfg3s", "sparse_edges", "shortcols", "shortrows"])
def test_restricted_gather_hessvec(name):
    """A2 / A5 restricted to lists C: empty, single, heaviest column, 1 %, half."""
    ds = dataset(name)
    w = random_w(ds.n, "pct", 3)
    o = oracle.Oracle(ds)
    o.set_w(w)
    o.eval_f_grad()
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    ctx.ml_eval_f_grad(want_g=False, want_h=False)
    rng = np.random.default_rng(8)
    A = absX(ds)
    _, r_o, D_o, _ = o.rows()
    zs = A @ np.abs(w)
    gs_all = A.T @ (np.abs(r_o) + 0.25 * zs)
    hs_all = A.multiply(A).T @ (D_o + 0.1 * zs)
    for key, C in _lists(ds, 4).items():
        if len(C) == 0:
            continue
        _, g_o, h_o = o.eval_f_grad(C)
        Fg, g_g, h_g = ctx.ml_eval_f_grad(dt(C, torch.int32))
        assert rel(g_g.cpu().numpy(), g_o) <= 1e-9, key
        assert rel(h_g.cpu().numpy(), h_o) <= 1e-9, key
        elem(g_g.cpu().numpy(), g_o, gs_all[C], what=("g", key))
        elem(h_g.cpu().numpy(), h_o, hs_all[C], what=("h", key))
        hd = ctx.ml_diag_hess(dt(C, torch.int32))
        assert rel(hd.cpu().numpy(), h_o) <= 1e-9, key
        elem(hd.cpu().numpy(), h_o, hs_all[C], what=("diag", key))
        v = rng.standard_normal(len(C))
        Hv_o = o.hessvec(C, v)
        Hv_g = ctx.ml_hessvec(dt(C, torch.int32), dt(v))
        assert rel(Hv_g.cpu().numpy(), Hv_o) <= 1e-9, key
        vfull = np.zeros(ds.n)
        vfull[C] = np.abs(v)
        AC = A[:, C]
        elem(Hv_g.cpu().numpy(), Hv_o, AC.T @ ((D_o + 0.1 * zs) * (A @ vfull)), what=("Hv", key))
    v = rng.standard_normal(ds.n)
    assert rel(ctx.ml_hessvec(None, dt(v)).cpu().numpy(), o.hessvec(None, v)) <= 1e-9


@pytest.mark.parametrize("name", ["cfg1", "cfg3s", "sparse_edges", "onehot"])
def test_select_coarse_exact(name):
    """A8: exact set equality given identical gradient bits (ties by index)."""
    ds = dataset(name)
    w = random_w(ds.n, "pct", 5)
    o = oracle.Oracle(ds)
    o.set_w(w)
    _, g, _ = o.eval_f_grad()
    g = g.copy()
    g[::7] = np.round(g[::7], 2)  # exact ties
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    nS = int(np.count_nonzero(w))
    for k in (0, nS, nS + 1, nS + 37, (ds.n + nS) // 2, ds.n, ds.n + 5):
        C_o = o.select_coarse(g, k)
        C_g = ctx.ml_select_coarse(dt(g), k).cpu().numpy()
        assert np.array_equal(C_g, C_o), (k, len(C_g), len(C_o))


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "sparse_edges"])
def test_shrink_linesearch_parity(name):
    """A7: PCD step (d = NULL) and a given long step; alpha and F_new (Eq. 4-5)."""
    ds = dataset(name)
    w = random_w(ds.n, "ten", 9)
    for mode in ("pcd", "given"):
        o = oracle.Oracle(ds)
        o.set_w(w)
        _, g, h = o.eval_f_grad()
        ctx = ml.Context(ds)
        ctx.ml_set_w(dt(w))
        ctx.ml_eval_f_grad(want_g=False, want_h=False)
        C = np.arange(ds.n, dtype=np.int32)
        if mode == "pcd":
            a_o, F_o, st_o = o.shrink_linesearch(C, g, h=h)
            a_g, F_g, st_g = ctx.ml_shrink_linesearch(dt(C, torch.int32), dt(g), h=dt(h))
        else:
            rng = np.random.default_rng(2)
            d = -np.sign(g) * np.abs(rng.normal(0, 2.0, ds.n))
            a_o, F_o, st_o = o.shrink_linesearch(C, g, d=d)
            a_g, F_g, st_g = ctx.ml_shrink_linesearch(dt(C, torch.int32), dt(g), d=dt(d))
        assert st_o == st_g
        assert a_o == a_g, (mode, a_o, a_g)
        assert abs(F_g - F_o) <= 1e-9 * abs(F_o)
        assert rel(ctx.ml_get_w().cpu().numpy(), o.get_w()) <= 1e-12


def _support_check(ds, w_g, w_o, g_o):
    band = np.abs(np.abs(g_o) - ds.lam) < 1e-4
    sg, so = w_g != 0, w_o != 0
    assert np.all((sg == so) | band), int(np.sum((sg != so) & ~band))


@pytest.mark.parametrize("name,opts", [("cfg1", {}), ("cfg2s", {}), ("cfg3s", {}), ("sparse_edges", {}),
                                       ("onehot", {}), ("n1", {}), ("m1", {}),
                                       ("cfg3s", {"multilevel": 0, "K_fine": 10}),
                                       ("cfg1", {"inner_cg": 0, "K_mid": 2, "K_coarse": 5}),
                                       ("cfg2s", {"continuation": 1}), ("cfg3s", {"continuation": 1}),
                                       ("mid6k", {"continuation": 1}), ("onehot", {"continuation": 1}),
                                       ("lasso2s", {}), ("lasso4s", {}), ("lasso_mid6k", {}),
                                       ("lasso2s", {"continuation": 1}), ("lasso4s", {"multilevel": 0, "K_fine": 10}),
                                       ("tail3", {"multilevel": 0}), ("tail2", {"continuation": 1}),
                                       ("shortcols", {}), ("shortrows", {})])
def test_solve_parity(name, opts):
    """A9: ml_solve vs the oracle's solve (Algorithm 1 P:155-173 per P:798), both to kappa <= 1e-6."""
    ds = dataset(name)
    o = oracle.Oracle(ds)
    r_o = o.solve(oracle.default_opts(**opts))
    ctx = ml.Context(ds)
    r_g = ctx.ml_solve(ml.default_opts(**opts))
    assert r_o["status"] == 0 and r_g["status"] == 0, (r_o, r_g)
    assert r_g["kappa"] <= 1e-6 and r_o["kappa"] <= 1e-6
    assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
    w_o = o.get_w()
    _, g_o, _ = o.eval_f_grad()
    _support_check(ds, ctx.ml_get_w().cpu().numpy(), w_o, g_o)
    tr = ctx.trace()
    for row in tr:   # Lemma P:207-243
        assert row["F_after"] <= row["F_before"] * (1 + 1e-12) + 1e-12


def test_solve_onehot_closed_form():
    """GPU solve against the one-hot closed form with no oracle involved, n = 20000."""
    ds, a, p, q = mlgen.onehot(20000, 11)
    lam = ds.lam
    d = np.abs(p - q).astype(np.float64)
    act = lam < a * d / 2
    wref = np.zeros(ds.n)
    big, small = np.maximum(p, q).astype(np.float64), np.minimum(p, q).astype(np.float64)
    wref[act] = np.sign(p - q)[act] / a[act] * np.log((a[act] * big[act] - lam) / (a[act] * small[act] + lam))
    F = np.sum(p * np.logaddexp(0, -a * wref) + q * np.logaddexp(0, a * wref) + lam * np.abs(wref))
    ctx = ml.Context(ds)
    r = ctx.ml_solve(ml.default_opts(tol_kkt=1e-12))
    w = ctx.ml_get_w().cpu().numpy()
    assert r["status"] == 0
    assert set(np.nonzero(w)[0]) == set(np.nonzero(wref)[0])
    nz = wref != 0
    assert np.max(np.abs(w[nz] - wref[nz]) / np.abs(wref[nz])) <= 1e-8
    assert abs(r["F"] - F) <= 1e-12 * F


def test_lambda_max_zero_solution_gpu():
    ds = dataset("cfg1")
    ctx = ml.Context(ds, lam=ds.lambda_max * (1 + 1e-9))
    r = ctx.ml_solve()
    assert r["status"] == 0 and r["cycles"] == 0 and r["nnz_w"] == 0


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_solve_parity_full_configs(name):
    """Solve parity at BASELINE configs 2, 3 and 4 (full size; cfg 4's oracle solve takes ~20-40 s on one core)."""
    ds = _full(int(name[-1]))
    o = oracle.Oracle(ds)
    r_o = o.solve()
    ctx = ml.Context(ds)
    r_g = ctx.ml_solve()
    assert r_o["status"] == 0 and r_g["status"] == 0
    assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
    w_o = o.get_w()
    _, g_o, _ = o.eval_f_grad()
    _support_check(ds, ctx.ml_get_w().cpu().numpy(), w_o, g_o)


@pytest.mark.parametrize("name,opts", [("cfg2s", {"inner_cg": 1, "pcd_snap": 0}), ("cfg1", {"inner_cg": 1, "pcd_snap": 0}),
                                       ("onehot", {"inner_cg": 1, "pcd_snap": 0}), ("cfg2s", {"pcd_snap": 0}),
                                       ("cfg4s", {"pcd_snap": 0}), ("cfg4s", {}), ("cfg4s", {"inner_cg": 0}),
                                       ("mid6k", {}), ("mid6k", {"inner_cg": 1, "pcd_snap": 0})])
def test_solve_parity_inner_variants(name, opts):
    """The other inner solvers (DESIGN Q9b, Q27): plain PCD-CG, PCD-CG with a shrinkage step after every kink without
    the snap path, plain PCD with the snap path; small-m (persistent) and large-m (generic) relaxation paths."""
    test_solve_parity(name, opts)


@pytest.mark.parametrize("name,opts", [("cfg2s", {}), ("cfg4s", {}), ("onehot", {}), ("mid6k", {}), ("cfg2s", {"inner_cg": 0}),
                                       ("cfg4s", {"inner_cg": 0}), ("cfg4s", {"inner_cg": 1, "pcd_snap": 0}),
                                       ("cfg2s", {"continuation": 1}), ("cfg4s", {"continuation": 1}),
                                       ("lasso2s", {}), ("lasso4s", {}),
                                       ("tail1", {}), ("tail2", {}), ("tail3", {}), ("tail3", {"inner_cg": 0})])
def test_trace_parity(name, opts):
    """Relaxation by relaxation (Algorithm 1, DESIGN S1-S18/R1-R18): level, |A|, outcome, inner iterations and
    F after each of the first relaxations agree with the oracle's trace (decisions identical while rounding
    differences stay below the decision margins)."""
    ds = dataset(name)
    o = oracle.Oracle(ds)
    o.solve(oracle.default_opts(max_cycles=3, **opts))
    ctx = ml.Context(ds)
    ctx.ml_solve(ml.default_opts(max_cycles=3, **opts))
    to, tg = o.trace(), ctx.trace()
    n = min(len(to), len(tg), 12)
    assert n >= 5
    for k in range(n):
        a, b = to[k], tg[k]
        for f in ("level", "nA", "outcome", "inner_iters"):
            assert a[f] == b[f], (k, f, a, b)
        assert abs(a["F_after"] - b["F_after"]) <= 1e-9 * abs(a["F_after"]), (k, a, b)


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_sampled_eval_parity(cfg):
    """BASELINE configs 4 and 5 at full size: F, g_C, h_C on a sampled column list (random + the 20 heaviest
    columns), in the launch configuration the bench uses, against the oracle's one-by-one evaluation."""
    ds = _full(cfg)
    rng = np.random.default_rng(cfg)
    lens = np.diff(ds.csc_colptr)
    C = np.unique(np.r_[rng.choice(ds.n, 2000, replace=False), np.argsort(lens)[-20:]]).astype(np.int32)
    w = np.zeros(ds.n)
    idx = rng.choice(ds.n, 5000, replace=False)
    w[idx] = rng.normal(0, 0.2, len(idx))
    w[np.argsort(lens)[-5:]] = 0.1   # heavy columns in the support
    o = oracle.Oracle(ds)
    o.set_w(w)
    F_o, g_o, h_o = o.eval_f_grad(C)
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    F_g, g_g, h_g = ctx.ml_eval_f_grad(dt(C, torch.int32))
    assert abs(F_g - F_o) <= 1e-9 * abs(F_o)
    assert rel(g_g.cpu().numpy(), g_o) <= 1e-9
    assert rel(h_g.cpu().numpy(), h_o) <= 1e-9
    v = rng.standard_normal(len(C))
    Hv_g, Hv_o = ctx.ml_hessvec(dt(C, torch.int32), dt(v)).cpu().numpy(), o.hessvec(C, v)
    assert rel(Hv_g, Hv_o) <= 1e-9
    # elementwise, each sampled column against the sum of its absolute terms
    A = absX(ds)
    _, r_o, D_o, _ = o.rows()
    zs = A @ np.abs(w)
    AC = A[:, C]
    elem(g_g.cpu().numpy(), g_o, AC.T @ (np.abs(r_o) + 0.25 * zs), what="g")
    elem(h_g.cpu().numpy(), h_o, AC.multiply(AC).T @ (D_o + 0.1 * zs), what="h")
    vfull = np.zeros(ds.n)
    vfull[C] = np.abs(v)
    elem(Hv_g, Hv_o, AC.T @ ((D_o + 0.1 * zs) * (A @ vfull)), what="Hv")


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_solve_kkt_by_oracle(cfg):
    """Full-size GPU solve; the oracle re-evaluates the gradient at the GPU's w and checks the KKT conditions
    (|g_j| <= lam(1+1e-6) off the support, |g_j + lam sign w_j| <= 1e-6 lam on it) and F."""
    ds = _full(cfg)
    ctx = ml.Context(ds)
    r = ctx.ml_solve()
    assert r["status"] == 0 and r["kappa"] <= 1e-6, r
    w = ctx.ml_get_w().cpu().numpy()
    del ctx
    o = oracle.Oracle(ds)
    o.set_w(w)
    F_o, g_o, _ = o.eval_f_grad()
    S = w != 0
    lam = ds.lam
    assert np.max(np.abs(g_o[~S])) <= lam * (1 + 1e-6)
    assert np.max(np.abs(g_o[S] + lam * np.sign(w[S]))) <= 1e-6 * lam
    assert abs(F_o - r["F"]) <= 1e-9 * abs(F_o)


@pytest.mark.parametrize("name", ["cfg2s", "cfg1", "sparse_edges", "mid6k"])
def test_small_m_solve_bitwise_reproducible(name):
    """The small-m persistent path reduces in fixed orders only (slot-major partials, block-ordered row sums,
    position-ordered compaction): two solves from w = 0 return bitwise identical w and F (DESIGN 8.2, Determinism)."""
    ds = dataset(name)
    ctx = ml.Context(ds)
    r1 = ctx.ml_solve()
    w1 = ctx.ml_get_w().cpu().numpy().copy()
    ctx.ml_set_w(torch.zeros(ds.n, dtype=torch.float64, device="cuda"))
    r2 = ctx.ml_solve()
    w2 = ctx.ml_get_w().cpu().numpy()
    assert r1["status"] == 0 and r2["status"] == 0
    assert r1["F"] == r2["F"] and r1["cycles"] == r2["cycles"]
    assert np.array_equal(w1, w2)


def test_create_rejects_malformed_index():
    """ABI error behaviour (include/ml.h): unsorted rows inside a CSC column and out-of-range CSR columns are rejected
    by ml_create with ML_E_INVAL (the column passes rely on distinct rows within a column)."""
    import dataclasses
    good = mlgen.from_dense(np.eye(4, 3, dtype=np.float32) + 1.0, np.array([1, -1, 1, -1], np.int8), 0.1)
    ml.Context(good)   # well formed: accepted
    row = good.csc_row.copy()
    row[0], row[1] = row[1], row[0]   # column 0's rows out of order
    col = good.csr_col.copy()
    col[-1] = good.n                  # a CSR column index out of range
    dup = good.csc_row.copy()
    dup[1] = dup[0]                   # a repeated row inside column 0
    last = good.csc_row.copy()
    last[3], last[2] = last[2], last[3]   # the descent at a column's last element (next to a legal one at its end)
    for bad in (dataclasses.replace(good, csc_row=row), dataclasses.replace(good, csr_col=col),
                dataclasses.replace(good, csc_row=dup), dataclasses.replace(good, csc_row=last)):
        with pytest.raises(ml.MLError) as e:
            ml.Context(bad)
        assert "status 1" in str(e.value), str(e.value)
    # empty rows and columns (equal consecutive pointers) are well formed
    a = np.zeros((5, 4), np.float32)
    a[0, 1], a[3, 1], a[3, 3] = 1.0, 2.0, 3.0
    ml.Context(mlgen.from_dense(a, np.array([1, -1, 1, -1, 1], np.int8), 0.1))


def test_lasso_orthogonal_closed_form_gpu():
    """Squared loss (Q29) on an orthogonal (one-hot) design, n = 20000, no oracle involved:
    w*_j = soft(x_j^T b, lam) / ||x_j||^2."""
    base = mlgen.onehot(20000, 11)[0]
    ds = mlgen.lasso(base, 6, k=2000, noise=0.5, lam_factor=0.1)
    cp, ri, rv = base.csc_colptr, base.csc_row, base.csc_val.astype(np.float64)
    xtb = np.add.reduceat(rv * ds.b[ri], cp[:-1])
    nrm = np.add.reduceat(rv * rv, cp[:-1])
    wref = np.sign(xtb) * np.maximum(np.abs(xtb) - ds.lam, 0.0) / nrm
    ctx = ml.Context(ds)
    r = ctx.ml_solve(ml.default_opts(tol_kkt=1e-12))
    w = ctx.ml_get_w().cpu().numpy()
    assert r["status"] == 0
    assert set(np.nonzero(w)[0]) == set(np.nonzero(wref)[0])
    nz = wref != 0
    assert np.max(np.abs(w[nz] - wref[nz]) / np.abs(wref[nz])) <= 1e-10


def test_columns_only_context():
    """include/ml.h: the CSR may be NULL for m <= 8192 (every pass reads X by columns there); the solve is bitwise
    the one with both layouts.  Above that size ml_create rejects a missing CSR with ML_E_INVAL."""
    ds = dataset("cfg2s")
    a = ml.Context(ds)
    ra = a.ml_solve()
    b = ml.Context(ds, csr=False)
    rb = b.ml_solve()
    assert ra["F"] == rb["F"] and ra["cycles"] == rb["cycles"]
    assert np.array_equal(a.ml_get_w().cpu().numpy(), b.ml_get_w().cpu().numpy())
    F1, g1, h1 = a.ml_eval_f_grad()
    F2, g2, h2 = b.ml_eval_f_grad()
    assert F1 == F2 and torch.equal(g1, g2) and torch.equal(h1, h2)
    with pytest.raises(ml.MLError) as e:
        ml.Context(dataset("cfg4s"), csr=False)
    assert "status 1" in str(e.value)


def test_replicas_side_by_side():
    """ml_set_sm_share (batched replicas): two contexts on their own streams and host threads, each
    with half of the SMs, solve concurrently and both match the oracle; a share too small for m is rejected."""
    import threading
    ds = dataset("cfg2s")
    r_o = oracle.Oracle(ds).solve()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    streams = [torch.cuda.Stream() for _ in range(2)]
    ctxs = [ml.Context(ds, stream=s) for s in streams]
    for c in ctxs:
        c.ml_set_sm_share(sms // 2)
    out = [None, None]

    def work(k):
        out[k] = [ctxs[k].ml_solve() for _ in range(3)]

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for rs in out:
        for r in rs:
            assert r["status"] == 0 and r["kappa"] <= 1e-6
            assert abs(r["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
    big = ml.Context(dataset("mid6k"))   # m = 6000 on the small-m path: needs >= 94 blocks (64 rows each)
    with pytest.raises(ml.MLError):
        big.ml_set_sm_share(16)
    big.ml_set_sm_share(0)   # the whole GPU again


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_random_designs_parity(seed):
    """Randomised solve parity (tools/random_parity.py in small): random shapes on both solver paths, densities,
    empty rows / columns, logistic or squared loss, option sets; GPU and oracle both converge to the same F."""
    rng = np.random.default_rng(seed)
    pool = [{}, {"inner_cg": 1, "pcd_snap": 0}, {"multilevel": 0}, {"continuation": 1}]
    for _ in range(4):
        m = int(rng.choice([37, 300, 777, 2000, 9000]))
        n = int(rng.choice([13, 150, 1301]))
        base = mlgen.random_sparse(m, n, float(rng.choice([0.01, 0.05, 0.3])), seed=int(rng.integers(1 << 30)),
                                   lam_factor=float(rng.choice([0.05, 0.1, 0.3])),
                                   empty_rows=int(rng.integers(0, min(5, m // 2) + 1)),
                                   empty_cols=int(rng.integers(0, min(20, n // 2) + 1)))
        ds = mlgen.lasso(base, int(rng.integers(1 << 30)), k=5) if rng.random() < 0.3 else base
        opts = pool[int(rng.integers(len(pool)))]
        r_o = oracle.Oracle(ds).solve(oracle.default_opts(**opts))
        r_g = ml.Context(ds).ml_solve(ml.default_opts(**opts))
        assert r_o["status"] == r_g["status"] == 0, (m, n, opts, r_o["status"], r_g["status"])
        assert r_g["kappa"] <= 1e-6
        assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"]), (m, n, opts, r_g["F"], r_o["F"])


def test_solve_with_stale_workspace():
    """ml_create must not depend on the workspace's previous contents.  The workspace is pre-filled with words that
    look like look-back statuses of epochs 0..63 (flag 1, count 5) before ml_create; the large-m solve (64-column
    coarse tiles) must still match the oracle."""
    # m > 8192 (large-m path) and coarse sets wider than m / 4 columns: their 64-column tiles reach past the status
    # words of the 256-row tiles
    ds = mlgen.random_sparse(9000, 6000, 0.1, seed=3, lam_factor=0.02)
    r_o = oracle.Oracle(ds).solve()
    ctx = ml.Context(ds, ws_fill="epochs")
    r_g = ctx.ml_solve()
    assert r_g["status"] == 0 and r_g["kappa"] <= 1e-6
    assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])


def _ls_pair(ds, w, mode, seed=2):
    """One ml_shrink_linesearch on both sides from the same w: PCD step (d = NULL), a given long step, or an ascent
    direction (every Armijo trial fails: ML_E_STAGNATION, iterate unchanged)."""
    o = oracle.Oracle(ds)
    o.set_w(w)
    _, g, h = o.eval_f_grad()
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    ctx.ml_eval_f_grad(want_g=False, want_h=False)
    C = np.arange(ds.n, dtype=np.int32)
    rng = np.random.default_rng(seed)
    if mode == "pcd":
        res_o = o.shrink_linesearch(C, g, h=h)
        res_g = ctx.ml_shrink_linesearch(dt(C, torch.int32), dt(g), h=dt(h))
    else:
        d = np.abs(rng.normal(0, 2.0, ds.n))
        if mode == "ascent":   # uphill on both the smooth part and the l1 term: Delta > 0, no alpha passes
            d = d * np.sign(g)
            d[w != 0] = np.abs(d[w != 0]) * np.sign(w[w != 0])
            d[(w == 0) & (g == 0)] = 0.0
        else:                  # a long step along minus the min-norm subgradient: a descent direction
            v = np.where(w != 0, g + ds.lam * np.sign(w), np.sign(g) * np.maximum(np.abs(g) - ds.lam, 0.0))
            d = -d * v
        res_o = o.shrink_linesearch(C, g, d=d)
        res_g = ctx.ml_shrink_linesearch(dt(C, torch.int32), dt(g), d=dt(d))
    return o, ctx, res_o, res_g


@pytest.mark.parametrize("name", ["cfg4s", "cfg4"])
@pytest.mark.parametrize("mode", ["pcd", "given", "ascent"])
def test_shrink_linesearch_parity_large_m(name, mode):
    """A7 on the large-m API path (m > 8192: the fp64 X_C d scatter and k_outer_ls over all rows), including a forced
    stagnation (Eq. 4; include/ml.h: alpha = 0, ML_E_STAGNATION, iterate unchanged)."""
    ds = _full(4) if name == "cfg4" else dataset(name)
    w = random_w(ds.n, "pct", 9)
    o, ctx, (a_o, F_o, st_o), (a_g, F_g, st_g) = _ls_pair(ds, w, mode)
    assert st_o == st_g
    if mode == "ascent":
        assert st_g == ml.ML_E_STAGNATION and a_g == 0.0 and a_o == 0.0
        assert np.array_equal(ctx.ml_get_w().cpu().numpy(), w)
    else:
        assert st_g == 0 and a_o == a_g, (a_o, a_g)
    assert abs(F_g - F_o) <= 1e-9 * abs(F_o)
    assert rel(ctx.ml_get_w().cpu().numpy(), o.get_w()) <= 1e-12


@pytest.mark.parametrize("cfg", [4, 5])
def test_select_coarse_exact_full_size(cfg):
    """A8 at BASELINE configs 4 and 5 (n = 1e6 / 2e7 candidates): exact set equality with the oracle given the
    oracle's gradient bits (ties by ascending index, DESIGN Q14), at the level sizes a solve uses."""
    ds = _full(cfg)
    rng = np.random.default_rng(cfg)
    w = np.zeros(ds.n)
    idx = rng.choice(ds.n, 3000, replace=False)
    w[idx] = rng.normal(0, 0.2, len(idx))
    o = oracle.Oracle(ds)
    o.set_w(w)
    _, g, _ = o.eval_f_grad()
    g = g.copy()
    g[::5] = np.round(g[::5], 3)   # exact ties
    ctx = ml.Context(ds)
    ctx.ml_set_w(dt(w))
    nS = int(np.count_nonzero(w))
    gd = dt(g)
    for k in (nS, nS + 1, nS + 4321, 2 * nS + 100000, (ds.n + nS) // 2):
        C_o = o.select_coarse(g, k)
        C_g = ctx.ml_select_coarse(gd, k).cpu().numpy()
        assert np.array_equal(C_g, C_o), (k, len(C_g), len(C_o))


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_solve_vs_oracle_golden(cfg):
    """Full-size solve at BASELINE configs 4 and 5 against the oracle's own solution, committed under tests/golden/
    by tools/make_golden.py (which calls only oracle/): F within 1e-6 relative, both kappa <= 1e-6, supports equal
    outside the band ||g_j| - lambda| < 1e-4 (BASELINE.json north_star), and w on the common support close.  cfg 5 runs
    the default heavy-column path (its X_A s from the row-major copy), cfg 4 the column units only."""
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", f"cfg{cfg}_solution.npz"))
    meta = json.loads(str(z["meta"]))
    ds = _full(cfg)
    assert (meta["m"], meta["n"], meta["nnz"]) == (ds.m, ds.n, ds.nnz) and meta["lam"] == ds.lam
    ctx = ml.Context(ds)
    r = ctx.ml_solve()
    info = ctx.ml_heavy_info()   # cfg 5 takes the heavy-column path by default (include/ml.h, ml_set_engine)
    assert (info["built"] == 1 and info["relaxations"] > 0) if cfg == 5 else info["relaxations"] == 0, info
    assert r["status"] == 0 and r["kappa"] <= 1e-6 and meta["kappa"] <= 1e-6
    assert abs(r["F"] - meta["F"]) <= 1e-6 * abs(meta["F"]), (r["F"], meta["F"])
    w = ctx.ml_get_w().cpu().numpy()
    sg = np.flatnonzero(w)
    so = z["supp"].astype(np.int64)
    band = set(z["band"].tolist())
    diff = set(sg.tolist()) ^ set(so.tolist())
    outside = [j for j in diff if j not in band]
    assert not outside, outside[:10]
    common = np.intersect1d(sg, so)
    wo = np.zeros(ds.n)
    wo[so] = z["w_supp"]
    assert np.linalg.norm(w[common] - wo[common]) <= 1e-6 * np.linalg.norm(wo[common])   # (oracle variants: 2e-10)


# ----------------------------------------------------------------------------- boundary error behaviour
def test_nonfinite_inputs_rejected():
    """include/ml.h ML_E_NONFINITE (SPEC S:24 'finite entries only'): NaN / Inf among X's values (CSC or CSR) or the
    LASSO targets -> ml_create fails; a NaN in ml_set_w's vector -> ML_E_NONFINITE with w unchanged."""
    import dataclasses
    good = mlgen.from_dense(np.eye(4, 3, dtype=np.float32) + 1.0, np.array([1, -1, 1, -1], np.int8), 0.1)
    for field, val in (("csc_val", np.nan), ("csc_val", np.inf), ("csr_val", -np.inf)):
        a = getattr(good, field).copy()
        a[2] = val
        with pytest.raises(ml.MLError) as e:
            ml.Context(dataclasses.replace(good, **{field: a}))
        assert e.value.status == ml.ML_E_NONFINITE, str(e.value)
    las = mlgen.lasso(mlgen.make(1), 1, k=5)
    b = las.b.copy()
    b[7] = np.nan
    with pytest.raises(ml.MLError) as e:
        ml.Context(dataclasses.replace(las, b=b))
    assert e.value.status == ml.ML_E_NONFINITE
    ctx = ml.Context(dataset("cfg1"))
    w0 = random_w(ctx.n, "ten", 1)
    ctx.ml_set_w(dt(w0))
    bad = w0.copy()
    bad[3] = np.nan
    with pytest.raises(ml.MLError) as e:
        ctx.ml_set_w(dt(bad))
    assert e.value.status == ml.ML_E_NONFINITE
    assert np.array_equal(ctx.ml_get_w().cpu().numpy(), w0)
    ctx.ml_set_w(dt(w0))   # the context stays usable
    F, _, _ = ctx.ml_eval_f_grad(want_g=False, want_h=False)
    assert np.isfinite(F)


def test_bad_index_list_rejected():
    """include/ml.h: C must be strictly ascending in [0, n); every API entry taking C checks it on the device and
    returns ML_E_INVAL (unsorted, duplicate, out of range, negative), then keeps working on a good list."""
    ds = dataset("cfg3s")
    ctx = ml.Context(ds)
    good = np.array([3, 17, 400, ds.n - 1], np.int32)
    bads = [np.array([17, 3, 400], np.int32), np.array([3, 3, 400], np.int32), np.array([3, ds.n], np.int32),
            np.array([-1, 3], np.int32)]
    for C in bads:
        Ct = dt(C, torch.int32)
        v = dt(np.ones(len(C)))
        for call in (lambda: ctx.ml_eval_f_grad(Ct), lambda: ctx.ml_diag_hess(Ct), lambda: ctx.ml_hessvec(Ct, v),
                     lambda: ctx.ml_shrink_linesearch(Ct, v, h=v)):
            with pytest.raises(ml.MLError) as e:
                call()
            assert e.value.status == ml.ML_E_INVAL, (C, str(e.value))
    o = oracle.Oracle(ds)
    o.eval_f_grad()
    _, g_o, h_o = o.eval_f_grad(good)
    _, g_g, h_g = ctx.ml_eval_f_grad(dt(good, torch.int32))
    assert rel(g_g.cpu().numpy(), g_o) <= 1e-9 and rel(h_g.cpu().numpy(), h_o) <= 1e-9


def test_misaligned_arrays_rejected():
    """include/ml.h alignment: X's index / value arrays 16-byte aligned (16-byte vector loads, TMA bulk copies);
    an array starting 4 bytes into an allocation is rejected with ML_E_INVAL instead of faulting the context."""
    import ctypes
    ds = dataset("cfg1")
    L = ml.load()
    dev = "cuda:0"
    arrs = {k: torch.from_numpy(getattr(ds, k)).to(dev) for k in ("csr_rowptr", "csr_col", "csr_val", "csc_colptr",
                                                                    "csc_row", "csc_val", "y")}
    shifted = torch.zeros(ds.nnz + 4, dtype=torch.float32, device=dev)
    shifted[1:1 + ds.nnz] = arrs["csc_val"]
    ws = torch.empty(int(L.ml_workspace_bytes(ds.m, ds.n, ds.nnz)) + 512, dtype=torch.uint8, device=dev)
    for bad in ("csc_val",):
        ptrs = {k: v.data_ptr() for k, v in arrs.items()}
        ptrs[bad] = shifted.data_ptr() + 4
        data = ml.MLData(ds.m, ds.n, ds.nnz, ptrs["csr_rowptr"], ptrs["csr_col"], ptrs["csr_val"], ptrs["csc_colptr"],
                         ptrs["csc_row"], ptrs["csc_val"], ptrs["y"])
        h = ctypes.c_void_p()
        st = L.ml_create(ctypes.byref(data), ds.lam, None, ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.byref(h))
        assert st == ml.ML_E_INVAL
    torch.cuda.synchronize()
    ml.Context(ds).ml_solve()   # the process's CUDA context is intact


@pytest.mark.parametrize("name", ["cfg4s", "lasso4s", "sparse_big"])
def test_column_engines_agree(name):
    """The large-m engines (ml_set_engine: merge-path or per-column gathers; static or dynamic unit schedules in the
    inner solver) agree inside the solve: every combination matches the oracle, with identical relaxation traces
    (levels, |A|, outcomes)."""
    ds = mlgen.random_sparse(12000, 9000, 0.01, seed=7, lam_factor=0.05, empty_rows=20, empty_cols=300) \
        if name == "sparse_big" else dataset(name)
    r_o = oracle.Oracle(ds).solve()
    res = []
    for eng in (1, 0, 8):   # bit 0: merge-path gathers; bit 3: dynamic unit claims (ml_set_engine)
        ctx = ml.Context(ds)
        ctx.ml_set_engine(eng)
        r = ctx.ml_solve()
        assert r["status"] == 0 and r["kappa"] <= 1e-6
        assert abs(r["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
        res.append([(t["level"], t["nA"], t["outcome"]) for t in ctx.trace()])
    assert res[0] == res[1]


def test_merge_path_gather_bitwise_reproducible():
    """The merge-path pass sums in a fixed order (threads, then tiles): two solves on cfg4s give identical bits."""
    ds = dataset("cfg4s")
    ctx = ml.Context(ds)
    ctx.ml_set_engine(1)
    r1 = ctx.ml_solve()
    ctx.ml_set_w(torch.zeros(ds.n, dtype=torch.float64, device="cuda"))
    F1, g1, h1 = ctx.ml_eval_f_grad()
    ctx2 = ml.Context(ds)
    r2 = ctx2.ml_solve()
    assert r1["cycles"] == r2["cycles"] and r1["nnz_w"] == r2["nnz_w"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg2m", "n1"])
def test_dense_index_free_bitwise(name):
    """Index-free dense X (include/ml.h): values only, no CSR / CSC pointers / row indices on the
    device.  The arithmetic is the indexed path's, so every output is bitwise equal to it: F, g, h, Hv, the line search,
    the coarse selection and the whole solve (and therefore the oracle parity of the indexed path carries over)."""
    ds = dataset(name)
    assert ds.nnz == ds.m * ds.n
    a, b = ml.Context(ds), ml.Context(ds, dense=True)
    assert b.csc_row is None and b.csc_colptr is None and b.csr_col is None
    rng = np.random.default_rng(3)
    w = random_w(ds.n, "ten", 5)
    for c in (a, b):
        c.ml_set_w(dt(w))
    Fa, ga, ha = a.ml_eval_f_grad()
    Fb, gb, hb = b.ml_eval_f_grad()
    assert Fa == Fb and torch.equal(ga, gb) and torch.equal(ha, hb)
    C = np.sort(rng.choice(ds.n, max(1, ds.n // 3), replace=False)).astype(np.int32)
    v = dt(rng.standard_normal(len(C)))
    assert torch.equal(a.ml_hessvec(dt(C, torch.int32), v), b.ml_hessvec(dt(C, torch.int32), v))
    assert torch.equal(a.ml_diag_hess(dt(C, torch.int32)), b.ml_diag_hess(dt(C, torch.int32)))
    g = ga.clone()
    assert torch.equal(a.ml_select_coarse(g, ds.n // 2 + 3), b.ml_select_coarse(g, ds.n // 2 + 3))
    la = a.ml_shrink_linesearch(None, g, h=ha)
    lb = b.ml_shrink_linesearch(None, g, h=hb)
    assert la == lb and torch.equal(a.ml_get_w(), b.ml_get_w())
    ra = ml.Context(ds).ml_solve()
    cb = ml.Context(ds, dense=True)
    rb = cb.ml_solve()
    assert ra["F"] == rb["F"] and ra["cycles"] == rb["cycles"] and ra["relaxations"] == rb["relaxations"]
    r_o = oracle.Oracle(ds).solve()
    assert rb["status"] == 0 and abs(rb["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])


def test_dense_full_cfg2_solve():
    """BASELINE config 2 (2000 x 20000 dense) solved index-free: bitwise the indexed solve, and the oracle's F."""
    ds = _full(2)
    ra = ml.Context(ds).ml_solve()
    rb = ml.Context(ds, dense=True).ml_solve()
    assert ra["F"] == rb["F"] and ra["cycles"] == rb["cycles"]
    r_o = oracle.Oracle(ds).solve()
    assert abs(rb["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])


@pytest.mark.parametrize("name,flags", [("cfg4s", 0), ("cfg4s", 8), ("lasso4s", 0), ("cfg4s_cg", 8)])
def test_large_m_solve_bitwise_reproducible(name, flags):
    """The large-m path is bitwise reproducible: X_A s is reduced in 64-bit fixed point (integer
    addition does not depend on the order of the reductions), every other sum has a fixed order, and dynamic unit
    claims (flags 8) change only which warp sums a unit.  Two solves from w = 0 return identical w, F and traces."""
    ds = dataset("cfg4s" if name == "cfg4s_cg" else name)
    opts = {"inner_cg": 1, "pcd_snap": 0} if name == "cfg4s_cg" else {}
    out = []
    for rep in range(2):
        ctx = ml.Context(ds)
        ctx.ml_set_engine(flags)
        r = ctx.ml_solve(ml.default_opts(**opts))
        out.append((r["F"], r["cycles"], ctx.ml_get_w().cpu().numpy(), [(t["nA"], t["inner_iters"], t["F_after"])
                                                                       for t in ctx.trace()]))
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    assert np.array_equal(out[0][2], out[1][2])
    assert out[0][3] == out[1][3]


def _sparse_big():
    key = "sparse_big"
    if key not in _CACHE:
        _CACHE[key] = mlgen.random_sparse(12000, 9000, 0.01, seed=7, lam_factor=0.05, empty_rows=20, empty_cols=300)
    return _CACHE[key]


@pytest.mark.parametrize("name,opts", [("cfg4s", {}), ("cfg4s", {"inner_cg": 0}), ("cfg4s", {"inner_cg": 1, "pcd_snap": 0}),
                                       ("lasso4s", {}), ("sparse_big", {}), ("cfg4s", {"continuation": 1})])
def test_heavy_path_parity(name, opts):
    """The large-m heavy-column path (ml_heavy.cuh: X_A s of the longest columns from their row-major copy without
    atomics, DESIGN 8.2) forced in every relaxation (ml_set_engine bit 4) against the oracle: the same
    relaxation decisions (level, |A|, outcome, inner iterations) and F after each of the first relaxations to 1e-9,
    the final F to 1e-6 and the support outside the band."""
    ds = _sparse_big() if name == "sparse_big" else dataset(name)
    o = oracle.Oracle(ds)
    r_o = o.solve(oracle.default_opts(**opts))
    ctx = ml.Context(ds)
    ctx.ml_set_engine(16)
    r_g = ctx.ml_solve(ml.default_opts(**opts))
    info = ctx.ml_heavy_info()
    assert info["built"] == 1 and info["nh"] > 0 and info["relaxations"] > 0, info
    assert r_o["status"] == 0 and r_g["status"] == 0, (r_o, r_g)
    assert r_g["kappa"] <= 1e-6
    assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
    w_o = o.get_w()
    _, g_o, _ = o.eval_f_grad()
    _support_check(ds, ctx.ml_get_w().cpu().numpy(), w_o, g_o)
    to, tg = o.trace(), ctx.trace()
    n = min(len(to), len(tg), 12)
    assert n >= 5
    for k in range(n):
        a, b = to[k], tg[k]
        for f in ("level", "nA", "outcome"):
            assert a[f] == b[f], (k, f, a, b)
        # a one-column inner solve is exact after one step; whether a second, rounding-sized step is taken depends on
        # the summation order (both are correct), so the count is compared above that size only
        assert a["inner_iters"] == b["inner_iters"] or a["nA"] <= 1, (k, a, b)
        assert abs(a["F_after"] - b["F_after"]) <= 1e-9 * abs(a["F_after"]), (k, a, b)


@pytest.mark.parametrize("flags", [16, 24, 32])
def test_heavy_path_bitwise_reproducible(flags):
    """Heavy path on (16; with dynamic unit claims 24) or off (32): every heavy row sum has a fixed order (groups of
    lanes per row, a fixed shuffle tree), so two contexts solving cfg4s give identical bits."""
    ds = dataset("cfg4s")
    out = []
    for rep in range(2):
        ctx = ml.Context(ds)
        ctx.ml_set_engine(flags)
        r = ctx.ml_solve()
        out.append((r["F"], ctx.ml_get_w().cpu().numpy(), [(t["nA"], t["inner_iters"], t["F_after"]) for t in ctx.trace()]))
        if flags == 32:
            assert ctx.ml_heavy_info()["relaxations"] == 0
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


def test_heavy_path_not_built_small_m():
    """m <= 8192 (the shared-memory solver) has no heavy path: ml_set_engine bit 4 is rejected."""
    ctx = ml.Context(dataset("cfg2s"))
    assert ctx.ml_heavy_info()["built"] == 0
    with pytest.raises(Exception):
        ctx.ml_set_engine(16)


@pytest.mark.parametrize("fill", [-1, 0x7FF8000000000000])
def test_heavy_path_stale_workspace(fill):
    """The heavy path must not depend on the workspace's previous contents either: with every word of the workspace
    set to all-ones (or a NaN pattern) before ml_create, the forced heavy-path solve of cfg4s matches the oracle (the
    copies' padding entries past a chunk hold stale indices; their products are discarded)."""
    ds = dataset("cfg4s")
    r_o = oracle.Oracle(ds).solve()
    ctx = ml.Context(ds, ws_fill=fill)
    ctx.ml_set_engine(16)
    r_g = ctx.ml_solve()
    assert ctx.ml_heavy_info()["relaxations"] > 0
    assert r_g["status"] == 0 and r_g["kappa"] <= 1e-6
    assert abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"])
