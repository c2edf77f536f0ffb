"""Randomised parity of the API passes (ml_eval_f_grad, ml_diag_hess, ml_hessvec on a random column list) against
the oracle on random designs, including ones whose last nonzeros are past X's last 16-byte boundary."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import oracle  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=30)
    ap.add_argument("--seed", type=int, default=5)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    fails = 0
    for k in range(a.cases):
        m = int(rng.choice([37, 300, 2000, 9000, 12000]))
        n = int(rng.choice([13, 150, 1301, 4000]))
        base = mlgen.random_sparse(m, n, float(rng.choice([0.005, 0.05, 0.3])), seed=int(rng.integers(1 << 30)),
                                   empty_rows=int(rng.integers(0, min(5, m // 2) + 1)),
                                   empty_cols=int(rng.integers(0, min(20, n // 2) + 1)))
        ds = mlgen.lasso(base, int(rng.integers(1 << 30)), k=5) if rng.random() < 0.3 else base
        w = np.zeros(ds.n)
        idx = rng.choice(ds.n, max(1, ds.n // 7), replace=False)
        w[idx] = rng.normal(0, 0.3, len(idx))
        o = oracle.Oracle(ds)
        o.set_w(w)
        ctx = ml.Context(ds)
        ctx.ml_set_w(torch.from_numpy(w).cuda())
        F_o, g_o, h_o = o.eval_f_grad()
        F_g, g_g, h_g = ctx.ml_eval_f_grad()
        C = np.sort(rng.choice(ds.n, max(1, ds.n // 3), replace=False)).astype(np.int32)
        v = rng.standard_normal(len(C))
        hv_o = o.hessvec(C, v)
        hv_g = ctx.ml_hessvec(torch.from_numpy(C).cuda(), torch.from_numpy(v).cuda()).cpu().numpy()
        dh_o = o.diag_hess(C)
        dh_g = ctx.ml_diag_hess(torch.from_numpy(C).cuda()).cpu().numpy()
        errs = {"F": abs(F_g - F_o) / abs(F_o), "g": rel(g_g.cpu().numpy(), g_o), "h": rel(h_g.cpu().numpy(), h_o),
                "hv": rel(hv_g, hv_o), "dh": rel(dh_g, dh_o)}
        ok = all(e <= 1e-9 for e in errs.values())
        fails += not ok
        print(json.dumps({"case": k, "m": m, "n": n, "nnz": ds.nnz, "nnz_mod4": ds.nnz % 4, "lasso": ds.b is not None,
                          "errs": {kk: float(f"{vv:.2e}") for kk, vv in errs.items()}, "ok": ok}))
    print(json.dumps({"cases": a.cases, "failures": fails}))


if __name__ == "__main__":
    main()
