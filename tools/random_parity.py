"""Randomised solve parity: many small random designs (shapes, densities, lambda factors, solver options), GPU solve
vs oracle solve: both converged, F within 1e-6 relative.  One JSON line per case and a summary line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import mlgen  # noqa: E402
import oracle  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=40)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--big", action="store_true", help="large-m designs only (m > 8192)")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    opts_pool = [{}, {"inner_cg": 1, "pcd_snap": 0}, {"inner_cg": 0}, {"multilevel": 0}, {"continuation": 1}]
    fails = 0
    for k in range(a.cases):
        m = int(rng.choice([9000, 20000, 40000] if a.big else [37, 200, 777, 2000, 5000, 9000, 12000]))
        n = int(rng.choice([500, 5000, 30000] if a.big else [13, 150, 1301, 4000, 9000]))
        dens = float(rng.choice([0.001, 0.005, 0.02] if a.big else [0.005, 0.02, 0.1, 0.5]))
        base = mlgen.random_sparse(m, n, dens, seed=int(rng.integers(1 << 30)), lam_factor=float(rng.choice([0.05, 0.1, 0.3])),
                                   empty_rows=int(rng.integers(0, min(5, m // 2) + 1)), empty_cols=int(rng.integers(0, min(20, n // 2) + 1)))
        ds = mlgen.lasso(base, int(rng.integers(1 << 30)), k=5) if rng.random() < 0.25 else base
        opts = opts_pool[int(rng.integers(len(opts_pool)))]
        if opts.get("inner_cg") == 0:
            opts = {**opts, "max_cycles": 3000}
        r_o = oracle.Oracle(ds).solve(oracle.default_opts(**opts))
        r_g = ml.Context(ds).ml_solve(ml.default_opts(**opts))
        ok = (r_o["status"] == r_g["status"] == 0 and r_g["kappa"] <= 1e-6
              and abs(r_g["F"] - r_o["F"]) <= 1e-6 * abs(r_o["F"]))
        fails += not ok
        print(json.dumps({"case": k, "m": m, "n": n, "density": dens, "lasso": ds.b is not None, "opts": opts,
                          "status": [r_o["status"], r_g["status"]], "F_rel": abs(r_g["F"] - r_o["F"]) / max(abs(r_o["F"]), 1e-300),
                          "kappa_gpu": r_g["kappa"], "cycles": [r_o["cycles"], r_g["cycles"]], "ok": ok}))
    print(json.dumps({"cases": a.cases, "failures": fails}))


if __name__ == "__main__":
    main()
