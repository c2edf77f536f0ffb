"""Replays one case of tools/random_parity.py (same seeds) and compares the GPU solution with the oracle's, evaluating
the GPU iterate with the oracle as well."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import oracle  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def case(idx, seed=7):
    """The dataset and options of case `idx` of tools/random_parity.py --seed `seed`."""
    rng = np.random.default_rng(seed)
    opts_pool = [{}, {"inner_cg": 1, "pcd_snap": 0}, {"inner_cg": 0}, {"multilevel": 0}, {"continuation": 1}]
    opts = {}
    for k in range(idx + 1):
        m = int(rng.choice([37, 200, 777, 2000, 5000, 9000, 12000]))
        n = int(rng.choice([13, 150, 1301, 4000, 9000]))
        dens = float(rng.choice([0.005, 0.02, 0.1, 0.5]))
        base = mlgen.random_sparse(m, n, dens, seed=int(rng.integers(1 << 30)), lam_factor=float(rng.choice([0.05, 0.1, 0.3])),
                                   empty_rows=int(rng.integers(0, min(5, m // 2) + 1)), empty_cols=int(rng.integers(0, min(20, n // 2) + 1)))
        ds = mlgen.lasso(base, int(rng.integers(1 << 30)), k=5) if rng.random() < 0.25 else base
        opts = opts_pool[int(rng.integers(len(opts_pool)))]
        if opts.get("inner_cg") == 0:
            opts = {**opts, "max_cycles": 3000}
    return ds, opts


if __name__ == "__main__":
    ds, opts = case(int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    print(json.dumps({"m": ds.m, "n": ds.n, "nnz": ds.nnz, "lasso": ds.b is not None, "opts": opts}), flush=True)
    o = oracle.Oracle(ds)
    r_o = o.solve(oracle.default_opts(**opts))
    ctx = ml.Context(ds)
    r_g = ctx.ml_solve(ml.default_opts(**opts))
    w_g = ctx.ml_get_w().cpu().numpy()
    o2 = oracle.Oracle(ds)
    o2.set_w(w_g)
    F2, g2, _ = o2.eval_f_grad()
    tg = ctx.trace()
    to = o.trace()
    print(json.dumps({"opts": opts, "F_oracle": r_o["F"], "F_gpu": r_g["F"], "F_of_gpu_w_by_oracle": F2,
                      "kappa_gpu": r_g["kappa"], "cycles": [r_o["cycles"], r_g["cycles"]], "nnz_w": [r_o["nnz_w"], r_g["nnz_w"]],
                      "max_abs_w_diff": float(np.abs(w_g - o.get_w()).max())}))
    for k in range(min(len(to), len(tg), 40)):
        a, b = to[k], tg[k]
        print(k, (a["level"], a["nA"], a["outcome"], a["inner_iters"], round(a["F_after"], 9)), (b["level"], b["nA"], b["outcome"], b["inner_iters"], round(b["F_after"], 9)))
