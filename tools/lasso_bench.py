"""Squared-loss (LASSO, DESIGN Q29) solves on the designs of BASELINE configs: ms per solve (CUDA events, median of
--reps after one warm solve), cycles, X GB/s (8 B x nonzeros streamed / time).  --oracle also times one oracle solve."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mlgen  # noqa: E402
import paper_1607_00315_b200 as ml  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--lam-factor", type=float, default=0.05)
    ap.add_argument("--oracle", action="store_true")
    a = ap.parse_args()
    base = mlgen.make(a.config)
    ds = mlgen.lasso(base, 7, k=max(20, base.n // 200), noise=0.1, lam_factor=a.lam_factor)
    ctx = ml.Context(ds)
    ctx.ml_solve()
    ts, rep = [], None
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        rep = ctx.ml_solve()
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    out = {"workload": ds.name, "m": ds.m, "n": ds.n, "nnz": ds.nnz, "lambda": ds.lam, "ms": round(ms, 3),
           "cycles": rep["cycles"], "relaxations": rep["relaxations"], "kappa": rep["kappa"], "nnz_w": rep["nnz_w"],
           "F": rep["F"], "x_gbs": round(8.0 * rep["nnz_touched"] / (ms * 1e-3) / 1e9, 1)}
    if a.oracle:
        import oracle
        o = oracle.Oracle(ds)
        t0 = time.perf_counter()
        r_o = o.solve()
        out["oracle_s"] = round(time.perf_counter() - t0, 3)
        out["oracle_F"] = r_o["F"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
